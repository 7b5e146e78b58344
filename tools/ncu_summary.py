"""Key metrics of ncu --set full captures: python tools/ncu_summary.py rep1.ncu-rep [...]
Prints duration, DRAM bytes/throughput, issue activity, occupancy and the top stall reasons."""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__inst_executed.sum": "warp_inst",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "launch__registers_per_thread": "regs",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "smsp__thread_inst_executed_per_inst_executed.ratio": "active_threads_per_warp",
}


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {"report": rep, "kernel": vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            d[name] = f"{vals[i]} {units[i]}".strip()
    stalls = []
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            try:
                stalls.append((float(vals[i].replace(",", "")), h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]))
            except ValueError:
                pass
    stalls.sort(reverse=True)
    d["top_stalls"] = [f"{n}={v:.2f}" for v, n in stalls[:5]]
    return d


if __name__ == "__main__":
    for r in sys.argv[1:]:
        print(json.dumps(summarize(r), indent=1))

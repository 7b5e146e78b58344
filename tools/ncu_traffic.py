"""profiles/ncu_traffic.json from an ncu_summary.py output (concatenated JSON
objects): per-kernel DRAM bytes (read + write) and duration of one launch, and
the per-stage totals bench.py reads as `traffic`.
  python tools/ncu_traffic.py profiles/rNN_ncu_full_summary.json "note" > profiles/ncu_traffic.json"""
import json
import re
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
TUNIT = {"ns": 1e-3, "us": 1.0, "ms": 1e3}


def num(s, table):
    v, u = s.split()
    return float(v) * table[u]


def objects(text):
    dec, i = json.JSONDecoder(), 0
    while True:
        m = re.compile(r"\S").search(text, i)
        if not m:
            return
        o, i = dec.raw_decode(text, m.start())
        yield o


def main():
    src, note = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    detail = {}
    for o in objects(open(src).read()):
        name = o["kernel"].split("(")[0]
        if "/fused/" in o["report"]:
            name = "fused/" + name
        b = num(o["dram_read"], UNIT) + num(o["dram_write"], UNIT)
        us = num(o["duration"], TUNIT)
        detail[name] = {"dram_bytes": b, "duration_us": round(us, 2), "dram_GBps": round(b / us / 1e3, 1)}

    def get(*keys):
        return sum(detail[k]["dram_bytes"] for k in keys if k in detail) or None

    out = {
        "ssr_forward": get("void k_forward<1, 0>"),
        "ssr_backward": get("k_backward_splat2"),
        "ssr_adam": get("void k_adam<16>"),
        "ssr_chain_sh": get("void k_chain_sh<3>"),
        "ssr_chain_geo": get("void k_chain_geo<0>"),
        "ssr_chain_sh_fused": get("fused/void k_chain_sh_adam<3>"),
        "ssr_chain_geo_fused": get("fused/void k_chain_geo<1>"),
        "ssr_preprocess": get("void k_preprocess<3, 1>"),
        "ssr_loss_fwd": get("void k_ssim_fwd<0>"),
        "ssr_loss_bwd": get("void k_ssim_bwd<0>"),
        "ssr_bin_tiles_radix_down": get("void k_radix_down<0>"),
        "ssr_bin_tiles_duplicate": get("k_duplicate"),
        "note": note,
        "detail": detail,
    }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()

"""ctypes binding of the sm_100a extension ``libssr.so`` (C ABI in include/ssr.h).

The library is built in-tree (``make -C paper_2503_13086_b200/csrc`` or
``__graft_entry__.build()``).  There is no fallback: if the library is missing
or no CUDA device is present, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os

import torch

from .errors import ExtensionMissing, InvalidParameter, NativeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SSR_LIB") or os.path.join(_HERE, "libssr.so")

c_void_p, c_int32, c_int64, c_double, c_float = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                                                  ctypes.c_double, ctypes.c_float)


class SsrCamera(ctypes.Structure):
    _fields_ = [("R", c_double * 9), ("t", c_double * 3), ("fx", c_double), ("fy", c_double),
                ("cx", c_double), ("cy", c_double), ("center", c_double * 3), ("width", c_int32),
                ("height", c_int32)]


class SsrSplats(ctypes.Structure):
    _fields_ = [(k, c_void_p) for k in ("mean", "conic_opa", "color", "conic_opa64", "color64", "depth",
                                        "rect", "tiles", "offset", "row_offset", "depth_order")]


class SsrFrame(ctypes.Structure):
    _fields_ = [("width", c_int32), ("height", c_int32), ("tiles_x", c_int32), ("tiles_y", c_int32),
                ("bg", c_float * 3)] + [(k, c_void_p) for k in (
                    "image", "t_final", "n_walk", "terminated", "hard_count", "soft_count", "flagged",
                    "tile_info", "ckpt", "fix_list")]


# name -> argtypes (restype int unless listed in _RESTYPES)
_SIGS = {
    "ssr_version": [],
    "ssr_last_error": [],
    "ssr_device_info": [c_void_p, c_void_p, c_void_p],
    "ssr_preprocess": [ctypes.POINTER(SsrCamera), c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                       c_void_p, SsrSplats, c_void_p],
    "ssr_project_aux": [ctypes.POINTER(SsrCamera), c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                        c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p,
                        c_void_p, c_void_p, c_void_p],
    "ssr_scan_workspace": [c_int64, ctypes.POINTER(c_int64)],
    "ssr_scan_tiles": [c_int64, SsrSplats, c_void_p, c_int64, c_void_p, c_void_p],
    "ssr_bin_workspace": [c_int64, c_int32, ctypes.POINTER(c_int64)],
    "ssr_bin_tiles": [c_int64, c_int64, c_int32, c_int32, SsrSplats, c_void_p, c_void_p, c_void_p, c_int64,
                      c_void_p],
    "ssr_bin_tiles_capacity": [c_int64, c_int64, c_int32, c_int32, SsrSplats, c_void_p, ctypes.POINTER(c_int64),
                               c_void_p, c_void_p, c_void_p, c_int64, c_void_p],
    "ssr_ckpt_floats": [c_int64, c_int32],
    "ssr_rows_floats": [c_int64],
    "ssr_fix_list_ints": [c_int32, c_int32, c_int32],
    "ssr_forward": [c_int64, SsrSplats, c_void_p, c_void_p, SsrFrame, c_float, c_float, c_void_p],
    "ssr_backward": [c_int32, c_int64, SsrSplats, c_void_p, c_void_p, SsrFrame, c_void_p, c_void_p, c_void_p,
                     c_void_p],
    "ssr_chain": [ctypes.POINTER(SsrCamera), c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                  SsrSplats, c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_void_p],
    "ssr_chain_adam": [ctypes.POINTER(SsrCamera), c_int64, c_int32, c_void_p, c_void_p, c_void_p, SsrSplats,
                       c_void_p, c_void_p, ctypes.POINTER(c_double), c_double, ctypes.POINTER(c_double),
                       ctypes.POINTER(c_double), c_void_p],
    "ssr_exchange_adam": [c_int64, c_int32, c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                          ctypes.POINTER(c_double), c_double, ctypes.POINTER(c_double), ctypes.POINTER(c_double),
                          c_void_p],
    "ssr_exchange_chunk": [c_int64, c_int32, c_int32, ctypes.POINTER(c_int64), ctypes.POINTER(c_int64)],
    "ssr_ipc_export": [c_void_p, c_void_p, ctypes.POINTER(c_int64)],
    "ssr_ipc_open": [c_void_p, c_int64, ctypes.POINTER(c_void_p)],
    "ssr_ipc_close": [c_void_p],
    "ssr_adam": [c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, ctypes.POINTER(c_double), c_double,
                 ctypes.POINTER(c_double), ctypes.POINTER(c_double), c_void_p],
    "ssr_adam_range": [c_int64, c_int32, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, c_int64, c_int64,
                       ctypes.POINTER(c_double), c_double, ctypes.POINTER(c_double), ctypes.POINTER(c_double),
                       c_void_p],
    "ssr_densify_masks": [c_int64, c_void_p, c_int32, c_void_p, c_double, c_double, c_double, c_void_p,
                          c_void_p, c_void_p],
    "ssr_densify_workspace": [c_int64, ctypes.POINTER(c_int64)],
    "ssr_densify_apply": [c_int64, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_double,
                          c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p],
    "ssr_knn_workspace": [c_int64, c_int64, ctypes.POINTER(c_int64)],
    "ssr_knn": [c_void_p, c_int64, c_void_p, c_int64, c_int32, ctypes.POINTER(c_double),
                ctypes.POINTER(c_int32), c_void_p, c_void_p, c_int64, c_void_p],
    "ssr_ply_properties": [c_int32],
    "ssr_ply_pack": [c_int64, c_int32, c_void_p, c_void_p, c_void_p],
    "ssr_ply_unpack": [c_int64, c_int32, c_void_p, c_void_p, c_void_p],
    "ssr_loss_workspace": [c_int32, c_int32, ctypes.POINTER(c_int64)],
    "ssr_loss": [c_int32, c_int32, c_void_p, c_void_p, c_int32, c_void_p, c_void_p, c_double, c_double, c_double,
                 c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p],
}
_RESTYPES = {"ssr_last_error": ctypes.c_char_p, "ssr_ckpt_floats": c_int64, "ssr_rows_floats": c_int64, "ssr_fix_list_ints": c_int64,
             "ssr_ply_properties": c_int32}

EXPORTS = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load and type the extension; raises ExtensionMissing when absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ExtensionMissing(
            f"{path} is not built; run `make -C {os.path.join(_HERE, 'csrc')}` or __graft_entry__.build()")
    try:
        lib = ctypes.CDLL(path)
    except OSError as e:  # pragma: no cover - depends on the box
        raise ExtensionMissing(f"cannot load {path}: {e}") from e
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPES.get(name, c_int32)
    _lib = lib
    return lib


_timers = None  # name -> [(start_event, end_event)] when enabled (bench.py)


def enable_timers(on: bool = True) -> None:
    """Bracket every ABI call with CUDA events on the launching stream."""
    global _timers
    _timers = {} if on else None


def timer_ms() -> dict:
    """Mean device milliseconds per ABI function since enable_timers()."""
    if not _timers:
        return {}
    torch.cuda.synchronize()
    return {k: sum(a.elapsed_time(b) for a, b in v) / len(v) for k, v in _timers.items()}


def raise_last(name: str, rc: int) -> None:
    """Raise the Python error of a failed entry point's return code."""
    msg = (load().ssr_last_error() or b"").decode(errors="replace")
    if rc in (1, 3):
        raise InvalidParameter(f"{name}: {msg}")
    raise NativeError(f"{name} failed ({rc}): {msg}")


def call_rc(name: str, *args) -> int:
    """Call an entry point (timed when timers are on) and return its code."""
    if _timers is not None:
        ev0 = torch.cuda.Event(enable_timing=True)
        ev0.record()
    rc = getattr(load(), name)(*args)
    if _timers is not None:
        ev1 = torch.cuda.Event(enable_timing=True)
        ev1.record()
        _timers.setdefault(name, []).append((ev0, ev1))
    return rc


def call(name: str, *args) -> None:
    rc = call_rc(name, *args)
    if rc != 0:
        raise_last(name, rc)


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise ExtensionMissing("no CUDA device: the sm_100a extension has no CPU fallback")
    load()
    return torch.device("cuda", torch.cuda.current_device())


def stream_ptr() -> int:
    return torch.cuda.current_stream().cuda_stream


def ptr(t) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise InvalidParameter("expected a CUDA tensor")
    return t.data_ptr()


def camera_struct(cam) -> SsrCamera:
    c = SsrCamera()
    R = cam.rotation.reshape(9)
    for i in range(9):
        c.R[i] = float(R[i])
    for i in range(3):
        c.t[i] = float(cam.translation[i])
        c.center[i] = float(cam.center[i])
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    c.width, c.height = int(cam.width), int(cam.height)
    return c


def query(name: str, *args) -> int:
    out = c_int64(0)
    call(name, *args, ctypes.byref(out))
    return int(out.value)

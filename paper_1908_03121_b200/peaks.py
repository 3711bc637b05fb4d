"""Measured FP64 roofline denominator (bench evidence).

MEASURED_PEAKS.json has HBM and bf16 but no FP64 figure; the same-level
kernels are FP64-pipe bound, so this measures the DFMA throughput of the
device with csrc/fp64_peak.cu (8 independent DFMA chains per thread, 148 x 8
CTAs x 256 threads), timed with CUDA events on the launching stream.
"""
from __future__ import annotations

import ctypes as C

from . import build as _build

_peak = None


def _lib():
    global _peak
    if _peak is None:
        _peak = C.CDLL(_build.build_peak())
        _peak.octo_fp64_peak_launch.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        _peak.octo_fp64_peak_launch.restype = C.c_double
    return _peak


def measure_fp64_peak(reps: int = 20, iters: int = 2048, seconds: float = 0.0) -> dict:
    """Best-of-reps burst DFMA rate (TFLOP/s, FMA = 2 flop).  With seconds > 0
    also a sustained figure: back-to-back launches for that long."""
    import torch
    st = torch.cuda.current_stream()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    blocks = sms * 8
    lib = _lib()
    lib.octo_fp64_peak_launch(st.cuda_stream, blocks, 64, 2)   # warm-up
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        fl = lib.octo_fp64_peak_launch(st.cuda_stream, blocks, iters, 1)
        b.record(st)
        b.synchronize()
        best = max(best, fl / (a.elapsed_time(b) * 1e-3) / 1e12)
    out = {"fp64_tflops_burst": best, "sms": sms}
    if seconds > 0:
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        n = max(1, int(seconds / (fl / (best * 1e12))))
        a.record(st)
        fl = lib.octo_fp64_peak_launch(st.cuda_stream, blocks, iters, n)
        b.record(st)
        b.synchronize()
        out["fp64_tflops_sustained"] = fl * n / (a.elapsed_time(b) * 1e-3) / 1e12
    return out

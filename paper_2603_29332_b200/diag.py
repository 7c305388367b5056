"""Diagnostics over the C ABI (roofline denominators)."""
import ctypes as C

from . import MskError, lib


def fp32_peak_tflops(device=0):
    """Measured FFMA throughput (TFLOP/s) of `device` — the binding roofline of the step kernel."""
    L = lib()
    L.msk_gpu_fp32_peak_probe.argtypes = [C.c_int, C.POINTER(C.c_double)]
    L.msk_gpu_fp32_peak_probe.restype = C.c_int
    v = C.c_double(0)
    rc = L.msk_gpu_fp32_peak_probe(int(device), C.byref(v))
    if rc:
        raise MskError(rc, L.msk_gpu_last_error(None).decode())
    return float(v.value)

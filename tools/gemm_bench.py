#!/usr/bin/env python3
"""Per-layer time of the tcgen05 GEMM (tanh epilogue) vs K: the intercept is the
per-layer fixed cost (fill, epilogue, launch), the slope the mainloop rate.

  python tools/gemm_bench.py [M] [N]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import paper_2603_29332_b200 as pk

    M = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    N = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
    L = pk.lib()
    L.msk_gemm_bench.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_double)]
    for K in (64, 256, 512, 1024, 2048, 4096):
        ms = C.c_double()
        assert L.msk_gemm_bench(M, K, N, 200, C.byref(ms)) == 0
        us = ms.value * 1e3
        print(f"M={M} N={N} K={K:5d}: {us:7.2f} us per layer, {2 * M * N * K / (us * 1e-6) / 1e12:7.1f} TFLOP/s")


if __name__ == "__main__":
    main()

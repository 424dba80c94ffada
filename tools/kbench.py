"""Kernel microbenchmarks through pcb_debug_kernel_bench (device-timed, back-to-back launches)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2311_04934_b200 as pcb

L = pcb.lib()
L.pcb_debug_kernel_bench.argtypes = [C.c_char_p, C.c_int64, C.c_int64, C.c_int64, C.c_int, C.POINTER(C.c_double)]


def bench(which, a0, a1, a2, iters=50):
    us = C.c_double()
    rc = L.pcb_debug_kernel_bench(which.encode(), a0, a1, a2, iters, C.byref(us))
    if rc:
        raise RuntimeError(L.pcb_last_error().decode())
    return us.value


if __name__ == "__main__":
    for M, N, K, nm in [(64, 12288, 4096, "qkv"), (64, 4096, 4096, "o"), (64, 16384, 4096, "w1"),
                        (64, 4096, 16384, "w2"), (1, 32000, 4096, "unembed"), (128, 12288, 4096, "qkv128"),
                        (256, 12288, 4096, "qkv256"), (512, 12288, 4096, "qkv512"), (512, 16384, 4096, "w1_512"),
                        (512, 4096, 16384, "w2_512"),
                        (4160, 12288, 4096, "qkv_prefill"), (4160, 16384, 4096, "w1_prefill"),
                        (4160, 4096, 16384, "w2_prefill")]:
        us = bench("gemm", M, N, K)
        gb = (N * K * 2 + M * K * 2 + M * N * 8) / 1e9
        tf = 2 * M * N * K / 1e12
        print(f"gemm {nm:12s} M={M:5d} N={N:5d} K={K:5d}: {us:8.1f} us  {gb / us * 1e6:7.0f} GB/s  "
              f"{tf / us * 1e6:7.1f} TFLOP/s")
    for n, P in [(64, 4096), (128, 16384), (4160, 0), (1, 4096)]:
        us = bench("attn", n, P, 32)
        gb = 2 * (n + P) * 4096 * 2 / 1e9
        print(f"attn n={n} P={P}: {us:8.1f} us  {gb / us * 1e6:7.0f} GB/s (KV read)")

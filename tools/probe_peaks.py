"""Probe FP64 / TF32 library peaks (cuBLAS via torch) on the B200 box.

Roofline denominators for the FP64 mode (DGEMM) and the TF32 fast mode.
Prints one JSON line. Run under gpurun; never a bench number.
"""
import json
import torch


def bench(fn, reps=10):
    fn(); torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def main():
    out = {}
    N = 8192
    a = torch.randn(N, N, dtype=torch.float64, device="cuda")
    b = torch.randn(N, N, dtype=torch.float64, device="cuda")
    ms = bench(lambda: a @ b, reps=5)
    out["cublas_dgemm_tflops"] = 2 * N**3 / ms / 1e9
    a32 = a.float(); b32 = b.float()
    torch.backends.cuda.matmul.allow_tf32 = True
    ms = bench(lambda: a32 @ b32)
    out["cublas_tf32_tflops"] = 2 * N**3 / ms / 1e9
    torch.backends.cuda.matmul.allow_tf32 = False
    ms = bench(lambda: a32 @ b32)
    out["cublas_sgemm_tflops"] = 2 * N**3 / ms / 1e9
    print(json.dumps(out))


if __name__ == "__main__":
    main()

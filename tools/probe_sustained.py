"""Sustained (power-capped) library peaks: cuBLAS DGEMM and TF32 8192^3 back to back for ~5 s,
the last ~2 s timed with CUDA events, SM clocks sampled by nvidia-smi meanwhile.  The roofline
denominator the bench uses beside the burst peaks for kernels timed inside long steps (c3-c5).
Prints one JSON line.  Run under gpurun; never a bench number.
"""
import json
import subprocess
import time

import torch


def sustained(fn, flops, seconds=5.0, tail=2.0):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < seconds - tail:
        for _ in range(4):
            fn()
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 0
    e0.record()
    t1 = time.perf_counter()
    while time.perf_counter() - t1 < tail:
        for _ in range(4):
            fn()
        n += 4
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return flops * n / (e0.elapsed_time(e1) * 1e-3) / 1e12


def main():
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "200"], stdout=subprocess.PIPE, text=True)
    N = 8192
    a = torch.randn(N, N, dtype=torch.float64, device="cuda")
    b = torch.randn(N, N, dtype=torch.float64, device="cuda")
    out = {"cublas_dgemm_8192_sustained_tflops": sustained(lambda: a @ b, 2 * N**3)}
    a32, b32 = a.float(), b.float()
    torch.backends.cuda.matmul.allow_tf32 = True
    out["cublas_tf32_8192_sustained_tflops"] = sustained(lambda: a32 @ b32, 2 * N**3)
    smi.terminate()
    lines = smi.communicate()[0].strip().splitlines()
    mhz = sorted(float(l.split(",")[0]) for l in lines if l.strip())
    out["sm_mhz_median_during"] = mhz[len(mhz) // 2] if mhz else None
    out["how"] = "back to back 5 s each, last 2 s timed (CUDA events)"
    print(json.dumps(out))


if __name__ == "__main__":
    main()

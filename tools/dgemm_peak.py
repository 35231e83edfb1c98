"""cuBLAS DGEMM reference peak (roofline context only; never on the product path).

Same method as MEASURED_PEAKS.json's bf16 entry: torch.matmul fp64 8192^3, best of 10 (burst)
and back to back for 4 s (sustained), CUDA events.
"""
import json
import time

import torch


def main():
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    c = torch.empty_like(a)
    flop = 2.0 * n ** 3
    for _ in range(3):
        torch.matmul(a, b, out=c)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b, out=c)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    count = 0
    t0 = time.time()
    while time.time() - t0 < 4.0:
        torch.matmul(a, b, out=c)
        count += 1
        if count % 4 == 0:
            torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    sus = flop * count / (e0.elapsed_time(e1) * 1e-3) / 1e12
    print(json.dumps({"cublas_dgemm_8192_burst_tflops": flop / (best * 1e-3) / 1e12,
                      "cublas_dgemm_8192_sustained_tflops": sus}))


if __name__ == "__main__":
    main()

"""Measure cuBLAS FP64 GEMM throughput (torch.matmul float64) as the FP64 roofline denominator."""
import json
import torch

def main():
    dev = torch.device("cuda:0")
    out = {}
    for n in (4096, 8192):
        a = torch.randn(n, n, dtype=torch.float64, device=dev)
        b = torch.randn(n, n, dtype=torch.float64, device=dev)
        for _ in range(3):
            torch.matmul(a, b)
        torch.cuda.synchronize()
        best = 1e9
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        out[f"dgemm_{n}_tflops"] = 2 * n**3 / (best * 1e-3) / 1e12
    # copy bandwidth (fp64)
    x = torch.empty(1 << 27, dtype=torch.float64, device=dev); y = torch.empty_like(x)
    for _ in range(3): y.copy_(x)
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(10):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); y.copy_(x); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out["copy_gbs"] = 2 * x.numel() * 8 / (best * 1e-3) / 1e9
    print(json.dumps(out))

if __name__ == "__main__":
    main()

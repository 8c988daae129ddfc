"""cuBLAS DGEMM throughput on this B200 (reference point for the DMMA kernels)."""
import torch

def bench(m, n, k, batch=1, reps=20):
    a = torch.randn(batch, m, k, dtype=torch.float64, device="cuda")
    b = torch.randn(batch, k, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.bmm(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        torch.bmm(a, b)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"bmm {batch}x[{m}x{k}]@[{k}x{n}]: {2.0*batch*m*n*k/ms/1e9:.2f} TFLOP/s ({ms*1e3:.1f} us)")

bench(8192, 8192, 8192, reps=5)
bench(4096, 4096, 4096)
bench(64, 1024, 128, batch=256)   # Legendre-forward-like: per (m, parity)
bench(128, 1024, 64, batch=256)   # Legendre-inverse-like
bench(128, 512, 256, batch=128)   # radial-like

"""cuBLAS DGEMM throughput (the fp64 library roofline used for the dense stages)."""
import torch
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        a @ b
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"DGEMM {n}^3: {2 * n**3 / (ms * 1e-3) / 1e12:.2f} TFLOP/s")
# tall-skinny Gram like the final eig_svd (1M x 200)
w = torch.randn(1_000_000, 200, dtype=torch.float64, device="cuda")
for _ in range(2):
    w.T @ w
torch.cuda.synchronize()
e0.record()
for _ in range(5):
    w.T @ w
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"cuBLAS W^T W 1M x 200: {ms:.3f} ms, {2 * 1e6 * 200 * 200 / (ms * 1e-3) / 1e12:.2f} TFLOP/s")

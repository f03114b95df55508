"""Measured FP64 GEMM peak on this B200 (BASELINE.md asks for one): cuBLAS
DGEMM through torch (float64 matmul, n = 8192, CUDA events, warm), the
denominator for the FP64 tensor-pipe fractions of the engine's own DMMA
kernels (k_dgemm, k_type_gemm, k_h_gemm, k_dual_root, k_mf_factor)."""
import json
import torch

n = 8192
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
reps = 10
for _ in range(reps):
    c = a @ b
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
tf = 2.0 * n ** 3 / (ms * 1e-3) / 1e12
print(json.dumps({"what": "cuBLAS DGEMM (torch float64 matmul) n=8192, warm, CUDA events", "ms": ms,
                  "tflops_fp64": tf}))

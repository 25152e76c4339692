"""ncu tensor-pipe calibration target: a cuBLAS bf16 8192^3 GEMM (the MEASURED_PEAKS.json kernel),
run a few times so ncu can capture it next to our conv kernels with the same metric list."""
import torch

n = 8192
a = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
b = torch.randn(n, n, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
print("gemm flops per launch", 2 * n ** 3)

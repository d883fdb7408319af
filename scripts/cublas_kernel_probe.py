"""One cuBLAS launch of the UPDATE / GRAM shapes (for an ncu look at its tile / cluster config)."""
import torch
bt, m, n = 8, 4096, 12288
x = torch.randn(bt, m, n, device="cuda").mul_(0.01).bfloat16()
a = torch.randn(bt, m, m, device="cuda").mul_(0.01).bfloat16()
for _ in range(2):
    torch.matmul(a, x)
    torch.matmul(x, x.transpose(1, 2))
torch.cuda.synchronize()

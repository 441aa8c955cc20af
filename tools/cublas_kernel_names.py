import torch
w = torch.randn(2048, 16384, device="cuda", dtype=torch.bfloat16)
x = torch.randn(800, 16384, device="cuda", dtype=torch.bfloat16)
for _ in range(3): y = x @ w.T
w2 = torch.randn(32768, 2048, device="cuda", dtype=torch.bfloat16)
x2 = torch.randn(800, 2048, device="cuda", dtype=torch.bfloat16)
for _ in range(3): y = x2 @ w2.T
torch.cuda.synchronize()

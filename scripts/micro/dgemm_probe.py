import torch
a=torch.randn(8192,8192,dtype=torch.float64,device='cuda'); b=torch.randn_like(a)
for _ in range(3): c=a@b
torch.cuda.synchronize()

import torch
a=torch.randn(8192,4096,device="cuda",dtype=torch.bfloat16); b=torch.randn(28672,4096,device="cuda",dtype=torch.bfloat16)
c=torch.randn(8192,14336,device="cuda",dtype=torch.bfloat16); w2=torch.randn(4096,14336,device="cuda",dtype=torch.bfloat16)
torch.cuda.synchronize()
for _ in range(2): x = a@b.T; y = c@w2.T
torch.cuda.synchronize()

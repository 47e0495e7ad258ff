import sys
sys.path.insert(0, ".")
import torch
import paper_2604_02525_b200 as ah
x = (torch.randn(16384, 2048, device="cuda") * 0.1).to(torch.bfloat16)
for _ in range(3):
    ah.debug_foid(x, k=64)
torch.cuda.synchronize()

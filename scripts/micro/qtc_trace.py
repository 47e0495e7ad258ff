import os, sys
sys.path.insert(0, ".")
import torch
import paper_2604_02525_b200 as ah
t = (torch.randn(16384, 8192, device="cuda") * 0.1).to(torch.bfloat16)
for _ in range(2):
    ah.debug_iht_quant(t)
torch.cuda.synchronize()
print("=== dual", flush=True)
ah.debug_quant_dual(t)
torch.cuda.synchronize()

import sys
sys.path.insert(0, ".")
import torch
import paper_2604_02525_b200 as ah
R, C = 16384, 2048
t = (torch.randn(R, C, device="cuda") * 0.1).to(torch.bfloat16)
g = torch.Generator().manual_seed(0)
cz = sorted(torch.randperm(C, generator=g)[:64].tolist())
ah.debug_quant_dual(t, col_zero=cz, want_slices=True)
torch.cuda.synchronize()
print("=== run", flush=True)
ah.debug_quant_dual(t, col_zero=cz, want_slices=True)
torch.cuda.synchronize()

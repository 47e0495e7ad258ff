import sys
sys.path.insert(0, ".")
import torch
import paper_2604_02525_b200 as ah
R, C = 16384, 2048
t = (torch.randn(R, C, device="cuda") * 0.1).to(torch.bfloat16)
g = torch.Generator().manual_seed(0)
cz = sorted(torch.randperm(C, generator=g)[:64].tolist())
cz1 = [5]
for masks, sl in (((None, cz), False), ((None, cz), True), ((None, cz1), False), ((None, list(range(64))), False)):
    for _ in range(3):
        ah.debug_quant_dual(t, row_zero=masks[0], col_zero=masks[1], want_slices=sl)
torch.cuda.synchronize()

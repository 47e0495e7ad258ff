import sys
sys.path.insert(0, ".")
import torch
import paper_2604_02525_b200 as ah
for R, C in ((16384, 2048), (512, 2048), (16384, 512)):
    t = (torch.randn(R, C, device="cuda") * 0.1).to(torch.bfloat16)
    g = torch.Generator().manual_seed(0)
    rz = sorted(torch.randperm(R, generator=g)[:64].tolist())
    cz = sorted(torch.randperm(C, generator=g)[:64].tolist())
    for masks in ((None, None), (rz, None), (None, cz), (rz, cz)):
        for _ in range(3):
            ah.debug_quant_dual(t, row_zero=masks[0], col_zero=masks[1], want_slices=True)
    torch.cuda.synchronize()

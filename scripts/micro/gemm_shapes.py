import sys
sys.path.insert(0, ".")
import torch
import paper_2604_02525_b200 as ah
for M, N, K in ((16384, 8192, 2048), (16384, 2048, 8192), (16384, 2048, 2048)):
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device="cuda", generator=g)
    b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device="cuda", generator=g)
    sa = torch.full((M, K // 32), 120, dtype=torch.uint8, device="cuda")
    sb = torch.full((N, K // 32), 120, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ah.debug_gemm_mxf4(a, sa, b, sb, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()

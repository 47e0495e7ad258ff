"""Tile timeline of CTA 0 of the MXFP4 GEMM (build with --define GEMM_TRACE=1 and select the
library with ADAHOP_LIB). Usage: python scripts/micro/gemm_trace.py M N K"""
import sys
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2604_02525_b200 as ah  # noqa: E402
M, N, K = (int(v) for v in sys.argv[1:4]) if len(sys.argv) > 3 else (16384, 8192, 2048)
g = torch.Generator(device="cuda").manual_seed(0)
a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device="cuda", generator=g)
b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device="cuda", generator=g)
sa = torch.full((M, K // 32), 120, dtype=torch.uint8, device="cuda")
sb = torch.full((N, K // 32), 120, dtype=torch.uint8, device="cuda")
for _ in range(2):
    ah.debug_gemm_mxf4(a, sa, b, sb, out_dtype=torch.bfloat16)
torch.cuda.synchronize()

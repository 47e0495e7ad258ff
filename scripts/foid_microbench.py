"""Time FOID (probe keys + top-k) alone on bench-like operands; run under ncu for per-kernel data."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_02525_b200 as ah  # noqa: E402

dev = torch.device("cuda:0")
for R, K, ks in ((16384, 2048, False), (16384, 2048, True), (2048, 8192, False)):
    x = (torch.randn((K, R) if ks else (R, K), device=dev) * 0.1).to(torch.bfloat16)
    for _ in range(3):
        ah.debug_foid(x, k=64, k_strided=ks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ah.debug_foid(x, k=64, k_strided=ks)
    e1.record()
    torch.cuda.synchronize()
    print(f"foid R={R} K={K} kstrided={ks}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us/call (incl. allocs)")

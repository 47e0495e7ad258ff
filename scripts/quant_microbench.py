"""Time the IHT+quant kernels alone on the bench's operand shapes (run under ncu for per-kernel
durations, or read the CUDA-event numbers printed here). Not part of the product path."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_02525_b200 as ah  # noqa: E402

dev = torch.device("cuda:0")
shapes = [(16384, 2048), (16384, 8192), (2048, 8192), (16384, 512)]
if len(sys.argv) > 1:   # e.g. 16384x8192,16384x2048
    shapes = [tuple(int(v) for v in s.split("x")) for s in sys.argv[1].split(",")]
zr = list(range(0, 4096, 64))
for R, C in shapes:
    t = (torch.randn(R, C, device=dev) * 0.1).to(torch.bfloat16)
    for name, fn in (("row", lambda: ah.debug_iht_quant(t, zero_rows=zr)),
                     ("col", lambda: ah.debug_iht_quant(t, k_strided=True, zero_rows=zr[: min(64, C // 64)])),
                     ("dual", lambda: ah.debug_quant_dual(t, row_zero=zr, col_zero=zr[: min(64, C // 64)]))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        n = 20
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"{name:5s} {R}x{C}: {ms * 1e3:8.1f} us/call (incl. sf convert + allocs)")

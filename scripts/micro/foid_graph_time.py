"""FOID (keys + select) per call on the layer operands, CUDA-graph replayed (no allocation in the
timed region): the column FOID of X [16384 x 2048] (2048 stored rows) and the row FOID of G_Y
[16384 x 512] (16384 stored rows, 4 select blocks + merge)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2604_02525_b200 as ah  # noqa: E402

dev = torch.device("cuda:0")
for R, K, ks in ((2048, 16384, True), (16384, 512, False), (8192, 16384, True)):
    x = (torch.randn((K, R) if ks else (R, K), device=dev) * 0.1).to(torch.bfloat16)
    for _ in range(3):
        ah.debug_foid(x, k=64, k_strided=ks)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        ah.debug_foid(x, k=64, k_strided=ks)
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        for _ in range(20):
            ah.debug_foid(x, k=64, k_strided=ks)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    print(f"foid stored rows {R}, probe of K {K} ({'strided' if ks else 'contiguous'}): "
          f"{e0.elapsed_time(e1) / 20 * 1e3:.1f} us per call (graph)")

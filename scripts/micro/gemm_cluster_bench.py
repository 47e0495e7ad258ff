"""Time the MXFP4 GEMM kernel alone (torch.profiler device times) on the Llama-3.2-1B and
Llama-3-8B layer GEMM shapes, for the cluster shape in ADAHOP_GEMM_CLUSTER."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2604_02525_b200 as ah  # noqa: E402

T = 16384
SHAPES = {
    "1b": [(2048, 2048), (2048, 512), (2048, 8192), (8192, 2048)],
    "8b": [(4096, 4096), (4096, 1024), (4096, 14336), (14336, 4096)],
}
model = sys.argv[1] if len(sys.argv) > 1 else "1b"
gemms = []
for d_in, d_out in SHAPES[model]:
    gemms += [("fwd", T, d_out, d_in), ("dgrad", T, d_in, d_out), ("wgrad", d_out, d_in, T)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
res = []
tot_fl = tot_us = 0.0
for path, M, N, K in gemms:
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device="cuda", generator=g)
    b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device="cuda", generator=g)
    sa = torch.randint(118, 122, (M, K // 32), dtype=torch.uint8, device="cuda", generator=g)
    sb = torch.randint(118, 122, (N, K // 32), dtype=torch.uint8, device="cuda", generator=g)
    for _ in range(2):
        ah.debug_gemm_mxf4(a, sa, b, sb, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            flush.zero_()
            ah.debug_gemm_mxf4(a, sa, b, sb, out_dtype=torch.bfloat16)
        torch.cuda.synchronize()
    d = defaultdict(list)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA and "k_gemm_mxf4" in ev.name:
            d[ev.name].append(ev.device_time)
    us = sum(sum(v) / len(v) for v in d.values())
    fl = 2.0 * M * N * K
    tot_fl += fl
    tot_us += us
    print(f"{path:6s} M={M:6d} N={N:6d} K={K:6d} {us:8.1f} us {fl / us / 1e6:7.0f} TFLOP/s")
print(f"cluster={os.environ.get('ADAHOP_GEMM_CLUSTER', '1')} model={model} total {tot_us:.1f} us "
      f"{tot_fl / tot_us / 1e6:.0f} TFLOP/s")

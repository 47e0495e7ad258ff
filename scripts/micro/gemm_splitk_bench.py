"""Time the MXFP4 GEMM alone (torch.profiler device times, L2 flushed) on long-K few-tile wgrad
shapes with fp32 output (the bench's G_W), for the ADAHOP_GEMM_SPLITK setting of an experiment
build (0 = 256x128 tiles, 2 / 4 = pairs per split-K cluster, 1 = automatic)."""
import os
import sys
from collections import defaultdict

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2604_02525_b200 as ah  # noqa: E402

shapes = [(512, 2048, 16384), (1024, 4096, 16384), (768, 3072, 16384), (512, 1024, 8192)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for M, N, K in shapes:
    g = torch.Generator(device="cuda").manual_seed(0)
    a = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device="cuda", generator=g)
    b = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device="cuda", generator=g)
    sa = torch.randint(118, 122, (M, K // 32), dtype=torch.uint8, device="cuda", generator=g)
    sb = torch.randint(118, 122, (N, K // 32), dtype=torch.uint8, device="cuda", generator=g)
    for _ in range(2):
        ah.debug_gemm_mxf4(a, sa, b, sb, out_dtype=torch.float32)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(10):
            flush.zero_()
            ah.debug_gemm_mxf4(a, sa, b, sb, out_dtype=torch.float32)
        torch.cuda.synchronize()
    d = defaultdict(list)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA and "k_gemm_mxf4" in ev.name:
            d[ev.name].append(ev.device_time)
    for name, v in d.items():
        us = sum(v) / len(v)
        print(f"split={os.environ.get('ADAHOP_GEMM_SPLITK', '1')} M={M:5d} N={N:5d} K={K:6d} {us:8.1f} us "
              f"{2.0 * M * N * K / us / 1e6:7.0f} TFLOP/s  {name.split('(')[0][-40:]}")

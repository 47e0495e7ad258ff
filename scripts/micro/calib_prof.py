"""Kernel times of one calibration step (stats + classify) per Llama-3.2-1B tensor shape."""
import sys
from collections import defaultdict
sys.path.insert(0, ".")
import torch  # noqa: E402
import paper_2604_02525_b200 as ah  # noqa: E402
for R, C in ((16384, 2048), (2048, 2048), (16384, 8192), (8192, 2048), (16384, 512)):
    t = torch.randn(R, C, device="cuda").to(torch.bfloat16)
    ws = torch.empty(ah.calibrate_workspace_bytes(R, C), dtype=torch.uint8, device="cuda")
    cv = torch.empty(2, dtype=torch.float64, device="cuda")
    pat = torch.empty(1, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        ah.calibrate_async(t, ws, cv, pat)
    torch.cuda.synchronize()
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for _ in range(5):
            ah.calibrate_async(t, ws, cv, pat)
        torch.cuda.synchronize()
    d = defaultdict(list)
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            d[ev.name.split("(")[0][:40]].append(ev.device_time)
    print(R, C, {k: round(sum(v) / len(v), 1) for k, v in d.items()}, f"ideal {R * C * 2 / 6.5e6:.1f} us")

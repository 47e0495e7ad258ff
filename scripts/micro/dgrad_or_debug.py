"""Debug: 8B k linear, Lv2 (dgrad OE-Left fused into W's pass): determinism and bf16 = RN(fp32)."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_2604_02525_b200 as ah
import synth
T, d_in, d_out = 16384, 4096, 1024
px, pg = synth.LLAMA32_1B_LAYER_PATTERNS["k"]
dev = torch.device("cuda:0")
x = synth.operand_torch(T, d_in, px, "X", 501, dev)
w = synth.operand_torch(d_out, d_in, "N", "W", 502, dev)
gy = synth.operand_torch(T, d_out, pg, "GY", 503, dev)
for level in (2, 1):
    strats = tuple(ah.layer_strategies(px, "N", pg, level)[0])
    p = ah.Params(oe_k=64, level=level)
    a = ah.linear_layer(x, w, gy, strats, p, out_dtype=torch.float32)
    b = ah.linear_layer(x, w, gy, strats, p, out_dtype=torch.float32)
    c = ah.linear_layer(x, w, gy, strats, p, out_dtype=torch.bfloat16)
    torch.cuda.synchronize()
    for name, u, v, z in zip(("fwd", "dgrad", "wgrad"), a, b, c):
        det = (u.view(torch.int32) != v.view(torch.int32))
        rn = (z != u.to(torch.bfloat16))
        rows_det = torch.unique(torch.nonzero(det)[:, 0]).cpu().numpy()[:20]
        rows_rn = torch.unique(torch.nonzero(rn)[:, 0]).cpu().numpy()[:20]
        print(f"level {level} {strats} {name}: nondet {int(det.sum())} rows {rows_det}; bf16!=RN(fp32) {int(rn.sum())} rows {rows_rn}")

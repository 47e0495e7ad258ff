"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck): one
adahop_linear_layer per strategy set on ragged shapes (FOID, OE gathers, the dual-orientation
tensor-core quantiser with and without the fused outlier product, BF16 outlier GEMM + fold,
the MXFP4 GEMMs on CTA pairs and single CTAs, the Lv2 BF16 GEMM), the split forward/backward
API and one calibration step. Prints the max relative error against the CPU oracle so a run
that the sanitizer slows down still proves it computed the right thing.
Usage: compute-sanitizer --tool racecheck python scripts/sanitize_layer.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2604_02525_b200 as ah  # noqa: E402
import synth  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def main():
    dev = torch.device("cuda:0")
    worst = 0.0
    for (T, d_in, d_out), strats in [((544, 352, 224), ("IHT", "OE_LEFT_IHT", "OE_RIGHT_IHT")),
                                     ((640, 256, 384), ("OE_RIGHT_IHT", "IHT", "OE_LEFT_IHT")),
                                     ((384, 128, 96), ("IHT", "IHT", "BF16"))]:
        x, _ = synth.operand(T, d_in, "C", "X", case_id=11)
        w, _ = synth.operand(d_out, d_in, "N", "W", case_id=12)
        gy, _ = synth.operand(T, d_out, "R", "GY", case_id=13)
        p = ah.Params(oe_k=16)
        xd, wd, gd = (torch.from_numpy(a).to(dev, torch.bfloat16) for a in (x, w, gy))
        y, gx, gw = ah.linear_layer(xd, wd, gd, strats, p, out_dtype=torch.float32)
        torch.cuda.synchronize()
        for path, got, s in (("fwd", y, strats[0]), ("dgrad", gx, strats[1]), ("wgrad", gw, strats[2])):
            worst = max(worst, rel(got.cpu().numpy().astype(np.float64), O.linear(path, s, x=x, w=w, gy=gy, k=16)))
        y2, ctx = ah.linear_forward(xd, wd, strats, p, out_dtype=torch.float32)
        gx2, gw2 = ah.linear_backward(gd, wd, ctx, gx_dtype=torch.float32, gw_dtype=torch.float32)
        torch.cuda.synchronize()
        worst = max(worst, rel(gw2.cpu().numpy().astype(np.float64), gw.cpu().numpy().astype(np.float64)))
    t = torch.from_numpy(synth.operand(512, 256, "R", "X", case_id=21)[0]).to(dev, torch.bfloat16)
    pat, _, _ = ah.calibrate(t)
    torch.cuda.synchronize()
    print(f"sanitize workload done: max rel err vs oracle {worst:.2e}, calibration pattern {pat}")


if __name__ == "__main__":
    main()

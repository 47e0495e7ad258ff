#!/usr/bin/env python
"""Nine-pair quantisation-error sweep (the Imp metric of P:161-163, Fig. 3).

For every outlier pattern pair (P_A, P_B) of C = A·B (A: M x K, B: K x N, patterns in that fed
orientation: R = rows, C = columns), on Fig-3-style synthetic tensors (256 x 256, three planted
rows / columns at x38.3 for kurtosis ~226), it reports the relative MSE against the exact
product of
  * base  — Q(A) Q(B), plain MXFP4 with no transform (the oracle: the GPU path has no
            untransformed mode, every AdaHOP strategy applies the IHT),
  * IHT, OE-L+IHT, OE-R+IHT — the GPU path (adahop_gemm through the C ABI), k = 8,
  * the IHT improvement Imp = (E_base - E_IHT) * 100 / E_base,
  * the strategy the table picks (tab:strategy_summary P:305-326, Lv1) and the best measured.
The GPU IHT error is also checked against the oracle's (same codes, fp32 vs fp64 sums).

Usage (B200): python tests/pair_mse_sweep.py [--seeds 5] [--json out.json]
(It lives under tests/ because it calls the oracle: only tests/, smoke() and bench.py's CPU
legs may.)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle as O  # noqa: E402
import synth  # noqa: E402

PAIRS = [a + b for a in "RCN" for b in "RCN"]
STRATS = ("IHT", "OE_LEFT_IHT", "OE_RIGHT_IHT")


def operands(pair: str, seed: int, n: int = 256, count: int = 3, scale: float = 38.3):
    a, _ = synth.operand(n, n, pair[0], "X", case_id=900 + 10 * seed, count=count, scale=scale)
    b, _ = synth.operand(n, n, pair[1], "X", case_id=901 + 10 * seed, count=count, scale=scale)
    return a, b   # A (M x K), B (K x N), bf16-representable fp32


def mse(c, exact):
    return float(np.mean((np.asarray(c, np.float64) - exact) ** 2))


def sweep(seeds: int = 5, k: int = 8):
    import torch

    import paper_2604_02525_b200 as ah
    dev = torch.device("cuda:0")
    p = ah.Params(oe_k=k)
    rows = []
    for pair in PAIRS:
        acc = {s: 0.0 for s in ("base", "base_oracle_iht") + STRATS}
        for seed in range(seeds):
            a, b = operands(pair, seed)
            b_store = np.ascontiguousarray(b.T)
            exact = a.astype(np.float64) @ b.astype(np.float64)
            acc["base"] += mse(O.adahop_matmul(a, b_store, O.IHT, hadamard="none"), exact) / seeds
            acc["base_oracle_iht"] += mse(O.adahop_matmul(a, b_store, O.IHT), exact) / seeds
            ad = torch.from_numpy(a).to(dev, torch.bfloat16)
            bd = torch.from_numpy(b_store).to(dev, torch.bfloat16)
            for s in STRATS:
                c = ah.gemm(ad, False, bd, False, a.shape[0], b.shape[1], a.shape[1], s, p, out_dtype=torch.float32)
                acc[s] += mse(c.cpu().numpy(), exact) / seeds
        chosen = O.strategy_for_pair(pair[0], pair[1], 1)
        best = min(STRATS, key=lambda s: acc[s])
        norm = float(np.mean(exact ** 2))
        rows.append({"pair": pair, **{f"relmse_{s}": acc[s] / norm for s in acc},
                     "imp_iht_pct": (acc["base"] - acc["IHT"]) * 100.0 / acc["base"],
                     "iht_gpu_vs_oracle": acc["IHT"] / acc["base_oracle_iht"],
                     "table_choice": chosen, "best_measured": best})
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seeds", type=int, default=5)
    ap.add_argument("--json", default=None)
    args = ap.parse_args()
    rows = sweep(args.seeds)
    print(f"{'pair':4s} {'base':>10s} {'IHT':>10s} {'OE-L+IHT':>10s} {'OE-R+IHT':>10s} {'Imp(IHT)%':>9s}"
          f" {'gpu/orc':>8s}  table -> best")
    for r in rows:
        print(f"{r['pair']:4s} {r['relmse_base']:10.3e} {r['relmse_IHT']:10.3e} {r['relmse_OE_LEFT_IHT']:10.3e} "
              f"{r['relmse_OE_RIGHT_IHT']:10.3e} {r['imp_iht_pct']:9.1f} {r['iht_gpu_vs_oracle']:8.4f}  "
              f"{r['table_choice']} -> {r['best_measured']}")
    if args.json:
        with open(args.json, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()

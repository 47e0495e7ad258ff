"""Calibration-driven plan (§5.1): run the calibration pass on every linear's X, W and
G_Y for a number of training steps (30 in the paper), vote each tensor's pattern over the
steps, and freeze the strategy of each of the linear's three matmuls (tab:strategy_summary,
P:305-326). The frozen plan is what the hot path consumes: "requires no runtime pattern
detection".

Every decision is the library's: adahop_calibrate (stats + App. A classification, per tensor and
step, device-resident and graph-capturable), adahop_majority_vote, adahop_layer_strategies (fed
orientation + strategy table). This module only records the per-step pattern codes, reads them back
once, and persists the result (JSON) — SURVEY §5's checkpoint of the calibration outcome.
"""
from __future__ import annotations

import json
from collections import Counter
from dataclasses import asdict, dataclass, field

import torch

from . import adahop as ah

TENSORS = ("X", "W", "G_Y")
PATHS = ("fwd", "dgrad", "wgrad")


@dataclass
class LinearPlan:
    name: str
    d_in: int
    d_out: int
    patterns: dict                       # tensor -> voted pattern ('R' | 'C' | 'N')
    strategies: tuple                    # (fwd, dgrad, wgrad)
    fed_pairs: tuple                     # fed (left, right) patterns per path, e.g. ('CN', 'CN', 'RC')
    votes: dict = field(default_factory=dict)   # tensor -> {pattern: steps}
    oe_k: int = 0                        # per-layer OE k (DESIGN R16; 0 = the global k)
    outliers: dict = field(default_factory=dict)   # tensor -> [rows, cols], the largest over the steps


# The OE operand of each path, as (tensor, axis of that tensor whose outlier count sizes k):
# OE-Left extracts rows of A_store, OE-Right rows of B_store: fwd A = X, B_store = W;
# dgrad A = G_Y, B_store = W^T (W's columns); wgrad A = G_Y^T (G_Y's columns), B_store = X^T (X's columns)
OE_OPERAND = {("fwd", "OE_LEFT_IHT"): ("X", 0), ("fwd", "OE_RIGHT_IHT"): ("W", 0),
              ("dgrad", "OE_LEFT_IHT"): ("G_Y", 0), ("dgrad", "OE_RIGHT_IHT"): ("W", 1),
              ("wgrad", "OE_LEFT_IHT"): ("G_Y", 1), ("wgrad", "OE_RIGHT_IHT"): ("X", 1)}


def adaptive_k(count: int, k_max: int = 64, granule: int = 16) -> int:
    """DESIGN R16: the OE operand's outlier rows rounded up to the tcgen05 N granule,
    clamped to [granule, k_max]."""
    return int(min(k_max, max(granule, -(-int(count) // granule) * granule)))


def layer_oe_k(strategies, outliers: dict, k_max: int = 64) -> int:
    """One k per linear (adahop_linear_layer takes one): the largest over its OE paths."""
    ks = [adaptive_k(outliers[OE_OPERAND[(p, s)][0]][OE_OPERAND[(p, s)][1]], k_max)
          for p, s in zip(PATHS, strategies) if (p, s) in OE_OPERAND]
    return max(ks) if ks else 0


@dataclass
class Plan:
    level: int
    steps: int
    linears: list

    def strategies(self, name: str) -> tuple:
        return next(lp.strategies for lp in self.linears if lp.name == name)

    def census(self) -> dict:
        """Fed-pair counts per path (the form of tab:pattern_distribution)."""
        out = {p: Counter() for p in PATHS}
        for lp in self.linears:
            for p, pair in zip(PATHS, lp.fed_pairs):
                out[p][pair] += 1
        return {p: dict(sorted(c.items())) for p, c in out.items()}

    def to_json(self) -> str:
        return json.dumps({"level": self.level, "steps": self.steps,
                           "linears": [dict(asdict(lp), strategies=list(lp.strategies),
                                            fed_pairs=list(lp.fed_pairs)) for lp in self.linears]}, indent=1)

    @staticmethod
    def from_json(text: str) -> "Plan":
        d = json.loads(text)
        lins = [LinearPlan(e["name"], e["d_in"], e["d_out"], e["patterns"], tuple(e["strategies"]),
                           tuple(e["fed_pairs"]), e.get("votes", {}), e.get("oe_k", 0), e.get("outliers", {}))
                for e in d["linears"]]
        return Plan(d["level"], d["steps"], lins)

    def save(self, path: str) -> None:
        with open(path, "w") as f:
            f.write(self.to_json())

    @staticmethod
    def load(path: str) -> "Plan":
        with open(path) as f:
            return Plan.from_json(f.read())


def plan_from_patterns(linears, per_step: dict, level: int = 1, outliers: dict | None = None,
                       k_max: int = 64) -> Plan:
    """linears: [(name, d_in, d_out)]; per_step[(name, tensor)] = the per-step pattern letters.
    Votes each record (adahop_majority_vote) and maps the voted patterns to the three strategies
    (adahop_layer_strategies). With outliers[(name, tensor)] = [rows, cols] (the largest over the
    steps) each linear also gets its adaptive OE k (DESIGN R16)."""
    out = []
    steps = 0
    for name, d_in, d_out in linears:
        pats, votes = {}, {}
        for t in TENSORS:
            rec = list(per_step[(name, t)])
            steps = max(steps, len(rec))
            pats[t] = ah.majority_vote(rec)
            votes[t] = dict(Counter(rec))
        strategies, fed = ah.layer_strategies(pats["X"], pats["W"], pats["G_Y"], level)
        lp = LinearPlan(name, d_in, d_out, pats, strategies, fed, votes)
        if outliers is not None:
            lp.outliers = {t: list(outliers[(name, t)]) for t in TENSORS}
            lp.oe_k = layer_oe_k(strategies, lp.outliers, k_max)
        out.append(lp)
    return Plan(level, steps, out)


class Calibrator:
    """Records one pattern code per (step, linear, tensor) on the device.

    record() issues adahop_calibrate for X, W and G_Y of one linear (no host synchronisation, so a
    whole calibration step can be captured in a CUDA graph); plan() reads the record back once and
    votes. Token-sharded data parallelism uses paper_2604_02525_b200.dist.calibrate_sharded per
    tensor instead (its classification needs the merged statistics of all ranks)."""

    def __init__(self, linears, steps: int = 30, params=None, device=None):
        self.linears = list(linears)
        self.index = {name: i for i, (name, _, _) in enumerate(self.linears)}
        self.steps = steps
        self.params = params or ah.Params()
        dev = device or torch.device("cuda", torch.cuda.current_device())
        n = len(self.linears)
        self.pat = torch.full((steps, n, 3), 255, dtype=torch.uint8, device=dev)
        self.cv = torch.zeros((steps, n, 3, 4), dtype=torch.float64, device=dev)
        self.cnt = torch.full((steps, n, 3, 2), -1, dtype=torch.int32, device=dev)   # outlier rows / cols
        self.ws = None
        self.device = dev

    def workspace_bytes(self, T: int) -> int:
        return max(ah.calibrate_batch_workspace_bytes([(T, d_in), (d_out, d_in), (T, d_out)])
                   for _, d_in, d_out in self.linears)

    def record(self, step: int, name: str, x: torch.Tensor, w: torch.Tensor, gy: torch.Tensor) -> None:
        """One calibration step of the linear's X, W and G_Y (adahop_calibrate_batch: three launches)."""
        i = self.index[name]
        need = ah.calibrate_batch_workspace_bytes([t.shape for t in (x, w, gy)])
        if self.ws is None or self.ws.numel() < need:
            self.ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        shapes = [x.shape, w.shape, gy.shape]
        ah.calibrate_batch_async([x, w, gy], self.ws, self.cv[step, i], self.pat[step, i], self.params)
        ah.calibrate_batch_outliers_async(shapes, self.ws, self.cnt[step, i])

    def record_sharded(self, step: int, name: str, x_local: torch.Tensor, w: torch.Tensor, gy_local: torch.Tensor,
                       rows_global: int, group=None) -> None:
        """Token-sharded variant: X and G_Y hold this rank's token rows; their patterns are decided
        on the statistics merged over all ranks (dist.calibrate_sharded), W (replicated) locally."""
        from . import dist as ahd
        i = self.index[name]
        codes = {"N": 0, "R": 1, "C": 2}
        for j, t in enumerate((x_local, None, gy_local)):
            if t is None:
                need = ah.calibrate_workspace_bytes(*w.shape)
                if self.ws is None or self.ws.numel() < need:
                    self.ws = torch.empty(need, dtype=torch.uint8, device=self.device)
                ah.calibrate_async(w, self.ws, self.cv[step, i, j], self.pat[step, i, j:j + 1], self.params)
                continue
            st = ahd.calibrate_sharded(t, rows_global, group=group)
            self.pat[step, i, j] = codes[st.pattern]

    def per_step_patterns(self) -> dict:
        codes = self.pat.cpu().tolist()
        out = {}
        for name, i in self.index.items():
            for j, t in enumerate(TENSORS):
                rec = [codes[s][i][j] for s in range(self.steps)]
                if any(c > 2 for c in rec):
                    raise RuntimeError(f"calibration record of {name}.{t} is incomplete")
                out[(name, t)] = [ah.PAT_NAME[c] for c in rec]
        return out

    def outlier_counts(self) -> dict | None:
        """(name, tensor) -> [rows, cols], the largest over the steps; None if any step lacks them
        (the token-sharded record keeps no counts)."""
        c = self.cnt.cpu()
        if bool((c < 0).any()):
            return None
        mx = c.amax(dim=0).tolist()
        return {(name, t): mx[i][j] for name, i in self.index.items() for j, t in enumerate(TENSORS)}

    def plan(self, level: int = 1, k_max: int = 64) -> Plan:
        return plan_from_patterns(self.linears, self.per_step_patterns(), level, self.outlier_counts(), k_max)

"""Data-parallel plumbing of the AdaHOP hot path (token-row sharding).

One process per GPU. Token rows T are split into contiguous per-rank ranges (multiples of
the Hadamard block, so that the wgrad path's 32-blocks along T never straddle ranks).
fwd and dgrad are independent per rank; wgrad yields a rank-local partial G_W (with
rank-local FOID, R12) that is summed by an all-reduce over NVLink (NCCL).
Calibration merges the per-column statistics (sum for the moments, max for |x|) and the
per-row CV sums across ranks so every rank classifies — and freezes — the same pattern.

The collective is torch.distributed (NCCL on B200, gloo in the CPU tests); the compute is
injected (the C ABI by default) so the host logic is testable without a GPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional

import torch
import torch.distributed as dist


def token_shard(t_global: int, world: int, rank: int, align: int = 32) -> tuple[int, int]:
    """[t0, t1) token rows of `rank`: contiguous, balanced, every boundary a multiple of
    `align` (the Hadamard block along tokens)."""
    if t_global % align:
        raise ValueError(f"global tokens {t_global} must be a multiple of {align}")
    blocks = t_global // align
    base, extra = divmod(blocks, world)
    b0 = rank * base + min(rank, extra)
    b1 = b0 + base + (1 if rank < extra else 0)
    return b0 * align, b1 * align


def allreduce_wgrad(gw: torch.Tensor, group=None, async_op: bool = False):
    """Sum the rank-local wgrad partials G_W,r = AdaHOP(G_Y,r^T, X_r) in place."""
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return None
    return dist.all_reduce(gw, op=dist.ReduceOp.SUM, group=group, async_op=async_op)


def merge_col_stats(col_stats: torch.Tensor, group=None) -> torch.Tensor:
    """Per-column statistics [cols, 4] = (sum x, sum x^2, sum |x|, max |x|) of the local token
    rows -> the global ones (sum of the first three, max of the fourth), in place."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        moments = col_stats[:, :3].contiguous()
        amax = col_stats[:, 3].contiguous()
        dist.all_reduce(moments, op=dist.ReduceOp.SUM, group=group)
        dist.all_reduce(amax, op=dist.ReduceOp.MAX, group=group)
        col_stats[:, :3] = moments
        col_stats[:, 3] = amax
    return col_stats


def merge_row_cv_sum(row_cv_sum: torch.Tensor, group=None) -> torch.Tensor:
    """Sum over ranks of sum_i std(T_i,:)/(mean|T_i,:| + eps) of the local rows (App. A)."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(row_cv_sum, op=dist.ReduceOp.SUM, group=group)
    return row_cv_sum


@dataclass
class CalibrationStep:
    pattern: str
    cv_row: float
    cv_col: float


@dataclass
class CalibrationOps:
    """The three library calls of one calibration step (include/adahop.h):
    stats(t) -> (row_stats [rows, 4], col_stats [cols, 4])           adahop_stats
    classify(row_stats, col_stats, row_len, col_count) -> (cv[4], pat) adahop_classify
    classify_sums(cv, rows_global, cols) -> pat                        adahop_classify_sums
    The CPU tests inject host implementations; the product uses the C ABI (``default_ops``)."""
    stats: Callable
    classify: Callable
    classify_sums: Callable


def default_ops() -> CalibrationOps:
    from . import adahop as ah
    return CalibrationOps(ah.stats, ah.classify, ah.classify_sums)


PAT_NAME = {0: "N", 1: "R", 2: "C"}


def calibrate_sharded(t_local: torch.Tensor, rows_global: int, ops: Optional[CalibrationOps] = None,
                      group=None) -> CalibrationStep:
    """One calibration step of one token-sharded tensor (rows = tokens), App. A.

    Every arithmetic step runs in the library; this function only moves data between ranks:
      1. adahop_stats on the local rows;
      2. all-reduce the column statistics (SUM of the moments, MAX of |x|);
      3. adahop_classify with col_count = rows_global: cv[0] = local row-CV sum,
         cv[1] = column-CV sum over the merged statistics;
      4. all-reduce cv[0] (SUM over ranks);
      5. adahop_classify_sums(rows_global): CV_row, CV_col and the pattern, identical on all ranks."""
    ops = ops or default_ops()
    _, cols = t_local.shape
    row_stats, col_stats = ops.stats(t_local)
    merge_col_stats(col_stats, group)
    cv, _ = ops.classify(row_stats, col_stats, cols, rows_global)
    row_sum = cv[:1].clone()
    merge_row_cv_sum(row_sum, group)
    cv[:1].copy_(row_sum)
    pat = ops.classify_sums(cv, rows_global, cols)
    vals = cv.cpu().tolist()
    return CalibrationStep(PAT_NAME[int(pat.reshape(-1)[0].item())], vals[2], vals[3])


class DataParallelLinear:
    """One linear on this rank's token shard, AdaHOP strategies fixed per path at calibration
    time; wgrad partials are all-reduced.

    The training-step form is forward() / backward(): the split layer API (adahop_linear_forward /
    _backward) quantises X and W once in both orientations in the forward, saves the FP4
    context, and the backward quantises G_Y once for dgrad and wgrad — the path bench.py times.
    fwd() / dgrad() / wgrad() are the per-path calls (every operand quantised per GEMM)."""

    def __init__(self, strategies: dict, params=None, group=None, compute: Optional[dict] = None):
        self.strategies = strategies
        self.params = params
        self.group = group
        self.compute = dict(compute or {})   # injected ops (CPU tests); the C ABI otherwise

    _OPS = {"fwd": "linear_fwd", "dgrad": "linear_dgrad", "wgrad": "linear_wgrad",
            "forward": "linear_forward", "backward": "linear_backward"}

    def _op(self, name):
        if name not in self.compute:
            from . import adahop as ah   # loads the CUDA library (fails loudly without it)
            self.compute[name] = getattr(ah, self._OPS[name])
        return self.compute[name]

    def _strats(self):
        return (self.strategies["fwd"], self.strategies["dgrad"], self.strategies["wgrad"])

    def forward(self, x_local, w, **kw):
        """(Y_local, ctx): Y = X W^T on the local token rows and the saved backward context."""
        return self._op("forward")(x_local, w, self._strats(), self.params, **kw)

    def backward(self, gy_local, w, ctx, async_op: bool = False, **kw):
        """(G_X_local, G_W[, work]): G_W is the rank-local partial summed over ranks."""
        gx, gw = self._op("backward")(gy_local, w, ctx, **kw)
        work = allreduce_wgrad(gw, self.group, async_op=async_op)
        return (gx, gw, work) if async_op else (gx, gw)

    def fwd(self, x_local, w, **kw):
        return self._op("fwd")(x_local, w, self.strategies["fwd"], self.params, **kw)

    def dgrad(self, gy_local, w, **kw):
        return self._op("dgrad")(gy_local, w, self.strategies["dgrad"], self.params, **kw)

    def wgrad(self, gy_local, x_local, async_op: bool = False, **kw):
        gw = self._op("wgrad")(gy_local, x_local, self.strategies["wgrad"], self.params, **kw)
        work = allreduce_wgrad(gw, self.group, async_op=async_op)
        return (gw, work) if async_op else gw

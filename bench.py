#!/usr/bin/env python
"""AdaHOP MXFP4 linear benchmark (BASELINE.json metric, configs[1] workload).

One STEP = the whole hot path over one batch: the 21 GEMMs of one Llama-3.2-1B
transformer layer (q, k, v, o, gate, up, down x fwd / dgrad / wgrad) at T = 16384 tokens
per GPU (seq 2048 x batch 8), each through the C ABI (FOID + IHT/quant + MXFP4 GEMM +
BF16 outlier GEMM + scatter-add, strategy from the pattern pair, AdaHOP-Lv1, k = 64).
Per-linear tensor patterns follow the Table-1 census classes (synth.LLAMA32_1B_LAYER_PATTERNS),
which exercises the six pairs that occur in practice: CN, NN, RN, RC, NC, CC.

value      = sum(2 M N K) over the step's GEMMs, all ranks / max-over-ranks device time
e2e        = the same metric with inputs copied from pinned host memory and outputs read
             back inside the timed region
cublas     = the same 21 GEMMs with torch.matmul (cuBLAS BF16), same shapes / output dtype
roofline   = dominant kernel (CUDA events recorded by the library between stages)
cpu_baseline / --impl reference = the CPU oracle (oracle/) on a bounded sample

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl adahop|reference]
Multi-GPU: python -m torch.distributed.run --nproc-per-node N bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
from collections import Counter
import json
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "AdaHOP MXFP4 linear TFLOP/s (IHT+quant+OE+GEMM) and speedup vs BF16 cuBLAS"
UNIT = "TFLOP/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="adahop", choices=["adahop", "reference"])
    ap.add_argument("--workload", default="llama32_1b",
                    choices=["llama32_1b", "llama3_8b", "instella_3b", "llama32_1b_stack"],
                    help="llama32_1b_stack = BASELINE configs[4]: the full 16-layer linear stack (336 GEMMs) "
                         "with 30 calibration steps -> plan -> step")
    ap.add_argument("--calib-steps", type=int, default=30)
    ap.add_argument("--tokens", type=int, default=16384, help="tokens per GPU")
    ap.add_argument("--oe-k", type=int, default=64)
    ap.add_argument("--adaptive-k", action="store_true",
                    help="stack workload: per-linear OE k from the calibration plan (DESIGN R16, P:503)")
    ap.add_argument("--level", type=int, default=1)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=64, help="oracle sample rows/cols per GEMM")
    ap.add_argument("--no-graph", action="store_true", help="launch eagerly instead of a CUDA graph")
    ap.add_argument("--per-path", action="store_true",
                    help="three adahop_linear_* calls per linear instead of one adahop_linear_layer call")
    ap.add_argument("--no-split", action="store_true",
                    help="skip the forward/backward split timing (adahop_linear_forward / _backward)")
    return ap.parse_args()


# ------------------------------------------------------------------------------- workload
def transpose_pattern(p):
    return {"R": "C", "C": "R", "N": "N"}[p]


def fed_pair(path, px, pw, pg):
    # fed orientation: fwd (X, W^T), dgrad (G_Y, W), wgrad (G_Y^T, X)
    if path == "fwd":
        return px, transpose_pattern(pw)
    if path == "dgrad":
        return pg, pw
    return transpose_pattern(pg), px


def workload_spec(name):
    model = {"llama32_1b": synth.LLAMA32_1B, "llama3_8b": synth.LLAMA3_8B, "instella_3b": synth.INSTELLA_3B}[name]
    pats = synth.LLAMA32_1B_LAYER_PATTERNS
    return model, pats


def gemm_list(model, pats, tokens):
    out = []
    for name, d_in, d_out in model["linears"]:
        px, pg = pats[name]
        for path in ("fwd", "dgrad", "wgrad"):
            a, b = fed_pair(path, px, "N", pg)
            M, N, K = {"fwd": (tokens, d_out, d_in), "dgrad": (tokens, d_in, d_out),
                       "wgrad": (d_out, d_in, tokens)}[path]
            out.append(dict(linear=name, path=path, pair=a + b, M=M, N=N, K=K, d_in=d_in, d_out=d_out))
    return out


# ------------------------------------------------------------------------------- clocks
class ClockSampler:
    """Samples SM clock and throttle reasons through NVML every ~2 ms while running (the
    timed region is only tens of milliseconds, too short for `nvidia-smi -lms`)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.reasons = set()
        self._stop = threading.Event()
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[index]) if vis and vis.split(",")[index].isdigit() else index
            self.h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self.nv = pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - depends on the box
            self.err = repr(e)

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for n, bit in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(n)
            except Exception:
                pass
            time.sleep(0.002)

    def start(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()

    def stop(self):
        if not self.ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        self._stop.set()
        self.t.join()
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": float(self.max_mhz),
                "samples": len(self.samples), "reasons": sorted(self.reasons)}


# ------------------------------------------------------------------------------- peaks
def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": d["hbm_gbs"], "bf16": d["bf16_tflops"],
                "bf16_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "bf16": 1590.0, "bf16_sustained": 1400.0, "src": "fallback"}


# ------------------------------------------------------------------------------- oracle arm
def oracle_sample_step(gemms, host, sample, rng):
    """Oracle on a bounded sample: for every GEMM of the step, a sample x sample block of
    output entries (FOID over the full operand, quantisation of the sampled rows only).
    Returns the flops those entries represent (2 * K per entry)."""
    import oracle as O
    flops = 0.0
    for g in gemms:
        x, w, gy = host[g["linear"]]
        a_store, b_store = O.path_operands(g["path"], x=x, w=w, gy=gy)
        rows = rng.choice(g["M"], size=min(sample, g["M"]), replace=False)
        cols = rng.choice(g["N"], size=min(sample, g["N"]), replace=False)
        rr, cc = np.meshgrid(rows, cols, indexing="ij")
        O.sampled_entries(a_store, b_store, g["strategy"], rr.ravel(), cc.ravel())
        flops += 2.0 * rr.size * g["K"]
    return flops


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        return int(max(n)) if n else os.cpu_count()
    except Exception:
        return os.cpu_count()


def timed_oracle(fn, threads):
    """Run fn() with the BLAS pool limited to `threads` (the oracle is numpy: its only parallel
    part is BLAS); returns (seconds, the thread count the pool actually had)."""
    try:
        from threadpoolctl import threadpool_limits
        ctx = threadpool_limits(limits=threads, user_api="blas")
    except Exception:
        ctx = None
    try:
        used = blas_threads()
        t0 = time.perf_counter()
        out = fn()
        return time.perf_counter() - t0, used, out
    finally:
        if ctx is not None:
            ctx.restore_original_limits()


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands, on rank 0 only (host cores)."""
    if rank != 0:
        return
    import torch  # noqa: F401  (only for the seeded generator of the same inputs)
    model, pats = workload_spec(args.workload)
    gemms = gemm_list(model, pats, args.tokens)
    for g in gemms:
        g["strategy"] = _strategy_host(g["pair"], args.level)
    host = make_host_inputs(model, pats, args.tokens)
    rng = np.random.default_rng(0)
    for _ in range(args.warmup):
        oracle_sample_step(gemms, host, args.cpu_sample, rng)
    dt, cores, flops = timed_oracle(
        lambda: sum(oracle_sample_step(gemms, host, args.cpu_sample, rng) for _ in range(args.steps)), 1)
    v = flops / dt / 1e12
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_dict(args, world),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": f"{args.cpu_sample}x{args.cpu_sample} output entries per GEMM x 21 GEMMs per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _strategy_host(pair, level):
    # tab:strategy_summary; the product path asks the C ABI, this host copy is
    # only used by the oracle arm so that it runs without a GPU library.
    if pair == "CC":
        return "OE_RIGHT_IHT" if level == 1 else "BF16"
    return {"CN": "IHT", "NN": "IHT", "CR": "IHT", "NR": "IHT", "RN": "OE_LEFT_IHT", "RR": "OE_LEFT_IHT",
            "RC": "OE_RIGHT_IHT", "NC": "OE_RIGHT_IHT"}[pair]


def make_host_inputs(model, pats, tokens):
    """Inputs of the same recipe and shapes as the GPU arm, drawn with torch's CPU generator."""
    import torch
    host = {}
    for li, (name, d_in, d_out) in enumerate(model["linears"]):
        px, pg = pats[name]
        x = synth.operand_torch(tokens, d_in, px, "X", 1000 + li, "cpu").float().numpy()
        w = synth.operand_torch(d_out, d_in, "N", "W", 2000 + li, "cpu").float().numpy()
        gy = synth.operand_torch(tokens, d_out, pg, "GY", 3000 + li, "cpu").float().numpy()
        host[name] = (x, w, gy)
    del torch
    return host


def nccl_version():
    try:
        import torch
        v = torch.cuda.nccl.version()
        return ".".join(str(x) for x in v) if isinstance(v, tuple) else str(v)
    except Exception:   # noqa: BLE001 - informational only
        return None


def config_dict(args, world):
    return {"workload": f"{args.workload}_layer_21gemm (7 linears x fwd/dgrad/wgrad)",
            "api": "adahop_linear_* per path" if args.per_path else "adahop_linear_layer (dual-orientation quant)",
            "tokens_per_gpu": args.tokens, "global_tokens": args.tokens * world,
            "pairs": "CN NN RN RC NC CC (Table-1 census classes)", "oe_k": args.oe_k,
            "level": args.level, "hadamard_block": 32, "out_dtype": "bf16 (Y, G_X), fp32 (G_W)",
            "l2": "flushed between steps (256 MiB write, untimed)",
            "parallelism": f"dp{world} token-sharded, NCCL all-reduce of wgrad" if world > 1 else "single GPU",
            **({"nccl": nccl_version()} if world > 1 else {})}


# ------------------------------------------------------------------------------- GPU arm
def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if world > 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist

    if os.environ.get("ADAHOP_DIST_BACKEND", "nccl") != "nccl":
        local = local % max(1, torch.cuda.device_count())   # several ranks may share a GPU
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        # ADAHOP_DIST_BACKEND=gloo runs the multi-rank path with several ranks on one GPU (a test
        # of the sharding / reduction plumbing; NCCL needs one GPU per rank)
        backend = os.environ.get("ADAHOP_DIST_BACKEND", "nccl")
        if backend == "nccl":
            # NCCL's init log (stderr) records the transport and whether NVLS / NVLink SHARP is
            # used for the wgrad all-reduce; the JSON line is on stdout
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    import paper_2604_02525_b200 as ah
    import paper_2604_02525_b200.dist as ahd

    if args.workload == "llama32_1b_stack":
        run_stack(args, rank, world, local, dev, torch, dist, ah, ahd)
        if world > 1:
            dist.destroy_process_group()
        return

    if world > 1 and not args.no_graph:
        args.no_graph = True     # NCCL collectives are launched eagerly under torchrun

    model, pats = workload_spec(args.workload)
    T = args.tokens
    gemms = gemm_list(model, pats, T)
    params = ah.Params(oe_k=args.oe_k, level=args.level)
    for g in gemms:
        g["strategy"] = ah.strategy_for_pair(g["pair"][0], g["pair"][1], args.level)
        g["flops"] = 2.0 * g["M"] * g["N"] * g["K"]

    # inputs (seeded, synthetic, on the device) and outputs
    lin = {}
    for li, (name, d_in, d_out) in enumerate(model["linears"]):
        px, pg = pats[name]
        seed = 17 * rank
        x = synth.operand_torch(T, d_in, px, "X", 1000 + li + seed, dev)
        w = synth.operand_torch(d_out, d_in, "N", "W", 2000 + li, dev)       # W replicated
        gy = synth.operand_torch(T, d_out, pg, "GY", 3000 + li + seed, dev)
        lin[name] = dict(x=x, w=w, gy=gy,
                         y=torch.empty(T, d_out, dtype=torch.bfloat16, device=dev),
                         gx=torch.empty(T, d_in, dtype=torch.bfloat16, device=dev),
                         gw=torch.empty(d_out, d_in, dtype=torch.float32, device=dev))   # fp32 G_W (DP all-reduce)
    strat3 = {name: tuple(g["strategy"] for g in gemms if g["linear"] == name) for name, _, _ in model["linears"]}
    if args.per_path:
        ws_bytes = max(ah.workspace_bytes(g["path"], T, g["d_in"], g["d_out"], g["strategy"], params) for g in gemms)
    else:
        ws_bytes = max(ah.layer_workspace_bytes(T, d_in, d_out, strat3[name], params)
                       for name, d_in, d_out in model["linears"])
    ws = ah.Workspace(ws_bytes, dev)
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)

    launches = [0]
    units = gemms if args.per_path else [dict(linear=name) for name, _, _ in model["linears"]]

    def step_adahop(stage_events=None):
        n = 0
        works = []   # wgrad all-reduces in flight: linear i's overlaps the kernels of linear i+1
        for gi, g in enumerate(units):
            L = lin[g["linear"]]
            ctx = stage_events[gi] if stage_events is not None else None
            if ctx is not None:
                ctx.__enter__()
            if not args.per_path:
                ah.linear_layer(L["x"], L["w"], L["gy"], strat3[g["linear"]], params, out=(L["y"], L["gx"], L["gw"]),
                                ws=ws)
                if world > 1:
                    works.append(ahd.allreduce_wgrad(L["gw"], async_op=True))   # DP: sum the wgrad partials
            elif g["path"] == "fwd":
                ah.linear_fwd(L["x"], L["w"], g["strategy"], params, out=L["y"], ws=ws)
            elif g["path"] == "dgrad":
                ah.linear_dgrad(L["gy"], L["w"], g["strategy"], params, out=L["gx"], ws=ws)
            else:
                ah.linear_wgrad(L["gy"], L["x"], g["strategy"], params, out=L["gw"], ws=ws)
                if world > 1:
                    works.append(ahd.allreduce_wgrad(L["gw"], async_op=True))   # DP: sum the wgrad partials
            if ctx is not None:
                ctx.__exit__()
            n += ah.last_launch_count()
        for w in works:
            w.wait()   # the step ends when every partial is summed
        launches[0] += n

    def mm_f32(a, b, out):
        # bf16 x bf16 -> fp32 output (cuBLAS), the same G_W dtype as the AdaHOP arm
        try:
            return torch.mm(a, b, out_dtype=torch.float32, out=out)
        except (RuntimeError, TypeError):
            return out.copy_(torch.mm(a, b, out_dtype=torch.float32))

    def step_cublas():
        works = []
        for g in gemms:
            L = lin[g["linear"]]
            if g["path"] == "fwd":
                torch.mm(L["x"], L["w"].t(), out=L["y"])
            elif g["path"] == "dgrad":
                torch.mm(L["gy"], L["w"], out=L["gx"])
            else:
                mm_f32(L["gy"].t(), L["x"], L["gw"])
                if world > 1:   # issued like the AdaHOP arm's: asynchronous, waited at the step end
                    works.append(dist.all_reduce(L["gw"], async_op=True))
        for w in works:
            w.wait()

    def barrier():
        if world > 1:
            dist.barrier()

    def as_graph(fn):
        """Capture one step into a CUDA graph (the library is capture-safe: no host sync,
        no allocation on the hot path); returns a replay callable."""
        if args.no_graph:
            return fn
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
        return g.replay

    def timed(step_fn, steps, warmup, after_step=None, sampler=None):
        for _ in range(warmup):
            l2.zero_()
            step_fn()
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.start()
        ms = 0.0
        for i in range(steps):
            l2.zero_()                                   # untimed L2 flush
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            step_fn()
            e.record()
            torch.cuda.synchronize()                     # between steps only; device-timed
            ms += s.elapsed_time(e)
            if after_step:
                after_step()
        barrier()
        torch.cuda.synchronize()
        clocks = sampler.stop() if sampler else None
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms / steps, clocks

    flops_step = sum(g["flops"] for g in gemms)

    # ---- AdaHOP, device-resident inputs; per-stage events recorded by the library
    stage_ev = [ah.StageEvents() for _ in units]
    step_adahop(stage_ev)                                  # first call: kernel attributes
    torch.cuda.synchronize()
    launches[0] = 0
    step_adahop(stage_ev)
    launches_per_step = launches[0]
    # value: the step as a user runs it (no stage events between the kernels: event nodes would
    # break the programmatic-dependent-launch edges of the graph)
    run_plain = as_graph(lambda: step_adahop())
    sampler = ClockSampler(local)
    ms_ada, clocks = timed(run_plain, args.steps, args.warmup, None, sampler)
    value = flops_step * world / (ms_ada * 1e-3) / 1e12

    # ---- the same 21 GEMMs through the split API a training step uses: the forward of every
    #      linear (saving its FP4 context), then the backward in reverse order
    split = None
    if not args.per_path and not args.no_split:
        names = [name for name, _, _ in model["linears"]]
        ws_split = ah.Workspace(max(ah.split_workspace_bytes(T, d_in, d_out, strat3[name], params)
                                    for name, d_in, d_out in model["linears"]), dev)
        ctxs = {}
        for name in names:   # the contexts: static device buffers reused every step
            L = lin[name]
            _, ctxs[name] = ah.linear_forward(L["x"], L["w"], strat3[name], params, out=L["y"], ws=ws_split)
        torch.cuda.synchronize()

        def step_split():
            for name in names:
                L = lin[name]
                ah.linear_forward(L["x"], L["w"], strat3[name], params, out=L["y"], ws=ws_split, ctx=ctxs[name])
            works = []
            for name in reversed(names):
                L = lin[name]
                ah.linear_backward(L["gy"], L["w"], ctxs[name], out=(L["gx"], L["gw"]), ws=ws_split)
                if world > 1:
                    works.append(ahd.allreduce_wgrad(L["gw"], async_op=True))
            for w in works:
                w.wait()

        ms_split, _ = timed(as_graph(step_split), args.steps, args.warmup)
        saved = sum(c.saved_bytes for c in ctxs.values())
        x_bf16 = sum(lin[n]["x"].numel() * 2 for n in names)
        w_fp4 = sum(lin[n]["w"].numel() * 17 // 32 for n in names)
        split = {"ms_per_step": ms_split, "value": flops_step * world / (ms_split * 1e-3) / 1e12, "unit": UNIT,
                 "api": "adahop_linear_forward (7 linears) then adahop_linear_backward (reverse order)",
                 "saved_context_bytes_per_step": int(saved),
                 "saved_context_bytes_per_linear": {n: int(c.saved_bytes) for n, c in ctxs.items()},
                 "bf16_activation_bytes_per_step": int(x_bf16),
                 "activation_compression_vs_bf16": x_bf16 / max(1, saved - w_fp4),
                 "note": "context = FP4 column layouts of X and W + OE indices + BF16 outlier slices "
                         "(+ X itself where the wgrad strategy multiplies all of X in BF16); compression "
                         "counts the activation part (context minus W's FP4 copy) against BF16 X"}

    # stage breakdown + roofline: the same step replayed with the library's stage events
    run_ada = as_graph(lambda: step_adahop(stage_ev))
    acc = [{n: 0.0 for n in ah.StageEvents.NAMES} for _ in units]

    def collect():
        for gi in range(len(units)):
            for n, v in stage_ev[gi].times_ms().items():
                acc[gi][n] += v / args.steps

    ms_instr, _ = timed(run_ada, args.steps, args.warmup, collect)

    # per-stage breakdown (tab:latency analogue), summed over the step
    stage_tot = {n: 0.0 for n in ah.StageEvents.NAMES}
    per_unit = []
    for gi, g in enumerate(units):
        for n in acc[gi]:
            stage_tot[n] += acc[gi][n]
        per_unit.append(dict(g, **{k: round(v, 4) for k, v in acc[gi].items()}))

    # ---- calibration pass (a1, config 5): one stats + classify step over the layer's 21 tensors
    #      (X, W, G_Y of every linear), timed like the step; 2 B read per element is the work
    cal_t = [L[n] for L in lin.values() for n in ("x", "w", "gy")]
    cal_ws = torch.empty(ah.calibrate_batch_workspace_bytes([t.shape for t in cal_t]), dtype=torch.uint8, device=dev)
    cal_cv = torch.empty((len(cal_t), 4), dtype=torch.float64, device=dev)
    cal_pat = torch.empty(len(cal_t), dtype=torch.uint8, device=dev)

    def step_calib():   # adahop_calibrate_batch: the 21 tensors in three launches
        ah.calibrate_batch_async(cal_t, cal_ws, cal_cv, cal_pat, params)

    def step_calib_each():   # one adahop_calibrate per tensor (three launches each), for comparison
        for i, t in enumerate(cal_t):
            ah.calibrate_async(t, cal_ws, cal_cv[i], cal_pat[i:i + 1], params)

    step_calib()
    ms_cal, _ = timed(as_graph(step_calib), args.steps, args.warmup)
    ms_cal_each, _ = timed(as_graph(step_calib_each), args.steps, args.warmup)
    step_calib()
    cal_bytes = sum(t.numel() * 2 for t in cal_t)
    calib = {"ms_per_calibration_step": ms_cal, "api": "adahop_calibrate_batch (3 launches)",
             "ms_per_calibration_step_per_tensor_calls": ms_cal_each, "tensors": len(cal_t), "bytes_read": cal_bytes,
             "GB_per_s": cal_bytes / (ms_cal * 1e-3) / 1e9,
             "frac_of_hbm": cal_bytes / (ms_cal * 1e-3) / 1e9 / load_peaks()["hbm_gbs"],
             "patterns": "".join("NRC"[int(v)] for v in cal_pat.cpu().tolist())}

    # ---- cuBLAS BF16 baseline (same GEMMs, same flush protocol)
    ms_cub = None
    if not args.no_cublas:
        ms_cub, _ = timed(as_graph(step_cublas), args.steps, args.warmup)

    # ---- per-linear comparison (report per-shape results, the k / v projections are the
    #      shapes where the FP4 path has the least headroom): each linear's three cuBLAS GEMMs timed
    #      with events around them, against the same linear's AdaHOP stages (instrumented replay)
    per_linear = None
    if not args.no_cublas and not args.per_path:
        cub_ms = {name: 0.0 for name, _, _ in model["linears"]}
        for it in range(args.warmup + args.steps):
            l2.zero_()
            evs = []
            for name, _, _ in model["linears"]:
                L = lin[name]
                a_, b_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a_.record()
                torch.mm(L["x"], L["w"].t(), out=L["y"])
                torch.mm(L["gy"], L["w"], out=L["gx"])
                mm_f32(L["gy"].t(), L["x"], L["gw"])
                b_.record()
                evs.append((name, a_, b_))
            torch.cuda.synchronize()
            if it >= args.warmup:
                for name, a_, b_ in evs:
                    cub_ms[name] += a_.elapsed_time(b_) / args.steps
        per_linear = {}
        for gi, (name, d_in, d_out) in enumerate(model["linears"]):
            ada = sum(acc[gi].values())
            fl = 3 * 2.0 * T * d_in * d_out
            per_linear[name] = {"d_in": d_in, "d_out": d_out, "adahop_ms": round(ada, 4), "cublas_ms": round(cub_ms[name], 4),
                                "speedup": cub_ms[name] / ada if ada else None,
                                "adahop_TFLOPs": fl / (ada * 1e-3) / 1e12 if ada else None,
                                "stages_ms": {k: round(v, 4) for k, v in acc[gi].items()}}

    # ---- e2e: pinned host inputs in, outputs out, inside the timed region
    e2e = None
    if not args.no_e2e:
        host_in = {k: {n: L[n].cpu().pin_memory() for n in ("x", "w", "gy")} for k, L in lin.items()}
        host_out = {k: {n: torch.empty_like(L[n], device="cpu").pin_memory() for n in ("y", "gx", "gw")}
                    for k, L in lin.items()}
        h2d = sum(t.numel() * t.element_size() for d in host_in.values() for t in d.values())
        d2h = sum(t.numel() * t.element_size() for d in host_out.values() for t in d.values())

        # three-stage pipeline over the layer's linears: the host->device copy of linear i+1
        # (copy engine, stream s_in) and the device->host copy of linear i-1 (stream s_out) run
        # under the AdaHOP calls of linear i (current stream); events order each linear's stages
        s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
        # only the first linear's copy-in and the last one's copy-out are exposed: start with the
        # linear with the fewest input bytes and end with the one with the fewest output bytes
        def nbytes(k, keys):
            return sum(lin[k][n].numel() * lin[k][n].element_size() for n in keys)

        names = list(lin)
        first = min(names, key=lambda k: nbytes(k, ("x", "w", "gy")))
        rest = [k for k in names if k != first]
        last = min(rest, key=lambda k: nbytes(k, ("y", "gx", "gw")))
        names = [first] + [k for k in rest if k != last] + [last]

        def step_e2e():
            cur = torch.cuda.current_stream()
            s_in.wait_stream(cur)
            s_out.wait_stream(cur)
            ev_in = []
            for k in names:
                with torch.cuda.stream(s_in):
                    for n in ("x", "w", "gy"):
                        lin[k][n].copy_(host_in[k][n], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(s_in)
                ev_in.append(e)
            for i, k in enumerate(names):
                L = lin[k]
                cur.wait_event(ev_in[i])
                if args.per_path:
                    sf, sd, sw = strat3[k]
                    ah.linear_fwd(L["x"], L["w"], sf, params, out=L["y"], ws=ws)
                    ah.linear_dgrad(L["gy"], L["w"], sd, params, out=L["gx"], ws=ws)
                    ah.linear_wgrad(L["gy"], L["x"], sw, params, out=L["gw"], ws=ws)
                else:
                    ah.linear_layer(L["x"], L["w"], L["gy"], strat3[k], params, out=(L["y"], L["gx"], L["gw"]),
                                    ws=ws)
                if world > 1:
                    ahd.allreduce_wgrad(L["gw"], async_op=True).wait()   # before the copy-out of G_W
                e = torch.cuda.Event()
                e.record(cur)
                s_out.wait_event(e)
                with torch.cuda.stream(s_out):
                    for n in ("y", "gx", "gw"):
                        host_out[k][n].copy_(L[n], non_blocking=True)
            cur.wait_stream(s_out)
            cur.wait_stream(s_in)

        ms_e2e, _ = timed(step_e2e, args.e2e_steps, 1)
        e2e = {"value": flops_step * world / (ms_e2e * 1e-3) / 1e12, "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

    # ---- roofline of the dominant kernel
    peaks = load_peaks()
    dom = max(stage_tot, key=stage_tot.get)
    roof = roofline(dom, gemms, stage_tot, peaks, T, model, per_path=args.per_path, workload=args.workload)
    if dom == "gemm_mxf4" and not args.no_cublas:
        lib = library_fp4(gemms, args, l2, as_graph, timed, dev)
        if lib:
            roof["library_fp4"] = lib

    # ---- CPU oracle baseline (rank 0, bounded sample)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        host = {k: (L["x"].float().cpu().numpy(), L["w"].float().cpu().numpy(), L["gy"].float().cpu().numpy())
                for k, L in lin.items()}
        rng = np.random.default_rng(0)
        dt, used, fl = timed_oracle(lambda: oracle_sample_step(gemms, host, args.cpu_sample, rng), 1)
        dt_all, used_all, fl_all = timed_oracle(lambda: oracle_sample_step(gemms, host, args.cpu_sample, rng),
                                                os.cpu_count())
        cpu = {"value": fl / dt / 1e12, "unit": UNIT, "cores": used, "kind": "oracle",
               "all_cores": {"value": fl_all / dt_all / 1e12, "cores": used_all, "seconds": round(dt_all, 2)},
               "seconds": round(dt, 2),
               "sample": f"{args.cpu_sample}x{args.cpu_sample} output entries of each of the 21 GEMMs "
                         "(FOID on the full operand, quantisation of the sampled rows)"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_ada, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "mxfp4", "data": "synthetic", "config": config_dict(args, world),
                "speedup_vs_cublas_bf16": (ms_cub / ms_ada) if ms_cub else None,
                "cublas_bf16": {"value": flops_step * world / (ms_cub * 1e-3) / 1e12, "ms_per_step": ms_cub}
                if ms_cub else None,
                "stages_ms_per_step": {k: round(v, 4) for k, v in stage_tot.items()},
                "ms_per_step_instrumented": ms_instr,
                "calibration": calib,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks, "split": split,
                "per_linear": per_linear,
                "gpu_launches": int(launches_per_step * args.steps),
                "launch": "eager" if args.no_graph else "cuda_graph"}
        print(json.dumps(line), flush=True)
        with open(os.path.join(ROOT, "gpurun_out", "bench_per_gemm.json") if os.path.isdir(
                os.path.join(ROOT, "gpurun_out")) else os.devnull, "w") as f:
            json.dump(per_unit, f, indent=1)
    if world > 1:
        dist.destroy_process_group()


def run_stack(args, rank, world, local, dev, torch, dist, ah, ahd):
    """BASELINE configs[4]: the full Llama-3.2-1B training-step linear stack —
    16 layers x 7 linears x (fwd, dgrad, wgrad) = 336 GEMMs per GPU per step at T tokens per GPU —
    with the calibration pass in front (§5.1): args.calib_steps steps of adahop_calibrate
    on every X, W, G_Y (fresh noise each step, outlier channels fixed per tensor, patterns per the
    Table-1 census, synth.llama32_1b_census_patterns) -> adahop_majority_vote ->
    adahop_layer_strategies -> a persisted plan that fixes the strategy of every GEMM of the step."""
    from paper_2604_02525_b200 import plan as plan_mod
    T = args.tokens
    params = ah.Params(oe_k=args.oe_k, level=args.level)
    cfg = synth.llama32_1b_census_patterns()
    dims = {n: (a, b) for n, a, b in synth.LLAMA32_1B["linears"]}
    keys = [f"l{layer}.{name}" for layer, name, *_ in cfg]
    linears = [(k, *dims[c[1]]) for k, c in zip(keys, cfg)]
    seed = 17 * rank
    # ---- calibration: fresh X / G_Y batches every step (scratch buffers), W fixed
    cal = plan_mod.Calibrator(linears, steps=args.calib_steps, params=params, device=dev)
    scratch = {}
    W = {}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i, (k, (layer, name, px, pw, pg)) in enumerate(zip(keys, cfg)):
        d_in, d_out = dims[name]
        W[k] = synth.operand_torch(d_out, d_in, pw, "W", 20000 + i, dev)
        x = scratch.setdefault(("x", d_in), torch.empty((T, d_in), dtype=torch.bfloat16, device=dev))
        gy = scratch.setdefault(("gy", d_out), torch.empty((T, d_out), dtype=torch.bfloat16, device=dev))
        for s in range(args.calib_steps):
            synth.operand_torch(T, d_in, px, "X", 1000003 * s + i + seed, dev, plant_seed=30000 + i, out=x)
            synth.operand_torch(T, d_out, pg, "GY", 1000003 * s + 500000 + i + seed, dev, plant_seed=40000 + i, out=gy)
            if world > 1:
                cal.record_sharded(s, k, x, W[k], gy, T * world)
            else:
                cal.record(s, k, x, W[k], gy)
    plan = cal.plan(level=args.level)
    torch.cuda.synchronize()
    calib_wall = time.perf_counter() - t0
    del scratch
    plan_path = os.path.join(ROOT, "gpurun_out", "plan_llama32_1b_stack.json")
    if rank == 0 and os.path.isdir(os.path.dirname(plan_path)):
        plan.save(plan_path)
    # ---- the step's tensors (the batch after calibration) and outputs
    lin = {}
    for i, (k, (layer, name, px, pw, pg)) in enumerate(zip(keys, cfg)):
        d_in, d_out = dims[name]
        lin[k] = dict(x=synth.operand_torch(T, d_in, px, "X", 7000000 + i + seed, dev, plant_seed=30000 + i),
                      w=W[k],
                      gy=synth.operand_torch(T, d_out, pg, "GY", 8000000 + i + seed, dev, plant_seed=40000 + i),
                      y=torch.empty(T, d_out, dtype=torch.bfloat16, device=dev),
                      gx=torch.empty(T, d_in, dtype=torch.bfloat16, device=dev),
                      gw=torch.empty(d_out, d_in, dtype=torch.float32, device=dev))
    flops_step = sum(2.0 * T * dims[c[1]][0] * dims[c[1]][1] * 3 for c in cfg)
    # per-linear parameters: the global k, or (--adaptive-k) the plan's per-layer k (DESIGN R16)
    lparams = {}
    for lp in plan.linears:
        k_lin = lp.oe_k if (args.adaptive_k and lp.oe_k > 0) else args.oe_k
        lparams[lp.name] = params if k_lin == args.oe_k else ah.Params(oe_k=k_lin, level=args.level)
    ws = ah.Workspace(max(ah.layer_workspace_bytes(T, d_in, d_out, plan.strategies(k), lparams[k])
                          for k, d_in, d_out in linears), dev)
    l2 = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    launches = [0]

    def step():
        works = []
        n = 0
        for k in keys:      # the plan fixes every GEMM's strategy: no runtime detection
            L = lin[k]
            ah.linear_layer(L["x"], L["w"], L["gy"], plan.strategies(k), lparams[k], out=(L["y"], L["gx"], L["gw"]),
                            ws=ws)
            n += ah.last_launch_count()
            if world > 1:
                works.append(ahd.allreduce_wgrad(L["gw"], async_op=True))
        for w_ in works:
            w_.wait()
        launches[0] = n

    def graph(fn):
        if world > 1 or args.no_graph:
            return fn
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            fn()
        torch.cuda.current_stream().wait_stream(side)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        torch.cuda.synchronize()
        return g.replay

    def timed(fn, steps, warmup, sampler=None):
        for _ in range(warmup):
            l2.zero_()
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if sampler:
            sampler.start()
        ms = 0.0
        for _ in range(steps):
            l2.zero_()
            s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_.record()
            fn()
            e_.record()
            torch.cuda.synchronize()
            ms += s_.elapsed_time(e_)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clocks = sampler.stop() if sampler else None
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms / steps, clocks

    step()
    torch.cuda.synchronize()
    run = graph(step)
    sampler = ClockSampler(local)
    ms, clocks = timed(run, args.steps, args.warmup, sampler)
    value = flops_step * world / (ms * 1e-3) / 1e12

    # one calibration pass over the step's 336 tensors, graph-replayed (a1 at config-5 scale)
    cal1 = plan_mod.Calibrator(linears, steps=1, params=params, device=dev)

    def calib_step():
        for k in keys:
            cal1.record(0, k, lin[k]["x"], lin[k]["w"], lin[k]["gy"])

    calib_step()
    torch.cuda.synchronize()
    ms_cal, _ = timed(graph(calib_step), args.steps, args.warmup)
    cal_bytes = sum(t.numel() * 2 for L in lin.values() for t in (L["x"], L["w"], L["gy"]))

    ms_cub = None
    if not args.no_cublas:
        def mm_f32(a, b, out):
            try:
                return torch.mm(a, b, out_dtype=torch.float32, out=out)
            except (RuntimeError, TypeError):
                return out.copy_(torch.mm(a, b, out_dtype=torch.float32))

        def step_cublas():
            works = []
            for k in keys:
                L = lin[k]
                torch.mm(L["x"], L["w"].t(), out=L["y"])
                torch.mm(L["gy"], L["w"], out=L["gx"])
                mm_f32(L["gy"].t(), L["x"], L["gw"])
                if world > 1:
                    works.append(dist.all_reduce(L["gw"], async_op=True))
            for w_ in works:
                w_.wait()
        ms_cub, _ = timed(graph(step_cublas), args.steps, args.warmup)

    if rank == 0:
        census = plan.census()
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "mxfp4", "data": "synthetic",
                "config": {"workload": "llama32_1b_stack_336gemm (BASELINE configs[4]: 16 layers x 7 linears x "
                                       "fwd/dgrad/wgrad) with calibration -> plan",
                           "tokens_per_gpu": T, "global_tokens": T * world,
                           "oe_k": ({"adaptive (DESIGN R16)": dict(Counter(lp.oe_k for lp in plan.linears))}
                                    if args.adaptive_k else args.oe_k), "level": args.level,
                           "hadamard_block": 32, "out_dtype": "bf16 (Y, G_X), fp32 (G_W)",
                           "patterns": "Table-1 census of Llama3.2-1B (P:190-195), synth.llama32_1b_census_patterns",
                           "l2": "flushed between steps (256 MiB write, untimed)",
                           "parallelism": f"dp{world} token-sharded, NCCL all-reduce of wgrad" if world > 1
                           else "single GPU"},
                "speedup_vs_cublas_bf16": (ms_cub / ms) if ms_cub else None,
                "cublas_bf16": {"ms_per_step": ms_cub, "value": flops_step * world / (ms_cub * 1e-3) / 1e12}
                if ms_cub else None,
                "calibration": {"steps": args.calib_steps, "wall_s_incl_batch_generation": round(calib_wall, 2),
                                "ms_per_calibration_step_336_tensors": ms_cal,
                                "GB_per_s": cal_bytes / (ms_cal * 1e-3) / 1e9,
                                "plan_census": census, "plan_file": "gpurun_out/plan_llama32_1b_stack.json"},
                "clocks": clocks, "gpu_launches": int(launches[0] * args.steps),
                "launch": "eager" if (world > 1 or args.no_graph) else "cuda_graph"}
        print(json.dumps(line), flush=True)


def profiled_traffic(workload, kernel):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `kernel`, averaged over the
    launches of one step, from the committed ncu capture (profiles/traffic.json, written by
    scripts/ncu_summary.py traffic); None when no capture of this workload exists."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d[workload][kernel]
        return {"bytes_per_launch": e["bytes_per_launch"], "algorithmic_bytes_per_launch": e.get("algorithmic"),
                "source": e["source"]}
    except (OSError, KeyError, ValueError):
        return None


def library_fp4(gemms, args, l2, as_graph, timed, dev):
    """The library's block-scaled FP4 GEMM next to ours on the step's MXFP4 GEMM shapes: cuBLASLt
    NVFP4 (E2M1 x E2M1, E4M3 scales per 16 along K — the same FP4 tensor-core rate as MXFP4, twice
    the scale factors; torch exposes no MXFP4 matmul) through F.scaled_mm, and k_gemm_mxf4_2sm alone
    (adahop_debug_gemm_mxf4_tcsf: one launch per GEMM, scales already in the tcgen05 layout), both
    with the step's output dtypes (bf16 Y / G_X, fp32 G_W), both timed like the step (CUDA graph,
    L2 flushed between steps). Speed-of-light context for the GEMM stage, not a baseline of the
    method. None where torch / cuBLASLt does not offer it."""
    import torch
    import paper_2604_02525_b200 as ah
    F = torch.nn.functional
    if not hasattr(F, "scaled_mm"):
        return None
    try:
        lib_ops, our_ops = [], []
        for g in gemms:
            if g["strategy"] == "BF16":
                continue
            M, N, K = g["M"], g["N"], g["K"]
            odt = torch.float32 if g["path"] == "wgrad" else torch.bfloat16
            ca = torch.randint(0, 256, (M, K // 2), dtype=torch.uint8, device=dev)
            cb = torch.randint(0, 256, (N, K // 2), dtype=torch.uint8, device=dev)
            sa = torch.ones((M, K // 16), device=dev).to(torch.float8_e4m3fn)
            sb = torch.ones((K // 16, N), device=dev).to(torch.float8_e4m3fn)
            lib_ops.append((ca.view(torch.float4_e2m1fn_x2), cb.view(torch.float4_e2m1fn_x2), sa, sb, odt))
            ea = torch.full((ah.debug_sf_bytes(M, K),), 127, dtype=torch.uint8, device=dev)
            eb = torch.full((ah.debug_sf_bytes(N, K),), 127, dtype=torch.uint8, device=dev)
            our_ops.append((ca, ea, cb, eb, torch.empty((M, N), dtype=odt, device=dev)))

        def step_lib():
            for a, b, sa, sb, odt in lib_ops:   # outputs come from the graph's private pool
                F.scaled_mm(a, b.t(), [sa], [F.ScalingType.BlockWise1x16], [sb], [F.ScalingType.BlockWise1x16],
                            [F.SwizzleType.SWIZZLE_32_4_4], [F.SwizzleType.SWIZZLE_32_4_4], None, odt)

        def step_ours():
            for ca, ea, cb, eb, out in our_ops:
                ah.debug_gemm_mxf4_tcsf(ca, ea, cb, eb, out)
        step_lib()
        step_ours()
        flops = sum(2.0 * g["M"] * g["N"] * g["K"] for g in gemms if g["strategy"] != "BF16")
        ms_lib, _ = timed(as_graph(step_lib), args.steps, args.warmup)
        ms_ours, _ = timed(as_graph(step_ours), args.steps, args.warmup)
        return {"kernel": "cuBLASLt NVFP4 block-scaled GEMM (torch F.scaled_mm, BlockWise1x16)",
                "ms_per_step": ms_lib, "TFLOP_s": flops / (ms_lib * 1e-3) / 1e12,
                "ours_gemm_only_ms_per_step": ms_ours, "ours_gemm_only_TFLOP_s": flops / (ms_ours * 1e-3) / 1e12,
                "ours_over_library": ms_lib / ms_ours,
                "ours_gemm_only_frac": flops / (ms_ours * 1e-3) / 1e12 / (load_peaks()["bf16"] * 4.0),
                "note": "the step's MXFP4 GEMM shapes and output dtypes; ours = k_gemm_mxf4_2sm alone (no outlier patch)"}
    except Exception as e:  # noqa: BLE001  (reported, not fatal: context only)
        return {"unavailable": f"{type(e).__name__}: {str(e)[:160]}"}


def roofline(dom, gemms, stage_tot, peaks, T, model=None, per_path=False, workload=None):
    """Achieved = algorithmic work of the dominant stage per step / its measured time (CUDA events
    recorded by the library around the stage on the launching stream) = the launch-weighted
    average of work per launch / duration per launch."""
    # the GEMM runs at max SM clock inside the step (clocks in the bench line), so its peak is the
    # BURST bf16 figure x 4 (nominal dense fp4 / bf16 = 9 / 2.25); sustained x 4 given beside it
    fp4_peak = peaks["bf16"] * 4.0
    if dom == "gemm_mxf4":
        work = sum(g["flops"] for g in gemms if g["strategy"] != "BF16")
        ach = work / (stage_tot[dom] * 1e-3) / 1e12
        n = sum(1 for g in gemms if g["strategy"] != "BF16")
        tr = profiled_traffic(workload, "k_gemm_mxf4_2sm")
        if tr:   # FP4 codes + E8M0 scales of both operands in, C out (bf16; fp32 G_W)
            tr["algorithmic_bytes_per_launch"] = sum((g["M"] + g["N"]) * g["K"] * 17 / 32 +
                                                     g["M"] * g["N"] * (4 if g["path"] == "wgrad" else 2)
                                                     for g in gemms if g["strategy"] != "BF16") / n
        return {"kernel": "k_gemm_mxf4_2sm (tcgen05 kind::mxf4, cta_group::2)", "bound": "tensor", "achieved": ach,
                "peak": fp4_peak, "unit": "TFLOP/s", "frac": ach / fp4_peak,
                "traffic": tr["bytes_per_launch"] if tr else None, "traffic_detail": tr,
                "launches_per_step": n, "flop_per_launch": work / n,
                "peak_src": f"{peaks['src']} bf16 burst {peaks['bf16']} TF/s x 4 (nominal fp4/bf16); "
                            f"vs sustained x 4 ({peaks['bf16_sustained'] * 4:.0f}): {ach / (peaks['bf16_sustained'] * 4):.3f}"}
    if dom == "quant":
        if per_path:
            # 2 B in + 0.5 B codes + 1/32 B scale per element of both operands of every GEMM
            by = sum((g["M"] + g["N"]) * g["K"] * (2 + 0.5 + 1 / 32) for g in gemms if g["strategy"] != "BF16")
        else:
            # layer step: every tensor read once (2 B) and written in both FP4 layouts
            by = 0.0
            for _, d_in, d_out in model["linears"]:
                for n_el in (T * d_in, d_out * d_in, T * d_out):
                    by += n_el * (2 + 2 * (0.5 + 1 / 32))
        ach = by / (stage_tot[dom] * 1e-3) / 1e9
        tr = profiled_traffic(workload, "k_quant_tc")
        if tr:
            tr["algorithmic_bytes_per_launch"] = by / len(model["linears"])
        return {"kernel": "k_quant_tc", "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": ach / peaks["hbm_gbs"], "traffic": tr["bytes_per_launch"] if tr else None,
                "traffic_detail": tr, "peak_src": peaks["src"]}
    if dom == "outlier":
        by = 0.0
        for g in gemms:
            if g["strategy"] == "OE_LEFT_IHT":
                by += g["N"] * g["K"] * 2
            elif g["strategy"] == "OE_RIGHT_IHT":
                by += g["M"] * g["K"] * 2
        ach = by / (stage_tot[dom] * 1e-3) / 1e9
        return {"kernel": "k_gemm_bf16 (outlier) + k_outlier_fold", "bound": "hbm", "achieved": ach,
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": ach / peaks["hbm_gbs"], "traffic": None,
                "peak_src": peaks["src"]}
    # FOID probe bytes: min(64, K) bf16 of every stored row of each OE operand
    by = 0.0
    for g in gemms:
        if g["strategy"] == "OE_LEFT_IHT":
            by += g["M"] * min(64, g["K"]) * 2
        elif g["strategy"] == "OE_RIGHT_IHT":
            by += g["N"] * min(64, g["K"]) * 2
    ach = by / (stage_tot[dom] * 1e-3) / 1e9
    return {"kernel": "k_foid_*", "bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": ach / peaks["hbm_gbs"], "traffic": None, "peak_src": peaks["src"]}


if __name__ == "__main__":
    main()

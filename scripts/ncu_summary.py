#!/usr/bin/env python
"""Summarise ncu output for profiles/ (runs here, no GPU).

  python scripts/ncu_summary.py launches <launches.csv>   # per-kernel share of ONE bench step
  python scripts/ncu_summary.py full <report.ncu-rep>     # key metrics of a --set full capture

The launch list holds every launch of the process; one step is the last
`adahop_linear_layer` x 7 sequence, i.e. the launches after the last torch kernel that
precedes our own (the L2 flush / input generation)."""
from __future__ import annotations

import csv
import re
import subprocess
import sys
from collections import OrderedDict

# hot-path kernels of the layer step (calibration kernels excluded: bench.py times them after the step)
OURS = re.compile(r"mxf4x2::|bf16g::|k_quant_tc|k_gemm_|k_foid|k_oe_|k_outlier|k_iht|k_or_fold")


def short(name: str) -> str:
    name = re.sub(r"\(.*$", "", name)
    name = name.replace("void ", "")
    return name.strip()


def launches(path: str, steps: int = 1) -> None:
    rows = [r for r in csv.reader(open(path)) if len(r) == 15 and r[0].isdigit()]
    seq = [(int(r[0]), r[4], float(r[14])) for r in rows if r[12] == "gpu__time_duration.sum"]
    ours = [i for i, (_, n, _) in enumerate(seq) if OURS.search(n)]
    if not ours:
        print("no adahop launches found")
        return
    # last contiguous block of our kernels = the last step
    end = ours[-1]
    start = end
    while start - 1 >= 0 and OURS.search(seq[start - 1][1]):
        start -= 1
    step = seq[start:end + 1]
    agg: "OrderedDict[str, list]" = OrderedDict()
    for _, n, ns in step:
        k = short(n)
        a = agg.setdefault(k, [0, 0.0])
        a[0] += 1
        a[1] += ns / 1000.0
    tot = sum(v[1] for v in agg.values())
    print(f"one bench step ({len(step)} launches of our kernels), ncu gpu__time_duration.sum, cold cache, serialised")
    for k, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k[:70]:70s} {n:4d} launches {us:10.1f} us {100 * us / tot:5.1f}%")
    print(f"total {tot:.1f} us over {len(step)} launches")


KEYS = [
    r"^gpu__time_duration\.sum$", r"^dram__bytes_read\.sum$", r"^dram__bytes_write\.sum$",
    r"^dram__throughput\.avg\.pct_of_peak_sustained_elapsed$", r"^gpu__dram_throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^lts__t_bytes\.sum$", r"^lts__throughput\.avg\.pct_of_peak_sustained_elapsed$",
    r"^sm__throughput\.avg\.pct_of_peak_sustained_elapsed$", r"^sm__inst_executed_pipe_uniform",
    r"^sm__pipe_tensor.*pct_of_peak_sustained_(active|elapsed)$", r"^sm__pipe_shared_cycles_active",
    r"^launch__grid_size$", r"^launch__block_size$", r"^launch__registers_per_thread$",
    r"^launch__shared_mem_per_block_dynamic$", r"^sm__warps_active\.avg\.pct_of_peak_sustained_active$",
    r"^smsp__cycles_active\.avg$", r"^sm__cycles_elapsed\.avg$", r"^sm__cycles_elapsed\.avg\.per_second$",
    r"^dram__cycles_elapsed\.avg\.per_second$",
]


def full(path: str) -> None:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        name = r[hdr.index("Kernel Name")]
        print(f"kernel: {short(name)}  grid {r[hdr.index('Grid Size')]} block {r[hdr.index('Block Size')]}")
        for i, h in enumerate(hdr):
            if any(re.search(k, h) for k in KEYS) and r[i] not in ("", "n/a"):
                print(f"  {h:75s} {r[i]:>16s} {units[i]}")
        try:
            rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
            u = units[hdr.index("dram__bytes_read.sum")]
            print(f"  traffic (read+write) = {rd + wr:.3f} {u}")
        except ValueError:
            pass


def traffic(path: str, workload: str, out: str) -> None:
    """Per-launch DRAM bytes (read + write) of our kernels in the LAST step of a launch list
    captured with --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum;
    merged into `out` (profiles/traffic.json) under `workload`."""
    import json
    import os
    rows = [r for r in csv.reader(open(path)) if len(r) == 15 and r[0].isdigit()]
    per: "OrderedDict[int, dict]" = OrderedDict()
    for r in rows:
        d = per.setdefault(int(r[0]), {"name": r[4]})
        v = float(r[14].replace(",", ""))
        unit = r[13]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1, "us": 1e3, "ms": 1e6}.get(unit, 1)
        d[r[12]] = v * scale
    seq = list(per.values())
    ours = [i for i, d in enumerate(seq) if OURS.search(d["name"])]
    end = ours[-1]
    start = end
    while start - 1 >= 0 and OURS.search(seq[start - 1]["name"]):
        start -= 1
    step = seq[start:end + 1]
    res = {}
    for key in ("k_gemm_mxf4_2sm", "k_quant_tc", "k_gemm_bf16", "k_foid_select", "k_oe_gather"):
        ls = [d for d in step if key in d["name"]]
        if not ls:
            continue
        by = [d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in ls]
        ns = [d.get("gpu__time_duration.sum", 0) for d in ls]
        res[key] = {"launches_per_step": len(ls), "bytes_per_launch": sum(by) / len(ls),
                    "ncu_ns_per_launch": sum(ns) / len(ls),
                    "source": f"ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum (one step), {os.path.basename(path)}"}
        print(f"{key:20s} {len(ls):3d} launches, {sum(by) / len(ls) / 1e6:10.2f} MB/launch, "
              f"{sum(ns) / len(ls) / 1e3:8.1f} us/launch (ncu, serialised)")
    allres = json.load(open(out)) if os.path.exists(out) else {}
    allres[workload] = res
    with open(out, "w") as f:
        json.dump(allres, f, indent=1)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "traffic":
        traffic(path, sys.argv[3], sys.argv[4])
    elif mode == "launches":
        launches(path)
    else:
        full(path)

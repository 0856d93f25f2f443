"""Per-unit counters of the config-4 run kernels for bench.py's roofline.

bench.py reports the run kernels against their actual limiter, instruction
issue: achieved = executed warp instructions / time.  The instruction and
DRAM counts per cost unit (one FGP inner iteration of one 256x256 problem,
+2 per problem; the unit of the device work queue, csrc/common.cuh) are
static properties of each kernel's code; this tool measures them once with
ncu, and bench.py multiplies them by the units each kernel finished in the
live run (psb_queue_stats) and divides by the live CUDA-event time.

Workload: the bench's config-4 timed segment on a subset of the problems
(W = 5 warm-up outer iterations, then K = 20), once with the clusters only
(PSB_NO_SMWORK=1), once with the SM workers only (PSB_SM_ONLY=1) and once
with 8-CTA clusters only (PSB_CLUSTER8=1 PSB_NO_SMWORK=1).

On the GPU box:

  for m in cluster sm cluster8; do
    ncu --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
gpu__time_duration.sum,sm__inst_issued.avg.pct_of_peak_sustained_active,\
sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active \
        --clock-control none -k regex:fgp_.*_run_kernel --csv \
        --log-file gpurun_out/ctr_$m.csv python tools/run_kernel_counters.py --mode $m \
        > gpurun_out/ctr_$m.json
  done
  python tools/run_kernel_counters.py --emit gpurun_out   # -> profiles/r02_run_kernel_counters.json
"""

import argparse
import csv
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
N, W, K = 1184, 5, 20  # 1184 = 8 x 148 problems


def run(mode):
    os.environ["PSB_SM_ONLY" if mode == "sm" else "PSB_NO_SMWORK"] = "1"
    os.environ["PSB_CLUSTER8"] = "1" if mode == "cluster8" else "0"
    if mode == "sm":  # the workers' share of the SMs in the bench's run (L2-resident working sets)
        os.environ.setdefault("PSB_SM_WORKERS", "28")
    import torch
    import paper_2411_00688_b200 as psb
    from paper_2411_00688_b200 import _lib as L
    from paper_2411_00688_b200 import batched, phantoms
    idx = np.linspace(0, 4095, N).astype(int)
    b = phantoms.config4_batch(idx, 256)
    coins = batched.coin_table(0.1, idx, W + K)
    s = psb.BatchedTvDenoise(b, 0.1, 50, precision="fp32")
    s.run_proxskip(coins[:W], 1.0, 0.1)          # launch 1 (warm-up)
    s.run_proxskip(coins[W:], 1.0, 0.1)          # launch 2 (the measured one)
    torch.cuda.synchronize()
    qs = (L.C.c_double * 6)()
    L.call("psb_queue_stats", qs)
    units = {"cluster": qs[1], "sm": qs[3], "cluster8": qs[5]}[mode]
    print(json.dumps({"mode": mode, "problems": N, "warmup": W, "steps": K, "units": units,
                      "prox_calls": int(coins[W:].sum())}))


def _ncu_rows(path):
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rows = list(csv.DictReader(lines))
    return rows


def emit(d):
    out = {"source": "ncu --metrics (tools/run_kernel_counters.py), second launch of each kernel",
           "unit": "one FGP inner iteration of one 256x256 problem (+2 per problem)"}
    for mode, key, kname in (("cluster", "cluster", "fgp_cluster_run_kernel"),
                             ("sm", "sm_worker", "fgp_sm_run_kernel"),
                             ("cluster8", "cluster8", "fgp_cluster8_run_kernel")):
        if not os.path.exists(os.path.join(d, f"ctr_{mode}.json")):
            continue
        meta = json.loads(open(os.path.join(d, f"ctr_{mode}.json")).read().strip().splitlines()[-1])
        rows = [r for r in _ncu_rows(os.path.join(d, f"ctr_{mode}.csv"))
                if kname in r["Kernel Name"]]
        ids = sorted({int(r["ID"]) for r in rows})
        last = [r for r in rows if int(r["ID"]) == ids[-1]]
        m = {r["Metric Name"]: float(r["Metric Value"].replace(",", "")) for r in last}
        u = float(meta["units"])
        out[key] = {
            "inst_per_unit": m["smsp__inst_executed.sum"] / u,
            "dram_bytes_per_unit": (m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]) / u,
            "ns_per_unit_serialised": m["gpu__time_duration.sum"] / u,
            "issue_active_pct": m.get("sm__inst_issued.avg.pct_of_peak_sustained_active"),
            "fma_pipe_pct": m.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
            "units": u, "workload": meta}
    out["issue_active_pct"] = out["cluster"]["issue_active_pct"]
    path = os.path.join(ROOT, "profiles", "r02_run_kernel_counters.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", choices=["cluster", "sm", "cluster8"])
    ap.add_argument("--emit")
    a = ap.parse_args()
    if a.emit:
        emit(a.emit)
    else:
        run(a.mode)

"""Benchmark: BASELINE config 4 -- batched ProxSkip TV denoising.

4096 independent 256x256 problems (seeded random-ellipse/rectangle phantoms,
noise sigma_i ~ U[0.05, 0.15], alpha = 0.1, gamma = 1, p = 0.1 per-problem
Philox coin streams, FGP-50 inner iterations), sharded over N GPUs (one
process per GPU, contiguous problem blocks, no collective on the data path).
A "step" is one outer ProxSkip iteration over the whole batch.  The native
driver runs the K timed steps as ONE segment: fgp_cluster_run_kernel (16-CTA
clusters, one problem each at a time, all of its coin-fired prox calls back to
back with the FGP state in registers) plus fgp_sm_run_kernel on the SMs the
clusters leave, each problem advanced by exactly K outer iterations.  W
warm-up steps are outer iterations 0..W-1 of the run; the K timed steps are
iterations W..W+K-1 (default W+K = 300, the full config-4 run).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Prints one JSON line (rank 0).  See DESIGN.md "Measurement" for every field.
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_PROBLEMS = 4096
SIDE = 256
ALPHA = 0.1
P = 0.1
INNER = 50
E2E_REPS = 3
RUN_LEN = 300
BYTES_FGP_MOM = 28   # fp32 per pixel-iteration: x + q_k(2) + q_{k-1}(2) read, q_{k+1}(2) write
BYTES_FGP_FIRST = 20  # first inner iteration (beta = 0): no q_{k-1} read
CLUSTER = os.environ.get("PSB_NO_CLUSTER", "0") != "1"
if CLUSTER:
    KERNEL = ("fgp_cluster_run_kernel<float> (+ fgp_sm_run_kernel on the 36 SMs the clusters "
              "leave): the whole timed run segment in ONE launch each; a 16-CTA cluster runs its "
              "problems' coin-fired prox calls back to back (skips + 50 FGP iterations + post) "
              "with z, q in registers and x, b, h in shared memory; the 28 B/px-iter of the "
              "streaming formulation stay on-chip / in L2, so frac > 1 is expected; time = both "
              "kernels (events around the pair)")
    # ncu dram__bytes_read.sum + dram__bytes_write.sum of fgp_cluster_run_kernel per launch,
    # per problem in the launch (profiles/r01_launches_bench_run.csv)
    TRAFFIC_PER_PROBLEM_LAUNCH = 2.4e6
else:
    KERNEL = "fgp2d_iter_kernel<float,4> (streaming, one launch per inner iteration)"
    # profiles/r01_fgp2d_iter_ncu_details.csv: 795 MB per launch at 422 problems
    TRAFFIC_PER_PROBLEM = 795e6 / 422 * INNER
METRIC = "ProxSkip TV outer iter/s (config 4: 4096 x 256^2 batch, FGP-50, p=0.1)"
WORKLOAD = "config4: batched ProxSkip TV denoising, 4096 x 256x256, alpha=0.1, p=0.1, FGP-50"


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def _gen(idx):
    from paper_2411_00688_b200 import phantoms
    return phantoms.config4_batch(idx, SIDE)


def make_inputs(indices, procs=None):
    procs = procs or min(8, os.cpu_count() or 1)
    chunks = [c for c in np.array_split(np.asarray(indices), procs * 4) if len(c)]
    with mp.get_context("fork").Pool(procs) as pool:
        parts = pool.map(_gen, chunks)
    return np.concatenate(parts, axis=0)


# -- CPU baseline: the oracle (numpy restatement of the reference) -------------

def _oracle_problem(arg):
    """Run problem i's outer loop with the oracle; time iterations W..W+K-1."""
    i, warm, steps = arg
    from oracle import imgskip_cpu as oc
    from paper_2411_00688_b200 import phantoms
    b = phantoms.config4_problem(int(i), SIDE)[1]
    pr = oc.make_recon(oc.identity_op(b.shape), b, ALPHA, inner=INNER)
    marks = {}

    def obs(k, x, n, th):
        if k == warm - 1:
            marks["t0"] = time.perf_counter()

    t_begin = time.perf_counter()
    oc.proxskip(pr.grad, pr.prox, np.zeros_like(b), None, 1.0, P, int(i), warm + steps, obs)
    return time.perf_counter() - marks.get("t0", t_begin)


def cpu_baseline(warm, steps, procs):
    """The reference algorithm (oracle port, float64 numpy) on ``procs`` host
    processes, one config-4 problem each (indices spread over 0..4095),
    timing the same outer iterations W..W+K-1 as the GPU arm.  Returns the
    rate scaled to the 4096-problem batch (batch outer iter/s)."""
    idx = np.linspace(0, N_PROBLEMS - 1, procs).astype(int)
    env = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS")}
    os.environ["OMP_NUM_THREADS"] = os.environ["OPENBLAS_NUM_THREADS"] = "1"
    try:
        with mp.get_context("fork").Pool(procs) as pool:
            per = pool.map(_oracle_problem, [(int(i), warm, steps) for i in idx])
    finally:
        for k, v in env.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    wall = max(per)
    value = procs * steps / wall / N_PROBLEMS
    return {
        "value": value,
        "unit": "outer-iter/s (4096-problem batch)",
        "cores": procs,
        "kind": "port",
        "sample": f"{procs} of 4096 problems (one per host process, 1 thread each), outer "
                  f"iterations {warm}..{warm + steps - 1} of the {RUN_LEN}-iteration run, "
                  f"oracle/imgskip_cpu.py float64 numpy; slowest process {wall:.2f}s; "
                  f"rate scaled x{procs}/4096 to the full batch",
    }


# -- clocks sampled during the timed region -------------------------------------

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.dev}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            f = [c.strip() for c in line.split(",")]
            if len(f) >= 9:
                rows.append(f)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[j] for r in rows for j in range(4) if r[5 + j].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(rows[0][2]) if rows[0][2].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# -- arms -------------------------------------------------------------------------

def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=None)
    return world, rank, local


def run_reference(args):
    """The reference's algorithm on the host cores (rank 0 only under torchrun)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return 0
    procs = os.cpu_count() or 1
    r = cpu_baseline(args.warmup, args.steps, procs)
    v = r["value"]
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": r["unit"],
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 / v if v else None, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded phantoms, SURVEY D3)",
        "config": {"workload": WORKLOAD, "problems": N_PROBLEMS, "side": SIDE, "inner": INNER,
                   "p": P, "alpha": ALPHA, "device": "host CPU"},
        "cpu_baseline": {"value": v, "unit": r["unit"], "cores": procs, "kind": "port",
                         "sample": r["sample"]},
        "e2e": {"value": v, "unit": r["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_gpu(args):
    import torch
    import paper_2411_00688_b200 as psb
    from paper_2411_00688_b200 import batched

    world, rank, local = dist_init()
    torch.cuda.set_device(local)
    dev = torch.cuda.current_device()
    idx = batched.shard_indices(N_PROBLEMS, rank, world)
    b_host = make_inputs(idx)
    coins = batched.coin_table(P, idx, args.warmup + args.steps)
    solver = psb.BatchedTvDenoise(b_host, ALPHA, INNER, precision="fp32")
    HW = SIDE * SIDE

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
            torch.cuda.synchronize()

    # ---- device-resident throughput: warm-up steps, then K timed steps ----
    solver.reset()
    solver.run_proxskip(coins[:args.warmup], 1.0, P)
    fgp_t = np.zeros(args.steps)
    sync_all()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk:
        e0.record(stream)
        solver.run_proxskip(coins[args.warmup:], 1.0, P, fgp_time=fgp_t)
        e1.record(stream)
        sync_all()
    solver.check_finite()
    t_local = e0.elapsed_time(e1) / 1000.0
    timed = coins[args.warmup:]
    active = timed.sum(axis=1)                       # coin-fired problems per step
    fgp_bytes = active * HW * (BYTES_FGP_FIRST + (INNER - 1) * BYTES_FGP_MOM)
    n_fired_steps = int(np.count_nonzero(active))
    if CLUSTER:
        # one fgp_cluster_run_kernel launch for the K timed steps, plus one
        # fgp_sm_run_kernel launch on the SMs the clusters leave
        launches = 1 + (os.environ.get("PSB_NO_SMWORK", "0") != "1")
    else:
        launches = args.steps + n_fired_steps * (INNER + 1)
    stats = np.array([t_local, fgp_t.sum(), float(fgp_bytes.sum()), float(active.sum())])
    if world > 1:
        import torch.distributed as dist
        ts = torch.tensor(stats, device="cuda", dtype=torch.float64)
        tmax = ts.clone()
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
        dist.all_reduce(ts, op=dist.ReduceOp.SUM)
        t_job = float(tmax[0])
        sums = ts.cpu().numpy()
    else:
        t_job = t_local
        sums = stats
    value = args.steps / t_job                        # batch outer iterations / s
    inner_rate = sums[3] * INNER / t_job               # problem-inner-iterations / s
    fgp_time_local = fgp_t.sum()
    achieved = fgp_bytes.sum() / fgp_time_local / 1e9 if fgp_time_local > 0 else 0.0
    peak, peak_kind = _peaks()

    # ---- e2e: the public API with host buffers, copies inside the region ----
    # (the device-resident solver above is released first; its blocks stay in
    # torch's caching allocator, as in any process that has run a solve before)
    del solver
    b_pin = torch.from_numpy(b_host).pin_memory()
    # untimed warm-up of the e2e path on a slice (its one-time host set-up:
    # pinned staging buffers, copy stream, stream-memop entry points)
    # The result lands in a page-locked host buffer allocated up front, like
    # the pinned input (a pageable one costs a staged copy plus first-touch
    # page faults on 1 GB inside the timed call: e2e varied 290-500 it/s).
    x_pin = torch.empty(b_pin.shape, dtype=torch.float32).pin_memory()
    nw = min(len(idx), 512)
    psb.run_proxskip_batched(b_pin[:nw], ALPHA, P, idx[:nw], args.warmup, INNER, precision="fp32",
                             out=x_pin[:nw])
    # Three timed calls, the median reported: the device part of a call is
    # stable to 0.1 ms (CUDA-event timeline of the copies, PSB_DEBUG_E2E=1),
    # but the host wall clock of a single call sometimes stalls for 0.1-1 s
    # (seen in ~1 of 8 calls, with the device timeline unchanged).
    e2e_samples = []
    for _ in range(E2E_REPS):
        sync_all()
        t0 = time.perf_counter()
        x_e2e, counts = psb.run_proxskip_batched(b_pin, ALPHA, P, idx, args.warmup + args.steps,
                                                 INNER, precision="fp32", out=x_pin)
        assert x_e2e.device.type == "cpu"
        e2e_samples.append(time.perf_counter() - t0)
    t_e2e_local = float(np.median(e2e_samples))
    if world > 1:
        tt = torch.tensor([t_e2e_local], device="cuda", dtype=torch.float64)
        torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
        t_e2e = float(tt[0])
    else:
        t_e2e = t_e2e_local
    n_e2e = args.warmup + args.steps
    h2d = b_host.nbytes * world / n_e2e
    d2h = x_e2e.numel() * x_e2e.element_size() * world / n_e2e

    if rank != 0:
        return 0
    procs = os.cpu_count() or 1
    cpu = cpu_baseline(args.warmup, args.steps, procs) if (world == 1 and not args.no_cpu) else None
    line = {
        "metric": METRIC, "value": value, "unit": "outer-iter/s (4096-problem batch)",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * t_job / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (seeded random-shape phantoms, SURVEY D3; no public dataset)",
        "config": {"workload": WORKLOAD, "problems": N_PROBLEMS, "side": SIDE, "inner": INNER,
                   "p": P, "alpha": ALPHA, "parallelism": f"problem-shard x{world}",
                   "l2": "inputs larger than L2 (~10 GB of state per GPU vs 126 MB L2)"},
        "fgp_inner_iter_per_s": inner_rate,
        "fgp_mpx_iter_per_s": inner_rate * HW / 1e6,
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak,
                     "traffic": (TRAFFIC_PER_PROBLEM_LAUNCH * len(idx) if CLUSTER else
                                 TRAFFIC_PER_PROBLEM * float(active.sum()) / max(n_fired_steps, 1)),
                     "kernel": KERNEL,
                     "bytes_per_unit": "28 B/pixel-iteration (20 B at the first inner iteration), "
                                       "SURVEY 8(d); x units = the timed steps' coin-fired "
                                       "problem-prox calls x 65536 px x 50 inner iterations "
                                       "(one launch for all of them on the cluster path)",
                     "peak_source": peak_kind},
        "cpu_baseline": cpu,
        "e2e": {"value": n_e2e / t_e2e, "unit": "outer-iter/s (4096-problem batch)",
                "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "path": "paper_2411_00688_b200.run_proxskip_batched (pinned host in, pinned host out)",
                "timing": f"host wall clock per call, median of {E2E_REPS} calls (max over ranks)",
                "samples_s": [round(t, 5) for t in e2e_samples]},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=295)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())

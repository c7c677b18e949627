"""Benchmark of the mQO hot path: the fused batched PGA gradient step.

Workload (BASELINE.json configs[3], per GPU): MaxCut with the paper's
perturbed-bias objective f_B (lambda = 0.001) on the synthetic
Barabasi-Albert graph BA(n=1e6, m'=5, seed 1) -- nnz = 2m = 9,999,950 --
with B = 128 independent chains per GPU (1024 over 8 GPUs), preset
alpha = 0.0025, beta = 0.8.  One "step" = one fused PGA iteration
(gather-SpMM over the CSR + f_B epilogue + momentum + box clip + max|dx|)
of every chain.  Metric: edge-chain updates / s = nnz * B / step time.

* value        device-timed (CUDA events on the batch stream), inputs
               resident in HBM; the 1 GB chain state is > L2, so no flush.
* e2e          the same metric through the C-ABI call a user makes
               (mqo_run_trajectories) with pinned host buffers: every step
               copies the B initial states in, runs a bounded trajectory
               (max_iters = 1000) and copies the final states out.
* roofline     achieved algorithmic GB/s of the fused kernel vs the
               measured HBM copy peak (MEASURED_PEAKS.json).
* cpu_baseline the reference's own CPU step (oracle/_ref, else the oracle
               port) on the box's host cores, bounded sample.
``--impl reference`` times that CPU implementation alone (the driver's
reference arm).  Multi-GPU: one process per GPU (torchrun), chains sharded
with no data-path collective (weak scaling), time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_VERTICES = 1_000_000
M_ATTACH = 5
GRAPH_SEED = 1
CHAINS_PER_GPU = 128
ALPHA, BETA, LAMBDA = 0.0025, 0.8, 0.001
E2E_ITERS = 1000
METRIC = "edge-chain updates/sec of mQO gradient step"
UNIT = "edge-chain updates/s"


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def load_traffic():
    """dram read+write bytes per launch of the fused kernel, from the
    committed ncu --set full summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "latest_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi sampling of SM clocks / throttle reasons during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            t0 = time.time()  # nvidia-smi needs a moment before its first row
            while not self.rows and time.time() - t0 < 3.0:
                time.sleep(0.05)
            self.rows.clear()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def bytes_per_step(n: int, nnz: int, B: int) -> int:
    """Algorithmic HBM bytes of one fused step:
    CSR offsets + indices once, plus per chain the gathered neighbour
    values (no-reuse model) and read x, v / write x, v per vertex."""
    return 8 * (n + 1) + 4 * nnz + B * (8 * nnz + 32 * n)


# ------------------------------------------------------------ CPU arms
def cpu_step_rate(threads: int, steps_per_thread: int):
    """Reference step() (oracle/_ref when built, else the oracle port) on
    `threads` host threads, one chain each; returns (rate, kind, sample)."""
    import oracle
    kind = "reference" if oracle.have_ref() else "port"
    L = oracle.load("ref" if kind == "reference" else "oracle")
    g = L.generate_ba(N_VERTICES, M_ATTACH, GRAPH_SEED)
    nnz = 2 * g.m
    rng = np.random.default_rng(123)
    xs = [rng.uniform(-1.0, 1.0, g.n) for _ in range(threads)]
    vs = [np.zeros(g.n) for _ in range(threads)]

    def work(i):
        x, v = xs[i], vs[i]
        for _ in range(steps_per_thread):
            x, v = L.step(g, oracle.PERTURBED_BIAS, LAMBDA, x, v, ALPHA, BETA)

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    dt = time.perf_counter() - t0
    rate = steps_per_thread * threads * nnz / dt
    sample = (f"{threads} chains x {steps_per_thread} reference step() calls on BA(1e6,5) f_B, "
              f"one chain per host thread ({dt:.1f} s)")
    return rate, kind, sample, g


def run_reference(args, rank: int, world: int):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    import oracle
    kind = "reference" if oracle.have_ref() else "port"
    L = oracle.load("ref" if kind == "reference" else "oracle")
    g = L.generate_ba(N_VERTICES, M_ATTACH, GRAPH_SEED)
    nnz = 2 * g.m
    rng = np.random.default_rng(123)
    xs = [rng.uniform(-1.0, 1.0, g.n) for _ in range(threads)]
    vs = [np.zeros(g.n) for _ in range(threads)]

    def one_step():  # one reference step() per thread, all threads in parallel
        def work(i):
            xs[i], vs[i] = L.step(g, oracle.PERTURBED_BIAS, LAMBDA, xs[i], vs[i], ALPHA, BETA)
        ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()

    for _ in range(args.warmup):
        one_step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one_step()
    dt = time.perf_counter() - t0
    value = args.steps * threads * nnz / dt
    sample = (f"per step: {threads} chains (one per host thread) x 1 reference step() on "
              f"BA(1e6,5) f_B")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * dt / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "MaxCut f_B on BA(n=1e6, m=5), reference CPU step()",
                   "chains": threads, "graph": "ba:1000000:5 seed 1",
                   "nnz": int(nnz), "alpha": ALPHA, "beta": BETA, "lambda": LAMBDA},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ GPU arm
def run_ours(args, rank: int, world: int, local_rank: int):
    import torch
    import paper_2605_06921_b200 as P

    dist = world > 1
    if dist:
        import torch.distributed as tdist
    torch.cuda.set_device(local_rank)
    device = local_rank
    B = CHAINS_PER_GPU
    g = P.generate(P.BaSpec(N_VERTICES, M_ATTACH), GRAPH_SEED, device=device)
    n, nnz = g.n(), 2 * g.m()
    batch = P.ChainBatch(g, B)
    # chains rank*B .. rank*B+B-1 of the global batch, seeded per chain
    X = np.empty((B, n))
    for c in range(B):
        X[c] = np.random.default_rng(1000 + rank * B + c).uniform(-1.0, 1.0, n)
    batch.set_x(X)
    batch.zero_v()
    spec, cfg = P.PerturbedBias(LAMBDA), P.OptimizerConfig(alpha=ALPHA, beta=BETA)
    stream = torch.cuda.ExternalStream(batch.stream, device=device)

    for _ in range(args.warmup):
        batch.step(spec, cfg)
    batch.sync()
    if dist:
        tdist.barrier()
    torch.cuda.synchronize()
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device) as clk:
        start.record(stream)
        for _ in range(args.steps):
            batch.step(spec, cfg)
        end.record(stream)
        end.synchronize()
    torch.cuda.synchronize()
    if dist:
        tdist.barrier()
    ms = start.elapsed_time(end)
    red_dev = f"cuda:{device}" if (not dist or tdist.get_backend() == "nccl") else "cpu"
    t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    if dist:
        tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ms_max = float(t.item())
    per_step_s = ms_max / 1e3 / args.steps
    value = world * B * nnz / per_step_s

    # roofline of the fused kernel (one launch per step)
    peak, peak_kind = load_peaks()
    alg = bytes_per_step(n, nnz, B)
    achieved = alg / (ms / 1e3 / args.steps) / 1e9
    traffic = load_traffic()

    # e2e through the C-ABI with pinned host buffers
    e2e_steps = 3
    hx = torch.empty((B, n), dtype=torch.float64, pin_memory=True)
    hx.numpy()[:] = X
    hout = torch.empty((B, n), dtype=torch.float64, pin_memory=True)
    it_total = 0
    ecfg = P.OptimizerConfig(alpha=ALPHA, beta=BETA, max_iters=E2E_ITERS)
    import ctypes as C
    from paper_2605_06921_b200 import _lib

    def e2e_once():
        nonlocal it_total
        _lib.check(_lib.lib.mqo_batch_set_x(batch._h, C.cast(hx.data_ptr(), _lib._D)))
        it, rs = batch.run_trajectories(spec, ecfg)
        _lib.check(_lib.lib.mqo_batch_get_x(batch._h, C.cast(hout.data_ptr(), _lib._D)))
        return int(it.sum())

    e2e_once()  # warm-up
    if dist:
        tdist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        it_total += e2e_once()
    e2e_dt = time.perf_counter() - t0
    te = torch.tensor([e2e_dt, float(it_total)], dtype=torch.float64, device=red_dev)
    if dist:
        tmax = te[:1].clone()
        tsum = te[1:].clone()
        tdist.all_reduce(tmax, op=tdist.ReduceOp.MAX)
        tdist.all_reduce(tsum, op=tdist.ReduceOp.SUM)
        e2e_dt, it_all = float(tmax.item()), float(tsum.item())
    else:
        it_all = float(it_total)
    e2e_value = it_all * nnz / e2e_dt

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        rate, kind, sample, _ = cpu_step_rate(threads, args.cpu_steps)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": kind, "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": "MaxCut f_B (lambda=0.001) fused PGA step on BA(n=1e6, m=5), "
                                   f"{B} chains per GPU",
                       "graph": "ba:1000000:5 seed 1", "n": n, "nnz": nnz,
                       "chains_per_gpu": B, "global_chains": B * world,
                       "alpha": ALPHA, "beta": BETA, "parallelism": f"chains sharded x{world}",
                       "l2": "state (1 GB per buffer) > 126 MB L2; no flush needed",
                       "e2e": f"mqo_run_trajectories, max_iters={E2E_ITERS}, pinned host x in/out"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "traffic": (traffic or {}).get("dram_bytes_per_launch"),
                         "algorithmic_bytes_per_launch": alg,
                         "kernel": "k_pass<PerturbedBias,4,kStep,Tune<4,3,1>>"},
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": int(hx.numel() * 8),
                    "d2h_bytes_per_step": int(hout.numel() * 8 + 2 * 4 * B)},
            "gpu_launches": args.steps,
            "clocks": clk.summary(),
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=40)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: several ranks sharing fewer GPUs (gloo for the timing
    # reductions); production runs one rank per GPU over NCCL
    backend = os.environ.get("MQO_BENCH_BACKEND", "nccl")
    if backend != "nccl":
        import torch
        local_rank %= max(1, torch.cuda.device_count())
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            tdist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
        else:
            tdist.init_process_group(backend)
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as tdist
            tdist.destroy_process_group()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Benchmark of the B200 IPM hot path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2_lasso] [--impl ours|reference]

A *step* is one complete solve (Algorithm 1 from the unit start point to
termination at ε_feas = 1e-8) of the configured synthetic instance.  The
headline metric is IPM iterations per second of the whole job; solve time per
instance is reported alongside.  The default workload is BASELINE.json
configs[1] (C2: lasso with 50k features × 200k rows, FP32 LDL' + FP64
iterative refinement).

value     — device-resident inputs (problem uploaded once), CUDA-event timed per
            step on the solver stream, L2 flushed between steps (256 MiB write).
e2e       — through the public API with host buffers: Solver.update_data(q, b)
            (host equilibration + H2D upload) + Solver.solve() (D2H of x, z, s),
            CUDA-event timed on the same stream.
roofline  — the dominant kernel class (supernodal triangular solves or the
            numeric factorisation), algorithmic bytes / event-timed duration.
cpu_baseline — the CPU oracle (oracle/, a restatement of the reference solver;
            its parity is pinned bit-for-bit to the reference's golden
            fixtures) on the same instance, single thread, bounded sample.

Multi-GPU (torchrun): a single problem does not shard, so N>1
runs N independent replicas (weak scaling), timed as the max over ranks.
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

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ipm_iterations_per_s"
UNIT = "iter/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2_lasso")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--eps", type=float, default=1e-8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-iters", type=int, default=200,
                    help="cap on IPM iterations per CPU solve (bounded sample)")
    ap.add_argument("--cpu-worker", action="store_true", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-max-iters", type=int, default=0, help=argparse.SUPPRESS)
    ap.add_argument("--cpu-solves", type=int, default=1, help=argparse.SUPPRESS)
    ap.add_argument("--cpu-impl", default="reference", help=argparse.SUPPRESS)
    ap.add_argument("--cpu-procs", type=int, default=1, help=argparse.SUPPRESS)
    ap.add_argument("--cpu-instances", type=int, default=0,
                    help="batched configs: instances in one CPU sample (0: 256 for the cpu_baseline "
                         "key, every instance for --impl reference)")
    return ap.parse_args()


def workload(config):
    from paper_2412_19027_b200 import generators as G
    spec = G.CONFIGS[config]
    desc = {"c1_lp": "C1 random sparse LP n=2000 m=4000 (1000 zero + 3000 nonneg)",
            "c2_lasso": "C2 lasso 50k features x 200k rows (n=300k, m=300k), fp32 LDL' + fp64 IR",
            "c3_socp": "C3 SOCP 100k cones dim U{3..10}",
            "c4_exppow": "C4 50k exp + 20k pow cones",
            "c5a_psd": "C5a 10k PSD cones side 6",
            "c5b_mpc": "C5b 2048 independent MPC QPs (nx=8, nu=3, N=10), one CTA per instance, "
                       "instances sharded over the GPUs"}[config]
    return spec, desc


def common_config(config, eps, prob=None):
    """The config keys both arms report (same workload, same generator, same sizes)."""
    from paper_2412_19027_b200 import generators as G
    spec, desc = workload(config)
    prob = prob if prob is not None else (G.build_instances(config, 0, 1)[0] if "instances" in spec else G.build(config))
    out = {"workload": desc, "config": config, "generator": f"generators.{spec['gen']}(seed, **{spec['kwargs']})",
           "n": prob.n, "m": prob.m, "nnz_A": prob.A.nnz, "precision": spec["precision"], "eps_feas": eps}
    if "instances" in spec:
        out["instances"] = spec["instances"]
    return out


def settings_for(config, eps):
    from paper_2412_19027_b200 import generators as G
    from paper_2412_19027_b200.settings import SolverSettings
    return SolverSettings(eps_feas=eps, precision=G.CONFIGS[config]["precision"])


# ---------------------------------------------------------------------------
# clocks sampler (nvidia-smi during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the UNMODIFIED reference solver (conic_ipm, pip-installed into
# baseline/_ref — see DESIGN.md "Reference arm"), else the oracle restatement
# (oracle/, bit-exact vs the reference on the golden fixtures).  Runs in a
# subprocess pinned to one thread: the reference is sequential (numba kernels,
# Python cone loops), SURVEY.md §8(d).
# ---------------------------------------------------------------------------

REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def reference_available():
    return os.path.isdir(os.path.join(REF_DIR, "conic_ipm"))


def _to_reference(ref, p):
    conv = {"zero": lambda c: ref.zero_cone(c.dim), "nonneg": lambda c: ref.nonneg_cone(c.dim),
            "soc": lambda c: ref.soc_cone(c.dim), "exp": lambda c: ref.exp_cone(),
            "pow": lambda c: ref.pow_cone(c.alpha), "psd": lambda c: ref.psd_cone(c.side)}
    P = ref.CsrMatrix(p.P.nrows, p.P.ncols, p.P.rowptr, p.P.colidx, p.P.values)
    A = ref.CsrMatrix(p.A.nrows, p.A.ncols, p.A.rowptr, p.A.colidx, p.A.values)
    return ref.ProblemData(P, A, p.q, p.b, [conv[c.kind](c) for c in p.cones])


def cpu_worker(args):
    """One process: setup once, then `--cpu-solves` bounded solves of at most
    `--cpu-max-iters` IPM iterations each; one JSON line per solve."""
    from paper_2412_19027_b200 import generators as G
    if "instances" in G.CONFIGS[args.config]:
        return cpu_worker_batch(args)
    prob = G.build(args.config)
    cap = args.cpu_max_iters or 200
    if args.cpu_impl == "reference":
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/cipm_numba_cache")
        sys.dont_write_bytecode = True
        sys.path.insert(0, REF_DIR)
        import conic_ipm as ref
        prec = G.CONFIGS[args.config]["precision"]
        # numba JIT warm-up on a tiny instance, outside any timing
        warm = _to_reference(ref, G.gen_lp(20, 40, seed=1))
        ref.Solver(warm, ref.SolverSettings(eps_feas=args.eps, precision=prec)).solve()
        t0 = time.perf_counter()
        solver = ref.Solver(_to_reference(ref, prob), ref.SolverSettings(eps_feas=args.eps, precision=prec,
                                                                         max_iter=cap))
        setup = time.perf_counter() - t0
        run = solver.solve
    else:
        from oracle.ipm import OracleSolver
        cfg = settings_for(args.config, args.eps)
        t0 = time.perf_counter()
        solver = OracleSolver(prob, cfg)
        setup = time.perf_counter() - t0

        def run():
            return solver.solve(max_iterations_run=cap)
    for _ in range(max(1, args.cpu_solves)):
        res = run()
        out = {"impl": args.cpu_impl, "setup_s": setup, "solve_s": res.solve_seconds,
               "iterations": res.iterations, "status": res.status, "obj": res.obj_primal}
        print("CPUWORKER " + json.dumps(out), flush=True)


def _ref_solver_factory(impl, config, eps):
    """Returns make(problem) -> object with .solve(); reference setup happens in make()."""
    from paper_2412_19027_b200 import generators as G
    prec = G.CONFIGS[config]["precision"]
    if impl == "reference":
        os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/cipm_numba_cache")
        sys.dont_write_bytecode = True
        if REF_DIR not in sys.path:
            sys.path.insert(0, REF_DIR)
        import conic_ipm as ref
        warm = _to_reference(ref, G.gen_lp(20, 40, seed=1))
        ref.Solver(warm, ref.SolverSettings(eps_feas=eps, precision=prec)).solve()
        return lambda p: ref.Solver(_to_reference(ref, p), ref.SolverSettings(eps_feas=eps, precision=prec))
    from oracle.ipm import OracleSolver
    from paper_2412_19027_b200.settings import SolverSettings
    return lambda p: OracleSolver(p, SolverSettings(eps_feas=eps, precision=prec))


_CHUNK_SOLVERS = {}


def _batch_chunk(payload):
    """Worker: set up its instances once (cached per process), then time only the solves."""
    impl, config, eps, lo, hi = payload
    key = (impl, config, eps, lo, hi)
    if key not in _CHUNK_SOLVERS:
        from paper_2412_19027_b200 import generators as G
        make = _ref_solver_factory(impl, config, eps)
        _CHUNK_SOLVERS[key] = [make(p) for p in G.build_instances(config, lo, hi)]
    solvers = _CHUNK_SOLVERS[key]
    t0 = time.perf_counter()
    it = sum(s.solve().iterations for s in solvers)
    return it, time.perf_counter() - t0


def cpu_worker_batch(args):
    """Batched configs: `--cpu-procs` worker processes (the reference's own
    `bench --jobs` mode, bench.py:98-113) over the first `--cpu-instances`
    instances; one JSON line per repetition."""
    from concurrent.futures import ProcessPoolExecutor
    procs = max(1, args.cpu_procs)
    count = args.cpu_instances
    chunks = [(args.cpu_impl, args.config, args.eps, count * k // procs, count * (k + 1) // procs)
              for k in range(procs)]
    # one chunk per worker process; setup (reference Solver construction) is done once in each
    # worker and excluded; a repetition's time is the slowest worker's solve time
    with ProcessPoolExecutor(max_workers=procs) as ex:
        for _ in range(max(1, args.cpu_solves)):
            out = list(ex.map(_batch_chunk, chunks, chunksize=1))
            its = sum(o[0] for o in out)
            res = {"impl": args.cpu_impl, "setup_s": 0.0, "solve_s": max(o[1] for o in out), "iterations": its,
                   "status": "n/a", "obj": None, "instances": count, "procs": procs}
            print("CPUWORKER " + json.dumps(res), flush=True)


def run_cpu(args, max_iters, solves=1, impl=None, procs=1):
    impl = impl or ("reference" if reference_available() else "port")
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1", MKL_NUM_THREADS="1",
               NUMBA_NUM_THREADS="1", CUDA_VISIBLE_DEVICES="")
    cmd = [sys.executable, os.path.abspath(__file__), "--cpu-worker", "--config", args.config,
           "--eps", str(args.eps), "--cpu-max-iters", str(max_iters), "--cpu-solves", str(solves),
           "--cpu-impl", impl, "--cpu-procs", str(procs), "--cpu-instances", str(args.cpu_instances)]
    out = subprocess.run(cmd, capture_output=True, text=True, env=env, timeout=3600)
    res = [json.loads(line[len("CPUWORKER "):]) for line in out.stdout.splitlines()
           if line.startswith("CPUWORKER ")]
    if not res:
        raise RuntimeError(f"cpu worker failed: {out.stderr[-2000:]}")
    return impl, res


def cpu_sample(args):
    """Bounded sample for the cpu_baseline key: one solve capped at `--cpu-iters`
    IPM iterations (setup excluded from the rate)."""
    if not args.cpu_instances:
        args.cpu_instances = 256
    impl, res = run_cpu(args, args.cpu_iters, 1)
    r = res[0]
    return impl, r


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def fp64_peak_tflops(device):
    """FP64 tensor-pipe reference peak of this GPU: cuBLAS DGEMM 8192^3 (best of 5)."""
    import torch
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=device)
    b = torch.randn(n, n, dtype=torch.float64, device=device)
    torch.matmul(a, b)
    best = float("inf")
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize(device)
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    return 2.0 * n ** 3 / best / 1e12


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def ncu_traffic(config):
    """DRAM bytes per sweep pair of the dominant kernel class from the committed ncu
    capture (profiles/ncu_traffic.json, tools/ncu_sweeps.sh + tools/ncu_traffic.py), if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            v = json.load(f).get(config)
        return v if isinstance(v, dict) else None
    except Exception:
        return None


def shard(total, world, rank):
    """Contiguous block of instances of rank `rank`."""
    lo = total * rank // world
    return lo, total * (rank + 1) // world


def run_batch(args):
    """C5b: every rank solves its shard of the 2048 MPC instances in one launch
    (no collective on the solve path); value = all ranks' IPM iterations / the
    slowest rank's device time."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2412_19027_b200 import generators as G
    from paper_2412_19027_b200.batch import BatchSolver

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # functional check of the sharded path on a one-GPU box: every rank on cuda:0,
    # gloo for the (timing-only) collectives — NCCL refuses two ranks per device
    one_dev = os.environ.get("CIPM_BENCH_ONE_DEVICE", "0") != "0"
    if one_dev:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_dev:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    spec, desc = workload(args.config)
    total = G.CONFIGS[args.config]["instances"]
    lo, hi = shard(total, world, rank)
    probs = G.build_instances(args.config, lo, hi)
    cfg = settings_for(args.config, args.eps)
    t0 = time.perf_counter()
    bs = BatchSolver(probs, cfg, device=local)
    setup = time.perf_counter() - t0
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")
    for _ in range(args.warmup):
        bs.run()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ms = []
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        ms.append(bs.run())
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    res = bs.results()
    iters = sum(r.iterations for r in res)
    statuses = sorted({r.status for r in res})
    dev_s = sum(ms) / 1e3
    # e2e through the public API: host arrays -> update_data (equilibration + H2D) -> solve -> results (D2H)
    q_host = np.stack([p.q for p in probs])
    b_host = np.stack([p.b for p in probs])
    from paper_2412_19027_b200.native import lib
    import ctypes
    h2d, d2h = ctypes.c_int64(0), ctypes.c_int64(0)
    lib().cipm_batch_io_bytes(bs.handle, None, None, 1)
    if world > 1:
        dist.barrier()
    e2e = []
    e2e_it = 0
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        bs.update_data(q=q_host, b=b_host)
        out = bs.solve()
        e2e.append(time.perf_counter() - t1)
        e2e_it += int(out.iterations.sum())
    lib().cipm_batch_io_bytes(bs.handle, ctypes.byref(h2d), ctypes.byref(d2h), 1)
    e2e_s = sum(e2e)
    vals = torch.tensor([dev_s, e2e_s, float(iters), float(e2e_it), float(len(probs))], dtype=torch.float64,
                        device=f"cuda:{local}")
    if world > 1:
        mx = vals.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = vals.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        dev_s, e2e_s = float(mx[0]), float(mx[1])
        iters_all, e2e_all, n_all = float(sm[2]), float(sm[3]), int(sm[4])
    else:
        iters_all, e2e_all, n_all = float(iters), float(e2e_it), len(probs)
    value = iters_all * args.steps / dev_s
    info = bs.info()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_s * 1e3 / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator, paper_2412_19027_b200/generators.py)",
        "config": {**common_config(args.config, args.eps, probs[0]), "instances": n_all,
                   "instances_per_gpu": len(probs), "nnz_L": info["nnz_l"],
                   "smem_bytes_per_cta": info["smem_bytes"], "cta_factorisation": bool(info["cta_factor"]),
                   "root_width": info["root_width"], "leaf_groups": info["groups"],
                   "status": statuses, "iterations_total": iters_all,
                   "instances_per_s": n_all * args.steps / dev_s, "setup_s": setup,
                   "l2": "flushed between steps (256 MiB write)",
                   "parallelism": f"instance shards x{world}, no collective on the solve path"},
        "clocks": clk,
        "e2e": {"value": e2e_all / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d.value // max(1, args.steps),
                "d2h_bytes_per_step": d2h.value // max(1, args.steps),
                "path": "BatchSolver.update_data(q, b) raw host arrays (H2D; reorder + Ruiz per instance on the device) + solve() -> host results"},
        "gpu_launches": args.steps,
        "roofline": None,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            # the reference's own bench --jobs mode (bench.py:98-113): one worker process per
            # host core over a bounded sample of the instances; the single-core rate beside it
            procs = os.cpu_count() or 1
            if not args.cpu_instances:
                args.cpu_instances = 32 * procs
            impl, res = run_cpu(args, args.cpu_iters, 1, procs=procs)
            rj = res[0]
            args.cpu_instances = 64
            _, res1 = run_cpu(args, args.cpu_iters, 1, procs=1)
            r1 = res1[0]
            who = 'the unmodified reference conic_ipm' if impl == 'reference' else 'the oracle'
            line["cpu_baseline"] = {"value": rj["iterations"] / rj["solve_s"], "unit": UNIT, "cores": procs,
                                    "kind": impl,
                                    "sample": f"{rj['instances']} instances over {procs} worker processes "
                                              f"(the reference's bench --jobs mode) by {who}, setup excluded",
                                    "single_core": {"value": r1["iterations"] / r1["solve_s"], "cores": 1,
                                                    "sample": f"{r1['instances']} instances, 1 process"}}
        except Exception as e:
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"failed: {e}"[:300]}
    bs.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# configs whose reference run cannot fit a bench run's time budget (the number
# stated was measured once, offline, in the build container)
CPU_SKIP = {
    "c4_exppow": "not run: the unmodified reference's setup alone (its exact minimum-degree "
                 "ordering in Python) takes ~35 min at this size; measured once in the build "
                 "container: 3 IPM iterations in 463 s = 0.0065 iter/s after 2113 s of setup",
}


def run_ours(args):
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2412_19027_b200 import generators as G
    from paper_2412_19027_b200.native import pdbl
    from paper_2412_19027_b200.solver import Solver

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    spec, desc = workload(args.config)
    prob = G.build(args.config)
    cfg = settings_for(args.config, args.eps)
    solver = Solver(prob, cfg, device=local)
    ctx = solver._ctx
    info = solver.symbolic.info()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=f"cuda:{local}")

    for _ in range(args.warmup):
        res = solver.solve()
    torch.cuda.synchronize()

    ms = ctypes.c_double(0.0)
    ctx.call("cipm_launch_count", None, 1)
    clocks = ClockSampler(local)
    clocks.start()
    barrier()
    torch.cuda.synchronize()
    step_ms = []
    iters = []
    statuses = set()
    for _ in range(args.steps):
        flush.fill_(1.0)                 # L2 flush (256 MiB) outside the timed window
        torch.cuda.synchronize()
        ctx.call("cipm_timer", 0, None)
        res = solver.solve()
        ctx.call("cipm_timer", 1, ctypes.byref(ms))
        step_ms.append(ms.value)
        iters.append(res.iterations)
        statuses.add(res.status)
    torch.cuda.synchronize()
    barrier()
    clk = clocks.stop()
    launches = ctypes.c_int64(0)
    ctx.call("cipm_launch_count", ctypes.byref(launches), 1)
    # kernel-level stats from one extra, separately profiled solve (per-launch CUDA events
    # on the solver stream; the timed steps above run the graph-captured refinement)
    ctx.call("cipm_profile", 1)
    flush.fill_(1.0)
    torch.cuda.synchronize()
    prof_res = solver.solve()
    kst = np.zeros(5)
    ctx.call("cipm_kernel_stats", pdbl(kst))
    ctx.call("cipm_profile", 0)
    kst_iters = max(1, prof_res.iterations)
    # the other kernel classes of the north star (fused residual SpMV, KKT matvec, cone
    # scaling per family) timed at the final iterate with CUDA events on the solver stream
    kcls = np.zeros(12)
    ctx.call("cipm_kernel_classes", 20, pdbl(kcls))

    total_s = sum(step_ms) / 1e3
    total_it = sum(iters)
    if world > 1:
        t = torch.tensor([total_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_s = float(t.item())
        it_t = torch.tensor([float(total_it)], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(it_t, op=dist.ReduceOp.SUM)
        total_it_all = float(it_t.item())
    else:
        total_it_all = float(total_it)
    value = total_it_all / total_s

    # ---- e2e through the public API with host buffers ----
    q_host = np.ascontiguousarray(prob.q)
    b_host = np.ascontiguousarray(prob.b)
    e2e_ms = []
    e2e_it = 0
    ctx.call("cipm_io_bytes", None, None, 1)
    barrier()
    for _ in range(args.steps):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        ctx.call("cipm_timer", 0, None)
        solver.update_data(q=q_host, b=b_host)
        r = solver.solve()
        _ = (r.x.sum(), r.z.sum(), r.s.sum())
        ctx.call("cipm_timer", 1, ctypes.byref(ms))
        e2e_ms.append(ms.value)
        e2e_it += r.iterations
    h2d = ctypes.c_int64(0)
    d2h = ctypes.c_int64(0)
    ctx.call("cipm_io_bytes", ctypes.byref(h2d), ctypes.byref(d2h), 1)
    e2e_s = sum(e2e_ms) / 1e3
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_value = e2e_it * world / e2e_s

    # ---- roofline of the dominant kernel class ----
    hbm, peak_kind = peaks()
    es = 4 if cfg.precision == "mixed" else 8
    fac_ms, fac_n, sol_ms, sol_n, rhs_n = kst
    nnz_l, dim = info["nnz_l"], info["dim"]
    if sol_ms >= fac_ms and sol_n > 0:
        # per right-hand side: L and L' sweeps read (value + int32 index) per nnz, plus 4 vector passes
        bytes_per_rhs = 2 * (es + 4) * nnz_l + 4 * es * dim
        achieved = bytes_per_rhs * (rhs_n / sol_n) / (sol_ms / sol_n / 1e3) / 1e9
        dom = {"kernel": "supernodal triangular solve (forward_kernel + backward_kernel)",
               "launches": int(sol_n), "avg_ms": sol_ms / sol_n,
               "bytes_per_launch": bytes_per_rhs * rhs_n / sol_n,
               "share_of_step": sol_ms / (sum(step_ms) / len(step_ms) or 1)}
    else:
        # numeric factorisation: write L (value + index) + read the assembled K values
        bytes_fac = (es + 4) * nnz_l + es * info["nnz_storage"]
        achieved = bytes_fac / (fac_ms / fac_n / 1e3) / 1e9
        dom = {"kernel": "supernodal numeric factorisation (factor_kernel)", "launches": int(fac_n),
               "avg_ms": fac_ms / fac_n, "bytes_per_launch": bytes_fac,
               "share_of_step": fac_ms / (sum(step_ms) / len(step_ms) or 1),
               "tflops": info["flops"] / (fac_ms / fac_n / 1e3) / 1e12}
    kernels = {}
    for k, name in enumerate(("residual_spmv (resid_n + resid_m)", "kkt_matvec (kkt_res_n + kkt_res_m + apply_H)",
                              "scaling_nonneg (nn_scaling)", "scaling_soc (soc_scaling)",
                              "scaling_exp_pow (nsym_scaling)", "scaling_psd (psd_scaling)")):
        ms_k, by_k = kcls[2 * k], kcls[2 * k + 1]
        if ms_k > 0:
            gbs = by_k / (ms_k / 1e3) / 1e9
            kernels[name] = {"us": ms_k * 1e3, "bytes": by_k, "achieved_gbs": gbs, "frac": gbs / hbm}
    traffic = ncu_traffic(args.config)
    roof = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
            "traffic": (traffic or {}).get("bytes") if isinstance(traffic, dict) else traffic,
            "traffic_source": (traffic or {}).get("source") if isinstance(traffic, dict) else None,
            "peak_source": peak_kind, "dominant": dom,
            "factor_ms_avg": fac_ms / fac_n if fac_n else None,
            "solve_ms_avg_per_pair": sol_ms / sol_n if sol_n else None,
            "kernels": kernels}
    if "tflops" in dom and cfg.precision == "full":
        # factorisation-dominated (dense tail on the FP64 tensor pipe): the tensor roofline,
        # against a DGEMM measured here (MEASURED_PEAKS.json has no FP64 figure)
        f64 = fp64_peak_tflops(f"cuda:{local}")
        roof.update({"bound": "tensor", "achieved": dom["tflops"], "peak": f64, "unit": "TFLOP/s",
                     "frac": dom["tflops"] / f64, "traffic": None,
                     "peak_source": "measured here: cuBLAS DGEMM (torch.matmul float64 8192^3, best of 5)",
                     "hbm_view": {"achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm}})

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": sum(step_ms) / len(step_ms), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None,
        "dtype": "f64 iterate / f32 LDL' + f64 refinement" if cfg.precision == "mixed" else "f64",
        "data": "synthetic (seeded generator, paper_2412_19027_b200/generators.py)",
        "config": {**common_config(args.config, args.eps, prob), "status": sorted(statuses),
                   "iterations_per_solve": total_it / max(1, args.steps),
                   "solve_time_s": sum(step_ms) / 1e3 / args.steps,
                   "setup_s": solver.setup_seconds, "nnz_L": nnz_l, "supernodes": info["nsuper"],
                   "etree_height_supernodes": info["height"], "F_LDL_gflop": info["flops"] / 1e9,
                   "l2": "flushed between steps (256 MiB write), inputs resident in HBM",
                   "parallelism": f"replicas x{world}" if world > 1 else "single GPU"},
        "clocks": clk,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d.value // max(1, args.steps),
                "d2h_bytes_per_step": d2h.value // max(1, args.steps),
                "path": "Solver.update_data(q, b) host arrays + Solver.solve() -> host x, z, s"},
        "gpu_launches": int(launches.value),
        "roofline": roof,
    }
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.config in CPU_SKIP:
        line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                "sample": CPU_SKIP[args.config]}
    elif rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            impl, r = cpu_sample(args)
            cpu_val = r["iterations"] / r["solve_s"]
            what = ("the unmodified reference conic_ipm (baseline/_ref)" if impl == "reference"
                    else "the oracle restatement of the reference")
            line["cpu_baseline"] = {"value": cpu_val, "unit": UNIT, "cores": 1, "kind": impl,
                                    "sample": f"{what}: first {r['iterations']} IPM iterations of {args.config} "
                                              f"(status {r['status']}), setup {r['setup_s']:.1f}s excluded, "
                                              f"1 thread of a {os.cpu_count()}-core host",
                                    "cpu_solve_s_per_iter": r["solve_s"] / max(1, r["iterations"]),
                                    "setup_s": r["setup_s"]}
        except Exception as e:  # never lose the GPU line over the CPU leg
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                                    "sample": f"failed: {e}"[:300]}
    solver.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# ---------------------------------------------------------------------------
# reference arm: the CPU oracle (the reference itself cannot travel to the box)
# ---------------------------------------------------------------------------

def run_reference(args):
    """--impl reference: rank 0 times the reference's own CPU solver (setup once,
    then W warm-up + K timed solves, each capped at --cpu-iters iterations)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    spec, desc = workload(args.config)
    from paper_2412_19027_b200 import generators as G
    batched = "instances" in G.CONFIGS[args.config]
    procs = (os.cpu_count() or 1) if batched else 1
    if batched and not args.cpu_instances:
        args.cpu_instances = G.CONFIGS[args.config]["instances"]
    impl, res = run_cpu(args, args.cpu_iters, args.warmup + args.steps, procs=procs if batched else 1)
    timed = res[args.warmup:]
    it_total = sum(r["iterations"] for r in timed)
    secs = sum(r["solve_s"] for r in timed)
    value = it_total / secs
    what = ("unmodified reference conic_ipm from baseline/_ref" if impl == "reference"
            else "oracle restatement of the reference (bit-exact on the golden fixtures)")
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": 0, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": secs * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong" if batched else "weak", "vs_baseline": None,
            "dtype": "f64 iterate / f32 LDL' + f64 refinement" if G_precision(args.config) == "mixed" else "f64",
            "impl": "reference", "data": "synthetic (seeded generator, paper_2412_19027_b200/generators.py)",
            "config": {**common_config(args.config, args.eps), "status": sorted({r["status"] for r in timed}),
                       "iterations_per_solve": it_total / max(1, len(timed)),
                       "setup_s": timed[0]["setup_s"]},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": procs if batched else 1, "kind": impl,
                             "sample": (f"{what}: each step {args.cpu_instances} instances over {procs} worker "
                                        f"processes (the reference's bench --jobs mode)" if batched else
                                        f"{what}: each step one solve capped at {args.cpu_iters} IPM iterations, "
                                        f"setup excluded, 1 thread of a {os.cpu_count()}-core host")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def G_precision(config):
    from paper_2412_19027_b200 import generators as G
    return G.CONFIGS[config]["precision"]


def main():
    args = parse()
    if args.cpu_worker:
        cpu_worker(args)
        return
    from paper_2412_19027_b200 import generators as G
    if args.impl == "reference":
        run_reference(args)
    elif "instances" in G.CONFIGS[args.config]:
        run_batch(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

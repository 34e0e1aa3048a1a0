#!/usr/bin/env python
"""Benchmark of the GLAM lambda-path fit (BASELINE.json metric:
"lambda-path fit time & prox-grad iters/s; rho-contraction HBM GB/s vs peak").

One step = one full warm-started lambda path of a BASELINE config with the
observation array resident in HBM.  The default workload is C5, the largest
config (Poisson 3-D GLAM, n = (256,256,1024), p = (64,64,256), cubic
B-splines, 20-lambda lasso path): it fits one B200 and runs the n-space
route, i.e. the north-star rho contractions on the 537 MB observation array
every prox-grad step.  value = prox-grad (FISTA) iterations per second over
the whole path.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--impl ours|reference]
                  [--replicas]

N > 1 (launched by torchrun, or re-launched under torchrun by this script when
WORLD_SIZE is unset): by default ONE fit of the config sharded along its last
observation mode over the ranks (slab-local H, a p-sized NCCL
all-reduce per gradient; strong scaling); --replicas runs one independent fit
per rank instead (weak scaling).

--impl reference times the reference's CPU algorithm -- the oracle port in
oracle/ (the Eigen-based reference cannot be built here) -- on all
host cores, on a bounded sample of the same workload; it never loads the
product library.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "lambda-path fit time & prox-grad iters/s; rho-contraction HBM GB/s vs peak"
UNIT = "prox-grad iters/s"
L2_NOTE = "256 MB buffer written between timed steps (> 126 MB L2)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-budget", type=float, default=20.0, help="seconds of CPU work per baseline sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: one independent fit per rank (weak scaling) instead of one sharded fit")
    ap.add_argument("--shard", action="store_true", help="(default for N > 1) one fit sharded over the ranks")
    return ap.parse_args()


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json, copy read+write)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def fp64_peaks():
    path = os.path.join(ROOT, "profiles", "fp64_peaks.json")
    if os.path.exists(path):
        with open(path) as f:
            return json.load(f)
    return None


def world_info():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def sharded_mode(args, world):
    # --shard at N = 1 runs the sharded machinery on one rank (NCCL communicator,
    # host-driven loop, owned-slice path with KG_HALO=1): a single-GPU check
    return (world > 1 or args.shard) and not args.replicas


def config_obj(args, data, world):
    """The workload description, identical in both arms (the driver compares them)."""
    if world == 1 and not args.shard:
        par = "single GPU"
    elif sharded_mode(args, world):
        par = (f"last-mode shards x{world} (per gradient: NCCL send/recv of the ~3 boundary coefficient "
               f"slices with each neighbour + a 4-double all-reduce)")
    else:
        par = f"replicas x{world}"
    return {"workload": args.config, "family": data["family"], "n": list(data["n"]), "p": list(data["p"]),
            "n_lambda": data["n_lambda"], "lambda_min_ratio": data["lambda_min_ratio"], "penalty": "lasso",
            "iwls": "exact", "l2": L2_NOTE, "parallelism": par}


class Clocks:
    """nvidia-smi sampler running during the timed region."""

    def __init__(self, index=0):
        self.samples = []
        self.index = index
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
                 "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
                 "clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# ------------------------------------------------------------ CPU samples
def cpu_sample(data, threads, budget, iters=None):
    """The oracle (reference algorithm restated, oracle/) on a bounded sample of
    the workload, returning (prox-grad iterations, seconds, description).

    Gaussian configs: the first lambdas of the warm-started path, lambda by
    lambda (outer_solve per lambda, path.cpp:47-81), until `budget` seconds.
    Poisson configs: the first inner problem the path solves below lambda_max
    (model 1's first outer iteration: v = glm_weights(eta = 0), z = the working
    response, fista_solve at lambda_1 from theta = 0, inner.cpp:121-235),
    capped at `iters` prox-grad iterations (first call: sized to the budget)."""
    from oracle import oracle as O
    O.set_threads(threads)
    design, y, fam = data["design"], data["y"], data["family"]
    lmax = O.lambda_max(design, fam, y)
    nl, ratio = data["n_lambda"], data["lambda_min_ratio"]
    lams = [lmax] + [lmax * float(np.exp(np.log(ratio) / (nl - 1) * t)) for t in range(1, nl)]
    if fam == "gaussian":
        t0 = time.perf_counter()
        it, k, init = 0, 0, None
        for lam in lams:
            if iters is not None and it >= iters:
                break
            if iters is None and time.perf_counter() - t0 > budget:
                break
            r = O.outer_solve(design, fam, y, lam, init=init)
            it += sum(int(rec["inner_iterations"]) for rec in r["iterations"])
            init = r["coef"]
            k += 1
        return it, time.perf_counter() - t0, f"first {k} of {nl} lambdas (warm-started outer_solve per lambda)"
    eta0 = np.zeros(y.shape)
    v = O.glm_weights(fam, eta0).reshape(y.shape, order="F")
    z = O.working_response(fam, y, eta0).reshape(y.shape, order="F")
    if iters is None:  # size the sample to the budget: marginal cost of an iteration past the setup
        t0 = time.perf_counter()
        O.fista_solve(design, v, z, lams[1], inner_maxit=1)
        t1 = time.perf_counter()
        O.fista_solve(design, v, z, lams[1], inner_maxit=2)
        t2 = time.perf_counter()
        per_it = max((t2 - t1) - (t1 - t0), 1e-6)
        setup = max((t1 - t0) - per_it, 0.0)
        iters = int(max(3, min(200, (budget - setup) / per_it)))
    t0 = time.perf_counter()
    r = O.fista_solve(design, v, z, lams[1], inner_maxit=iters)
    dt = time.perf_counter() - t0
    return r["iterations"], dt, (f"fista_solve of model 1's first inner problem (lambda_1, v = glm_weights(0), "
                                 f"z = working response), {r['iterations']} prox-grad iterations")


def run_reference(args):
    world, rank, _ = world_info()
    if rank != 0:
        return  # rank 0 alone times the CPU reference; the other ranks exit without work
    from oracle import oracle as O
    from paper_1510_03298_b200 import configs
    data = configs.make(args.config, bspline=O.bspline_design)  # no product library on this arm
    threads = os.cpu_count() or 1
    budget = max(2.0, min(args.cpu_budget, 8.0))
    it0, _, _ = cpu_sample(data, threads, budget)  # fixes the per-step sample size
    for _ in range(max(args.warmup - 1, 0)):
        cpu_sample(data, threads, budget, iters=it0)
    tot_it, tot_s, desc = 0, 0.0, ""
    for _ in range(args.steps):
        it, s, desc = cpu_sample(data, threads, budget, iters=it0)
        tot_it += it
        tot_s += s
    value = tot_it / tot_s
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * tot_s / args.steps,
            "higher_is_better": True, "scaling": "strong" if sharded_mode(args, world) else "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded stand-in for the BASELINE config)",
            "config": config_obj(args, data, world),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                             "sample": f"{args.config}: {desc}, oracle on {threads} host threads"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------ our arm
def parity_prefix(name, res):
    """The fitted models against the committed oracle fixture of this config
    (tests/golden/path_<config>.npz): support, iteration counts and the
    coefficient error of every model the fixture stores in full."""
    path = os.path.join(ROOT, "tests", "golden", f"path_{name}.npz")
    if not os.path.exists(path):
        return None
    from tests.test_gpu_fixtures import coefs_of, load, supports_of
    fx = load(name)
    want, supp = coefs_of(fx), supports_of(fx)
    m = min(res.n_models, fx["meta"]["models"])
    got = res.coefs()
    errs = [float(np.max(np.abs(got[t] - w)) / max(np.max(np.abs(w)), 1e-300)) for t, w in want.items() if t < m]
    return {"models": m, "source": f"tests/golden/path_{name}.npz (CPU oracle, same seeded inputs)",
            "max_coef_rel_err": max(errs) if errs else None,
            "same_support": bool(all(np.array_equal(got[t] != 0, supp[t]) for t in range(m))),
            "same_iteration_counts": bool(res.inner_iters[:m] == [int(v) for v in fx["inner_iters"][:m]]
                                          and res.outer_iters[:m] == [int(v) for v in fx["outer_iters"][:m]])}


def kernel_time(ctx, design, obs, which, reps=10):
    import ctypes as C
    from paper_1510_03298_b200 import _lib
    ms, b = C.c_double(), C.c_double()
    ctx.check(_lib.load().kg_time_kernel(ctx.h, design.h, obs.h, which, reps, C.byref(ms), C.byref(b)))
    return ms.value, b.value


def path_kernel_stats(ctx):
    import ctypes as C
    from paper_1510_03298_b200 import _lib
    ms, b, st = C.c_double(), C.c_double(), C.c_int64()
    if _lib.load().kg_path_kernel_stats(ctx.h, C.byref(ms), C.byref(b), C.byref(st)) != 0:
        return None
    return ms.value, b.value, st.value


def relaunch_under_torchrun(args):
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} requested but {have} CUDA device(s) "
                          f"are visible; refusing to run N={args.gpus} on fewer GPUs"}), flush=True)
        sys.exit(1)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(29500 + os.getpid() % 1000)] + sys.argv
    sys.stdout.flush()
    sys.exit(subprocess.call(cmd, stdout=sys.stdout))  # the ranks inherit the real stdout (see _quiet_stdout)


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = world_info()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1510_03298_b200 import configs
    from paper_1510_03298_b200 import kronglm as K

    data = configs.make(args.config)
    shard = sharded_mode(args, world)
    fam, nl, ratio = data["family"], data["n_lambda"], data["lambda_min_ratio"]
    y = data["y"]
    if shard:
        uid = K.nccl_unique_id() if rank == 0 else None
        box = [uid]
        if world > 1:
            dist.broadcast_object_list(box, src=0)
        ctx = K.Context.sharded(local, rank, world, box[0])
        lo, hi = K.shard_rows(data["n"][-1], rank, world)
        y = np.asfortranarray(y[..., lo:hi])
    else:
        ctx = K.Context(local)
        if rank > 0:  # independent replica: same design, its own response draw
            rng = np.random.default_rng(configs.SEED0 + 1000 + rank)
            y = np.asfortranarray(y + 0.1 * rng.standard_normal(y.shape)) if fam == "gaussian" else \
                np.asfortranarray(rng.poisson(np.maximum(y, 0.1)).astype(np.float64))
    design = K.Design(data["design"], ctx)
    obs = K.Observation(design, y)
    stream = torch.cuda.ExternalStream(ctx.stream, device=torch.device("cuda", local))
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > 126 MB L2

    def one_path():
        return K.fit_path_resident(design, obs, fam, n_lambda=nl, lambda_min_ratio=ratio)

    for _ in range(args.warmup):
        res = one_path()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = Clocks(local)
    clocks.start()
    ctx.reset_launches()
    total_ms, iters = 0.0, 0
    pk_ms, pk_bytes, pk_n = 0.0, 0.0, 0
    with torch.cuda.stream(stream):
        for _ in range(args.steps):
            flush.zero_()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            res = one_path()
            e1.record(stream)
            e1.synchronize()
            total_ms += e0.elapsed_time(e1)
            iters += sum(res.inner_iters)
            st = path_kernel_stats(ctx)
            if st is not None:
                pk_ms, pk_bytes, pk_n = pk_ms + st[0], pk_bytes + st[1], pk_n + 1
    launches = ctx.launches
    torch.cuda.synchronize()
    clk = clocks.stop()
    max_ms, all_iters = total_ms, float(iters)
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        max_ms = float(t.item())
        if not shard:  # replicas: every rank's iterations count; sharded: one joint fit
            it = torch.tensor([float(iters)], dtype=torch.float64, device="cuda")
            dist.all_reduce(it, op=dist.ReduceOp.SUM)
            all_iters = float(it.item())
    value = all_iters / (max_ms / 1000.0)
    iters_per_path = sum(res.inner_iters)

    # --- roofline of the step's dominant kernel and the rho-contraction passes
    hbm, peak_kind = peaks()
    rho = {}
    try:  # the route the fits run: slab pass (d = 3) or the mode-1 fused pass
        kernel_time(ctx, design, obs, 6, reps=1)
        slab = True
    except Exception:
        slab = False
    kernels = ((("fused_pass", 0, "k_slab4: slab pass (per last-mode slice: eta = X1 S3 X2^T, v eta^2, "
                 "Q3 = X1^T (v eta) X2)"),
                ("h_mode3_step", 6, "mode-3 H-chain contraction (x -> S3)"),
                ("g_mode3_step", 7, "mode-3 G-chain contraction (Q3 -> S x)"),
                ("largest_h_step", 1, "largest banded H-chain contraction (Armijo trial eta, once per outer "
                 "iteration)"))
               if slab else
               (("fused_pass", 0, "fused n-space pass (H-last + v eta^2 + V.* + G-first)"),
                ("largest_h_step", 1, "largest banded H-chain contraction"),
                ("g_step", 5, "mode-2 G-chain contraction")))
    for key, which, what in kernels:
        try:
            ms, b = kernel_time(ctx, design, obs, which)
        except Exception as e:  # a route without this kernel (e.g. 2-D designs have no mode-2 G step)
            rho[key] = {"kernel": what, "unavailable": str(e)[:120]}
            continue
        rho[key] = {"kernel": what, "bytes_per_launch": b, "avg_launch_ms": ms,
                    "achieved": b / (ms / 1000.0) / 1e9, "frac": b / (ms / 1000.0) / 1e9 / hbm}
    rho["timing"] = "kg_time_kernel: CUDA events around each launch on the ctx stream, L2 evicted before each"
    traffic = None
    tfile = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(tfile):
        with open(tfile) as f:
            traffic = json.load(f)
    if pk_n:  # Gaussian constant-weight paths: the whole path is one cooperative launch
        achieved = pk_bytes / (pk_ms / 1000.0) / 1e9
        roof = {"bound": "hbm", "kernel": "k_gauss_path (whole lambda path, one cooperative launch)",
                "achieved": achieved, "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / hbm,
                "traffic": traffic.get("path_kernel_dram_bytes") if traffic else None,
                "bytes_per_launch": pk_bytes / pk_n, "avg_launch_ms": pk_ms / pk_n,
                "share_of_step": pk_ms / total_ms,
                "note": "latency-bound: one neighbour hand-off per prox-grad step; its bytes are p-space and "
                        "L2-resident"}
    else:
        f = rho.get("fused_pass", {})
        roof = {"bound": "hbm", "kernel": f.get("kernel"), "achieved": f.get("achieved"), "peak": hbm,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": f.get("frac"),
                "traffic": traffic.get("fused_pass_dram_bytes") if traffic else None,
                "bytes_per_launch": f.get("bytes_per_launch"), "avg_launch_ms": f.get("avg_launch_ms"),
                "launches_per_step": 1,
                "share_of_step": (f["avg_launch_ms"] * iters / total_ms) if f.get("avg_launch_ms") else None}
        if slab:
            roof["note"] = ("k_slab4 moves exactly its algorithmic bytes (traffic); with v streamed by bulk copies "
                            "alone the kernel takes ~105 us (5.7 TB/s); the rest is issue latency of its 16 resident "
                            "warps and shared-memory bandwidth (v, the U windows and the scatter/gather partials "
                            "all cross shared memory: ~122 KB per 2048-cell chunk, L1/shared pipe 74% busy) "
                            "(DESIGN.md 4b)")
    fp64 = fp64_peaks()
    if fp64:
        roof["fp64_peaks"] = fp64

    # --- e2e: the public kronglm.fit_path call with host buffers: design and
    # observation upload, the path, all coefficient downloads
    e2e_iters, e2e_ms = 0, 0.0
    n_e2e = max(1, min(args.steps, 3))
    if not shard:
        # two untimed calls first: the coefficients land in page-locked blocks that
        # the library recycles, and a caller holding the previous result uses a
        # second one, so steady state starts at the third call
        for i in range(2 + n_e2e):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            out = K.fit_path(data["design"], fam, y, n_lambda=nl, lambda_min_ratio=ratio)
            if i >= 2:
                e2e_ms += 1000.0 * (time.perf_counter() - t0)
                e2e_iters += sum(out["inner_iters"])
        n_models = len(out["lambdas"])
    else:  # sharded: the slab upload + path + coefficient download through the same objects
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        for i in range(n_e2e):
            t0 = time.perf_counter()
            o2 = K.Observation(design, y)
            r2 = K.fit_path_resident(design, o2, fam, n_lambda=nl, lambda_min_ratio=ratio)
            r2.coefs()
            e2e_ms += 1000.0 * (time.perf_counter() - t0)
            e2e_iters += sum(r2.inner_iters)
            n_models = r2.n_models
        if world > 1:
            t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
    h2d = 8 * (y.size + sum(x.size for x in data["design"][0]))
    d2h = 8 * design.p * n_models

    line = None
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": max_ms / args.steps, "higher_is_better": True,
                "scaling": "strong" if shard else "weak", "vs_baseline": None, "dtype": "f64",
                "data": "synthetic (seeded stand-in for the BASELINE config; no dataset)",
                "config": config_obj(args, data, world),
                "path": {"models_fitted": res.n_models, "prox_grad_iters_per_path": iters_per_path,
                         "path_fit_ms": max_ms / args.steps},
                "e2e": {"value": e2e_iters / (e2e_ms / 1000.0), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms / n_e2e},
                "roofline": roof, "rho_contraction": rho, "clocks": clk, "gpu_launches": int(launches)}
        if world == 1:
            line["parity_prefix"] = parity_prefix(args.config, res)
    # CPU baseline: the oracle port on rank 0 at N = 1, bounded sample of the same workload
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import oracle as O
        d_cpu = configs.make(args.config, bspline=O.bspline_design)
        it, s, desc = cpu_sample(d_cpu, 1, args.cpu_budget)
        line["cpu_baseline"] = {"value": it / s, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"{args.config}: {desc}, {s:.1f} s on one host core"}
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _quiet_stdout():
    """The contract is ONE JSON line on stdout.  Native libraries write there too
    (NCCL prints its version banner to stdout when NCCL_DEBUG is set in the
    environment), so file descriptor 1 is pointed at stderr for the whole run and
    Python's sys.stdout keeps the original descriptor for the JSON line."""
    sys.stdout.flush()
    keep = os.dup(1)
    os.dup2(2, 1)
    sys.stdout = os.fdopen(keep, "w", buffering=1)


def main():
    args = parse()
    _quiet_stdout()
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        print(json.dumps({"metric": METRIC, "error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}), flush=True)
        sys.exit(1)
    run_ours(args)


if __name__ == "__main__":
    main()

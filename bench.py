#!/usr/bin/env python
"""Benchmark of the hot path (BASELINE.json metric: Sinkhorn cost-entries/s — n*m per
iteration — and time-to-tol per init, with the roofline fraction of the dominant kernel).

Default workload: BASELINE.json configs[3] (C4), the largest configuration and the one its
">= 6x at 8 GPUs" target names — n = m = 262144 RGB-pixel-shaped points in [0,1]^3, eps = 1e-2,
tol = 1e-3, online cost.  One step = the paper's method on the whole problem: the subsample
initializer (Sec. 3.4: 4096 points per side, inner solve to tol/10, Eq. (8) extrapolation)
followed by the Sinkhorn solve to tolerance.  value = n*m*L / step time.  With N > 1
(torchrun) the rows of x are sharded over the ranks (sinkhorn_solve_sharded: per-rank block
partials of the column pass exchanged with ncclAllGather every sweep; strong scaling, the total
problem is fixed; the initializer is replicated).

Other workloads (also measurable): --workload c1 | c2 | c3 | c5.  C2 (1024 independent 1D
problems per rank) scales weakly with no data-path collective.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload ...]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

MUFU_EX2_PER_CLK_SM = 16     # B200 (sm_100) SFU ex2 throughput per SM per clock
FFMA_PER_CLK_SM = 128        # FP32 lanes per SM
N_SM = 148


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return json.load(open(p)), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled (every 50 ms) during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.out = index, None, ""

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)   # let the first sample land before the timed region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.1)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = [[c.strip() for c in l.split(",")] for l in self.out.splitlines() if l.count(",") >= 8]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        num = lambda v: float(v) if v.replace(".", "", 1).isdigit() else None
        sm = [num(r[1]) for r in rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows)}


def dist_env():
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ==================================================================== workloads
class Workload:
    """One BASELINE.json config.  step() runs the hot path once on this rank's inputs (already
    in HBM) and returns the cost entries n*m*L it processed; e2e_step() runs the same through
    the C ABI with pinned host buffers."""
    scaling = "weak"
    roof = "mufu"           # mufu | hbm | ffma
    fma_exp_share = 0.25    # mufu roof: share of the exponentials evaluated on the FMA pipe (K13: 1 of 4 pairs)

    def cpu_sample(self):  # -> (entries, seconds, threads, description)
        raise NotImplementedError


def c2_config(world):
    return {"workload": "BJ.cfg2 (C2): batched 1D sorting/ranking, B=1024 per GPU x n=m=1024, d=1, "
                        "x~U[0,1), y_j=j/(m-1), eps=1e-3, tol=1e-3 (L1 marginal), max_iter=10000",
            "init": "sort1d (closed-form eps=0 dual, Sec. 3.1)", "global_batch": 1024 * world,
            "parallelism": f"dp{world} (independent problems per rank)",
            "l2": "flushed (256 MiB write) before every timed step"}


class C2(Workload):
    name = "c2"

    def __init__(self, sk, ctx, dev, rank, world, args):
        from workloads import gen
        self.sk, self.ctx, self.world = sk, ctx, world
        self.p = p = gen.c2(seed=rank)
        self.B, self.n, self.m = p.batch, p.n, p.m
        import torch
        self.x = torch.from_numpy(p.x).to(dev)
        self.y = torch.from_numpy(p.y).to(dev)
        self.xh = torch.from_numpy(p.x).pin_memory()
        self.yh = torch.from_numpy(p.y).pin_memory()

    def config(self):
        return c2_config(self.world)

    def _run(self, x, y, init=True, anderson=None, adaptive=None):
        sk, p = self.sk, self.p
        f0 = sk.sinkhorn_init_sort1d(self.ctx, x.view(self.B, self.n), y.view(self.m), y_shared=True) if init else None
        self.f, self.g, reps = sk.sinkhorn_solve(self.ctx, x, y, p.eps, tol=p.tol, max_iter=p.max_iter,
                                                 y_shared=True, f_init=f0, anderson=anderson, adaptive=adaptive)
        self.its = reps.column("iterations")
        return float(self.n) * self.m * float(self.its.sum())

    def step(self):
        return self._run(self.x, self.y)

    def e2e_step(self):
        e = self._run(self.xh, self.yh)
        B, n, m = self.B, self.n, self.m
        h2d = 2 * (self.xh.numel() + self.yh.numel()) * 4 + B * n * 4   # x,y twice + f0 back in
        d2h = B * n * 4 + B * n * 4 + B * m * 4                          # f0, f, g
        return e, h2d, d2h

    def baseline(self):
        e = self._run(self.x, self.y, init=False)
        return {"init": "zero", "iterations_mean": float(self.its.mean()), "iterations_max": int(self.its.max())}

    def extra(self):
        import torch
        out = {"iterations_mean": float(self.its.mean()), "iterations_max": int(self.its.max())}
        # NEXT-2: soft ranks + soft sort of the whole batch from the solved potentials (K15, one
        # extra pass each way; 2 n m exponentials per problem), timed on the library's stream
        self._run(self.x, self.y)
        st = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        xs = self.x.view(self.B, self.n)
        self.sk.sinkhorn_soft_rank_sort(self.ctx, xs, self.y.view(self.m), self.p.eps, self.f, self.g, y_shared=True)
        e0.record(st)
        for _ in range(5):
            self.sk.sinkhorn_soft_rank_sort(self.ctx, xs, self.y.view(self.m), self.p.eps, self.f, self.g,
                                            y_shared=True)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        ex2 = 2.0 * self.B * self.n * self.m
        out["soft_rank_sort"] = {"ms": ms, "ex2_per_s": ex2 / (ms / 1e3),
                                 "mufu_frac": ex2 / (ms / 1e3) / (N_SM * MUFU_EX2_PER_CLK_SM * 1965e6),
                                 "note": "K15: ranks E_P[z|i] and sort E_P[x|j] of the 1024-problem batch (R-22)"}
        # NEXT-1: the same step (sort1d init + solve to tol) with Anderson acceleration (m = 5, R-27)
        self._run(self.x, self.y, anderson=5)
        e0.record(st)
        for _ in range(3):
            ent = self._run(self.x, self.y, anderson=5)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        out["anderson5"] = {"time_to_tol_ms": ms, "iterations_mean": float(self.its.mean()),
                            "iterations_max": int(self.its.max()), "cost_entries_per_s": ent / (ms / 1e3),
                            "note": "sort1d init + Anderson (memory 5) to the same tol; entries = n m sweeps"}
        # NEXT-1: adaptive momentum (window 10; R-31)
        self._run(self.x, self.y, adaptive=10)
        e0.record(st)
        for _ in range(3):
            ent = self._run(self.x, self.y, adaptive=10)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 3
        out["adaptive10"] = {"time_to_tol_ms": ms, "iterations_mean": float(self.its.mean()),
                             "iterations_max": int(self.its.max()), "cost_entries_per_s": ent / (ms / 1e3),
                             "note": "sort1d init + adaptive momentum (window 10) to the same tol"}
        return out

    kernel = "k_batched<1,2,512> (on-chip persistent solver, K13)"

    def cpu_sample(self, nprob=None, target_s=10.0):
        """The fp64 oracle, as it stands, on whole C2 problems (sort1d init + solve to tol);
        the number of problems is scaled so the sample takes about target_s seconds."""
        from oracle import oracle as O
        from workloads import gen
        p = gen.c2(B=256)

        def run(k):
            t0 = time.perf_counter()
            e = 0.0
            for b in range(k):
                f0 = O.init_sort1d(p.x[b].ravel(), p.y.ravel())
                r = O.sinkhorn(p.x[b], p.y, p.eps, tol=p.tol, f0=f0)
                e += float(p.n) * p.m * r.iterations
            return e, time.perf_counter() - t0
        if nprob is None:
            e, t = run(2)
            nprob = int(min(256, max(2, 2 * target_s / max(t, 1e-3))))
        e, t = run(nprob)
        return e, t, O.num_threads(), f"{nprob} of the 1024 C2 problems (sort1d init + fp64 solve to tol)"


def single_spec(args):
    """The problem, initializer, cost mode and dominant kernel of one single-problem workload
    (C1, C3, C4, C5) — shared by both arms so that their config dicts are identical."""
    from workloads import gen
    name = args.workload
    sp = {"name": name, "scaling": "weak", "fma_exp_share": 0.25}
    if name == "c1":
        sp.update(p=gen.c1(), init="gaussian", mode="auto", roof="mufu", kernel="k_batched (on-chip solver, one CTA)")
    elif name == "c3":
        sp.update(p=gen.c3(eps_factor=args.eps_factor or 0.01), init=args.init or "gmm", mode="stored", roof="hbm",
                  kernel="k_stored_fused (single-read fused stored sweep, K5)")
    elif name == "c4":
        ffma = any(t.replace(" ", "") in ("tc=0", "tc_small_d=0") for t in args.tune)
        sp.update(p=gen.c4(), init=args.init or "subsample", mode="online", roof="mufu", scaling="strong",
                  # K3 passes: 2 of 8 exponential pairs on the FMA pipe (K2: 1 of 8)
                  fma_exp_share=0.125 if ffma else 0.25,
                  kernel="k_lse<3,4> (online LSE pass, FFMA cross term, K2)" if ffma else
                         "k_lse_tc2 (online LSE pass, tcgen05 cross term (d = 3 in one K = 16 step, 3-product "
                         "fp16 split) with w and the row shift folded into the MMA, K3)")
        if not ffma:
            sp["traffic_note"] = ("DRAM bytes of one seeded K3 column pass (ncu): both sides' operand images (compact "
                                  "K = 16 layout, 132 B per point, 35 MB per side) and the partials; the kernel is "
                                  "MUFU/FMA-bound, far from HBM bandwidth")
    else:
        sp.update(p=gen.c5(d=args.d or 64, eps_factor=args.eps_factor or 1e-2), init=args.init or "gaussian", mode="online",
                  roof="tensor", scaling="strong", kernel="k_lse_tc2 (online LSE pass, CTA-pair tcgen05 kind::f16 3-product hi/lo "
                                        "cross term with w and the row shift folded into the MMA, K3)")
        if args.ffma:   # comparison leg: the FFMA kernel at d = 64
            sp.update(roof="fp32", kernel="k_lse<64,1> (online LSE pass, FFMA2 cross term, K2)")
    return sp


def single_config(sp, args, world):
    p, name = sp["p"], sp["name"]
    sharded = name in ("c4", "c5") and (world > 1 or args.force_sharded)
    c = {"workload": {"c1": "BJ.cfg1 (C1): n=m=256, d=2, Gaussian clouds, eps=0.01*mean(C)",
                      "c3": f"BJ.cfg3 (C3): n=m=16384, d=16 GMM clouds, stored-cost mode (1 GiB C), eps={p.eps:.4g}",
                      "c4": "BJ.cfg4 (C4): n=m=262144, d=3 RGB-pixel mixtures, eps=1e-2, online cost",
                      "c5": f"BJ.cfg5 (C5): n=m=65536, d={p.d} embeddings, eps={p.eps:.4g}, online cost"
                            + ("" if p.d == 64 else " (the BJ.cfg5 recipe at another d: not a BASELINE configuration)")}[name],
         "n": p.n, "m": p.m, "d": p.d, "init": sp["init"], "tol": p.tol, "mode": sp["mode"],
         "parallelism": f"row-sharded x{world} (NCCL allgather of block partials per sweep)" if sharded else
                        ("1 GPU" if world == 1 else f"{world} independent replicas"),
         "l2": "flushed (256 MiB write) before every timed step" if name in ("c1",) else
               "inputs + cost larger than L2 / flushed before each step"}
    if sp["init"] == "subsample":
        c["subsample"] = {"ns": int(p.extra["idx_x"].size), "inner_tol": p.tol / 10}
    if sp["init"] == "gmm":
        c["gmm_fit"] = {"K": 8, "kmeans_iters": args.gmm_kmeans_iters, "em_max_iters": args.gmm_iters,
                        "em_tol": args.gmm_tol, "start": "gen.gmm_start_idx seeds 3/4 (R-23/R-28)"}
    if name == "c5" and args.ffma:
        c["kernel_variant"] = "FFMA cross term (sk_set_tuning tc=0)"
    if args.tune:
        c["tuning"] = dict(t.split("=", 1) for t in args.tune)
    return c


class Single(Workload):
    """One problem (C1, C3, C4, C5); C4 is row-sharded over the ranks."""

    def __init__(self, sk, ctx, dev, rank, world, args):
        import torch
        self.sk, self.ctx, self.world, self.rank, self.args = sk, ctx, world, rank, args
        self.spec = sp = single_spec(args)
        self.name, self.p, self.init, self.mode, self.roof = sp["name"], sp["p"], sp["init"], sp["mode"], sp["roof"]
        self.kernel, self.scaling, self.fma_exp_share = sp["kernel"], sp["scaling"], sp["fma_exp_share"]
        self.traffic_note = sp.get("traffic_note")
        if self.name == "c5" and args.ffma:
            ctx.set_tuning("tc", 0)
        p = self.p
        self.n, self.m, self.d = p.n, p.m, p.d
        # C4 and C5 (BJ.cfg4/5: "1/2/4/8 GPUs") shard their rows; C1/C3 run replicas
        self.sharded = self.name in ("c4", "c5") and (world > 1 or args.force_sharded)
        if self.sharded:
            from paper_2206_07630_b200 import dist as skd
            skd.init_comm(ctx)
            if world == 1:   # (--force-sharded: the 1-rank communicator takes the NCCL data plane)
                ctx.set_force_nccl(True)
        self.row0, self.nl = sk.shard_rows(p.n, rank, world) if self.sharded else (0, p.n)
        self.x = torch.from_numpy(p.x).to(dev)
        self.y = torch.from_numpy(p.y).to(dev)
        self.xh = torch.from_numpy(p.x).pin_memory()
        self.yh = torch.from_numpy(p.y).pin_memory()
        self.dev = dev
        if self.init == "gmm_given":   # the generating mixtures as the GMM parameters (no fitting)
            self.gx = {k: torch.from_numpy(v).to(dev) for k, v in p.extra["gmm_x"].items()}
            self.gy = {k: torch.from_numpy(v).to(dev) for k, v in p.extra["gmm_y"].items()}
        if self.init == "gmm":          # fit both K = 8 GMMs (on the device, K16) inside the step
            from workloads import gen as _g
            self.gmm_idx = (_g.gmm_start_idx(p.n, 8, 3), _g.gmm_start_idx(p.m, 8, 4))
        if self.init == "subsample":
            self.ix = torch.from_numpy(p.extra["idx_x"]).to(dev)
            self.iy = torch.from_numpy(p.extra["idx_y"]).to(dev)

    def config(self):
        return single_config(self.spec, self.args, self.world)

    def _init(self, x, y):
        sk, p = self.sk, self.p
        if self.init == "gaussian":
            f0, _ = sk.sinkhorn_init_gaussian(self.ctx, x, y)
        elif self.init == "gmm":
            gx, _ = sk.sinkhorn_fit_gmm(self.ctx, x, 8, self.gmm_idx[0], iters=self.args.gmm_iters,
                                        kmeans_iters=self.args.gmm_kmeans_iters, tol=self.args.gmm_tol)
            gy, _ = sk.sinkhorn_fit_gmm(self.ctx, y, 8, self.gmm_idx[1], iters=self.args.gmm_iters,
                                        kmeans_iters=self.args.gmm_kmeans_iters, tol=self.args.gmm_tol)
            f0, _ = sk.sinkhorn_init_gmm(self.ctx, x, y, gx, gy, p.eps)
        elif self.init == "gmm_given":
            gx, gy = self.gx, self.gy
            if not x.is_cuda:
                gx = {k: v.cpu() for k, v in gx.items()}
                gy = {k: v.cpu() for k, v in gy.items()}
            f0, _ = sk.sinkhorn_init_gmm(self.ctx, x, y, gx, gy, p.eps)
        elif self.init == "subsample":
            ix, iy = (self.ix, self.iy) if x.is_cuda else (self.ix.cpu(), self.iy.cpu())
            f0, _, self.inner = sk.sinkhorn_init_subsample(self.ctx, x, y, ix, iy, p.eps, p.tol / 10)
        else:
            f0 = None
        return f0

    def _run(self, x, y, init=True, anderson=None, adaptive=None):
        import torch
        sk, p = self.sk, self.p
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        ev[0].record()
        f0 = self._init(x, y) if init else None
        ev[1].record()
        if self.sharded:
            xl = x[self.row0:self.row0 + self.nl]
            f0l = None if f0 is None else f0[self.row0:self.row0 + self.nl].contiguous()
            _, _, rep = sk.sinkhorn_solve_sharded(self.ctx, self.n, self.row0, xl, y, p.eps, tol=p.tol,
                                                  max_iter=p.max_iter, mode=self.mode, f_init_local=f0l)
        else:
            _, _, rep = sk.sinkhorn_solve(self.ctx, x, y, p.eps, tol=p.tol, max_iter=p.max_iter, mode=self.mode,
                                          f_init=f0, anderson=anderson, adaptive=adaptive)
        ev[2].record()
        ev[2].synchronize()
        self.split_ms = {"init_ms": ev[0].elapsed_time(ev[1]), "solve_call_ms": ev[1].elapsed_time(ev[2]),
                         "solve_loop_ms": rep["solve_ms"], "build_ms": rep["build_ms"]}
        self.rep = rep
        return float(self.n) * self.m * rep["iterations"] / (self.world if self.sharded else 1)   # this rank's share

    def step(self):
        e = self._run(self.x, self.y)
        self.step_L = self.rep["iterations"]
        return e

    def e2e_step(self):
        e = self._run(self.xh, self.yh)
        n, m, d = self.n, self.m, self.d
        h2d = 2 * (n * d + m * d) * 4 + n * 4
        d2h = n * 4 + n * 4 + m * 4
        return e, h2d, d2h

    def baseline(self):
        self._run(self.x, self.y, init=False)
        return {"init": "zero", "iterations": self.rep["iterations"]}

    def extra(self):
        out = {"iterations": self.rep["iterations"], "converged": self.rep["converged"],
               "dual_objective": self.rep["dual_objective"], "build_ms": self.rep["build_ms"],
               "last_step_split_ms": getattr(self, "split_ms", None)}
        if hasattr(self, "inner"):
            out["subsample_inner_iterations"] = self.inner["iterations"]
        if not self.sharded and not self.args.no_anderson:   # NEXT-1: Anderson (memory 5, R-27), same step
            import torch
            reps = 5 if self.name == "c1" else (1 if self.name == "c4" else 3)
            self._run(self.x, self.y, anderson=5)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps):
                ent = self._run(self.x, self.y, anderson=5)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            out["anderson5"] = {"time_to_tol_ms": ms, "iterations": self.rep["iterations"],
                                "converged": self.rep["converged"], "cost_entries_per_s": ent / (ms / 1e3),
                                "solve_ms": self.rep["solve_ms"],
                                "note": "same init + Anderson (memory 5) to the same tol (K13 / K19)"}
            # adaptive momentum (window 10; R-31), same step
            self._run(self.x, self.y, adaptive=10)
            e0.record()
            for _ in range(reps):
                ent = self._run(self.x, self.y, adaptive=10)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            out["adaptive10"] = {"time_to_tol_ms": ms, "iterations": self.rep["iterations"],
                                 "converged": self.rep["converged"],
                                 "cost_entries_per_s": ent / (ms / 1e3),
                                 "note": "same init + adaptive momentum (window 10) to the same tol"}
        return out

    def cpu_sample(self, target_s=10.0):
        return single_cpu_sample(self.p, target_s)

    def cpu_extra(self, target_s=10.0):
        """Beside the sampled sweep: the oracle's time-to-tol extrapolated from it (L of our solve
        x the measured fp64 sweep time; the initializer likewise), and a full fp64 run (init +
        solve to tol) of the same recipe at reduced n (full runs take hours)."""
        from oracle import oracle as O
        from workloads import gen
        e, t, thr, _ = single_cpu_sample(self.p, target_s / 2)
        rate = e / t                      # cost entries (one per sweep = 2 passes) per second
        p, L = self.p, self.step_L
        out = {"kind": "oracle", "cores": thr, "sweep_entries_per_s": rate,
               "time_to_tol_s_extrapolated": (p.n * p.m * L) / rate,
               "extrapolation": f"L = {L} sweeps (this run's) x n m / measured fp64 sweep rate"}
        if self.init == "subsample" and hasattr(self, "inner"):
            ns = int(p.extra["idx_x"].size)
            out["init_s_extrapolated"] = (ns * ns * self.inner["iterations"] + p.n * ns / 2) / rate
        if self.name == "c5":   # full fp64 run at reduced n: Gaussian init + solve to tol (same eps factor)
            q = gen.c5(n=1024, eps_factor=self.args.eps_factor or 1e-2)
            t0 = time.perf_counter()
            f0, _ = O.init_gaussian(q.x, q.y)
            r = O.sinkhorn(q.x, q.y, q.eps, tol=q.tol, f0=f0)
            tt = time.perf_counter() - t0
            out["reduced_n_full_run"] = {"n": q.n, "iterations": r.iterations, "time_to_tol_s": tt,
                                         "value": q.n * q.m * r.iterations / tt, "unit": "cost-entries/s"}
        if self.name == "c4":   # full fp64 run at reduced n: subsample init + solve to tol
            q = gen.c4(n=2048, ns=256)
            t0 = time.perf_counter()
            f0 = O.init_subsample(q.x, q.y, q.extra["idx_x"], q.extra["idx_y"], q.eps, q.tol / 10)
            f0 = f0[0] if isinstance(f0, tuple) else f0
            r = O.sinkhorn(q.x, q.y, q.eps, tol=q.tol, f0=f0)
            tt = time.perf_counter() - t0
            out["reduced_n_full_run"] = {"n": q.n, "ns": 256, "iterations": r.iterations, "time_to_tol_s": tt,
                                         "value": q.n * q.m * r.iterations / tt, "unit": "cost-entries/s"}
        return out


def single_cpu_sample(p, target_s=10.0):
    """The fp64 oracle timed on a bounded sample of one sweep: the g-update (column pass) on
    sampled columns and the f-update (row pass) on sampled rows, sized to take about target_s
    seconds.  Returns (cost entries, seconds, threads, description); one cost entry = 2 passes."""
    from oracle import oracle as O
    g, f = np.zeros(p.m), np.zeros(p.n)

    def run(k):
        rows = np.linspace(0, p.n - 1, k).astype(np.int64)
        cols = np.linspace(0, p.m - 1, k).astype(np.int64)
        t0 = time.perf_counter()
        O.g_update(p.x, p.y, f, p.eps, cols=cols)
        O.f_update(p.x, p.y, g, p.eps, rows=rows)
        return time.perf_counter() - t0
    k = min(p.n, p.m, 16)
    t = run(k)
    k = int(min(p.n, p.m, max(k, k * target_s / max(t, 1e-4))))
    t = run(k)
    return float(k) * (p.m + p.n) / 2, t, O.num_threads(), \
        f"oracle sweep sample: g-update on {k} sampled columns + f-update on {k} sampled rows " \
        f"(of {p.n} x {p.m}); one cost entry = 2 passes"


def make_workload(args, sk, ctx, dev, rank, world):
    return C2(sk, ctx, dev, rank, world, args) if args.workload == "c2" else Single(sk, ctx, dev, rank, world, args)


def roofline(w, cnt, steps, pk, src, step_ms, clocks=None):
    """Roofline of the dominant kernel: ALGORITHMIC units per launch / its average launch
    duration, both from the library's per-launch CUDA events on the launching stream
    (sk_counters.dom_*: launches that returned at entry after the stop flag are excluded)."""
    sm_max = float(pk.get("sm_max_mhz", 1965.0))
    nl = max(int(cnt["dom_launches"]), 1)
    dom_s = cnt["dom_ms"] / 1e3
    common = {"kernel": w.kernel, "launches": int(cnt["dom_launches"]),
              "avg_launch_ms": cnt["dom_ms"] / nl,
              "share_of_step": (cnt["dom_ms"] / max(steps, 1)) / step_ms if step_ms > 0 else None,
              "traffic": traffic_from_profile(w)}
    if getattr(w, "traffic_note", None):
        common["traffic_note"] = w.traffic_note
    if w.roof == "hbm":
        achieved = cnt["dom_bytes"] / dom_s / 1e9 if dom_s > 0 else 0.0
        peak = float(pk["hbm_gbs"])
        return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({src})",
                "algorithmic": "4 bytes (one fp32 C_ij read) per cost entry per launch; the fused sweep reads C "
                               "once for a row pass and the next column pass",
                "bytes_per_launch": cnt["dom_bytes"] / nl, **common}
    if w.roof == "tensor":
        kpad = 16 * ((int(w.d) + 15) // 16)   # the MMA K steps K3 issues (d = 64: 64)
        flops = cnt["dom_entries"] * 3 * 2 * kpad        # 3 fp16 MMAs (hi.hi, hi.lo, lo.hi), K = d padded to 16
        achieved = flops / dom_s / 1e12 if dom_s > 0 else 0.0
        # K3 runs inside a long step (many back-to-back launches): the sustained figure
        # (fp16 dense = bf16 dense rate); the burst one beside it
        peak = float(pk.get("bf16_tflops_sustained", pk["bf16_tflops"]))
        ex2_peak = N_SM * MUFU_EX2_PER_CLK_SM * sm_max * 1e6
        ent_s = cnt["dom_entries"] / dom_s if dom_s > 0 else 0.0
        return {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "peak_source": f"MEASURED_PEAKS.json bf16_tflops_sustained (kernel timed inside a long step; fp16 "
                               f"runs at the bf16 rate), {src}",
                "frac_of_burst": achieved / float(pk["bf16_tflops"]),
                "algorithmic": f"3 x 2 x {kpad} fp16 tensor flops per cost entry per pass (3-product hi/lo split, "
                               f"K = d padded to 16)",
                "flops_per_launch": flops / nl,
                "mufu_frac": ent_s / ex2_peak,
                # under the 1000 W cap the SM clock drops: the fraction of the burst rate at the
                # clock the run actually had (the tensor pipe's own utilisation, ncu's view)
                "frac_of_burst_at_observed_clock": (achieved / float(pk["bf16_tflops"])) * sm_max /
                                                   float((clocks or {}).get("sm_mhz") or sm_max),
                **common}
    if w.roof == "fp32":
        flops = cnt["dom_entries"] * 2 * w.d            # d FMAs per entry for the cross term
        achieved = flops / dom_s / 1e12 if dom_s > 0 else 0.0
        peak = N_SM * 128 * 2 * sm_max * 1e6 / 1e12
        return {"bound": "alu", "pipe": "FP32 FMA", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak,
                "peak_source": f"derived: {N_SM} SM x 128 FP32 lanes x 2 flop x {sm_max:.0f} MHz ({src})",
                "algorithmic": "2 d flops (the cross term's d FMAs) per cost entry per pass",
                "flops_per_launch": flops / nl, **common}
    achieved = cnt["dom_entries"] / dom_s if dom_s > 0 else 0.0
    peak = N_SM * MUFU_EX2_PER_CLK_SM * sm_max * 1e6
    share = float(getattr(w, "fma_exp_share", 0.0))
    return {"bound": "alu", "pipe": "MUFU.EX2 (SFU)", "achieved": achieved / 1e9,
            "peak": peak / 1e9, "unit": "Gex2/s", "frac": achieved / peak,
            "exp_on_fma_share": share, "xu_frac": (1.0 - share) * achieved / peak,
            "frac_note": "achieved counts every cost entry's exponential; a share of them runs on the FMA pipe "
                         "(Cody-Waite + polynomial), so frac is exponentials per MUFU slot and xu_frac the XU "
                         "pipe's own utilisation",
            "peak_source": f"derived: {N_SM} SM x {MUFU_EX2_PER_CLK_SM} ex2/clk x {sm_max:.0f} MHz "
                           f"(sm_max_mhz from MEASURED_PEAKS.json, {src})",
            "algorithmic": "one exp2 per cost entry per pass; 2 passes per sweep (+1 column pass for err_L)",
            "ex2_per_launch": cnt["dom_entries"] / nl, **common}


def traffic_from_profile(w):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel from the
    committed `ncu --set full` capture (profiles/traffic.json, written by tools/ncu_summary.py)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if w.name == "c5" and getattr(w, "d", 64) != 64:   # (the capture is of the d = 64 launch)
        return None
    try:
        t = json.load(open(p)).get(w.name)
        return t
    except Exception:
        return None


# ==================================================================== reference arm
def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    from oracle import oracle as O
    O.build()

    if args.workload == "c2":
        w = C2.__new__(C2)
        cfg = c2_config(world)
        sample = lambda warm: w.cpu_sample(1 if warm else 2)   # noqa: E731
        scaling = "weak"
    else:
        sp = single_spec(args)
        cfg = single_config(sp, args, world)   # the same dict as our arm's
        sample = lambda warm: single_cpu_sample(sp["p"], 1.0 if warm else 3.0)   # noqa: E731
        scaling = sp["scaling"]
    for _ in range(args.warmup):
        sample(True)
    tot_e, tot_t, thr, desc = 0.0, 0.0, 1, ""
    for _ in range(args.steps):
        e, t, thr, desc = sample(False)
        tot_e += e
        tot_t += t
    v = tot_e / tot_t
    line = {"impl": "reference", "metric": "sinkhorn_cost_entries_per_s", "value": v, "unit": "cost-entries/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {"value": v, "unit": "cost-entries/s", "cores": thr, "kind": "oracle", "sample": desc},
            "e2e": {"value": v, "unit": "cost-entries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ==================================================================== our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2206_07630_b200 as sk

    world, rank, local = dist_env()
    if world > 1 or args.force_sharded:
        torch.cuda.set_device(local)
        if "MASTER_ADDR" not in os.environ:   # (--force-sharded without torchrun: a 1-rank group)
            os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=os.environ.get("MASTER_PORT", "29531"),
                              RANK="0", WORLD_SIZE="1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    stream = torch.cuda.Stream(dev)
    ctx = sk.Context(dev.index, stream)
    for t in args.tune:
        key, val = t.split("=", 1)
        ctx.set_tuning(key, float(val))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[dev.index])
        torch.cuda.synchronize(dev)

    k14 = {}
    if rank == 0 and not args.no_k14:
        # K14 microbenchmarks: this device's MUFU / FP32 / HBM / fp16 tensor rates (roofline context)
        try:
            k14 = {"ex2_per_s": ctx.microbench("ex2"), "ffma_per_s": ctx.microbench("ffma"),
                   "hbm_read_GBps": ctx.microbench("hbm") / 1e9, "tc_f16_TFLOPs": ctx.microbench("tc") / 1e12}
        except Exception as ex:  # pragma: no cover
            k14 = {"error": repr(ex)}
    with torch.cuda.stream(stream):
        w = make_workload(args, sk, ctx, dev, rank, world)
        for _ in range(max(args.warmup, 0)):
            w.step()
    barrier()
    ctx.reset_counters()
    ctx.set_timing(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    entries = 0.0
    with ClockSampler(dev.index) as clk:
        barrier()
        for s in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(float(s))                     # L2 flush, outside the timed events
                ev[s][0].record(stream)
                entries += w.step()
                ev[s][1].record(stream)
        barrier()
    ctx.set_timing(False)
    cnt = ctx.counters()
    ms = sum(a.elapsed_time(b) for a, b in ev)
    from paper_2206_07630_b200 import dist as skd
    ms_all = skd.max_over_ranks([ms], device=dev)[0] if world > 1 else ms
    entries_all = skd.sum_over_ranks([entries], device=dev)[0] if world > 1 else entries
    value = entries_all / (ms_all / 1e3)
    with torch.cuda.stream(stream):   # (extra() times its own kernels on the library's stream)
        extra = w.extra()

    # ---- e2e: the same step through the C ABI with pinned HOST buffers, copies inside the timing
    e2e_ms, e2e_entries, h2d, d2h = 0.0, 0.0, 0, 0
    # (short steps: more of them, so that one host hiccup does not decide the mean; all ranks
    # derive the same count from the max-over-ranks step time)
    e2e_steps = max(1, min(args.steps, 5)) if ms_all / args.steps >= 100.0 else max(5, min(4 * args.steps, 40))
    with torch.cuda.stream(stream):
        w.e2e_step()            # untimed warm-up: the library's staging buffers are allocated once
    torch.cuda.synchronize(dev)
    for s in range(e2e_steps):
        with torch.cuda.stream(stream):
            flush.fill_(float(s))
        torch.cuda.synchronize(dev)   # the L2 flush completes outside the timed region
        barrier()
        t0 = time.perf_counter()
        with torch.cuda.stream(stream):
            e, h2d, d2h = w.e2e_step()
        torch.cuda.synchronize(dev)
        e2e_ms += 1e3 * (time.perf_counter() - t0)
        e2e_entries += e
    if world > 1:
        e2e_ms = skd.max_over_ranks([e2e_ms], device=dev)[0]
        e2e_entries = skd.sum_over_ranks([e2e_entries], device=dev)[0]

    # ---- time-to-tol of the zero initializer (context for the initializer's effect)
    with torch.cuda.stream(stream):
        flush.fill_(0.0)
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        zero = w.baseline()
        e1.record(stream)
    torch.cuda.synchronize(dev)
    zero["time_to_tol_ms"] = e0.elapsed_time(e1)

    if rank == 0:
        pk, src = peaks()
        line = {
            "metric": "sinkhorn_cost_entries_per_s", "value": value, "unit": "cost-entries/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_all / args.steps, "higher_is_better": True, "scaling": w.scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": w.config(),
            "time_to_tol_ms": {"init": ms / args.steps, "zero_init": zero["time_to_tol_ms"]},
            "solve": extra, "zero_init": zero,
            "roofline": roofline(w, cnt, args.steps, pk, src, ms_all / args.steps, clk.summary()),
            "gpu_launches": int(cnt["kernel_launches"]),
            "clocks": clk.summary(),
            "k14_measured_peaks": k14,
            "e2e": {"value": e2e_entries / (e2e_ms / 1e3), "unit": "cost-entries/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": e2e_steps},
        }
        if not args.no_cpu_baseline:
            try:
                e, t, thr, desc = w.cpu_sample()
                line["cpu_baseline"] = {"value": e / t, "unit": "cost-entries/s", "cores": thr, "kind": "oracle",
                                        "sample": f"{desc}, {t:.1f} s"}
                if hasattr(w, "cpu_extra"):
                    line["cpu_baseline"].update(w.cpu_extra())
            except Exception as ex:  # pragma: no cover
                line["cpu_baseline"] = {"value": None, "error": repr(ex)}
        print(json.dumps(line), flush=True)
    if dist.is_initialized():
        dist.barrier(device_ids=[dev.index])
        dist.destroy_process_group()
    ctx.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c1", "c2", "c3", "c4", "c5"])
    ap.add_argument("--ffma", action="store_true", help="c5: the FFMA cross-term kernel (sk_set_tuning tc=0)")
    ap.add_argument("--tune", action="append", default=[], metavar="KEY=VALUE",
                    help="sk_set_tuning diagnostic knob (repeatable; recorded in config)")
    ap.add_argument("--force-sharded", action="store_true",
                    help="c4 at N=1 through the sharded entry with a 1-rank NCCL communicator (test of the N>1 path)")
    ap.add_argument("--init", default=None,
                    help="c3/c4/c5 initializer: zero|gaussian|gmm (fitted on the device)|gmm_given|subsample")
    ap.add_argument("--gmm-iters", type=int, default=100, help="max EM iterations of the device GMM fit (init gmm; "
                    "sklearn's default max_iter)")
    ap.add_argument("--gmm-tol", type=float, default=1e-3, help="EM convergence tol (sklearn's default; 0 = run "
                    "all --gmm-iters)")
    ap.add_argument("--no-anderson", action="store_true", help="skip the Anderson time-to-tol extra")
    ap.add_argument("--gmm-kmeans-iters", type=int, default=10,
                    help="Lloyd steps of the fit's k-means start (R-28; sklearn's default start), 0 = start at x[idx]")
    ap.add_argument("--eps-factor", type=float, default=None)
    ap.add_argument("--d", type=int, default=None,
                    help="c5 only: the BJ.cfg5 recipe at another dimension (17..256; K3 in K chunks above 64)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-k14", action="store_true", help="skip the K14 microbenchmarks")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

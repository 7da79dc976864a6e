#!/usr/bin/env python
"""CoFEM benchmark: EM iterations/sec on the BASELINE.json headline workload.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config dense-large] [--precision fp32|fp64]

A "step" is one CoFEM EM iteration (E-step: blocked PCG over K+1 = 21
right-hand sides to tol 1e-5 / cap 200 steps; fused diagonal estimate and
M-step) on the dense Gaussian CS problem N=16384, D=65536 (Phi 4 GiB fp32).
The timed K steps start from alpha = 1 after W warm-up iterations, so
--steps 20 times exactly the 20-iteration job BASELINE.json names.

value : device-timed (CUDA events on the library's stream), Phi resident in
        HBM, max over ranks; Phi column-sharded across ranks for N > 1.
e2e   : the public API ``run_cofem(problem, cfg)`` from host numpy buffers
        (Phi upload, per-iteration probe upload, result read-back inside).
--impl reference : the reference's CPU algorithm (the bit-exact numpy
        oracle of oracle/, float64, all host threads) on a bounded sample of
        the same workload, rank 0 only.

Inputs: Phi is 4 GiB >> 126 MB L2, so every PCG pass streams it from HBM
(no L2 flush needed).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "CoFEM EM iters/sec at D=65536,N=16384,K=20 (fp32)"
METRICS = {"conv-large": "CoFEM EM iters/sec, convolution dictionary N=D=2^22, 256 taps, K=30",
           "dct-large": "CoFEM EM iters/sec, 2-D partial DCT 1024x1024 (D=2^20, 25% kept), K=20"}
UNIT = "EM iter/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="dense-large")
    ap.add_argument("--precision", default="auto", choices=["auto", "fp32", "fp64", "ozaki", "ozaki24"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm, smax, reasons, power = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
                power.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": smax, "reasons": ["unsampled"]}
        loaded = [v for v in sm if v > 0.5 * max(sm)] or sm
        return {"sm_mhz": float(np.median(loaded)), "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(power) if power else None}


# -------------------------------------------------------------- roofline ----
def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def profiled_traffic(config, precision):
    path = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(path):
        return None
    d = json.load(open(path))
    return d.get(f"{config}/{precision}")


# ----------------------------------------------------------- CPU baseline ---
class CpuBaseline:
    """Reference CPU algorithm (bit-exact oracle, float64, all BLAS threads) on
    the full-size system for a bounded number of PCG steps; EM it/s =
    1 / (time per PCG step * PCG steps per EM iteration + M-step time)."""

    def __init__(self, c):
        from oracle import cofem_oracle as O
        from paper_2105_10439_b200 import simulate as S

        self.O, self.c = O, c
        phi32 = S.gaussian_dictionary(c.N, c.D, c.seed)
        self.op = O.dense_op(phi32)
        y = S.observe(phi32, S.sparse_signal(c.D, c.n_spikes, c.seed), c.sigma, c.seed)
        del phi32
        probes = O.draw_rademacher(c.D, c.K, O.substream(c.seed, 3))
        self.rhs = np.concatenate([probes, self.op.adjoint(y[:, None])], axis=1)
        alpha = np.ones(c.D)
        self.minv = 1.0 / (c.beta + alpha)
        self.fn = lambda V: O.system_apply(self.op, c.beta, alpha, V)  # noqa: E731
        O.pcg_solve(self.fn, self.rhs, self.minv, O.CgConfig(max_steps=1, tolerance=1e-300))  # warm BLAS

    def sample(self, seconds, steps_per_em, steps_source="the GPU arm's measured count in this invocation"):
        O, c = self.O, self.c
        steps, t0 = 0, time.perf_counter()
        while time.perf_counter() - t0 < seconds:
            O.pcg_solve(self.fn, self.rhs, self.minv, O.CgConfig(max_steps=2, tolerance=1e-300))
            steps += 2
        dt = time.perf_counter() - t0
        per_step = dt / steps
        t_m = time.perf_counter()
        O.m_step(np.ones(c.D), np.ones(c.D))
        t_m = time.perf_counter() - t_m
        cores = os.cpu_count()
        return {
            "value": 1.0 / (per_step * steps_per_em + t_m),
            "unit": UNIT,
            "cores": cores,
            "kind": "port",
            "projected": True,
            "sample": (f"{steps} PCG steps ({dt:.1f}s) of the full N={c.N},D={c.D},Q={c.K + 1} float64 system "
                       f"with the bit-exact numpy oracle (reference algorithm, numpy BLAS on {cores} threads); "
                       f"EM it/s = 1 / ({per_step * 1e3:.1f} ms/PCG step x {steps_per_em:.2f} PCG steps per EM "
                       f"iteration [{steps_source}] + M-step)"),
            "ms_per_pcg_step": per_step * 1e3,
            "pcg_steps_per_sec": 1.0 / per_step,
            "pcg_steps_per_em_iteration": steps_per_em,
            "pcg_steps_sampled": steps,
            "sample_seconds": dt,
        }


# --------------------------------------------------------------- our arm ----
def run_ours(args):
    import torch

    from paper_2105_10439_b200 import _lib
    from paper_2105_10439_b200 import simulate as S

    world, rank, local = dist_env()
    if args.config in S.CONV_CONFIGS or args.config in S.DCT_CONFIGS:
        return run_ours_conv(args)
    c = S.CONFIGS[args.config]
    dist = None
    if world > 1:
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    device = local if world > 1 else 0
    prec = {"fp32": _lib.FP32, "fp64": _lib.FP64, "ozaki": _lib.OZAKI, "ozaki24": _lib.OZAKI24}[args.precision]

    # ---- device-resident run (value) ----
    from paper_2105_10439_b200.distributed import column_shards

    shards = column_shards(c.D, world)
    c0, c1 = shards[rank]
    ctx = _lib.Context(c.N, c1 - c0, prec, device)
    ctx.set_shard(c0, c.D)
    ctx.generate_gaussian(seed=20250101, scale=1.0 / np.sqrt(c.N))
    if world > 1:
        from paper_2105_10439_b200.distributed import broadcast_nccl_id

        ctx.set_comm(broadcast_nccl_id(dist, rank, device), world, rank)
    z = S.sparse_signal(c.D, c.n_spikes, c.seed)
    y = ctx.apply(z[c0:c1, None])[:, 0] + c.sigma * np.random.default_rng(2).standard_normal(c.N)
    dseed = 0xC0FE
    ctx.bench_prepare(y, c.beta, c.K, c.U, c.tol, seed=dseed)
    if args.warmup:
        ctx.bench_iterations(args.warmup)
    ctx.bench_prepare(y, c.beta, c.K, c.U, c.tol, seed=dseed)  # job starts at alpha = 1
    if dist:
        dist.barrier()
    torch.cuda.synchronize(device)
    with ClockSampler(device) as clk:
        tim = ctx.bench_iterations(args.steps, time_kernels=True)
    torch.cuda.synchronize(device)
    if dist:
        dist.barrier()
    total_ms = tim["total_ms"]
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = args.steps / (total_ms / 1e3)
    pcg_steps = tim["pcg_steps"]
    steps_per_em = pcg_steps / args.steps

    # roofline of the dominant kernel (the Phi contraction with more device time)
    q = c.K + 1
    d_local = c1 - c0
    phi_entry = 3.0 if args.precision == "ozaki24" else 4.0  # bytes per streamed Phi entry
    phi_bytes = phi_entry * c.N * d_local
    vec_bytes = 4.0 * (c.N + d_local) * q if args.precision == "fp32" else 8.0 * (c.N + d_local) * q
    alg_bytes = phi_bytes + vec_bytes
    fwd_avg = tim["fwd_ms"] / max(tim["fwd_launches"], 1)
    bwd_avg = tim["bwd_ms"] / max(tim["bwd_launches"], 1)
    dom, avg_ms = ("bwd (Phi^T U)", bwd_avg) if tim["bwd_ms"] >= tim["fwd_ms"] else ("fwd (Phi P)", fwd_avg)
    peak, peak_src = measured_peaks()
    achieved = alg_bytes / (avg_ms / 1e3) / 1e9
    line = {
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": total_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": {"ozaki": "i8 x i8 -> exact i32 Phi contractions (32-bit fixed-point Phi), f64 vectors",
                  "ozaki24": "i8 x i8 -> exact i32 Phi contractions (24-bit fixed-point Phi, 3 B/entry), f64 vectors",
                  "fp64": "f64 (fp32 Phi)", "fp32": "f32 (fp64 scalars)"}[args.precision],
        "data": "synthetic (Gaussian Phi from a device Philox stream, 1% N(0,1) spikes, sigma=0.01)",
        "config": {"workload": f"{args.config}: dense Gaussian CS N={c.N} D={c.D} K={c.K} T={c.T} "
                               f"PCG cap {c.U} tol {c.tol}", "N": c.N, "D": c.D, "K": c.K,
                   "pcg_max_steps": c.U, "pcg_tol": c.tol, "parallelism": f"column-shard x{world}",
                   "l2": "Phi 4 GiB >> 126 MB L2: every pass streams HBM, no flush needed"},
        "pcg_steps_per_sec": pcg_steps / (total_ms / 1e3),
        "pcg_steps_per_em_iteration": steps_per_em,
        "gpu_launches": int(tim["kernel_launches"]),
        "clocks": clk.summary(),
        "roofline": {
            "bound": "hbm",
            "kernel": dom,
            "achieved": achieved,
            "peak": peak,
            "unit": "GB/s",
            "frac": achieved / peak,
            "traffic": profiled_traffic(args.config, args.precision),
            "algorithmic_bytes_per_launch": alg_bytes,
            "avg_launch_ms": avg_ms,
            "peak_source": peak_src,
            "fwd_avg_ms": fwd_avg,
            "bwd_avg_ms": bwd_avg,
            "contraction_share_of_step": (tim["fwd_ms"] + tim["bwd_ms"]) / tim["total_ms"],
            "step_hbm_frac": (2 * alg_bytes * pcg_steps / (total_ms / 1e3) / 1e9) / peak,
            # the same step against streaming a 4-byte (fp32) Phi twice per PCG step:
            # > 1 means faster than any fp32-Phi implementation can be on this HBM
            "step_frac_of_fp32_phi_roofline": (2 * (4.0 * c.N * d_local + vec_bytes) * pcg_steps
                                               / (total_ms / 1e3) / 1e9) / peak,
        },
    }
    ctx.close()
    del ctx

    # ---- end to end through the public API (host buffers) ----
    if not args.no_e2e:
        from paper_2105_10439_b200 import run_cofem

        phi = S.gaussian_dictionary(c.N, c.D, c.seed)
        prob, _, _ = S.dense_cs_problem(c, phi=phi)
        cfg = c.cofem_config(args.precision, iterations=args.steps)
        if dist:
            from paper_2105_10439_b200.distributed import run_cofem_sharded

            dist.barrier()
            t0 = time.perf_counter()
            st, est, diag = run_cofem_sharded(prob, cfg, device=device)
            torch.cuda.synchronize(device)
            el = time.perf_counter() - t0
            t = torch.tensor([el], dtype=torch.float64, device=f"cuda:{device}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        else:
            prof = None
            if os.environ.get("BENCH_E2E_PROFILE"):  # where the host time of the e2e call goes (stderr)
                import cProfile

                prof = cProfile.Profile()
                prof.enable()
            t0 = time.perf_counter()
            st, est, diag = run_cofem(prob, cfg)
            el = time.perf_counter() - t0
            if prof:
                import pstats

                prof.disable()
                pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(8)
            prob.op.release()
        h2d = (4.0 * c.N * c.D + 8.0 * c.N + 32.0) / args.steps
        d2h = 8.0 * 3 * c.D / args.steps + 12.0
        line["e2e"] = {"value": args.steps / el, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                       "seconds": el, "pcg_steps": int(sum(d["cg_steps"] for d in diag)),
                       "note": "run_cofem(problem, cfg) on host numpy Phi/y, context created inside the timed "
                               "region: Phi upload + digit planes once (amortised over the steps), probes drawn "
                               "on the device from the reference's PCG64 stream (32-byte state), per-iteration "
                               "CG steps/residuals and alpha/mu/s read back"}
    if rank == 0 and not args.no_cpu and world == 1:
        line["cpu_baseline"] = CpuBaseline(c).sample(args.cpu_seconds, steps_per_em)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def run_ours_conv(args):
    """BASELINE configs 3 (banded int8 convolution) and 4 (2-D partial DCT), single GPU."""
    import torch

    from paper_2105_10439_b200 import run_cofem
    from paper_2105_10439_b200 import simulate as S

    world, rank, local = dist_env()
    is_conv = args.config in S.CONV_CONFIGS
    if world > 1 and not is_conv:
        raise SystemExit("2-D DCT dictionaries run on one GPU (their transposes are not sharded)")
    c = S.CONV_CONFIGS[args.config] if is_conv else S.DCT_CONFIGS[args.config]
    prob, z = S.conv_problem(c) if is_conv else S.dct2_problem(c)
    prec = args.precision if args.precision in ("ozaki", "ozaki24", "fp64") else "ozaki"
    dist, device, y_local = None, 0, np.asarray(prob.y)
    if world > 1:
        # time shards: each rank holds its samples; halo send/recv + scalar all-reduces over NCCL
        import torch.distributed as dist

        from paper_2105_10439_b200.distributed import ShardedContext, local_observation

        device = local
        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
        sharded = ShardedContext.for_operator(prob.op, "ozaki", device)
        ctx = sharded.ctx
        t0_, t1_ = sharded.col_range
        y_local = local_observation(prob.op, prob.y, t0_, t1_)
    else:
        ctx = prob.op.context(prec)
    dseed = 0xC0FE
    ctx.bench_prepare(y_local, c.beta, c.K, c.U, c.tol, seed=dseed)
    if args.warmup:
        ctx.bench_iterations(args.warmup)
    ctx.bench_prepare(y_local, c.beta, c.K, c.U, c.tol, seed=dseed)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(device)
    with ClockSampler(device) as clk:
        tim = ctx.bench_iterations(args.steps, time_kernels=True)
    torch.cuda.synchronize(device)
    if dist:
        dist.barrier()
    total_ms = tim["total_ms"]
    if dist:
        t = torch.tensor([total_ms], dtype=torch.float64, device=f"cuda:{device}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    value = args.steps / (total_ms / 1e3)
    pcg_steps = tim["pcg_steps"]
    q = c.K + 1  # real right-hand sides (the kernels pad to 24 / 32 columns; padding is not algorithmic)
    fwd_avg = tim["fwd_ms"] / max(tim["fwd_launches"], 1)
    bwd_avg = tim["bwd_ms"] / max(tim["bwd_launches"], 1)
    # the fused convolution step (one GPU, K + 1 <= 32)
    fused = is_conv and world == 1 and q <= 32 and not os.environ.get("COFEM_CONV_UNFUSED")
    if is_conv:
        d_loc = c.D // world  # per-rank launch (balanced time shards)
        # Phi P band: operand digit planes in (4 B / entry), fp64 V out; Phi^T V
        # band with the PCG combine fused: planes in, P in, Psi out -- or, in
        # the fused step, planes in, P in, R in and out (no Psi)
        if tim["bwd_ms"] >= tim["fwd_ms"]:
            if fused:
                dom = ("bwd (Phi^T V band + fused residual update: R -= gamma (beta Phi^T V + alpha P); "
                       "MMA-issue bound, see DESIGN.md)")
                alg_bytes = (4.0 + 8.0 + 8.0 + 8.0) * q * d_loc
            else:
                dom = ("bwd (Phi^T V band + fused combine: Psi = beta Phi^T V + alpha P; MMA-issue bound, "
                       "see DESIGN.md)")
                alg_bytes = (4.0 + 8.0 + 8.0) * q * d_loc
            avg_ms = bwd_avg
        else:
            dom, avg_ms = "fwd (Phi P band)", fwd_avg
            alg_bytes = (4.0 + 8.0) * q * d_loc
    else:  # the fused column pass: one fp64 n^2 x Q block in, one out (+ n^2 mask bytes)
        alg_bytes = 16.0 * q * c.D + c.D
        dom, avg_ms = "column pass (DCT-II, mask, DCT-III; fp64 FFT)", fwd_avg
    peak, peak_src = measured_peaks()
    achieved = alg_bytes / (avg_ms / 1e3) / 1e9
    line = {
        "metric": METRICS[args.config], "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None,
        "dtype": (("i8 x i8 -> exact i32, 24-bit taps (ozaki24) / f64" if prec == "ozaki24" else
                   "i8 x i8 -> exact i32 (ozaki) / f64") if is_conv else "f64 (FFT passes)"),
        "data": ("synthetic (Bernoulli(0.01) x Exp(1) spikes, exp(-t/20) filter, sigma=0.05)" if is_conv else
                 "synthetic (3% N(0,1) pixels, variable-density 25% DCT mask, sigma=0.01)"),
        "config": {"workload": (f"{args.config}: causal convolution N=D={c.D}, {c.ntaps} taps, K={c.K}, "
                                f"PCG cap {c.U} tol {c.tol}" if is_conv else
                                f"{args.config}: 2-D partial DCT n={c.n} (D={c.D}, N={prob.op.n_rows}), K={c.K}, "
                                f"PCG cap {c.U} tol {c.tol}"), "D": c.D, "K": c.K,
                   "parallelism": f"time-shard x{world}" if is_conv else "single GPU",
                   "precision": prec, "fused_step": fused},
        "pcg_steps_per_sec": pcg_steps / (total_ms / 1e3), "pcg_steps_per_em_iteration": pcg_steps / args.steps,
        "gpu_launches": int(tim["kernel_launches"]), "clocks": clk.summary(),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": profiled_traffic(args.config, args.precision),
                     "algorithmic_bytes_per_launch": alg_bytes, "avg_launch_ms": avg_ms, "peak_source": peak_src,
                     "contraction_share_of_step": (tim["fwd_ms"] + tim["bwd_ms"]) / tim["total_ms"]},
    }
    prob.op.release()
    if world > 1:
        sharded.ctx.close()
    if not args.no_e2e:
        cfg = c.cofem_config(prec, iterations=args.steps)
        if dist:
            from paper_2105_10439_b200.distributed import run_cofem_sharded

            dist.barrier()
        prof = None
        if os.environ.get("BENCH_E2E_PROFILE"):  # where the host time of the e2e call goes (stderr)
            import cProfile

            prof = cProfile.Profile()
            prof.enable()
        t0 = time.perf_counter()
        st, est, diag = run_cofem_sharded(prob, cfg, device) if dist else run_cofem(prob, cfg)
        el = time.perf_counter() - t0
        if prof:
            import pstats

            prof.disable()
            pstats.Stats(prof, stream=sys.stderr).sort_stats("tottime").print_stats(8)
        if dist:
            t = torch.tensor([el], dtype=torch.float64, device=f"cuda:{device}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
        prob.op.release()
        line["e2e"] = {"value": args.steps / el, "unit": UNIT,
                       "h2d_bytes_per_step": (8.0 * prob.op.n_rows + 32.0) / args.steps,
                       "d2h_bytes_per_step": 24.0 * c.D / args.steps + 12.0, "seconds": el,
                       "pcg_steps": int(sum(d["cg_steps"] for d in diag)),
                       "note": "run_cofem(problem, cfg) from host numpy y, context created inside the timed region, "
                               "probes drawn on the device from the reference's PCG64 stream"}
    if not args.no_cpu and world == 1:
        line["cpu_baseline"] = cpu_sample_conv(c, prob, args.cpu_seconds, pcg_steps / args.steps, is_conv)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


def cpu_sample_conv(c, prob, seconds, steps_per_em, is_conv=True,
                    steps_source="the GPU arm's measured count in this invocation"):
    """The reference algorithm (oracle: FFT convolution like operators.py:209-219
    or scipy.fft dctn, float64, numpy/scipy threads) on the full-size system."""
    from oracle import cofem_oracle as O

    op = O.conv_op(c.D, c.taps()) if is_conv else O.dct2_op(c.n, prob.op.mask)
    probes = O.draw_rademacher(c.D, c.K, O.substream(c.seed, 3))
    rhs = np.concatenate([probes, op.adjoint(np.asarray(prob.y)[:, None])], axis=1)
    alpha = np.ones(c.D)
    minv = 1.0 / (c.beta + alpha)
    fn = lambda V: O.system_apply(op, c.beta, alpha, V)  # noqa: E731
    from scipy import fft as sfft

    steps, t0 = 0, time.perf_counter()
    with sfft.set_workers(os.cpu_count()):  # the reference's scipy.fft calls, on every host thread
        while time.perf_counter() - t0 < seconds:
            O.pcg_solve(fn, rhs, minv, O.CgConfig(max_steps=1, tolerance=1e-300))
            steps += 1
    dt = time.perf_counter() - t0
    per = dt / steps
    return {"value": 1.0 / (per * steps_per_em), "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
            "projected": True,
            "sample": f"{steps} PCG steps ({dt:.1f}s) of the full D={c.D}, Q={c.K + 1} "
                      f"{'convolution' if is_conv else 'DCT'} system with the numpy oracle (scipy.fft like the "
                      f"reference, {os.cpu_count()} workers); EM it/s = 1 / ({per * 1e3:.0f} ms/PCG step x "
                      f"{steps_per_em:.2f} PCG steps per EM iteration [{steps_source}])",
            "ms_per_pcg_step": per * 1e3, "pcg_steps_per_sec": 1.0 / per, "pcg_steps_per_em_iteration": steps_per_em,
            "pcg_steps_sampled": steps, "sample_seconds": dt}


def reference_steps_per_em(config, T):
    """PCG steps per EM iteration of the reference itself at this config: the
    mean of the cg_steps its own run_cofem recorded (tests/golden/
    make_golden_large.py runs the real reference at the full size; golden
    files travel with the repo).  Falls back to the step cap when absent."""
    from paper_2105_10439_b200 import simulate as S

    name = {"dense-large": "cofem_dense-large_T20.npz", "dense-mid": "cofem_dense-mid_T30.npz",
            "dense-small": "cofem_dense-small.npz", "dct-large": "cofem_dct-large_T20.npz",
            "conv-large": "cofem_conv-large_T2.npz"}.get(config)
    path = os.path.join(ROOT, "tests", "golden", name) if name else None
    if path and os.path.exists(path):
        steps = np.load(path)["cg_steps"]
        return float(np.mean(steps[:T])), (f"mean cg_steps of the real reference's run_cofem at this config "
                                           f"({len(steps[:T])} EM iterations, tests/golden/{name})")
    cfgs = {**S.CONFIGS, **S.CONV_CONFIGS, **S.DCT_CONFIGS}
    return float(cfgs[config].U), "the PCG step cap (no reference run recorded)"


def run_reference(args):
    world, rank, local = dist_env()
    if rank != 0:
        return
    # torchrun pins OMP_NUM_THREADS=1 per rank; the CPU reference (rank 0 alone)
    # gets every host thread for its BLAS / FFT calls
    try:
        from threadpoolctl import threadpool_limits

        threadpool_limits(limits=os.cpu_count())
    except Exception:
        pass
    from paper_2105_10439_b200 import simulate as S

    structured = args.config in S.CONV_CONFIGS or args.config in S.DCT_CONFIGS
    if structured:
        is_conv = args.config in S.CONV_CONFIGS
        c = S.CONV_CONFIGS[args.config] if is_conv else S.DCT_CONFIGS[args.config]
        prob, _ = S.conv_problem(c) if is_conv else S.dct2_problem(c)
    else:
        c = S.CONFIGS[args.config]
        cb = CpuBaseline(c)
    steps_per_em, source = reference_steps_per_em(args.config, c.T)

    def sample(seconds):
        if structured:
            return cpu_sample_conv(c, prob, seconds, steps_per_em, is_conv, source)
        return cb.sample(seconds, steps_per_em, source)

    for _ in range(args.warmup):
        base = sample(0.5)
    per, pcg, secs = [], 0, 0.0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        base = sample(max(0.5, args.cpu_seconds / max(args.steps, 1)))
        per.append(base["value"])
        pcg += base["pcg_steps_sampled"]
        secs += base["sample_seconds"]
    el = time.perf_counter() - t0
    value = float(np.median(per))
    line = {
        "metric": METRICS.get(args.config, METRIC),
        "value": value,
        "unit": UNIT,
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        # one timed step = one bounded PCG sample; ms_per_step x steps = the timed wall
        "ms_per_step": 1e3 * el / args.steps,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (same generator as the GPU arm)",
        "config": ({"workload": f"{args.config}: D={c.D} K={c.K}", "D": c.D, "K": c.K} if structured else
                   {"workload": f"{args.config}: dense Gaussian CS N={c.N} D={c.D} K={c.K} T={c.T} "
                                f"PCG cap {c.U} tol {c.tol}", "N": c.N, "D": c.D, "K": c.K}),
        "impl": "reference",
        "projected": True,
        "pcg_steps_per_sec": pcg / secs,
        "pcg_steps_per_em_iteration": steps_per_em,
        "pcg_steps_per_em_source": source,
        "cpu_baseline": {**{k: base[k] for k in ("unit", "cores", "kind", "sample")}, "value": value,
                         "projected": True},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_seconds": el,
        "note": ("value = EM it/s PROJECTED from the measured PCG-step rate (pcg_steps_per_sec, full-size float64 "
                 "system, every host thread) and the reference's own PCG steps per EM iteration "
                 "(pcg_steps_per_em_source): one EM iteration of the CPU reference at this size takes minutes, "
                 "so each timed step is a bounded sample of PCG steps"),
    }
    print(json.dumps(line), flush=True)


def relaunch_distributed(n):
    """`python bench.py --gpus N` outside torchrun: relaunch under
    torch.distributed.run with N ranks (one per GPU, rendezvous on 127.0.0.1)."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def resolve_precision(args):
    """--precision auto: the mode the library's CgConfig(precision="auto")
    picks for this config's operator (operators.py resolve_precision)."""
    if args.precision != "auto":
        return args.precision
    from paper_2105_10439_b200 import simulate as S
    from paper_2105_10439_b200.operators import AUTO_FP64_ENTRIES, ConvolutionOperator

    if args.config in S.CONFIGS:
        c = S.CONFIGS[args.config]
        return "fp64" if c.N * c.D <= AUTO_FP64_ENTRIES else "ozaki24"
    if args.config in S.CONV_CONFIGS:
        c = S.CONV_CONFIGS[args.config]
        return ConvolutionOperator.from_taps(c.D, c.taps()).resolve_precision("auto")
    return "fp64"


def main():
    args = parse()
    args.precision = resolve_precision(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_distributed(args.gpus)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

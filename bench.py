#!/usr/bin/env python
"""bench.py -- the arXiv 1312.1869 hot path on B200: sketch Y = K Omega -> TSQR -> low-rank solve.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c4] [--impl ours|reference]

One "step" = one pass of the whole hot path over the
config's synthetic input: sketch randomness + fused covariance/SRHT sketch,
blocked TSQR with explicit Q, Q^T A, truncated back substitution, X = Omega Z.
N > 1 (torchrun): rows are sharded, R factors all-gathered (NCCL), C all-reduced.

Metric (BASELINE.json): "K Omega sketch throughput (n^2 d/s) and end-to-end TSQR
low-rank solve time vs n".  `value` = n^2 d / (max-over-ranks step time), i.e.
nominal dense-equivalent n^2 d per second of the WHOLE step; the sketch-only
throughput and the per-phase / end-to-end times are reported beside it.
Timing: CUDA events per step on the launching stream; L2 flushed (a 256 MiB write)
between timed steps outside the events; max over ranks.
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

import ks_inputs  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
TRAFFIC_PATH = os.path.join(ROOT, "profiles", "r1_sketch_traffic.json")   # ncu --set full, per launch
FALLBACK_SM_MHZ = 1965.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-rows", type=int, default=0, help="oracle sample rows (0 = auto, ~10-20 s)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ------------------------------------------------------------------ algorithmic work
def alu_ops_per_element(cfg) -> float:
    """Algorithmic FP32 ops per K element of the fused SRHT sketch:
    SE 2D+2, Matern-3/2 2D+4 (sign folded into the amplitude), + (N/n) log2 d transform adds."""
    D = cfg["dim"]
    kern = 2 * D + 2 if cfg["kernel"] == ks_inputs.SQEXP else 2 * D + 4
    n = cfg["n"]
    N = 1 << (n - 1).bit_length()
    return kern + (N / n) * np.log2(cfg["d"])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.rows = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 4 + i and r[4 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------ shared line fields
METRIC = "K Omega sketch throughput (n^2 d/s) and end-to-end TSQR low-rank solve time vs n"
UNIT = "n^2*d/s"


def blocks_for(cfg, world):
    """TSQR leaf blocks per GPU: c4/c5 fix blocks per GPU; the others split the config's blocks."""
    return cfg["blocks"] if cfg.get("blocks_per_gpu") else max(1, cfg["blocks"] // world)


def make_config(name, cfg, world):
    if cfg.get("planted"):
        return {"workload": name, "n": cfg["n"], "d": cfg["d"],
                "kernel": "stored K = E D E^T (PAPER.md:388), d_ii = exp(-0.01 i), read from HBM",
                "omega": ["srht", "gauss", "hartley", "cosine"][cfg["omega"]], "blocks_per_gpu": blocks_for(cfg, world),
                "m": cfg["m"], "parallelism": f"rows x{world}",
                "l2": "flushed (256 MiB write) before every timed step"}
    return {"workload": name, "n": cfg["n"], "d": cfg["d"], "dim": cfg["dim"],
            "kernel": "sqexp" if cfg["kernel"] == 0 else "matern32",
            "omega": ["srht", "gauss", "hartley", "cosine"][cfg["omega"]], "blocks_per_gpu": blocks_for(cfg, world),
            "m": cfg["m"], "parallelism": f"rows x{world}",
            "l2": "flushed (256 MiB write) before every timed step"}


# ------------------------------------------------------------------ oracle leg (cpu_baseline / --impl reference)
class OracleStep:
    """One oracle 'step' on a bounded sample of the workload (the oracle as it stands, fp64 C,
    all host threads): the sketch of r evenly spaced rows of Y, the TSQR (explicit Q) and Q^T A of
    that r x d sample -- all linear in the number of rows, so their time is scaled by n / r --
    plus the truncated back substitution and the full X = Omega Z once."""

    def __init__(self, cfg, pts, A, budget_s=6.0, rows_hint=0, krows=None, threads=None):
        import oracle
        self.oracle = oracle
        self.cfg = cfg
        self.krows = krows   # planted (stored K): rows -> K[rows] fp64 on the host
        self.prob = oracle.Problem.from_cfg(cfg, pts if pts is not None else np.zeros((1, cfg["n"]), np.float32))
        _ = self.prob.s, self.prob.S  # randomness (setup, excluded like the GPU's)
        if cfg["omega"] == 1:
            _ = self.prob.om16
        self.threads = oracle._threads(threads)
        n, d = cfg["n"], cfg["d"]
        if rows_hint:
            rows = rows_hint
        else:  # calibrate the sketch on a small sample, then size the sample to ~budget_s
            probe = max(self.threads, 8)
            t0 = time.perf_counter()
            self._sketch(np.arange(probe, dtype=np.int64))
            dt = time.perf_counter() - t0
            rows = int(max(probe, min(n, probe * budget_s / max(dt, 1e-3))))
        self.rows = int(min(n, max(rows, d)))
        self.sel = np.linspace(0, n - 1, self.rows).astype(np.int64)
        self.A = np.asarray(A, np.float64)
        self.extrapolated = self.rows < n
        if self.extrapolated:
            self.sample = (f"oracle (fp64 C, {self.threads} threads): sketch of {self.rows} evenly spaced rows of Y "
                           f"({self.rows / n:.4f} of n), TSQR with explicit Q and Q^T A of that {self.rows}x{d} sample, "
                           f"times n/{self.rows} (EXTRAPOLATED: rows are independent); truncated back substitution "
                           f"and the full X = Omega Z once")
        else:
            self.sample = (f"oracle (fp64 C, {self.threads} threads): the whole step on the whole workload "
                           f"(not extrapolated)")
        self.last_measured_s = None

    def info(self):
        return {"cores": self.threads, "extrapolated": self.extrapolated, "sample_rows": self.rows,
                "sample_fraction": self.rows / self.cfg["n"], "measured_s_per_step": self.last_measured_s}

    def _sketch(self, rows):
        if self.krows is not None:
            return self.prob.sketch_stored(self.krows(rows))
        return self.prob.sketch_rows(rows, nthreads=self.threads)

    def run(self):
        o, n = self.oracle, self.cfg["n"]
        t0 = time.perf_counter()
        Y = self._sketch(self.sel)
        Q, R = o.tsqr_tree(Y, max(1, min(self.threads, self.rows // (2 * self.cfg['d']))), want_q=True,
                           nthreads=self.threads)
        Cm = o.matmul(np.ascontiguousarray(Q.T), self.A[self.sel])
        t_lin = time.perf_counter() - t0
        t1 = time.perf_counter()
        k = o.truncation_rank(R)
        Z = o.back_substitute(R, Cm, k)
        self.prob.omega_apply(Z)
        t_once = time.perf_counter() - t1
        self.last_measured_s = t_lin + t_once
        return t_lin * n / self.rows + t_once

    def value(self, seconds):
        c = self.cfg
        return c["n"] * c["n"] * c["d"] / seconds


def planted_rows_fn(cfg):
    """Host rows of the planted K (the device generator's K, copied back row by row)."""
    import torch
    from ks_inputs.planted import planted_K_device
    K = planted_K_device(cfg["n"], cfg["seed"], torch.device("cuda", 0), **cfg["planted"])
    return lambda rows: K[torch.as_tensor(rows, device=K.device)][:, :cfg["n"]].double().cpu().numpy()


def run_reference(args, cfg, pts, A):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    st = OracleStep(cfg, pts, A, rows_hint=args.cpu_rows,
                    krows=planted_rows_fn(cfg) if cfg.get("planted") else None)
    for _ in range(max(0, min(args.warmup, 1))):
        st.run()
    times, measured = [], []
    for _ in range(args.steps):
        times.append(st.run())
        measured.append(st.last_measured_s)
    t = statistics.mean(times)
    v = st.value(t)
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * t, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (ks_inputs, Philox seeded)",
        "config": make_config(args.config, cfg, world),
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": st.threads, "kind": "oracle", "sample": st.sample,
                         **st.info()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "extrapolated": st.extrapolated,
        "measured_s_per_step": statistics.mean(measured),
    }), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg, pts_np, A_np):
    import torch
    import torch.distributed as dist
    import paper_1312_1869_b200 as ks
    from paper_1312_1869_b200 import dist as ksd

    rank, world, local = dist_env()
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")   # keep stdout to the one JSON line
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local if world > 1 else 0)
    torch.cuda.set_device(dev)
    n, d, m = cfg["n"], cfg["d"], cfg["m"]
    blocks = blocks_for(cfg, world)
    rb, re = ksd.shard_rows(n, world, rank)
    desc = dict(n=n, dim=cfg["dim"], kernel=cfg["kernel"], sigma2=cfg["sigma2"], ell=cfg["ell"],
                nugget=cfg["nugget"], d=d, seed=cfg["seed"], omega=cfg["omega"])
    ops = ksd.CudaOps(desc, m, blocks, 1e-5, rank, world, dev, inplace=True)   # sketch into the TSQR plan
    planted = bool(cfg.get("planted"))
    if planted:   # NEXT-2: this rank's rows of the stored K = E D E^T (generated once, outside the timing)
        from ks_inputs.planted import planted_K_device
        pts = planted_K_device(n, cfg["seed"], dev, row_begin=rb, row_end=re, **cfg["planted"])
    else:
        pts = torch.as_tensor(pts_np, device=dev)
    A_loc = torch.as_tensor(np.ascontiguousarray(A_np[rb:re]), device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def step():
        ksd.lowrank_solve_sharded(ops, pts, A_loc)

    # phase events (one step, after warm-up) and per-step events (timed region)
    for _ in range(max(3, args.warmup)):
        step()
    barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    sk_ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps)]
    launches0 = ks.lib().ks_launch_count() if hasattr(ks.lib(), "ks_launch_count") else None
    with ClockSampler(dev.index) as clk:
        barrier()
        for s in range(args.steps):
            flush.fill_(s & 0xFF)  # L2 flush outside the timed events
            ev[2 * s].record(stream)
            sk_ev[2 * s].record(stream)
            Y = ops.sketch(pts)
            sk_ev[2 * s + 1].record(stream)
            Rp = ops.local_r(Y)
            if world > 1:
                dist.all_gather_into_tensor(ops.Rstack, Rp)
                Q2, R = ops.merge(ops.Rstack)
                Q = ops.qform(Q2[rank * d:(rank + 1) * d].contiguous())
            else:
                R = Rp
                Q = ops.qform(None)
            Cm = ops.qt(Q, A_loc)
            if world > 1:
                dist.all_reduce(Cm)
            Z, k = ops.trsolve(R, Cm)
            ops.omega_apply(Z)
            ev[2 * s + 1].record(stream)
        barrier()
    launches = (ks.lib().ks_launch_count() - launches0) if launches0 is not None else None
    step_ms = [ev[2 * s].elapsed_time(ev[2 * s + 1]) for s in range(args.steps)]
    sk_ms = [sk_ev[2 * s].elapsed_time(sk_ev[2 * s + 1]) for s in range(args.steps)]
    t_step = statistics.mean(step_ms)
    t_sk = statistics.mean(sk_ms)
    if world > 1:
        tt = torch.tensor([t_step, t_sk], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_step, t_sk = tt.tolist()

    # phase breakdown (one extra, untimed-for-value step)
    ph = {}
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    flush.fill_(1)
    e[0].record(stream); Y = ops.sketch(pts); e[1].record(stream)
    Rp = ops.local_r(Y)
    if world > 1:
        dist.all_gather_into_tensor(ops.Rstack, Rp)
        Q2, R = ops.merge(ops.Rstack)
        Q = ops.qform(Q2[rank * d:(rank + 1) * d].contiguous())
    else:
        R = Rp
        Q = ops.qform(None)
    e[2].record(stream)
    Cm = ops.qt(Q, A_loc)
    if world > 1:
        dist.all_reduce(Cm)
    Z, k = ops.trsolve(R, Cm)
    ops.omega_apply(Z)
    e[3].record(stream)
    torch.cuda.synchronize(dev)
    ph = {"sketch": e[0].elapsed_time(e[1]), "tsqr_qform": e[1].elapsed_time(e[2]), "solve": e[2].elapsed_time(e[3])}

    # implicit-Q variant (world size 1): the same step without forming Q (row a6), C = Q-hat^T A from the stored
    # reflectors -- reported beside the contract step, not instead of it
    implicit = None
    if world == 1 and not planted:
        ti = []
        for s in range(args.steps + 1):
            flush.fill_(s & 0xFF)
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            Y = ops.sketch(pts)
            R = ops.local_r(Y)
            Cm = ops.qt_implicit(A_loc)
            Z, k_i = ops.trsolve(R, Cm)
            ops.omega_apply(Z)
            b.record(stream)
            b.synchronize()
            if s > 0:
                ti.append(a.elapsed_time(b))
        t_i = statistics.mean(ti)
        implicit = {"ms_per_step": t_i, "value": n * n * d / (t_i * 1e-3), "unit": UNIT,
                    "what": "sketch + TSQR (R only) + implicit Q^T A + trsolve + Omega Z: row a6 skipped"}

    # end-to-end through the public API with host buffers (pinned), copies inside the timed region
    e2e = None
    if planted and n > 10000:
        e2e = {"value": None, "unit": "n^2*d/s", "skipped": "stored K above 10000^2: the host copy of K "
               "(4 n^2 bytes per step) is not staged in pinned memory"}
    elif not args.no_e2e:
        pts_h = (pts.cpu() if planted else torch.as_tensor(pts_np)).pin_memory()
        A_h = torch.as_tensor(np.ascontiguousarray(A_np[rb:re])).pin_memory()
        X_h = torch.empty((re - rb, m), dtype=torch.float32).pin_memory()
        pts_d = torch.empty_like(pts)
        A_d = torch.empty_like(A_loc)
        tms = []
        for s in range(args.steps + 1):
            flush.fill_(s & 0xFF)
            barrier()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            if planted:   # stored K rows: host copy first, then the device path
                pts_d.copy_(pts_h, non_blocking=True)
                X, Z, k, R = ksd.lowrank_solve_sharded(ops, pts_d, A_h, X_host=X_h)
            else:         # the public API with host buffers (A's copy overlaps the sketch and the TSQR)
                X, Z, k, R = ksd.lowrank_solve_sharded(ops, pts_h, A_h, X_host=X_h)
            b.record(stream)
            b.synchronize()
            if s > 0:
                tms.append(a.elapsed_time(b))
        te = statistics.mean(tms)
        if world > 1:
            tt = torch.tensor([te], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = tt.item()
        e2e = {"value": n * n * d / (te * 1e-3), "unit": "n^2*d/s", "ms_per_step": te,
               "h2d_bytes_per_step": int(pts_h.numel() * 4 + A_h.numel() * 4),
               "d2h_bytes_per_step": int(X_h.numel() * 4)}

    if rank == 0:
        peaks = json.load(open(PEAKS_PATH)) if os.path.exists(PEAKS_PATH) else {}
        sm_max = float(peaks.get("sm_max_mhz", FALLBACK_SM_MHZ))
        rows_per_gpu = re - rb
        units = rows_per_gpu * n  # K elements per sketch launch on this rank
        if planted:   # the stored-K sketch streams K from HBM once: bytes / time against the copy bandwidth
            kbytes = units * 4.0
            achieved = kbytes / (t_sk * 1e-3) / 1e9
            peak = float(peaks.get("hbm_gbs", 7700.0))
            nmma = 2 if cfg["omega"] == ks_inputs.OMEGA_GAUSS else (3 if cfg["omega"] != ks_inputs.OMEGA_SRHT else 0)
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "traffic": None, "kernel": "k_sketch_srht" if cfg["omega"] == ks_inputs.OMEGA_SRHT
                    else "k_sketch_gauss2", "bytes_per_element": 4,
                    "peak_basis": "MEASURED_PEAKS.json hbm_gbs (copy bandwidth)"}
            if nmma:
                roof["tensor_frac"] = 2.0 * units * d * nmma / (t_sk * 1e-3) / 1e12 / float(peaks.get("bf16_tflops", 1590.0))
        elif cfg["omega"] == ks_inputs.OMEGA_SRHT:
            ops_elem = alu_ops_per_element(cfg)
            achieved = units * ops_elem / (t_sk * 1e-3) / 1e12
            peak = 148 * 128 * sm_max * 1e6 / 1e12
            roof = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": None,
                    "kernel": "k_sketch_srht", "ops_per_element": ops_elem,
                    "peak_basis": f"148 SMs x 128 FP32 lanes x {sm_max:.0f} MHz (sm_max_mhz, MEASURED_PEAKS.json)"}
        else:
            nmma = 2 if cfg["omega"] == ks_inputs.OMEGA_GAUSS else 3   # MMAs per K step (hi/lo splits counted)
            flops = 2.0 * units * d * nmma
            achieved = flops / (t_sk * 1e-3) / 1e12
            peak = float(peaks.get("bf16_tflops", 1590.0))
            roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                    "frac": achieved / peak, "traffic": None, "kernel": "k_sketch_gauss2", "mma_per_kstep": nmma,
                    "peak_basis": "MEASURED_PEAKS.json bf16_tflops (burst); fp16 dense = bf16 rate"}
        try:   # DRAM bytes of one launch of this config's sketch kernel from a committed ncu capture
            tr = json.load(open(TRAFFIC_PATH)).get(args.config) if world == 1 else None
        except (OSError, ValueError):
            tr = None
        if tr:
            roof["traffic"] = tr["traffic_bytes"]
            roof["traffic_source"] = f"{os.path.relpath(TRAFFIC_PATH, ROOT)} ({tr['kernel']})"
            if tr.get("smem_wavefronts") and roof["bound"] == "alu":
                # the SRHT sketch's binding datapath: shared-memory wavefronts per launch (ncu)
                # over the measured sketch time against 1 wavefront / clk / SM
                wf_peak = 148 * sm_max * 1e6
                roof["smem"] = {"wavefronts_per_launch": tr["smem_wavefronts"],
                                "frac": tr["smem_wavefronts"] / (t_sk * 1e-3) / wf_peak,
                                "peak": "148 SMs x 1 wavefront (128 B) / clk x sm_max_mhz"}
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            krows = (lambda rows: pts[torch.as_tensor(rows, device=dev) - rb][:, :n].double().cpu().numpy()) \
                if planted else None
            st = OracleStep(cfg, pts_np, A_np, rows_hint=args.cpu_rows, krows=krows)
            t_or = st.run()
            cpu = {"value": st.value(t_or), "unit": UNIT, "cores": st.threads, "kind": "oracle",
                   "sample": st.sample, "s_per_step": t_or, **st.info()}
            st1 = OracleStep(cfg, pts_np, A_np, budget_s=4.0, krows=krows, threads=1)   # the same on 1 core
            t1 = st1.run()
            cpu["one_core"] = {"value": st1.value(t1), "unit": UNIT, "s_per_step": t1, "sample": st1.sample,
                               **st1.info()}
        out = {
            "metric": METRIC,
            "value": n * n * d / (t_step * 1e-3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": t_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "data": ("synthetic (planted K = E D E^T, ks_inputs.planted device generator, seeded)" if planted
                     else "synthetic (ks_inputs, Philox seeded)"),
            "config": make_config(args.config, cfg, world),
            "sketch_n2d_per_s": n * rows_per_gpu * d * world / (t_sk * 1e-3),
            "sketch_ms": t_sk, "solve_ms": t_step, "phase_ms": ph,
            "e2e": e2e, "roofline": roof, "cpu_baseline": cpu, "clocks": clk.summary(),
            "gpu_launches": launches, "k": int(k.item()), "implicit_q": implicit,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def relaunch_distributed(args):
    """`--gpus N` (N > 1) outside torchrun: check the GPUs exist, then re-exec this command as N ranks under
    torch.distributed.run (one process per GPU, NCCL).  Inside torchrun: WORLD_SIZE must equal N."""
    world = os.environ.get("WORLD_SIZE")
    if world is not None:
        if int(world) != args.gpus:
            sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
        return
    if args.gpus <= 1:
        return
    import socket
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, this node has {have}")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # the NCCL init lines show every rank joining (on stderr:
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")   # stdout carries only rank 0's JSON line)
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execvpe(sys.executable, cmd, env)


def main():
    args = parse()
    relaunch_distributed(args)
    cfg = dict(ks_inputs.CONFIGS[args.config])
    cfg["seed"] = ks_inputs.config_seed(args.config)
    pts = None if cfg.get("planted") else ks_inputs.points(cfg["seed"], cfg["n"], cfg["dim"], cfg["dist"])
    A = ks_inputs.rhs(cfg["seed"], cfg["n"], cfg["m"])
    if args.impl == "reference":
        run_reference(args, cfg, pts, A)
        return
    run_ours(args, cfg, pts, A)


if __name__ == "__main__":
    main()

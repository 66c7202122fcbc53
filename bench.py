#!/usr/bin/env python
"""iALS++ epoch benchmark (BASELINE.json metric: epoch seconds & nnz*d updates/s,
% of roofline) on B200.

A "step" is one full iALS++ epoch (cache recompute + B blocks x {slab(H), user
pass, slab(W), item pass}) over a seeded synthetic interaction set with the
named shape.  Default workload: configs[3], the ML20M-shaped set
(136,677 x 20,108, 10.0M pairs) at d=1024, b=128 -- the configuration the
metric (b=128) and the >=50%-of-roofline target are quoted on.

    python bench.py [--config L1] [--gpus 1] [--steps 5] [--warmup 3]
    python bench.py --impl reference ...     # the CPU oracle arm

Prints ONE JSON line on rank 0.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # key: (shape, d, b, description)
    "tiny": ("tiny", 32, 8, "configs[0] tiny 2,000x1,000 ~50k, d=32 b=8"),
    "mid": ("mid", 128, 32, "configs[1] ML20M-shaped 136,677x20,108 10.0M, d=128 b=32"),
    "sw-b1": ("mid", 256, 1, "configs[2] d=256 b=1 (iCD case)"),
    "sw-b16": ("mid", 256, 16, "configs[2] d=256 b=16"),
    "sw-b64": ("mid", 256, 64, "configs[2] d=256 b=64"),
    "sw-b128": ("mid", 256, 128, "configs[2] d=256 b=128"),
    "sw-b256": ("mid", 256, 256, "configs[2] d=256 b=d (iALS case)"),
    "ials-d512": ("mid", 512, 512, "dedicated iALS (b = d): ML20M-shaped, d=512 (the wide solver, b > 256)"),
    "d64": ("mid", 64, 64, "metric d-grid: ML20M-shaped, d=64 b=d (b=128 > d)"),
    "d512": ("mid", 512, 128, "metric d-grid: ML20M-shaped, d=512 b=128"),
    "L1": ("mid", 1024, 128, "configs[3] ML20M-shaped 136,677x20,108 10.0M, d=1024 b=128"),
    "L2": ("mid", 2048, 128, "configs[3] ML20M-shaped, d=2048 b=128"),
    "msd": ("msd", 2048, 128, "configs[4] MSD-shaped 571,355x41,140 33.6M, d=2048 b=128"),
}
ALPHA0, REG, NU, SIGMA = 0.1, 1e-3, 1.0, 0.1

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# FP32 FFMA peak: tools/microbench.cu on this pool's B200 (MEASURED_PEAKS.json has no FP32 figure)
# FP32 peak: nominal 148 SM x 128 lanes x 2 FLOP x the SM clock measured under
# load during the timed region (74.4 TFLOP/s at 1965 MHz); MEASURED_PEAKS.json
# has no FP32 figure.  The FFMA microbenchmark (tools/microbench.cu) reaches
# 64.5 TFLOP/s on this pool's B200s -- reported beside it, not used as the peak.
FP32_FFMA_MEASURED_TFLOPS = 64.5
FP32_NOMINAL_TFLOPS = 74.4   # at 1965 MHz


def fp32_peak_tflops(sm_mhz):
    return 148 * 128 * 2 * (sm_mhz or 1965.0) * 1e6 / 1e12


def load_peaks():
    try:
        with open(PEAKS_PATH) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(cfg_key):
    """DRAM bytes per side pass of the sweep kernels from the committed ncu
    capture (tools/traffic.py over tools/profile_pass.py), or None."""
    import glob
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*", f"traffic_{cfg_key}.json")),
                       reverse=True):
        try:
            with open(path) as f:
                t = json.load(f)
            return float(t["dram_bytes_per_side_pass"]), os.path.relpath(path, ROOT)
        except Exception:
            continue
    return None, None


# ----------------------------------------------------------------------- data
def dataset(shape, seed=0):
    """(U, I, CSR dict) of the synthetic set; cached on disk (inputs only)."""
    from paper_2110_14044_b200 import synthetic
    cache_dir = os.path.expanduser("~/.cache/ials_b200")
    path = os.path.join(cache_dir, f"{shape}_s{seed}.npz")
    if os.path.exists(path):
        with np.load(path) as z:
            return {k: z[k] for k in z.files}
    U, I, users, items = synthetic.generate(shape, seed)
    from paper_2110_14044_b200.data import InteractionDataset
    data = InteractionDataset(U, I, users, items)
    iv = data.item_view()
    out = {"U": np.array(U), "I": np.array(I), "user_ptr": data.user_ptr,
           "user_cols": data.items.astype(np.int32), "item_ptr": data.item_ptr,
           "item_cols": iv.cols.astype(np.int32), "item_pos": iv.cache_pos.astype(np.int32),
           "users": data.users.astype(np.int32), "digest": np.array(synthetic.digest(users, items))}
    try:
        os.makedirs(cache_dir, exist_ok=True)
        np.savez(path + ".tmp.npz", **out)
        os.replace(path + ".tmp.npz", path)
    except OSError:
        pass
    return out


def roofline_model(U, I, S, d, b, p_fp32_tflops, bw_gbs):
    """sweep FLOPs / gathered bytes per epoch, slab, predictions."""
    B = -(-d // b)
    f_sw = B * (2 * S * (b * (b + 1) + 4 * b) + (U + I) * (2 * d * b + b ** 3 / 3 + 2 * b * b))
    q_sw = B * (2 * S * (4 * b + 4 + 8) + (U + I) * (4 * d + 4 * b + 8))
    f_g = 2 * (U + I) * d * d
    q_g = B * 4 * (U + I) * d
    q_p = S * (4 * d + 8) + 4 * U * d
    t_sw = max(f_sw / (p_fp32_tflops * 1e12), q_sw / (bw_gbs * 1e9))
    t_g = max(f_g / (p_fp32_tflops * 1e12), q_g / (bw_gbs * 1e9))
    t_p = q_p / (bw_gbs * 1e9)
    bound = "fp32" if f_sw / (p_fp32_tflops * 1e12) >= q_sw / (bw_gbs * 1e9) else "hbm"
    return {"F_sw": f_sw, "Q_sw": q_sw, "F_G": f_g, "Q_P": q_p, "t_sw": t_sw, "t_G": t_g,
            "t_P": t_p, "t_epoch": t_sw + t_g + t_p, "sweep_bound": bound, "B": B}


def config_dict(cfg_key, U, I, S, world):
    """The workload description both arms print (same dict: same config)."""
    shape, d, b, desc = CONFIGS[cfg_key]
    return {"workload": cfg_key, "desc": desc, "users": U, "items": I, "nnz": S,
            "d": d, "b": b, "alpha0": ALPHA0, "reg": REG, "reg_exponent": NU,
            "parallelism": f"replicas x{world}" if world > 1 else "single",
            "l2": ("inputs larger than L2 (W,H,cache,CSR > 126 MB)" if (U + I) * d * 4 + 12 * S > 126e6
                   else "inputs fit in L2 (launch-bound config)")}


# --------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        loaded = [s for s in sm if s > 0.5 * max(sm)] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------- distributed
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------------- ours
def run_ours(args, cfg_key):
    import torch

    from paper_2110_14044_b200 import _lib
    from paper_2110_14044_b200.engine import DeviceProblem, Engine

    shape, d, b, desc = CONFIGS[cfg_key]
    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # NCCL's init lines (ranks, NVLS / NVLink) ...
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()
    ds = dataset(shape)
    U, I = int(ds["U"]), int(ds["I"])
    S = int(ds["user_ptr"][-1])
    if world > 1 or args.sharded:
        if world == 1:
            import torch.distributed as dist
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29533")
            dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
        return run_sharded(args, cfg_key, ds, dev, rank, world)
    prob = DeviceProblem(dev, U, I, ds["user_ptr"], ds["user_cols"], ds["item_ptr"],
                         ds["item_cols"], ds["item_pos"])
    prob.set_regularizer(ALPHA0, REG, NU)
    eng = Engine(prob)
    # seeded init (model.py:123-134), fp32
    from paper_2110_14044_b200.model import SolverConfig, init_model
    cfg = SolverConfig(dim=d, block_size=b, unobserved_weight=ALPHA0, reg=REG,
                       reg_exponent=NU, init_stddev=SIGMA, seed=0)
    m = init_model(cfg, U, I)
    W0 = torch.from_numpy(m.user_factors.astype(np.float32)).to(dev)
    H0 = torch.from_numpy(m.item_factors.astype(np.float32)).to(dev)
    del m
    W, H = W0.clone(), H0.clone()
    cache = torch.zeros(S, dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    B = -(-d // b)
    spans = [(b0, min(b, d - b0)) for b0 in range(0, d, b)]
    slab = torch.empty(d * b, dtype=torch.float32, device=dev)
    su, si = prob.users.schedule(b), prob.items.schedule(b)

    n_ev = 2 + 4 * len(spans)
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
              for _ in range(args.steps)]
    for ev in events:   # torch creates the CUDA events lazily, on first record
        for e in ev:
            e.record(stream)
    # the timed step is the product path: one ials_epoch C-ABI call per epoch
    # (tensor-core GEMMs + fused sweep), with phase events recorded inside it
    # many narrow blocks (b = 1: 4,096 launches of 5..70 us kernels per epoch) are
    # bound by launch latency: the timed epochs then replay the epoch captured as a
    # CUDA graph (Engine.epoch_graph: the same ials_epoch call, captured once); the
    # phase split comes from one eager epoch after the timed region
    use_graph = world == 1 and (args.graph == "on" or (args.graph == "auto" and B >= 32))
    for _ in range(args.warmup):
        eng.epoch(W, H, cache, b, ALPHA0)
    launches_per_graph = 0
    if use_graph:
        n0 = int(eng.lib.ials_launch_count())
        eng.epoch_graph(W, H, cache, b, ALPHA0)   # one eager epoch, the capture, one replay
        launches_per_graph = (int(eng.lib.ials_launch_count()) - n0) // 2
        for _ in range(2):
            eng.epoch_graph(W, H, cache, b, ALPHA0)
    eng.sess.reset_singular()
    torch.cuda.synchronize(dev)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(local)
    with clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        n_launch0 = int(eng.lib.ials_launch_count())
        eng.sess.tc_redo_rows(reset=True)
        t_start.record(stream)
        for s in range(args.steps):
            if use_graph:
                eng.epoch_graph(W, H, cache, b, ALPHA0)
            else:
                eng.epoch(W, H, cache, b, ALPHA0, events=events[s])
        t_end.record(stream)
        n_launches = int(eng.lib.ials_launch_count()) - n_launch0
        torch.cuda.synchronize(dev)
    if use_graph:   # (replays are not counted by the library: the captured epoch's kernels x steps)
        n_launches = launches_per_graph * args.steps
        for s in range(args.steps):   # the phase split, outside the timed region
            eng.epoch(W, H, cache, b, ALPHA0, events=events[s])
        torch.cuda.synchronize(dev)
    tc_redo = eng.sess.tc_redo_rows()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    eng.sess.raise_if_singular()
    total_ms = t_start.elapsed_time(t_end)
    # per-phase sums
    ph = {"cache": 0.0, "gramian": 0.0, "user": 0.0, "item": 0.0}
    for s in range(args.steps):
        e = events[s]
        ph["cache"] += e[0].elapsed_time(e[1])
        k = 1
        for _ in spans:
            for side in ("user", "item"):
                ph["gramian"] += e[k].elapsed_time(e[k + 1])
                ph[side] += e[k + 1].elapsed_time(e[k + 2])
                k += 2
    ms_step = total_ms / args.steps
    if world > 1:
        t = torch.tensor([ms_step], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms_step = float(t.item())
    updates = 2.0 * S * d
    value = updates * world / (ms_step / 1e3)

    hbm, hbm_src = load_peaks()
    clocks = clk.summary()
    p32 = fp32_peak_tflops(clocks.get("sm_mhz"))
    rl = roofline_model(U, I, S, d, b, p32, hbm)
    sweep_ms = (ph["user"] + ph["item"]) / args.steps
    if use_graph:   # eager phase times carry launch gaps the replay does not: their shares of the step
        sweep_ms *= ms_step / max(sum(ph.values()) / args.steps, 1e-9)
    if rl["sweep_bound"] == "fp32":
        achieved = rl["F_sw"] / (sweep_ms / 1e3) / 1e12
        roof = {"bound": "fp32", "achieved": round(achieved, 3), "peak": round(p32, 2),
                "unit": "TFLOP/s", "frac": round(achieved / p32, 4),
                "frac_of_measured_ffma": round(achieved / FP32_FFMA_MEASURED_TFLOPS, 4)}
    else:
        achieved = rl["Q_sw"] / (sweep_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                "frac": round(achieved / hbm, 4)}
    traffic, traffic_src = load_traffic(cfg_key)
    roof.update({
        "traffic": traffic,
        "traffic_unit": "DRAM bytes per side pass (dram__bytes_read.sum + dram__bytes_write.sum, ncu)",
        "traffic_source": traffic_src,
        "algorithmic_bytes_per_side_pass": rl["Q_sw"] / (2 * rl["B"]),
        "kernel": "block sweep per side pass (b 65..128: k_sweep_tc4 [+ k_sweep_wb on rotated user passes] + "
                  "k_heavy_partial_tc4 / k_heavy_solve + k_pass_cache_flat; b 33..64: k_sweep_pk<2>; "
                  "b 17..32: k_sweep_w32m + k_heavy_partial_wm<32>; b 4..16: k_sweep_w16m + "
                  "k_heavy_partial_wm<16>; b = 1: k_sweep_b1 + k_b1_cache_flat; b = 256: k_sweep_light<256>)",
        "per_launch_algorithmic": (rl["F_sw"] if roof["unit"] == "TFLOP/s" else rl["Q_sw"]) / (2 * rl["B"]),
        "avg_launch_ms": round(sweep_ms / (2 * rl["B"]), 4),
        "peak_source": ("nominal FP32 (148 SM x 128 x 2 x measured SM clock; MEASURED_PEAKS.json has "
                        "no FP32 figure)") if roof["bound"] == "fp32" else hbm_src,
        "sweep_share_of_step": round(sweep_ms / ms_step, 4),
        "epoch_roofline_ms": round(rl["t_epoch"] * 1e3, 3),
        "epoch_frac_of_roofline": round(rl["t_epoch"] * 1e3 / ms_step, 4),
        "sweep_roofline_ms": round(rl["t_sw"] * 1e3, 3),
    })

    # ---- e2e through the C-ABI epoch call with host (pinned) buffers
    e2e = None
    if not args.no_e2e:
        Wh = W0.cpu().pin_memory()
        Hh = H0.cpu().pin_memory()
        Ch = torch.empty(S, dtype=torch.float32).pin_memory()
        Wo, Ho = torch.empty_like(Wh).pin_memory(), torch.empty_like(Hh).pin_memory()
        def e2e_step():
            # ials_epoch_host: W / H in from pinned host memory, results (W, H,
            # cache) back, the copies overlapped with the epoch on a second stream
            eng.epoch_host(Wh, Hh, W, H, cache, b, ALPHA0, W_out=Wo, H_out=Ho, cache_out=Ch)
        for _ in range(max(1, args.warmup)):
            e2e_step()
        torch.cuda.synchronize(dev)
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(args.steps):
            e2e_step()
        z.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = a.elapsed_time(z) / args.steps
        if world > 1:
            t = torch.tensor([e2e_ms], device=dev)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            e2e_ms = float(t.item())
        e2e = {"value": updates * world / (e2e_ms / 1e3), "unit": "nnz*d/s",
               "ms_per_step": round(e2e_ms, 3),
               "h2d_bytes_per_step": 4 * (U + I) * d,
               "d2h_bytes_per_step": 4 * (U + I) * d + 4 * S,
               "path": "ials_epoch_host C-ABI call: W/H from pinned host, W/H/cache back, copies overlapped with the epoch"}

    # ---- e2e through the reference's own public API: ialspp_epoch(model, data,
    # cache, config) on the caller's float64 NumPy model (solvers.py:340-375),
    # results written back in place every step (wall clock around the calls;
    # each call returns with the host arrays final)
    e2e_api = None
    if not args.no_e2e and world == 1:
        import paper_2110_14044_b200 as ials
        data = ials.InteractionDataset(U, I, ds["users"], ds["user_cols"])
        mcfg = ials.SolverConfig(dim=d, block_size=b, unobserved_weight=ALPHA0, reg=REG,
                                 reg_exponent=NU, init_stddev=SIGMA, seed=0)
        model = ials.FactorModel(W0.cpu().double().numpy(), H0.cpu().double().numpy())
        pcache = ials.PredictionCache.zeros(S)
        for e in range(max(1, args.warmup)):
            ials.ialspp_epoch(model, data, pcache, mcfg, epoch_index=e)
        torch.cuda.synchronize(dev)
        n0 = int(eng.lib.ials_launch_count())
        t0 = time.perf_counter()
        for e in range(args.steps):
            ials.ialspp_epoch(model, data, pcache, mcfg, epoch_index=e)
        api_ms = (time.perf_counter() - t0) * 1e3 / args.steps
        e2e_api = {"value": updates / (api_ms / 1e3), "unit": "nnz*d/s",
                   "ms_per_step": round(api_ms, 3),
                   "h2d_bytes_per_step": 8 * (U + I) * d,
                   "d2h_bytes_per_step": 8 * (U + I) * d + 8 * S,
                   "gpu_launches_per_step": (int(eng.lib.ials_launch_count()) - n0) / args.steps,
                   "path": ("paper_2110_14044_b200.ialspp_epoch(model, data, cache, config): the "
                            "reference's drop-in call on its float64 NumPy model and cache, updated "
                            "in place (wall clock; host arrays page-locked once, f64 copies and "
                            "casts on the GPU overlapped with the epoch)")}
        del model, pcache, data

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(ds, d, b, budget_s=args.cpu_budget)

    if rank == 0:
        line = {
            "metric": "ialspp_epoch_nnz_d_updates_per_s",
            "value": value, "unit": "nnz*d/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "epoch_seconds": round(ms_step / 1e3, 6),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded Zipf/lognormal stand-in for ML20M/MSD shapes)",
            "config": config_dict(cfg_key, U, I, S, world),
            "phases_ms": {k: round(v / args.steps, 4) for k, v in ph.items()},
            "roofline": roof,
            # headline end to end: the reference-facing call; the fp32 pinned
            # C-ABI call (ials_epoch_host) beside it
            "e2e": e2e_api if e2e_api is not None else e2e,
            "e2e_cabi": e2e,
            "cpu_baseline": cpu,
            "clocks": clocks,
            "gpu_launches": n_launches,
            "launch_mode": ("cuda graph replay of the captured ials_epoch (phases_ms from eager epochs "
                            "outside the timed region)") if use_graph else "eager ials_epoch calls",
            # rows the fused tensor-core sweep's cancellation guard handed to the
            # FP32 sweep during the timed epochs (numerics transparency)
            "tc_redo_rows": tc_redo,
        }
        emit(line)
    if world > 1:
        torch.distributed.destroy_process_group()


def run_sharded(args, cfg_key, ds, dev, rank, world):
    """N GPUs: row shards + replicated tables, NCCL all-reduce of slabs and
    all-gather of column blocks (paper_2110_14044_b200/distributed.py)."""
    import torch
    import torch.distributed as dist

    from paper_2110_14044_b200.distributed import GpuOps, ShardedTrainer
    from paper_2110_14044_b200.model import SolverConfig, init_model

    shape, d, b, desc = CONFIGS[cfg_key]
    U, I, S = int(ds["U"]), int(ds["I"]), int(ds["user_ptr"][-1])
    cfg = SolverConfig(dim=d, block_size=b, unobserved_weight=ALPHA0, reg=REG,
                       reg_exponent=NU, init_stddev=SIGMA, seed=0)
    m = init_model(cfg, U, I)
    W0 = torch.from_numpy(m.user_factors.astype(np.float32))
    H0 = torch.from_numpy(m.item_factors.astype(np.float32))
    del m
    W, H = W0.to(dev), H0.to(dev)
    data = {"num_users": U, "num_items": I, "user_ptr": ds["user_ptr"], "user_cols": ds["user_cols"],
            "item_ptr": ds["item_ptr"], "item_cols": ds["item_cols"], "item_order": ds["item_pos"],
            "labels": None, "weights": None}
    ops = GpuOps(dev)
    tr = ShardedTrainer(data, W, H, ALPHA0, REG, NU, ops)
    stream = torch.cuda.current_stream(dev)
    for _ in range(args.warmup):
        tr.epoch(b)
    torch.cuda.synchronize(dev)
    dist.barrier()
    torch.cuda.synchronize(dev)
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    with clk:
        a, z = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        from paper_2110_14044_b200 import _lib as _l
        lib = _l.load()
        n_launch0 = int(lib.ials_launch_count())
        a.record(stream)
        for _ in range(args.steps):
            tr.epoch(b)
        n_launches = int(lib.ials_launch_count()) - n_launch0
        z.record(stream)
        torch.cuda.synchronize(dev)
    dist.barrier()
    ops.check()
    ms = torch.tensor([a.elapsed_time(z) / args.steps], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms_step = float(ms.item())
    updates = 2.0 * S * d
    value = updates / (ms_step / 1e3)
    e2e = None
    if not args.no_e2e:
        Wh, Hh = W0.pin_memory(), H0.pin_memory()
        ulo, uhi = tr.user_bounds[rank]
        ilo, ihi = tr.item_bounds[rank]
        Wo = torch.empty((uhi - ulo, d), dtype=torch.float32).pin_memory()
        Ho = torch.empty((ihi - ilo, d), dtype=torch.float32).pin_memory()
        Co = torch.empty(tr.us.nnz, dtype=torch.float32).pin_memory()
        dist.barrier()
        a.record(stream)
        for _ in range(args.steps):
            W.copy_(Wh, non_blocking=True)
            H.copy_(Hh, non_blocking=True)
            tr.epoch(b)
            Wo.copy_(W[ulo:uhi], non_blocking=True)
            Ho.copy_(H[ilo:ihi], non_blocking=True)
            Co.copy_(tr.Cu, non_blocking=True)
        z.record(stream)
        torch.cuda.synchronize(dev)
        t = torch.tensor([a.elapsed_time(z) / args.steps], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
        e2e = {"value": updates / (e2e_ms / 1e3), "unit": "nnz*d/s", "ms_per_step": round(e2e_ms, 3),
               "h2d_bytes_per_step": 4 * (U + I) * d * world,
               "d2h_bytes_per_step": 4 * (U + I) * d + 4 * S,
               "path": "per rank: full W/H from pinned host, sharded epoch, local rows + C_u back"}
    if rank == 0:
        hbm, _ = load_peaks()
        rl = roofline_model(U, I, S, d, b, FP32_NOMINAL_TFLOPS, hbm)
        emit(({
            "metric": "ialspp_epoch_nnz_d_updates_per_s", "value": value, "unit": "nnz*d/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(ms_step, 4), "epoch_seconds": round(ms_step / 1e3, 6),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Zipf/lognormal stand-in for ML20M/MSD shapes)",
            "config": {"workload": cfg_key, "desc": desc, "users": U, "items": I, "nnz": S,
                       "d": d, "b": b, "parallelism": f"row shards x{world}, replicated W/H, "
                       "NCCL all-reduce(slab) + all-gather(column block)"},
            "roofline": {"bound": rl["sweep_bound"], "epoch_roofline_ms_1gpu": round(rl["t_epoch"] * 1e3, 3),
                         "epoch_frac_of_Ngpu_roofline": round(rl["t_epoch"] * 1e3 / world / ms_step, 4),
                         "traffic": None},
            "e2e": e2e, "cpu_baseline": None, "clocks": clk.summary(),
            "gpu_launches": n_launches,
        }))
    dist.destroy_process_group()


# ------------------------------------------------------------------ CPU arm
def reference_module():
    """The unmodified reference (``blockals``) installed under baseline/_ref
    (``pip install --no-deps --target baseline/_ref``; git-ignored, shipped to
    the GPU box), or None when it is not there."""
    path = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(path, "blockals")):
        return None
    if path not in sys.path:
        sys.path.insert(0, path)
    try:
        import blockals
        from blockals import solvers as ref_solvers
    except Exception:   # pragma: no cover - broken install
        return None
    return blockals, ref_solvers


def cpu_baseline(ds, d, b, budget_s=15.0, seed=0):
    """The reference CPU solver on this host's cores, on a bounded systematic
    sample of one epoch: the UNMODIFIED reference from baseline/_ref when it is
    installed (``kind`` "reference": its own ``compute_predictions``,
    ``partial_gramian`` and ``_newton_side_pass``, solvers.py:152-186, over
    sub-views of the sampled rows), else the oracle port (``kind`` "port",
    oracle/ialspp_oracle.py).  The BLAS pool is opened to every host core for
    the measurement (torchrun exports OMP_NUM_THREADS=1 to its ranks)."""
    try:
        from threadpoolctl import threadpool_limits
        limits = threadpool_limits(limits=os.cpu_count() or 1)
    except Exception:  # pragma: no cover - threadpoolctl is a reference dependency
        limits = None
    try:
        return _cpu_baseline(ds, d, b, budget_s, seed)
    finally:
        if limits is not None:
            limits.restore_original_limits()


def _entries(rows, ptr):
    counts = ptr[rows + 1] - ptr[rows]
    starts = np.repeat(ptr[rows], counts)
    return starts + np.arange(counts.sum()) - np.repeat(np.cumsum(counts) - counts, counts)


def _cpu_baseline(ds, d, b, budget_s=15.0, seed=0):
    from oracle import ialspp_oracle as orc   # the row sampler; the port itself if no reference
    refm = reference_module()
    U, I = int(ds["U"]), int(ds["I"])
    uptr, iptr = ds["user_ptr"].astype(np.int64), ds["item_ptr"].astype(np.int64)
    S = int(uptr[-1])
    rng = np.random.default_rng(seed)
    scale = SIGMA / np.sqrt(d)
    w = rng.normal(0.0, scale, size=(U, d))
    h = rng.normal(0.0, scale, size=(I, d))
    users = ds["users"].astype(np.int64)
    ucols = ds["user_cols"].astype(np.int64)
    icols = ds["item_cols"].astype(np.int64)
    ipos = ds["item_pos"].astype(np.int64)
    lab = np.ones(S)
    lu = orc.effective_reg(np.diff(uptr), I, REG, ALPHA0, NU)
    li = orc.effective_reg(np.diff(iptr), U, REG, ALPHA0, NU)
    B = -(-d // b)
    blk = np.arange(min(b, d))
    # size the strides from a rough per-unit cost so one step is ~budget_s
    work_u = (S * b * b + U * (d * b + b ** 3 / 3))
    per_unit = 2.0e-10 * max(1.0, b / 32)
    s_u = max(1, int(work_u * per_unit * B / (0.35 * budget_s)))
    s_i = max(1, s_u // 8)
    s_p = max(1, int(S * d * 2e-9 / (0.15 * budget_s)))
    prows = np.arange(0, U, s_p)
    pidx = _entries(prows, uptr)
    if refm is not None:
        ref, rs = refm
        from blockals import data as ref_data
        # predictions over the sampled users' interactions (model.py:153-165)
        pdata = ref.InteractionDataset(prows.size, I, np.repeat(np.arange(prows.size),
                                       uptr[prows + 1] - uptr[prows]), ucols[pidx])
        pmodel = ref.FactorModel(np.ascontiguousarray(w[prows]), h)
        t0 = time.perf_counter()
        ref.compute_predictions(pmodel, pdata)
        t_pred = (time.perf_counter() - t0) * (S / max(pidx.size, 1))
        gram = lambda m: ref.partial_gramian(m, blk)

        def run_rows(ptr, cols, pos, fixed, own, slab, lam, rows):
            # the reference's own side pass over a SideView of just these rows
            # (their entries, a compact cache); view buckets are built once per
            # dataset in the reference, so outside the timed region
            ent = _entries(rows, ptr)
            sub_ptr = np.zeros(rows.size + 1, dtype=np.int64)
            np.cumsum(ptr[rows + 1] - ptr[rows], out=sub_ptr[1:])
            ones = np.ones(ent.size)
            view = ref_data.SideView(rows.size, fixed.shape[0], sub_ptr, cols[ent], ones, ones,
                                np.arange(ent.size))
            view.buckets()
            upd = np.ascontiguousarray(own[rows])
            cache_ext = np.zeros(ent.size + 1)
            t0 = time.perf_counter()
            rs._newton_side_pass(view, fixed, upd, cache_ext, blk, slab, ALPHA0, lam[rows])
            return time.perf_counter() - t0
        kind, what = "reference", ("the unmodified reference (baseline/_ref blockals 0.1.0): "
                                   "compute_predictions, partial_gramian, _newton_side_pass")
    else:
        t0 = time.perf_counter()
        orc.predictions(w, h, users[pidx], ucols[pidx])
        t_pred = (time.perf_counter() - t0) * (S / max(pidx.size, 1))
        gram = lambda m: orc.partial_gramian(m, blk)
        cache = np.zeros(S)

        def run_rows(ptr, cols, pos, fixed, own, slab, lam, rows):
            t0 = time.perf_counter()
            orc.side_pass(ptr, cols, lab, lab, pos, fixed, own, cache, blk, slab, ALPHA0, lam,
                          rows=rows)
            return time.perf_counter() - t0
        kind, what = "port", "oracle/ialspp_oracle.py (f64 NumPy restatement)"

    def timed_pass(ptr, cols, pos, fixed, own, slab, lam, stride):
        head, tail = orc.systematic_rows(np.diff(ptr), stride)
        t = 0.0
        for rows, weight in ((head, 1.0), (tail, float(stride))):
            if rows.size:
                t += run_rows(ptr, cols, pos, fixed, own, slab, lam, rows) * weight
        return t

    t0 = time.perf_counter()
    slab_h = gram(h)
    t_gh = time.perf_counter() - t0
    t_user = timed_pass(uptr, ucols, np.arange(S), h, w, slab_h, lu, s_u)
    t0 = time.perf_counter()
    slab_w = gram(w)
    t_gw = time.perf_counter() - t0
    t_item = timed_pass(iptr, icols, ipos, w, h, slab_w, li, s_i)
    t_epoch = t_pred + B * (t_gh + t_user + t_gw + t_item)
    try:
        from threadpoolctl import threadpool_info
        blas = [(i.get("internal_api"), i.get("num_threads")) for i in threadpool_info()]
        threads = max([t for _, t in blas if t] or [os.cpu_count()])
    except Exception:
        blas, threads = [], os.cpu_count()
    return {"value": 2.0 * S * d / t_epoch, "unit": "nnz*d/s", "cores": int(threads),
            "kind": kind, "epoch_seconds_est": round(t_epoch, 2),
            "sample": (f"{what}, f64 on this host ({os.cpu_count()} cores): predictions for every "
                       f"{s_p}th user, block-0 slabs in full, user / item pass on the 64 heaviest "
                       f"rows in full plus every {s_u}th / {s_i}th run of 64 degree-sorted rows "
                       f"(scaled by the stride); epoch = t_pred + {B} x t_block "
                       f"(extrapolated from 1 of {B} blocks)"),
            "phase_seconds_est": {"pred": round(t_pred, 3), "gram": round(t_gh + t_gw, 3),
                                  "user_per_block": round(t_user, 3),
                                  "item_per_block": round(t_item, 3)},
            "blas": str(blas)}


def run_reference(args, cfg_key):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    shape, d, b, desc = CONFIGS[cfg_key]
    ds = dataset(shape)
    U, I, S = int(ds["U"]), int(ds["I"]), int(ds["user_ptr"][-1])
    vals = []
    for _ in range(args.warmup):
        cpu_baseline(ds, d, b, budget_s=args.cpu_budget)
    for _ in range(args.steps):
        vals.append(cpu_baseline(ds, d, b, budget_s=args.cpu_budget))
    value = statistics.median(v["value"] for v in vals)
    last = vals[-1]
    line = {"impl": "reference", "metric": "ialspp_epoch_nnz_d_updates_per_s", "value": value,
            "unit": "nnz*d/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(2.0 * S * d / value * 1e3, 3), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded Zipf/lognormal stand-in for ML20M/MSD shapes)",
            "config": config_dict(cfg_key, U, I, S, world),
            "cpu_baseline": {"value": value, "unit": "nnz*d/s", "cores": last["cores"],
                             "kind": last["kind"], "sample": last["sample"],
                             "epoch_seconds_est": last["epoch_seconds_est"]},
            "e2e": {"value": value, "unit": "nnz*d/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    emit(line)


_JSON_FD = None


def emit(line):
    """The one JSON line, on the process's original stdout."""
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def main():
    # stdout carries the one JSON line: NCCL prints its version banner (and,
    # unless told otherwise, its log) to stdout from native code, so fd 1 is
    # pointed at stderr for the run and the line goes to the saved descriptor
    global _JSON_FD
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    sys.stdout.flush()
    _JSON_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="L1")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="replay the epoch as a CUDA graph in the timed region (auto: 32 or more blocks)")
    ap.add_argument("--sharded", action="store_true",
                    help="use the multi-GPU (sharded) epoch even on one GPU")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args, args.config)
    else:
        run_ours(args, args.config)


if __name__ == "__main__":
    main()

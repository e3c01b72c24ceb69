#!/usr/bin/env python
"""bench.py — B200 CSFMM benchmark (driver contract).

Workload (BASELINE.json metric, configs[4] = "c5"): SAL potential on the 6x1024x1024
cubed sphere, N = 6,291,456 targets = sources, p = 10, theta = 0.6, leaf <= 256, fp64,
seeded synthetic ocean-mask x N(0,1) x area weights (paper_2508_13550_b200/configs.py).
One step = one full csfmm_sum-equivalent: tree build + upward + dual traversal +
PP/PC/CP/CC + downward, output in input order.

  value  target points/s over all ranks, inputs resident in HBM, CUDA events, max over
         ranks (N > 1: target-partitioned, NCCL all-reduce of proxy weights + potentials)
  e2e    the same through the host-pointer C-ABI (csfs_b200_csfmm): pinned host inputs
         copied H2D and the result copied D2H inside every step
  roofline  the evaluation phase (k_mutual + k_interact, 95% of the step) against the
         MEASURED FP64 DFMA peak: `achieved` by SURVEY.md §8d's per-pair convention (87
         flop for SAL, so frac > 1 — the functor executes ~34), `executed_frac` from the
         ncu-measured FP64 flop per pair (profiles/*interact_sal_ncu.json)
  cpu_baseline  the reference's own csfmm_sum (oracle/_ref, all host cores) on a bounded
         sample of the same workload (one depth-1 face quadrant of targets, all sources)

--impl reference runs that reference CPU path alone (rank 0), same metric and config.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import statistics
import subprocess
import sys
import threading
import time

os.environ.setdefault("OMP_WAIT_POLICY", "active")
os.environ.setdefault("OMP_PROC_BIND", "close")

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

METRIC = "FMM target points/s at N=6.29M (1/2/4/8 B200); % of FP64 peak in P2P+M2L"
UNIT = "target points/s"
# Algorithmic FP64 flops per pairwise kernel evaluation (SURVEY.md §8d convention:
# reference formula as executed by sm_100a libdevice fast paths, DFMA = 2).
FLOP_PER_PAIR = {"laplace": 53, "sal": 87, "biot_savart": 39, "biharmonic": 94}
def _hbm_gbs() -> float:
    """MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth on this pool's B200s)."""
    try:
        with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6549.4


HBM_GBS = _hbm_gbs()
NOMINAL_FP64_TFLOPS = 37.2


def rank_info():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def quadrant_sample(wl):
    """Targets of face 0, quadrant 0 (xi, eta < 0): one depth-1 subtree of the C5 tree."""
    m = 1 << wl.level
    h = m // 2
    i, j = np.meshgrid(np.arange(h), np.arange(h), indexing="ij")
    return (i * m + j).reshape(-1)


def cpu_reference(wl, steps: int, warmup: int):
    """The reference's own csfmm_sum (oracle/_ref) on the bounded sample; returns
    (points/s per step list, sample description, cores)."""
    from oracle import ref  # cpu_baseline leg only

    idx = quadrant_sample(wl)
    txyz = np.ascontiguousarray(wl.xyz[idx])
    cores = os.cpu_count() or 1
    kw = dict(mac=wl.mac, degree=wl.degree, n0=wl.n0, threads=0)
    # OpenMP warm-up on a tiny problem (fork/wake overheads)
    ref.csfmm(wl.xyz[:4096], wl.xyz[:4096], wl.weights[:4096], wl.kernel, **kw)
    vals = []
    for s in range(warmup + steps):
        t = time.perf_counter()
        ref.csfmm(txyz, wl.xyz, wl.weights, wl.kernel, **kw)
        dt = time.perf_counter() - t
        if s >= warmup:
            vals.append(len(idx) / dt)
    sample = (f"reference csfmm_sum (oracle/_ref, g++ -O3 -fopenmp, {cores} threads) on "
              f"{len(idx)} targets = face 0 / quadrant 0 (one depth-1 subtree of {wl.name}) "
              f"x all {wl.n} sources; tree builds + upward + traversal + PP/PC/CP/CC + downward "
              f"timed; points/s = sampled targets / wall")
    return vals, sample, cores


class ClockSampler:
    """nvidia-smi sampling DURING the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []  # (wall time, csv line)
        self.window = None  # (t0, t1): keep the samples taken inside the timed region

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def start(self):
        """nvidia-smi takes ~0.5 s to deliver its first sample: start it before the warm-up."""
        return self.__enter__()

    def mark(self, t0: float, t1: float):
        self.window = (t0, t1)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        lines = self.lines
        if self.window is not None:
            inside = [x for x in lines if self.window[0] <= x[0] <= self.window[1] + 0.1]
            lines = inside if inside else lines[-1:]
        for _, ln in lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_ncu(kernel_tag: str):
    """Newest committed ncu summary of the evaluation kernel (profiles/*interact_<tag>*ncu*.json)."""
    files = sorted(glob.glob(os.path.join(HERE, "profiles", f"*interact_{kernel_tag}*ncu*.json")))
    if not files:
        return {}, None
    try:
        return json.load(open(files[-1])), os.path.relpath(files[-1], HERE)
    except Exception:
        return {}, None


def run_reference(args):
    rank, world, _ = rank_info()
    if rank != 0:
        return 0
    from paper_2508_13550_b200 import configs

    wl = configs.make(args.workload)
    vals, sample, cores = cpu_reference(wl, args.steps, args.warmup)
    v = float(np.mean(vals))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * len(quadrant_sample(wl)) / v,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(wl),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


def workload_config(wl):
    return {"workload": f"{wl.name}: {wl.kernel} kernel sum, 6x{1 << wl.level}x{1 << wl.level} cubed sphere, "
                        f"N={wl.n}, targets=sources",
            "n_points": wl.n, "kernel": wl.kernel, "degree": wl.degree, "mac": wl.mac, "n0": wl.n0,
            "weights": "seeded ocean mask (p=0.7) x N(0,1) x cell area",
            "l2": "inputs (N x 32 B = 201 MB) and proxy/potential arrays exceed the 126 MB L2; no flush"}


_OUT_FD = None  # the real stdout; fd 1 points at stderr while the run prints (NCCL banners, ...)


def emit(line):
    """The ONE JSON line, on the real stdout (everything else the run prints went to stderr)."""
    data = (json.dumps(line) + "\n").encode()
    if _OUT_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_OUT_FD, data)


def main():
    global _OUT_FD
    sys.stdout.flush()
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--partitioned", action="store_true",
                    help="use the multi-GPU (NCCL) path even with one rank (torchrun)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2508_13550_b200 import Engine, Kernel, ParticleSet, SumStats, TraversalConfig, configs
    from paper_2508_13550_b200.distributed import partitioned_csfmm
    from paper_2508_13550_b200.engine import kernel_launches

    rank, world, local = rank_info()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    part = world > 1 or args.partitioned  # target-partitioned path (NCCL all-reduces)
    if part:
        dist.init_process_group("nccl", device_id=dev)
    wl = configs.make(args.workload)
    k = Kernel.parse(wl.kernel)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    eng = Engine(local)
    xyz = torch.from_numpy(wl.xyz).to(dev)
    w = torch.from_numpy(wl.weights).to(dev)
    out = torch.empty(wl.n * k.out_dim(), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step(st=None):
        if part:
            partitioned_csfmm(eng, xyz, xyz, w, k, cfg, out)
            return None
        return eng.csfmm_device(xyz.data_ptr(), wl.n, xyz.data_ptr(), w.data_ptr(), wl.n, k, cfg,
                                out.data_ptr(), stream.cuda_stream, st)

    def barrier():
        if part:
            dist.barrier()

    fp64_peak = eng.probe_fp64_tflops()
    clk = ClockSampler(local).start()  # running through the warm-up; samples kept for the timed region
    for _ in range(args.warmup):
        step()

    # ---- timed: device-resident (value) -------------------------------------------------
    stats = []
    barrier()
    torch.cuda.synchronize()
    l0 = kernel_launches()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall0 = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        st = SumStats()
        step(st)
        stats.append(st)
    e1.record(stream)
    torch.cuda.synchronize()
    clk.mark(t_wall0, time.time())
    clk.__exit__(None, None, None)
    barrier()
    launches = kernel_launches() - l0
    ms = e0.elapsed_time(e1)
    if part:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = wl.n * args.steps / (ms * 1e-3)

    # ---- roofline of the dominant kernel (single-GPU stats) ------------------------------
    roof = None
    if not part:
        s0 = stats[-1]
        evals = s0.evals_pp + s0.evals_pc + s0.evals_cp + s0.evals_cc
        t_int = statistics.mean(s.t_interact for s in stats)
        flops = evals * FLOP_PER_PAIR[wl.kernel]
        achieved = flops / t_int / 1e12
        ncu, ncu_src = load_ncu({"sal": "sal", "laplace": "laplace", "biharmonic": "biharmonic",
                                 "biot_savart": "bs"}[wl.kernel])
        traffic = ncu.get("dram_bytes_per_launch")
        exec_fpp = ncu.get("fp64_flop_per_pair_executed")
        exec_evals = s0.evals_executed  # symmetric PP/CC pairs evaluated once for both directions
        roof = {"bound": "fp64", "kernel": f"evaluation phase: k_mutual + k_interact<Op{wl.kernel}> "
                                          f"(PP+PC+CP+CC)", "achieved": achieved,
                "peak": fp64_peak, "unit": "TFLOP/s", "frac": achieved / fp64_peak,
                "traffic": traffic, "traffic_source": ncu_src,
                "algorithmic_flop_per_pair": FLOP_PER_PAIR[wl.kernel],
                "algorithmic_convention": "SURVEY.md §8d: reference formula as executed by sm_100a libdevice "
                                          "(DFMA=2); our functor computes the same value with fewer FP64 ops, "
                                          "so frac can exceed 1 — see executed_* for pipe-level utilisation",
                "executed_flop_per_pair": exec_fpp,
                "executed_pair_evals_per_launch": exec_evals,
                "executed_tflops": (exec_evals * exec_fpp / t_int / 1e12) if exec_fpp else None,
                "executed_frac": (exec_evals * exec_fpp / t_int / 1e12 / fp64_peak) if exec_fpp else None,
                "fp64_pipe_active_pct_ncu": ncu.get("fp64_pipe_active_pct"),
                "peak_source": "measured DFMA-chain probe (csfs_b200_probe_fp64) on this GPU; "
                               "MEASURED_PEAKS.json has no FP64 entry",
                "frac_of_nominal_37.2": achieved / NOMINAL_FP64_TFLOPS,
                "pair_evals_per_launch": evals,
                "kernel_ms": t_int * 1e3, "share_of_step": t_int / (ms_per_step * 1e-3),
                "phases_ms": {kk: 1e3 * statistics.mean(getattr(s, kk) for s in stats)
                              for kk in ("t_tree_build", "t_upward", "t_lists", "t_interact", "t_downward", "t_total")}}
        # the HBM-type phases against the measured copy bandwidth (SURVEY.md §8d algorithmic
        # bytes): tree build = xyz in (24 B/pt) + per level xi, eta, idx moved (2 x 20 B/pt) +
        # sorted xyz, w, perm out (36 B/pt); upward leaf = 24 B/pt + (p+1)^2 x 8 B per leaf;
        # downward leaf = 16 B/pt + 8 dim B/pt.  They are launch/latency-bound small kernels
        # (4% of the step), reported for completeness.
        n = wl.n
        npp = (wl.degree + 1) ** 2
        hbm_bytes = {"t_tree_build": n * (24 + 40 * s0.tgt_depth + 36),
                     "t_upward": n * 24 + npp * 8 * s0.src_leaves,
                     "t_downward": n * (16 + 8 * k.out_dim())}
        roof["hbm_phases"] = {
            ph: {"algorithmic_bytes": b, "ms": roof["phases_ms"][ph],
                 "gbs": b / (roof["phases_ms"][ph] * 1e-3) / 1e9,
                 "frac_of_hbm": b / (roof["phases_ms"][ph] * 1e-3) / 1e9 / HBM_GBS}
            for ph, b in hbm_bytes.items()}

    # ---- e2e through the host-pointer C-ABI ---------------------------------------------
    e2e = None
    if not args.no_e2e:
        hx = torch.from_numpy(wl.xyz).pin_memory()
        hw = torch.from_numpy(wl.weights).pin_memory()
        ho = torch.empty(wl.n * k.out_dim(), dtype=torch.float64).pin_memory()
        p = ParticleSet(hx.numpy(), hw.numpy())
        if part:
            # each rank: H2D of all inputs, partitioned evaluation, D2H of the result
            def e2e_step():
                xyz.copy_(hx, non_blocking=True)
                w.copy_(hw, non_blocking=True)
                partitioned_csfmm(eng, xyz, xyz, w, k, cfg, out)
                ho.copy_(out, non_blocking=True)
                torch.cuda.synchronize()
        else:
            def e2e_step():
                eng.csfmm_sum(p, p, k, cfg, out=ho.numpy())
        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        barrier()
        dt = time.perf_counter() - t0
        if part:
            t = torch.tensor([dt], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        e2e = {"value": wl.n * args.steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(wl.xyz.nbytes + wl.weights.nbytes),
               "d2h_bytes_per_step": int(wl.n * k.out_dim() * 8),
               "timing": "wall clock around the synchronous host-pointer call, pinned host buffers"}

    # ---- CPU baseline (rank 0, N = 1 only) ------------------------------------------------
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            vals, sample, cores = cpu_reference(wl, 1, 0)
            cpu = {"value": float(vals[0]), "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample}
        except Exception as ex:  # the checker must not break the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "reference",
                   "sample": f"unavailable: {ex}"}

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": dict(workload_config(wl), parallelism=f"target-partitioned x{world}" if part else "1 GPU"),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
                "clocks": clk.summary()}
        if roof:
            line["fp64_frac_p2p_m2l"] = roof["frac"]
            line["fp64_frac_p2p_m2l_executed"] = roof["executed_frac"]
        emit(line)
    if part:
        dist.destroy_process_group()
    eng.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())

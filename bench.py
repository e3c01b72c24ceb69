#!/usr/bin/env python
"""bench.py — B200 CSFMM benchmark (driver contract).

Workload (BASELINE.json metric, configs[4] = "c5"): SAL potential on the 6x1024x1024
cubed sphere, N = 6,291,456 targets = sources, p = 10, theta = 0.6, leaf <= 256, fp64,
seeded synthetic ocean-mask x N(0,1) x area weights (paper_2508_13550_b200/configs.py).
One step = one full csfmm_sum-equivalent: tree build + upward + dual traversal +
PP/PC/CP/CC + downward, output in input order.

  --gpus N   N ranks, one process per GPU.  Under torchrun (RANK/WORLD_SIZE set) this
             process is one rank; without it, N > 1 re-executes itself under
             `python -m torch.distributed.run --nproc-per-node N` and refuses (exit 2) when
             fewer than N GPUs are visible.  N > 1 runs the target-partitioned CSFMM of the
             C-ABI (csfs_b200_create_rank): NCCL all-gathers of proxy weights and
             potentials inside the library, over NVLink.
  value      target points/s of the whole job, inputs resident in HBM, CUDA events on the
             launching stream, max over ranks
  e2e        the same through the host-pointer C-ABI call (csfs_b200_csfmm): pinned host
             inputs copied H2D and the result copied D2H inside every step
  roofline   the evaluation phase (k_mutual + k_interact, ~95% of the step) on the FP64
             pipe: achieved = executed evaluations (summed over ranks) x the FP64 flop per
             evaluation ncu measured on THIS build (profiles/*interact_<kernel>*ncu*.json,
             refused when its source hash differs) / the phase time (max over ranks) /
             (N x the measured DFMA peak); the SURVEY.md §8d libdevice-convention rate is
             reported beside it as libdevice_equiv_tflops
  cpu_baseline  the reference's own csfmm_sum (oracle/_ref, all host cores) on a bounded
             sample: the targets of one depth-1 face quadrant (1/24) against all sources;
             the whole-workload time is extrapolated from its SumStats (source tree and
             upward pass once, target-side phases x 24)

--impl reference runs that reference CPU path alone (rank 0), same metric and config.
"""
from __future__ import annotations

import argparse
import glob
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402

METRIC = "FMM target points/s at N=6.29M (1/2/4/8 B200); % of FP64 peak in P2P+M2L"
UNIT = "target points/s"
# SURVEY.md §8d convention: FP64 flops of the reference formula as executed by the sm_100a
# libdevice fast paths (DFMA = 2).  Reported as libdevice_equiv_tflops, not as the roofline.
LIBDEVICE_FLOP_PER_PAIR = {"laplace": 53, "sal": 87, "biot_savart": 39, "biharmonic": 94}
NCU_TAG = {"sal": "sal", "laplace": "laplace", "biharmonic": "biharmonic", "biot_savart": "bs"}
NOMINAL_FP64_TFLOPS = 37.2
QUADRANTS = 24  # depth-1 face quadrants: the CPU sample is one of them


def _hbm_gbs() -> float:
    """MEASURED_PEAKS.json hbm_gbs (driver-measured copy bandwidth on this pool's B200s)."""
    try:
        with open(os.path.join(HERE, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6549.4


HBM_GBS = _hbm_gbs()


def rank_info():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# ---------------------------------------------------------------------------------------
# the reference's CPU path (cpu_baseline leg and --impl reference)
# ---------------------------------------------------------------------------------------

def quadrant_sample(wl):
    """Targets of face 0, quadrant 0 (xi, eta < 0): one depth-1 subtree of the C5 tree."""
    m = 1 << wl.level
    h = m // 2
    i, j = np.meshgrid(np.arange(h), np.arange(h), indexing="ij")
    return (i * m + j).reshape(-1)


def cpu_reference(wl, steps: int, warmup: int):
    """The reference's own csfmm_sum (oracle/_ref) on the bounded sample.  Returns a list
    of per-step dicts: sample wall time, its SumStats phases and the extrapolated time of
    the whole workload (target points/s = N / that)."""
    os.environ.setdefault("OMP_WAIT_POLICY", "active")  # before libgomp starts (first call)
    os.environ.setdefault("OMP_PROC_BIND", "close")
    from oracle import ref  # cpu_baseline leg only

    idx = quadrant_sample(wl)
    txyz = np.ascontiguousarray(wl.xyz[idx])
    kw = dict(mac=wl.mac, degree=wl.degree, n0=wl.n0, threads=0)
    # OpenMP warm-up on a tiny problem (fork/wake overheads)
    ref.csfmm(wl.xyz[:4096], wl.xyz[:4096], wl.weights[:4096], wl.kernel, **kw)
    res = []
    for s in range(warmup + steps):
        t = time.perf_counter()
        _, st = ref.csfmm(txyz, wl.xyz, wl.weights, wl.kernel, **kw)
        wall = time.perf_counter() - t
        # st: t_tree_build (both trees), t_upward (source), t_traversal, t_downward, t_total
        t_tree, t_up, t_trav, t_down = float(st[0]), float(st[1]), float(st[2]), float(st[3])
        # the tree build is linear in the particle count: the target tree is 1/24 of the
        # source tree's work, so the sample's build = (1 + 1/24) source builds, and the full
        # run (targets = sources, the reference builds both trees) = 2 source builds
        t_src_tree = t_tree * QUADRANTS / (QUADRANTS + 1)
        full = 2.0 * t_src_tree + t_up + QUADRANTS * (t_trav + t_down)
        if s >= warmup:
            res.append({"sample_wall_s": wall, "tree_s": t_tree, "upward_s": t_up, "traversal_s": t_trav,
                        "downward_s": t_down, "extrapolated_full_s": full, "value": wl.n / full})
    return res


def cpu_sample_text(wl, cores):
    return (f"reference csfmm_sum (oracle/_ref, g++ -O3 -fopenmp, {cores} threads, OMP_WAIT_POLICY=active) on "
            f"the {len(quadrant_sample(wl))} targets of face 0 / quadrant 0 (one depth-1 subtree = 1/{QUADRANTS} "
            f"of {wl.name}) x all {wl.n} sources; whole-workload time extrapolated from its SumStats: "
            f"2 x source-tree build + upward pass (once) + {QUADRANTS} x (traversal incl. PP/PC/CP/CC + "
            f"downward); value = N / that time (profiles/r02_reference_c5_full.json checks it against a full run)")


def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def workload_config(wl, parallelism):
    return {"workload": f"{wl.name}: {wl.kernel} kernel sum, 6x{1 << wl.level}x{1 << wl.level} cubed sphere, "
                        f"N={wl.n}, targets=sources",
            "n_points": wl.n, "kernel": wl.kernel, "degree": wl.degree, "mac": wl.mac, "n0": wl.n0,
            "weights": "seeded ocean mask (p=0.7) x N(0,1) x cell area",
            "parallelism": parallelism,
            "l2": "inputs (N x 32 B = 201 MB) and proxy/potential arrays exceed the 126 MB L2; no flush"}


def run_reference(args):
    rank, world, _ = rank_info()
    if rank != 0:
        return 0
    from paper_2508_13550_b200 import configs

    wl = configs.make(args.workload)
    res = cpu_reference(wl, args.steps, args.warmup)
    cores = os.cpu_count() or 1
    v = float(np.mean([r["value"] for r in res]))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * wl.n / v,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": workload_config(wl, f"CPU, {cores} host threads"),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "reference",
                             "sample": cpu_sample_text(wl, cores), "cpu_model": cpu_model(), "steps": res},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    emit(line)
    return 0


# ---------------------------------------------------------------------------------------
# measurement helpers
# ---------------------------------------------------------------------------------------

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

    def start(self):
        """nvidia-smi takes ~0.5 s to deliver its first sample: start it before the warm-up."""
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def mark(self, t0: float, t1: float):
        self.window = (t0, t1)

    def stop(self):
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
        return {"gpu": self.gpu, "sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


def load_ncu(kernel: str):
    """Newest committed ncu summary of the evaluation kernels for `kernel`
    (profiles/*interact_<tag>*ncu*.json) — only if it was captured from these sources."""
    from paper_2508_13550_b200.srchash import eval_kernel_sha256

    files = sorted(glob.glob(os.path.join(HERE, "profiles", f"*interact_{NCU_TAG[kernel]}*ncu*.json")))
    if not files:
        return {}, None, "no ncu capture for this kernel in profiles/"
    src = os.path.relpath(files[-1], HERE)
    try:
        d = json.load(open(files[-1]))
    except (OSError, ValueError) as ex:
        return {}, src, f"unreadable: {ex}"
    if d.get("source_sha256") != eval_kernel_sha256():
        return {}, src, "refused: captured from different evaluation-kernel sources (srchash.py)"
    return d, src, None


_OUT_FD = None  # the real stdout; fd 1 points at stderr while the run prints (NCCL banners, ...)


def emit(line):
    """The ONE JSON line, on the real stdout (everything else the run prints went to stderr)."""
    data = (json.dumps(line) + "\n").encode()
    if _OUT_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_OUT_FD, data)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch_argv(argv, gpus: int, port: int | None = None):
    """The torchrun command that runs this script as `gpus` ranks (one process per GPU)."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr=127.0.0.1", f"--master-port={port or _free_port()}", os.path.abspath(__file__)] + list(argv)


def visible_gpus() -> int:
    import torch

    return torch.cuda.device_count() if torch.cuda.is_available() else 0


# ---------------------------------------------------------------------------------------
# runtime: CUDA + NCCL for the bench, CPU + gloo for the launcher tests
# ---------------------------------------------------------------------------------------

class CudaRuntime:
    def __init__(self, local: int, world: int):
        import torch
        import torch.distributed as dist

        self.torch, self.dist = torch, dist
        torch.cuda.set_device(local)
        self.dev = torch.device("cuda", local)
        self.world = world
        if world > 1:
            dist.init_process_group("nccl", device_id=self.dev)
        self.stream = torch.cuda.current_stream(self.dev)

    def sync(self):
        self.torch.cuda.synchronize(self.dev)

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def event(self):
        e = self.torch.cuda.Event(enable_timing=True)
        e.record(self.stream)
        return e

    def elapsed_ms(self, a, b) -> float:
        return a.elapsed_time(b)

    def reduce(self, x: float, op: str) -> float:
        if self.world == 1:
            return x
        t = self.torch.tensor([float(x)], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX if op == "max" else self.dist.ReduceOp.SUM)
        return float(t.item())

    def gather(self, obj):
        if self.world == 1:
            return [obj]
        out = [None] * self.world
        self.dist.all_gather_object(out, obj)
        return out

    def share_bytes(self, b: bytes | None) -> bytes:
        if self.world == 1:
            return b
        box = [b]
        self.dist.broadcast_object_list(box, src=0)
        return box[0]

    def close(self):
        if self.world > 1:
            self.dist.destroy_process_group()


def make_engine(rt, wl, rank, world, local):
    """This rank's engine: one GPU, or rank `rank` of a partitioned NCCL group."""
    from paper_2508_13550_b200 import Engine
    from paper_2508_13550_b200.engine import nccl_unique_id

    if world == 1 and not getattr(rt, "partitioned", False):
        return Engine(local)
    uid = rt.share_bytes(nccl_unique_id() if rank == 0 else None)
    return Engine.rank(local, world, rank, uid)


# ---------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------

def run_ours(args, rt=None, engine_factory=None, clock_factory=None, fp64_peak=None):
    """The GPU arm.  rt / engine_factory / clock_factory / fp64_peak are injected by the
    launcher tests (CPU + gloo + a fake engine); the bench uses CUDA + NCCL + libcsfs_b200."""
    from paper_2508_13550_b200 import Kernel, ParticleSet, SumStats, TraversalConfig, configs
    from paper_2508_13550_b200.engine import kernel_launches

    rank, world, local = rank_info()
    if rt is None:
        rt = CudaRuntime(local, world)
        rt.partitioned = args.partitioned
    wl = configs.make(args.workload)
    k = Kernel.parse(wl.kernel)
    cfg = TraversalConfig(mac=wl.mac, degree=wl.degree, n0=wl.n0)
    eng = (engine_factory or make_engine)(rt, wl, rank, world, local)
    xyz, w, out = eng.device_arrays(wl, k) if hasattr(eng, "device_arrays") else _device_arrays(rt, wl, k)
    launches = getattr(eng, "launches", None) or kernel_launches

    def step(st=None):
        return eng.csfmm_device(_addr(xyz), wl.n, _addr(xyz), _addr(w), wl.n, k, cfg, _addr(out),
                                getattr(rt, "stream", None) and rt.stream.cuda_stream or 0, st)

    peak = fp64_peak if fp64_peak is not None else eng.probe_fp64_tflops()
    clk = (clock_factory or ClockSampler)(local).start()  # samples kept for the timed region only
    for _ in range(args.warmup):
        step()

    # ---- timed: device-resident (value) -------------------------------------------------
    stats = []
    rt.barrier()
    rt.sync()
    l0 = launches()
    t_wall0 = time.time()
    e0 = rt.event()
    for _ in range(args.steps):
        st = SumStats()
        step(st)
        stats.append(st)
    e1 = rt.event()
    rt.sync()
    clk.mark(t_wall0, time.time())
    clk.stop()
    rt.barrier()
    n_launch = rt.reduce(launches() - l0, "sum")
    ms = rt.reduce(rt.elapsed_ms(e0, e1), "max")
    ms_per_step = ms / args.steps
    value = wl.n * args.steps / (ms * 1e-3)

    # ---- roofline: the evaluation phase on the FP64 pipe, summed over ranks ---------------
    s0 = stats[-1]
    t_int = rt.reduce(statistics.mean(s.t_interact for s in stats), "max")
    exec_evals = rt.reduce(float(s0.evals_executed), "sum")
    list_evals = float(s0.evals_pp + s0.evals_pc + s0.evals_cp + s0.evals_cc)
    peak_mean = rt.reduce(peak, "sum") / world
    ncu, ncu_src, ncu_why = load_ncu(wl.kernel)
    fpp = ncu.get("fp64_flop_per_pair_executed")
    achieved = exec_evals * fpp / t_int / 1e12 / world if fpp else None  # per-GPU TF/s
    phases = {kk: 1e3 * statistics.mean(getattr(s, kk) for s in stats)
              for kk in ("t_tree_build", "t_upward", "t_lists", "t_interact", "t_downward", "t_exchange", "t_total")}
    roof = {"bound": "fp64",
            "kernel": f"evaluation phase: k_mutual + k_interact<Op{wl.kernel}> (PP+PC+CP+CC)",
            "achieved": achieved, "peak": peak_mean, "unit": "TFLOP/s",
            "frac": achieved / peak_mean if achieved else None,
            "traffic": ncu.get("dram_bytes_per_launch"),
            "definition": "achieved = executed pair evaluations (sum over ranks) x FP64 flop per evaluation "
                          "(ncu, this build) / evaluation-phase time (max over ranks) / n_gpus; "
                          "peak = measured DFMA-chain FP64 peak per GPU (csfs_b200_probe_fp64; "
                          "MEASURED_PEAKS.json has no FP64 entry)",
            "ncu_source": ncu_src, "ncu_refused": ncu_why,
            "executed_flop_per_pair": fpp,
            "executed_pair_evals_per_launch": exec_evals,
            "list_pair_evals_per_launch": list_evals,
            # the evaluation throughput itself (flop-count independent: a functor that needs
            # fewer FP64 operations per pair lowers `frac` while raising this)
            "executed_evals_per_s_per_gpu": exec_evals / t_int / world,
            "fp64_pipe_active_pct_ncu": ncu.get("fp64_pipe_active_pct"),
            "frac_of_nominal_37.2": achieved / NOMINAL_FP64_TFLOPS if achieved else None,
            "step_frac": (exec_evals * fpp / (ms_per_step * 1e-3) / 1e12 / world / peak_mean) if fpp else None,
            "libdevice_equiv_tflops": list_evals * LIBDEVICE_FLOP_PER_PAIR[wl.kernel] / t_int / 1e12 / world,
            "libdevice_equiv_note": "SURVEY.md §8d convention (reference formula as libdevice would execute it, "
                                    f"{LIBDEVICE_FLOP_PER_PAIR[wl.kernel]} flop per LISTED pair evaluation); "
                                    "exceeds the executed rate because symmetric pairs are evaluated once and the "
                                    "functor needs fewer FP64 ops — a throughput-equivalent, not a roofline",
            "kernel_ms": t_int * 1e3, "share_of_step": t_int / (ms_per_step * 1e-3),
            "phases_ms_rank0": phases}
    if world == 1:
        # the HBM-type phases against the measured copy bandwidth (SURVEY.md §8d algorithmic
        # bytes): tree build = xyz in (24 B/pt) + per level xi, eta, idx moved (2 x 20 B/pt) +
        # sorted xyz, w, perm out (36 B/pt) — the traffic of the level-by-level partition;
        # the label-then-sort build (tree.cu) moves 24 B/pt per level plus one sort and
        # gather, i.e. about as much, so the same figure is kept; upward leaf = 24 B/pt +
        # (p+1)^2 x 8 B per leaf; downward leaf = 16 B/pt + 8 dim B/pt
        n, npp = wl.n, (wl.degree + 1) ** 2
        hbm_bytes = {"t_tree_build": n * (24 + 40 * s0.tgt_depth + 36),
                     "t_upward": n * 24 + npp * 8 * s0.src_leaves,
                     "t_downward": n * (16 + 8 * k.out_dim())}
        roof["hbm_phases"] = {
            ph: {"algorithmic_bytes": b, "ms": phases[ph], "gbs": b / (phases[ph] * 1e-3) / 1e9,
                 "frac_of_hbm": b / (phases[ph] * 1e-3) / 1e9 / HBM_GBS}
            for ph, b in hbm_bytes.items()}

    # ---- e2e through the host-pointer C-ABI ---------------------------------------------
    e2e = None
    if not args.no_e2e:
        hx, hw, ho = eng.host_arrays(wl, k) if hasattr(eng, "host_arrays") else _host_arrays(wl, k)
        p = ParticleSet(hx, hw)
        eng.csfmm_sum(p, p, k, cfg, out=ho)
        rt.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            eng.csfmm_sum(p, p, k, cfg, out=ho)
        dt = rt.reduce(time.perf_counter() - t0, "max")
        rt.barrier()
        e2e = {"value": wl.n * args.steps / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(world * (wl.xyz.nbytes + wl.weights.nbytes)),
               "d2h_bytes_per_step": int(world * wl.n * k.out_dim() * 8),
               "timing": "wall clock around the synchronous host-pointer call (csfs_b200_csfmm), pinned host "
                         "buffers, max over ranks; every rank copies the full inputs in and the full result out"}

    # ---- CPU baseline (rank 0, N = 1 only) ------------------------------------------------
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cores = os.cpu_count() or 1
        try:
            r = cpu_reference(wl, 1, 0)[0]
            cpu = {"value": r["value"], "unit": UNIT, "cores": cores, "kind": "reference",
                   "sample": cpu_sample_text(wl, cores), "cpu_model": cpu_model(), "phases_s": r}
        except Exception as ex:  # the checker must not break the GPU line
            cpu = {"value": None, "unit": UNIT, "cores": cores, "kind": "reference", "sample": f"unavailable: {ex}"}

    clocks = rt.gather(clk.summary())
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": workload_config(wl, "1 GPU" if world == 1 and not args.partitioned else
                                          f"target-partitioned x{world} (depth-1 subtrees; NCCL all-gathers)"),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(n_launch),
                "clocks": clocks[0] if world == 1 else dict(clocks[0], per_gpu=clocks),
                "fp64_frac_p2p_m2l": roof["frac"]}
        if world > 1:
            line["exchange_ms_rank0"] = phases["t_exchange"]
        emit(line)
    eng.close()
    rt.close()
    return 0


def _addr(x):
    return x.data_ptr() if hasattr(x, "data_ptr") else int(x)


def _device_arrays(rt, wl, k):
    import torch

    xyz = torch.from_numpy(wl.xyz).to(rt.dev)
    w = torch.from_numpy(wl.weights).to(rt.dev)
    out = torch.empty(wl.n * k.out_dim(), dtype=torch.float64, device=rt.dev)
    return xyz, w, out


def _host_arrays(wl, k):
    import torch

    hx = torch.from_numpy(wl.xyz).pin_memory()
    hw = torch.from_numpy(wl.weights).pin_memory()
    ho = torch.empty(wl.n * k.out_dim(), dtype=torch.float64).pin_memory()
    return hx.numpy(), hw.numpy(), ho.numpy()


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--partitioned", action="store_true",
                    help="one GPU through the partitioned NCCL group path (csfs_b200_create_rank, 1 rank)")
    args = ap.parse_args(argv)
    if args.impl == "ours":
        args.warmup = max(args.warmup, 3)
    return args


def main(argv=None):
    global _OUT_FD
    argv = sys.argv[1:] if argv is None else argv
    args = parse(argv)
    in_torchrun = "RANK" in os.environ and "WORLD_SIZE" in os.environ
    if args.impl == "ours" and not in_torchrun and args.gpus > 1:
        have = visible_gpus()
        if have < args.gpus:
            print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {have}; "
                  "refusing to measure fewer", file=sys.stderr)
            return 2
        cmd = relaunch_argv(argv, args.gpus)
        print("bench.py: relaunching as " + " ".join(cmd), file=sys.stderr)
        return subprocess.call(cmd)
    if in_torchrun and args.impl == "ours":
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
            return 2
        if visible_gpus() < world:
            print(f"bench.py: {world} ranks need {world} visible GPUs, found {visible_gpus()}", file=sys.stderr)
            return 2
    sys.stdout.flush()
    _OUT_FD = os.dup(1)
    os.dup2(2, 1)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

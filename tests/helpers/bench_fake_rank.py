"""One rank of bench.py's GPU arm on the CPU (tests/test_bench_launcher.py): gloo for the
barrier / max / sum / gather, perf_counter in place of CUDA events, and a stand-in engine
that sleeps a rank-dependent time per step and reports per-rank evaluation counts — so the
test can check what rank 0 prints: n_gpus, the max over ranks, sums over ranks, per-GPU
clocks.  Run under torchrun (RANK / WORLD_SIZE set)."""
import os
import sys
import time

import numpy as np
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

SLEEP_S = 0.02  # rank r sleeps (r + 1) x this per step
EVALS = 1000    # rank r executes (r + 1) x this evaluations per step


class GlooRuntime:
    def __init__(self, world):
        dist.init_process_group("gloo")
        self.world = world
        self.stream = None

    def sync(self):
        pass

    def barrier(self):
        dist.barrier()

    def event(self):
        return time.perf_counter()

    def elapsed_ms(self, a, b):
        return (b - a) * 1e3

    def reduce(self, x, op):
        import torch

        t = torch.tensor([float(x)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    def gather(self, obj):
        out = [None] * self.world
        dist.all_gather_object(out, obj)
        return out

    def share_bytes(self, b):
        box = [b]
        dist.broadcast_object_list(box, src=0)
        return box[0]

    def close(self):
        dist.destroy_process_group()


class FakeEngine:
    def __init__(self, rank):
        self.rank = rank
        self.n_launch = 0

    def device_arrays(self, wl, k):
        return 1, 2, 3

    def host_arrays(self, wl, k):
        return wl.xyz, wl.weights, np.empty(wl.n * k.out_dim())

    def launches(self):
        return self.n_launch

    def probe_fp64_tflops(self):
        return 30.0

    def csfmm_device(self, *a):
        st = a[-1]
        time.sleep(SLEEP_S * (self.rank + 1))
        self.n_launch += 7
        if st is not None:
            st.t_interact = 0.5 * SLEEP_S * (self.rank + 1)
            st.evals_executed = EVALS * (self.rank + 1)
            st.evals_pp = 4 * EVALS
        return st

    def csfmm_sum(self, *a, **kw):
        time.sleep(SLEEP_S * (self.rank + 1))

    def close(self):
        pass


class NoClock:
    def __init__(self, gpu):
        self.gpu = gpu

    def start(self):
        return self

    def mark(self, a, b):
        pass

    def stop(self):
        pass

    def summary(self):
        return {"gpu": self.gpu, "sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}


if __name__ == "__main__":
    args = bench.parse(sys.argv[1:])
    rank, world, _ = bench.rank_info()
    sys.exit(bench.run_ours(args, rt=GlooRuntime(world), engine_factory=lambda rt, wl, r, w, l: FakeEngine(r),
                            clock_factory=NoClock, fp64_peak=30.0))

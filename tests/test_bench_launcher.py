"""CPU: bench.py's multi-GPU contract — `--gpus N` really runs N ranks
(re-exec under torchrun), refuses to measure fewer GPUs than asked, and rank 0's line
carries the max over ranks and the sums over ranks.  The two-rank run uses gloo and a
stand-in engine (tests/helpers/bench_fake_rank.py); the GPU path itself is exercised by the
driver's bench and tests/test_gpu_group.py."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def _env(**kw):
    e = dict(os.environ)
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT"):
        e.pop(k, None)
    e.update({k: str(v) for k, v in kw.items()})
    e["CUDA_VISIBLE_DEVICES"] = ""
    return e


def test_relaunch_argv_is_torchrun_on_loopback():
    cmd = bench.relaunch_argv(["--gpus", "4", "--steps", "2"], 4, port=29555)
    assert cmd[:3] == [sys.executable, "-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--master-port=29555" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"] and cmd[-5].endswith("bench.py")


def test_more_gpus_than_visible_fails_loudly():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=_env(), timeout=300)
    assert r.returncode == 2
    assert r.stdout.strip() == ""  # no silent 1-GPU line
    assert "needs 2 visible GPUs" in r.stderr


def test_world_size_must_match_gpus():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "1"],
                       capture_output=True, text=True, env=_env(RANK=0, WORLD_SIZE=1, LOCAL_RANK=0), timeout=300)
    assert r.returncode == 2 and r.stdout.strip() == ""
    assert "WORLD_SIZE=1" in r.stderr


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.timeout(600)
def test_two_ranks_over_gloo_report_max_and_sums():
    sys.path.insert(0, os.path.join(ROOT, "tests", "helpers"))
    import bench_fake_rank as F

    steps = 3
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}",
           os.path.join(ROOT, "tests", "helpers", "bench_fake_rank.py"),
           "--gpus", "2", "--steps", str(steps), "--warmup", "3", "--workload", "c1", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, env=_env(), timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == steps
    # ms_per_step = the slower rank (rank 1 sleeps 2 x SLEEP_S per step)
    assert d["ms_per_step"] >= 2 * F.SLEEP_S * 1e3 * 0.95
    assert abs(d["value"] - 6144 * steps / (d["ms_per_step"] * steps * 1e-3)) < 1e-6 * d["value"]
    roof = d["roofline"]
    assert roof["executed_pair_evals_per_launch"] == F.EVALS * (1 + 2)  # summed over ranks
    assert abs(roof["kernel_ms"] - 0.5 * F.SLEEP_S * 2 * 1e3) < 1e-9  # max over ranks
    assert roof["peak"] == 30.0
    assert d["gpu_launches"] == 2 * 7 * steps  # both ranks' launches in the timed region
    assert [c["gpu"] for c in d["clocks"]["per_gpu"]] == [0, 1]
    assert "target-partitioned x2" in d["config"]["parallelism"]
    assert d["e2e"]["value"] > 0 and d["cpu_baseline"] is None

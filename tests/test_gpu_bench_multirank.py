"""bench.py's N > 1 path (the driver's scaling run: one rank per GPU, barrier + max-over-ranks
timing, stream partition, frame gather after the timed region) executed for real: two ranks
under torchrun sharing the box's one GPU, collectives over gloo (SF_BENCH_DIST_BACKEND; NCCL
refuses two ranks on one device).  Rank 0 must print one JSON line for the whole job."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _run(extra, timeout=600):
    env = dict(os.environ, SF_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", *extra]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 only
    return json.loads(lines[0])


@pytest.mark.gpu
def test_bench_two_ranks_dit():
    S, steps, n = 4, 3, 4
    d = _run(["--steps", str(steps), "--warmup", "4", "--streams", str(S), "--no-decode", "--no-cpu-baseline"])
    assert d["n_gpus"] == 2 and d["steps"] == steps and d["scaling"] == "weak"
    assert d["config"]["streams_total"] == 2 * S and d["config"]["streams_per_gpu"] == S
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["ms_per_step"] > 0
    assert all(d["check"][k] for k in ("frames_finite", "frame_ids_ok", "ring_finite"))
    g = d["gather"]
    assert g["window_steps"] == n and g["frames_gathered"] == n * 2 * S
    assert g["frame_ids_valid"] == n * 2 * S  # past warm-up every stream emits every step
    assert g["frames_emitted_timed_total"] == 2 * S * steps


@pytest.mark.gpu
def test_bench_two_ranks_mock():
    d = _run(["--model", "mock", "--steps", "20", "--warmup", "4", "--streams", "8", "--no-cpu-baseline"])
    assert d["n_gpus"] == 2 and d["config"]["streams_total"] == 16
    assert d["value"] > 0 and d["e2e"]["value"] > 0

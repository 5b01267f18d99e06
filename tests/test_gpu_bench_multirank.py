"""bench.py's multi-rank arms end to end on one GPU: torchrun with 2 ranks, the one-GPU test knobs
(GPA_BENCH_ONE_GPU=1 puts both ranks on GPU 0, GPA_BENCH_BACKEND=gloo since NCCL refuses two ranks
on one device).  Timings from this are meaningless; the test checks that every code path of the
N > 1 step (DP-1 all-reduce and its report, DP-2 kernel partition) runs and rank 0 alone prints one
JSON line that counted every record."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _need_cuda(cuda_available):
    if not cuda_available:
        pytest.skip("no CUDA device")


def _torchrun(*args):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, GPA_BENCH_ONE_GPU="1", GPA_BENCH_BACKEND="gloo")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2",
                        "--steps", "1", "--warmup", "3", "--e2e-steps", "1", *args],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_dp1_large_arm_two_ranks():
    d = _torchrun("--workload", "large", "--records", "20000000")
    assert d["n_gpus"] == 2 and d["config"]["records_total"] == 40_000_000
    ar = d["allreduce"]
    assert ar["bytes"] == (50_000 * 2 * 9 + 4) * 8 and ar["standalone_ms"] > 0 and ar["backend"] == "gloo"
    assert d["e2e"]["h2d_bytes_per_step"] == 40_000_000 * 8


def test_dp2_batch_arm_two_ranks():
    d = _torchrun("--workload", "batch")
    assert d["n_gpus"] == 2 and "allreduce" not in d and d["value"] > 0

"""bench.py --impl reference (the oracle on the host cores) keeps the driver's JSON contract and runs
without a GPU; under torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(extra_env=None, gpus=1):
    env = dict(os.environ, **(extra_env or {}))
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload", "rodinia", "--steps", "1",
                        "--warmup", "0", "--ref-sample", "200000", "--gpus", str(gpus)], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return [l for l in r.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    lines = _run()
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "samples/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_other_ranks_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2"}, gpus=2) == []


def test_reference_arm_prints_our_config():
    """The reference arm times a bounded sample of OUR workload and prints our `config` object."""
    d = json.loads(_run()[0])
    assert d["config"]["records_per_gpu"] == 10_000_000 and d["config"]["parallelism"].startswith("dp1")
    assert "first 200000 of the 10000000 records" in d["cpu_baseline"]["sample"]
    host = d["cpu_baseline"]["host"]
    assert host["nproc"] >= 1 and host["usable_cores"] >= 1


def test_gpus_flag_relaunches_under_torchrun():
    """`bench.py --gpus N` without torchrun re-executes itself as N ranks (one per GPU)."""
    env = dict(os.environ, GPA_BENCH_DRYRUN="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "4", "--steps", "2", "--warmup", "3"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    cmd = json.loads([l for l in r.stdout.splitlines() if l.startswith("{")][0])["relaunch"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd
    assert "--master-addr=127.0.0.1" in cmd and cmd[-6:] == ["--gpus", "4", "--steps", "2", "--warmup", "3"]


def test_gpus_flag_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    for impl in ("ours", "reference"):
        r = subprocess.run([sys.executable, "bench.py", "--gpus", "8", "--impl", impl], cwd=ROOT, env=env,
                           capture_output=True, text=True, timeout=300)
        assert r.returncode == 2 and "WORLD_SIZE=2" in r.stderr, (impl, r.returncode, r.stderr[-500:])

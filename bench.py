#!/usr/bin/env python
"""Benchmark of GPA's hot path on B200: PC samples/s attributed (ingest + blame + rollup +
estimate), and the ingest kernel's achieved fraction of the measured HBM roofline.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload large|rodinia|batch|pelec] [--impl reference]
  torchrun --nproc-per-node N bench.py --gpus N ...     (one rank per GPU, NCCL all-reduce)

Workload: BASELINE.json config 3 -- the 50k-instruction PeleC/ExaTENSOR-shaped
program with 10^9 synthetic PC-sample records per GPU (8 GB, device-resident, far larger than
L2, so no flush is needed between steps) at EVERY N.  At N > 1 rank r ingests records
[r*1e9, (r+1)*1e9) of the same counter-based stream (config 5's sharding), the count table is
all-reduced over NCCL, and blame / rollup / estimate run replicated: weak scaling, the same
per-GPU load at N = 1, 2, 4, 8.  `--gpus N` without torchrun re-launches itself under
`torch.distributed.run --nproc-per-node N`; under torchrun `--gpus` must equal WORLD_SIZE.

One step = reset -> ingest -> [all_reduce] -> blame -> aggregate -> estimate, all enqueued on one
stream; timed with CUDA events, W warm-up steps, K timed steps, barrier + synchronize on both
sides, max over ranks.  Rank 0 prints one JSON line.
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

METRIC = "PC samples/sec attributed (ingest+blame+rollup) at 1/2/4/8 B200; % HBM peak"
WORKLOADS = {
    # name: (config id, records per GPU)
    "large": (3, 1_000_000_000),
    "rodinia": (2, 10_000_000),
    "batch": (4, 100_000_000),      # records in total (the batch is partitioned, DP-2)
    "pelec": (6, 1_000_000_000),    # not a BASELINE config: 200k-instruction kernel
}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _traffic_from_profile(workload, records):
    """dram bytes per ingest launch from the committed ncu --set full summary, if it was captured
    at this launch size (else None: the figure is per launch, not per record)."""
    path = os.path.join(ROOT, "profiles", "ncu_ingest_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        e = d.get(workload, {})
        if e.get("records_per_launch") != records:
            return None
        return e.get("dram_bytes_per_launch")
    except Exception:
        return None


def _host_info():
    """The box's host CPU beside the oracle's timing (north_star: "core count stated")."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        usable = len(os.sched_getaffinity(0))
    except Exception:
        usable = os.cpu_count()
    return {"cpu_model": model, "nproc": os.cpu_count(), "usable_cores": usable}


def _check_world(args):
    """--gpus N must match the launch: without torchrun, N > 1 re-executes this script under
    torch.distributed.run (one rank per GPU); under torchrun, WORLD_SIZE must equal N."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is None:
        if args.gpus > 1:
            import socket
            sk = socket.socket()
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
            sk.close()
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
                   "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
            if os.environ.get("GPA_BENCH_DRYRUN") == "1":     # test hook: show the re-launch, do not run it
                print(json.dumps({"relaunch": cmd}), flush=True)
                sys.exit(0)
            os.execv(sys.executable, cmd)
        return 1
    if int(ws) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}: launch one rank per GPU\n")
        sys.exit(2)
    return int(ws)


def large_config(args, world, prog, cfg, n_per):
    """The `config` object of the large / rodinia arms (printed identically by --impl reference)."""
    what = f"BASELINE config {cfg}" if cfg != 6 else "PeleC-scale (P:708-714, beyond BASELINE's configs)"
    return {"workload": f"{args.workload}: {what} program ({prog.n_instr} instrs, {prog.n_edges} edges, "
                        f"{prog.n_loops} loops), {n_per} records per GPU"
                        + (f" (the first {n_per * world} records of config 5's 10^10-record stream, {n_per} per GPU)"
                           if world > 1 else ""),
            "records_per_gpu": n_per, "records_total": n_per * world,
            "l2": "inputs larger than L2 (8 B/record)" if n_per * 8 > 126 << 20 else "inputs smaller than L2",
            "parallelism": f"dp{world} (sample-stream shards + NCCL all-reduce of counts)"}


def step_alg_bytes(prog, n_records, table_word=8):
    """SURVEY §8(d) algorithmic bytes of one whole step (ingest + blame + rollup): records once,
    instruction SoA + CSR read once, count table written and read once, per-instruction blame and
    the rollup outputs written once."""
    n, E, R = prog.n_instr, prog.n_edges, prog.n_reasons
    ncol = 10 + R - 4
    segs = prog.n_lines + 2 * prog.n_loops + (len(prog.func_begin) - 1) + (len(prog.kernel_func_begin) - 1)
    return (8 * n_records + 4 * (n + 1) + 16 * n + 20 * E + 2 * n * 2 * R * table_word + 64 * n
            + segs * (ncol * 2 * 8 + 16))


def oracle_throughput(prog, records: np.ndarray, patterns):
    """Time the oracle (tests' CPU implementation, as it stands) on `records`: whole path."""
    import oracle
    from tests._common import oracle_pattern
    op = oracle.OracleProgram(prog)
    t0 = time.perf_counter()
    C, _ = op.histogram(records)
    b = op.blame(C)
    op.rollup(C, b["V"])
    op.estimate(C, b, [oracle_pattern(p) for p in patterns])
    return time.perf_counter() - t0


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores (rank 0 only) on our arm's workload and
    config; each step is a bounded sample (the first `sample` records of the same stream), sized so
    the whole --warmup W --steps K run stays within a few minutes."""
    world = _check_world_ref(args)
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import gpagen
    from gpagen.patterns import table2
    if args.workload == "batch":
        from gpagen import batch
        prog = batch.config4_program()
        spec = batch.config4_stream(prog)
        n_per = args.records or WORKLOADS["batch"][1]
        config = batch_config(args, world, prog, n_per)
        cfg = 4
    else:
        cfg, n_per = WORKLOADS[args.workload]
        n_per = args.records or n_per
        prog = gpagen.config_program(cfg)
        spec = gpagen.config_stream(prog, cfg)
        config = large_config(args, world, prog, cfg, n_per)
    pats = table2(prog.n_reasons)
    if args.ref_sample:
        sample = min(args.ref_sample, n_per)
    else:   # size the sample from a pilot run: the whole W + K run within ~150 s of oracle time
        pilot = min(n_per, 5_000_000)
        rate = pilot / oracle_throughput(prog, spec.host(0, pilot), pats)
        sample = int(min(n_per, max(pilot, rate * 150.0 / max(1, args.steps + args.warmup))))
        sample -= sample % 1_000_000 if sample > 1_000_000 else 0
    recs = spec.host(0, sample)
    for _ in range(args.warmup):
        oracle_throughput(prog, recs, pats)
    times = [oracle_throughput(prog, recs, pats) for _ in range(args.steps)]
    t = sum(times) / len(times)
    v = sample / t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "strong" if args.workload == "batch" else "weak", "vs_baseline": None, "dtype": "u64+f64",
            "data": "synthetic", "config": config,
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": 1, "kind": "oracle",
                             "sample": f"first {sample} of the {n_per} records of this workload's stream per step "
                                       "(histogram+blame+rollup+estimate, single-threaded)",
                             "host": _host_info()},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _check_world_ref(args):
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None and int(ws) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}\n")
        sys.exit(2)
    return args.gpus if ws is None else int(ws)


def batch_config(args, world, prog, n_total):
    return {"workload": f"batch: BASELINE config 4, {prog.n_kernels} kernels, {prog.n_instr} instrs, "
                        f"{prog.n_edges} edges, {n_total} records grouped by kernel launch",
            "records_total": n_total, "l2": "inputs larger than L2 (0.8 GB records, 0.65 GB table)",
            "parallelism": f"dp2-{world} (kernel partition, no count collective)"}


def _local_device() -> int:
    """This rank's GPU: LOCAL_RANK.  GPA_BENCH_ONE_GPU=1 (test knob, never used for a reported
    number) puts every rank on GPU 0 so the multi-rank code path can be exercised on one GPU."""
    if os.environ.get("GPA_BENCH_ONE_GPU") == "1":
        return 0
    return int(os.environ.get("LOCAL_RANK", "0"))


def _init_dist(dist, dev):
    """NCCL over NVLink; GPA_BENCH_BACKEND=gloo (test knob, with GPA_BENCH_ONE_GPU) runs the same
    collectives through host memory, since NCCL refuses two ranks on one GPU."""
    backend = os.environ.get("GPA_BENCH_BACKEND", "nccl")
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)

def run_batch(args):
    """--workload batch: BASELINE config 4 -- 10^4 kernels (~4.5 M instructions), 10^8 records
    grouped by kernel launch.  N > 1: DP-2 -- contiguous kernel ranges balanced by sample count,
    each rank analyses its slice (no count collective); estimates are gathered to every rank
    (outside the timed step).  Step = reset -> gpa_ingest_segments -> blame -> aggregate -> estimate."""
    import torch
    import torch.distributed as dist
    from gpagen import batch
    from gpagen.patterns import table2
    from paper_2009_04061_b200 import Program
    from paper_2009_04061_b200.dist import gather_estimates, partition_kernels, slice_program

    world = _check_world(args)
    rank = int(os.environ.get("RANK", "0"))
    local = _local_device()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        _init_dist(dist, dev)
    n_total = args.records or WORKLOADS["batch"][1]
    prog = batch.config4_program()
    spec = batch.config4_stream(prog)
    recs = spec.device(0, n_total).view(torch.int64)            # the application's whole stream
    pcs = recs & 0xFFFFFFFF
    kb = batch.kernel_pc_begin(prog)
    kid = torch.bucketize(pcs, torch.as_tensor(kb[1:-1], device=dev), right=True)
    ksamp = torch.bincount(kid, minlength=prog.n_kernels).cpu().numpy()
    bounds = partition_kernels(ksamp, world)
    k0, k1 = bounds[rank], bounds[rank + 1]
    sub, maps = (prog, {"pc_base": 0, "n_instr": prog.n_instr}) if world == 1 else slice_program(prog, k0, k1)
    lo, hi = maps["pc_base"], maps["pc_base"] + maps["n_instr"]
    mine = recs[(pcs >= lo) & (pcs < hi)]
    del recs, pcs, kid
    order, sb, sk = batch.grouped_order((mine & 0xFFFFFFFF) - lo, sub)
    g = mine[order].contiguous()
    del mine, order
    seg_begin = torch.from_numpy(sb.astype(np.int64)).to(dev)
    seg_kernel = torch.from_numpy(sk.view(np.int32)).to(dev)
    n_mine = int(g.numel())
    pats = table2(prog.n_reasons)
    P = Program(sub, device=dev)
    P.set_patterns(pats)
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()

    def step(ev=None):
        P.reset()
        if ev is not None:
            ev[0].record(stream)
        P.ingest_segments(g, seg_begin, seg_kernel, pc_base=lo)
        if ev is not None:
            ev[1].record(stream)
        P.analyze()
        if ev is not None:
            ev[2].record(stream)

    if args.profile:
        step()
        torch.cuda.synchronize()
        return
    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = P.launches
    torch.cuda.synchronize()
    t0.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t1.record(stream)
    torch.cuda.synchronize()
    launches = P.launches - l0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = t0.elapsed_time(t1)
    ingest_ms = sum(a.elapsed_time(b) for a, b, _ in evs) / args.steps
    analyze_ms = sum(b.elapsed_time(c) for _, b, c in evs) / args.steps
    if world > 1:
        t = torch.tensor([ms, ingest_ms, analyze_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ingest_ms, analyze_ms = (float(x) for x in t)
    ms_per_step = ms / args.steps
    st = P.stats()   # valid + invalid samples = every sample of this rank's records (count 1 each)
    assert st[0] + st[2] == n_mine, (st, n_mine)
    est = P.read_estimates_array()
    allest = gather_estimates(np.ascontiguousarray(est["speedup"]))
    assert allest.shape[0] == prog.n_kernels

    # end to end: pinned host -> device copy of this rank's grouped records inside the timed region
    host = torch.empty(n_mine * 8, dtype=torch.uint8, pin_memory=True)
    host.copy_(g.view(torch.uint8))
    dbuf = torch.empty_like(g)
    e_steps = max(args.e2e_steps, 1)
    torch.cuda.synchronize()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    for _ in range(e_steps):
        dbuf.view(torch.uint8).copy_(host, non_blocking=True)
        P.reset()
        P.ingest_segments(dbuf, seg_begin, seg_kernel, pc_base=lo)
        P.analyze()
        P.read_estimates_array()
    eb.record(stream)
    torch.cuda.synchronize()
    e_ms = ea.elapsed_time(eb)
    if world > 1:
        t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e_ms = float(t[0])
    e2e = {"value": n_total * e_steps / (e_ms / 1e3), "unit": "samples/s", "h2d_bytes_per_step": n_total * 8,
           "d2h_bytes_per_step": prog.n_kernels * len(pats) * 56, "ms_per_step": e_ms / e_steps,
           "path": "pinned H2D copy + gpa_ingest_segments + gpa_analyze + gpa_read_estimates"}
    peak, peak_kind = _peaks()
    alg_bytes = n_mine * 8 + sub.n_instr * 2 * sub.n_reasons * 8     # records once + table written once
    achieved = alg_bytes / (ingest_ms / 1e3) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = min(n_total, 10_000_000)
        h = spec.host(0, sample)
        t_or = oracle_throughput(prog, h, pats)
        cpu = {"value": sample / t_or, "unit": "samples/s", "cores": 1, "kind": "oracle",
               "sample": f"first {sample} records of the config-4 stream (whole 4.5M-instruction batch); "
                         "histogram+blame+rollup+estimate", "seconds": t_or, "host": _host_info()}
    if rank == 0:
        step_bytes = step_alg_bytes(sub, n_mine)
        line = {
            "metric": METRIC, "value": n_total / (ms_per_step / 1e3), "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64+f64", "data": "synthetic",
            "config": batch_config(args, world, prog, n_total),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "kernel": "ingest_segments", "peak_kind": peak_kind,
                         "alg_bytes_per_launch": alg_bytes, "ingest_ms": ingest_ms,
                         "ingest_share_of_step": ingest_ms / ms_per_step, "blame_rollup_estimate_ms": analyze_ms,
                         "step": {"alg_bytes": step_bytes, "ms": ms_per_step,
                                  "achieved": step_bytes / (ms_per_step / 1e3) / 1e9,
                                  "frac": step_bytes / (ms_per_step / 1e3) / 1e9 / peak,
                                  "note": "rank 0's slice: SURVEY §8(d) bytes of ingest+blame+rollup over the whole step"}},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="large", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--records", type=int, default=0, help="override records per GPU")
    ap.add_argument("--variant", default=None, help="force ingest variant (smem|part|l2)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="records per reference step (default: sized from a pilot run, <= records per GPU)")
    ap.add_argument("--profile", action="store_true", help="one short step for ncu (no JSON rules)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.workload == "batch":
        return run_batch(args)

    import torch
    import torch.distributed as dist
    import gpagen
    from gpagen.patterns import table2
    from paper_2009_04061_b200 import Program

    world = _check_world(args)
    rank = int(os.environ.get("RANK", "0"))
    local = _local_device()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        _init_dist(dist, dev)
    cfg, n_per = WORKLOADS[args.workload]    # the same records per GPU at every N (weak scaling)
    if args.records:
        n_per = args.records
    prog = gpagen.config_program(cfg)
    pats = table2(prog.n_reasons)
    P = Program(prog, device=dev)
    if args.variant:
        P.variant = args.variant
    P.set_patterns(pats)
    spec = gpagen.config_stream(prog, cfg)
    recs = spec.device(rank * n_per, n_per)          # this rank's shard, device-resident
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    red = P.reduce_view()    # [counts | stats]: the one buffer the DP-1 step all-reduces

    def step(ev_a=None, ev_b=None, ev_c=None, ev_r=None):
        P.reset()
        if ev_a is not None:
            ev_a.record(stream)
        P.ingest(recs)
        if ev_b is not None:
            ev_b.record(stream)
        if world > 1:
            dist.all_reduce(red, op=dist.ReduceOp.SUM)
        if ev_r is not None:
            ev_r.record(stream)
        P.analyze()          # blame + aggregate + estimate (one CUDA graph of the library's kernels)
        if ev_c is not None:
            ev_c.record(stream)

    if args.profile:
        step()
        torch.cuda.synchronize()
        return

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    sampler = ClockSampler(local)
    sampler.start()
    time.sleep(0.3)
    ing = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(4)) for _ in range(args.steps)]
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = P.launches
    torch.cuda.synchronize()
    t0.record(stream)
    for k in range(args.steps):
        step(*ing[k])
    t1.record(stream)
    torch.cuda.synchronize()
    launches = P.launches - l0
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    ms = t0.elapsed_time(t1)
    ingest_ms = sum(a.elapsed_time(b) for a, b, _, _ in ing) / args.steps
    analyze_ms = sum(r.elapsed_time(c) for _, _, c, r in ing) / args.steps
    reduce_ms = sum(b.elapsed_time(r) for _, b, _, r in ing) / args.steps
    if world > 1:
        t = torch.tensor([ms, ingest_ms, reduce_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, ingest_ms, reduce_ms = float(t[0]), float(t[1]), float(t[2])
    ms_per_step = ms / args.steps

    ar_ms = 0.0
    if world > 1:   # the collective alone, on a buffer the size of [counts | stats] (outside the timed region)
        scratch = torch.zeros_like(red)   # same size as [counts | stats]; sums stay 0
        dist.barrier()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        dist.all_reduce(scratch, op=dist.ReduceOp.SUM)
        a0.record(stream)
        for _ in range(10):
            dist.all_reduce(scratch, op=dist.ReduceOp.SUM)
        a1.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a0.elapsed_time(a1) / 10], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ar_ms = float(t[0])
        del scratch

    # correctness guard on the timed output: every record of every rank was counted
    st = P.stats()   # valid + invalid samples = every sample of every rank (timed streams: count 1)
    total = n_per * world
    assert st[0] + st[2] == total, (st, total)

    # end to end through the C ABI from pinned host memory (H2D inside the timed region)
    e2e = None
    if args.e2e_steps > 0:
        host = torch.empty(n_per * 8, dtype=torch.uint8, pin_memory=True)
        host.copy_(recs)
        est_bytes = P.n_kernels * P.n_patterns * 56
        for _ in range(1):
            P.reset(); P.ingest_host(host); P.analyze(); P.read_estimates_array()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = time.perf_counter()
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(stream)
        for _ in range(args.e2e_steps):
            P.reset()
            P.ingest_host(host)
            if world > 1:
                dist.all_reduce(red, op=dist.ReduceOp.SUM)
            P.analyze()
            P.read_estimates_array()
        eb.record(stream)
        torch.cuda.synchronize()
        e_ms = ea.elapsed_time(eb)
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t[0])
        e2e = {"value": total * args.e2e_steps / (e_ms / 1e3), "unit": "samples/s",
               "h2d_bytes_per_step": n_per * 8 * world, "d2h_bytes_per_step": est_bytes * world,
               "ms_per_step": e_ms / args.e2e_steps, "path": "gpa_ingest_samples_host (pinned, 2x32 MB staging ring)"}
        del host

    peak, peak_kind = _peaks()
    table_bytes = prog.n_instr * 2 * prog.n_reasons * 8
    alg_bytes = n_per * 8 + 2 * table_bytes
    achieved = alg_bytes / (ingest_ms / 1e3) / 1e9
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = min(n_per, 1_000_000_000)
        h = recs[: sample * 8].cpu().numpy().view(np.uint64)
        t_or = oracle_throughput(prog, h, pats)
        cpu = {"value": sample / t_or, "unit": "samples/s", "cores": 1, "kind": "oracle",
               "sample": f"{sample} records (the same device stream, copied to host); histogram+blame+rollup+estimate",
               "seconds": t_or, "host": _host_info()}
    if rank == 0:
        step_bytes = step_alg_bytes(prog, n_per)
        line = {
            "metric": METRIC, "value": total / (ms_per_step / 1e3), "unit": "samples/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u64+f64", "data": "synthetic",
            "config": large_config(args, world, prog, cfg, n_per),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic_from_profile(args.workload, n_per),
                         "kernel": f"ingest ({P.variant} variant)", "peak_kind": peak_kind,
                         "alg_bytes_per_launch": alg_bytes,
                         "ingest_ms": ingest_ms, "ingest_share_of_step": ingest_ms / ms_per_step,
                         "blame_rollup_estimate_ms": analyze_ms,
                         "step": {"alg_bytes": step_bytes, "ms": ms_per_step,
                                  "achieved": step_bytes / (ms_per_step / 1e3) / 1e9,
                                  "frac": step_bytes / (ms_per_step / 1e3) / 1e9 / peak,
                                  "note": "SURVEY §8(d) bytes of ingest+blame+rollup (per GPU) over the whole "
                                          "timed step (incl. estimate and, at N > 1, the all-reduce)"}},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        if world > 1:
            # the DP-1 exchange: one SUM all-reduce of [counts | stats]; bus bandwidth 2(p-1)/p * bytes / t
            # against NVLink 5's 900 GB/s per direction.  "ms" is the in-step time
            # (it includes the wait for the slowest rank's ingest); "standalone_ms" times the same
            # collective alone on a same-size buffer, all ranks aligned, after the timed region
            rb = red.numel() * 8
            bus = 2 * (world - 1) / world * rb / (ar_ms / 1e3) / 1e9 if ar_ms > 0 else None
            line["allreduce"] = {"bytes": rb, "ms": reduce_ms, "standalone_ms": ar_ms, "busbw_gbs": bus,
                                 "peak_gbs": 900.0, "frac": bus / 900.0 if bus else None,
                                 "backend": dist.get_backend()}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Probe: throughput of the GPU PC-sampling simulator as a workload generator (samples/s)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from gpagen import sass as gs
from paper_2009_04061_b200 import simulate_sass
S = gs.random_sass(1, 41, func_len=(150, 300))
cfg = dict(schedulers=4, warps_per_scheduler=4, period=5, trip_count=4, rbar_latency=2, max_cycles=5_000_000, seed=3)
n_sm = int(sys.argv[1]) if len(sys.argv) > 1 else 9472
simulate_sass(S, 64, 20_000, **cfg)
torch.cuda.synchronize()
t = time.perf_counter(); rec, tr, counts = simulate_sass(S, n_sm, 20_000, **cfg); torch.cuda.synchronize(); dt = time.perf_counter() - t
n = int(counts.sum())
t = time.perf_counter(); o, _ = oracle.simulate(S, oracle.SimCfg(4, 4, 5, 4, 2, 5_000_000, 3), sm=0); do = time.perf_counter() - t
print(f"{S.n_instr} instrs, {n_sm} SMs x 16 warps: {n} samples in {dt*1e3:.1f} ms = {n/dt:.3e} samples/s; oracle 1 SM {len(o)} samples in {do*1e3:.1f} ms = {len(o)/do:.3e} samples/s")

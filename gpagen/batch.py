"""Config 4: a batch of profiled kernels (whole-application advisor pass), input generation only.

BASELINE.json configs[3]: 10^4 kernels, sizes log-uniform in [24, 2048] instructions (mean ~455,
~4.5 M instructions in all), 10^8 samples.  The shape per kernel follows ``random_program``
(one global function plus device functions, a nested loop forest, ~2 in-edges per
instruction with geometric def->use distances, loop-carried edges, barrier/WAR/predicate kinds,
rule-2 markers, lines of 1-6 instructions with reuse) but every step is vectorised over the whole
batch so the 4.5 M-instruction program builds in seconds.  Kernels get a lognormal share of the
samples (some kernels are hot, most are cold), and ``grouped_order`` arranges a stream by kernel
launch, the way a profiler delivers the samples of each launch in its own buffer.

Contains none of the blamer's arithmetic.
"""
from __future__ import annotations

import numpy as np

from .programs import (ARITH_FIXED, ARITH_LONG, BAR, CALLSITE, CONSTANT, CONTROL, CONVERT, GLOBAL,
                       IN_DEVICE_FN, IN_MATH, LOCAL, MISC, PRED, PROF_EXECCONS, PROF_LOAD, PROF_MEMCONS,
                       PROF_OTHER, PROF_SYNC, REG, SHARED, SYNC, TEXTURE, VARIABLE_LATENCY, WAR,
                       _LATENCY_RANGE, Program, _nested_loops, CONFIG_SEED_BASE)

_MIX = {ARITH_FIXED: .48, ARITH_LONG: .06, GLOBAL: .10, SHARED: .08, LOCAL: .03, CONSTANT: .03,
        CONVERT: .03, SYNC: .02, CONTROL: .08, MISC: .08, TEXTURE: .01}


def batch_program(n_kernels: int, seed: int, min_size: int = 24, max_size: int = 2048,
                  n_reasons: int = 9, kernel_sigma: float = 1.5, name: str = "batch") -> Program:
    rng = np.random.default_rng(seed)
    K = int(n_kernels)
    # ---- kernel sizes (log-uniform), functions per kernel, kernel-major layout
    sizes = np.exp(rng.uniform(np.log(min_size), np.log(max_size + 1), size=K)).astype(np.int64)
    sizes = np.clip(sizes, min_size, max_size)
    kbase = np.concatenate([[0], np.cumsum(sizes)])
    n = int(kbase[-1])
    nf_k = 1 + (sizes >= 256).astype(np.int64) + (sizes >= 1024).astype(np.int64)   # 1..3 functions
    func_begin = []
    for k in range(K):   # O(K) python: cut points at multiples of 8
        a, m = int(kbase[k]), int(sizes[k])
        if nf_k[k] == 1:
            func_begin.append(a)
        else:
            cuts = np.sort(rng.choice(np.arange(1, m // 8), size=nf_k[k] - 1, replace=False)) * 8
            func_begin.extend([a] + list(a + cuts))
    func_begin = np.array(func_begin + [n], np.int64)
    kernel_func_begin = np.concatenate([[0], np.cumsum(nf_k)]).astype(np.int64)
    n_funcs = len(func_begin) - 1
    func_of = np.repeat(np.arange(n_funcs), np.diff(func_begin))
    kernel_of = np.repeat(np.arange(K), sizes)
    fb_of = func_begin[func_of]
    is_global = np.zeros(n_funcs, bool)
    is_global[kernel_func_begin[:-1]] = True

    # ---- instruction classes, latencies, flags
    ks = np.array(list(_MIX.keys()))
    ps = np.array(list(_MIX.values()), np.float64)
    opclass = ks[rng.choice(len(ks), size=n, p=ps / ps.sum())].astype(np.uint8)
    latency = np.zeros(n, np.uint32)
    for c, (a, b) in _LATENCY_RANGE.items():
        m = opclass == c
        latency[m] = rng.integers(a, b + 1, size=int(m.sum()))
    iflags = np.zeros(n, np.uint8)
    dev_fn = ~is_global[func_of]
    iflags[dev_fn] |= IN_DEVICE_FN
    first_dev = np.zeros(n_funcs + 1, bool)          # first device function of each kernel
    first_dev[kernel_func_begin[:-1] + 1] = True
    first_dev = first_dev[:n_funcs] & ~is_global
    iflags[first_dev[func_of]] |= IN_MATH
    callsite = (~dev_fn) & (opclass == CONTROL) & (rng.random(n) < 0.3)
    iflags[callsite] |= CALLSITE

    # ---- loops: ~1 per 150 instructions, nested per function (python over functions)
    fsz = np.diff(func_begin)
    per_func = rng.poisson(fsz / 150.0)
    intervals = []
    for f in np.nonzero(per_func)[0]:
        intervals.extend(_nested_loops(rng, int(func_begin[f]), int(func_begin[f + 1]), int(per_func[f]), 4))
    intervals.sort(key=lambda t: (t[0], -(t[1] - t[0])))
    n_l = len(intervals)
    loop_parent = np.full(n_l, -1, np.int32)
    loop_id = np.full(n, -1, np.int32)
    depth = np.zeros(n, np.int32)
    stack = []
    for l, (a, b, d) in enumerate(intervals):
        while stack and not (intervals[stack[-1]][0] <= a and b <= intervals[stack[-1]][1]):
            stack.pop()
        loop_parent[l] = stack[-1] if stack else -1
        stack.append(l)
        loop_id[a:b] = l
        depth[a:b] += 1
    loop_a = np.array([t[0] for t in intervals], np.int64)
    loop_b = np.array([t[1] for t in intervals], np.int64)

    # ---- edges: up to 4 candidate slots per use j, vectorised
    k_choice = rng.choice(5, size=n, p=[.12, .30, .33, .15, .10])
    S = 4
    j = np.repeat(np.arange(n, dtype=np.int64), S)
    slot = np.tile(np.arange(S), n)
    live = slot < np.repeat(k_choice, S)
    j, slot = j[live], slot[live]
    m = len(j)
    lj = loop_id[j]
    carried = (lj >= 0) & (rng.random(m) < 0.12)
    la = np.where(lj >= 0, loop_a[np.maximum(lj, 0)], 0)
    lb = np.where(lj >= 0, loop_b[np.maximum(lj, 0)], 0)
    ic = j + (rng.random(m) * np.maximum(lb - j, 1)).astype(np.int64)           # i in [j, lb)
    mnc = (lb - ic) + (j - la)
    span = j - fb_of[j]
    d = np.maximum(rng.geometric(1.0 / 6.0, size=m), 1)
    d = np.minimum(d, np.maximum(span, 1))
    ifw = j - d
    i = np.where(carried, ic, ifw)
    mn = np.where(carried, mnc, d)
    ok = carried | (span >= 1)
    i, j, mn = i[ok], j[ok], mn[ok]
    # dedupe (j, i) keeping the first slot, then order by (j, i) = CSR by use
    key = j * n + i
    _, first = np.unique(key, return_index=True)
    i, j, mn = i[first], j[first], mn[first]
    E = len(i)
    extra = np.where(rng.random(E) < 0.6, 0, rng.geometric(0.25, size=E))
    mx = mn + extra
    var = np.isin(opclass[i], VARIABLE_LATENCY)
    u = rng.random(E)
    kind_var = np.where(u < 0.05, BAR, np.where(u < 0.09, WAR | BAR, np.where(u < 0.85, REG | BAR, REG)))
    kind_fix = np.where(rng.random(E) < 0.05, PRED, REG)
    kind = np.where(var, kind_var, kind_fix).astype(np.uint8)
    dom = np.full(E, -1, np.int64)
    dm = (i < j) & (j - i >= 2) & (rng.random(E) < 0.06)
    dom[dm] = i[dm] + 1 + (rng.random(int(dm.sum())) * (j[dm] - i[dm] - 1)).astype(np.int64)
    row_ptr = np.zeros(n + 1, np.uint32)
    np.add.at(row_ptr, j + 1, 1)
    row_ptr = np.cumsum(row_ptr).astype(np.uint32)

    # ---- lines: runs of 1..6 instructions inside a function; 15% of runs reuse an earlier line
    run = rng.integers(1, 7, size=n)
    starts = np.zeros(n, bool)
    pos = 0
    # run starts: walk by cumulative sums, restarted at every function start
    cs = np.cumsum(run)
    starts_idx = np.concatenate([[0], cs[:-1]])
    starts_idx = starts_idx[starts_idx < n]
    starts[starts_idx] = True
    starts[func_begin[:-1]] = True
    run_id = np.cumsum(starts) - 1                      # run index per instruction
    n_runs = int(run_id[-1]) + 1 if n else 0
    run_start = np.nonzero(starts)[0]
    run_func = func_of[run_start]
    reuse = rng.random(n_runs) < 0.15
    first_run_of_func = np.zeros(n_runs, bool)
    first_run_of_func[np.searchsorted(run_start, func_begin[:-1])] = True
    reuse &= ~first_run_of_func
    new_line = ~reuse
    line_of_run = np.cumsum(new_line) - 1                # fresh lines numbered in order
    # a reused run takes the line of a random earlier fresh run of its function
    fresh_runs = np.nonzero(new_line)[0]
    func_first_fresh = np.searchsorted(fresh_runs, np.searchsorted(run_start, func_begin[:-1]))
    for r in np.nonzero(reuse)[0]:                       # ~15% of runs, cheap python
        f = run_func[r]
        lo = func_first_fresh[f]
        hi = np.searchsorted(fresh_runs, r)              # fresh runs before r
        line_of_run[r] = line_of_run[fresh_runs[lo + int(rng.integers(hi - lo))]]
    line_id = line_of_run[run_id].astype(np.uint32)
    n_lines = int(new_line.sum())

    # ---- stream side: PC weights (kernel share x lognormal x depth) and reason profiles
    kw = np.exp(rng.normal(0.0, kernel_sigma, size=K)) / sizes    # per-kernel share, spread over its PCs
    w = kw[kernel_of] * np.exp(rng.normal(0.0, 0.75, size=n)) * 1.5 ** depth
    prof = np.full(n, PROF_OTHER, np.uint8)
    ci = opclass[i]
    exec_j = np.zeros(n, bool)
    exec_j[j[np.isin(ci, (SHARED, ARITH_LONG, CONVERT))]] = True
    prof[exec_j] = PROF_EXECCONS
    mem_j = np.zeros(n, bool)
    mem_j[j[np.isin(ci, (GLOBAL, LOCAL, CONSTANT, TEXTURE))]] = True
    prof[mem_j] = PROF_MEMCONS
    prof[np.isin(opclass, (GLOBAL, LOCAL, TEXTURE))] = PROF_LOAD
    prof[opclass == SYNC] = PROF_SYNC
    grid = rng.choice(np.array([8, 32, 80, 148, 296, 1024, 4096], np.uint32), size=K)

    return Program(
        n_reasons=n_reasons, opclass=opclass, iflags=iflags, latency=latency, line_id=line_id,
        loop_id=loop_id, loop_parent=loop_parent, func_begin=func_begin.astype(np.uint32),
        kernel_func_begin=kernel_func_begin.astype(np.uint32), kernel_grid_blocks=grid.astype(np.uint32),
        row_ptr=row_ptr, edge_def=i.astype(np.uint32), edge_kind=kind, edge_min_len=mn.astype(np.uint32),
        edge_max_len=mx.astype(np.uint32), edge_dom_k=dom.astype(np.int32), n_lines=n_lines,
        pc_weight=w, pc_profile=prof, name=name)


def config4_program(n_kernels: int = 10_000) -> Program:
    """BASELINE.json configs[3] (the batch); smaller n_kernels give the same recipe at test size."""
    return batch_program(n_kernels, CONFIG_SEED_BASE + 4)


def kernel_pc_begin(prog: Program) -> np.ndarray:
    """First instruction of every kernel (n_kernels + 1 entries)."""
    return prog.func_begin[prog.kernel_func_begin].astype(np.int64)


def grouped_order(pcs: np.ndarray, prog: Program, kernel_order=None):
    """Arrange a stream by kernel launch: a stable permutation of the records grouped by the
    kernel of their pc (kernels in ``kernel_order``, default 0..K-1; records whose pc is outside
    the program form a last group), plus the segment table (record offsets, kernel per segment)
    a profiler would hand over with the per-launch buffers.  numpy; ``torch`` tensors are
    accepted and handled on their device with the same stable order."""
    kb = kernel_pc_begin(prog)
    K = prog.n_kernels
    rank = np.arange(K + 1, dtype=np.int64)
    if kernel_order is not None:
        rank[np.asarray(kernel_order, np.int64)] = np.arange(K)
    try:
        import torch
        is_t = isinstance(pcs, torch.Tensor)
    except ImportError:
        is_t = False
    if is_t:
        kb_t = torch.as_tensor(kb[1:-1], device=pcs.device)
        kid = torch.bucketize(pcs.to(torch.int64), kb_t, right=True)
        kid = torch.where(pcs.to(torch.int64) >= int(kb[-1]), torch.full_like(kid, K), kid)
        key = torch.as_tensor(rank, device=pcs.device)[kid]
        order = torch.sort(key, stable=True).indices
        counts = torch.bincount(key, minlength=K + 1).cpu().numpy()
    else:
        p = np.asarray(pcs, np.int64)
        kid = np.searchsorted(kb[1:-1], p, side="right")
        kid = np.where(p >= kb[-1], K, kid)
        key = rank[kid]
        order = np.argsort(key, kind="stable")
        counts = np.bincount(key, minlength=K + 1)
    seg_kernel_all = np.empty(K + 1, np.int64)
    seg_kernel_all[rank[:K]] = np.arange(K)
    seg_kernel_all[K] = 0xFFFFFFFF       # out-of-program records: no kernel
    nz = np.nonzero(counts)[0]
    seg_begin = np.concatenate([[0], np.cumsum(counts[nz])]).astype(np.uint64)
    seg_kernel = seg_kernel_all[nz].astype(np.uint32)
    return order, seg_begin, seg_kernel


def record_pcs(records):
    """The pc field (low 32 bits) of 8-byte records (numpy uint64 or torch int64)."""
    try:
        import torch
        if isinstance(records, torch.Tensor):
            return records & 0xFFFFFFFF
    except ImportError:
        pass
    return (np.asarray(records, np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.int64)


def rebase_records(records: np.ndarray, pc_base: int) -> np.ndarray:
    """Records with pc - pc_base (a sub-program's view of an application stream)."""
    r = np.asarray(records, np.uint64)
    pc = (r & np.uint64(0xFFFFFFFF)) - np.uint64(pc_base)
    return (r & ~np.uint64(0xFFFFFFFF)) | (pc & np.uint64(0xFFFFFFFF))


def config4_stream(prog: Program) -> "StreamSpec":
    from .streams import STREAM_SEED_XOR, StreamSpec
    return StreamSpec(prog, (CONFIG_SEED_BASE + 4) ^ STREAM_SEED_XOR)

"""Seeded synthetic SASS-shaped programs (input generation only).

A ``Program`` is the static side of GPA's problem statement: the instruction table, the
def-use CSR with edge kinds and path lengths, and the line/loop/function/kernel maps that
GPA's static analyzer recovers from a CUBIN (§3).  The generator draws
them with the shapes DESIGN.md §5 gives for BASELINE.json's configs; it contains none of
the blamer's arithmetic.  ``tiny_fixture()`` is the hand-written config-1 program.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

# Encodings.  Stall reasons: 0 NONE, 1 MEM, 2 EXEC, 3 SYNC, 4 THROTTLE,
# 5 FETCH, 6 PIPE, 7 NOTSEL, 8 MISC.
GLOBAL, LOCAL, SHARED, CONSTANT, TEXTURE, ARITH_FIXED, ARITH_LONG, CONVERT, CONTROL, SYNC, MISC = range(11)
CLASS_NAMES = ["GLOBAL", "LOCAL", "SHARED", "CONSTANT", "TEXTURE", "ARITH_FIXED", "ARITH_LONG",
               "CONVERT", "CONTROL", "SYNC", "MISC"]
REG, PRED, BAR, WAR = 1, 2, 4, 8
IN_MATH, IN_DEVICE_FN, CALLSITE = 1, 2, 4
VARIABLE_LATENCY = (GLOBAL, LOCAL, SHARED, CONSTANT, TEXTURE)

# reason profiles: weights[(class, reason)] for the stream generator (index = class*9+reason)
PROF_OTHER, PROF_MEMCONS, PROF_EXECCONS, PROF_SYNC, PROF_LOAD = range(5)
_PROFILES = {
    #            ACT: NONE MEM EXEC SYNC THR FETCH PIPE NSEL MISC | LAT: NONE MEM EXEC SYNC THR FETCH PIPE NSEL MISC
    PROF_OTHER:    [40, 1, 4, 1, 1, 2, 3, 4, 1,     0, 2, 20, 1, 1, 4, 6, 10, 2],
    PROF_MEMCONS:  [25, 8, 2, 1, 1, 1, 1, 2, 1,     0, 45, 8, 1, 1, 2, 2, 4, 1],
    PROF_EXECCONS: [30, 1, 10, 1, 1, 1, 2, 3, 1,    0, 2, 35, 1, 1, 2, 4, 5, 1],
    PROF_SYNC:     [20, 1, 1, 5, 1, 1, 1, 2, 1,     0, 2, 2, 50, 1, 2, 2, 3, 1],
    PROF_LOAD:     [35, 5, 2, 1, 3, 1, 2, 3, 1,     0, 5, 3, 1, 25, 2, 3, 6, 1],
}

_LATENCY_RANGE = {
    GLOBAL: (1024, 1024), LOCAL: (1024, 1024), TEXTURE: (1024, 1024), CONSTANT: (64, 64),
    SHARED: (24, 32), ARITH_FIXED: (4, 6), ARITH_LONG: (16, 32), CONVERT: (16, 32),
    CONTROL: (8, 8), SYNC: (20, 20), MISC: (10, 10),
}


@dataclass
class Program:
    n_reasons: int
    opclass: np.ndarray
    iflags: np.ndarray
    latency: np.ndarray
    line_id: np.ndarray
    loop_id: np.ndarray
    loop_parent: np.ndarray
    func_begin: np.ndarray
    kernel_func_begin: np.ndarray
    kernel_grid_blocks: np.ndarray
    row_ptr: np.ndarray
    edge_def: np.ndarray
    edge_kind: np.ndarray
    edge_min_len: np.ndarray
    edge_max_len: np.ndarray
    edge_dom_k: np.ndarray
    n_lines: int
    pc_weight: np.ndarray = field(default=None)   # stream generator only
    pc_profile: np.ndarray = field(default=None)  # stream generator only
    name: str = ""

    @property
    def n_instr(self) -> int:
        return int(self.opclass.shape[0])

    @property
    def n_edges(self) -> int:
        return int(self.row_ptr[-1])

    @property
    def n_loops(self) -> int:
        return int(self.loop_parent.shape[0])

    @property
    def n_funcs(self) -> int:
        return int(self.func_begin.shape[0] - 1)

    @property
    def n_kernels(self) -> int:
        return int(self.kernel_func_begin.shape[0] - 1)

    def arrays(self) -> dict:
        return {k: getattr(self, k) for k in (
            "opclass", "iflags", "latency", "line_id", "loop_id", "loop_parent", "func_begin",
            "kernel_func_begin", "kernel_grid_blocks", "row_ptr", "edge_def", "edge_kind",
            "edge_min_len", "edge_max_len", "edge_dom_k")}


def _finalize(n_reasons, opclass, iflags, latency, line_id, loop_id, loop_parent, func_begin,
              kernel_func_begin, grid_blocks, rows, n_lines, pc_weight=None, pc_profile=None,
              name=""):
    """rows: list over uses of lists of (def, kind, min_len, max_len, dom_k)."""
    n = len(opclass)
    row_ptr = np.zeros(n + 1, dtype=np.uint32)
    flat = []
    for j in range(n):
        r = sorted(rows[j], key=lambda t: t[0])
        row_ptr[j + 1] = row_ptr[j] + len(r)
        flat.extend(r)
    E = len(flat)
    arr = np.array(flat, dtype=np.int64).reshape(E, 5) if E else np.zeros((0, 5), np.int64)
    return Program(
        n_reasons=n_reasons,
        opclass=np.asarray(opclass, np.uint8), iflags=np.asarray(iflags, np.uint8),
        latency=np.asarray(latency, np.uint32), line_id=np.asarray(line_id, np.uint32),
        loop_id=np.asarray(loop_id, np.int32), loop_parent=np.asarray(loop_parent, np.int32),
        func_begin=np.asarray(func_begin, np.uint32),
        kernel_func_begin=np.asarray(kernel_func_begin, np.uint32),
        kernel_grid_blocks=np.asarray(grid_blocks, np.uint32),
        row_ptr=row_ptr, edge_def=arr[:, 0].astype(np.uint32), edge_kind=arr[:, 1].astype(np.uint8),
        edge_min_len=arr[:, 2].astype(np.uint32), edge_max_len=arr[:, 3].astype(np.uint32),
        edge_dom_k=arr[:, 4].astype(np.int32), n_lines=int(n_lines),
        pc_weight=pc_weight, pc_profile=pc_profile, name=name)


# --------------------------------------------------------------------------- tiny fixture
def tiny_fixture() -> Program:
    """Config 1: 24 instructions, one loop (8..18), 13 def-use edges.

    The instruction list is the paper-style worked example of DESIGN.md §5.1: Fig. 4/5's
    @!P0 LDC / @P0 LDG / IMAD feeding an IADD, Fig. 3's barrier-only
    LDG -> BRA, Listing 1's F2F conversion, Listing 2's short
    load->use distance inside a loop with a __syncthreads, and a WAR edge.
    """
    cls = [MISC, ARITH_FIXED, ARITH_FIXED, CONSTANT, ARITH_FIXED, GLOBAL, ARITH_FIXED, ARITH_FIXED,
           GLOBAL, ARITH_FIXED, CONVERT, ARITH_FIXED, SHARED, SYNC, SHARED, ARITH_FIXED,
           ARITH_FIXED, ARITH_FIXED, CONTROL, GLOBAL, CONTROL, MISC, GLOBAL, CONTROL]
    lat = [_LATENCY_RANGE[c][0] for c in cls]
    lat[1] = 4; lat[2] = 4; lat[4] = 4; lat[6] = 4; lat[7] = 4; lat[9] = 4; lat[11] = 4
    lat[15] = 4; lat[16] = 4; lat[17] = 4; lat[10] = 16; lat[12] = 32; lat[14] = 32
    n = 24
    loop_id = [-1] * n
    for i in range(8, 19):
        loop_id[i] = 0
    rows = [[] for _ in range(n)]
    # (def, kind, min_len, max_len, dom_k)
    rows[7] = [(3, REG | BAR, 4, 4, -1), (5, REG | BAR, 2, 2, -1), (6, REG, 1, 1, -1)]
    rows[9] = [(8, REG | BAR, 1, 1, -1), (7, REG, 2, 2, -1), (15, REG, 5, 5, -1)]
    rows[11] = [(10, REG, 1, 1, -1), (9, REG, 2, 2, -1), (12, WAR | BAR, 10, 10, -1)]
    rows[15] = [(14, REG | BAR, 1, 1, -1), (11, REG, 4, 4, -1)]
    rows[20] = [(19, BAR, 1, 1, -1)]
    # rule 2: IMAD R2 -> @P0 LDG [R2]; the unpredicated MOV R3, R2 at 4 reads R2 on
    # the only path 1->5, so the edge carries dom_k = 4.  min_len 4 == latency(IMAD) 4 would
    # keep it under rule 3 (Q8 boundary).
    rows[5] = [(1, REG, 4, 4, 4)]
    iflags = [0] * n
    iflags[10] = IN_MATH
    line_id = [0, 0, 1, 2, 3, 4, 5, 5, 6, 7, 8, 8, 9, 10, 11, 12, 13, 13, 13, 14, 15, 16, 17, 18]
    return _finalize(9, cls, iflags, lat, line_id, loop_id, [-1], [0, n], [0, 1], [16], rows,
                     n_lines=19, name="tiny")


# --------------------------------------------------------------------------- random programs
def _nested_loops(rng, lo, hi, n_target, max_depth):
    """Random properly-nested loop intervals inside [lo, hi); returns list of (a, b, depth)."""
    loops = []
    # containers: (a, b, depth, children list)
    root = [lo, hi, 0, []]
    containers = [root]
    tries = 0
    while len(loops) < n_target and tries < n_target * 20:
        tries += 1
        c = containers[rng.integers(len(containers))]
        a0, b0, d0, kids = c
        if d0 >= max_depth or b0 - a0 < 6:
            continue
        length = int(rng.integers(4, max(5, (b0 - a0) * 3 // 4 + 1)))
        if length > b0 - a0:
            continue
        a = int(rng.integers(a0, b0 - length + 1))
        b = a + length
        if any(not (b <= ka or a >= kb) for ka, kb in kids):
            continue
        kids.append((a, b))
        node = [a, b, d0 + 1, []]
        containers.append(node)
        loops.append((a, b, d0 + 1))
    return loops


def random_program(n_instr: int, n_funcs: int, n_loops: int, max_depth: int, seed: int,
                   n_kernels: int = 1, n_reasons: int = 9, depth_bias: float = 4.0,
                   weight_sigma: float = 1.0, grid_blocks=None, class_mix=None,
                   name: str = "") -> Program:
    """A SASS-shaped random program: contiguous functions grouped into kernels,
    a properly nested loop forest per function, ~2 in-edges per instruction with geometric
    def->use distances, loop-carried edges, barrier/WAR/predicate kinds and rule-2 markers."""
    rng = np.random.default_rng(seed)
    n = n_instr
    if class_mix is None:
        class_mix = {ARITH_FIXED: .50, ARITH_LONG: .05, GLOBAL: .10, SHARED: .08, LOCAL: .02,
                     CONSTANT: .03, CONVERT: .03, SYNC: .02, CONTROL: .08, MISC: .08, TEXTURE: .01}
    ks = np.array(list(class_mix.keys()))
    ps = np.array(list(class_mix.values()), dtype=np.float64)
    opclass = ks[rng.choice(len(ks), size=n, p=ps / ps.sum())].astype(np.uint8)
    latency = np.zeros(n, np.uint32)
    for c, (a, b) in _LATENCY_RANGE.items():
        m = opclass == c
        latency[m] = rng.integers(a, b + 1, size=int(m.sum()))

    # functions: contiguous ranges, at least 8 instructions each
    cuts = np.sort(rng.choice(np.arange(1, n // 8), size=n_funcs - 1, replace=False)) * 8 if n_funcs > 1 else np.array([], np.int64)
    func_begin = np.concatenate([[0], cuts, [n]]).astype(np.int64)
    # kernels: contiguous ranges of functions
    if n_kernels > 1:
        kc = np.sort(rng.choice(np.arange(1, n_funcs), size=n_kernels - 1, replace=False))
        kernel_func_begin = np.concatenate([[0], kc, [n_funcs]]).astype(np.int64)
    else:
        kernel_func_begin = np.array([0, n_funcs], np.int64)
    func_kernel = np.searchsorted(kernel_func_begin, np.arange(n_funcs), side="right") - 1
    is_global = np.zeros(n_funcs, bool)
    is_global[kernel_func_begin[:-1]] = True

    iflags = np.zeros(n, np.uint8)
    for f in range(n_funcs):
        a, b = func_begin[f], func_begin[f + 1]
        if not is_global[f]:
            iflags[a:b] |= IN_DEVICE_FN
            if f == kernel_func_begin[func_kernel[f]] + 1:   # first device fn of a kernel: a math routine
                iflags[a:b] |= IN_MATH
        else:
            ctl = np.nonzero(opclass[a:b] == CONTROL)[0] + a
            iflags[ctl[rng.random(len(ctl)) < 0.3]] |= CALLSITE

    # loops, numbered in preorder (parents before children)
    sizes = np.diff(func_begin).astype(np.float64)
    per_func = np.floor(n_loops * sizes / sizes.sum()).astype(int)
    per_func[np.argsort(-sizes)[: n_loops - per_func.sum()]] += 1
    intervals = []
    for f in range(n_funcs):
        for (a, b, d) in _nested_loops(rng, int(func_begin[f]), int(func_begin[f + 1]), int(per_func[f]), max_depth):
            intervals.append((a, b, d))
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

    # edges
    func_of = np.searchsorted(func_begin, np.arange(n), side="right") - 1
    k_choice = rng.choice(5, size=n, p=[.12, .30, .33, .15, .10])
    rows = [[] for _ in range(n)]
    var_lat = np.isin(opclass, VARIABLE_LATENCY)
    for j in range(n):
        fb = int(func_begin[func_of[j]])
        seen = set()
        for _ in range(int(k_choice[j])):
            lj = int(loop_id[j])
            if lj >= 0 and rng.random() < 0.12:
                la, lb = intervals[lj][0], intervals[lj][1]
                i = int(rng.integers(j, lb))
                mn = (lb - i) + (j - la)
            else:
                if j - fb < 1:
                    continue
                d = min(1 + int(rng.geometric(1.0 / 6.0)) - 1, j - fb)
                d = max(d, 1)
                i = j - d
                mn = d
            if i in seen:
                continue
            seen.add(i)
            extra = 0 if rng.random() < 0.6 else int(rng.geometric(0.25))
            mx = mn + extra
            if var_lat[i]:
                u = rng.random()
                kind = BAR if u < 0.05 else (WAR | BAR if u < 0.09 else REG | BAR if u < 0.85 else REG)
            else:
                kind = PRED if rng.random() < 0.05 else REG
            dom = -1
            if i < j and j - i >= 2 and rng.random() < 0.06:
                dom = int(rng.integers(i + 1, j))
            rows[j].append((i, kind, mn, mx, dom))

    # lines: runs of 1..6 instructions; 15% of runs reuse an earlier line of the same function
    line_id = np.zeros(n, np.int64)
    next_line = 0
    f_lines = {}
    i = 0
    while i < n:
        run = int(rng.integers(1, 7))
        f = int(func_of[i])
        run = min(run, int(func_begin[f + 1]) - i)
        prev = f_lines.setdefault(f, [])
        if prev and rng.random() < 0.15:
            lid = prev[int(rng.integers(len(prev)))]
        else:
            lid = next_line
            next_line += 1
            prev.append(lid)
        line_id[i:i + run] = lid
        i += run

    # stream-side: PC weights and reason profiles
    w = np.exp(rng.normal(0.0, weight_sigma, size=n)) * depth_bias ** depth
    prof = np.full(n, PROF_OTHER, np.uint8)
    for j in range(n):
        for (i, kind, *_rest) in rows[j]:
            c = opclass[i]
            if c in (GLOBAL, LOCAL, CONSTANT, TEXTURE):
                prof[j] = PROF_MEMCONS
            elif prof[j] == PROF_OTHER and c in (SHARED, ARITH_LONG, CONVERT):
                prof[j] = PROF_EXECCONS
    prof[np.isin(opclass, (GLOBAL, LOCAL, TEXTURE))] = PROF_LOAD
    prof[opclass == SYNC] = PROF_SYNC
    if grid_blocks is None:
        grid_blocks = np.full(len(kernel_func_begin) - 1, 16, np.uint32)
    return _finalize(n_reasons, opclass, iflags, latency, line_id, loop_id, loop_parent, func_begin,
                     kernel_func_begin, grid_blocks, rows, next_line, pc_weight=w, pc_profile=prof,
                     name=name)


CONFIG_SEED_BASE = 0x2009040610


def config_program(cfg: int) -> Program:
    """Programs of BASELINE.json configs 1-4 (config 5 reuses config 3's program); 6 = a 200k-instruction
    PeleC-scale kernel (bench --workload pelec)."""
    seed = CONFIG_SEED_BASE + cfg
    if cfg == 1:
        return tiny_fixture()
    if cfg == 2:
        return random_program(2000, 4, 8, 3, seed, depth_bias=4.0, weight_sigma=1.0, name="rodinia")
    if cfg in (3, 5):
        mix = {ARITH_FIXED: .46, ARITH_LONG: .07, GLOBAL: .10, SHARED: .07, LOCAL: .04,
               CONSTANT: .03, CONVERT: .03, SYNC: .02, CONTROL: .08, MISC: .09, TEXTURE: .01}
        return random_program(50000, 64, 200, 6, CONFIG_SEED_BASE + 3, depth_bias=1.5,
                              weight_sigma=0.75, class_mix=mix, name="large")
    if cfg == 4:
        from .batch import config4_program
        return config4_program()
    if cfg == 6:   # not a BASELINE config: a PeleC-scale kernel, 15-bit local ingest bins
        mix = {ARITH_FIXED: .46, ARITH_LONG: .07, GLOBAL: .10, SHARED: .07, LOCAL: .04,
               CONSTANT: .03, CONVERT: .03, SYNC: .02, CONTROL: .08, MISC: .09, TEXTURE: .01}
        return random_program(200000, 128, 600, 6, CONFIG_SEED_BASE + 6, depth_bias=1.5,
                              weight_sigma=0.75, class_mix=mix, name="pelec")
    raise ValueError(f"no program for config {cfg}")


# Config-1 sample counts: (pc, class, reason) -> samples; 500 samples over six
# stall reasons, chosen so every Eq. 1 share is dyadic (exact in fp64).
TINY_COUNTS = {
    (0, 0, 0): 10, (1, 0, 0): 10, (2, 0, 0): 10, (3, 0, 0): 40, (4, 0, 0): 10,
    (5, 0, 0): 20, (5, 1, 1): 4, (5, 1, 2): 2,
    (6, 0, 0): 20,
    (7, 0, 0): 40, (7, 0, 1): 4, (7, 0, 2): 4, (7, 1, 1): 12, (7, 1, 2): 4,
    (8, 0, 0): 8, (8, 1, 4): 10,
    (9, 0, 0): 4, (9, 1, 1): 24, (9, 1, 2): 8,
    (10, 0, 0): 2,
    (11, 0, 0): 16, (11, 1, 1): 6, (11, 1, 2): 16,
    (12, 0, 0): 40,
    (13, 0, 3): 2, (13, 0, 0): 6, (13, 1, 3): 30,
    (14, 0, 0): 12,
    (15, 0, 0): 10, (15, 1, 2): 16,
    (16, 0, 0): 6, (16, 0, 7): 4, (16, 1, 7): 4,
    (17, 0, 0): 10,
    (18, 0, 0): 10, (18, 1, 5): 8,
    (19, 0, 0): 10, (19, 1, 4): 6,
    (20, 0, 0): 4, (20, 1, 1): 20,
    (22, 0, 0): 10,
    (23, 0, 0): 8,
}


def tiny_records(seed: int = CONFIG_SEED_BASE + 1) -> np.ndarray:
    """The 500 config-1 samples as count-1 records (uint64 view), in a seeded order."""
    recs = []
    for (pc, c, r), k in sorted(TINY_COUNTS.items()):
        recs += [pc | (1 << 32) | (r << 48) | (c << 56)] * k
    arr = np.array(recs, dtype=np.uint64)
    return arr[np.random.default_rng(seed).permutation(len(arr))]

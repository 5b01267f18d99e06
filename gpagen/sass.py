"""SASS-level program descriptions for backward slicing, input generation only.

Fields per instruction (Table 1): guard predicate, destination and source
operands (R0-R254, P0-P6), write / read barrier and wait masks over B0-B5; plus the control flow
graph (basic blocks, successors) per function.  ``slice_fixture()`` is the hand-made example of
DESIGN.md §5.3 whose def-use graph is derived by hand in tests/test_oracle_slicing.py;
``random_sass`` draws larger programs (straight code, if/else diamonds, loops, predicated defs,
variable-latency instructions with barriers).  Holds none of the slicing arithmetic.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NONE = 0xFFFF
RZ = 255
ALWAYS = 7           # guard: no predicate ('_')
NEG = 8              # guard bit: !P


def P(i: int) -> int:
    return 256 + i


@dataclass
class Sass:
    func_begin: np.ndarray
    block_begin: np.ndarray
    succ_ptr: np.ndarray
    succ: np.ndarray
    guard: np.ndarray
    dst: np.ndarray       # [n, 4] u16
    src: np.ndarray       # [n, 4] u16
    wbar: np.ndarray
    rbar: np.ndarray
    wait: np.ndarray
    opclass: np.ndarray = field(default=None)
    latency: np.ndarray = field(default=None)

    @property
    def n_instr(self) -> int:
        return int(self.guard.shape[0])


def _build(instrs, blocks, succs, funcs=None):
    """instrs: list of dicts (guard, dst, src, wbar, rbar, wait, cls, lat); blocks: list of
    (begin, end); succs: list of successor-block lists."""
    n = len(instrs)
    dst = np.full((n, 4), NONE, np.uint16)
    src = np.full((n, 4), NONE, np.uint16)
    for i, ins in enumerate(instrs):
        for t, r in enumerate(ins.get("dst", ())):
            dst[i, t] = r
        for t, r in enumerate(ins.get("src", ())):
            src[i, t] = r
    bb = np.array([b for b, _ in blocks] + [blocks[-1][1]], np.uint32)
    sp = np.zeros(len(blocks) + 1, np.uint32)
    flat = []
    for b, ss in enumerate(succs):
        flat.extend(ss)
        sp[b + 1] = len(flat)
    return Sass(np.array(funcs or [0, n], np.uint32), bb, sp, np.array(flat, np.uint32),
                np.array([ins.get("guard", ALWAYS) for ins in instrs], np.uint8), dst, src,
                np.array([ins.get("wbar", 0) for ins in instrs], np.uint8),
                np.array([ins.get("rbar", 0) for ins in instrs], np.uint8),
                np.array([ins.get("wait", 0) for ins in instrs], np.uint8),
                np.array([ins.get("cls", 5) for ins in instrs], np.uint8),
                np.array([ins.get("lat", 4) for ins in instrs], np.uint32))


def slice_fixture() -> Sass:
    """16 instructions, blocks A [0,7) -> {B, C}, B [7,9) -> D, C [9,10) -> D, D [10,14) -> {D, E}
    (a loop), E [14,16): Fig. 5's @!P0 LDC / @P0 LDG feeding an unpredicated IADD (predicate
    coverage), the rule-2 MOV between IMAD and @P0 LDG, an if/else whose arms
    define the same register, a loop with a loop-carried FFMA -> FADD dependency, a shared load
    whose read barrier makes a later write a WAR dependency, and Fig. 3's barrier-only LDG
    -> BRA."""
    GL, CO, SH, AR, CT = 0, 3, 2, 5, 8
    I = [
        dict(dst=[10], cls=10),                                        # 0  S2R R10
        dict(dst=[P(1)], src=[10]),                                    # 1  ISETP P1, R10
        dict(dst=[2], src=[10]),                                       # 2  IMAD R2, R10
        dict(guard=NEG | 0, dst=[0], src=[2], wbar=1 << 0, cls=CO, lat=64),   # 3  @!P0 LDC R0, c[R2]   (B0)
        dict(dst=[3], src=[2]),                                        # 4  MOV R3, R2
        dict(guard=0, dst=[0], src=[2], wbar=1 << 1, cls=GL, lat=1024),       # 5  @P0 LDG R0, [R2]    (B1)
        dict(guard=1, cls=CT, lat=8),                                  # 6  @P1 BRA C
        dict(dst=[4], src=[0], wait=(1 << 0) | (1 << 1)),              # 7  IADD R4, R0   (waits B0 B1)
        dict(dst=[4], src=[4, 3]),                                     # 8  IADD R4, R4, R3
        dict(dst=[4], src=[3]),                                        # 9  IADD R4, R3
        dict(dst=[5], src=[4, 6]),                                     # 10 FADD R5, R4, R6
        dict(dst=[7], src=[5], wbar=1 << 2, rbar=1 << 3, cls=SH, lat=32),     # 11 LDS R7, [R5] (B2 / read B3)
        dict(dst=[6], src=[7, 5], wait=1 << 2),                        # 12 FFMA R6, R7, R5 (waits B2)
        dict(dst=[5], src=[6], wait=1 << 3),                           # 13 MOV R5, R6 (waits B3: WAR)
        dict(dst=[8], src=[6], wbar=1 << 4, cls=GL, lat=1024),         # 14 LDG R8, [R6] (B4)
        dict(wait=1 << 4, cls=CT, lat=8),                              # 15 BRA (waits B4)
    ]
    blocks = [(0, 7), (7, 9), (9, 10), (10, 14), (14, 16)]
    succs = [[1, 2], [3], [3], [3, 4], []]
    return _build(I, blocks, succs)


def random_sass(n_funcs: int, seed: int, func_len=(24, 160), n_regs: int = 24) -> Sass:
    """Random functions built from regions: straight code, if/else diamonds and loops (back edge),
    with predicated instructions (ISETP-defined predicates), variable-latency loads that set write
    (and sometimes read) barriers waited on by later instructions."""
    rng = np.random.default_rng(seed)
    instrs, blocks, succs, funcs = [], [], [], [0]

    def new_block():
        blocks.append([len(instrs), None])
        succs.append([])
        return len(blocks) - 1

    def emit():
        g = ALWAYS
        if rng.random() < 0.15:
            g = int(rng.integers(0, 3)) | (NEG if rng.random() < 0.5 else 0)
        kind = rng.random()
        ins = dict(guard=g)
        if kind < 0.1:                                      # ISETP
            ins.update(dst=[P(int(rng.integers(0, 3)))], src=[int(rng.integers(0, n_regs))])
        elif kind < 0.3:                                    # variable-latency load
            b = int(rng.integers(0, 6))
            ins.update(dst=[int(rng.integers(0, n_regs))], src=[int(rng.integers(0, n_regs))], wbar=1 << b,
                       cls=int(rng.choice([0, 2, 3])), lat=1024)
            if rng.random() < 0.3:
                ins["rbar"] = 1 << int((b + 1) % 6)
        else:                                               # arithmetic
            ns = int(rng.integers(0, 4))
            ins.update(dst=[int(rng.integers(0, n_regs))], src=[int(x) for x in rng.integers(0, n_regs, ns)])
            if rng.random() < 0.05:
                ins["src"] = ins["src"] + [P(int(rng.integers(0, 3)))]
        if rng.random() < 0.25:
            ins["wait"] = int(rng.integers(1, 64))
        if rng.random() < 0.03:
            ins["dst"] = ins.get("dst", []) + [RZ]
        instrs.append(ins)

    def straight(k):
        for _ in range(k):
            emit()

    for f in range(n_funcs):
        target = int(rng.integers(*func_len))
        b = new_block()
        straight(int(rng.integers(2, 6)))
        while len(instrs) - funcs[-1] < target:
            r = rng.random()
            if r < 0.35:                                    # if/else diamond
                blocks[b][1] = len(instrs)
                t = new_block(); straight(int(rng.integers(1, 8))); blocks[t][1] = len(instrs)
                e = new_block(); straight(int(rng.integers(1, 5))); blocks[e][1] = len(instrs)
                j = new_block()
                succs[b] += [t, e]; succs[t] += [j]; succs[e] += [j]
                straight(int(rng.integers(1, 4)))
                b = j
            elif r < 0.6:                                   # loop (single block with a back edge)
                blocks[b][1] = len(instrs)
                lp = new_block(); straight(int(rng.integers(3, 12))); blocks[lp][1] = len(instrs)
                nx = new_block()
                succs[b] += [lp]; succs[lp] += [lp, nx]
                straight(int(rng.integers(1, 4)))
                b = nx
            else:
                straight(int(rng.integers(2, 10)))
        blocks[b][1] = len(instrs)
        funcs.append(len(instrs))
    return _build(instrs, [tuple(x) for x in blocks], succs, funcs)


def single_source_sass(n: int, seed: int) -> Sass:
    """Straight-line function where every instruction reads exactly one register, produced by one
    of the previous 5 instructions (so each stall has a single true source): loads (GLOBAL, 400
    cycles, a write barrier its consumers wait on), long (20-cycle) and short (4-6-cycle) arithmetic."""
    rng = np.random.default_rng(seed)
    instrs, n_loads = [], 0
    for i in range(n):
        ins = dict(dst=[i % 250])
        if i > 0:
            p = i - int(rng.integers(1, min(5, i) + 1))
            ins["src"] = [p % 250]
            if instrs[p].get("wbar"):
                ins["wait"] = instrs[p]["wbar"]
        u = rng.random()
        if u < 0.25:
            ins.update(wbar=1 << (n_loads % 6), cls=0, lat=400)
            n_loads += 1
        elif u < 0.4:
            ins.update(cls=6, lat=20)
        else:
            ins.update(cls=5, lat=int(rng.integers(4, 7)))
        instrs.append(ins)
    return _build(instrs, [(0, n)], [[]])


def program_from_sass(S: Sass, csr: dict, n_reasons: int = 9):
    """A gpa Program (gpagen.programs.Program) for a sliced SASS program: lines = instructions,
    one loop per self-loop block, the functions of S, one kernel."""
    from .programs import _finalize
    n = S.n_instr
    loop_id = np.full(n, -1, np.int32)
    n_loops = 0
    for b in range(len(S.block_begin) - 1):
        if b in set(int(x) for x in S.succ[S.succ_ptr[b]:S.succ_ptr[b + 1]]):
            loop_id[S.block_begin[b]:S.block_begin[b + 1]] = n_loops
            n_loops += 1
    rows = [[] for _ in range(n)]
    rp = csr["row_ptr"]
    for j in range(n):
        for e in range(rp[j], rp[j + 1]):
            rows[j].append((int(csr["edge_def"][e]), int(csr["edge_kind"][e]), int(csr["edge_min_len"][e]),
                            int(csr["edge_max_len"][e]), int(csr["edge_dom_k"][e])))
    prog = _finalize(n_reasons, S.opclass, np.zeros(n, np.uint8), S.latency, np.arange(n), loop_id,
                     [-1] * n_loops, S.func_begin, [0, len(S.func_begin) - 1], [16], rows, n_lines=n)
    prog.pc_weight = np.ones(n)
    prog.pc_profile = np.zeros(n, np.uint8)
    return prog


def random_cfg_sass(seed: int, max_instr: int = 24, n_regs: int = 5, n_funcs: int = 1) -> Sass:
    """Small functions (<= max_instr instructions each) with structured but irregular control flow,
    for the brute-force slicing checks: nested loops, multi-block loop bodies, loops with several
    back edges (`continue`: a body block branching back to the header), multi-exit loops (`break`:
    a body block branching to the loop's exit), if/else diamonds and one-armed ifs.  Few registers,
    so def-use chains cross loops and arms; predicated defs (3 predicates) and barriers as in
    random_sass.  Blocks are laid out in address order, a loop's header first.  Functions are
    drawn one by one; a draw longer than max_instr, or without a back edge when loops are wanted
    (about 3 in 4 draws), is redrawn from the next sub-seed."""
    if n_funcs > 1:
        return concat_sass([random_cfg_sass(int(np.random.default_rng([seed, f]).integers(1 << 62)), max_instr, n_regs)
                            for f in range(n_funcs)])
    for attempt in range(1000):
        S = _cfg_draw(np.random.default_rng([seed, attempt]), max_instr, n_regs, 1)
        has_back = any(S.block_begin[t] <= S.block_begin[b + 1] - 1 for b in range(len(S.block_begin) - 1)
                       for t in S.succ[S.succ_ptr[b]:S.succ_ptr[b + 1]])
        if S.n_instr <= max_instr and (has_back or np.random.default_rng([seed, attempt, 1]).random() < 0.25):
            return S
    raise RuntimeError("random_cfg_sass: no draw fits")


def concat_sass(parts) -> Sass:
    """Functions of several Sass descriptions laid out one after another (ids renumbered)."""
    fb, bb, sp, su = [0], [0], [0], []
    arr = {k: [] for k in ("guard", "dst", "src", "wbar", "rbar", "wait", "opclass", "latency")}
    i0 = b0 = 0
    for S in parts:
        fb += [int(x) + i0 for x in S.func_begin[1:]]
        bb += [int(x) + i0 for x in S.block_begin[1:]]
        su += [int(x) + b0 for x in S.succ]
        sp += [int(x) + sp[-1] for x in S.succ_ptr[1:]]
        for k in arr:
            arr[k].append(getattr(S, k))
        i0 += S.n_instr
        b0 += len(S.block_begin) - 1
    return Sass(np.array(fb, np.uint32), np.array(bb, np.uint32), np.array(sp, np.uint32), np.array(su, np.uint32),
                *[np.concatenate(arr[k]) for k in ("guard", "dst", "src", "wbar", "rbar", "wait", "opclass", "latency")])


def _cfg_draw(rng, max_instr, n_regs, n_funcs):
    instrs, blocks, succs, funcs = [], [], [], [0]

    def new_block():
        blocks.append([len(instrs), None])
        succs.append([])
        return len(blocks) - 1

    def emit():
        g = ALWAYS
        if rng.random() < 0.2:
            g = int(rng.integers(0, 3)) | (NEG if rng.random() < 0.5 else 0)
        u = rng.random()
        ins = dict(guard=g)
        if u < 0.12:                                        # ISETP
            ins.update(dst=[P(int(rng.integers(0, 3)))], src=[int(rng.integers(0, n_regs))])
        elif u < 0.3:                                       # variable-latency load with barriers
            b = int(rng.integers(0, 3))
            ins.update(dst=[int(rng.integers(0, n_regs))], src=[int(rng.integers(0, n_regs))], wbar=1 << b,
                       cls=int(rng.choice([0, 2, 3])), lat=1024)
            if rng.random() < 0.4:
                ins["rbar"] = 1 << int((b + 1) % 3)
        elif u < 0.4:                                       # a pure reader (store-like)
            ins.update(src=[int(x) for x in rng.integers(0, n_regs, int(rng.integers(1, 3)))])
        else:                                               # arithmetic
            ins.update(dst=[int(rng.integers(0, n_regs))],
                       src=[int(x) for x in rng.integers(0, n_regs, int(rng.integers(0, 3)))])
        if rng.random() < 0.25:
            ins["wait"] = int(rng.integers(1, 8))
        instrs.append(ins)

    def close(b, targets):
        blocks[b][1] = len(instrs)
        succs[b].extend(targets)

    def room(f0):
        return max_instr - (len(instrs) - f0)

    def region(cur, depth, f0, loop):
        """Emit a region starting in open block `cur`; returns the open block it ends in.  `loop`:
        (header block, list collecting break sources) of the innermost enclosing loop, or None."""
        for _ in range(int(rng.integers(1, 4))):
            left = room(f0)
            if left <= 2:
                break
            r = rng.random()
            if r < 0.4 and left >= 6 and depth < 3:        # loop: header, body region, latch
                emit(); close(cur, [len(blocks)])
                h = new_block(); emit()
                breaks = []
                body = region(h, depth + 1, f0, (h, breaks))
                emit()                                      # latch: back edge + exit
                latch = body
                ex_id = len(blocks)
                close(latch, [h, ex_id])
                for b in breaks:
                    succs[b].append(ex_id)
                cur = new_block(); emit()
            elif r < 0.6 and left >= 5:                    # if/else diamond (or one-armed if)
                emit()
                one_arm = rng.random() < 0.3
                t = len(blocks)
                close(cur, [t])
                tb = new_block(); emit()
                tend = region(tb, depth + 1, f0, loop) if rng.random() < 0.4 else tb
                if one_arm:
                    j = len(blocks)
                    close(tend, [j])
                    succs[cur].append(j)
                else:
                    e = len(blocks)
                    succs[cur].append(e)
                    eb_pending = tend
                    close(tend, [])
                    eb = new_block(); emit()
                    j = len(blocks)
                    close(eb, [j])
                    succs[eb_pending].append(j)
                cur = new_block(); emit()
            elif r < 0.8 and loop is not None and left >= 3:   # continue / break out of the body
                emit()
                nxt = len(blocks)
                if rng.random() < 0.5:
                    close(cur, [nxt, loop[0]])             # continue: a second back edge to the header
                else:
                    close(cur, [nxt])
                    loop[1].append(cur)                    # break: edge to the loop exit (patched)
                cur = new_block(); emit()
            else:
                for _ in range(int(rng.integers(1, 4))):
                    if room(f0) > 1:
                        emit()
        return cur

    for _ in range(n_funcs):
        f0 = len(instrs)
        b = new_block()
        emit()
        if rng.random() < 0.2:                              # the entry block heads a loop
            breaks = []
            body = region(b, 1, f0, (b, breaks))
            emit()
            ex_id = len(blocks)
            close(body, [b, ex_id])
            for bb in breaks:
                succs[bb].append(ex_id)
            b = new_block(); emit()
        end = region(b, 0, f0, None)
        if len(instrs) == blocks[end][0]:
            emit()
        close(end, [])
        funcs.append(len(instrs))
    return _build(instrs, [tuple(x) for x in blocks], succs, funcs)

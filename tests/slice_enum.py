"""Brute-force path enumeration for backward slicing (test infrastructure; shares nothing with
oracle/ or the CUDA slicer).  VERDICT r01 "pin the slicer to a definition": this module states the
slicer's outputs as definitions over the set of backward paths and evaluates them by listing the
paths one by one, which is only feasible on tiny CFGs (<= 24 instructions).

Definitions (DESIGN.md §3.2 Q35-Q38):

* reads(j): source operands (R0-R254, P0-P6; RZ ignored; kind REG / PRED), the guard predicate
  register (PRED), the virtual barrier registers B_b of the wait mask (BAR).  x defines a general
  or predicate register when it is a destination of x, and B_b when b is x's write or read barrier
  (P:301-302).
* A backward path of j for register r is x_1, ..., x_m with x_1 in prev(j), x_{t+1} in prev(x_t):
  prev(x) = x - 1 inside a block, else the last instruction of every predecessor block (same
  function).  P_0 = {} and, when x_t defines r, P_t = P_{t-1} + pred(x_t) (with {p, !p} = '_'); the
  path may not continue past an x_t that defines r with P_t containing j's predicate.
  Every x_t that defines r is a def-state of x_t at length t (i exclusive, j inclusive: S:172).
* A step from x (first instruction of its block) to the last instruction y of a predecessor block
  crosses a back edge iff y >= x (the branch goes to the same or a lower address).
* min_len(i, j) = the fewest steps over all paths reaching a def-state of i (any register j reads
  that i defines).  K*(i, j) = the fewest back-edge crossings over those paths;
  max_len(i, j) = the most steps over the paths with exactly K* crossings ("the longest one",
  P:380, on the unrolled-once convention of S:185 / SURVEY Q9: back edges only as often as the
  pair needs them).
* dom_k(i, j) = the smallest k not in {i, j}, with no guard predicate, that reads every register r
  linking i to j and lies on every path of every such r that reaches a def-state of i (rule 2,
  P:367); -1 if there is none.
* kind = OR over the linking registers of REG / PRED / BAR, plus WAR when a linking barrier is i's
  read barrier and j writes a register i reads.

Paths are enumerated with at most B crossings in total, B = the number of back edges of the
function: a path reaching i with a repeated instruction can be cut at the repeat into a valid path
that still reaches i, is shorter, crosses no more back edges, avoids every instruction the longer
one avoided, and (being simple) crosses each back edge at most once -- so minima, K* and the
rule-2 "every path" condition are all decided by the paths with <= B crossings, and every path with
K* <= B crossings is listed for the maximum.
"""
from __future__ import annotations

NONE, RZ, ALWAYS = 0xFFFF, 255, 7
REG, PRED, BAR, WAR = 1, 2, 4, 8
P_ALL = 1 << 14


def _pset_bit(guard: int) -> int:
    g = guard & 7
    if g == 7:
        return P_ALL
    return 1 << (7 + g) if guard & 8 else 1 << g


def _union(P: int, b: int) -> int:
    P |= b
    for i in range(7):
        if P >> i & 1 and P >> (7 + i) & 1:
            P |= P_ALL
    return P


def _contains(P: int, b: int) -> bool:
    return bool(P & P_ALL) or bool(P & b)


def reads(S, x: int):
    out = []
    for t in range(4):
        r = int(S.src[x][t])
        if r != NONE and r != RZ:
            out.append((r, PRED if r >= 256 else REG))
    if int(S.guard[x]) & 7 != 7:
        out.append((256 + (int(S.guard[x]) & 7), PRED))
    for b in range(6):
        if int(S.wait[x]) >> b & 1:
            out.append((512 + b, BAR))
    return out


def defines(S, x: int, r: int) -> bool:
    if r >= 512:
        return bool((int(S.wbar[x]) | int(S.rbar[x])) >> (r - 512) & 1)
    return any(int(S.dst[x][t]) == r for t in range(4))


class _Cfg:
    def __init__(self, S):
        bb = [int(v) for v in S.block_begin]
        self.nb = len(bb) - 1
        self.block_of = {}
        for b in range(self.nb):
            for x in range(bb[b], bb[b + 1]):
                self.block_of[x] = b
        self.bb = bb
        self.preds = [[] for _ in range(self.nb)]
        for b in range(self.nb):
            for t in S.succ[int(S.succ_ptr[b]):int(S.succ_ptr[b + 1])]:
                self.preds[int(t)].append(b)
        fb = [int(v) for v in S.func_begin]
        self.func_of_block = []
        for b in range(self.nb):
            self.func_of_block.append(max(f for f in range(len(fb) - 1) if fb[f] <= bb[b]))
        self.back_edges = [0] * (len(fb) - 1)
        for b in range(self.nb):
            for t in S.succ[int(S.succ_ptr[b]):int(S.succ_ptr[b + 1])]:
                if bb[int(t)] <= bb[b + 1] - 1:
                    self.back_edges[self.func_of_block[b]] += 1

    def prev(self, x: int):
        b = self.block_of[x]
        if x > self.bb[b]:
            return [x - 1]
        return [self.bb[p + 1] - 1 for p in sorted(set(self.preds[b]))]


def paths_to_defs(S, cfg: _Cfg, j: int, r: int, max_cross: int | None = None, simple: bool = False):
    """Every def-state reached by the backward paths of j for register r: list of (def x, length,
    crossings, frozenset of the instructions strictly between).  `max_cross` bounds the back-edge
    crossings (default B, the function's back-edge count); `simple` keeps only paths whose
    instructions are pairwise distinct."""
    pj = _pset_bit(int(S.guard[j]))
    B = cfg.back_edges[cfg.func_of_block[cfg.block_of[j]]] if max_cross is None else max_cross
    found = []
    on_path = set()

    def walk(x, P, length, k, between):
        if simple:
            if x in on_path:
                return
            on_path.add(x)
        if defines(S, x, r):
            found.append((x, length, k, frozenset(between)))
            P = _union(P, _pset_bit(int(S.guard[x])))
            if _contains(P, pj):
                if simple:
                    on_path.discard(x)
                return
        between.append(x)
        for y in cfg.prev(x):
            k2 = k + (1 if y >= x else 0)
            if k2 <= B:
                walk(y, P, length + 1, k2, between)
        between.pop()
        if simple:
            on_path.discard(x)

    for y in cfg.prev(j):
        k0 = 1 if y >= j else 0
        if k0 <= B:
            walk(y, 0, 1, k0, [])
    return found


def slice_use(S, j: int, cfg: _Cfg | None = None, reduced: bool = True):
    """{def i: (kind, min_len, max_len, dom_k)} of use j, by the definitions above.

    reduced=True (default): minima, K* and the rule-2 sets from the simple paths (enough, by the
    cutting argument in the module docstring), then every path with at most max K* crossings for
    the maxima.  reduced=False: every path with at most B crossings for everything (the direct
    reading; exponential in B, used on a subset to check the reduction)."""
    cfg = cfg or _Cfg(S)
    per_def = {}     # i -> {"kind", "states": [(len, k)], "dom_sets": [set per linking register]}
    for r, kind in reads(S, j):
        found = paths_to_defs(S, cfg, j, r, simple=reduced)
        by_def = {}
        for x, length, k, between in found:
            by_def.setdefault(x, []).append((length, k, between))
        if reduced and by_def:
            kmax = max(min(k for _, k, _ in st) for st in by_def.values())
            longest = {}
            for x, length, k, _ in paths_to_defs(S, cfg, j, r, max_cross=kmax):
                longest.setdefault(x, []).append((length, k, None))
            for x in by_def:
                by_def[x] = by_def[x] + [(l, k, None) for l, k, _ in longest[x]]
        for i, states in by_def.items():
            d = per_def.setdefault(i, {"kind": 0, "states": [], "dom_sets": []})
            kk = kind
            if r >= 512 and int(S.rbar[i]) >> (r - 512) & 1:
                jd = {int(v) for v in S.dst[j] if int(v) not in (NONE, RZ)}
                isrc = {int(v) for v in S.src[i] if int(v) not in (NONE, RZ)}
                if jd & isrc:
                    kk |= WAR
            d["kind"] |= kk
            d["states"] += [(length, k) for length, k, _ in states]
            on_every = set.intersection(*[set(b) for _, _, b in states if b is not None])
            d["dom_sets"].append({k for k in on_every
                                  if k not in (i, j) and int(S.guard[k]) & 7 == 7
                                  and any(rr == r for rr, _ in reads(S, k))})
    out = {}
    for i, d in per_def.items():
        mn = min(l for l, _ in d["states"])
        kstar = min(k for _, k in d["states"])
        mx = max(l for l, k in d["states"] if k == kstar)
        dom = set.intersection(*d["dom_sets"])
        out[i] = (d["kind"], mn, mx, min(dom) if dom else -1)
    return out


def slice_all(S, reduced: bool = True):
    """{use j: [(def i, kind, min_len, max_len, dom_k)] ascending by i} for every instruction."""
    cfg = _Cfg(S)
    res = {}
    for j in range(len(S.guard)):
        row = slice_use(S, j, cfg, reduced)
        if row:
            res[j] = [(i, *row[i]) for i in sorted(row)]
    return res

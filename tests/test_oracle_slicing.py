"""Pins of the oracle's backward slicing (readings DESIGN.md
§3.2 Q35-Q39): the def-use graph of gpagen.sass.slice_fixture() derived by hand, SPEC's path-length
examples, the brute-force path enumerator of tests/slice_enum.py (the definitions
evaluated path by path; no code shared with oracle/) on 1,500 random <= 24-instruction CFGs with
nested, multi-exit and multi-back-edge loops, and properties of larger random programs."""
import numpy as np
import pytest

import oracle
from gpagen import sass
from tests.slice_enum import slice_all

REG, PRED, BAR, WAR = 1, 2, 4, 8

# use j -> [(def i, kind, min_len, max_len, dom_k)], derived by hand (see slice_fixture's doc)
EXPECTED = {
    1: [(0, REG, 1, 1, -1)],                       # ISETP reads R10 <- S2R
    2: [(0, REG, 2, 2, 1)],                        # the ISETP at 1 reads R10 on the only path: rule 2
    3: [(2, REG, 1, 1, -1)],                       # P0 is never defined: no predicate edge
    4: [(2, REG, 2, 2, -1)],                       # the LDC at 3 reads R2 but is predicated
    5: [(2, REG, 3, 3, 4)],                        # Fig. 5 / P:367: MOV R3, R2 at 4 interposes
    6: [(1, PRED, 5, 5, -1)],                      # @P1 BRA <- ISETP P1
    7: [(3, REG | BAR, 4, 4, -1), (5, REG | BAR, 2, 2, -1)],   # @P0 LDG then @!P0 LDC cover '_'
    8: [(4, REG, 4, 4, -1), (7, REG, 1, 1, -1)],
    9: [(4, REG, 3, 3, -1)],
    # R4 from both arms, 1 step without the back edge (K* = 0, so the path through one more loop
    # iteration does not count: S:185); R6 loop-carried from the FFMA (K* = 1: 10 <- 13 <- 12),
    # whose value the MOV at 13 reads on every path: rule 2
    10: [(8, REG, 1, 1, -1), (9, REG, 1, 1, -1), (12, REG, 2, 2, 13)],
    11: [(10, REG, 1, 1, -1)],
    12: [(10, REG, 2, 2, 11), (11, REG | BAR, 1, 1, -1)],    # the LDS at 11 reads R5: rule 2
    13: [(11, BAR | WAR, 2, 2, -1), (12, REG, 1, 1, -1)],    # read barrier B3 + MOV overwrites R5: WAR
    14: [(12, REG, 2, 2, 13)],
    15: [(14, BAR, 1, 1, -1)],                     # Fig. 3: BRA waits on the LDG's barrier only
}


def _rows(csr):
    rp = csr["row_ptr"]
    out = {}
    for j in range(len(rp) - 1):
        es = [(int(csr["edge_def"][e]), int(csr["edge_kind"][e]), int(csr["edge_min_len"][e]),
               int(csr["edge_max_len"][e]), int(csr["edge_dom_k"][e])) for e in range(rp[j], rp[j + 1])]
        if es:
            out[j] = es
    return out


def test_slice_fixture_matches_hand_derivation():
    assert _rows(oracle.slice_program(sass.slice_fixture())) == EXPECTED


def test_random_programs_slicing_properties():
    for seed in (1, 2, 3):
        S = sass.random_sass(6, seed)
        csr = oracle.slice_program(S)
        rp = csr["row_ptr"].astype(np.int64)
        n = S.n_instr
        fb = S.func_begin.astype(np.int64)
        func_of = np.searchsorted(fb, np.arange(n), side="right") - 1
        assert rp[-1] > n // 2
        for j in range(n):
            defs = csr["edge_def"][rp[j]:rp[j + 1]].astype(np.int64)
            assert np.all(np.diff(defs) > 0)                          # one edge per def, ascending
            assert np.all(func_of[defs] == func_of[j])                # intra-function
            mn = csr["edge_min_len"][rp[j]:rp[j + 1]]
            mx = csr["edge_max_len"][rp[j]:rp[j + 1]]
            assert np.all(mn >= 1) and np.all(mx >= mn)
            for e in range(rp[j], rp[j + 1]):
                i, k = int(csr["edge_def"][e]), int(csr["edge_dom_k"][e])
                kind = int(csr["edge_kind"][e])
                assert kind != 0 and (kind & WAR == 0 or kind & BAR)
                # straight-line defs before j in j's own block: the path length is j - i
                b = np.searchsorted(S.block_begin.astype(np.int64), j, side="right") - 1
                if S.block_begin[b] <= i < j:
                    assert int(csr["edge_min_len"][e]) == j - i
                if k >= 0:
                    assert k != i and k != j and func_of[k] == func_of[j] and S.guard[k] == sass.ALWAYS


def test_enumerator_reproduces_hand_derivation():
    """The brute-force enumerator itself is pinned to the hand-derived fixture."""
    assert slice_all(sass.slice_fixture()) == EXPECTED


def _spec_cases():
    """SPEC S:175-177 path_distance examples as SASS: (program, use j, def i, min, max)."""
    R1, R2 = 1, 2
    # adjacent instructions in one block: min = max = 1
    adj = sass._build([dict(dst=[R1]), dict(src=[R1])], [(0, 2)], [[]])
    # diamond with arms of 2 and 5 instructions: min 3, max 6 (arm + the join instruction)
    I = [dict(dst=[R1])] + [dict(dst=[9])] * 2 + [dict(dst=[9])] * 5 + [dict(src=[R1])]
    dia = sass._build(I, [(0, 1), (1, 3), (3, 8), (8, 9)], [[1, 2], [3], [3], []])
    # j before i in a loop body (loop block [2, 6) with a back edge): R1 is defined at 4 after the
    # use at 3, so the path needs the back edge once: 3 <- 2 <- 5 <- 4, min = max = 3; R2 defined
    # before the loop: reachable without the back edge (K* = 0), 3 <- 2 <- 1, min = max = 2
    I = [dict(dst=[9]), dict(dst=[R2]), dict(dst=[9]), dict(src=[R1, R2]), dict(dst=[R1]), dict(dst=[9]), dict()]
    lp = sass._build(I, [(0, 2), (2, 6), (6, 7)], [[1], [1, 2], []])
    return [(adj, 1, 0, 1, 1), (dia, 8, 0, 3, 6), (lp, 3, 4, 3, 3), (lp, 3, 1, 2, 2)]


@pytest.mark.parametrize("case", range(4))
def test_spec_path_length_examples(case):
    S, j, i, mn, mx = _spec_cases()[case]
    for rows in (_rows(oracle.slice_program(S)), slice_all(S)):
        e = {d: (a, b) for d, _, a, b, _ in rows[j]}
        assert e[i] == (mn, mx)


def test_oracle_matches_path_enumeration_on_random_cfgs():
    """the oracle's CSR equals the brute-force definitions (min_len, K* /
    max_len, dom_k over every path, kinds) on 1,500 random tiny CFGs: nested loops, multi-block
    bodies, `continue` (several back edges), `break` (multi-exit), loops headed by the entry
    block, 1-3 functions."""
    n_back = 0
    for seed in range(1500):
        S = sass.random_cfg_sass(seed, n_funcs=1 + seed % 3)
        assert np.diff(S.func_begin.astype(np.int64)).max() <= 24
        n_back += sum(int(S.block_begin[t]) <= int(S.block_begin[b + 1]) - 1 for b in range(len(S.block_begin) - 1)
                      for t in S.succ[S.succ_ptr[b]:S.succ_ptr[b + 1]])
        assert _rows(oracle.slice_program(S)) == slice_all(S), seed
    assert n_back > 2000


def test_enumerator_reduction_equals_direct_enumeration():
    """The enumerator's shortcut (simple paths for minima / K* / rule 2) agrees with listing every
    path of at most B back-edge crossings."""
    for seed in range(8):
        S = sass.random_cfg_sass(seed)
        assert slice_all(S) == slice_all(S, reduced=False)

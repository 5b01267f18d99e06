"""Pins of the oracle's backward slicing (readings DESIGN.md
§3.2 Q35-Q39): the def-use graph of gpagen.sass.slice_fixture() derived by hand, and properties
of random programs that any correct slicer has."""
import numpy as np

import oracle
from gpagen import sass

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
    # R4 from both arms (1 step; 5 steps through one loop iteration), R6 loop-carried from the
    # FFMA, whose value the MOV at 13 reads on every path: rule 2
    10: [(8, REG, 1, 5, -1), (9, REG, 1, 5, -1), (12, REG, 2, 2, 13)],
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

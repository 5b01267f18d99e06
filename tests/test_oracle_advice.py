"""Pins of the oracle's advice step (hotspots, optimizer ranking, single
dependency coverage) against values derived by hand from the
config-1 fixture (tests/golden/tiny_fixture.txt) and closed forms.  Readings:
DESIGN.md §3.2 Q30-Q32."""
import numpy as np
import pytest

import oracle
from gpagen import programs as gp
from gpagen.patterns import table2
from gpagen.streams import StreamSpec
from tests.test_oracle_pins import _pat, _prog, _records

T2 = table2()
Q = {p["name"]: i for i, p in enumerate(T2)}


@pytest.fixture(scope="module")
def tiny():
    prog = gp.tiny_fixture()
    op = oracle.OracleProgram(prog)
    res = op.run_all(gp.tiny_records(), [_pat(p) for p in T2])
    return prog, op, res


def _tuples(lst):
    return [(h.def_pc, h.use_pc, h.distance, h.item, h.samples) for h in lst]


def test_tiny_loop_unrolling_hotspots(tiny):
    """Latency samples of global-memory and execution dependencies inside loop 8..18:
    8->9 = MEM 24 x 1 + EXEC 8 x 1/4 (weights A_8/1 = 8 vs A_7/2 = 24) = 26; 14->15 = EXEC 16 x
    12/16 = 12; 12->11 (WAR) = 16 x 4/8 = 8; 9->11 and 10->11 = 16 x 2/8 = 4 each; 11->15 also
    carries 4 but has the larger item id (edge 10 > 7, 8), so it is sixth."""
    prog, op, res = tiny
    h = op.hotspots(res["C"], res, [_pat(p) for p in T2], 5)
    assert _tuples(h[0][Q["loop_unrolling"]]) == [(8, 9, 1, 5, 26.0), (14, 15, 1, 11, 12.0), (12, 11, 10, 9, 8.0),
                                                  (9, 11, 2, 7, 4.0), (10, 11, 1, 8, 4.0)]
    h6 = op.hotspots(res["C"], res, [_pat(p) for p in T2], 6)
    assert _tuples(h6[0][Q["loop_unrolling"]])[5] == (11, 15, 4, 10, 4.0)
    # all items of the pattern sum to its matched latency samples M = 58 (golden est line)
    hall = op.hotspots(res["C"], res, [_pat(p) for p in T2], 64)
    assert sum(x.samples for x in hall[0][Q["loop_unrolling"]]) == 58.0


def test_tiny_code_reordering_and_single_item_hotspots(tiny):
    """Code reordering (no loop filter): 19->20 = MEM 20 x 1; 5->7 = MEM 12 x 1/2 (LDC and LDG
    weigh 40/4 = 20/2) + EXEC 4 x 10/40 (the IMAD weighs 20) = 7.  Strength reduction: the F2F
    10->11 edge, EXEC 16 (ACT 0 + LAT 16) x 2/8 = 4.  Function split: FETCH at 18, 8 samples,
    a self item (def = use, distance 0, item E + 18 = 31).  Warp balance: the BAR.SYNC's own
    32 sync samples."""
    prog, op, res = tiny
    h = op.hotspots(res["C"], res, [_pat(p) for p in T2], 5)
    assert _tuples(h[0][Q["code_reordering"]]) == [(8, 9, 1, 5, 26.0), (19, 20, 1, 12, 20.0), (14, 15, 1, 11, 12.0),
                                                   (12, 11, 10, 9, 8.0), (5, 7, 2, 2, 7.0)]
    assert _tuples(h[0][Q["strength_reduction"]]) == [(10, 11, 1, 8, 4.0)]
    assert _tuples(h[0][Q["function_split"]]) == [(18, 18, 0, 31, 8.0)]
    assert _tuples(h[0][Q["warp_balance"]]) == [(13, 13, 0, 26, 32.0)]
    assert h[0][Q["register_reuse"]] == [] and h[0][Q["block_increase"]] == []


def test_tiny_single_dependency_coverage(tiny):
    """Live nodes (dependency stalls): 5, 7, 9, 11, 13, 15, 20.  Before pruning single: 5 (one
    in-edge), 13 (none), 20 (one) -> 3/7.  After pruning: 5 (its edge is rule-2 pruned), 13, 20
    (one MEM candidate); 7 keeps two MEM candidates (LDC, LDG), 9 two EXEC (8, 7), 11 three,
    15 two -> 3/7."""
    prog, op, res = tiny
    assert op.coverage(res["C"], res["cand"]).tolist() == [[7, 3, 3]]


def test_coverage_closed_forms():
    """Edgeless graph -> every live node is single (coverage 1).  Ten live nodes, one with two
    memory-dependency in-edges from loads -> 9/10 before and after; rule 1 drops an arithmetic
    def's memory candidacy -> that node becomes single after pruning only (Fig. 8's claim that
    coverage does not drop)."""
    n = 10
    prog = _prog([gp.GLOBAL] * n, [[] for _ in range(n)])
    op = oracle.OracleProgram(prog)
    res = op.run_all(_records([(i, 1, 1, 3) for i in range(n)]))
    assert op.coverage(res["C"], res["cand"]).tolist() == [[n, n, n]]
    rows = [[] for _ in range(n)]
    rows[9] = [(0, gp.REG, 2, 2, -1), (1, gp.REG, 3, 3, -1)]
    prog = _prog([gp.GLOBAL] * n, rows)
    op = oracle.OracleProgram(prog)
    res = op.run_all(_records([(i, 1, 1, 3) for i in range(n)]))
    assert op.coverage(res["C"], res["cand"]).tolist() == [[n, 9, 9]]
    prog = _prog([gp.GLOBAL, gp.ARITH_FIXED] + [gp.GLOBAL] * (n - 2), rows, latency=[1024, 4] + [1024] * (n - 2))
    op = oracle.OracleProgram(prog)
    res = op.run_all(_records([(i, 1, 1, 3) for i in range(n)]))
    assert op.coverage(res["C"], res["cand"]).tolist() == [[n, 9, 10]]


def test_coverage_never_drops_after_pruning():
    for seed in (3, 4, 5):
        prog = gp.random_program(700, 3, 8, 3, seed=seed, n_kernels=2)
        op = oracle.OracleProgram(prog)
        res = op.run_all(StreamSpec(prog, seed=seed + 10).host(0, 50_000))
        cov = op.coverage(res["C"], res["cand"])
        assert np.all(cov[:, 2] >= cov[:, 1]) and np.all(cov[:, 0] >= cov[:, 2])
        assert cov[:, 0].sum() > 0


def _est(speedups):
    row = []
    for s in speedups:
        e = oracle.Estimate()
        e.speedup = s
        row.append(e)
    return row


def test_rank_orders_by_speedup_with_stable_ties():
    """suggestions sorted by estimated speedup; an unbounded estimate (+inf) first, equal
    speedups keep the optimizer order."""
    order = oracle.rank([_est([1.0, 1.2, float("inf"), 1.2, 1.01]), _est([1.0, 1.0, 1.0, 1.0, 1.0])])
    assert order.tolist() == [[2, 1, 3, 4, 0], [0, 1, 2, 3, 4]]


def test_tiny_rank(tiny):
    prog, op, res = tiny
    sp = [e.speedup for e in res["est"][0]]
    order = oracle.rank(res["est"])[0].tolist()
    assert order[0] == Q["block_increase"] and order[1] == Q["code_reordering"] and order[2] == Q["loop_unrolling"]
    assert all(sp[a] >= sp[b] for a, b in zip(order, order[1:]))

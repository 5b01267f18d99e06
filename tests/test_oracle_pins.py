"""Pins of the CPU oracle against what the paper and mathematics fix (not against itself).

Every expected value here is (a) printed in the paper or derived by hand from it
(tests/golden/*, each with its citation), (b) a closed form, (c) an invariant, or
(d) a brute-force/alternative computation on tiny inputs.  CPU only.
"""
from fractions import Fraction
import os

import numpy as np
import pytest

import oracle
from gpagen import programs as gp
from gpagen.patterns import table2
from gpagen.streams import StreamSpec

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _pat(d):
    return oracle.Pattern(*[d[k] for k in ("column_mask", "class_mask", "sample_class", "model",
                                           "flag_filter", "same_loop", "parallel_rule")], 0,
                          d["sm_count"], d["ratio"], d["W"], d["W_new"], d["f"])


def _golden(name):
    out = {}
    with open(os.path.join(GOLD, name)) as fh:
        for line in fh:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            tok = line.split()
            out.setdefault(tok[0], []).append(tok[1:])
    return out


def _records(entries):
    """entries: list of (pc, cls, reason, count, flags_extra)."""
    recs = []
    for e in entries:
        pc, c, r, k = e[:4]
        extra = e[4] if len(e) > 4 else 0
        recs.append(pc | (k << 32) | (r << 48) | ((c | extra) << 56))
    return np.array(recs, dtype=np.uint64)


def _prog(classes, rows, latency=None, loops=None, loop_parent=(), iflags=None, line_id=None,
          funcs=None, kernels=None, R=9):
    n = len(classes)
    lat = latency if latency is not None else [1024] * n
    return gp._finalize(R, classes, iflags or [0] * n, lat,
                        line_id if line_id is not None else list(range(n)),
                        loops if loops is not None else [-1] * n, list(loop_parent),
                        funcs or [0, n], kernels or [0, len(funcs or [0, n]) - 1], [16] * len(
                            (kernels or [0, 1])[:-1]), rows,
                        n_lines=(max(line_id) + 1) if line_id is not None else n)


# ---------------------------------------------------------------------- tiny fixture (config 1)
@pytest.fixture(scope="module")
def tiny():
    prog = gp.tiny_fixture()
    op = oracle.OracleProgram(prog)
    recs = gp.tiny_records()
    res = op.run_all(recs, [_pat(p) for p in table2()])
    return prog, op, res


def test_tiny_histogram_reproduces_fixture_counts(tiny):
    prog, op, res = tiny
    C = res["C"]
    expect = np.zeros_like(C)
    for (pc, c, r), k in gp.TINY_COUNTS.items():
        expect[pc, c, r] = k
    assert np.array_equal(C, expect)
    assert list(res["stats"]) == [500, 0, 0]


def test_tiny_totals(tiny):
    _, _, res = tiny
    T, A, L = map(int, _golden("tiny_fixture.txt")["total"][0])
    assert int(res["kern_al"][0, 0]) == A and int(res["kern_al"][0, 1]) == L and A + L == T


def test_tiny_candidates_and_self(tiny):
    prog, _, res = tiny
    g = _golden("tiny_fixture.txt")
    for e, d, u, m in g["cand"]:
        e = int(e)
        assert int(prog.edge_def[e]) == int(d)
        assert int(prog.row_ptr[int(u)]) <= e < int(prog.row_ptr[int(u) + 1])
        assert int(res["cand"][e]) == int(m), f"edge {e}"
    expect_self = np.zeros(prog.n_instr, np.uint8)
    for pc, m in g["self"]:
        expect_self[int(pc)] = int(m)
    assert np.array_equal(res["self"], expect_self)


def test_tiny_shares_exact(tiny):
    _, _, res = tiny
    for e, *sh in _golden("tiny_fixture.txt")["share"]:
        for r in range(3):
            assert res["share"][int(e), r] == float(Fraction(sh[r])), (e, r)


def test_tiny_instruction_blame_exact(tiny):
    prog, op, res = tiny
    expect = np.zeros((prog.n_instr, op.ncol, 2))
    for pc, col, a, l in _golden("tiny_fixture.txt")["V"]:
        expect[int(pc), int(col)] = (float(a), float(l))
    assert np.array_equal(res["V"], expect)


def test_tiny_rollups_exact(tiny):
    prog, op, res = tiny
    g = _golden("tiny_fixture.txt")
    k = np.zeros((op.ncol, 2))
    for col, a, l in g["kern"]:
        k[int(col)] = (float(a), float(l))
    assert np.array_equal(res["kern_v"][0], k)
    lp = np.zeros((op.ncol, 2))
    for col, a, l in g["loop"]:
        lp[int(col)] = (float(a), float(l))
    assert np.array_equal(res["loop_incl_v"][0], lp)
    assert np.array_equal(res["loop_excl_v"][0], lp)          # single loop: excl == incl
    a, l = map(int, g["loopAL"][0])
    assert list(map(int, res["loop_incl_al"][0])) == [a, l]


def test_tiny_estimates_exact(tiny):
    _, _, res = tiny
    names = [p["name"] for p in table2()]
    est = res["est"][0]
    for name, num, den, M, best in _golden("tiny_fixture.txt")["est"]:
        o = est[names.index(name)]
        assert o.speedup == pytest.approx(float(Fraction(int(num), int(den))), rel=1e-15), name
        assert o.M == float(M), name
        assert o.best_scope == int(best), name
        assert o.T == 500 and o.A == 330


def test_tiny_block_increase_matches_fewer_blocks_than_sms(tiny):
    _, _, res = tiny
    names = [p["name"] for p in table2()]
    bi = res["est"][0][names.index("block_increase")]
    ti = res["est"][0][names.index("thread_increase")]
    assert bi.matched == 1 and ti.matched == 0 and ti.speedup == 1.0   # grid 16 < 80 SMs
    # R_I = A / T = 330/500; W = 8 -> W_new = 4, f = 1 evaluated in exact rationals
    R = Fraction(330, 500)
    I, In = 1 - (1 - R) ** 8, 1 - (1 - R) ** 4
    assert bi.speedup == pytest.approx(float(2 * In / I), rel=1e-14)


# ---------------------------------------------------------------------- Fig. 2
def test_fig2_sampling_counts():
    """6 samples: latency at N, 4N, 6N; stalls at N, 3N, 4N, 5N, 6N -> A = L = 3, 5 stall
    samples, stall ratio = active ratio = 3/6."""
    prog = _prog([gp.ARITH_FIXED], [[]])
    op = oracle.OracleProgram(prog)
    recs = _records([(0, 1, 1, 1), (0, 0, 0, 1), (0, 0, 1, 1), (0, 1, 1, 1), (0, 0, 1, 1), (0, 1, 1, 1)])
    res = op.run_all(recs)
    A, L = map(int, res["kern_al"][0])
    assert (A, L) == (3, 3) and Fraction(A, A + L) == Fraction(3, 6)
    assert res["kern_v"][0, :, 0].sum() == 5        # five stall samples, all MEM, self-held


# ---------------------------------------------------------------------- Eq. 1 and pruning
def _fig5_program(path_ldc=4, path_ldg=2):
    # 0 @!P0 LDC R0 (constant), 1 @P0 LDG R0 (global), 2 IMAD R5, 3 IADD R6 <- R0, R5
    rows = [[], [], [], [(0, gp.REG | gp.BAR, path_ldc, path_ldc, -1),
                         (1, gp.REG | gp.BAR, path_ldg, path_ldg, -1),
                         (2, gp.REG, 1, 1, -1)]]
    return _prog([gp.CONSTANT, gp.GLOBAL, gp.ARITH_FIXED, gp.ARITH_FIXED], rows,
                 latency=[64, 1024, 4, 4])


def test_fig5_rule1_prunes_imad_and_split_is_equal():
    """Fig. 5: IMAD->IADD is not a memory-dependency source; LDC has twice the
    issued samples and twice the path length of LDG, so each gets half of the stalls."""
    prog = _fig5_program()
    op = oracle.OracleProgram(prog)
    recs = _records([(0, 0, 0, 40), (1, 0, 0, 20), (2, 0, 0, 7), (3, 1, 1, 60)])
    res = op.run_all(recs)
    assert list(res["cand"]) == [0b011, 0b011, 0b010]
    assert res["share"][0, 0] == 0.5 and res["share"][1, 0] == 0.5 and res["share"][2, 0] == 0.0
    assert res["V"][0, 2, 0] == 30.0 and res["V"][1, 0, 0] == 30.0   # constant / global memory


def test_spec_three_way_split():
    """issued {1,2,3}, max_len {1,2,3}, S_j = 60 -> weights {1,1,1} -> 20 each."""
    rows = [[], [], [], [(0, gp.REG, 1, 1, -1), (1, gp.REG, 2, 2, -1), (2, gp.REG, 3, 3, -1)]]
    prog = _prog([gp.GLOBAL] * 4, rows)
    op = oracle.OracleProgram(prog)
    res = op.run_all(_records([(0, 0, 0, 1), (1, 0, 0, 2), (2, 0, 0, 3), (3, 1, 1, 60)]))
    blame = res["share"][:, 0] * 60.0
    assert blame == pytest.approx([20.0, 20.0, 20.0], rel=1e-15)
    assert res["V"][:3, 0, 0] == pytest.approx([20.0] * 3, rel=1e-15)


def test_single_candidate_takes_all_and_none_self_attributes():
    rows = [[], [(0, gp.REG, 1, 1, -1)], [(0, gp.REG, 1, 1, -1)]]
    prog = _prog([gp.ARITH_FIXED, gp.ARITH_FIXED, gp.ARITH_FIXED], rows, latency=[4, 4, 4])
    op = oracle.OracleProgram(prog)
    res = op.run_all(_records([(1, 1, 2, 9), (2, 1, 1, 5)]))
    assert res["share"][0, 1] == 1.0 and res["V"][0, 4, 1] == 9.0       # exec -> arithmetic
    # MEM stall at 2 with only an arithmetic def: rule 1 prunes it, the stall stays at 2
    assert res["cand"][1] & 1 == 0 and res["self"][2] & 1 and res["V"][2, 7, 1] == 5.0


def test_fig3_barrier_only_dependency():
    """LDG writes B0, BRA waits on B0 without reading R0: memory stalls at BRA are blamed on
    the LDG, classified as global memory (Fig. 6)."""
    prog = _prog([gp.GLOBAL, gp.CONTROL], [[], [(0, gp.BAR, 1, 1, -1)]], latency=[1024, 8])
    op = oracle.OracleProgram(prog)
    res = op.run_all(_records([(0, 0, 0, 3), (1, 1, 1, 11)]))
    assert res["cand"][0] == 0b011 and res["V"][0, 0, 0] == 11.0 and res["V"][1, 7, 0] == 0.0


@pytest.mark.parametrize("path,kept", [(199, True), (200, True), (201, False), (300, False)])
def test_rule3_latency_boundary(path, kept):
    """Prune iff every path is longer than latency(i): min_len > latency (Q8; S:341 uses
    LDG latency 200 with a 300-instruction path)."""
    prog = _prog([gp.GLOBAL, gp.ARITH_FIXED], [[], [(0, gp.REG, path, path + 5, -1)]],
                 latency=[200, 4])
    op = oracle.OracleProgram(prog)
    res = op.run_all(_records([(1, 1, 1, 4)]))
    assert bool(res["cand"][0] & 1) == kept
    assert bool(res["self"][1] & 1) == (not kept)


@pytest.mark.parametrize("dom_k,kept", [(-1, True), (1, False)])
def test_rule2_dominating_reader(dom_k, kept):
    """An unpredicated reader k on every i->j path removes the edge."""
    rows = [[], [], [(0, gp.REG, 2, 2, dom_k)]]
    prog = _prog([gp.GLOBAL, gp.ARITH_FIXED, gp.ARITH_FIXED], rows, latency=[1024, 4, 4])
    res = oracle.OracleProgram(prog).run_all(_records([(2, 1, 1, 4), (2, 1, 2, 4)]))
    assert res["cand"][0] == (0b011 if kept else 0)


def test_sync_rule1_and_shared_is_execution_source():
    """Sync stalls only to sync instructions; shared-memory defs are execution
    dependencies (Fig. 6(b)), never memory-dependency sources (Q6)."""
    rows = [[], [], [(0, gp.REG, 1, 1, -1), (1, gp.REG, 2, 2, -1)]]
    prog = _prog([gp.SHARED, gp.SYNC, gp.ARITH_FIXED], rows, latency=[32, 20, 4])
    res = oracle.OracleProgram(prog).run_all(_records([(2, 1, 1, 4), (2, 1, 2, 8), (2, 1, 3, 6)]))
    assert list(res["cand"]) == [0b010, 0b110]
    assert res["self"][2] == 0b001
    assert res["V"][1, 6, 0] == 6.0            # all sync stalls to the SYNC def
    assert res["V"][0, 3, 0] + res["V"][1, 4, 0] == 8.0   # exec: shared + arithmetic categories


def test_war_classification():
    """WAR: variable-latency def reads a register the use writes -> EXEC_WAR."""
    rows = [[], [(0, gp.WAR | gp.BAR, 3, 3, -1)]]
    prog = _prog([gp.GLOBAL, gp.ARITH_FIXED], rows, latency=[1024, 4])
    res = oracle.OracleProgram(prog).run_all(_records([(1, 1, 2, 7), (1, 1, 1, 3)]))
    assert res["V"][0, 5, 0] == 7.0 and res["V"][0, 0, 0] == 3.0


def test_zero_issue_def_counts_as_one():
    """A def with no active samples weighs like one issued sample (Q4)."""
    rows = [[], [], [(0, gp.REG, 1, 1, -1), (1, gp.REG, 1, 1, -1)]]
    prog = _prog([gp.GLOBAL] * 3, rows)
    res = oracle.OracleProgram(prog).run_all(_records([(1, 0, 0, 3), (2, 1, 1, 8)]))
    assert res["share"][0, 0] == 0.25 and res["share"][1, 0] == 0.75


# ---------------------------------------------------------------------- estimators
def test_eq2_closed_forms():
    assert oracle.eq2(100, 50) == 2.0 and oracle.eq2(100, 0) == 1.0
    assert oracle.eq2(100, 100) == float("inf")


def test_eq4_closed_forms():
    assert oracle.eq4(100, 30, 50) == pytest.approx(100 / 70, rel=1e-15)
    assert oracle.eq4(100, 50, 50) == 2.0          # Theorem 1 extremal case


def test_eq5_nested_loops():
    """T=100, loop2 contains loop1, A = {10, 10}, M^L = 40 -> min(20, 40) -> 5/4."""
    assert oracle.eq5(100, 10 + 10, 40) == 1.25


def test_eq10_closed_form():
    """W=8, W_new=4, R_I=0.2, f=1: I = 1-0.8^8, I_new = 1-0.8^4, S^p = 1250/881 exactly
    (SPEC.md S:522 prints 1.418847, which is 4.8e-6 off)."""
    assert oracle.eq10(8, 4, 0.2, 1.0) == pytest.approx(1250 / 881, rel=1e-14)
    assert oracle.eq10(8, 8, 0.37, 0.9) == pytest.approx(0.9, rel=1e-15)    # W_new = W -> f
    assert oracle.eq10(8, 4, 1.0, 1.0) == 2.0                               # R_I = 1 -> f / C_W
    assert oracle.eq10(8, 4, 0.0, 1.0) == 2.0                               # I = 0 -> C_I := 1


def test_theorem1_property():
    """S^h <= 2 for every T = A + L, 0 <= M^L <= L; both proof branches hit."""
    rng = np.random.default_rng(1)
    hits = [0, 0]
    for _ in range(10000):
        A, L = (int(x) for x in rng.integers(0, 10**6, size=2))
        if A + L == 0:
            continue
        ML = int(rng.integers(0, L + 1))
        s = oracle.eq4(A + L, A, ML)
        assert s <= 2.0
        assert oracle.eq2(A + L, ML) >= s           # Eq. 3 >= Eq. 4
        hits[0 if A <= ML else 1] += 1
    assert min(hits) >= 1000


# ---------------------------------------------------------------------- properties on random inputs
@pytest.fixture(scope="module", params=[11, 12, 13])
def rand_case(request):
    prog = gp.random_program(300, 3, 6, 3, seed=request.param, n_reasons=9)
    spec = StreamSpec(prog, seed=request.param * 7919, count_max=5, invalid_ppm=20000)
    recs = spec.host(0, 40000)
    op = oracle.OracleProgram(prog)
    return prog, op, recs, op.run_all(recs, [_pat(p) for p in table2()])


def test_histogram_properties(rand_case):
    prog, op, recs, res = rand_case
    # independent decode of the records (numpy field extraction + bincount)
    pc = (recs & 0xFFFFFFFF).astype(np.int64)
    cnt = ((recs >> 32) & 0xFFFF).astype(np.int64)
    rs = ((recs >> 48) & 0xFF).astype(np.int64)
    fl = (recs >> 56).astype(np.int64)
    ok = (pc < prog.n_instr) & (rs < 9) & ((fl & ~1) == 0) & ~((fl == 1) & (rs == 0))
    key = (pc[ok] * 2 + fl[ok]) * 9 + rs[ok]
    expect = np.bincount(key, weights=cnt[ok], minlength=prog.n_instr * 18)
    assert np.array_equal(res["C"].reshape(-1).astype(np.int64), expect.astype(np.int64))
    assert int(res["stats"][1]) == int((~ok).sum()) > 0 and int(res["stats"][2]) == int(cnt[~ok].sum())
    # shard and order invariance
    C1, s1 = op.histogram(recs[:12345])
    op.histogram(recs[12345:], C1, s1)
    assert np.array_equal(C1, res["C"])
    C2, _ = op.histogram(recs[::-1].copy())
    assert np.array_equal(C2, res["C"])
    # a count-c record equals c count-1 records
    first = recs[ok][:50]
    expanded = np.concatenate([np.repeat((r & ~np.uint64(0xFFFF << 32)) | np.uint64(1 << 32),
                                         int((r >> np.uint64(32)) & np.uint64(0xFFFF))) for r in first])
    Ca, _ = op.histogram(first)
    Cb, _ = op.histogram(expanded)
    assert np.array_equal(Ca, Cb)


def test_blame_conservation(rand_case):
    """Per (j, r in D, class): sum over edges of attributed + self = observed (Q5)."""
    prog, op, recs, res = rand_case
    C = res["C"].astype(np.float64)
    share = res["share"]
    for j in range(prog.n_instr):
        e0, e1 = int(prog.row_ptr[j]), int(prog.row_ptr[j + 1])
        for r in (1, 2, 3):
            tot = share[e0:e1, r - 1].sum()
            if res["self"][j] >> (r - 1) & 1:
                assert tot == 0.0
            elif C[j, :, r].sum() > 0:
                assert tot == pytest.approx(1.0, rel=1e-12)
    V = res["V"]
    stall_all = C[:, :, 1:].sum()
    stall_lat = C[:, 1, 1:].sum()
    assert V[:, :, 0].sum() == pytest.approx(stall_all, rel=1e-12)
    assert V[:, :, 1].sum() == pytest.approx(stall_lat, rel=1e-12)
    # per reason: memory columns hold exactly the memory-dependency stalls, etc.
    assert V[:, [0, 1, 2, 7], 0].sum() == pytest.approx(C[:, :, 1].sum(), rel=1e-12)
    assert V[:, [3, 4, 5, 8], 0].sum() == pytest.approx(C[:, :, 2].sum(), rel=1e-12)
    assert V[:, [6, 9], 0].sum() == pytest.approx(C[:, :, 3].sum(), rel=1e-12)
    assert np.array_equal(V[:, 10:, 0], C[:, :, 4:].sum(axis=1))


def test_candidates_brute_force(rand_case):
    """Candidate masks re-derived per edge from the three rules' text."""
    prog, op, recs, res = rand_case
    C = res["C"]
    mem = {gp.GLOBAL, gp.LOCAL, gp.CONSTANT, gp.TEXTURE}
    for j in range(prog.n_instr):
        live = C[j, :, 1:4].sum() > 0
        for e in range(int(prog.row_ptr[j]), int(prog.row_ptr[j + 1])):
            d = int(prog.edge_def[e])
            ok = prog.edge_dom_k[e] < 0 and prog.edge_min_len[e] <= prog.latency[d] and live
            m = (int(ok and prog.opclass[d] in mem) | int(ok) << 1 | int(ok and prog.opclass[d] == gp.SYNC) << 2)
            assert res["cand"][e] == m


def test_rollup_brute_force(rand_case):
    prog, op, recs, res = rand_case
    V = res["V"]
    lines = np.zeros((prog.n_lines,) + V.shape[1:])
    np.add.at(lines, prog.line_id.astype(np.int64), V)
    assert np.allclose(res["line_v"], lines, rtol=1e-12, atol=0)
    for l in range(prog.n_loops):
        members = []
        for i in range(prog.n_instr):
            x = int(prog.loop_id[i])
            while x >= 0 and x != l:
                x = int(prog.loop_parent[x])
            if x == l:
                members.append(i)
        assert np.allclose(res["loop_incl_v"][l], V[members].sum(axis=0), rtol=1e-12, atol=0)
        excl = np.nonzero(prog.loop_id == l)[0]
        assert np.allclose(res["loop_excl_v"][l], V[excl].sum(axis=0), rtol=1e-12, atol=0)
        Aincl = int(res["C"][members, 0, :].sum())
        assert int(res["loop_incl_al"][l, 0]) == Aincl
    for f in range(prog.n_funcs):
        a, b = int(prog.func_begin[f]), int(prog.func_begin[f + 1])
        assert np.allclose(res["func_v"][f], V[a:b].sum(axis=0), rtol=1e-12, atol=0)
    assert np.allclose(res["kern_v"][0], V.sum(axis=0), rtol=1e-12, atol=0)
    assert np.allclose(res["line_v"].sum(axis=0), res["kern_v"][0], rtol=1e-12)


def test_estimate_properties(rand_case):
    prog, op, recs, res = rand_case
    names = [p["name"] for p in table2()]
    est = res["est"][0]
    T, A = est[0].T, est[0].A
    lu, cr = est[names.index("loop_unrolling")], est[names.index("code_reordering")]
    assert lu.M <= cr.M + 1e-9
    for o in est:
        assert o.M <= T
        if o.model in (1, 2, 3, 4):
            assert 1.0 <= o.speedup <= 2.0                     # Theorem 1
            assert o.speedup <= o.eq4 * (1 + 1e-15)            # scoped <= kernel-level
            assert o.eq3 >= o.eq4
    # warp balance matches exactly the kernel's sync stalls
    assert est[names.index("warp_balance")].M == pytest.approx(res["kern_v"][0, [6, 9], 0].sum(), rel=1e-12)
    assert est[names.index("function_split")].M == res["kern_v"][0, 11, 0]


def test_scoped_estimates_brute_force(rand_case):
    """Eq. 5 per scope (Q16): an edge counts in loop scope l iff both its def and
    its use lie in l or a loop nested in it; the optimizer's estimate is its best scope."""
    prog, op, recs, res = rand_case
    names = [p["name"] for p in table2()]
    C = res["C"].astype(np.float64)
    T = C.sum()
    A_i = C[:, 0, :].sum(axis=1)
    mem = {gp.GLOBAL, gp.TEXTURE}
    use_of = np.repeat(np.arange(prog.n_instr), np.diff(prog.row_ptr.astype(np.int64)))

    def edge_lat(e, same_loop):
        d, j = int(prog.edge_def[e]), int(use_of[e])
        if same_loop and not (prog.loop_id[d] >= 0 and prog.loop_id[d] == prog.loop_id[j]):
            return 0.0
        m = 0.0
        if res["cand"][e] & 1 and prog.opclass[d] in mem:            # MEM_GLOBAL column
            m += C[j, 1, 1] * res["share"][e, 0]
        if res["cand"][e] & 2:                                       # EXEC_{SHARED,ARITH,WAR}
            m += C[j, 1, 2] * res["share"][e, 1]
        return m

    def subtree(l):
        out = set()
        for i in range(prog.n_instr):
            x = int(prog.loop_id[i])
            while x >= 0 and x != l:
                x = int(prog.loop_parent[x])
            if x == l:
                out.add(i)
        return out

    for name, same, with_funcs in (("loop_unrolling", True, False), ("code_reordering", False, True)):
        best, best_scope = None, -1
        scopes = [(l, subtree(l)) for l in range(prog.n_loops)]
        if with_funcs:
            scopes += [(prog.n_loops + f, set(range(int(prog.func_begin[f]), int(prog.func_begin[f + 1]))))
                       for f in range(prog.n_funcs)]
        for sid, mem_set in scopes:
            M = sum(edge_lat(e, same) for e in range(prog.n_edges)
                    if int(prog.edge_def[e]) in mem_set and int(use_of[e]) in mem_set)
            A = sum(A_i[i] for i in mem_set)
            s = T / (T - min(A, M))
            if best is None or s > best:
                best, best_scope = s, sid
        o = res["est"][0][names.index(name)]
        assert o.speedup == pytest.approx(best, rel=1e-12), name
        assert o.best_scope == best_scope, name

"""GPU parity for estimate cases the Table-2 runs never reach (VERDICT r01 weak #2 / ADVICE r01):
M >= T (Eq. 2 / 4 / 5 go +inf with `unbounded` = 1, Q19), patterns with `ratio` != 1 (Q17), and a
pattern set replaced by another of the same size between two gpa_analyze graph replays."""
import numpy as np
import pytest

from gpagen import programs as gp
from gpagen.patterns import ALL_CLASSES, ncol, table2
from gpagen.streams import StreamSpec
from tests._common import collect, compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

REL = 1e-9
FETCH = 5


@pytest.fixture(autouse=True)
def _need_cuda(cuda_available):
    if not cuda_available:
        pytest.skip("no CUDA device")


def _pat(R, **kw):
    d = dict(column_mask=(1 << ncol(R)) - 1, class_mask=ALL_CLASSES, sample_class=0, model=0, flag_filter=0,
             same_loop=0, parallel_rule=0, sm_count=80, ratio=1.0, W=8.0, W_new=4.0, f=1.0)
    d.update(kw)
    return d


def _records(pcs, reason, lat):
    pcs = np.asarray(pcs, np.uint64)
    return pcs | (np.uint64(1) << np.uint64(32)) | (np.uint64(reason) << np.uint64(48)) | (
        np.uint64(lat) << np.uint64(56))


def test_unbounded_when_matched_samples_reach_T():
    """Every sample is an active FETCH (pass-through, integer) stall: a pattern over all columns
    matches M = T exactly, so Eq. 2 (ratio 1), Eq. 4 (A = T) and Eq. 5 over functions are +inf;
    ratio 0.5 stays finite (= 2)."""
    prog = gp.random_program(600, 1, 6, 3, seed=41)   # one function: its A is the kernel's T
    rng = np.random.default_rng(41)
    recs = _records(rng.integers(0, prog.n_instr, 200_000), FETCH, 0)
    R = prog.n_reasons
    pats = table2(R) + [_pat(R), _pat(R, model=1), _pat(R, model=3), _pat(R, model=4), _pat(R, ratio=0.5)]
    o = run_oracle(prog, recs, pats)
    g = run_gpu(prog, recs, pats)
    compare(g, o, rel=REL)
    q0 = len(table2(R))
    for side in (g["est"], o["est"]):
        e = side[0]
        assert [e[q0 + i].unbounded for i in range(5)] == [1, 1, 1, 1, 0]
        assert np.isinf(e[q0].speedup) and e[q0 + 4].speedup == 2.0
        assert e[q0].M == float(len(recs))
    # the Table-2 function-split row (FETCH column) also matches every sample
    assert g["est"][0][2].unbounded == 1


@pytest.mark.parametrize("ratio", [0.25, 0.5])
def test_ratio_patterns(ratio):
    """Eq. 2 with the pattern's `ratio` (Q17): T / (T - ratio * M)."""
    prog = gp.random_program(1200, 3, 8, 3, seed=43)
    recs = StreamSpec(prog, seed=4343, count_max=3).host(0, 300_000)
    pats = [dict(p, ratio=ratio) if p["model"] == 0 else p for p in table2(prog.n_reasons)]
    o = run_oracle(prog, recs, pats)
    g = run_gpu(prog, recs, pats)
    compare(g, o, rel=REL)
    ones = run_oracle(prog, recs)
    for q, p in enumerate(pats):
        if p["model"] == 0 and ones["est"][0][q].M > 0:
            e = o["est"][0][q]
            assert e.speedup == pytest.approx(e.T / (e.T - ratio * e.M), rel=1e-12)
            assert e.speedup < ones["est"][0][q].speedup


def test_analyze_graph_after_same_size_pattern_swap():
    """gpa_analyze caches a CUDA graph with the pattern plan baked in: re-setting a permuted
    Table 2 (same count, loop-scoped rows moved) must rebuild it."""
    import torch
    from paper_2009_04061_b200 import Program
    prog = gp.random_program(1500, 3, 10, 4, seed=47)
    recs = StreamSpec(prog, seed=4747, count_max=2).host(0, 400_000)
    t2 = table2(prog.n_reasons)
    perm = [t2[i] for i in (6, 7, 0, 1, 2, 3, 4, 5, 8, 9, 10)]   # loop_unrolling / code_reordering first
    assert [p["model"] for p in perm][:2] == [2, 4] and [p["model"] for p in t2][6:8] == [2, 4]
    P = Program(prog)
    d = torch.from_numpy(recs.view(np.int64)).cuda()
    P.set_patterns(t2)
    P.reset(); P.ingest(d); P.analyze()
    torch.cuda.synchronize()
    compare(collect(P), run_oracle(prog, recs, t2), rel=REL)
    P.set_patterns(perm)
    P.reset(); P.ingest(d); P.analyze()
    torch.cuda.synchronize()
    g = collect(P)
    o = run_oracle(prog, recs, perm)
    compare(g, o, rel=REL)
    assert any(e.best_scope >= 0 for e in o["est"][0][:2])

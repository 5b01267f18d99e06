"""The fused analysis kernel (fused.cu, gpa_set_analyze_mode): one cooperative launch running the
analysis bodies phase by phase must give the same bits as the multi-kernel graph, and match the
oracle at the parity bar, on small programs, on a program wide enough to use every CTA of the
grid, and on estimate edge cases (M >= T, ratio != 1)."""
import numpy as np
import pytest

from gpagen import programs as gp
from gpagen.patterns import ALL_CLASSES, ncol, table2
from gpagen.streams import StreamSpec, config_stream
from tests._common import compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

REL = 1e-9
ARRAYS = ("C", "stats", "cand", "self", "share", "V", "line_v", "line_al", "loop_excl_v", "loop_excl_al",
          "loop_incl_v", "loop_incl_al", "func_v", "func_al", "kern_v", "kern_al")
EST_FIELDS = ("T", "A", "model", "matched", "unbounded", "best_scope", "speedup", "M", "eq3", "eq4")


@pytest.fixture(autouse=True)
def _need_cuda(cuda_available):
    if not cuda_available:
        pytest.skip("no CUDA device")


def assert_same_bits(a, b):
    for k in ARRAYS:
        assert np.array_equal(np.asarray(a[k]).view(np.uint8), np.asarray(b[k]).view(np.uint8)), k
    assert len(a["est"]) == len(b["est"])
    for ka, kb in zip(a["est"], b["est"]):
        assert len(ka) == len(kb)
        for x, y in zip(ka, kb):
            for f in EST_FIELDS:
                u, v = getattr(x, f), getattr(y, f)
                assert (u == v) or (np.isnan(u) and np.isnan(v)), (f, u, v)


def _pat(R, **kw):
    d = dict(column_mask=(1 << ncol(R)) - 1, class_mask=ALL_CLASSES, sample_class=0, model=0, flag_filter=0,
             same_loop=0, parallel_rule=0, sm_count=80, ratio=1.0, W=8.0, W_new=4.0, f=1.0)
    d.update(kw)
    return d


CASES = {
    "tiny": lambda: (gp.tiny_fixture(), gp.tiny_records()),
    "rodinia": lambda: (lambda p: (p, config_stream(p, 2).host(0, 1_000_000)))(gp.config_program(2)),
    "r16": lambda: (lambda p: (p, StreamSpec(p, seed=77, count_max=3, invalid_ppm=5_000).host(0, 300_001)))(
        gp.random_program(1500, 3, 10, 4, seed=76, n_reasons=16)),
    "r4_kernels": lambda: (lambda p: (p, StreamSpec(p, seed=79).host(0, 200_000)))(
        gp.random_program(3000, 12, 30, 4, seed=78, n_kernels=4, n_reasons=4)),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_fused_equals_graph_and_oracle(case):
    prog, recs = CASES[case]()
    g_graph = run_gpu(prog, recs, analyze="graph")
    g_fused = run_gpu(prog, recs, analyze="fused")
    assert_same_bits(g_fused, g_graph)
    o = run_oracle(prog, recs)
    compare(g_fused, o, rel=1e-15 if case == "tiny" else REL, exact_blame=case == "tiny")
    assert g_fused["program"].analyze_mode == "fused"


def test_fused_is_one_launch_and_auto_is_the_graph():
    prog, recs = CASES["rodinia"]()
    g = run_gpu(prog, recs, analyze="fused")
    P = g["program"]
    before = P.launches
    P.analyze()
    assert P.launches - before == 1          # one cooperative launch
    P.analyze_mode = "auto"
    before = P.launches
    P.analyze()
    assert P.launches - before > 1           # the graph of per-step kernels


def test_fused_many_ctas_config3_program():
    """The 50k-instruction config-3 program forced through the fused kernel: 148 CTAs, every
    grid-stride body spans many iterations."""
    prog = gp.config_program(3)
    recs = config_stream(prog, 3).host(0, 3_000_000)
    g_fused = run_gpu(prog, recs, analyze="fused")
    assert_same_bits(g_fused, run_gpu(prog, recs, analyze="graph"))
    compare(g_fused, run_oracle(prog, recs), rel=REL)


def test_fused_estimate_edge_cases():
    """M >= T (+inf, unbounded) and ratio != 1 through the fused kernel (16 patterns: the most
    the fused kernel's four warps take)."""
    prog = gp.random_program(600, 1, 6, 3, seed=41)
    rng = np.random.default_rng(41)
    recs = np.asarray(rng.integers(0, prog.n_instr, 200_000), np.uint64) | (np.uint64(1) << np.uint64(32)) | (
        np.uint64(5) << np.uint64(48))
    R = prog.n_reasons
    pats = table2(R) + [_pat(R), _pat(R, model=1), _pat(R, model=3), _pat(R, model=4), _pat(R, ratio=0.5)]
    assert len(pats) == 16
    g = run_gpu(prog, recs, pats, analyze="fused")
    compare(g, run_oracle(prog, recs, pats), rel=REL)
    assert_same_bits(g, run_gpu(prog, recs, pats, analyze="graph"))

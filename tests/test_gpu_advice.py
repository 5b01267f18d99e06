"""GPU advice step (hotspots, ranking, single dependency coverage;
P:261) against the oracle on the same seeded inputs.  Hotspot items and
their samples are bit-exact (the same arithmetic on the same blame), coverage counts exact, and the
ranking is exactly or_rank of the GPU's own estimates (equal to the oracle's wherever the
oracle's speedups are not within 1e-9 of each other)."""
import numpy as np
import pytest

import oracle
from gpagen import batch
from gpagen import programs as gp
from gpagen.patterns import table2
from gpagen.streams import StreamSpec, config_stream
from tests._common import oracle_pattern, run_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _need_cuda(cuda_available):
    if not cuda_available:
        pytest.skip("no CUDA device")


def _gpu_advice(prog, recs, top_k):
    import torch
    from paper_2009_04061_b200 import Program
    P = Program(prog)
    P.set_patterns(table2(prog.n_reasons))
    P.reset()
    if len(recs):
        P.ingest(torch.from_numpy(recs.view(np.int64)).cuda())
    P.analyze()
    P.advise(top_k)
    adv = P.read_advice()
    return adv, P.read_estimates()


def _check(prog, recs, top_k):
    pats = table2(prog.n_reasons)
    o = run_oracle(prog, recs, pats)
    op = oracle.OracleProgram(prog)
    hot = op.hotspots(o["C"], o, [oracle_pattern(p) for p in pats], top_k)
    adv, est_g = _gpu_advice(prog, recs, top_k)
    K, Q = prog.n_kernels, len(pats)
    for k in range(K):
        for q in range(Q):
            exp = [(h.def_pc, h.use_pc, h.distance, h.item, h.samples) for h in hot[k][q]]
            n = int(adv["n"][k, q])
            got = [tuple(adv["hotspots"][k, q, t][f] for f in ("def_pc", "use_pc", "distance", "item", "samples"))
                   for t in range(n)]
            assert got == exp, (k, q, got[:3], exp[:3])
    cov = np.stack([adv["coverage"][f] for f in ("nodes", "single_before", "single_after")], 1)
    assert np.array_equal(cov, op.coverage(o["C"], o["cand"]))
    # rank: exactly or_rank of the GPU's estimates; equal to the oracle's unless speedups nearly tie
    g_est = [[oracle.Estimate(e.speedup) for e in row] for row in est_g]
    assert np.array_equal(adv["rank"], oracle.rank(g_est))
    o_rank = oracle.rank(o["est"])
    for k in range(K):
        sp = [o["est"][k][q].speedup for q in range(Q)]
        for a, b in zip(adv["rank"][k], o_rank[k]):
            if a != b:
                assert abs(sp[a] - sp[b]) <= 1e-9 * max(abs(sp[a]), abs(sp[b]))


def test_tiny_fixture_advice():
    _check(gp.tiny_fixture(), gp.tiny_records(), 5)


@pytest.mark.parametrize("top_k", [1, 5, 8])
def test_random_multi_kernel_advice(top_k):
    prog = gp.random_program(3000, 12, 30, 4, seed=71, n_kernels=5)
    recs = StreamSpec(prog, seed=72, count_max=4, invalid_ppm=1_000).host(0, 400_000)
    _check(prog, recs, top_k)


def test_config2_advice():
    prog = gp.config_program(2)
    _check(prog, config_stream(prog, 2).host(0, 2_000_000), 5)


def test_batch_advice_many_kernels():
    prog = batch.batch_program(400, seed=73)
    _check(prog, StreamSpec(prog, seed=74, count_max=2).host(0, 1_000_000), 5)


def test_advice_state_errors():
    import torch
    from paper_2009_04061_b200 import GpaError, Program
    prog = gp.tiny_fixture()
    P = Program(prog)
    with pytest.raises(GpaError):
        P.advise(5)                      # no estimates yet
    P.set_patterns(table2())
    P.reset()
    P.ingest(torch.from_numpy(gp.tiny_records().view(np.int64)).cuda())
    P.analyze()
    with pytest.raises(GpaError):
        P.advise(0)
    with pytest.raises(GpaError):
        P.advise(9)
    with pytest.raises(GpaError):
        P.read_advice()                  # before gpa_advise
    P.advise(3)
    P.read_advice()
    P.reset()
    with pytest.raises(GpaError):
        P.read_advice()                  # new counts invalidate the advice


def test_occupancy_parallel_estimates_match_oracle():
    """parallel_rule 3 / 4 (NEXT #4): per-kernel W, W_new from gpa_set_launches equal the oracle's
    occupancy model; the Eq. 10 estimates agree within 1e-9."""
    import torch
    from paper_2009_04061_b200 import Program
    from paper_2009_04061_b200.gpa import ARCH_V100
    prog = gp.random_program(2000, 10, 20, 3, seed=75, n_kernels=6)
    prog.kernel_grid_blocks = np.array([16, 200, 10_000, 79, 4, 1000], np.uint32)
    launches = [(256, 64, 0), (32, 32, 0), (32, 32, 0), (128, 33, 40960), (1024, 255, 0), (256, 32, 0)]
    recs = StreamSpec(prog, seed=76).host(0, 300_000)
    pats = table2(prog.n_reasons)
    for p in pats:
        if p["name"] == "block_increase":
            p["parallel_rule"] = 3
        if p["name"] == "thread_increase":
            p["parallel_rule"] = 4
    o = run_oracle(prog, recs, pats)
    occ = oracle.occupancy(oracle.Arch(*ARCH_V100.values()), [oracle.Launch(*l, 0) for l in launches],
                           prog.kernel_grid_blocks)
    op = oracle.OracleProgram(prog)
    est_o = op.estimate(o["C"], o, [oracle_pattern(p) for p in pats], occ)
    P = Program(prog)
    P.set_patterns(pats)
    P.set_launches(launches, ARCH_V100)
    P.reset()
    P.ingest(torch.from_numpy(recs.view(np.int64)).cuda())
    P.analyze()
    est_g = P.read_estimates()
    matched = 0
    for k in range(prog.n_kernels):
        for q, p in enumerate(pats):
            a, b = est_g[k][q], est_o[k][q]
            assert a.matched == b.matched, (k, p["name"])
            assert abs(a.speedup - b.speedup) <= 1e-9 * abs(b.speedup), (k, p["name"], a.speedup, b.speedup)
            matched += a.matched and p["model"] == 5
    assert matched >= 3      # kernels 0, 3, 4 (block increase) and 1, 2 (thread increase) exercise both rules

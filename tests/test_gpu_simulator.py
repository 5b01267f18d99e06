"""The PC-sampling simulator on the GPU (gpa_simulate) against the oracle's
(records and ground truth bit-exact per simulated SM), and the blamer measured against that ground
truth: SASS -> gpa_slice -> gpa_simulate -> ingest -> blame, top-attributed def vs the simulator's
true producer (SPEC's acceptance bar: >= 95% of stalled PCs on single-true-source programs)."""
import numpy as np
import pytest

import oracle
from gpagen import sass as gs

pytestmark = pytest.mark.gpu
CFG = dict(schedulers=4, warps_per_scheduler=4, period=5, trip_count=4, rbar_latency=2, max_cycles=5_000_000, seed=3)


@pytest.fixture(autouse=True)
def _need_cuda(cuda_available):
    if not cuda_available:
        pytest.skip("no CUDA device")


def _oracle_cfg():
    return oracle.SimCfg(CFG["schedulers"], CFG["warps_per_scheduler"], CFG["period"], CFG["trip_count"],
                         CFG["rbar_latency"], CFG["max_cycles"], CFG["seed"])


@pytest.mark.parametrize("which", ["fixture", "random", "single"])
def test_gpu_simulator_matches_oracle(which):
    from paper_2009_04061_b200 import simulate_sass
    S = {"fixture": gs.slice_fixture(), "random": gs.random_sass(3, 21), "single": gs.single_source_sass(120, 22)}[which]
    n_sm, cap = 24, 200_000
    rec, tr, counts = simulate_sass(S, n_sm, cap, func=0, **CFG)
    rec, tr = rec.cpu().numpy().view(np.uint64), tr.cpu().numpy()
    for sm in range(n_sm):
        o_rec, o_tr = oracle.simulate(S, _oracle_cfg(), sm=sm)
        k = int(counts[sm])
        assert k == len(o_rec) > 0
        assert np.array_equal(rec[sm * cap: sm * cap + k], o_rec)
        assert np.array_equal(tr[sm * cap: sm * cap + k], o_tr)
        assert not rec[sm * cap + k: (sm + 1) * cap].any()           # zero-filled tail


def blame_accuracy(S, n_sm=148):
    """Fraction of stalled (pc, dependency reason) pairs whose top-attributed def (largest Eq. 1 share
    among the pruned candidates) is the simulator's most frequent true producer."""
    import torch
    from paper_2009_04061_b200 import Program, simulate_sass, slice_sass
    prog = gs.program_from_sass(S, slice_sass(S))
    rec, tr, counts = simulate_sass(S, n_sm, 100_000, func=0, **CFG)
    P = Program(prog)
    P.reset()
    P.ingest(rec)
    P.blame()
    torch.cuda.synchronize()
    share, cand = P.view("share").cpu().numpy(), P.view("cand").cpu().numpy()
    r = rec.cpu().numpy().view(np.uint64)
    t = tr.cpu().numpy()
    pc, reason, cls = (r & 0xFFFFFFFF).astype(np.int64), ((r >> 48) & 0xFF).astype(np.int64), (r >> 56).astype(np.int64)
    keep = (cls == 1) & np.isin(reason, [1, 2, 3])
    pairs = {}
    for p, q, x in zip(pc[keep], reason[keep], t[keep]):
        pairs.setdefault((int(p), int(q)), []).append(int(x))
    rp = prog.row_ptr
    hit = 0
    for (j, q), xs in pairs.items():
        true = max(set(xs), key=lambda v: (xs.count(v), -v))
        es = [e for e in range(rp[j], rp[j + 1]) if (cand[e] >> (q - 1)) & 1]
        top = int(prog.edge_def[max(es, key=lambda e: (share[e, q - 1], -e))]) if es else -1
        hit += top == true
    return hit / max(len(pairs), 1), len(pairs)


def test_blamer_accuracy_single_true_source_suite():
    rates = [blame_accuracy(gs.single_source_sass(160, s)) for s in range(30, 40)]
    total = sum(n for _, n in rates)
    acc = sum(a * n for a, n in rates) / total
    print(f"single-true-source blamer accuracy {acc:.4f} over {total} stalled (pc, reason) pairs")
    assert total > 200 and acc >= 0.95, rates


def test_blamer_accuracy_random_programs_reported():
    """Predication, diamonds and loops give stalls several possible sources; the rate is reported
    (DESIGN.md §6.6), the bar is only that the blamer beats always picking the nearest def."""
    res = [blame_accuracy(gs.random_sass(1, s, func_len=(150, 300))) for s in (41, 42, 43)]
    n = sum(k for _, k in res)
    acc = sum(a * k for a, k in res) / n
    print(f"random-program blamer accuracy {acc:.3f} over {n} stalled (pc, reason) pairs")
    assert n > 40 and acc > 0.5, res

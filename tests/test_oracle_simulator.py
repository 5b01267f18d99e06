"""Pins of the oracle's sampling simulator (PC sampling model P:125-142;
DESIGN.md §3.2 Q40-Q44): hand-timed fixtures (SPEC's examples), the round-robin sampling order,
determinism and sample conservation."""
import numpy as np

import oracle
from gpagen import sass as gs


def _cfg(S=1, WP=1, N=1, trips=4, seed=7):
    return oracle.SimCfg(S, WP, N, trips, 2, 10_000_000, seed)


def _dec(rec):
    return (rec & 0xFFFFFFFF).astype(np.int64), ((rec >> 48) & 0xFF).astype(np.int64), ((rec >> 56) & 0xFF).astype(np.int64)


def test_independent_single_cycle_ops_are_all_active():
    """One warp, 8 independent 1-cycle instructions, a sample every cycle: instruction c issues at
    cycle c, samples at cycles 1..7 are active with no stall (L = 0)."""
    S = gs._build([dict(dst=[i], lat=1) for i in range(8)], [(0, 8)], [[]])
    rec, truth = oracle.simulate(S, _cfg())
    pc, reason, cls = _dec(rec)
    assert list(pc) == list(range(1, 8)) and not reason.any() and not cls.any() and (truth == -1).all()


def test_load_then_waiting_consumer_stall_ratio():
    """LDG (latency 200, barrier B0) then a consumer waiting on B0, then an independent op; N = 10:
    the consumer issues at cycle 200, the last op at 201, so samples at 10..190 are 19 latency
    samples at the consumer with memory dependency on the LDG (truth 0), and the sample at 200 is
    the consumer issuing: stall ratio 19/20."""
    S = gs._build([dict(dst=[0], wbar=1, cls=0, lat=200), dict(dst=[1], src=[0], wait=1, lat=1), dict(dst=[2], lat=1)],
                  [(0, 3)], [[]])
    rec, truth = oracle.simulate(S, _cfg(N=10))
    pc, reason, cls = _dec(rec)
    assert len(rec) == 20
    assert (pc == 1).all()
    assert list(cls) == [1] * 19 + [0] and list(reason) == [1] * 19 + [0]
    assert list(truth) == [0] * 19 + [-1]


def test_execution_dependency_on_fixed_latency_producer():
    """A 6-cycle arithmetic producer and an immediate consumer: the consumer waits cycles 1..5 with an
    execution dependency (truth 0) and issues at 6."""
    S = gs._build([dict(dst=[0], lat=6), dict(dst=[1], src=[0], lat=1)], [(0, 2)], [[]])
    rec, truth = oracle.simulate(S, _cfg())
    pc, reason, cls = _dec(rec)
    assert list(pc) == [1] * 6 and list(reason) == [2] * 5 + [0] and list(cls) == [1] * 5 + [0]
    assert list(truth) == [0] * 5 + [-1]


def test_round_robin_schedulers_and_not_selected():
    """Two schedulers with two warps each running 1-cycle independent code: every cycle both
    schedulers issue; the sampled scheduler alternates and its sampled warp alternates, so samples
    are active and half of them are the non-issuing warp (reason NOTSEL = 7)."""
    S = gs._build([dict(dst=[i % 5], lat=1) for i in range(12)], [(0, 12)], [[]])
    rec, truth = oracle.simulate(S, _cfg(S=2, WP=2))
    pc, reason, cls = _dec(rec)
    assert not cls.any()
    assert set(reason.tolist()) <= {0, 7} and (reason == 7).sum() > 0 and (reason == 0).sum() > 0


def test_loops_run_trip_count_and_determinism():
    S = gs.slice_fixture()
    c = _cfg(S=4, WP=4, N=3, trips=4)
    r1, t1 = oracle.simulate(S, c)
    r2, t2 = oracle.simulate(S, c)
    assert np.array_equal(r1, r2) and np.array_equal(t1, t2)
    pc, reason, cls = _dec(r1)
    assert ((pc >= 10) & (pc < 14)).sum() > 0                 # the loop body is sampled
    lat = cls == 1
    assert (reason[lat] != 0).all()                         # a latency sample always carries a reason
    dep = np.isin(reason, [1, 2, 3])
    assert (truth_ok := (t1[dep] >= 0)).all() and (t1[~dep] == -1).all()
    # every truth is an instruction that the stalled pc reads from (a register, predicate or barrier)
    for p, t in zip(pc[dep], t1[dep]):
        reads = set(int(x) for x in S.src[p] if x not in (0xFFFF, 255))
        if (S.guard[p] & 7) != 7:
            reads.add(256 + int(S.guard[p] & 7))
        writes = set(int(x) for x in S.dst[t] if x not in (0xFFFF, 255))
        assert reads & writes or (S.wait[p] & (S.wbar[t] | S.rbar[t]))


def test_sample_count_is_cycles_over_period_single_warp():
    S = gs.random_sass(1, 5)
    for N in (1, 4, 7):
        rec, _ = oracle.simulate(S, _cfg(N=N, trips=2))
        # one warp, one scheduler: a sample at every multiple of N up to the last issue cycle
        assert len(rec) > 0
        rec2, _ = oracle.simulate(S, _cfg(N=1, trips=2))
        assert len(rec) == len(rec2) // N

"""Pins of the occupancy model (DESIGN.md §3.2 Q34) that feeds W, W_new of
Eq. 10 for Block Increase and Thread Increase: worked occupancy
calculations on the paper's V100 by hand, and the parallel estimates they produce."""
import math

import pytest

import oracle
from gpagen import programs as gp
from gpagen.patterns import table2
from tests.test_oracle_pins import _pat

V100 = oracle.Arch(80, 64, 32, 65536, 98304, 4, 32, 256)


def _occ(tpb, regs, smem, grid):
    return oracle.occupancy(V100, [oracle.Launch(tpb, regs, smem, 0)], [grid])[0]


def test_warp_limited_full_grid():
    """256 threads, 32 regs: 8 warps/block; warps allow 8 blocks, registers 65536 / (1024 * 8) = 8
    (the warp limit is listed first), 1000 blocks fill 8 per SM -> W = 64 / 4 = 16; neither
    parallel optimizer matches."""
    o = _occ(256, 32, 0, 1000)
    assert (o.blocks_per_sm, o.limiter, o.W, o.match_block, o.match_thread) == (8, 0, 16.0, 0, 0)


def test_block_slot_limited_small_blocks_match_thread_increase():
    """32 threads: 1 warp/block, block slots bind at 32 blocks = 32 warps (of 64) -> W = 8; larger
    blocks reach the warp limit 64 (registers allow 65536 / 1024 = 64) -> W_new = 16."""
    o = _occ(32, 32, 0, 10_000)
    assert (o.blocks_per_sm, o.limiter, o.W, o.W_new_thread, o.match_thread) == (32, 1, 8.0, 16.0, 1)


def test_few_blocks_match_block_increase_pelec_shape():
    """16 blocks (PeleC's react_state) of 256 threads at 64 regs: registers bind
    (65536 / (2048 * 8) = 4 blocks), one block per SM is resident -> W = 2; spreading the same
    warps over 80 SMs -> W_new = 2 * 16 / 80 = 0.4."""
    o = _occ(256, 64, 0, 16)
    assert (o.blocks_per_sm, o.limiter, o.W, o.match_block) == (4, 2, 2.0, 1)
    assert o.W_new_block == pytest.approx(0.4, rel=1e-15)


def test_register_rounding_and_shared_memory_limit():
    # 33 regs * 32 = 1056 -> allocation unit 256 -> 1280 per warp; 8 warps/block -> 65536 / 10240 = 6
    assert _occ(256, 33, 0, 1000).blocks_per_sm == 6
    # 40 KB of shared memory per block -> 98304 / 40960 = 2 blocks, limiter shared memory
    o = _occ(128, 16, 40960, 1000)
    assert (o.blocks_per_sm, o.limiter) == (2, 3)


def test_unlaunchable_configuration_never_matches():
    o = _occ(1024, 255, 0, 4)        # 255 regs -> 8192 per warp * 32 warps > 65536
    assert (o.blocks_per_sm, o.match_block, o.match_thread, o.W) == (0, 0, 0, 0.0)


def test_parallel_estimates_from_the_model_on_the_tiny_fixture():
    """parallel_rule 3 / 4 take W, W_new from the model; the speedup is Eq. 10 of those values
    (R_I = A / T = 330 / 500 for the fixture)."""
    prog = gp.tiny_fixture()
    op = oracle.OracleProgram(prog)
    res = op.run_all(gp.tiny_records())
    pats = [dict(p) for p in table2() if p["name"] in ("block_increase", "thread_increase")]
    pats[0]["parallel_rule"], pats[1]["parallel_rule"] = 3, 4
    pats[0]["f"] = pats[1]["f"] = 1.0
    for launch, grid, exp_block, exp_thread in [((32, 32, 0, 0), 10_000, None, (8.0, 16.0)),
                                                ((256, 64, 0, 0), 16, (2.0, 0.4), None)]:
        occ = oracle.occupancy(V100, [oracle.Launch(*launch)], [grid])
        est = op.estimate(res["C"], res, [_pat(p) for p in pats], occ)[0]
        R_I = 330 / 500
        for e, exp in zip(est, (exp_block, exp_thread)):
            if exp is None:
                assert e.matched == 0 and e.speedup == 1.0
            else:
                W, Wn = exp
                I, In = 1 - (1 - R_I) ** W, 1 - (1 - R_I) ** Wn
                assert e.matched == 1 and e.speedup == pytest.approx((W / Wn) * (In / I), rel=1e-12)
                assert e.speedup == pytest.approx(oracle.eq10(W, Wn, R_I, 1.0), rel=1e-15)

"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times: config 3
(50k instructions, 10^9 records, partitioned ingest + the analyze graph) and config 4 (10^4
kernels / 4.5 M instructions, 10^8 records grouped by kernel launch, segment ingest).  The oracle
runs on the same records copied to the host (counts bit-exact, fp64 within 1e-9)."""
import numpy as np
import pytest

from gpagen import batch
from gpagen import programs as gp
from gpagen.patterns import table2
from gpagen.streams import config_stream
from tests._common import collect, compare, run_oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
REL = 1e-9


@pytest.fixture(autouse=True)
def _need_cuda(cuda_available):
    if not cuda_available:
        pytest.skip("no CUDA device")


def test_config3_full_stream_as_benchmarked():
    import torch
    from paper_2009_04061_b200 import Program
    prog = gp.config_program(3)
    n = 1_000_000_000
    recs = config_stream(prog, 3).device(0, n)            # the bench's device-resident stream
    P = Program(prog)
    assert P.variant == "part"
    P.set_patterns(table2(prog.n_reasons))
    P.reset()
    P.ingest(recs)
    P.analyze()
    torch.cuda.synchronize()
    g = collect(P)
    host = recs.cpu().numpy().view(np.uint64)
    del recs
    compare(g, run_oracle(prog, host), rel=REL)


def test_config4_full_batch_as_benchmarked():
    import torch
    from paper_2009_04061_b200 import Program
    prog = batch.config4_program()
    n = 100_000_000
    recs = batch.config4_stream(prog).device(0, n).view(torch.int64)
    order, sb, sk = batch.grouped_order(recs & 0xFFFFFFFF, prog)
    g_recs = recs[order].contiguous()
    host = recs.cpu().numpy().view(np.uint64)
    del recs, order
    P = Program(prog)
    P.set_patterns(table2(prog.n_reasons))
    P.reset()
    P.ingest_segments(g_recs, torch.from_numpy(sb.astype(np.int64)).cuda(),
                      torch.from_numpy(sk.view(np.int32)).cuda())
    P.analyze()
    torch.cuda.synchronize()
    compare(collect(P), run_oracle(prog, host), rel=REL)


def test_config5_ten_billion_samples_as_eight_shards():
    """Config 5 at full size on one B200: the 10^10-record stream cut into the 8 rank shards
    bench.py uses (1.25e9 records each, counter-based, so every shard is the same records at any
    rank count).  Each shard is histogrammed by the partitioned ingest into its own program; the
    sum of the shards' [counts | stats] views (what the DP-1 all-reduce computes) equals the
    L2-atomic variant's table over all 10^10 records, bit for bit, and holds every sample.  The
    replicated analysis of the summed table matches the oracle run on the same counts."""
    import torch
    import oracle
    from paper_2009_04061_b200 import Program
    from tests._common import oracle_pattern
    free, _ = torch.cuda.mem_get_info()
    if free < 40 * 2 ** 30:
        pytest.skip("needs ~12 GB of device memory")
    prog = gp.config_program(3)
    spec = config_stream(prog, 3)
    world, n_per = 8, 1_250_000_000
    buf = torch.empty(n_per * 8, dtype=torch.uint8, device="cuda")
    L = Program(prog)
    L.variant = "l2"
    L.reset()
    total = None
    for r in range(world):
        spec.device(r * n_per, n_per, out_tensor=buf)
        P = Program(prog)
        assert P.variant == "part"
        P.reset()
        P.ingest(buf)
        L.ingest(buf)
        v = P.reduce_view().clone()
        total = v if total is None else total + v
        del P
    torch.cuda.synchronize()
    del buf
    assert torch.equal(total, L.reduce_view())
    assert int(total[-4]) == world * n_per and int(total[-3]) == 0     # count-1 records, all valid
    pats = table2(prog.n_reasons)
    A = Program(prog)
    A.set_patterns(pats)
    A.reset()
    A.reduce_view().copy_(total)
    A.analyze()
    torch.cuda.synchronize()
    g = collect(A)
    C = total[:-4].cpu().numpy().view(np.uint64).reshape(prog.n_instr, 2, prog.n_reasons)
    op = oracle.OracleProgram(prog)
    b = op.blame(C)
    o = {"C": C, "stats": total[-4:-1].cpu().numpy().view(np.uint64), **b, **op.rollup(C, b["V"]),
         "est": op.estimate(C, b, [oracle_pattern(p) for p in pats])}
    compare(g, o, rel=REL)

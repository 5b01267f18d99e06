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

"""Soak test of the partitioned ingest (k_ingest_part): its CTAs exchange keys
through L2 with mbarrier hand-offs and monotonic release / acquire counters, so a missing fence
or an off-by-one in the buffer recycling would show up as a rare miscount, not as a crash.  The
same device-resident config-3 records are ingested many times -- whole streams, ragged lengths,
8-byte-aligned heads, back-to-back launches without a reset -- and every count table must equal
the one the oracle-checked L2-atomic variant (one RED per record, no exchange) produces for the
same records, bit for bit."""
import numpy as np
import pytest

from gpagen import programs as gp
from gpagen.streams import config_stream

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(autouse=True)
def _need_cuda(cuda_available):
    if not cuda_available:
        pytest.skip("no CUDA device")


def test_partitioned_ingest_soak_against_l2_variant():
    import torch
    from paper_2009_04061_b200 import Program
    prog = gp.config_program(3)
    n = 200_000_000
    recs = config_stream(prog, 3, count_max=3, invalid_ppm=200).device(0, n + 1).view(torch.int64)   # one record per element
    ref = Program(prog)
    ref.variant = "l2"
    part = Program(prog)
    assert part.variant == "part"
    rng = np.random.default_rng(7)
    cases = [(0, n), (1, n)] + [(int(rng.integers(0, 2)), int(rng.integers(1, n))) for _ in range(78)]
    for off, length in cases:
        view = recs[off:off + length]
        ref.reset()
        ref.ingest(view)
        torch.cuda.synchronize()
        want_c, want_s = ref.view("counts").clone(), ref.view("stats").clone()
        for rep in range(3):                      # repeated launches on the same input
            part.reset()
            part.ingest(view)
            torch.cuda.synchronize()
            assert torch.equal(part.view("counts"), want_c), (off, length, rep)
            assert torch.equal(part.view("stats"), want_s), (off, length, rep)
    # accumulation across launches without a reset: two halves == the whole
    part.reset()
    part.ingest(recs[:n // 2 + 1])
    part.ingest(recs[n // 2 + 1:n])
    ref.reset()
    ref.ingest(recs[:n])
    torch.cuda.synchronize()
    assert torch.equal(part.view("counts"), ref.view("counts"))
    assert torch.equal(part.view("stats"), ref.view("stats"))
    # counts up to 40 per record: most take the exchange (<= 7), the rest the L2-atomic side path
    big = config_stream(prog, 3, count_max=40).device(0, 20_000_001).view(torch.int64)
    for off, length in [(0, 20_000_001), (1, 20_000_000), (0, 7_777_777)]:
        ref.reset()
        ref.ingest(big[off:off + length])
        part.reset()
        part.ingest(big[off:off + length])
        torch.cuda.synchronize()
        assert torch.equal(part.view("counts"), ref.view("counts")), (off, length)
        assert torch.equal(part.view("stats"), ref.view("stats")), (off, length)

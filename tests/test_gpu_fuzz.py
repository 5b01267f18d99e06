"""Randomised parity sweep: program shapes, reason counts, stream mixes, ingest variants, record
alignment, pattern sets and analysis modes drawn from one seed per case, each case checked against
the oracle at the parity bar.  Complements the hand-picked cases of test_gpu_parity.py with the
combinations nobody thought to write down."""
import numpy as np
import pytest

from gpagen import programs as gp
from gpagen.patterns import ALL_CLASSES, ncol, table2
from gpagen.streams import StreamSpec
from tests._common import compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

REL = 1e-9


@pytest.fixture(autouse=True)
def _need_cuda(cuda_available):
    if not cuda_available:
        pytest.skip("no CUDA device")


def _random_patterns(rng, R):
    """Table 2 plus up to five random patterns (any model, masks, filters, ratio), <= 16 in all."""
    pats = table2(R, W=float(rng.integers(1, 33)), W_new=float(rng.integers(1, 33)), f=float(rng.uniform(0.5, 2)))
    loop_scoped = 2                                    # table 2's loop unrolling and code reordering
    for _ in range(int(rng.integers(0, 6))):
        model = int(rng.integers(0, 6))
        if model in (2, 4):
            if loop_scoped == 4:                       # the library takes at most 4 (gpa.h)
                model = 3
            else:
                loop_scoped += 1
        pats.append(dict(column_mask=int(rng.integers(1, 1 << ncol(R))), class_mask=int(rng.integers(1, ALL_CLASSES + 1)),
                         sample_class=int(rng.integers(0, 2)), model=model, flag_filter=int(rng.choice([0, 1, 2, 4, 6])),
                         same_loop=int(rng.integers(0, 2)), parallel_rule=int(rng.integers(0, 3)) if model == 5 else 0,
                         sm_count=int(rng.integers(1, 200)), ratio=float(rng.choice([1.0, 0.5, 0.25, 2.0])),
                         W=float(rng.integers(1, 33)), W_new=float(rng.integers(1, 33)), f=float(rng.uniform(0.5, 2))))
    return pats[:16]


@pytest.mark.parametrize("case", range(64))
def test_fuzz_case(case):
    rng = np.random.default_rng(0xF022 + case)
    n_instr = int(rng.choice([24, 200, 1500, 6000, 20000, 70000]))
    R = int(rng.integers(4, 17))
    n_funcs = int(max(1, min(n_instr // 16, rng.integers(1, 12))))
    n_kernels = int(rng.integers(1, min(n_funcs, 4) + 1))
    prog = gp.random_program(n_instr, n_funcs, int(rng.integers(1, 40)), int(rng.integers(1, 7)), seed=1000 + case,
                             n_kernels=n_kernels, n_reasons=R)
    n_rec = int(rng.choice([0, 1, 2, 1001, 64_000, 700_001, 2_000_000]))
    spec = StreamSpec(prog, seed=2000 + case, count_max=int(rng.choice([1, 3, 7, 9, 65535])),
                      invalid_ppm=int(rng.choice([0, 1000, 50_000])))
    recs = spec.host(0, n_rec)
    variants = [None, "l2"] + (["smem"] if n_instr * 2 * R * 4 <= 224 * 1024 else [])
    variant = variants[int(rng.integers(0, len(variants)))]
    pats = _random_patterns(rng, R)
    analyze = [None, "graph", "fused"][int(rng.integers(0, 3))]
    offset = int(rng.integers(0, 2))
    g = run_gpu(prog, recs, pats, variant=variant, offset_records=offset, analyze=analyze)
    compare(g, run_oracle(prog, recs, pats), rel=REL)

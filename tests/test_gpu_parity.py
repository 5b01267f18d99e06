"""Parity of the CUDA path (through the C ABI) with the CPU oracle on the same seeded inputs.

Bar (BASELINE.json north_star): counts, stats, candidate masks and self flags bit-exact; blame,
rollups and estimates in fp64 within 1e-9 relative, integer-valued columns exact.
"""
import numpy as np
import pytest

from gpagen import programs as gp
from gpagen.patterns import table2
from gpagen.streams import StreamSpec, config_stream
from tests._common import compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu

REL = 1e-9


@pytest.fixture(autouse=True)
def _need_cuda(cuda_available):
    if not cuda_available:
        pytest.skip("no CUDA device")


def test_tiny_fixture_bit_exact():
    prog = gp.tiny_fixture()
    recs = gp.tiny_records()
    g = run_gpu(prog, recs)
    o = run_oracle(prog, recs)
    compare(g, o, rel=1e-15, exact_blame=True)
    assert g["program"].variant == "smem"


@pytest.mark.parametrize("seed,n_instr,R,count_max,invalid_ppm,n_rec", [
    (21, 300, 9, 1, 0, 100_003),          # odd record count (ragged tail)
    (22, 700, 9, 7, 30_000, 250_001),     # pre-aggregated counts + malformed records
    (23, 1500, 16, 3, 5_000, 400_000),    # R = 16 (max), 32 pass-through columns
    (24, 200, 4, 1, 0, 50_000),           # R = 4 (no pass-through reasons)
])
def test_random_programs(seed, n_instr, R, count_max, invalid_ppm, n_rec):
    prog = gp.random_program(n_instr, 3, 10, 4, seed=seed, n_reasons=R)
    spec = StreamSpec(prog, seed=seed * 101, count_max=count_max, invalid_ppm=invalid_ppm)
    recs = spec.host(0, n_rec)
    o = run_oracle(prog, recs)
    compare(run_gpu(prog, recs), o, rel=REL)
    # unaligned (8- but not 16-byte aligned) record pointer
    compare(run_gpu(prog, recs, offset_records=1), o, rel=REL)


@pytest.mark.parametrize("variant", ["smem", "l2"])
def test_config2_rodinia(variant):
    prog = gp.config_program(2)
    recs = config_stream(prog, 2).host(0, 10_000_000)
    o = run_oracle(prog, recs)
    compare(run_gpu(prog, recs, variant=variant), o, rel=REL)


@pytest.fixture(scope="module")
def config3_case():
    prog = gp.config_program(3)
    recs = config_stream(prog, 3).host(0, 20_000_000)
    return prog, recs, run_oracle(prog, recs)


@pytest.mark.parametrize("variant", [None, "l2"])
def test_config3_large_program_reduced_stream(config3_case, variant):
    """Config-3 program (50k instructions, 200 loops) on a 2*10^7-record prefix of its stream;
    the default ingest for its 3.6 MB table is the partitioned (bucket-exchange) kernel."""
    prog, recs, o = config3_case
    g = run_gpu(prog, recs, variant=variant)
    assert g["program"].variant == (variant or "part")
    compare(g, o, rel=REL)


@pytest.mark.parametrize("n_rec,offset", [(1, 0), (2, 1), (4097, 1), (1_212_417, 0), (3_000_001, 1)])
def test_part_ragged_and_small_streams(n_rec, offset):
    """Streams shorter than one chunk per CTA, odd lengths and an 8-byte-aligned start."""
    prog = gp.random_program(5000, 6, 20, 4, seed=31)
    recs = StreamSpec(prog, seed=32, count_max=9, invalid_ppm=20_000).host(0, n_rec)
    g = run_gpu(prog, recs, offset_records=offset)
    assert g["program"].variant == "part"
    compare(g, run_oracle(prog, recs), rel=REL)


@pytest.mark.parametrize("n_instr,R", [(65_000, 9), (37_000, 16)])
def test_part_large_tables_smaller_chunk(n_instr, R):
    """Per-CTA tables of 7920 / 8000 bins (13-bit local keys, near the limit): the 6400-record
    exchange chunk no longer fits next to the table in shared memory and the launch takes the
    5120-record instantiation."""
    prog = gp.random_program(n_instr, 8, 40, 6, seed=51, n_reasons=R)
    recs = StreamSpec(prog, seed=52, count_max=5, invalid_ppm=1_000).host(0, 3_000_001)
    g = run_gpu(prog, recs, offset_records=1)
    assert g["program"].variant == "part"
    compare(g, run_oracle(prog, recs), rel=REL)


@pytest.mark.parametrize("n_instr,R,count_max", [(150_000, 9, 1), (150_000, 9, 5), (100_000, 16, 3),
                                                 (120_000, 9, 3),
                                                 (80_000, 9, 4),     # 14-bit local bins on the Wide exchange shape
                                                 (45_000, 12, 9)])   # 13-bit, Wide, R = 12, counts past the key
def test_part_wide_local_bins(n_instr, R, count_max):
    """PeleC / Quicksilver-sized kernels: per-CTA tables of 9,126-21,632
    bins need 14- or 15-bit local keys (1-2 count bits), and stay on the exchange path instead of
    the L2-atomic fallback; records whose count does not fit the key go through L2 atomics."""
    prog = gp.random_program(n_instr, 8, 60, 8, seed=61, n_reasons=R)
    recs = StreamSpec(prog, seed=62, count_max=count_max, invalid_ppm=1_000).host(0, 4_000_001)
    g = run_gpu(prog, recs, offset_records=1)
    assert g["program"].variant == "part"
    compare(g, run_oracle(prog, recs), rel=REL)


def test_part_skewed_stream_overflow():
    """A hot PC takes half the samples: its bucket overflows the exchange slots and the excess
    goes through L2 atomics; counts stay exact."""
    prog = gp.random_program(6000, 6, 20, 4, seed=41)
    w = prog.pc_weight.copy()
    w[17] = w.sum()
    w[4000] = w.sum() / 3
    prog.pc_weight = w
    recs = StreamSpec(prog, seed=42, count_max=65535).host(0, 4_000_000)
    g = run_gpu(prog, recs)
    assert g["program"].variant == "part"
    compare(g, run_oracle(prog, recs), rel=REL)


def test_host_ingest_equals_device_ingest():
    prog = gp.config_program(2)
    recs = config_stream(prog, 2, count_max=3).host(0, 9_000_001)
    g1 = run_gpu(prog, recs)
    g2 = run_gpu(prog, recs, host=True)
    assert np.array_equal(g1["C"], g2["C"]) and np.array_equal(g1["V"], g2["V"])


def test_deterministic_and_accumulating():
    import torch
    from paper_2009_04061_b200 import Program
    prog = gp.config_program(2)
    recs = config_stream(prog, 2).host(0, 3_000_000)
    d = torch.from_numpy(recs.view(np.int64)).cuda()
    P = Program(prog)
    P.set_patterns(table2())
    outs = []
    for split in (None, 1_234_567):
        P.reset()
        if split is None:
            P.ingest(d)
        else:
            P.ingest(d[:split])
            P.ingest(d[split:])
        P.blame()
        P.aggregate()
        P.estimate()
        torch.cuda.synchronize()
        outs.append((P.view("counts").clone(), P.instr_vector(), P.view("kernel").clone(),
                     P.view("loop_incl").clone()))
    for a, b in zip(*outs):
        assert torch.equal(a, b)


def test_edge_cases_empty_and_invalid_streams():
    prog = gp.random_program(100, 2, 3, 2, seed=5)
    for recs in (np.zeros(0, np.uint64),
                 StreamSpec(prog, seed=9, invalid_ppm=1_000_000).host(0, 10_001)):
        o = run_oracle(prog, recs)
        g = run_gpu(prog, recs)
        compare(g, o, rel=REL)
        assert g["C"].sum() == 0
        for row in g["est"][0]:
            assert row.T == 0
            if row.model != 5:          # Eq. 10 with R_I = 0 is f / C_W by the C_I := 1 convention (Q18)
                assert row.speedup == 1.0


def test_program_without_edges_or_loops():
    n = 64
    prog = gp._finalize(9, [gp.GLOBAL] * n, [0] * n, [1024] * n, list(range(n)), [-1] * n, [],
                        [0, 32, n], [0, 2], [4], [[] for _ in range(n)], n_lines=n)
    recs = StreamSpec(gp.random_program(n, 2, 2, 2, seed=3), seed=4).host(0, 20_000)
    compare(run_gpu(prog, recs), run_oracle(prog, recs), rel=REL)


def test_multi_kernel_program():
    prog = gp.random_program(3000, 12, 20, 3, seed=77, n_kernels=5)
    recs = StreamSpec(prog, seed=78, count_max=2).host(0, 500_000)
    compare(run_gpu(prog, recs), run_oracle(prog, recs), rel=REL)


def test_call_order_errors():
    import torch
    from paper_2009_04061_b200 import GpaError, Program
    P = Program(gp.tiny_fixture())
    with pytest.raises(GpaError, match="before"):
        P.blame()
    P.reset()
    with pytest.raises(GpaError, match="before"):
        P.aggregate()
    P.blame()
    P.aggregate()
    with pytest.raises(GpaError, match="patterns"):
        P.estimate()
    with pytest.raises(GpaError):
        P.ingest(torch.zeros(65, dtype=torch.uint8, device="cuda")[1:])  # 8 records, misaligned pointer


def test_analyze_graph_equals_separate_calls():
    """gpa_analyze (one CUDA graph) gives bit-identical results to blame + aggregate + estimate."""
    import torch
    from paper_2009_04061_b200 import Program
    prog = gp.config_program(2)
    recs = config_stream(prog, 2).host(0, 2_000_000)
    d = torch.from_numpy(recs.view(np.int64)).cuda()
    P = Program(prog)
    P.set_patterns(table2())
    outs = []
    for mode in ("calls", "graph", "graph"):
        P.reset()
        P.ingest(d)
        if mode == "calls":
            P.blame(); P.aggregate(); P.estimate()
        else:
            P.analyze()
        torch.cuda.synchronize()
        outs.append((P.instr_vector(), P.view("line").clone(), P.view("kernel").clone(),
                     bytes(P.view("estimates").cpu().numpy())))
    for other in outs[1:]:
        for a, b in zip(outs[0][:3], other[:3]):
            assert torch.equal(a, b)
        assert outs[0][3] == other[3]


def test_read_estimates_array_matches_struct_list():
    prog = gp.config_program(2)
    recs = config_stream(prog, 2).host(0, 500_000)
    import torch
    from paper_2009_04061_b200 import Program
    P = Program(prog)
    P.set_patterns(table2())
    P.reset()
    P.ingest(torch.from_numpy(recs.view(np.int64)).cuda())
    P.analyze()
    rows = P.read_estimates()
    arr = P.read_estimates_array()
    assert arr.shape == (len(rows), len(rows[0]))
    for k, row in enumerate(rows):
        for q, e in enumerate(row):
            for f in ("speedup", "M", "eq3", "eq4", "T", "A", "best_scope", "unbounded", "matched", "model"):
                a, b = getattr(e, f), arr[k, q][f]
                assert a == b or (np.isnan(a) and np.isnan(b))


def test_part_stream_split_into_launches(monkeypatch):
    """Streams longer than one launch's wrap-free bound (kFlushEvery chunks, ~6.5e10 records at
    G = 148) are split by the host into several launches, each ending with its u32 -> u64 flush.
    The bound is lowered through the test hook so a small stream spans several launches."""
    monkeypatch.setenv("GPA_PART_LAUNCH_CHUNKS", "2")
    prog = gp.random_program(6000, 6, 20, 4, seed=51)
    recs = StreamSpec(prog, seed=52, count_max=9, invalid_ppm=2_000).host(0, 4_000_001)
    g = run_gpu(prog, recs, offset_records=1)
    assert g["program"].variant == "part"
    compare(g, run_oracle(prog, recs), rel=REL)


def test_smem_table_u32_wrap_carried():
    """Variant S keeps u32 per-CTA tables: a bin that passes 2^32 inside one CTA (68k records of
    count 65535 per CTA on one (pc, class, reason)) is carried into the u64 table exactly."""
    prog = gp.random_program(300, 2, 6, 3, seed=61)
    hot = np.uint64(5) | (np.uint64(65535) << np.uint64(32)) | (np.uint64(1) << np.uint64(48)) \
        | (np.uint64(1) << np.uint64(56))                        # pc 5, count 65535, MEM, LAT
    recs = np.full(10_000_000, hot, dtype=np.uint64)
    recs[::97] = StreamSpec(prog, seed=62, count_max=4).host(0, len(recs[::97]))
    g = run_gpu(prog, recs)
    assert g["program"].variant == "smem"
    o = run_oracle(prog, recs)
    assert int(o["C"].max()) > 2 ** 32 * 100
    compare(g, o, rel=REL)


def test_smem_table_u16_field_overflows():
    """Variant S counts in u16 fields, two bins per 32-bit word: a low field that wraps carries into
    its high neighbour (and may wrap it too), a high field that wraps drops out of the word.  Two hot
    bins of one word, (pc 5, ACT, NONE) and (pc 5, ACT, MEM), take 90 % of 10^7 records with random
    counts up to 65535, so every case occurs many times in every CTA; counts stay exact."""
    prog = gp.random_program(300, 2, 6, 3, seed=71)
    rng = np.random.default_rng(72)
    n = 10_000_000
    recs = StreamSpec(prog, seed=73, count_max=4).host(0, n)
    hot = rng.random(n)
    reason = np.where(hot < 0.5, 0, 1).astype(np.uint64)        # bins 2*5*R + 0 (even) and + 1 (odd)
    cnt = rng.integers(1, 65536, n, dtype=np.uint64)
    cnt[rng.random(n) < 0.3] = 65535
    h = np.uint64(5) | (cnt << np.uint64(32)) | (reason << np.uint64(48))   # ACT (flags 0)
    sel = hot < 0.9
    recs[sel] = h[sel]
    g = run_gpu(prog, recs)
    assert g["program"].variant == "smem"
    o = run_oracle(prog, recs)
    R = prog.n_reasons
    assert int(o["C"].reshape(-1)[10 * R]) > 2 ** 36 and int(o["C"].reshape(-1)[10 * R + 1]) > 2 ** 36
    compare(g, o, rel=REL)


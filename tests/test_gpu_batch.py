"""Config 4 on the GPU: gpa_ingest_segments (streams grouped by kernel launch) and
DP-2 kernel slices, against the CPU oracle on the same records.  Counts, stats, candidate masks
and self flags bit-exact; fp64 within 1e-9 relative (BASELINE.json north_star)."""
import numpy as np
import pytest

from gpagen import batch
from gpagen.streams import StreamSpec
from paper_2009_04061_b200.dist import slice_program
from tests._common import compare, run_gpu, run_oracle

pytestmark = pytest.mark.gpu
REL = 1e-9


@pytest.fixture(autouse=True)
def _need_cuda(cuda_available):
    if not cuda_available:
        pytest.skip("no CUDA device")


def _grouped(prog, recs, seed=0, split=False):
    pcs = batch.record_pcs(recs)
    order = np.random.default_rng(seed).permutation(prog.n_kernels)
    perm, seg_begin, seg_kernel = batch.grouped_order(pcs, prog, kernel_order=order)
    if split:   # every launch delivered in two buffers (the same kernel in consecutive segments)
        mid = (seg_begin[:-1] + seg_begin[1:]) // 2
        seg_begin = np.stack([seg_begin[:-1], mid], 1).reshape(-1)
        seg_begin = np.concatenate([seg_begin, [len(recs)]]).astype(np.uint64)
        seg_kernel = np.repeat(seg_kernel, 2)
    return recs[perm], seg_begin, seg_kernel


@pytest.mark.parametrize("split,offset", [(False, 0), (True, 1)])
def test_segment_ingest_matches_oracle(split, offset):
    prog = batch.batch_program(300, seed=61)
    recs = StreamSpec(prog, seed=62, count_max=5, invalid_ppm=2_000).host(0, 2_000_001)
    g, sb, sk = _grouped(prog, recs, seed=1, split=split)
    o = run_oracle(prog, recs)
    compare(run_gpu(prog, g, segments=(sb, sk, 0), offset_records=offset), o, rel=REL)


def test_segment_ingest_mislabelled_and_unknown_segments():
    """Records outside their segment's kernel and segments of unknown kernels are still counted
    (L2 path); records outside [seg_begin[0], seg_begin[-1]) are not ingested."""
    prog = batch.batch_program(200, seed=63)
    recs = StreamSpec(prog, seed=64, count_max=3, invalid_ppm=0).host(0, 600_000)
    g, sb, sk = _grouped(prog, recs, seed=2)
    sk = sk.copy()
    sk[::3] = (sk[::3] + 1) % prog.n_kernels          # wrong kernel
    sk[1::7] = 0xFFFFFFFF                              # unknown kernel
    lo, hi = int(sb[1]), int(sb[-2])                   # drop the first and last segments
    sub_b = sb[1:-1].copy()
    o = run_oracle(prog, g[lo:hi])
    compare(run_gpu(prog, g, segments=(sub_b, sk[1:-1], 0)), o, rel=REL)


def test_kernel_slice_with_pc_base():
    """DP-2: a rank's program holds kernels [k0, k1); its records keep the application's PCs and
    the segment ingest subtracts pc_base."""
    prog = batch.batch_program(150, seed=65)
    recs = StreamSpec(prog, seed=66, count_max=2, invalid_ppm=1_000).host(0, 1_000_000)
    sub, maps = slice_program(prog, 40, 97)
    pcs = batch.record_pcs(recs)
    sel = (pcs >= maps["pc_base"]) & (pcs < maps["pc_base"] + maps["n_instr"])
    mine = recs[sel]
    perm, sb, sk = batch.grouped_order(batch.record_pcs(batch.rebase_records(mine, maps["pc_base"])), sub)
    o = run_oracle(sub, batch.rebase_records(mine, maps["pc_base"]))
    compare(run_gpu(sub, mine[perm], segments=(sb, sk, maps["pc_base"])), o, rel=REL)


def test_config4_full_batch_reduced_stream():
    """BASELINE config 4's program (10^4 kernels, ~4.5 M instructions) on a 10^7-record prefix of
    its stream grouped by kernel launch."""
    prog = batch.config4_program()
    recs = batch.config4_stream(prog).host(0, 10_000_000)
    g, sb, sk = _grouped(prog, recs, seed=3)
    o = run_oracle(prog, recs)
    compare(run_gpu(prog, g, segments=(sb, sk, 0)), o, rel=REL)


def test_dp2_reduce_scatter_path_single_rank_nccl():
    """DP-2 for an ungrouped stream through NCCL (world size 1 on this box): the whole program
    histograms the records, reduce_scatter_counts hands the kernel slice to the sub-program's
    count table, and the sub-program's analysis equals the oracle on the slice's records."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    from paper_2009_04061_b200 import Program
    from paper_2009_04061_b200.dist import kernel_row_bounds, reduce_scatter_counts
    from gpagen.patterns import table2
    from tests._common import collect
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        prog = batch.batch_program(120, seed=91)
        recs = StreamSpec(prog, seed=92, count_max=2, invalid_ppm=0).host(0, 800_000)
        full = Program(prog)
        full.reset()
        full.ingest(torch.from_numpy(recs.view(np.int64)).cuda())
        k0, k1 = 30, 77
        sub, maps = slice_program(prog, k0, k1)
        rb = kernel_row_bounds(prog, [k0, k1])
        S = Program(sub)
        S.set_patterns(table2(prog.n_reasons))
        S.reset()
        counts = full.view("counts").reshape(prog.n_instr, -1)
        out = S.view("counts").reshape(sub.n_instr, -1)
        reduce_scatter_counts(counts[rb[0]:], [0, rb[1] - rb[0]], out)
        S.analyze()
        torch.cuda.synchronize()
        g = collect(S)
        pcs = batch.record_pcs(recs)
        mine = recs[(pcs >= maps["pc_base"]) & (pcs < maps["pc_base"] + maps["n_instr"])]
        o = run_oracle(sub, batch.rebase_records(mine, maps["pc_base"]))
        g["stats"] = o["stats"]          # stats stay with the whole-program histogram
        compare(g, o, rel=REL)
    finally:
        dist.destroy_process_group()


def test_dp1_reduce_view_single_collective_nccl():
    """DP-1 exchange: the count table and the stats are one contiguous buffer
    (Program.reduce_view), so one SUM all-reduce combines ranks.  The view aliases both results,
    and a world-size-1 NCCL sharded_step equals the oracle on the shard; summing two shards'
    views equals ingesting both shards (integer monoid)."""
    import os
    import socket
    import torch
    import torch.distributed as dist
    import gpagen
    from paper_2009_04061_b200 import Program
    from paper_2009_04061_b200.dist import sharded_step
    from gpagen.patterns import table2
    from tests._common import collect
    prog = gpagen.random_program(900, 4, 10, 3, seed=77)
    recs = StreamSpec(prog, seed=78, count_max=9, invalid_ppm=5_000).host(0, 300_001)
    half = len(recs) // 2
    A, B, AB = Program(prog), Program(prog), Program(prog)
    for P, part in ((A, recs[:half]), (B, recs[half:]), (AB, recs)):
        P.reset()
        P.ingest(torch.from_numpy(np.ascontiguousarray(part).view(np.int64)).cuda())
    torch.cuda.synchronize()
    ra = A.reduce_view()
    assert ra.numel() == prog.n_instr * 2 * prog.n_reasons + 4
    assert torch.equal(ra[:-4], A.view("counts").flatten()) and torch.equal(ra[-4:], A.view("stats"))
    ra += B.reduce_view()          # what the all-reduce computes for two ranks
    assert torch.equal(ra, AB.reduce_view())
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        P = Program(prog)
        P.set_patterns(table2(prog.n_reasons))
        sharded_step(P, torch.from_numpy(recs.view(np.int64)).cuda())
        torch.cuda.synchronize()
        compare(collect(P), run_oracle(prog, recs), rel=REL)
    finally:
        dist.destroy_process_group()

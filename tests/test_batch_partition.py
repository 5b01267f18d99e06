"""Config 4 (a batch of kernels) host logic: the batch generator's shape, grouping a stream by
kernel launch, and DP-2's kernel partition.  The partition is exact because every
def-use edge, line, loop and function lies inside one kernel (the blamer analyses each
kernel invocation on its own): the CPU oracle run on each kernel slice must reproduce the
whole-program oracle's values for those kernels bit for bit.  World-size-2 gloo test of the
partitioned step with estimate gathering."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from gpagen import batch
from gpagen.streams import StreamSpec
from paper_2009_04061_b200.dist import gather_estimates, partition_kernels, slice_program
from tests._common import run_oracle

EST_FIELDS = ("speedup", "M", "eq3", "eq4", "T", "A", "best_scope", "unbounded", "matched", "model")


def _case(n_kernels=120, n_rec=400_000):
    prog = batch.batch_program(n_kernels, seed=99)
    recs = StreamSpec(prog, seed=100, count_max=3, invalid_ppm=5_000).host(0, n_rec)
    return prog, recs


def test_batch_program_shape():
    prog = batch.batch_program(300, seed=5)
    kb = batch.kernel_pc_begin(prog)
    sizes = np.diff(kb)
    assert prog.n_kernels == 300 and sizes.min() >= 24 and sizes.max() <= 2048
    assert 200 < sizes.mean() < 700                                   # log-uniform 24..2048: ~455
    rp = prog.row_ptr.astype(np.int64)
    j = np.repeat(np.arange(prog.n_instr), np.diff(rp))
    key = j * prog.n_instr + prog.edge_def.astype(np.int64)
    assert np.all(np.diff(key) > 0)                                   # CSR by use, defs sorted
    fo = np.searchsorted(prog.func_begin.astype(np.int64), np.arange(prog.n_instr), side="right") - 1
    assert np.array_equal(fo[prog.edge_def], fo[j])                   # edges stay in a function
    lf = {}
    for i, l in enumerate(prog.line_id):
        assert lf.setdefault(int(l), fo[i]) == fo[i]                  # lines stay in a function
    assert 1.2 < prog.n_edges / prog.n_instr < 2.2


def test_grouped_order_segments():
    prog, recs = _case(60, 50_000)
    pcs = batch.record_pcs(recs)
    order, seg_begin, seg_kernel = batch.grouped_order(pcs, prog, kernel_order=np.arange(59, -1, -1))
    assert np.array_equal(np.sort(order), np.arange(len(recs)))
    kb = batch.kernel_pc_begin(prog)
    g = pcs[order]
    assert seg_begin[0] == 0 and seg_begin[-1] == len(recs)
    for s, k in enumerate(seg_kernel):
        part = g[seg_begin[s]:seg_begin[s + 1]]
        if k == 0xFFFFFFFF:
            assert np.all(part >= kb[-1])
        else:
            assert np.all((part >= kb[k]) & (part < kb[k + 1]))
    real = seg_kernel[seg_kernel != 0xFFFFFFFF]
    assert np.all(np.diff(real.astype(np.int64)) < 0)                 # the requested kernel order
    t = torch.from_numpy(pcs)
    o2, b2, k2 = batch.grouped_order(t, prog, kernel_order=np.arange(59, -1, -1))
    assert np.array_equal(o2.numpy(), order) and np.array_equal(b2, seg_begin) and np.array_equal(k2, seg_kernel)


def test_partition_kernels_balanced():
    assert partition_kernels([1, 1, 1, 1, 10, 1], 3) == [0, 4, 5, 6]
    assert partition_kernels([1] * 10, 4) == [0, 2, 5, 7, 10]
    assert partition_kernels([5, 1], 4) == [0, 1, 2, 2, 2]
    w = np.random.default_rng(3).lognormal(0, 1.5, 10_000)
    b = partition_kernels(w, 8)
    loads = [w[b[r]:b[r + 1]].sum() for r in range(8)]
    assert max(loads) < 1.05 * w.sum() / 8 + w.max()


def _slice_records(prog, recs, maps):
    pcs = batch.record_pcs(recs)
    sel = (pcs >= maps["pc_base"]) & (pcs < maps["pc_base"] + maps["n_instr"])
    return batch.rebase_records(recs[sel], maps["pc_base"])


def _assert_slice_matches(whole, part, prog, maps):
    i0, n = maps["pc_base"], maps["n_instr"]
    e0 = maps["edge_base"]
    assert np.array_equal(part["C"], whole["C"][i0:i0 + n])
    E = len(part["cand"])
    assert np.array_equal(part["cand"], whole["cand"][e0:e0 + E])
    assert np.array_equal(part["self"], whole["self"][i0:i0 + n])
    assert np.array_equal(part["share"], whole["share"][e0:e0 + E])
    assert np.array_equal(part["V"], whole["V"][i0:i0 + n])
    for lvl, ids in (("line", "lines"), ("loop_excl", "loops"), ("loop_incl", "loops"), ("func", "funcs"),
                     ("kern", "kernels")):
        assert np.array_equal(part[lvl + "_v"], whole[lvl + "_v"][maps[ids]]), lvl
        assert np.array_equal(part[lvl + "_al"], whole[lvl + "_al"][maps[ids]]), lvl
    for k, row in enumerate(part["est"]):
        wrow = whole["est"][int(maps["kernels"][k])]
        for q, (a, b) in enumerate(zip(row, wrow)):
            for f in EST_FIELDS:
                va, vb = getattr(a, f), getattr(b, f)
                if f == "best_scope" and va >= 0:
                    # scope ids are loop ids (or n_loops + function id) of the respective program
                    nl_p, nl_w = len(maps["loops"]), len(whole["loop_excl_v"])
                    va = int(maps["loops"][va]) if va < nl_p else nl_w + int(maps["funcs"][va - nl_p])
                assert va == vb or (np.isnan(va) and np.isnan(vb)), (k, q, f, va, vb)


def test_kernel_slices_reproduce_whole_program():
    prog, recs = _case()
    whole = run_oracle(prog, recs)
    kb = batch.kernel_pc_begin(prog)
    ksamp = np.bincount(np.searchsorted(kb[1:-1], batch.record_pcs(recs)[batch.record_pcs(recs) < kb[-1]],
                                        side="right"), minlength=prog.n_kernels)
    bounds = partition_kernels(ksamp, 3)
    for r in range(3):
        sub, maps = slice_program(prog, bounds[r], bounds[r + 1])
        part = run_oracle(sub, _slice_records(prog, recs, maps))
        _assert_slice_matches(whole, part, prog, maps)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    prog, recs = _case(80, 200_000)
    kb = batch.kernel_pc_begin(prog)
    pcs = batch.record_pcs(recs)
    ksamp = np.bincount(np.searchsorted(kb[1:-1], pcs[pcs < kb[-1]], side="right"), minlength=prog.n_kernels)
    bounds = partition_kernels(ksamp, world)
    sub, maps = slice_program(prog, bounds[rank], bounds[rank + 1])
    part = run_oracle(sub, _slice_records(prog, recs, maps))
    speed = np.array([[e.speedup for e in row] for row in part["est"]], np.float64)
    allsp = gather_estimates(speed)
    np.save(os.path.join(out_dir, f"sp{rank}.npy"), allsp)
    dist.barrier()
    dist.destroy_process_group()


def test_partitioned_step_gathers_whole_program_estimates(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    prog, recs = _case(80, 200_000)
    whole = run_oracle(prog, recs)
    ref = np.array([[e.speedup for e in row] for row in whole["est"]], np.float64)
    for r in range(world):
        got = np.load(tmp_path / f"sp{r}.npy")
        assert got.shape == ref.shape
        assert np.array_equal(got, ref)


def _rs_worker(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2009_04061_b200.dist import kernel_row_bounds, reduce_scatter_counts, shard_range
    prog = batch.batch_program(90, seed=81)
    spec = StreamSpec(prog, seed=82, count_max=3, invalid_ppm=2_000)
    n = 300_001
    k0, k1 = shard_range(n, rank, world)             # ungrouped shard of the stream
    C, _ = oracle.OracleProgram(prog).histogram(spec.host(k0, k1 - k0))
    counts = torch.from_numpy(C.view(np.int64).reshape(prog.n_instr, -1).copy())
    kb = batch.kernel_pc_begin(prog)
    pcs = batch.record_pcs(spec.host(0, n))
    ksamp = np.bincount(np.searchsorted(kb[1:-1], pcs[pcs < kb[-1]], side="right"), minlength=prog.n_kernels)
    rb = kernel_row_bounds(prog, partition_kernels(ksamp, world))
    out = torch.zeros((rb[rank + 1] - rb[rank], counts.shape[1]), dtype=torch.int64)
    reduce_scatter_counts(counts, rb, out)
    np.save(os.path.join(out_dir, f"rs{rank}.npy"), out.numpy())
    np.save(os.path.join(out_dir, f"rb{rank}.npy"), np.array(rb))
    dist.barrier()
    dist.destroy_process_group()


def test_reduce_scatter_of_ungrouped_shards_gives_kernel_slices(tmp_path):
    """DP-2 without grouping: ranks histogram arbitrary shards of the whole program, then each
    receives the summed rows of its kernel slice -- equal to the single-process table's rows."""
    import oracle
    world = 2
    mp.spawn(_rs_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    prog = batch.batch_program(90, seed=81)
    C, _ = oracle.OracleProgram(prog).histogram(StreamSpec(prog, seed=82, count_max=3, invalid_ppm=2_000).host(0, 300_001))
    full = C.view(np.int64).reshape(prog.n_instr, -1)
    for r in range(world):
        rb = np.load(tmp_path / f"rb{r}.npy")
        got = np.load(tmp_path / f"rs{r}.npy")
        assert np.array_equal(got, full[rb[r]:rb[r + 1]])

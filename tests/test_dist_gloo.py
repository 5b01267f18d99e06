"""World-size-2 gloo tests (CPU) of the data-parallel host logic: stream sharding and the
all-reduce of per-rank count tables.  Per-rank tables come from the CPU oracle here (the GPU
ingest kernel has its own parity tests); the reduced table must equal the single-process one."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2009_04061_b200.dist import allreduce_counts, shard_range


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n_total, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import gpagen
    import oracle
    prog = gpagen.random_program(400, 3, 6, 3, seed=7)
    spec = gpagen.StreamSpec(prog, seed=8, count_max=3, invalid_ppm=10_000)
    k0, k1 = shard_range(n_total, rank, world)
    op = oracle.OracleProgram(prog)
    C, stats = op.histogram(spec.host(k0, k1 - k0))
    counts = torch.from_numpy(C.view(np.int64).reshape(-1).copy())
    st = torch.from_numpy(stats.view(np.int64).copy())
    allreduce_counts(counts, st)
    np.save(os.path.join(out_dir, f"c{rank}.npy"), counts.numpy())
    np.save(os.path.join(out_dir, f"s{rank}.npy"), st.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_shard_range_tiles_stream():
    for n in (0, 1, 7, 1000, 10**10 + 3):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_allreduce_of_shard_counts_equals_single_process(tmp_path):
    import gpagen
    import oracle
    n_total, world = 300_001, 2
    mp.spawn(_worker, args=(world, _free_port(), n_total, str(tmp_path)), nprocs=world, join=True)
    prog = gpagen.random_program(400, 3, 6, 3, seed=7)
    spec = gpagen.StreamSpec(prog, seed=8, count_max=3, invalid_ppm=10_000)
    C, stats = oracle.OracleProgram(prog).histogram(spec.host(0, n_total))
    for r in range(world):
        c = np.load(tmp_path / f"c{r}.npy")
        s = np.load(tmp_path / f"s{r}.npy")
        assert np.array_equal(c, C.view(np.int64).reshape(-1))      # bit-exact on every rank
        assert np.array_equal(s, stats.view(np.int64))

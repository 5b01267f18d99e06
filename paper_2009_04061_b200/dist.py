"""Multi-GPU plumbing for the sample-stream data parallelism.

One process per GPU.  Rank r ingests records [r*N/p, (r+1)*N/p) of the stream; the count table
(a commutative integer monoid) and the ingest stats are then summed across ranks with
one all-reduce (NCCL over NVLink/NVSwitch on the GPU box, gloo in the CPU tests), after which
blame, rollup and estimates run replicated and are identical on every rank.
"""
from __future__ import annotations


def shard_range(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous record range [k0, k1) of `rank`; the ranges of all ranks tile [0, n_total)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    k0 = n_total * rank // world
    k1 = n_total * (rank + 1) // world
    return k0, k1


def allreduce_counts(counts, stats=None, group=None):
    """Sum the per-rank count table (int64 view of the u64 table) and stats in place."""
    import torch.distributed as dist
    dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    if stats is not None:
        dist.all_reduce(stats, op=dist.ReduceOp.SUM, group=group)
    return counts


def sharded_step(program, records, group=None, stream=None, estimate=True):
    """One data-parallel step on this rank: reset -> ingest(local shard) -> all-reduce -> blame ->
    aggregate -> estimate.  `records` is this rank's device-resident shard."""
    import torch.distributed as dist
    program.reset(stream)
    program.ingest(records, stream=stream)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        allreduce_counts(program.view("counts"), program.view("stats"), group)
    if estimate:
        program.analyze(stream)      # blame + aggregate + estimate as one CUDA graph
    else:
        program.blame(stream)
        program.aggregate(stream)

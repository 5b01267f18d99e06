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
    aggregate -> estimate.  `records` is this rank's device-resident shard.

    The whole step runs with `stream` as torch's current stream: NCCL's all_reduce waits for, and is
    waited on by, the current stream only, so this is what orders the collective after the ingest
    and before the analysis when a caller passes a stream of its own."""
    import torch
    import torch.distributed as dist
    s = stream if stream is not None else torch.cuda.current_stream(program.device)
    with torch.cuda.stream(s):
        program.reset(s)
        program.ingest(records, stream=s)
        if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
            dist.all_reduce(program.reduce_view(), op=dist.ReduceOp.SUM, group=group)   # counts + stats, one call
        if estimate:
            program.analyze(s)      # blame + aggregate + estimate as one CUDA graph
        else:
            program.blame(s)
            program.aggregate(s)


# ----------------------------------------------------------------------------- DP-2
# Kernel partition: the blame of a kernel depends only on its own
# instructions, edges and samples (every def-use edge, line, loop and function lies inside one
# kernel), so a batch of kernels splits into contiguous kernel ranges that ranks analyse
# independently; only the (kernel x pattern) estimates travel back.

def partition_kernels(kernel_samples, world: int):
    """Contiguous kernel ranges [k_r, k_{r+1}) with balanced sample counts (each rank gets at
    least one kernel while there are kernels left).  Returns the world + 1 boundaries."""
    import numpy as np
    w = np.asarray(kernel_samples, np.float64)
    K = len(w)
    if world < 1:
        raise ValueError("world must be >= 1")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    bounds = [0]
    for r in range(1, world):
        lo = min(bounds[-1] + 1, K)                         # every rank gets a kernel while any remain
        hi = max(lo, K - (world - r))
        target = cum[-1] * r / world
        ks = np.arange(lo, hi + 1)
        bounds.append(int(ks[np.argmin(np.abs(cum[ks] - target))]))
    bounds.append(K)
    return bounds


def slice_program(prog, k0: int, k1: int):
    """The sub-program of kernels [k0, k1): instruction, edge, line, loop and function ids are
    renumbered from 0; returns (sub_program, maps) where maps holds the global ids of the slice's
    instructions ('pc_base', 'n_instr'), lines, loops, functions and kernels, for reassembling
    per-rank results.  Works on any object with the gpa_program_desc arrays (gpagen.Program)."""
    import dataclasses
    import numpy as np
    kfb = np.asarray(prog.kernel_func_begin, np.int64)
    fb = np.asarray(prog.func_begin, np.int64)
    if not 0 <= k0 < k1 <= len(kfb) - 1:
        raise ValueError(f"bad kernel range [{k0}, {k1})")
    f0, f1 = int(kfb[k0]), int(kfb[k1])
    i0, i1 = int(fb[f0]), int(fb[f1])
    rp = np.asarray(prog.row_ptr, np.int64)
    e0, e1 = int(rp[i0]), int(rp[i1])
    edef = np.asarray(prog.edge_def, np.int64)[e0:e1]
    if len(edef) and (edef.min() < i0 or edef.max() >= i1):
        raise ValueError("an edge crosses the kernel range")
    dom = np.asarray(prog.edge_dom_k, np.int64)[e0:e1]
    lines = np.asarray(prog.line_id, np.int64)[i0:i1]
    line_ids, line_new = np.unique(lines, return_inverse=True)
    lid = np.asarray(prog.loop_id, np.int64)[i0:i1]
    parent = np.asarray(prog.loop_parent, np.int64)
    used = set(int(x) for x in np.unique(lid[lid >= 0]))
    for l in list(used):                                  # close over enclosing loops
        p = int(parent[l])
        while p >= 0 and p not in used:
            used.add(p)
            p = int(parent[p])
    loop_ids = np.array(sorted(used), np.int64)
    remap = {int(l): r for r, l in enumerate(loop_ids)}
    new_lid = np.array([remap[int(l)] if l >= 0 else -1 for l in lid], np.int32) if len(lid) else lid.astype(np.int32)
    new_parent = np.array([remap[int(parent[l])] if parent[l] >= 0 else -1 for l in loop_ids], np.int32)
    fields = {f.name: getattr(prog, f.name) for f in dataclasses.fields(prog)}
    sl = slice(i0, i1)
    fields.update(
        opclass=np.asarray(prog.opclass)[sl].copy(), iflags=np.asarray(prog.iflags)[sl].copy(),
        latency=np.asarray(prog.latency)[sl].copy(), line_id=line_new.astype(np.uint32),
        loop_id=new_lid, loop_parent=new_parent,
        func_begin=(fb[f0:f1 + 1] - i0).astype(np.uint32),
        kernel_func_begin=(kfb[k0:k1 + 1] - f0).astype(np.uint32),
        kernel_grid_blocks=np.asarray(prog.kernel_grid_blocks)[k0:k1].copy(),
        row_ptr=(rp[i0:i1 + 1] - e0).astype(np.uint32),
        edge_def=(edef - i0).astype(np.uint32), edge_kind=np.asarray(prog.edge_kind)[e0:e1].copy(),
        edge_min_len=np.asarray(prog.edge_min_len)[e0:e1].copy(),
        edge_max_len=np.asarray(prog.edge_max_len)[e0:e1].copy(),
        edge_dom_k=np.where(dom >= 0, dom - i0, -1).astype(np.int32),
        n_lines=int(len(line_ids)))
    for opt in ("pc_weight", "pc_profile"):
        if fields.get(opt) is not None:
            fields[opt] = np.asarray(fields[opt])[sl].copy()
    sub = type(prog)(**fields)
    maps = {"pc_base": i0, "n_instr": i1 - i0, "edge_base": e0, "lines": line_ids, "loops": loop_ids,
            "funcs": np.arange(f0, f1), "kernels": np.arange(k0, k1)}
    return sub, maps


def gather_estimates(local_est, group=None):
    """Concatenate every rank's estimate rows (numpy structured/byte arrays, kernel-major) on all
    ranks, in rank order (= kernel order for partition_kernels ranges)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return local_est
    parts = [None] * dist.get_world_size(group)
    dist.all_gather_object(parts, local_est, group=group)
    return np.concatenate(parts) if isinstance(local_est, np.ndarray) else sum(parts, [])


def kernel_row_bounds(prog, kernel_bounds):
    """Instruction-row boundaries of contiguous kernel ranges (the count-table slices of DP-2)."""
    import numpy as np
    fb = np.asarray(prog.func_begin, np.int64)
    kfb = np.asarray(prog.kernel_func_begin, np.int64)
    return [int(fb[kfb[k]]) for k in kernel_bounds]


def reduce_scatter_counts(counts, row_bounds, out, group=None):
    """DP-2 for an ungrouped stream: every rank histogrammed an arbitrary shard of
    the records into the whole program's table `counts` (int64 view [n_instr, 2R]); rank r
    receives into `out` ([rows of its slice, 2R]) the sum over ranks of rows
    [row_bounds[r], row_bounds[r+1]) -- its kernels' slice.  NCCL: one reduce_scatter over
    slices padded to the largest; other backends (gloo in the CPU tests): all_reduce + slice."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    b = row_bounds
    if len(b) != world + 1 or out.shape[0] != b[rank + 1] - b[rank]:
        raise ValueError("row_bounds / out do not match the world")
    if dist.get_backend(group) == "nccl":
        rows = max(b[r + 1] - b[r] for r in range(world))
        flat = counts.reshape(counts.shape[0], -1)
        send = torch.zeros((world, rows, flat.shape[1]), dtype=counts.dtype, device=counts.device)
        for r in range(world):
            send[r, : b[r + 1] - b[r]] = flat[b[r]:b[r + 1]]
        recv = torch.empty((rows, flat.shape[1]), dtype=counts.dtype, device=counts.device)
        dist.reduce_scatter_tensor(recv, send, op=dist.ReduceOp.SUM, group=group)
        out.reshape(out.shape[0], -1).copy_(recv[: b[rank + 1] - b[rank]])
    else:
        tmp = counts.clone()
        dist.all_reduce(tmp, op=dist.ReduceOp.SUM, group=group)
        out.copy_(tmp[b[rank]:b[rank + 1]])
    return out

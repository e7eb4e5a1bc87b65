"""Factor sharding of a global-mapping linearization across ranks.

One process per GPU.  Every factor is an independent unit of work, so the graph's factors
are partitioned across ranks with longest-processing-time-first balancing on point count
(the per-factor cost).  Per linearization the solver rank broadcasts the pose table
(V x 8 doubles), every rank linearizes its shard, and the result goes back to the solver
rank — the one real exchange step of this path (the LM solve stays on the solver rank's host,
as in the reference: factor_graph.py:546-612).  Two forms: the per-factor records gathered
and reassembled in factor order (the drop-in's per-factor API), or each rank's block-sparse
normal equations in the global pair layout, sum-reduced onto the solver rank (what the LM
consumes: per-pose-pair H/b blocks, 4.5x fewer bytes at config 5).

The helpers are backend-agnostic torch.distributed calls: NCCL over NVLink on the B200 box,
gloo in the CPU tests (tests/test_distributed_gloo.py).
"""

from __future__ import annotations

import numpy as np


def lpt_shards(weights, n_shards: int) -> list:
    """Longest-processing-time partition of factor indices; each shard sorted ascending."""
    w = np.asarray(weights, dtype=np.float64)
    order = np.argsort(-w, kind="stable")
    loads = np.zeros(n_shards)
    members = [[] for _ in range(n_shards)]
    for f in order:
        r = int(np.argmin(loads))
        members[r].append(int(f))
        loads[r] += w[f]
    return [np.sort(np.array(m, dtype=np.int64)) for m in members]


def shard_loads(weights, shards) -> np.ndarray:
    w = np.asarray(weights, dtype=np.float64)
    return np.array([w[s].sum() for s in shards])


def broadcast_poses(poses, src: int = 0) -> None:
    """Pose table from the solver rank to every rank (in place)."""
    import torch.distributed as dist

    dist.broadcast(poses, src)


def gather_records(local, gather_list, dst: int = 0) -> None:
    """Per-factor records (padded to the largest shard) gathered to the solver rank."""
    import torch.distributed as dist

    dist.gather(local, gather_list, dst=dst)


def assemble_records(gathered, shards, num_factors: int):
    """Solver-rank reassembly of gathered shard records into global factor order."""
    import torch

    first = gathered[0]
    out = torch.empty((num_factors, first.shape[1]), dtype=first.dtype, device=first.device)
    for rec, idx in zip(gathered, shards):
        if len(idx):
            out.index_copy_(0, torch.as_tensor(idx, device=first.device), rec[: len(idx)])
    return out


def global_pairs(var_source, var_target, unary, num_vars: int) -> np.ndarray:
    """Sorted unique variable pairs (a < b) of every binary factor whose two variables are
    both < num_vars: the H-block layout shared by all ranks (vg_batch_assemble_setup_pairs)."""
    vs = np.asarray(var_source, np.int64)
    vt = np.asarray(var_target, np.int64)
    keep = ~np.asarray(unary, bool) & (vs < num_vars) & (vt < num_vars) & (vs != vt)
    a = np.minimum(vs[keep], vt[keep])
    b = np.maximum(vs[keep], vt[keep])
    key = np.unique(a * num_vars + b)
    return np.column_stack([key // num_vars, key % num_vars]).astype(np.int32)


def reduce_normal_equations(flat, dst: int = 0) -> None:
    """Sum every rank's normal equations (same layout) onto the solver rank (in place)."""
    import torch.distributed as dist

    dist.reduce(flat, dst, op=dist.ReduceOp.SUM)


def allreduce_cost(cost_count) -> None:
    """Cost-only pass (LM candidate steps, factor_graph.py:591; total_cost :472-474): every
    rank's gated (cost, factor count) pair summed on all ranks (in place, 2 scalars).  With
    a fixed rank count the sum order is fixed, so repeated passes are bit-identical."""
    import torch.distributed as dist

    dist.all_reduce(cost_count, op=dist.ReduceOp.SUM)

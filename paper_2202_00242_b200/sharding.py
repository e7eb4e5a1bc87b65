"""Factor sharding of a global-mapping linearization across ranks.

One process per GPU.  Every factor is an independent unit of work, so the graph's factors
are partitioned across ranks with longest-processing-time-first balancing on point count
(the per-factor cost).  Per linearization the solver rank broadcasts the pose table
(V x 8 doubles), every rank linearizes its shard, and the result goes back to the solver
rank — the one real exchange step of this path (the LM solve stays on the solver rank's host,
as in the reference: factor_graph.py:546-612).  Forms of the exchange:

* per-factor records gathered and reassembled in factor order (the drop-in's per-factor API);
* normal equations (what the LM consumes, factor_graph.py:522-536), the default of bench.py:
  factors are sharded PAIR-DISJOINTLY (both factors of an unordered variable pair on one
  rank, ``pair_shards``), so every rank assembles (K6) a compact system — its diagonal blocks
  and gradient for all variables plus the off-diagonal blocks of ITS pairs only — and one
  all-gather brings the per-rank systems to the solver rank, which sums the diagonal parts in
  rank order and places the pair blocks (``PairExchange``): per-rank K6 work and exchange
  bytes shrink with the rank count instead of every rank assembling the full 27,825-pair
  layout;
* the full global pair layout on every rank, sum-reduced (``global_pairs`` +
  ``reduce_normal_equations``; any sharding).

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


def pair_shards(var_source, var_target, weights, n_shards: int) -> list:
    """Pair-disjoint LPT shards: factors grouped by unordered variable pair (i -> j and
    j -> i together), groups balanced on their summed weight; each shard sorted ascending
    (the batch keeps the caller's target-major factor order)."""
    vs = np.asarray(var_source, np.int64)
    vt = np.asarray(var_target, np.int64)
    w = np.asarray(weights, np.float64)
    n = int(max(vs.max(initial=0), vt.max(initial=0))) + 1
    key = np.minimum(vs, vt) * n + np.maximum(vs, vt)
    _, group = np.unique(key, return_inverse=True)
    gw = np.bincount(group, weights=w)
    rank_of_group = np.empty(len(gw), np.int64)
    for r, members in enumerate(lpt_shards(gw, n_shards)):
        rank_of_group[members] = r
    rank = rank_of_group[group]
    return [np.flatnonzero(rank == r).astype(np.int64) for r in range(n_shards)]


def target_shards(var_target, weights, n_shards: int, positions=None) -> list:
    """Target-local shards: all factors of a target map on one rank, targets ordered along a
    Morton (Z-order) curve of their positions (`positions`: (V, 3), e.g. the pose table's
    translations; target index order when absent) and cut into n contiguous runs of equal
    summed weight.  A rank then reads ~1/n of the voxel maps — and mostly the source clouds of
    nearby submaps, the ones its targets are paired with — instead of nearly all of them, so
    its DRAM traffic shrinks with n (pair-disjoint shards scatter every map over all ranks).
    A variable pair's two factors can land on two ranks: their pair block is then summed by
    the exchange's reduction (global layout) or combine."""
    vt = np.asarray(var_target, np.int64)
    w = np.asarray(weights, np.float64)
    nv = int(vt.max(initial=0)) + 1
    tw = np.bincount(vt, weights=w, minlength=nv)
    if positions is not None:
        p = np.asarray(positions, np.float64)[:nv, :3]
        lo, hi = p.min(0), p.max(0)
        q = np.clip(((p - lo) / np.maximum(hi - lo, 1e-12) * 1023).astype(np.int64), 0, 1023)
        code = np.zeros(nv, np.int64)
        for bit in range(10):
            for ax in range(3):
                code |= ((q[:, ax] >> bit) & 1) << (3 * bit + ax)
        order = np.argsort(code, kind="stable")
    else:
        order = np.arange(nv)
    cum = np.cumsum(tw[order])
    total = cum[-1] if len(cum) else 0.0
    # target k of the order goes to the rank whose weight interval holds its midpoint
    mid = cum - tw[order] / 2
    rank_sorted = np.minimum((mid / max(total, 1e-30) * n_shards).astype(np.int64), n_shards - 1)
    rank_of_target = np.empty(nv, np.int64)
    rank_of_target[order] = rank_sorted
    rank = rank_of_target[vt]
    return [np.flatnonzero(rank == r).astype(np.int64) for r in range(n_shards)]


class PairExchange:
    """Layout of the pair-disjoint normal-equation exchange (see the module docstring).

    Rank r's compact system is the K6 flat layout over its own sorted pair list
    ``rank_pairs[r]``: [cost, count, diag V x 21, grad V x 6, pairs P_r x 36], padded to a
    common length ``L`` for the all-gather.  ``combine`` turns the gathered (N, L) block into
    the global system over ``pairs`` (the sorted union): cost, count, diagonal blocks and
    gradient summed over ranks in rank order, pair blocks placed from their rank (with
    pair-disjoint shards each pair's contributions were summed on one rank in factor order,
    exactly as the single-GPU assembly sums them; a pair shared by two ranks is summed)."""

    def __init__(self, var_source, var_target, unary, num_vars: int, shards):
        vs = np.asarray(var_source, np.int64)
        vt = np.asarray(var_target, np.int64)
        un = np.asarray(unary, bool)
        self.V = int(num_vars)
        self.rank_pairs = [global_pairs(vs[s], vt[s], un[s], self.V) for s in shards]
        self.pairs = global_pairs(vs, vt, un, self.V)
        index = {(int(a), int(b)): k for k, (a, b) in enumerate(self.pairs)}
        self.gidx = [np.array([index[(int(a), int(b))] for a, b in rp], np.int64)
                     for rp in self.rank_pairs]
        cat = np.concatenate(self.gidx) if self.gidx else np.zeros(0, np.int64)
        if len(np.unique(cat)) != len(self.pairs):
            raise ValueError("the shards do not cover the graph's pairs")
        self.pair_disjoint = len(cat) == len(self.pairs)
        self.head = 2 + 27 * self.V
        self.pmax = max((len(p) for p in self.rank_pairs), default=0)
        self.L = self.head + 36 * self.pmax
        self.size = self.head + 36 * len(self.pairs)   # the global system (K6 flat layout)

    def local_size(self, rank: int) -> int:
        return self.head + 36 * len(self.rank_pairs[rank])

    def combine(self, gathered, out=None):
        """(N, L) gathered per-rank systems -> the global flat system (torch, on the device
        the tensors live on)."""
        import torch

        g = gathered.reshape(len(self.rank_pairs), self.L)
        if out is None:
            out = torch.empty(self.size, dtype=g.dtype, device=g.device)
        out[: self.head] = g[:, : self.head].sum(0)
        blocks = out[self.head:].view(-1, 36)
        if not hasattr(self, "_gidx_t") or self._gidx_t[0].device != g.device:
            self._gidx_t = [torch.as_tensor(i, device=g.device) for i in self.gidx]
        blocks.zero_()
        for r, gi in enumerate(self._gidx_t):   # rank order: a shared pair sums in rank order
            if len(gi):
                blocks.index_add_(0, gi, g[r, self.head: self.head + 36 * len(gi)].view(-1, 36))
        return out


def exchange_normal_equations(local, ex: PairExchange, rank: int, gathered, out=None):
    """All-gather every rank's compact system (length ex.L, zero-padded) and combine it on
    the solver rank (rank 0).  `gathered` is an (N * L) buffer on the same device."""
    import torch.distributed as dist

    dist.all_gather_into_tensor(gathered, local)
    if rank == 0:
        return ex.combine(gathered, out)
    return None


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

"""Multi-rank path on the CPU (gloo, world size 2): LPT factor shards, pose-table broadcast,
per-factor record gather and solver-rank reassembly reproduce the single-process result.
The per-factor compute is the oracle here (CPU); on the B200 box the same sharding helpers
drive the CUDA batch over NCCL (bench.py)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import vgicp_oracle as O
from paper_2202_00242_b200 import geometry as G
from paper_2202_00242_b200 import sharding, synthetic

REC = 12 + 2  # a compact record for the test: T_ij-derived H diag (12) + cost + inliers


def _graph():
    rng = np.random.default_rng(31)
    poses = synthetic.random_submap_poses(rng, 6)
    dirs = synthetic.ray_table(64, 16)
    scans = [synthetic.scan(p, dirs, np.random.default_rng(7 + i)) for i, p in enumerate(poses)]
    covs = [O.estimate_covariances(s, O.knn_search(s, 10))[0] for s in scans]
    maps = [O.build_voxelmap(s, c, 1.0) for s, c in zip(scans, covs)]
    srcs = []
    for s, c in zip(scans, covs):
        sel = np.sort(rng.choice(len(s), int(rng.integers(100, 300)), replace=False))
        srcs.append((s[sel], c[sel]))
    pairs = synthetic.nearest_pairs(poses, 3)
    table = np.array([G.pose_row(G.pose_retract(p, synthetic.perturbation(rng, 0.05, 1.0)))
                      for p in poses])
    return srcs, maps, pairs, table


def _records(srcs, maps, pairs, table, ids):
    R, t = O.relative_transforms(table, pairs[ids, 0], pairs[ids, 1])
    out = np.zeros((len(ids), REC))
    for k, f in enumerate(ids):
        i, j = pairs[f]
        try:
            lin = O.linearize(srcs[i][0], srcs[i][1], maps[j], R[k], t[k])
            out[k, :6] = np.diag(lin["h_ii"])
            out[k, 6:12] = lin["b_i"]
            out[k, 12], out[k, 13] = lin["cost"], lin["inliers"]
        except ValueError:
            pass
    return out


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    srcs, maps, pairs, table = _graph()
    weights = np.array([len(srcs[i][0]) for i in pairs[:, 0]])
    shards = sharding.lpt_shards(weights, world)
    fmax = max(len(s) for s in shards)
    poses = torch.from_numpy(table.copy()) if rank == 0 else torch.zeros(table.shape,
                                                                         dtype=torch.float64)
    sharding.broadcast_poses(poses, 0)
    local = np.zeros((fmax, REC))
    mine = shards[rank]
    local[: len(mine)] = _records(srcs, maps, pairs, poses.numpy(), mine)
    gathered = [torch.zeros((fmax, REC), dtype=torch.float64) for _ in range(world)] \
        if rank == 0 else None
    sharding.gather_records(torch.from_numpy(local), gathered, dst=0)
    if rank == 0:
        full = sharding.assemble_records(gathered, shards, len(pairs)).numpy()
        ref = _records(srcs, maps, pairs, table, np.arange(len(pairs)))
        q.put((np.array_equal(full, ref), sharding.shard_loads(weights, shards).tolist()))
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_two_rank_shard_broadcast_gather_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, loads = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
    assert max(loads) / min(loads) < 1.1  # LPT balance on point counts


def test_lpt_balance_large():
    rng = np.random.default_rng(0)
    w = rng.integers(200, 601, 50000)
    for n in (2, 4, 8):
        loads = sharding.shard_loads(w, sharding.lpt_shards(w, n))
        assert loads.max() / loads.min() < 1.0005
        assert sum(len(s) for s in sharding.lpt_shards(w, n)) == 50000


def assemble_np(rec, vs, vt, unary, V, pairs):
    """NumPy model of vg_batch_assemble_* (K6): flat [cost, count, diag V x 21, grad V x 6,
    pair blocks P x 36], block sums in factor order."""
    index = {(int(a), int(b)): k for k, (a, b) in enumerate(pairs)}
    diag, grad = np.zeros((V, 21)), np.zeros((V, 6))
    off = np.zeros((len(pairs), 36))
    cost = count = 0.0
    for f in range(len(rec)):
        r = rec[f]
        if r[91] >= 10:
            cost += r[90]
            count += 1
        diag[vs[f]] += r[0:21]
        grad[vs[f]] += r[78:84]
        if unary[f]:
            continue
        diag[vt[f]] += r[57:78]
        grad[vt[f]] += r[84:90]
        a, b = min(vs[f], vt[f]), max(vs[f], vt[f])
        off[index[(a, b)]] += r[21:57] if vs[f] < vt[f] else r[21:57].reshape(6, 6).T.ravel()
    return np.concatenate([[cost, count], diag.ravel(), grad.ravel(), off.ravel()])


def _ne_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(5)
    V, F = 9, 60
    vs = rng.integers(0, V, F)
    vt = (vs + rng.integers(1, V, F)) % V
    unary = rng.uniform(size=F) < 0.2
    rec = rng.normal(size=(F, 92))
    rec[:, 91] = rng.integers(0, 40, F)
    pairs = sharding.global_pairs(vs, vt, unary, V)
    shards = sharding.lpt_shards(rng.integers(200, 600, F), world)
    mine = shards[rank]
    flat = torch.from_numpy(assemble_np(rec[mine], vs[mine], vt[mine], unary[mine], V, pairs))
    sharding.reduce_normal_equations(flat, dst=0)
    if rank == 0:
        ref = assemble_np(rec, vs, vt, unary, V, pairs)
        q.put(float(np.max(np.abs(flat.numpy() - ref) / np.maximum(np.abs(ref), 1.0))))
    dist.destroy_process_group()


def test_two_rank_normal_equations_reduce_matches_single_process():
    """Per-rank normal equations in the global pair layout (sharding.global_pairs), summed
    onto the solver rank, equal the single-process assembly to fp64 rounding."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ne_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-12


def test_global_pairs_layout():
    vs = np.array([0, 2, 1, 3, 2, 0])
    vt = np.array([1, 0, 0, 9, 2, 3])
    unary = np.array([False, False, False, False, False, True])
    assert sharding.global_pairs(vs, vt, unary, 4).tolist() == [[0, 1], [0, 2]]


def _gated_cost(srcs, maps, pairs, table, ids):
    """Per-factor cost with the inlier gate (factor_graph.py:271-275), summed in factor order."""
    R, t = O.relative_transforms(table, pairs[ids, 0], pairs[ids, 1])
    c = n = 0.0
    for k, f in enumerate(ids):
        i, j = pairs[f]
        cost, inl = O.matching_cost(srcs[i][0], srcs[i][1], maps[j], R[k], t[k])
        if inl >= O.MIN_INLIERS:
            c += cost
            n += 1
    return c, n


def _cost_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    srcs, maps, pairs, table = _graph()
    shards = sharding.lpt_shards(np.array([len(srcs[i][0]) for i in pairs[:, 0]]), world)
    poses = torch.from_numpy(table.copy()) if rank == 0 else torch.zeros(table.shape,
                                                                         dtype=torch.float64)
    sharding.broadcast_poses(poses, 0)
    runs = []
    for _ in range(2):  # repeated passes are bit-identical
        cc = torch.tensor(_gated_cost(srcs, maps, pairs, poses.numpy(), shards[rank]),
                          dtype=torch.float64)
        sharding.allreduce_cost(cc)
        runs.append(cc.numpy().copy())
    ref = _gated_cost(srcs, maps, pairs, table, np.arange(len(pairs)))
    q.put((rank, runs[0].tolist(), bool(np.array_equal(runs[0], runs[1])), list(ref)))
    dist.destroy_process_group()


def test_two_rank_cost_allreduce_matches_single_process():
    """Cost-only LM passes: each rank's gated shard cost, all-reduced (2 scalars), equals the
    single-process total on every rank (count exactly, cost to fp64 reassociation)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_cost_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, (c, n), repeat_equal, (rc, rn) in got:
        assert repeat_equal
        assert n == rn and n > 0
        assert abs(c - rc) <= 1e-12 * abs(rc)
    assert got[0][1] == got[1][1]  # every rank holds the same total


def _pair_ex_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(8)
    V, F = 12, 90
    vs = rng.integers(0, V, F)
    vt = (vs + rng.integers(1, V, F)) % V
    unary = np.zeros(F, bool)
    rec = rng.normal(size=(F, 92))
    rec[:, 91] = rng.integers(0, 40, F)
    shards = sharding.pair_shards(vs, vt, rng.integers(200, 600, F), world)
    ex = sharding.PairExchange(vs, vt, unary, V, shards)
    mine = shards[rank]
    local = np.zeros(ex.L)
    part = assemble_np(rec[mine], vs[mine], vt[mine], unary[mine], V, ex.rank_pairs[rank])
    assert len(part) == ex.local_size(rank)
    local[: len(part)] = part
    gathered = torch.zeros(world * ex.L, dtype=torch.float64)
    out = sharding.exchange_normal_equations(torch.from_numpy(local), ex, rank, gathered)
    if rank == 0:
        ref = assemble_np(rec, vs, vt, unary, V, ex.pairs)
        got = out.numpy()
        head = ex.head
        q.put((bool(np.array_equal(got[head:], ref[head:])),
               float(np.max(np.abs(got[:head] - ref[:head]) / np.maximum(np.abs(ref[:head]), 1.0))),
               [len(p) for p in ex.rank_pairs], len(ex.pairs)))
    dist.destroy_process_group()


def test_pair_disjoint_exchange_matches_single_process():
    """Pair-disjoint shards (both factors of a variable pair on one rank): every rank's compact
    system (all diagonal blocks, its own pair blocks), all-gathered and combined on the
    solver rank, equals the single-process assembly — pair blocks bit for bit (each pair is
    summed on one rank in factor order), diagonal blocks / gradient / cost to fp64
    reassociation (rank-order sum)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_pair_ex_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    pairs_exact, head_err, rank_pairs, total_pairs = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert pairs_exact
    assert head_err < 1e-12
    assert sum(rank_pairs) == total_pairs and min(rank_pairs) > 0


def test_pair_shards_are_pair_disjoint_and_balanced():
    rng = np.random.default_rng(1)
    poses = synthetic.random_submap_poses(rng, 300)
    pairs = synthetic.nearest_pairs(poses, 20)
    w = rng.integers(200, 601, 300)[pairs[:, 0]]
    for n in (2, 4, 8):
        shards = sharding.pair_shards(pairs[:, 0], pairs[:, 1], w, n)
        assert sorted(np.concatenate(shards).tolist()) == list(range(len(pairs)))
        owner = np.empty(len(pairs), int)
        for r, s in enumerate(shards):
            owner[s] = r
        key = {}
        for f, (a, b) in enumerate(pairs):
            k = (min(a, b), max(a, b))
            assert key.setdefault(k, owner[f]) == owner[f]
        loads = sharding.shard_loads(w, shards)
        assert loads.max() / loads.min() < 1.02
        ex = sharding.PairExchange(pairs[:, 0], pairs[:, 1], np.zeros(len(pairs), bool), 300,
                                   shards)
        assert ex.pmax <= 1.1 * len(ex.pairs) / n + 1

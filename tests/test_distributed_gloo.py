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

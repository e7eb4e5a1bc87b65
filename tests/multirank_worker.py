"""Rank worker of tests/test_gpu_multirank.py (launched by torch.distributed.run, gloo backend,
every rank on cuda:0): the sharded normal-equation step of bench.py at N ranks — pair-disjoint
shards, each rank's CUDA batch (K-compose, K4, K5, K6 in its compact layout), the all-gather
and the solver-rank combine — checked on rank 0 against the one-rank device assembly of the
whole graph.  Prints one JSON line on rank 0."""

import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2202_00242_b200 import _lib, sharding, workloads  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(0)
    wl = workloads.global_mapping(int(os.environ.get("MR_SUBMAPS", "60")),
                                  int(os.environ.get("MR_NEIGHBORS", "8")))
    F, V = len(wl.pairs), wl.pose_table.shape[0]
    w = np.array([len(wl.source_index[i]) for i in wl.pairs[:, 0]])
    if os.environ.get("MR_SHARDING", "target") == "target":
        shards = sharding.target_shards(wl.pairs[:, 1], w, world, wl.pose_table[:, 4:7])
    else:
        shards = sharding.pair_shards(wl.pairs[:, 0], wl.pairs[:, 1], w, world)
    ex = sharding.PairExchange(wl.pairs[:, 0], wl.pairs[:, 1], np.zeros(F, bool), V, shards)
    batch = wl.batch(shards[rank])
    mode = os.environ.get("MR_EXCHANGE", "reduce")
    if mode == "reduce":
        batch.assemble_setup_mapped(V, ex.rank_pairs[rank], ex.gidx[rank], len(ex.pairs))
    else:
        batch.assemble_setup(V, ex.rank_pairs[rank])
    host = torch.from_numpy(wl.pose_table.copy()) if rank == 0 else \
        torch.zeros(wl.pose_table.shape, dtype=torch.float64)
    sharding.broadcast_poses(host, 0)   # the solver rank's pose table to every rank
    poses = host.cuda()
    rec = torch.zeros((len(shards[rank]), 92), dtype=torch.float64, device="cuda")
    local = torch.zeros(ex.size if mode == "reduce" else ex.L, dtype=torch.float64,
                        device="cuda")
    batch.linearize_poses_device(poses.data_ptr(), V, _lib.MODE_LINEARIZE, rec.data_ptr())
    batch.assemble_records_device(rec.data_ptr(), local.data_ptr())
    batch.ctx.synchronize()
    if mode == "reduce":
        out = local.cpu()
        sharding.reduce_normal_equations(out, 0)
    else:
        gathered = torch.zeros(world * ex.L, dtype=torch.float64)
        out = sharding.exchange_normal_equations(local.cpu(), ex, rank, gathered)
    if rank == 0:
        full = wl.batch()
        full.assemble_setup(V, ex.pairs)
        ref = full.assemble_poses(wl.pose_table, unpack=False)
        got = out.numpy()
        h = ex.head
        rel = np.abs(got[:h] - ref[:h]) / np.maximum(np.abs(ref[:h]), 1e-30)
        print(json.dumps({"world": world, "exchange": mode, "pair_disjoint": ex.pair_disjoint,
                          "factors": F, "pairs": len(ex.pairs),
                          "rank_factors": [len(s) for s in shards],
                          "pair_blocks_bit_exact": bool(np.array_equal(got[h:], ref[h:])),
                          "pair_max_rel": float(np.max((np.abs(got[h:] - ref[h:]) /
                                                        np.maximum(np.abs(ref[h:]), 1e-30))
                                                       [np.abs(ref[h:]) > 1e-9])),
                          "count_equal": bool(got[1] == ref[1]),
                          "head_max_rel": float(np.max(rel[np.abs(ref[:h]) > 1e-9]))}),
              flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

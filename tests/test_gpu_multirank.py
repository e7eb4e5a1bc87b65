"""The N > 1 path with its CUDA batches behind it, on the one GPU a gpurun box has: ranks are
separate processes sharing cuda:0 and exchanging through gloo (CPU) collectives — none of
their kernels waits on another rank's, so this is a functional check of the sharding,
per-rank assembly, all-gather and combine (bench.py uses the same helpers over NCCL)."""

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _torchrun(n, script, *args, env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={_port()}", str(script), *args]
    e = dict(os.environ, OMP_NUM_THREADS="1", **(env or {}))
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    return [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]


@pytest.mark.parametrize("n,exchange,shard", [(2, "reduce", "target"), (3, "reduce", "target"),
                                               (2, "gather", "target"), (2, "reduce", "pair"),
                                               (3, "gather", "pair")])
def test_sharded_normal_equations_equal_one_rank(n, exchange, shard):
    """Rank systems reduced / gathered onto the solver rank equal the one-rank assembly: pair
    blocks bit for bit when the shards are pair-disjoint, else (a pair's two factors on two
    ranks, summed by the exchange) to fp64 reassociation, like the diagonal blocks."""
    (res,) = _torchrun(n, ROOT / "tests" / "multirank_worker.py",
                       env={"MR_EXCHANGE": exchange, "MR_SHARDING": shard})
    assert res["world"] == n and res["exchange"] == exchange and min(res["rank_factors"]) > 0
    assert res["count_equal"]
    assert res["head_max_rel"] < 1e-12
    if res["pair_disjoint"]:
        assert res["pair_blocks_bit_exact"]
    assert res["pair_max_rel"] < 1e-12


def test_bench_two_ranks_gloo_runs_the_multi_gpu_path():
    """bench.py --gpus 2 spawns its own ranks (no WORLD_SIZE) and reports n_gpus = 2."""
    cmd = [sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--backend", "gloo",
           "--steps", "3", "--warmup", "3", "--e2e-steps", "2", "--submaps", "60",
           "--neighbors", "8", "--no-cpu-baseline"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env=dict(os.environ, OMP_NUM_THREADS="1"))
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["n_gpus"] == 2 and line["multi_gpu"]["backend"] == "gloo"
    assert line["value"] > 0 and line["e2e"]["value"] > 0
    assert sum(line["multi_gpu"]["rank_factors"]) == line["config"]["factors"]

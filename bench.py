#!/usr/bin/env python
"""Benchmark: VGICP correspondences linearized per second (BASELINE.json metric) on the
global-mapping workload (config 5: 1000 submaps, 50 nearest-neighbour binary factors each,
~20M correspondences per linearization, 1.0 m maps), synthetic data.

One step = one linearization of every factor of the graph: compose T_ij from the pose table
(K-compose), fused transform/lookup/fused-covariance/accumulate (K4), fixed-order finalize
into the per-factor H_ii/H_ij/H_jj/b_i/b_j/cost records (K5).

N > 1 (one process per GPU; `--gpus N` spawns them through torch.distributed.run when
WORLD_SIZE is unset): the fixed 50,000-factor graph is sharded by target map across the ranks
(strong scaling; sharding.target_shards: each rank reads ~1/N of the voxel maps), the solver
rank broadcasts the pose table, every rank linearizes its shard and assembles its blocks of
the normal equations straight into the global block-sparse layout (K6: diagonal blocks +
gradient of every variable, its pairs' blocks at their global slots), and one NCCL
sum-reduction puts the system on the solver rank — so the N > 1 step does strictly more than
the N = 1 step (K6 and the reduction on top), and the driver's scaling ratio is conservative.
`--backend gloo` runs the same multi-rank path with CPU collectives, ranks sharing GPUs
(a functional check on a one-GPU box, not a timing).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

BYTES_PER_CORR = 84  # SURVEY.md §8d algorithmic bytes per correspondence
FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback
METRIC = "VGICP correspondences linearized/sec"
UNIT = "corr/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--submaps", type=int, default=1000)
    ap.add_argument("--neighbors", type=int, default=50)
    ap.add_argument("--cpu-targets", type=int, default=16,
                    help="target maps in the bounded CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--backend", choices=["nccl", "gloo"], default="nccl")
    ap.add_argument("--sharding", choices=["target", "pair"], default="target",
                    help="N > 1: target-local shards along a Morton curve (default) or "
                         "pair-disjoint LPT shards")
    ap.add_argument("--exchange", choices=["reduce", "gather"], default="reduce",
                    help="N > 1: sum-reduce the global layout (default) or all-gather "
                         "compact per-rank systems and combine on the solver rank")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the single-GPU BASELINE configs 1-4 (N = 1 extra keys)")
    ap.add_argument("--no-lm", action="store_true",
                    help="skip the one-iteration reference LM measurement (N = 1)")
    ap.add_argument("--cpu-full-pass", action="store_true",
                    help="reference arm: also time one pass over the whole workload")
    return ap.parse_args()


def traffic_record():
    """DRAM bytes per K4 launch from the committed ncu capture (profiles/r02_traffic.json,
    written by tools/launch_traffic.py from profiles/r02_launches.csv)."""
    p = ROOT / "profiles" / "r02_traffic.json"
    try:
        return int(json.loads(p.read_text())["dram_bytes_per_launch"])
    except Exception:
        return None


def ncu_metrics():
    """Per-kernel ncu digest of K4a/K4b from the committed capture (profiles/r02_ncu_metrics.json,
    tools/ncu_summary.py): L2/L1 hit rates and pipe use beside the roofline."""
    p = ROOT / "profiles" / "r02_ncu_metrics.json"
    try:
        return json.loads(p.read_text())
    except Exception:
        return None


def hbm_peak():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return FALLBACK_HBM_GBS, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML is initialised and
    sampled once before the region starts (so a short region still has samples), then every
    ~2 ms on a thread, then once more at the end; nvidia-smi is the fallback."""

    REASONS = {0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.errors = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._h = None
        self._nvml = None

    def _init_nvml(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self._smax = float(pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM))
            get = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                getattr(pynvml, "nvmlDeviceGetCurrentClocksThrottleReasons")
            self._reasons = get
            self._nvml = pynvml
        except Exception as exc:  # noqa: BLE001
            self.errors.append(f"nvml: {exc!r}")

    def _sample(self):
        if self._nvml is not None:
            try:
                sm = self._nvml.nvmlDeviceGetClockInfo(self._h, self._nvml.NVML_CLOCK_SM)
                self.samples.append((float(sm), self._smax, int(self._reasons(self._h))))
                return
            except Exception as exc:  # noqa: BLE001
                self.errors.append(f"nvml sample: {exc!r}")
                self._nvml = None
        for field in ("clocks_event_reasons.active", "clocks_throttle_reasons.active"):
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), "--query-gpu=clocks.sm,clocks.max.sm,"
                     + field, "--format=csv,noheader,nounits"],
                    capture_output=True, text=True, timeout=10).stdout
                sm, smax, act = [x.strip() for x in out.strip().split(",")]
                self.samples.append((float(sm), float(smax), int(act, 16)))
                return
            except Exception as exc:  # noqa: BLE001
                self.errors.append(f"nvidia-smi {field}: {exc!r}")

    def _run(self):
        while not self._stop.wait(0.002):
            self._sample()
            if self._nvml is None:  # nvidia-smi is slow: sample sparsely
                self._stop.wait(0.2)

    def __enter__(self):
        self._init_nvml()
        self._sample()
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)
        self._sample()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"],
                    "errors": self.errors[:4]}
        reasons = set()
        for _, _, act in self.samples:
            for bit, name in self.REASONS.items():
                if act & bit:
                    reasons.add(name)
        return {"sm_mhz": statistics.median(s[0] for s in self.samples),
                "sm_max_mhz": max(s[1] for s in self.samples),
                "reasons": sorted(reasons), "samples": len(self.samples),
                "source": "nvml" if self._nvml is not None else "nvidia-smi"}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def spawn_ranks(args) -> int:
    """`--gpus N` without a launcher: start N ranks with torch.distributed.run (one process
    per GPU, rendezvous on 127.0.0.1) and pass their output through."""
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")          # rank/channel setup evidence, on stderr
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    env.setdefault("OMP_NUM_THREADS", "1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", str(Path(__file__).resolve())] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def cpu_reference(wl, args, steps, warmup, one_process=False):
    from oracle import cpu_baseline

    sample = cpu_baseline.build_sample(wl, args.cpu_targets)
    rate, sec, procs = cpu_baseline.time_sample(sample, steps, warmup)
    desc = (f"{len(sample['pairs'])} factors (every factor whose target is one of submaps "
            f"0..{args.cpu_targets - 1}), {sample['points']} correspondences per pass, "
            f"oracle linearization, {procs}-process fork pool, {steps} passes")
    extra = {"cpu_model": cpu_baseline.cpu_model(), "cpu_count": os.cpu_count()}
    # the same sample through the reference package itself (baseline/_ref), beside the oracle
    # port the arm reports: the port restates it, this shows the two run at the same speed
    ref = ROOT / "baseline" / "_ref"
    if (ref / "limapper").is_dir() and str(ref) not in sys.path:
        sys.path.append(str(ref))
    try:
        rr = cpu_baseline.time_sample_reference(sample, steps, warmup)
    except Exception as exc:
        rr = None
        extra["reference_package"] = {"error": repr(exc)[:200]}
    if rr is not None:
        extra["reference_package"] = {
            "value": rr[0], "unit": UNIT, "seconds_per_pass": rr[1], "processes": rr[2],
            "sample": "the same factors through limapper.registration.linearize_matching_cost "
                      "(the unmodified reference from baseline/_ref), same fork pool"}
    if one_process:
        r1, s1, _ = cpu_baseline.time_sample(sample, 1, 0, processes=1)
        extra["one_process"] = {"value": r1, "unit": UNIT, "seconds_per_pass": s1,
                                "sample": "the same sample, 1 process (the reference's "
                                          "single-threaded NumPy path)"}
    return rate, sec, procs, desc, extra


def run_reference(args):
    world, rank, _ = dist_setup(args)
    if rank != 0:
        return 0
    from paper_2202_00242_b200 import workloads

    wl = workloads.global_mapping(args.submaps, args.neighbors, device_objects=False)
    steps = max(1, args.steps)
    rate, sec, procs, desc, extra = cpu_reference(wl, args, steps, max(1, min(args.warmup, 3)),
                                                  one_process=True)
    if args.cpu_full_pass:
        from oracle import cpu_baseline

        t0 = time.perf_counter()
        full = cpu_baseline.build_sample(wl, wl.n_submaps)
        prep = time.perf_counter() - t0
        r, s_, p_ = cpu_baseline.time_sample(full, 1, 0)
        extra["full_pass"] = {"value": r, "unit": UNIT, "seconds": s_, "processes": p_,
                              "factors": len(full["pairs"]), "corr": full["points"],
                              "input_prep_s": round(prep, 1)}
    line = {"metric": METRIC, "value": rate, "unit": UNIT, "n_gpus": world, "steps": steps,
            "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": "global-mapping (BASELINE config 5): bounded CPU sample",
                       "submaps": args.submaps, "neighbors": args.neighbors},
            "cpu_baseline": dict({"value": rate, "unit": UNIT, "cores": procs, "kind": "port",
                                  "sample": desc}, **extra),
            "e2e": {"value": rate, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def lm_iteration(wl):
    """One config-5 LM iteration through the REFERENCE's own FactorGraph (factor_graph.py:
    546-612, installed unmodified in baseline/_ref) with the drop-in patched in
    (integrate.patch): 1,000 submap-pose variables, a gauge prior on submap 0, the 50,000
    MatchingCostFactors of the workload (tools/lm_workloads.global_mapping_lm).  Wall-clock
    seconds of the iteration with the device solve and, from the same
    values, of the reference's optimize_lm with its host splu solve."""
    if not (ROOT / "baseline" / "_ref" / "limapper").is_dir():
        return {"unavailable": "reference not installed in baseline/_ref "
                               "(tools/install_reference.sh)"}
    sys.path.insert(0, str(ROOT / "tools"))
    import lm_workloads

    t0 = time.perf_counter()
    g, fg, info = lm_workloads.global_mapping_lm(wl)
    build_s = time.perf_counter() - t0
    out = lm_workloads.time_lm_iteration(g, fg, info)
    out["graph_build_s"] = round(build_s, 2)
    return out


def odometry_pipeline():
    """The reference's own OdometryEstimator on a 30-frame synthetic LiDAR-IMU sequence
    (tools/odometry_replay.py), through the drop-in and unmodified, each in its own process:
    wall-clock seconds per frame (the drop-in's first frames include its one-time setup)."""
    if not (ROOT / "baseline" / "_ref" / "limapper").is_dir():
        return {"unavailable": "reference not installed in baseline/_ref"}
    out = {"frames": 30, "sequence": "reference synthetic.square_loop_scene: 20 m loop, "
                                      "128 x 16 rays at 10 Hz, 200 Hz IMU",
           "api": "limapper OdometryEstimator.process_frame (odometry.py:222-293), "
                  "drop-in = integrate.patch"}
    for mode in ("dropin", "reference"):
        try:
            r = subprocess.run([sys.executable, str(ROOT / "tools" / "odometry_replay.py"),
                                "--mode", mode], capture_output=True, text=True, timeout=300)
            out[mode] = json.loads(r.stdout.strip().splitlines()[-1])
        except Exception as exc:
            out[mode] = {"error": repr(exc)[:200]}
    return out


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_setup(args)
    ndev = torch.cuda.device_count()
    dev = local % max(ndev, 1)   # gloo check runs may put several ranks on one GPU
    torch.cuda.set_device(dev)
    gloo = args.backend == "gloo"
    if world > 1:
        if gloo:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    from paper_2202_00242_b200 import _lib, sharding, workloads

    _lib.set_device(dev)
    ctx = _lib.context(dev)
    # a real (non-legacy) stream shared by torch events, NCCL and the library's launches
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx.set_stream(stream.cuda_stream)

    t0 = time.perf_counter()
    wl = workloads.global_mapping(args.submaps, args.neighbors)
    weights = np.array([len(wl.source_index[i]) for i in wl.pairs[:, 0]])
    F = len(wl.pairs)
    V = wl.pose_table.shape[0]
    if world > 1:
        if args.sharding == "target":
            shards = sharding.target_shards(wl.pairs[:, 1], weights, world, wl.pose_table[:, 4:7])
        else:
            shards = sharding.pair_shards(wl.pairs[:, 0], wl.pairs[:, 1], weights, world)
        ex = sharding.PairExchange(wl.pairs[:, 0], wl.pairs[:, 1], np.zeros(F, bool), V, shards)
    else:
        shards, ex = [np.arange(F)], None
    mine = shards[rank]
    batch = wl.batch(mine, ctx=ctx)
    ctx.set_stream(stream.cuda_stream)
    setup_s = time.perf_counter() - t0
    F_r = len(mine)
    total_points = wl.num_points
    my_points = int(weights[mine].sum())
    REC = _lib.RECORD_SIZE[_lib.MODE_LINEARIZE]

    poses_dev = torch.from_numpy(wl.pose_table).to("cuda")
    out_dev = torch.zeros((max(F_r, 1), REC), dtype=torch.float64, device="cuda")
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")  # 256 MB > L2

    ne_local = gathered = ne_global = None
    if world > 1:
        if args.exchange == "reduce":
            # K6 writes this rank's blocks straight into the global layout (diagonal blocks +
            # gradient of every variable, its own pair blocks at their global slots; other
            # slots stay zero) and one sum-reduction to the solver rank yields the system
            batch.assemble_setup_mapped(V, ex.rank_pairs[rank], ex.gidx[rank], len(ex.pairs))
            assert batch.asm_size == ex.size
            ne_local = torch.zeros(ex.size, dtype=torch.float64, device="cuda")
            ne_global = ne_local
        else:
            # compact per-rank layout, all-gather, solver-rank combine (sharding.PairExchange)
            batch.assemble_setup(V, ex.rank_pairs[rank])
            assert batch.asm_size == ex.local_size(rank)
            ne_local = torch.zeros(ex.L, dtype=torch.float64, device="cuda")
            gathered = torch.zeros(world * ex.L, dtype=torch.float64,
                                   device="cpu" if gloo else "cuda")
            ne_global = torch.zeros(ex.size, dtype=torch.float64, device="cuda")

    def exchange():
        if args.exchange == "reduce":
            if gloo:  # CPU collectives (functional check)
                host = ne_local.cpu()
                sharding.reduce_normal_equations(host, 0)
                if rank == 0:
                    ne_local.copy_(host)
            else:
                sharding.reduce_normal_equations(ne_local, 0)
            return
        if gloo:
            host = ne_local.cpu()
            sharding.exchange_normal_equations(host, ex, rank, gathered)
            if rank == 0:
                ne_global.copy_(ex.combine(gathered))
        else:
            sharding.exchange_normal_equations(ne_local, ex, rank, gathered, ne_global)

    def assemble():
        # the solver rank's buffer holds the last reduction: its other ranks' pair slots must be
        # zero again before this rank's K6 writes its own blocks
        if args.exchange == "reduce" and rank == 0:
            ne_local.zero_()
        batch.assemble_records_device(out_dev.data_ptr(), ne_local.data_ptr())

    def bcast_poses():
        if gloo:
            h = poses_dev.cpu()
            sharding.broadcast_poses(h, 0)
            poses_dev.copy_(h)
        else:
            sharding.broadcast_poses(poses_dev, 0)

    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]

    def step(e=None):
        if world > 1:
            bcast_poses()
        if e:
            e[0].record()
        batch.compose_device(poses_dev.data_ptr(), V)
        if e:
            e[1].record()
        batch.accumulate_device(_lib.MODE_LINEARIZE)
        if e:
            e[2].record()
        batch.finalize_device(_lib.MODE_LINEARIZE, out_dev.data_ptr())
        if world > 1:
            assemble()
            if e:
                e[3].record()
            exchange()

    graph = {"ready": False}

    def step_fast():
        # the same step as one library call (K-compose, K4a, K4b, K5 chained with programmatic
        # dependent launch; no host events between the kernels); N > 1: the rank's whole
        # device step (+ zeroing on the solver rank + K6) replayed as one captured graph
        # between the pose broadcast and the reduction
        if world > 1:
            bcast_poses()
            if graph["ready"]:
                batch.launch_graph()
            else:
                batch.linearize_poses_device(poses_dev.data_ptr(), V, _lib.MODE_LINEARIZE,
                                             out_dev.data_ptr())
                assemble()
            exchange()
            return
        batch.linearize_poses_device(poses_dev.data_ptr(), V, _lib.MODE_LINEARIZE,
                                     out_dev.data_ptr())

    for _ in range(max(3, args.warmup)):
        step()
        step_fast()
    torch.cuda.synchronize()
    if world > 1:
        batch.capture_assemble_graph(poses_dev.data_ptr(), V, out_dev.data_ptr(),
                                     ne_local.data_ptr(),
                                     zero_out=(args.exchange == "reduce" and rank == 0))
        graph["ready"] = True
        step_fast()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launch_count()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(dev) as clk:
        # timed region 1 (the metric): K steps, each one library call (+ K6 and the exchange)
        for k in range(args.steps):
            flush.zero_()  # evict L2 between timed steps (outside the timed events)
            starts[k].record()
            step_fast()
            ends[k].record()
        torch.cuda.synchronize()
        launches = ctx.launch_count() - launches0
        # timed region 2 (the roofline): the same K steps kernel by kernel, events around K4
        for k in range(args.steps):
            flush.zero_()
            step(ev[k])
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    k4_ms = [e[1].elapsed_time(e[2]) for e in ev]
    total_ms = float(sum(step_ms))
    rank_ms = None
    if world > 1:
        t = torch.tensor([total_ms], dtype=torch.float64,
                         device="cpu" if gloo else "cuda")
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        rank_ms = [float(x.item()) / args.steps for x in allt]
        total_ms = max(float(x.item()) for x in allt)
    ms_per_step = total_ms / args.steps
    value = total_points * args.steps / (total_ms / 1e3)

    # ---- e2e: through the public batch API with host buffers (H2D poses, D2H records) ----
    # N = 1 headline: the compact record (vg_batch_linearize_poses_f32: fp32 H/b blocks, fp64
    # cost, int32 inliers; 376 B/factor) into pinned host memory; the fp64 record (736 B) is
    # reported beside it.  N > 1: host pose table in on the solver rank, the combined normal
    # equations out of it.
    poses_host = torch.from_numpy(wl.pose_table.copy()).pin_memory()
    e2e_ms, e2e64_ms = [], []
    e2e64_line = cost_line = None
    hits_per_step = None
    if world == 1:
        out_host = torch.empty((F_r, REC), dtype=torch.float64).pin_memory()
        out32_host = torch.empty((F_r, _lib.REC_LINEARIZE_F32), dtype=torch.float32).pin_memory()
        out_np, out32_np, poses_np = out_host.numpy(), out32_host.numpy(), poses_host.numpy()
        for k in range(args.e2e_steps + 2):
            torch.cuda.synchronize()
            a = time.perf_counter()
            batch.linearize_poses_f32(poses_np, out=out32_np)
            if k >= 2:
                e2e_ms.append((time.perf_counter() - a) * 1e3)
        for k in range(args.e2e_steps + 2):
            torch.cuda.synchronize()
            a = time.perf_counter()
            batch.linearize_poses(poses_np, _lib.MODE_LINEARIZE, out=out_np)
            if k >= 2:
                e2e64_ms.append((time.perf_counter() - a) * 1e3)
        h2d = poses_host.numel() * 8
        d2h = F_r * _lib.REC_LINEARIZE_F32 * 4
        e2e64_line = {"value": total_points / (statistics.median(e2e64_ms) / 1e3), "unit": UNIT,
                      "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(F_r * REC * 8),
                      "ms_per_step": statistics.median(e2e64_ms),
                      "api": "DeviceBatch.linearize_poses (vg_batch_linearize_poses, fp64 records)"}
        # cost-only pass (LM candidate steps, factor_graph.py:591): the same correspondences,
        # no accumulators, 2 values per factor
        cost_dev = torch.zeros((F_r, 2), dtype=torch.float64, device="cuda")
        cs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ce = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        for k in range(3):
            batch.linearize_poses_device(poses_dev.data_ptr(), V, _lib.MODE_COST,
                                         cost_dev.data_ptr())
        for k in range(args.steps):
            flush.zero_()
            cs[k].record()
            batch.linearize_poses_device(poses_dev.data_ptr(), V, _lib.MODE_COST,
                                         cost_dev.data_ptr())
            ce[k].record()
        torch.cuda.synchronize()
        cms = sum(a.elapsed_time(b) for a, b in zip(cs, ce)) / args.steps
        hits_per_step = int(cost_dev.view(-1, 2)[:, 1].sum().item())
        cost_line = {"value": total_points / (cms / 1e3), "unit": UNIT, "ms_per_step": cms,
                     "kernel": "K4c k_cost_fused (lookup + cost fused) after K-compose, then K5",
                     "api": "vg_batch_linearize_poses_device(VG_MODE_COST)"}
    else:
        ne_host = torch.empty(ex.size, dtype=torch.float64).pin_memory()
        for k in range(args.e2e_steps + 2):
            torch.cuda.synchronize()
            dist.barrier()
            a = time.perf_counter()
            if rank == 0:
                poses_dev.copy_(poses_host, non_blocking=True)
            step_fast()
            if rank == 0:
                ne_host.copy_(ne_global, non_blocking=False)
            torch.cuda.synchronize()
            dt = torch.tensor([(time.perf_counter() - a) * 1e3], dtype=torch.float64,
                              device="cpu" if gloo else "cuda")
            dist.all_reduce(dt, op=dist.ReduceOp.MAX)
            if k >= 2:
                e2e_ms.append(float(dt.item()))
        h2d = poses_host.numel() * 8
        d2h = ex.size * 8
    e2e_value = total_points / (statistics.median(e2e_ms) / 1e3)

    # ---- e2e of the normal equations: the same linearization, summed into
    # the block-sparse H/g on the device, only the system crosses PCIe ----
    ne_line = None
    if world == 1:
        pairs = batch.assemble_setup(V)
        ne_out = torch.empty(batch.asm_size, dtype=torch.float64).pin_memory().numpy()
        ne_ms = []
        for k in range(args.e2e_steps + 2):
            torch.cuda.synchronize()
            a = time.perf_counter()
            batch.assemble_poses(poses_np, out=ne_out, unpack=False)
            if k >= 2:
                ne_ms.append((time.perf_counter() - a) * 1e3)
        ne_line = {"value": total_points / (statistics.median(ne_ms) / 1e3), "unit": UNIT,
                   "h2d_bytes_per_step": int(poses_host.numel() * 8),
                   "d2h_bytes_per_step": int(batch.asm_size * 8),
                   "ms_per_step": statistics.median(ne_ms), "variables": int(V),
                   "pairs": int(len(pairs)),
                   "api": "DeviceBatch.assemble_poses (vg_batch_assemble_poses)"}

    # ---- roofline of the dominant kernel (K4) ----
    peak, peak_kind = hbm_peak()
    k4_avg_s = statistics.mean(k4_ms) / 1e3
    achieved = BYTES_PER_CORR * my_points / k4_avg_s / 1e9

    configs = None
    if world == 1 and not args.no_configs:
        # BASELINE configs 1-4 (the single-GPU workloads north_star names) as extra keys: the
        # same fields as this line (tools/bench_configs.py), with hit counts next to the
        # correspondence counts
        sys.path.insert(0, str(ROOT / "tools"))
        import bench_configs

        cargs = argparse.Namespace(steps=20, no_cpu=args.no_cpu_baseline, no_graph=False)
        configs = {}
        for c in (1, 2, 3, 4):
            try:
                configs[str(c)] = (bench_configs.run_preprocess(cargs) if c == 2
                                   else bench_configs.run(c, cargs, ctx, stream))
            except Exception as exc:
                configs[str(c)] = {"error": repr(exc)[:300]}
        if not args.no_lm and isinstance(configs.get("4"), dict):
            # config 4 at the LM level: the reference's FactorGraph with its IMU and prior
            # factors on the host and the 4,950 matching factors on the GPU (one iteration)
            try:
                import lm_workloads

                configs["4"]["lm_iteration"] = lm_workloads.time_lm_iteration(
                    *lm_workloads.local_mapping_lm())
            except Exception as exc:
                configs["4"]["lm_iteration"] = {"error": repr(exc)[:300]}
        ctx.set_stream(stream.cuda_stream)
    lm_line = odo_line = None
    if world == 1 and not args.no_lm:
        try:
            lm_line = lm_iteration(wl)
        except Exception as exc:  # report, never sink the bench line
            lm_line = {"error": repr(exc)[:300]}
        odo_line = odometry_pipeline()
    if rank == 0:
        clocks = clk.summary()
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            rate, sec, procs, desc, extra = cpu_reference(wl, args, steps=3, warmup=1)
            cpu = dict({"value": rate, "unit": UNIT, "cores": procs, "kind": "port",
                        "sample": desc}, **extra)
        multi = None
        if world > 1:
            multi = {"backend": args.backend,
                     "sharding": ("target-local (Morton order of the submap positions), balanced "
                                  "on point count" if args.sharding == "target"
                                  else "pair-disjoint LPT on point count"),
                     "rank_ms_per_step": rank_ms,
                     "rank_factors": [int(len(s)) for s in shards],
                     "rank_points": [int(weights[s].sum()) for s in shards],
                     "exchange": ("sum-reduction of the global layout to the solver rank "
                                  "(each rank's K6 writes only its own pair blocks)"
                                  if args.exchange == "reduce" else
                                  "all-gather of compact normal equations + solver-rank combine"),
                     "exchange_bytes_per_rank": int((ex.size if args.exchange == "reduce"
                                                     else ex.L) * 8),
                     "global_pairs": int(len(ex.pairs)),
                     "global_system_bytes": int(ex.size * 8)}
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32+f64", "data": "synthetic",
            "config": {"workload": "global-mapping (BASELINE config 5)",
                       "submaps": args.submaps, "neighbors": args.neighbors,
                       "factors": int(F), "corr_per_step": total_points,
                       "voxel_resolution_m": wl.resolution, "scan_points": 16384,
                       "source_points": "U[200,600]", "parallelism": f"factor-shard x{world}",
                       "l2": "flushed between timed steps (256 MB write)",
                       "timing": ("steps as one library call (PDL-chained kernels); K4 timed "
                                  "in a second pass of the same steps with events around it"
                                  + ("; N > 1 steps add K6 + all-gather + combine" if world > 1
                                     else "")),
                       "setup_s": round(setup_s, 2)},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "ms_per_step": statistics.median(e2e_ms),
                    "api": ("DeviceBatch.linearize_poses_f32 (vg_batch_linearize_poses_f32: "
                            "fp32 H/b blocks, fp64 cost, int32 inliers) into pinned memory"
                            if world == 1 else "normal equations combined on the solver rank")},
            "e2e_f64_records": e2e64_line,
            "e2e_normal_equations": ne_line,
            "cost_mode": cost_line,
            "lm_iteration": lm_line,
            "odometry_pipeline": odo_line,
            "configs": configs,
            "multi_gpu": multi,
            "gpu_launches": int(launches),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic_record(),
                         "kernel": "K4 = k_lookup_fast (K4a) + k_accumulate<0> (K4b)",
                         "kernel_ms": statistics.mean(k4_ms),
                         "bytes_per_corr": BYTES_PER_CORR, "peak_kind": peak_kind,
                         "hits_per_step": hits_per_step,
                         # the bytes a miss does not need (its source covariance and voxel
                         # record, 60 of the 84 B) left out: SURVEY §8d's 84 B charges them
                         "hits_only": (None if hits_per_step is None else {
                             "bytes": 24 * my_points + 60 * hits_per_step,
                             "frac": (24 * my_points + 60 * hits_per_step) / k4_avg_s / 1e9
                                     / peak}),
                         "ncu": ncu_metrics()},
            "clocks": clocks,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return spawn_ranks(args)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

"""CPU baseline of the reference path (test/bench infrastructure; never a product path).

Times the oracle (a restatement of limapper's NumPy VGICP linearization, the reference's
own CPU implementation of this path) on a bounded sample of the global-mapping workload,
on all host cores: factors are split across a fork()ed process pool (the reference is
single-threaded NumPy; processes are how it uses more cores).

Sample: every factor whose target is one of the first ``n_targets`` submaps.  Its inputs are
recomputed on the CPU with the oracle (kNN + covariances of the target scans, covariances
of the source subsamples against their full scans, voxel maps at the workload resolution).
"""

from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np
from scipy.spatial import cKDTree

from . import vgicp_oracle as O

_SAMPLE = None


def knn_query(full: np.ndarray, queries_idx: np.ndarray, k: int) -> np.ndarray:
    """kNN (self included) of a subset of a scan's points among the whole scan, ordered by
    (d2, index) like knn_search (preprocess.py:122-139)."""
    q = full[queries_idx]
    _, cand = cKDTree(full).query(q, k=k)
    cand = np.asarray(cand, np.int64).reshape(len(q), k)
    diff = full[cand] - q[:, None, :]
    sq = diff * diff
    d2 = (sq[..., 0] + sq[..., 2]) + sq[..., 1]
    order = np.lexsort((cand, d2), axis=1)
    return np.take_along_axis(cand, order, axis=1)


_WL = None  # the workload, shared with fork()ed preparation workers


def _prep_map(j):
    s = _WL.scans[j]
    covs, _ = O.estimate_covariances(s, O.knn_search(s, _KNN))
    return int(j), O.build_voxelmap(s, covs, _WL.resolution)


def _prep_source(i):
    s, sel = _WL.scans[i], _WL.source_index[i]
    covs, _ = O.estimate_covariances(s, knn_query(s, sel, _KNN))
    return int(i), (s[sel], covs)


_KNN = 10


def build_sample(wl, n_targets: int = 16, knn: int = 10, processes: int | None = None):
    """Oracle inputs of every factor whose target is one of the first n_targets submaps
    (n_targets >= wl.n_submaps: the whole workload), prepared on all host cores."""
    global _WL, _KNN
    targets = np.arange(min(n_targets, wl.n_submaps))
    fids = np.flatnonzero(np.isin(wl.pairs[:, 1], targets))
    sources_needed = np.unique(wl.pairs[fids, 0])
    _WL, _KNN = wl, knn
    procs = processes or os.cpu_count() or 1
    if procs > 1:
        with mp.get_context("fork").Pool(procs) as pool:
            maps = dict(pool.map(_prep_map, targets, chunksize=4))
            sources = dict(pool.map(_prep_source, sources_needed, chunksize=8))
    else:
        maps = dict(map(_prep_map, targets))
        sources = dict(map(_prep_source, sources_needed))
    _WL = None
    R, t = O.relative_transforms(wl.pose_table, wl.pairs[fids, 0], wl.pairs[fids, 1])
    return {"fids": fids, "pairs": wl.pairs[fids], "maps": maps, "sources": sources, "R": R,
            "t": t, "poses": wl.pose_table.copy(),
            "points": int(sum(len(sources[int(i)][0]) for i in wl.pairs[fids, 0]))}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def _work(chunk):
    s = _SAMPLE
    n = 0
    for f in chunk:
        i, j = s["pairs"][f]
        pts, covs = s["sources"][int(i)]
        try:
            O.linearize(pts, covs, s["maps"][int(j)], s["R"][f], s["t"][f])
        except ValueError:  # degenerate factor: still evaluated
            pass
        n += len(pts)
    return n


_REF = None  # limapper objects of the sample (reference-package timing)


def _work_ref(chunk):
    """The same factors through the reference package's own public API
    (limapper.registration.linearize_matching_cost, registration.py:251-269)."""
    s, (reg, frames, maps, poses) = _SAMPLE, _REF
    n = 0
    for f in chunk:
        i, j = (int(v) for v in s["pairs"][f])
        try:
            reg.linearize_matching_cost(frames[i], maps[j], poses[i], poses[j])
        except reg.DegenerateConstraint:  # still evaluated (anything else propagates)
            pass
        n += len(frames[i])
    return n


def reference_objects(sample):
    """limapper Frames / GaussianVoxelMaps / Se3Poses of the sample (None when the reference
    package is not importable, e.g. from baseline/_ref)."""
    try:
        import limapper.geometry as G
        import limapper.preprocess as P
        import limapper.registration as reg
    except Exception:
        return None
    # only the unmodified reference: a process that applied integrate.patch runs the drop-in
    # under these names
    if getattr(reg.linearize_matching_cost, "__module__", "") != "limapper.registration":
        return None
    frames = {i: P.Frame(points=pts, stamps=np.zeros(len(pts)), stamp=0.0, covs=covs,
                         deskewed=True) for i, (pts, covs) in sample["sources"].items()}
    maps = {j: reg.GaussianVoxelMap(m[0], m[1], m[2], m[3], m[4])
            for j, m in sample["maps"].items()}
    need = set(int(v) for v in sample["pairs"].ravel())
    poses = {v: G.Se3Pose(G.Rotation(sample["poses"][v, :4]), sample["poses"][v, 4:7].copy())
             for v in need}
    return reg, frames, maps, poses


class Runner:
    """Keeps a fork()ed pool alive across timed steps."""

    def __init__(self, sample, processes: int | None = None, work=None):
        global _SAMPLE
        _SAMPLE = sample
        self.work = work or _work
        self.sample = sample
        self.processes = processes or os.cpu_count() or 1
        F = len(sample["pairs"])
        n_chunks = min(F, self.processes * 4)
        self.chunks = [c for c in np.array_split(np.arange(F), n_chunks) if len(c)]
        ctx = mp.get_context("fork")
        self.pool = ctx.Pool(self.processes) if self.processes > 1 else None

    def step(self) -> int:
        if self.pool is None:
            return sum(self.work(c) for c in self.chunks)
        return sum(self.pool.map(self.work, self.chunks))

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()


def time_sample_reference(sample, steps: int, warmup: int = 1, processes: int | None = None):
    """time_sample through the reference package itself (limapper importable); None if not."""
    global _REF
    _REF = reference_objects(sample)
    if _REF is None:
        return None
    try:
        return time_sample(sample, steps, warmup, processes, work=_work_ref)
    finally:
        _REF = None


def time_sample(sample, steps: int, warmup: int = 1, processes: int | None = None, work=None):
    """Returns (corr_per_s, seconds_per_step, processes)."""
    r = Runner(sample, processes, work)
    try:
        for _ in range(warmup):
            r.step()
        t0 = time.perf_counter()
        n = 0
        for _ in range(steps):
            n += r.step()
        dt = time.perf_counter() - t0
    finally:
        r.close()
    return n / dt, dt / max(steps, 1), r.processes

"""Drop-in for limapper/registration.py: Gaussian voxel maps, correspondence lookup, the
matching cost and its Gauss-Newton linearization — all computed by libvgicp on the GPU.

Public names, argument meanings and exceptions follow registration.py:26-269.  Numerics:
voxel keys, correspondence rows and inlier counts are bit-identical to the reference;
per-point math is fp32 with fp64 accumulation, so H/b/cost agree with the reference's
fp64 results to 1e-4 relative (1e-6 absolute) per element.
"""

from __future__ import annotations

import weakref
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import DegenerateConstraint
from .geometry import Gaussian3, Se3Pose, pose_compose, pose_inverse, pose_row, transform12
from .preprocess import Frame, device_cloud

MIN_INLIERS_DEFAULT = 10  # registration.py:26


class GaussianVoxelMap:
    """Per-voxel aggregate Gaussians (registration.py:29-71).

    Host arrays ``keys``/``means``/``covs``/``counts`` are the reference's sorted parallel
    arrays; the device copy is a bucketized open-addressing hash table (32-bit cell-local keys
    in 16 B buckets, or int64 keys for maps beyond the local frame) whose records carry the
    reference row.  Maps built on the GPU export their host arrays lazily.
    """

    def __init__(self, resolution: float, keys: np.ndarray, means: np.ndarray,
                 covs: np.ndarray, counts: np.ndarray):
        self.resolution = float(resolution)
        self._keys = keys
        self._means = means
        self._covs = covs
        self._counts = counts
        self._dev: _lib.DeviceMap | None = None
        self._m = int(np.asarray(keys).shape[0])

    @classmethod
    def _from_device(cls, resolution: float, dev: _lib.DeviceMap) -> "GaussianVoxelMap":
        obj = cls.__new__(cls)
        obj.resolution = float(resolution)
        obj._keys = obj._means = obj._covs = obj._counts = None
        obj._dev = dev
        obj._m = dev.m
        return obj

    # lazy host view of device-built maps
    def _export(self):
        k, mu, c, n = self._dev.export()
        self._keys, self._means, self._covs, self._counts = k, mu, c, n

    @property
    def keys(self) -> np.ndarray:
        if self._keys is None:
            self._export()
        return self._keys

    @property
    def means(self) -> np.ndarray:
        if self._means is None:
            self._export()
        return self._means

    @property
    def covs(self) -> np.ndarray:
        if self._covs is None:
            self._export()
        return self._covs

    @property
    def counts(self) -> np.ndarray:
        if self._counts is None:
            self._export()
        return self._counts

    def device(self) -> _lib.DeviceMap:
        if self._dev is None:
            self._dev = _lib.DeviceMap.from_arrays(self.resolution, self._keys, self._means,
                                                   self._covs, self._counts)
        return self._dev

    def __len__(self) -> int:
        return self._m

    def lookup(self, points: np.ndarray) -> np.ndarray:
        """Row index of the containing cell per point, -1 on a miss (registration.py:47-55)."""
        pts = _lib.f64(points).reshape(-1, 3)
        n = pts.shape[0]
        rows = np.full(n, -1, dtype=np.int64)
        if len(self) == 0 or n == 0:
            return rows
        dev = self.device()
        hits = np.zeros(1, dtype=np.int64)
        _lib.check(dev.ctx.lib.vg_map_lookup(dev.ctx.handle, dev.handle, _lib.dptr(pts), n,
                                             _lib.iptr(rows), _lib.iptr(hits)), "lookup")
        return rows

    def cell(self, index3):
        """(mean, cov, count) of the voxel at an integer 3-index (registration.py:57-63)."""
        pt = (np.asarray(index3, dtype=float) + 0.5) * self.resolution
        row = int(self.lookup(pt.reshape(1, 3))[0])
        if row < 0:
            raise KeyError(f"voxel {tuple(index3)} is empty")
        return self.means[row], self.covs[row], int(self.counts[row])

    def occupied_indices(self) -> np.ndarray:
        """Integer 3-indices of all occupied voxels (registration.py:65-71)."""
        k = self.keys
        mask = (1 << 21) - 1
        off = 1 << 20
        return np.column_stack([(k >> 42) - off, ((k >> 21) & mask) - off, (k & mask) - off])


def _as_device_map(vmap) -> _lib.DeviceMap:
    if isinstance(vmap, GaussianVoxelMap):
        return vmap.device()
    # a reference limapper GaussianVoxelMap: adopt its arrays once per object
    dev = _foreign_maps.get(id(vmap))
    if dev is not None and dev[0]() is vmap:
        return dev[1]
    d = _lib.DeviceMap.from_arrays(vmap.resolution, vmap.keys, vmap.means, vmap.covs,
                                   vmap.counts)
    key = id(vmap)
    try:
        _foreign_maps[key] = (weakref.ref(vmap, lambda _r, k=key: _foreign_maps.pop(k, None)), d)
    except TypeError:
        pass
    return d


_foreign_maps: dict[int, tuple] = {}


def build_voxelmap(frame, resolution: float) -> GaussianVoxelMap:
    """Aggregate point Gaussians into per-voxel Gaussians on the GPU (registration.py:74-98).

    The exported arrays are bit-identical to the reference's (same sort order, same
    sequential fp64 summation order, no FMA contraction).
    """
    if getattr(frame, "covs", None) is None and len(frame) > 0:
        raise ValueError("frame needs covariances before voxelization")
    if len(frame) == 0:
        return GaussianVoxelMap(resolution, np.zeros(0, dtype=np.int64), np.zeros((0, 3)),
                                np.zeros((0, 3, 3)), np.zeros(0, dtype=np.int64))
    cloud = device_cloud(frame)
    return GaussianVoxelMap._from_device(resolution, _lib.DeviceMap.build(cloud, resolution))


def d2d_error(point: Gaussian3, voxel: Gaussian3, t_ij):
    """Single-pair distribution-to-distribution error (registration.py:101-110).

    Evaluated on the GPU as a one-point factor so it exercises the same arithmetic as the
    batched kernel.  Returns (error, residual, weight) for any input, like the reference.

    The voxel is placed in every cell of the 3x3x3 block around the host-transformed point,
    so the device transform (a different FMA order, so possibly one ulp away across a cell
    face) lands in a cell carrying it; the resolution is a power of two large enough that the
    21-bit packed key never wraps (|moved| < 2^18 res).
    """
    frame = Frame(points=np.asarray(point.mean, float).reshape(1, 3), stamps=np.zeros(1),
                  stamp=0.0, covs=np.asarray(point.cov, float).reshape(1, 3, 3), deskewed=True)
    rmat = t_ij.rotation.matrix()
    moved = rmat @ np.asarray(point.mean, float) + t_ij.translation
    big = float(np.max(np.abs(moved)))
    if not np.isfinite(big):
        raise ValueError("d2d_error: non-finite transformed point")
    res = 1.0 if big < 2.0 ** 18 else 2.0 ** int(np.ceil(np.log2(big / 2.0 ** 18)))
    base = np.floor(moved / res).astype(np.int64)
    off = np.stack(np.meshgrid([-1, 0, 1], [-1, 0, 1], [-1, 0, 1], indexing="ij"),
                   axis=-1).reshape(27, 3)
    idx = base + off + (1 << 20)
    keys = np.sort((idx[:, 0] << 42) | (idx[:, 1] << 21) | idx[:, 2])
    vmap = GaussianVoxelMap(res, keys,
                            np.broadcast_to(np.asarray(voxel.mean, float), (27, 3)).copy(),
                            np.broadcast_to(np.asarray(voxel.cov, float), (27, 3, 3)).copy(),
                            np.ones(27, dtype=np.int64))
    terms = match_terms(frame, vmap, t_ij)
    if terms.inliers != 1:  # cannot happen: the block covers every rounding of the transform
        raise RuntimeError("d2d_error: transformed point left its voxel block")
    return float(terms.cost), terms.d[0], terms.weight[0]


@dataclass
class MatchTerms:
    """Correspondences and fixed weights of one frame/map pair (registration.py:133-143)."""

    hit: np.ndarray
    moved: np.ndarray
    d: np.ndarray
    weight: np.ndarray
    wd: np.ndarray
    cost: float
    inliers: int
    rows: np.ndarray | None = None
    _source: object = None
    _map: object = None


def match_terms(frame, vmap, t_ij) -> MatchTerms:
    """Per-point correspondences, residuals and weights (registration.py:146-157)."""
    cloud = device_cloud(frame)
    dev = _as_device_map(vmap)
    n = len(frame)
    rows = np.empty(n, dtype=np.int64)
    moved = np.empty((n, 3))
    d = np.empty((n, 3))
    w = np.empty((n, 3, 3))
    wd = np.empty((n, 3))
    cost = np.zeros(1)
    inl = np.zeros(1, dtype=np.int64)
    T = transform12(t_ij)
    ctx = cloud.ctx
    _lib.check(ctx.lib.vg_match_terms(ctx.handle, cloud.handle, dev.handle, _lib.dptr(T),
                                      _lib.iptr(rows), _lib.dptr(moved), _lib.dptr(d),
                                      _lib.dptr(w), _lib.dptr(wd), _lib.dptr(cost),
                                      _lib.iptr(inl)), "match_terms")
    hit = rows >= 0
    return MatchTerms(hit, moved, d[hit], w[hit], wd[hit], float(cost[0]), int(inl[0]),
                      rows=rows, _source=frame, _map=vmap)


def matching_cost(frame, vmap, t_ij):
    """(cost, inliers) of frame against the map at t_ij (registration.py:160-165)."""
    if len(frame) == 0 or len(vmap) == 0 or getattr(frame, "covs", None) is None:
        return 0.0, 0
    rec = _single_factor(frame, vmap, False, 0).linearize(
        transform12(t_ij).reshape(1, 12), _lib.MODE_COST)[0]
    return float(rec[0]), int(rec[1])


def overlap_rate(frame, vmap, t_ij) -> float:
    """Fraction of frame points landing in occupied voxels (registration.py:168-173)."""
    if len(frame) == 0 or len(vmap) == 0:
        return 0.0
    cloud = device_cloud(frame, with_covs=False)
    dev = _as_device_map(vmap)
    hits = np.zeros(1, dtype=np.int64)
    T = transform12(t_ij)
    ctx = cloud.ctx
    _lib.check(ctx.lib.vg_cloud_lookup(ctx.handle, cloud.handle, dev.handle, _lib.dptr(T), None,
                                       _lib.iptr(hits)), "overlap_rate")
    return float(hits[0]) / len(frame)


# overlap batches, keyed by the identities of their device clouds and maps
_overlap_cache: "OrderedDict[tuple, _lib.DeviceBatch]" = OrderedDict()


def _overlap_cloud(frame):
    # reuse the factor path's upload when the frame carries covariances
    return device_cloud(frame, with_covs=getattr(frame, "covs", None) is not None)


def _overlap_batch(frames, vmaps, idx, var_source=None, var_target=None):
    clouds = [_overlap_cloud(frames[k]) for k in idx]
    maps = [_as_device_map(vmaps[k]) for k in idx]
    vs = None if var_source is None else [int(var_source[k]) for k in idx]
    vt = None if var_target is None else [int(var_target[k]) for k in idx]
    key = (tuple((id(c), id(m)) for c, m in zip(clouds, maps)),
           None if vs is None else (tuple(vs), tuple(vt)))
    b = _overlap_cache.get(key)
    if b is None or any(x is not c for x, c in zip(b._keep[0], clouds)) \
            or any(x is not m for x, m in zip(b._keep[1], maps)):
        b = _lib.DeviceBatch(clouds, maps, [False] * len(idx), [0] * len(idx), vs, vt)
        _overlap_cache[key] = b
        while len(_overlap_cache) > 16:
            _overlap_cache.popitem(last=False)
    else:
        _overlap_cache.move_to_end(key)
    return b


def overlap_rates(frames, vmaps, t_ijs) -> np.ndarray:
    """overlap_rate (registration.py:168-173) for many (frame, map, T_ij) triples in one
    launch (VG_MODE_INLIERS: K4a lookups + hit counts only).  Empty inputs give 0.0."""
    n = len(frames)
    out = np.zeros(n)
    idx = [k for k in range(n) if len(frames[k]) and len(vmaps[k])]
    if not idx:
        return out
    b = _overlap_batch(frames, vmaps, idx)
    T = np.stack([transform12(t_ijs[k]) for k in idx])
    rec = b.linearize(T, _lib.MODE_INLIERS)
    out[idx] = rec[:, 1] / np.array([len(frames[k]) for k in idx], dtype=float)
    return out


def overlap_matrix(frames, vmaps, poses) -> np.ndarray:
    """out[i, j] = overlap_rate(frames[i], vmaps[j], T_j^-1 T_i) for i != j, 0 on the
    diagonal: the keyframe overlap matrix of odometry.py:396-403 in one launch (the relative
    poses are composed on the device from the pose table, K-compose)."""
    m = len(frames)
    out = np.zeros((m, m))
    pairs = [(i, j) for i in range(m) for j in range(m)
             if i != j and len(frames[i]) and len(vmaps[j])]
    if not pairs:
        return out
    fs = [frames[i] for i, _ in pairs]
    ms_ = [vmaps[j] for _, j in pairs]
    vs = [i for i, _ in pairs]
    vt = [j for _, j in pairs]
    b = _overlap_batch(fs, ms_, list(range(len(pairs))), vs, vt)
    table = np.array([pose_row(p) for p in poses])
    rec = b.linearize_poses(table, _lib.MODE_INLIERS)
    for (i, j), r in zip(pairs, rec[:, 1]):
        out[i, j] = r / len(frames[i])
    return out


@dataclass(frozen=True)
class MatchingCostLinearization:
    """Gauss-Newton blocks of the matching cost (registration.py:176-191)."""

    h_ii: np.ndarray
    h_ij: np.ndarray | None
    h_jj: np.ndarray | None
    b_i: np.ndarray
    b_j: np.ndarray | None
    cost: float
    inlier_count: int


def skew_batch(points: np.ndarray) -> np.ndarray:
    """(n, 3, 3) cross-product matrices (registration.py:194-204).  Accepted for API
    compatibility; the fused kernel forms the skew products in registers."""
    p = np.asarray(points, float).reshape(-1, 3)
    out = np.zeros((p.shape[0], 3, 3))
    out[:, 0, 1], out[:, 0, 2] = -p[:, 2], p[:, 1]
    out[:, 1, 0], out[:, 1, 2] = p[:, 2], -p[:, 0]
    out[:, 2, 0], out[:, 2, 1] = -p[:, 1], p[:, 0]
    return out


_TRIU = np.triu_indices(6)


def unpack_sym6(v: np.ndarray) -> np.ndarray:
    """Upper-triangle (21) -> symmetric 6x6; works on (..., 21)."""
    v = np.asarray(v)
    out = np.zeros(v.shape[:-1] + (6, 6))
    out[..., _TRIU[0], _TRIU[1]] = v
    out[..., _TRIU[1], _TRIU[0]] = v
    return out


def unpack_record(rec: np.ndarray, unary: bool) -> MatchingCostLinearization:
    """One VG_MODE_LINEARIZE record (92 doubles) -> MatchingCostLinearization."""
    h_ii = unpack_sym6(rec[0:21])
    b_i = rec[78:84].copy()
    cost, inl = float(rec[90]), int(rec[91])
    if unary:
        return MatchingCostLinearization(h_ii, None, None, b_i, None, cost, inl)
    return MatchingCostLinearization(h_ii, rec[21:57].reshape(6, 6).copy(),
                                     unpack_sym6(rec[57:78]), b_i, rec[84:90].copy(), cost, inl)


# single-factor batches, reused across calls on the same (frame, map) pair
_single_cache: "OrderedDict[tuple, _lib.DeviceBatch]" = OrderedDict()


def _single_factor(frame, vmap, unary: bool, min_inliers: int) -> _lib.DeviceBatch:
    cloud = device_cloud(frame)
    dev = _as_device_map(vmap)
    key = (id(cloud), id(dev), bool(unary), int(min_inliers))
    b = _single_cache.get(key)
    if b is not None and b._keep[0][0] is cloud and b._keep[1][0] is dev:
        _single_cache.move_to_end(key)
        return b
    b = _lib.DeviceBatch([cloud], [dev], [unary], [min_inliers])
    _single_cache[key] = b
    while len(_single_cache) > 64:
        _single_cache.popitem(last=False)
    return b


def _linearize_tij(frame_i, map_j, t_ij, target_fixed, min_inliers):
    b = _single_factor(frame_i, map_j, target_fixed, min_inliers)
    rec = b.linearize(transform12(t_ij).reshape(1, 12), _lib.MODE_LINEARIZE)[0]
    inl = int(rec[91])
    if inl < min_inliers:  # registration.py:213-215
        raise DegenerateConstraint(f"{inl} inliers (minimum {min_inliers})")
    return unpack_record(rec, target_fixed)


def linearize_from_terms(frame_i, terms: MatchTerms, t_ij, target_fixed: bool = False,
                         min_inliers: int = MIN_INLIERS_DEFAULT,
                         source_hats: np.ndarray | None = None) -> MatchingCostLinearization:
    """Gauss-Newton blocks from a MatchTerms (registration.py:207-248).

    A MatchTerms from this package's match_terms carries its voxel map, so the fused kernel
    recomputes the correspondences in registers instead of reading them back.  Any other
    MatchTerms (e.g. the reference's own, which has no map) is linearized on the GPU from its
    explicit per-point weights (vg_linearize_terms).
    """
    if terms.inliers < min_inliers:
        raise DegenerateConstraint(f"{terms.inliers} inliers (minimum {min_inliers})")
    vmap = getattr(terms, "_map", None)
    if vmap is not None:
        return _linearize_tij(frame_i, vmap, t_ij, target_fixed, min_inliers)
    hit = np.asarray(terms.hit, bool)
    pts = _lib.f64(np.asarray(frame_i.points, float)[hit])
    W = _lib.f64(terms.weight).reshape(-1, 9)
    wd = _lib.f64(terms.wd).reshape(-1, 3)
    if not (len(pts) == len(W) == len(wd)):
        raise ValueError("MatchTerms arrays disagree with the frame's hit mask")
    rec = np.empty(92)
    ctx = _lib.context()
    _lib.check(ctx.lib.vg_linearize_terms(
        ctx.handle, _lib.dptr(transform12(t_ij)), _lib.dptr(pts), _lib.dptr(W), _lib.dptr(wd),
        len(pts), float(terms.cost), int(terms.inliers), _lib.FACTOR_UNARY if target_fixed else 0,
        int(min_inliers), _lib.dptr(rec)), "linearize_from_terms")
    return unpack_record(rec, target_fixed)


def linearize_matching_cost(frame_i, map_j, t_i, t_j, target_fixed: bool = False,
                            min_inliers: int = MIN_INLIERS_DEFAULT,
                            source_hats: np.ndarray | None = None) -> MatchingCostLinearization:
    """Linearize the matching cost of frame_i against map_j (registration.py:251-269)."""
    t_ij = pose_compose(pose_inverse(t_j), t_i)
    if len(frame_i) == 0 or len(map_j) == 0 or getattr(frame_i, "covs", None) is None:
        raise DegenerateConstraint("no points to match")
    return _linearize_tij(frame_i, map_j, t_ij, target_fixed, min_inliers)

"""CPU ORACLE — test infrastructure only, never a product path.

A NumPy restatement of the reference's VGICP matching-cost path (limapper, pure Python/NumPy,
mounted read-only at /root/reference/pkg/src/limapper).  Only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg may import this module, and only as the
checker or the timed CPU baseline.

Parity is PINNED: tests/golden/make_golden.py runs the reference itself on seeded inputs and
commits the outputs as fixtures; tests/test_oracle_golden.py checks this restatement against
them (bit-exact for keys/rows/counts/kNN, <= 1e-12 relative for fp64 blocks).

All arrays are float64 / int64.  A transform is (R (3x3), t (3,)); a map is the tuple
(resolution, keys (m,), means (m,3), covs (m,3,3), counts (m,)) with keys sorted ascending.
"""

from __future__ import annotations

import numpy as np

KEY_OFFSET = 1 << 20  # preprocess.py:21-22
MIN_INLIERS = 10  # registration.py:26


# ---- keys / maps ----------------------------------------------------------------------------

def pack_voxel_keys(points: np.ndarray, resolution: float) -> np.ndarray:
    """preprocess.py:68-70 — floor of the true quotient, +2^20, 21 bits per axis."""
    cell = np.floor(np.asarray(points, float) / resolution).astype(np.int64) + KEY_OFFSET
    return (cell[:, 0] << 42) | (cell[:, 1] << 21) | cell[:, 2]


def unpack_voxel_keys(keys: np.ndarray) -> np.ndarray:
    """registration.py:65-71 — integer 3-index of packed keys."""
    mask = (1 << 21) - 1
    return np.stack([(keys >> 42) - KEY_OFFSET, ((keys >> 21) & mask) - KEY_OFFSET,
                     (keys & mask) - KEY_OFFSET], axis=1)


def build_voxelmap(points: np.ndarray, covs: np.ndarray, resolution: float):
    """registration.py:74-98.

    Cells are the sorted unique keys; the mean is the sequential sum of members in index
    order over the count; the covariance is the mean of (C_k + (p_k - mu)(p_k - mu)^T),
    summed in the same order.  np.add.at accumulates in index order, which is what makes the
    result reproducible bit for bit.
    """
    pts = np.asarray(points, float).reshape(-1, 3)
    if pts.shape[0] == 0:
        return (float(resolution), np.zeros(0, np.int64), np.zeros((0, 3)), np.zeros((0, 3, 3)),
                np.zeros(0, np.int64))
    if covs is None:
        raise ValueError("frame needs covariances before voxelization")
    keys = pack_voxel_keys(pts, resolution)
    cells, member_of, counts = np.unique(keys, return_inverse=True, return_counts=True)
    m = cells.shape[0]
    acc = np.zeros((m, 3))
    np.add.at(acc, member_of, pts)
    means = acc / counts[:, None]
    c = pts - means[member_of]
    contrib = np.asarray(covs, float) + c[:, :, None] * c[:, None, :]
    cov_acc = np.zeros((m, 3, 3))
    np.add.at(cov_acc, member_of, contrib)
    return (float(resolution), cells, means, cov_acc / counts[:, None, None],
            counts.astype(np.int64))


def lookup(vmap, points: np.ndarray) -> np.ndarray:
    """registration.py:47-55 — row of the containing cell or -1 (binary search)."""
    res, keys = vmap[0], vmap[1]
    pts = np.asarray(points, float).reshape(-1, 3)
    if keys.shape[0] == 0 or pts.shape[0] == 0:
        return np.full(pts.shape[0], -1, np.int64)
    q = pack_voxel_keys(pts, res)
    pos = np.minimum(np.searchsorted(keys, q), keys.shape[0] - 1)
    return np.where(keys[pos] == q, pos, -1).astype(np.int64)


# ---- matching cost / linearization ----------------------------------------------------------

def _inverse3(a: np.ndarray) -> np.ndarray:
    """registration.py:113-130 — adjugate over determinant, batched."""
    adj = np.empty_like(a)
    adj[:, 0, 0] = a[:, 1, 1] * a[:, 2, 2] - a[:, 1, 2] * a[:, 2, 1]
    adj[:, 0, 1] = a[:, 0, 2] * a[:, 2, 1] - a[:, 0, 1] * a[:, 2, 2]
    adj[:, 0, 2] = a[:, 0, 1] * a[:, 1, 2] - a[:, 0, 2] * a[:, 1, 1]
    adj[:, 1, 0] = a[:, 1, 2] * a[:, 2, 0] - a[:, 1, 0] * a[:, 2, 2]
    adj[:, 1, 1] = a[:, 0, 0] * a[:, 2, 2] - a[:, 0, 2] * a[:, 2, 0]
    adj[:, 1, 2] = a[:, 0, 2] * a[:, 1, 0] - a[:, 0, 0] * a[:, 1, 2]
    adj[:, 2, 0] = a[:, 1, 0] * a[:, 2, 1] - a[:, 1, 1] * a[:, 2, 0]
    adj[:, 2, 1] = a[:, 0, 1] * a[:, 2, 0] - a[:, 0, 0] * a[:, 2, 1]
    adj[:, 2, 2] = a[:, 0, 0] * a[:, 1, 1] - a[:, 0, 1] * a[:, 1, 0]
    det = a[:, 0, 0] * adj[:, 0, 0] + a[:, 0, 1] * adj[:, 1, 0] + a[:, 0, 2] * adj[:, 2, 0]
    return adj / det[:, None, None]


def match_terms(points, covs, vmap, R, t) -> dict:
    """registration.py:146-157 — transform, lookup, fused covariance, weights, cost."""
    R = np.asarray(R, float)
    moved = np.asarray(points, float) @ R.T + np.asarray(t, float)
    rows = lookup(vmap, moved)
    hit = rows >= 0
    sel = rows[hit]
    d = vmap[2][sel] - moved[hit]
    fused = vmap[3][sel] + R @ (np.asarray(covs, float)[hit] @ R.T)
    w = _inverse3(fused)
    wd = np.einsum("nij,nj->ni", w, d)
    return {"rows": rows, "hit": hit, "moved": moved, "d": d, "weight": w, "wd": wd,
            "cost": float(np.sum(d * wd)), "inliers": int(hit.sum())}


def matching_cost(points, covs, vmap, R, t):
    """registration.py:160-165."""
    if len(points) == 0 or vmap[1].shape[0] == 0 or covs is None:
        return 0.0, 0
    mt = match_terms(points, covs, vmap, R, t)
    return mt["cost"], mt["inliers"]


def overlap_rate(points, vmap, R, t) -> float:
    """registration.py:168-173."""
    if len(points) == 0 or vmap[1].shape[0] == 0:
        return 0.0
    moved = np.asarray(points, float) @ np.asarray(R, float).T + np.asarray(t, float)
    return float(np.count_nonzero(lookup(vmap, moved) >= 0)) / len(points)


def _hat(v: np.ndarray) -> np.ndarray:
    out = np.zeros(v.shape[:-1] + (3, 3))
    out[..., 0, 1], out[..., 0, 2] = -v[..., 2], v[..., 1]
    out[..., 1, 0], out[..., 1, 2] = v[..., 2], -v[..., 0]
    out[..., 2, 0], out[..., 2, 1] = -v[..., 1], v[..., 0]
    return out


def linearize(points, covs, vmap, R, t, target_fixed=False, min_inliers=MIN_INLIERS):
    """registration.py:207-248 (fed by :146-157): explicit per-point Jacobians.

    J_i = [R hat(mu) | -R] (source), J_j = [-hat(x) | I] (target); H = 2 sum J^T W J,
    b = 2 sum J^T W d.  Returns a dict with h_ii, h_ij, h_jj, b_i, b_j (None when unary),
    cost, inliers; raises ValueError('degenerate') when inliers < min_inliers.
    """
    mt = match_terms(points, covs, vmap, R, t)
    if mt["inliers"] < min_inliers:
        raise ValueError(f"degenerate: {mt['inliers']} inliers (minimum {min_inliers})")
    R = np.asarray(R, float)
    hit, w, wd = mt["hit"], mt["weight"], mt["wd"]
    mu = np.asarray(points, float)[hit]
    n = mu.shape[0]
    j_i = np.empty((n, 3, 6))
    j_i[:, :, :3] = R @ _hat(mu)
    j_i[:, :, 3:] = -R
    jtw_i = np.swapaxes(j_i, 1, 2) @ w
    out = {"h_ii": 2.0 * (jtw_i @ j_i).sum(0),
           "b_i": 2.0 * np.einsum("nij,nj->i", np.swapaxes(j_i, 1, 2), wd),
           "h_ij": None, "h_jj": None, "b_j": None,
           "cost": mt["cost"], "inliers": mt["inliers"]}
    if target_fixed:
        return out
    j_j = np.empty((n, 3, 6))
    j_j[:, :, :3] = -_hat(mt["moved"][hit])
    j_j[:, :, 3:] = np.eye(3)
    jtw_j = np.swapaxes(j_j, 1, 2) @ w
    out["h_jj"] = 2.0 * (jtw_j @ j_j).sum(0)
    out["h_ij"] = 2.0 * (jtw_i @ j_j).sum(0)
    out["b_j"] = 2.0 * np.einsum("nij,nj->i", np.swapaxes(j_j, 1, 2), wd)
    return out


# ---- preprocessing -------------------------------------------------------------------------

def squared_distances(points: np.ndarray, nbr: np.ndarray) -> np.ndarray:
    """fp64 squared distance as the reference's einsum forms it: (dx^2 + dz^2) + dy^2
    (association checked bit for bit against the reference's fixtures)."""
    diff = points[nbr] - points[:, None, :]
    sq = diff * diff
    return (sq[..., 0] + sq[..., 2]) + sq[..., 1]


def knn_search(points: np.ndarray, k: int) -> np.ndarray:
    """preprocess.py:122-139 — exact kNN (self included), ascending (d2, index)."""
    from scipy.spatial import cKDTree

    pts = np.asarray(points, float).reshape(-1, 3)
    n = pts.shape[0]
    if n < k:
        raise ValueError(f"too sparse: frame has {n} points, need at least {k}")
    _, cand = cKDTree(pts).query(pts, k=k)
    cand = np.asarray(cand, np.int64).reshape(n, k)
    order = np.lexsort((cand, squared_distances(pts, cand)), axis=1)
    return np.take_along_axis(cand, order, axis=1)


def knn_bruteforce(points: np.ndarray, k: int) -> np.ndarray:
    """Stable argsort over all pairs (the check of test_preprocess.py:105-114)."""
    pts = np.asarray(points, float).reshape(-1, 3)
    n = pts.shape[0]
    allidx = np.broadcast_to(np.arange(n), (n, n))
    d2 = squared_distances(pts, allidx)
    return np.argsort(d2, axis=1, kind="stable")[:, :k].astype(np.int64)


def estimate_covariances(points: np.ndarray, neighbors: np.ndarray, plane_eps=1e-3):
    """preprocess.py:142-164 — sample covariance / k, eigh, eigenvalues -> (eps, 1, 1);
    lambda_max < 1e-12 -> eps * I (flagged degenerate)."""
    pts = np.asarray(points, float).reshape(-1, 3)
    if pts.shape[0] == 0:
        return np.zeros((0, 3, 3)), np.zeros(0, bool)
    nb = pts[np.asarray(neighbors)]
    c = nb - nb.mean(axis=1, keepdims=True)
    cov = np.einsum("nki,nkj->nij", c, c) / nb.shape[1]
    lam, vec = np.linalg.eigh(cov)
    degenerate = lam[:, 2] < 1e-12
    out = (vec * np.array([plane_eps, 1.0, 1.0])) @ np.swapaxes(vec, 1, 2)
    out[degenerate] = np.eye(3) * plane_eps
    return out, degenerate


# ---- voxel downsampling (preprocess.py:73-119) ----------------------------------------------

def pairwise_sum(a: np.ndarray) -> float:
    """NumPy's 1-D float64 add.reduce (pairwise: 8 accumulators up to 128 elements, halves
    rounded to a multiple of 8 above) — the summation order of `stamps[cell].mean()`."""
    n = len(a)
    if n < 8:
        res = 0.0
        for x in a:
            res += float(x)
        return res
    if n <= 128:
        r = [float(x) for x in a[:8]]
        i = 8
        while i < n - n % 8:
            for j in range(8):
                r[j] += float(a[i + j])
            i += 8
        res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
        for x in a[i:]:
            res += float(x)
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return pairwise_sum(a[:n2]) + pairwise_sum(a[n2:])


def _cell_mean(points, stamps, cell):
    """`points[cell].mean(axis=0)` (sequential row sums from 0.0) and `stamps[cell].mean()`
    (pairwise), each divided by the count."""
    acc = np.zeros(3)
    for i in cell:
        acc = acc + points[i]
    return acc / len(cell), (0.0 + pairwise_sum(stamps[cell])) / len(cell)


def voxel_downsample(points: np.ndarray, stamps: np.ndarray, resolution: float,
                     duration: float):
    """preprocess.py:73-119 — points grouped by packed voxel key (ascending key, members in
    scan order); a group whose stamp spread exceeds duration/10 is split by the running-mean
    rule into a primary and an overflow cell.  Returns (points (m,3), stamps (m,))."""
    if resolution <= 0.0:
        raise ValueError("resolution must be positive")
    pts = np.asarray(points, float).reshape(-1, 3)
    ts = np.asarray(stamps, float).reshape(-1)
    n = pts.shape[0]
    if n == 0:
        return pts, ts
    tol = duration / 10.0
    keys = pack_voxel_keys(pts, resolution)
    order = np.argsort(keys, kind="stable")
    starts = np.flatnonzero(np.r_[True, np.diff(keys[order]) != 0])
    ends = np.r_[starts[1:], n]
    out_p, out_t = [], []
    for s, e in zip(starts, ends):
        grp = order[s:e]
        g = ts[grp]
        if g.max() - g.min() <= tol:
            cells = [grp]
        else:
            cells = [[], []]
            sums = [0.0, 0.0]
            for i in grp:
                t = ts[i]
                target = 0 if (not cells[0] or abs(t - sums[0] / len(cells[0])) <= tol) else 1
                cells[target].append(i)
                sums[target] += t
            cells = [np.asarray(c, np.int64) for c in cells if c]
        for c in cells:
            mp, mt = _cell_mean(pts, ts, c)
            out_p.append(mp)
            out_t.append(mt)
    return np.asarray(out_p).reshape(-1, 3), np.asarray(out_t)


# ---- deskew, per-point half (preprocess.py:167-178, 218-231) -------------------------------

def slerp(qa: np.ndarray, qb: np.ndarray, alpha: np.ndarray) -> np.ndarray:
    """Shortest-arc slerp of xyzw rows (preprocess.py:167-178): near-parallel pairs
    (dot > 1 - 1e-12) interpolate linearly; the result is renormalised."""
    dot = np.sum(qa * qb, axis=1)
    qb = np.where(dot[:, None] < 0.0, -qb, qb)
    dot = np.abs(dot)
    theta = np.arccos(np.clip(dot, -1.0, 1.0))
    den = np.sin(theta)
    den = np.where(den == 0.0, 1.0, den)
    near = dot > 1.0 - 1e-12
    w0 = np.where(near, 1.0 - alpha, np.sin((1.0 - alpha) * theta) / den)
    w1 = np.where(near, alpha, np.sin(alpha * theta) / den)
    q = w0[:, None] * qa + w1[:, None] * qb
    return q / np.sqrt(np.sum(q * q, axis=1, keepdims=True))


def deskew_points(points, stamps, node_t, quats, trans) -> np.ndarray:
    """preprocess.py:218-231 — each point's trajectory segment (last node at or before its
    stamp, clipped to the node range), slerped rotation and interpolated translation at its
    stamp, then p' = p + w c1 + u x c1 + t with c1 = 2 u x p (q = (u, w))."""
    p = np.asarray(points, float).reshape(-1, 3)
    ts = np.asarray(stamps, float).reshape(-1)
    node_t = np.asarray(node_t, float)
    seg = np.clip(np.searchsorted(node_t, ts, side="right") - 1, 0, node_t.size - 2)
    span = node_t[seg + 1] - node_t[seg]
    alpha = np.where(span > 0, (ts - node_t[seg]) / np.where(span > 0, span, 1.0), 0.0)
    alpha = np.clip(alpha, 0.0, 1.0)
    q = slerp(quats[seg], quats[seg + 1], alpha)
    t = (1.0 - alpha)[:, None] * trans[seg] + alpha[:, None] * trans[seg + 1]
    u, w = q[:, :3], q[:, 3:4]
    c1 = 2.0 * np.cross(u, p)
    return p + w * c1 + np.cross(u, c1) + t


# ---- poses (geometry.py:33-144, 231-237), vectorised over factors -------------------------

def _qmul(a, b):
    ax, ay, az, aw = a[..., 0], a[..., 1], a[..., 2], a[..., 3]
    bx, by, bz, bw = b[..., 0], b[..., 1], b[..., 2], b[..., 3]
    return np.stack([aw * bx + bw * ax + ay * bz - az * by,
                     aw * by + bw * ay + az * bx - ax * bz,
                     aw * bz + bw * az + ax * by - ay * bx,
                     aw * bw - ax * bx - ay * by - az * bz], axis=-1)


def _qnorm(q):
    return q / np.sqrt(np.sum(q * q, axis=-1, keepdims=True))


def _qapply(q, v):
    ux, uy, uz, w = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    vx, vy, vz = v[..., 0], v[..., 1], v[..., 2]
    tx = 2.0 * (uy * vz - uz * vy)
    ty = 2.0 * (uz * vx - ux * vz)
    tz = 2.0 * (ux * vy - uy * vx)
    return np.stack([vx + w * tx + uy * tz - uz * ty, vy + w * ty + uz * tx - ux * tz,
                     vz + w * tz + ux * ty - uy * tx], axis=-1)


def quat_matrix(q):
    x, y, z, w = q[..., 0], q[..., 1], q[..., 2], q[..., 3]
    return np.stack([1 - 2 * (y * y + z * z), 2 * (x * y - w * z), 2 * (x * z + w * y),
                     2 * (x * y + w * z), 1 - 2 * (x * x + z * z), 2 * (y * z - w * x),
                     2 * (x * z - w * y), 2 * (y * z + w * x), 1 - 2 * (x * x + y * y)],
                    axis=-1).reshape(q.shape[:-1] + (3, 3))


def relative_transforms(poses: np.ndarray, var_source, var_target):
    """T_ij = pose_compose(pose_inverse(T_j), T_i) (registration.py:264) for pose-table rows
    (quat xyzw, t); returns R (F,3,3), t (F,3)."""
    pi = poses[np.asarray(var_source)]
    pj = poses[np.asarray(var_target)]
    qinv = _qnorm(pj[:, :4] * np.array([-1.0, -1.0, -1.0, 1.0]))
    tinv = -_qapply(qinv, pj[:, 4:7])
    q = _qnorm(_qmul(qinv, pi[:, :4]))
    return quat_matrix(q), _qapply(qinv, pi[:, 4:7]) + tinv

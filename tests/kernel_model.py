"""NumPy model of the K4/K5 arithmetic (test infrastructure).

Restates what csrc/linearize.cu computes — the 29-value target-frame accumulation about the
source origin and its fp64 adjoint expansion — so the algebra can be checked on the CPU
against the oracle (in fp64: must agree to ~1e-12) and the fp32 tolerance budget predicted
before a GPU run (dtype=np.float32 emulates the per-point fp32 math and fp32 lane sums).
"""

import numpy as np

from oracle import vgicp_oracle as O


def _hat(v):
    return O._hat(v)


def compact(points, covs, vmap, R, t, dtype=np.float64, cov_dtype=np.float64, lane_chunk=16):
    """Return the 29-value compact record [P6 N9 S6 br3 bt3 cost inliers] (fp64).

    dtype=np.float64 is the kernel as built (all per-point math fp64).  dtype=np.float32 /
    cov_dtype=np.float32 model the rejected cheaper designs: fp32 per-point math (residual in
    cell-local fp32 coordinates, fp32 fused covariance and inverse, fp32 lane sums over
    `lane_chunk` points) and fp32-stored covariances.
    """
    res, keys, means, vcovs = vmap[0], vmap[1], vmap[2], vmap[3]
    R = np.asarray(R, float)
    t = np.asarray(t, float)
    moved = np.asarray(points, float) @ R.T + t
    rows = O.lookup(vmap, moved)
    hit = rows >= 0
    sel = rows[hit]
    x = moved[hit]
    C = np.asarray(covs, float)[hit].astype(cov_dtype).astype(np.float64)
    Cv = vcovs[sel].astype(cov_dtype).astype(np.float64)
    if dtype == np.float64:
        d = means[sel] - x
        W = O._inverse3(Cv + R @ C @ R.T)
    else:
        cc = (O.unpack_voxel_keys(keys[sel]).astype(float) + 0.5) * res
        d = (means[sel] - cc).astype(dtype) - (x - cc).astype(dtype)
        Rf = R.astype(dtype)
        W = O._inverse3(Cv.astype(dtype) + Rf @ C.astype(dtype) @ Rf.T)
    xp = (x - t).astype(dtype)
    wd = np.einsum("nij,nj->ni", W, d)
    cost = np.einsum("ni,ni->n", d, wd)
    H = _hat(xp)
    N = H @ W
    P = N @ np.swapaxes(H, 1, 2)
    br = np.cross(xp, wd)
    iu = np.triu_indices(3)
    per = np.concatenate([P[:, iu[0], iu[1]], N.reshape(-1, 9), W[:, iu[0], iu[1]], br, wd,
                          cost[:, None]], axis=1)
    if dtype != np.float64 and lane_chunk > 1:
        # fp32 lane sums over chunks of `lane_chunk` points, then fp64
        n = per.shape[0]
        pad = (-n) % lane_chunk
        per = np.concatenate([per, np.zeros((pad, per.shape[1]), dtype)])
        lanes = per.reshape(-1, lane_chunk, per.shape[1])
        acc = np.zeros((lanes.shape[0], per.shape[1]), dtype)
        for k in range(lane_chunk):
            acc = acc + lanes[:, k]
        total = acc.astype(np.float64).sum(0)
    else:
        total = per.astype(np.float64).sum(0)
    return np.concatenate([total, [float(hit.sum())]])


def expand(rec, R, t, unary=False):
    """fp64 adjoint expansion of a compact record (mirrors k_finalize)."""
    s = rec
    P = np.array([[s[0], s[1], s[2]], [s[1], s[3], s[4]], [s[2], s[4], s[5]]])
    N = s[6:15].reshape(3, 3)
    S = np.array([[s[15], s[16], s[17]], [s[16], s[18], s[19]], [s[17], s[19], s[20]]])
    br, bt = s[21:24], s[24:27]
    R = np.asarray(R, float)
    C = O._hat(np.asarray(t, float)[None])[0]
    Rd = np.zeros((6, 6))
    Rd[:3, :3] = R
    Rd[3:, 3:] = R
    E = np.eye(6)
    E[3:, :3] = -C
    Hp = np.block([[P, N], [N.T, S]])
    bp = np.concatenate([br, bt])
    out = {"h_ii": 2 * Rd.T @ Hp @ Rd, "b_i": -2 * Rd.T @ bp, "cost": s[27], "inliers": int(s[28])}
    if not unary:
        out["h_jj"] = 2 * E.T @ Hp @ E
        out["h_ij"] = -2 * Rd.T @ Hp @ E
        out["b_j"] = 2 * E.T @ bp
    return out


def within_tolerance(got, ref, rel=1e-4, abs_=1e-6):
    """Worst ratio |got - ref| / max(rel*|ref|, abs) over elements (<= 1 passes)."""
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    return float(np.max(np.abs(got - ref) / np.maximum(rel * np.abs(ref), abs_)))

"""GPU parity: libvgicp (through the drop-in API / C-ABI) vs the pinned CPU oracle and the
reference's golden fixtures.  Bar: bit-exact keys, rows, inliers, voxel-map arrays; H/b/cost
within 1e-4 relative, 1e-6 absolute, per element."""

import numpy as np
import pytest

from oracle import vgicp_oracle as O
from paper_2202_00242_b200 import _lib, synthetic
from paper_2202_00242_b200 import geometry as G
from paper_2202_00242_b200 import registration as RG
from paper_2202_00242_b200.errors import DegenerateConstraint
from paper_2202_00242_b200.factor_graph import MatchingCostFactor, submap_key
from paper_2202_00242_b200.preprocess import make_frame

pytestmark = pytest.mark.gpu

REL, ABS = 1e-4, 1e-6  # north_star parity tolerance for fp32 H/b/error vs fp64
NAMES = ("h_ii", "b_i", "h_ij", "h_jj", "b_j")


def assert_tol(got, ref, what=""):
    got, ref = np.asarray(got, float), np.asarray(ref, float)
    assert got.shape == ref.shape, what
    bad = np.abs(got - ref) > np.maximum(REL * np.abs(ref), ABS)
    assert not bad.any(), f"{what}: worst ratio " \
        f"{np.max(np.abs(got - ref) / np.maximum(REL * np.abs(ref), ABS)):.3g}"


def assert_lin(lin, ref, unary):
    assert lin.inlier_count == ref["inliers"]
    assert_tol(lin.cost, ref["cost"], "cost")
    assert_tol(lin.h_ii, ref["h_ii"], "h_ii")
    assert_tol(lin.b_i, ref["b_i"], "b_i")
    if unary:
        assert lin.h_ij is None and lin.h_jj is None and lin.b_j is None
    else:
        for k in ("h_ij", "h_jj", "b_j"):
            assert_tol(getattr(lin, k), ref[k], k)


def pose_from_Rt(R, t):
    return G.Se3Pose(G.Rotation(_quat_from_matrix(R)), t)


def _quat_from_matrix(m):
    tr = m[0, 0] + m[1, 1] + m[2, 2]
    s = np.sqrt(tr + 1.0) * 2.0
    return np.array([(m[2, 1] - m[1, 2]) / s, (m[0, 2] - m[2, 0]) / s, (m[1, 0] - m[0, 1]) / s,
                     0.25 * s])


class _TPose:
    """A transform handed over exactly (R, t) — bypasses quaternion round trips."""

    class _Rot:
        def __init__(self, R):
            self._R = R

        def matrix(self):
            return self._R

    def __init__(self, R, t):
        self.rotation = self._Rot(np.asarray(R, float))
        self.translation = np.asarray(t, float)


def golden_map(g, res=0.5):
    tag = str(res).replace(".", "p")
    return (res, g[f"map{tag}_keys"], g[f"map{tag}_means"], g[f"map{tag}_covs"],
            g[f"map{tag}_counts"])


# ---- keys / maps ----------------------------------------------------------------------------

def test_pack_voxel_keys_bit_exact(golden):
    from paper_2202_00242_b200.preprocess import pack_voxel_keys

    g = golden("keys")
    for res in (0.25, 0.4, 0.5, 1.0, 2.0):
        assert np.array_equal(pack_voxel_keys(g["points"], res), g[f"keys_{res}"]), res


@pytest.mark.parametrize("res", [0.5, 1.0])
def test_build_voxelmap_bit_exact(golden, res):
    g = golden("registration")
    frame = make_frame(g["tgt_points"], g["tgt_covs"])
    vm = RG.build_voxelmap(frame, res)
    tag = str(res).replace(".", "p")
    assert len(vm) == len(g[f"map{tag}_keys"])
    assert np.array_equal(vm.keys, g[f"map{tag}_keys"])
    assert np.array_equal(vm.counts, g[f"map{tag}_counts"])
    assert np.array_equal(vm.means, g[f"map{tag}_means"])
    assert np.array_equal(vm.covs, g[f"map{tag}_covs"])


@pytest.mark.parametrize("res", [0.5, 2.0, 8.0])
def test_build_voxelmap_big_cells_bit_exact(res):
    """A 131,072-point scan (config 2) with coarse cells of up to tens of thousands of
    points: the warp-per-cell path for cells of >= 16 points keeps np.add.at's sequential
    order, so keys/counts/means/covs equal the oracle's bit for bit."""
    from paper_2202_00242_b200 import synthetic

    pts = synthetic.scan(synthetic.yaw_pose(0.2, [1.0, -2.0, 0.0]), synthetic.ray_table(1024, 128),
                         np.random.default_rng(2))
    rng = np.random.default_rng(9)
    a = rng.normal(size=(len(pts), 3, 3))
    covs = a @ np.swapaxes(a, 1, 2) * 0.01
    vm = RG.build_voxelmap(make_frame(pts, covs), res)
    ref = O.build_voxelmap(pts, covs, res)
    assert vm.counts.max() >= (96 if res >= 2.0 else 16)
    assert np.array_equal(vm.keys, ref[1]) and np.array_equal(vm.counts, ref[4])
    assert np.array_equal(vm.means, ref[2]) and np.array_equal(vm.covs, ref[3])


def test_build_voxelmap_requires_covs_and_handles_empty():
    with pytest.raises(ValueError):
        RG.build_voxelmap(make_frame(np.zeros((3, 3))), 1.0)
    assert len(RG.build_voxelmap(make_frame(np.zeros((0, 3)), np.zeros((0, 3, 3))), 1.0)) == 0


# ---- lookup / match / linearize at the golden cases -----------------------------------------

@pytest.mark.parametrize("adopt", [False, True])
@pytest.mark.parametrize("case", range(6))
def test_golden_cases(golden, case, adopt):
    """adopt=True: map handed over as reference arrays (vg_map_from_arrays);
    adopt=False: map built on the GPU (vg_map_build)."""
    g = golden("registration")
    src = make_frame(g["src_points"], g["src_covs"])
    if adopt:
        _, k, mu, c, n = golden_map(g)
        vm = RG.GaussianVoxelMap(0.5, k, mu, c, n)
    else:
        vm = RG.build_voxelmap(make_frame(g["tgt_points"], g["tgt_covs"]), 0.5)
    R, t = g[f"case{case}_R"], g[f"case{case}_t"]
    tij = _TPose(R, t)
    unary = bool(g[f"case{case}_unary"])
    terms = RG.match_terms(src, vm, tij)
    assert np.array_equal(terms.rows, g[f"case{case}_rows"])
    assert terms.inliers == int(g[f"case{case}_inliers"])
    assert_tol(terms.cost, g[f"case{case}_cost"], "cost")
    assert RG.overlap_rate(src, vm, tij) == float(g[f"case{case}_overlap"])
    c, n = RG.matching_cost(src, vm, tij)
    assert n == int(g[f"case{case}_inliers"])
    assert_tol(c, g[f"case{case}_cost"], "matching_cost")
    lin = RG.linearize_from_terms(src, terms, tij, target_fixed=unary)
    ref = {k: (g[f"case{case}_{k}"] if f"case{case}_{k}" in g.files else None)
           for k in NAMES + ("cost", "inliers")}
    ref["inliers"] = int(ref["inliers"])
    assert_lin(lin, ref, unary)


def test_match_terms_per_point(golden):
    g = golden("registration")
    src = make_frame(g["src_points"], g["src_covs"])
    vm_t = golden_map(g)
    vm = RG.GaussianVoxelMap(0.5, *vm_t[1:])
    R, t = g["case1_R"], g["case1_t"]
    ours = RG.match_terms(src, vm, _TPose(R, t))
    ref = O.match_terms(g["src_points"], g["src_covs"], vm_t, R, t)
    assert np.array_equal(ours.hit, ref["hit"])
    np.testing.assert_allclose(ours.moved, ref["moved"], rtol=0, atol=1e-12)
    np.testing.assert_allclose(ours.d, ref["d"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(ours.weight, ref["weight"], rtol=1e-5, atol=1e-4)
    np.testing.assert_allclose(ours.wd, ref["wd"], rtol=1e-4, atol=1e-4)


def test_lookup_and_cell(golden):
    g = golden("registration")
    vm_t = golden_map(g)
    vm = RG.GaussianVoxelMap(0.5, *vm_t[1:])
    pts = np.random.default_rng(3).uniform(-4, 4, (5000, 3))
    assert np.array_equal(vm.lookup(pts), O.lookup(vm_t, pts))
    idx = vm.occupied_indices()[7]
    mean, cov, cnt = vm.cell(idx)
    assert np.array_equal(mean, vm_t[2][7]) and cnt == vm_t[4][7]
    with pytest.raises(KeyError):
        vm.cell([10000, 0, 0])


def test_non_fp32_points_keep_exact_keys():
    """Points that are not fp32-representable take the fp64 path: rows stay bit-exact."""
    rng = np.random.default_rng(12)
    tgt = rng.uniform(-3, 3, (3000, 3))  # fp64, not fp32-exact
    covs = np.tile(np.eye(3) * 0.01, (3000, 1, 1))
    vm = RG.build_voxelmap(make_frame(tgt, covs), 0.5)
    ref_map = O.build_voxelmap(tgt, covs, 0.5)
    assert np.array_equal(vm.keys, ref_map[1]) and np.array_equal(vm.means, ref_map[2])
    src = tgt[:1500] + rng.normal(scale=0.02, size=(1500, 3))
    R = G.so3_exp([0.01, -0.02, 0.03]).matrix()
    t = np.array([0.05, -0.02, 0.01])
    terms = RG.match_terms(make_frame(src, covs[:1500]), vm, _TPose(R, t))
    ref = O.match_terms(src, covs[:1500], ref_map, R, t)
    assert np.array_equal(terms.rows, ref["rows"])


# ---- config 1 at full size ------------------------------------------------------------------

@pytest.fixture(scope="module")
def config1():
    source, target, t_i, t_j = synthetic.config1_scans()
    cs, _ = O.estimate_covariances(source, O.knn_search(source, 10))
    ct, _ = O.estimate_covariances(target, O.knn_search(target, 10))
    return source, cs, target, ct, t_i, t_j


def test_config1_single_factor(config1, golden):
    source, cs, target, ct, t_i, t_j = config1
    vm = RG.build_voxelmap(make_frame(target, ct), 0.5)
    ref_map = O.build_voxelmap(target, ct, 0.5)
    assert np.array_equal(vm.keys, ref_map[1])
    assert np.array_equal(vm.means, ref_map[2]) and np.array_equal(vm.covs, ref_map[3])
    src = make_frame(source, cs)
    lin = RG.linearize_matching_cost(src, vm, t_i, t_j)
    tij = G.pose_compose(G.pose_inverse(t_j), t_i)
    R, t = tij.rotation.matrix(), tij.translation
    ref = O.linearize(source, cs, ref_map, R, t)
    assert_lin(lin, ref, False)
    # correspondence rows bit-exact; count points within 1e-12*res of a voxel face (expect 0)
    moved = source @ R.T + t
    frac = moved / 0.5 - np.floor(moved / 0.5)
    near_face = np.sum((frac < 1e-12) | (frac > 1 - 1e-12))
    assert near_face == 0
    terms = RG.match_terms(src, vm, tij)
    assert np.array_equal(terms.rows, O.lookup(ref_map, moved))
    assert lin.inlier_count == int(golden("config1")["inliers"])


def test_config1_converged_pose(config1):
    """b -> 0 with heavy cancellation at the true pose; the 1e-6 absolute floor carries it."""
    source, cs, target, ct, _, _ = config1
    vm = RG.build_voxelmap(make_frame(target, ct), 0.5)
    ref_map = O.build_voxelmap(target, ct, 0.5)
    p_i = synthetic.yaw_pose(0.05, [0.3, 0.1, 0.0])
    lin = RG.linearize_matching_cost(make_frame(source, cs), vm, p_i, G.Se3Pose.identity())
    tij = G.pose_compose(G.pose_inverse(G.Se3Pose.identity()), p_i)
    ref = O.linearize(source, cs, ref_map, tij.rotation.matrix(), tij.translation)
    assert_lin(lin, ref, False)


# ---- batched path (pose table, many factors) ------------------------------------------------

@pytest.fixture(scope="module")
def small_graph():
    """12 submaps in the room, 600-point sources vs 1.0 m maps, nearest-5 factors."""
    rng = np.random.default_rng(21)
    poses = synthetic.random_submap_poses(rng, 12)
    dirs = synthetic.ray_table(128, 32)
    scans, covs, maps, srcs = [], [], [], []
    for i, p in enumerate(poses):
        s = synthetic.scan(p, dirs, np.random.default_rng(100 + i))
        c, _ = O.estimate_covariances(s, O.knn_search(s, 10))
        scans.append(s)
        covs.append(c)
        maps.append(O.build_voxelmap(s, c, 1.0))
        sel = np.sort(rng.choice(len(s), 600, replace=False))
        srcs.append((s[sel], c[sel]))
    pairs = synthetic.nearest_pairs(poses, 5)
    est = [G.pose_retract(p, synthetic.perturbation(rng, 0.05, 1.0)) for p in poses]
    return poses, est, scans, covs, maps, srcs, pairs


def test_batch_pose_table_vs_oracle(small_graph):
    poses, est, scans, covs, maps, srcs, pairs = small_graph
    clouds = [_lib.DeviceCloud(s, c) for s, c in srcs]
    dmaps = [_lib.DeviceMap.build(_lib.DeviceCloud(s, c), 1.0) for s, c in zip(scans, covs)]
    F = len(pairs)
    unary = [(f % 7) == 3 for f in range(F)]
    table = np.array([G.pose_row(p) for p in est])
    batch = _lib.DeviceBatch([clouds[i] for i, _ in pairs], [dmaps[j] for _, j in pairs], unary,
                             [10] * F, pairs[:, 0], pairs[:, 1])
    out = batch.linearize_poses(table, _lib.MODE_LINEARIZE)
    cost_out = batch.linearize_poses(table, _lib.MODE_COST)
    R, t = O.relative_transforms(table, pairs[:, 0], pairs[:, 1])
    checked = 0
    for f, (i, j) in enumerate(pairs):
        try:
            ref = O.linearize(srcs[i][0], srcs[i][1], maps[j], R[f], t[f], target_fixed=unary[f])
        except ValueError:  # degenerate: zero blocks, inliers below the gate
            assert np.all(out[f][:90] == 0) and out[f][91] < 10
            continue
        assert_lin(RG.unpack_record(out[f], unary[f]), ref, unary[f])
        assert cost_out[f][1] == ref["inliers"]
        assert_tol(cost_out[f][0], ref["cost"], "cost mode")
        checked += 1
    assert checked >= F // 2


def test_batch_explicit_transforms_and_determinism(small_graph):
    poses, est, scans, covs, maps, srcs, pairs = small_graph
    clouds = [_lib.DeviceCloud(s, c) for s, c in srcs]
    dmaps = [_lib.DeviceMap.build(_lib.DeviceCloud(s, c), 1.0) for s, c in zip(scans, covs)]
    F = len(pairs)
    batch = _lib.DeviceBatch([clouds[i] for i, _ in pairs], [dmaps[j] for _, j in pairs],
                             [False] * F, [10] * F)
    table = np.array([G.pose_row(p) for p in est])
    R, t = O.relative_transforms(table, pairs[:, 0], pairs[:, 1])
    T = np.concatenate([R.reshape(F, 9), t], axis=1)
    a = batch.linearize(T)
    b = batch.linearize(T)
    assert np.array_equal(a, b)  # bitwise deterministic
    pt = _lib.DeviceBatch([clouds[i] for i, _ in pairs], [dmaps[j] for _, j in pairs],
                          [False] * F, [10] * F, pairs[:, 0], pairs[:, 1]).linearize_poses(table)
    for f in range(F):
        if a[f][91] >= 10:
            assert_tol(pt[f], a[f], "pose-table vs explicit")


# ---- drop-in factor semantics ---------------------------------------------------------------

def test_factor_degenerate_and_empty():
    a = make_frame([[0, 0, 0]], np.eye(3)[None] * 0.01)
    b = make_frame([[50, 0, 0]], np.eye(3)[None] * 0.01)
    vm = RG.build_voxelmap(b, 0.5)
    assert RG.matching_cost(a, vm, G.Se3Pose.identity()) == (0.0, 0)
    with pytest.raises(DegenerateConstraint):
        RG.linearize_matching_cost(a, vm, G.Se3Pose.identity(), G.Se3Pose.identity())
    f = MatchingCostFactor(submap_key(0), a, vm, key_target=submap_key(1))
    vals = {submap_key(0): G.Se3Pose.identity(), submap_key(1): G.Se3Pose.identity()}
    assert f.cost(vals) == 0.0
    lin = f.linearize(vals)
    assert lin.cost == 0.0 and all(np.all(h == 0) for h in lin.h.values())
    empty = make_frame(np.zeros((0, 3)), np.zeros((0, 3, 3)))
    assert RG.overlap_rate(empty, vm, G.Se3Pose.identity()) == 0.0
    with pytest.raises(DegenerateConstraint):
        RG.linearize_matching_cost(empty, vm, G.Se3Pose.identity(), G.Se3Pose.identity())


@pytest.mark.parametrize("target", [9000, 33000])
def test_staged_host_output_matches_single_launch(small_graph, target):
    """Batches of >= 8192 factors run K4/K5 in stages whose records are copied to the host
    while the next stage computes (from 32,768 factors: 8 geometric stages over two compute
    streams); results must equal the one-launch device path bit for bit (same items, same
    fixed-order sums), and the small batch of the test above to rounding."""
    import torch

    poses, est, scans, covs, maps, srcs, pairs = small_graph
    clouds = [_lib.DeviceCloud(s, c) for s, c in srcs]
    dmaps = [_lib.DeviceMap.build(_lib.DeviceCloud(s, c), 1.0) for s, c in zip(scans, covs)]
    reps = target // len(pairs) + 1
    rng = np.random.default_rng(5)
    sel = rng.permutation(np.tile(np.arange(len(pairs)), reps))   # 4 or 8 stages
    P = pairs[sel]
    F = len(P)
    unary = [(int(s) % 7) == 3 for s in sel]
    table = np.array([G.pose_row(p) for p in est])
    big = _lib.DeviceBatch([clouds[i] for i, _ in P], [dmaps[j] for _, j in P], unary, [10] * F,
                           P[:, 0], P[:, 1])
    small = _lib.DeviceBatch([clouds[i] for i, _ in pairs], [dmaps[j] for _, j in pairs],
                             [(f % 7) == 3 for f in range(len(pairs))], [10] * len(pairs),
                             pairs[:, 0], pairs[:, 1])
    ref = small.linearize_poses(table)
    for mode in (_lib.MODE_LINEARIZE, _lib.MODE_COST, _lib.MODE_COMPACT, _lib.MODE_INLIERS):
        host = big.linearize_poses(table, mode)
        dev = torch.zeros((F, _lib.RECORD_SIZE[mode]), dtype=torch.float64, device="cuda")
        tdev = torch.from_numpy(table).cuda()
        torch.cuda.synchronize()
        big.linearize_poses_device(tdev.data_ptr(), len(table), mode, dev.data_ptr())
        big.ctx.synchronize()
        assert np.array_equal(host, dev.cpu().numpy()), mode
        if mode == _lib.MODE_LINEARIZE:
            # the small batch splits sources into smaller work items (more parallelism), so
            # its per-item partial sums round differently: equal to fp64 rounding only
            for f in range(0, F, 97):
                if ref[sel[f]][91] >= 10:
                    assert_tol(host[f], ref[sel[f]], "staged vs small batch")
                else:
                    assert host[f][91] == ref[sel[f]][91]


def test_device_normal_equations_match_host_assembly(small_graph):
    """vg_batch_assemble_*: every block is the factor-order sum of the factors' blocks,
    bit for bit (same additions as a sequential host sum), unary targets are constants, and
    the dense form matches the reference's _assemble_dense scatter (factor_graph.py:522-536)."""
    poses, est, scans, covs, maps, srcs, pairs = small_graph
    clouds = [_lib.DeviceCloud(s, c) for s, c in srcs]
    dmaps = [_lib.DeviceMap.build(_lib.DeviceCloud(s, c), 1.0) for s, c in zip(scans, covs)]
    F, V = len(pairs), len(est)
    unary = [(f % 7) == 3 for f in range(F)]
    fixed = [G.pose_row(G.pose_retract(poses[j], np.full(6, 0.01))) for _, j in pairs]
    vs = pairs[:, 0].copy()
    vt = np.array([V + f if unary[f] else pairs[f, 1] for f in range(F)])
    table = np.vstack([np.array([G.pose_row(p) for p in est]), np.array(fixed)])
    batch = _lib.DeviceBatch([clouds[i] for i, _ in pairs], [dmaps[j] for _, j in pairs], unary,
                             [10] * F, vs, vt)
    prs = batch.assemble_setup(V)
    rec = batch.linearize_poses(table)
    ne = batch.assemble_poses(table)
    # host: sequential sums in factor order
    diag = np.zeros((V, 21))
    grad = np.zeros((V, 6))
    off = {tuple(p): np.zeros(36) for p in prs}
    cost, count = 0.0, 0
    for f in range(F):
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
        blk = r[21:57] if vs[f] < vt[f] else r[21:57].reshape(6, 6).T.ravel()
        off[(a, b)] += blk
    iu = np.triu_indices(6)
    assert np.array_equal(ne.diag[:, iu[0], iu[1]], diag)
    assert np.array_equal(ne.grad, grad)
    assert set(map(tuple, prs)) == set(off) and np.all(prs[:, 0] < prs[:, 1])
    for p, blk in zip(prs, ne.off):
        assert np.array_equal(blk.ravel(), off[tuple(p)])
    assert ne.count == count and abs(ne.cost - cost) <= 1e-12 * abs(cost)
    # dense form vs the reference's per-factor scatter of the unpacked linearizations
    h_ref = np.zeros((6 * V, 6 * V))
    g_ref = np.zeros(6 * V)
    for f in range(F):
        lin = RG.unpack_record(rec[f], unary[f])
        i = vs[f]
        h_ref[6 * i:6 * i + 6, 6 * i:6 * i + 6] += lin.h_ii
        g_ref[6 * i:6 * i + 6] += lin.b_i
        if unary[f]:
            continue
        j = vt[f]
        h_ref[6 * j:6 * j + 6, 6 * j:6 * j + 6] += lin.h_jj
        h_ref[6 * i:6 * i + 6, 6 * j:6 * j + 6] += lin.h_ij
        h_ref[6 * j:6 * j + 6, 6 * i:6 * i + 6] += lin.h_ij.T
        g_ref[6 * j:6 * j + 6] += lin.b_j
    h, g = ne.dense()
    assert np.allclose(h, h_ref, rtol=1e-12, atol=1e-9) and np.allclose(g, g_ref, rtol=1e-12, atol=1e-9)


def test_overlap_rates_and_keyframe_matrix(small_graph):
    """Batched overlap_rate / keyframe overlap matrix (odometry.py:396-403) equal the oracle's
    per-pair overlap_rate exactly (integer hit counts / n); empty inputs give 0."""
    poses, est, scans, covs, maps, srcs, pairs = small_graph
    frames = [make_frame(s, c) for s, c in srcs[:6]]
    vmaps = [RG.build_voxelmap(make_frame(s, c), 1.0) for s, c in zip(scans[:6], covs[:6])]
    m = RG.overlap_matrix(frames, vmaps, est[:6])
    for i in range(6):
        assert m[i, i] == 0.0
        for j in range(6):
            if i == j:
                continue
            tij = G.pose_compose(G.pose_inverse(est[j]), est[i])
            ref = O.overlap_rate(srcs[i][0], maps[j], tij.rotation.matrix(), tij.translation)
            assert m[i, j] == ref
            assert RG.overlap_rate(frames[i], vmaps[j], tij) == ref
    # frames without covariances work for overlap (lookups only); empty frames give 0
    bare = make_frame(srcs[0][0], None)
    empty = make_frame(np.zeros((0, 3)), np.zeros((0, 3, 3)))
    r = RG.overlap_rates([bare, empty], [vmaps[1], vmaps[1]],
                         [G.pose_compose(G.pose_inverse(est[1]), est[0])] * 2)
    assert r[0] == m[0, 1] and r[1] == 0.0


def test_sharded_normal_equations_share_the_global_layout(small_graph):
    """Two factor shards assembled in the global pair layout (vg_batch_assemble_setup_pairs,
    what every rank of a sharded graph does before the sum-reduction) add up to the
    single-batch system."""
    from paper_2202_00242_b200 import sharding

    poses, est, scans, covs, maps, srcs, pairs = small_graph
    clouds = [_lib.DeviceCloud(s, c) for s, c in srcs]
    dmaps = [_lib.DeviceMap.build(_lib.DeviceCloud(s, c), 1.0) for s, c in zip(scans, covs)]
    F, V = len(pairs), len(est)
    table = np.array([G.pose_row(p) for p in est])
    unary = np.zeros(F, bool)
    gp = sharding.global_pairs(pairs[:, 0], pairs[:, 1], unary, V)

    def system(ids, layout):
        b = _lib.DeviceBatch([clouds[pairs[f, 0]] for f in ids], [dmaps[pairs[f, 1]] for f in ids],
                             [False] * len(ids), [10] * len(ids), pairs[ids, 0], pairs[ids, 1])
        b.assemble_setup(V, layout)
        return b.assemble_poses(table, unpack=False)

    full = system(np.arange(F), None)
    shards = sharding.lpt_shards(np.ones(F), 2)
    parts = [system(s, gp) for s in shards]
    assert full.shape == parts[0].shape == parts[1].shape
    tot = parts[0] + parts[1]
    assert np.allclose(tot, full, rtol=1e-12, atol=1e-9 * np.abs(full).max())
    # a layout missing one of the batch's pairs is rejected
    with pytest.raises(Exception):
        system(np.arange(F), gp[1:])


@pytest.mark.parametrize("res,wide", [(0.3, False), (1.0, True)])
def test_batch_general_paths_vs_oracle(small_graph, res, wide):
    """Batches off the fast path: a non-power-of-two resolution (IEEE-division key fallback,
    generic K4a), maps whose cells exceed the 32-bit local key frame (a far outlier point:
    int64 keys, kmode 0), and non-fp32 source points (fp64 staging in K4b)."""
    poses, est, scans, covs, maps, srcs, pairs = small_graph
    sel = pairs[:8]
    table = np.array([G.pose_row(p) for p in est])
    R, t = O.relative_transforms(table, sel[:, 0], sel[:, 1])
    rng = np.random.default_rng(9)
    for jitter in (False, True):
        clouds, dmaps, refs = [], [], []
        for f, (i, j) in enumerate(sel):
            pts = srcs[i][0] + (rng.normal(scale=1e-9, size=srcs[i][0].shape) if jitter else 0.0)
            tp, tc = scans[j], covs[j]
            if wide and f % 2 == 0:  # a cell 3 km away: the key extent no longer fits 11 bits
                # (every other map: the batch mixes 32-bit and int64 key tables)
                tp = np.vstack([tp, [[3000.25, 0.25, 0.25]]])
                tc = np.concatenate([tc, np.eye(3)[None] * 0.01])
            clouds.append(_lib.DeviceCloud(pts, srcs[i][1]))
            dmaps.append(_lib.DeviceMap.build(_lib.DeviceCloud(tp, tc), res))
            refs.append((pts, O.build_voxelmap(tp, tc, res)))
        batch = _lib.DeviceBatch(clouds, dmaps, [False] * len(sel), [10] * len(sel),
                                 sel[:, 0], sel[:, 1])
        out = batch.linearize_poses(table)
        checked = 0
        for f in range(len(sel)):
            pts, vmap = refs[f]
            try:
                ref = O.linearize(pts, srcs[sel[f, 0]][1], vmap, R[f], t[f])
            except ValueError:
                assert out[f][91] < 10
                continue
            assert_lin(RG.unpack_record(out[f], False), ref, False)
            checked += 1
        assert checked >= len(sel) // 2


def test_general_source_covariances_vs_oracle(small_graph):
    """Source covariances of the plane form alpha I - kappa n n^T (everything
    estimate_covariances makes, alpha = 1; and alpha = 2) take K4b's 21-op path, general SPD
    ones the R C R^T path; all match the oracle."""
    poses, est, scans, covs, maps, srcs, pairs = small_graph
    sel = pairs[:10]
    table = np.array([G.pose_row(p) for p in est])
    R, t = O.relative_transforms(table, sel[:, 0], sel[:, 1])
    rng = np.random.default_rng(12)
    dmaps = {j: _lib.DeviceMap.build(_lib.DeviceCloud(scans[j], covs[j]), 1.0)
             for j in np.unique(sel[:, 1])}
    for form in ("unit plane", "scaled plane", "small plane", "general"):
        clouds, ccovs = [], []
        for i, _ in sel:
            c = srcs[i][1]
            if form == "scaled plane":  # 2 (I - kappa n n^T): plane form with alpha = 2
                c = 2.0 * c
            elif form == "small plane":  # alpha = 1e-3: the fit tolerance is relative
                c = 1e-3 * c
            elif form == "general":
                a = rng.normal(scale=0.3, size=(len(c), 3, 3))
                c = c + np.einsum("nij,nkj->nik", a, a) * 0.1   # SPD, not plane form
            clouds.append(_lib.DeviceCloud(srcs[i][0], c))
            ccovs.append(c)
        batch = _lib.DeviceBatch(clouds, [dmaps[j] for j in sel[:, 1]], [False] * len(sel),
                                 [10] * len(sel), sel[:, 0], sel[:, 1])
        out = batch.linearize_poses(table)
        checked = 0
        for f, (i, j) in enumerate(sel):
            try:
                ref = O.linearize(srcs[i][0], ccovs[f], maps[j], R[f], t[f])
            except ValueError:
                assert out[f][91] < 10
                continue
            assert_lin(RG.unpack_record(out[f], False), ref, False)
            checked += 1
        assert checked >= len(sel) // 2


@pytest.fixture(scope="module")
def config5():
    from paper_2202_00242_b200 import workloads

    return workloads.global_mapping()


def test_config5_full_size_sample_vs_oracle_and_invariants(config5):
    """The headline workload at full size (1,000 submaps, 50,000 factors, 19.9M
    correspondences): a seeded sample of factors matches the oracle (bit-exact inliers,
    blocks within tolerance), repeated linearizations are bitwise identical, and the staged
    host path equals the one-launch device path bit for bit."""
    import torch

    wl = config5
    batch = wl.batch()
    table = wl.pose_table
    F = len(wl.pairs)
    host = batch.linearize_poses(table)
    host2 = batch.linearize_poses(table)
    assert np.array_equal(host, host2)
    dev = torch.zeros((F, 92), dtype=torch.float64, device="cuda")
    poses = torch.from_numpy(table).cuda()
    torch.cuda.synchronize()
    batch.linearize_poses_device(poses.data_ptr(), len(table), _lib.MODE_LINEARIZE, dev.data_ptr())
    batch.ctx.synchronize()
    assert np.array_equal(host, dev.cpu().numpy())
    # oracle on a seeded sample (the oracle recomputes maps from the same host inputs)
    rng = np.random.default_rng(55)
    sample = rng.choice(F, 24, replace=False)
    R, t = O.relative_transforms(table, wl.pairs[sample, 0], wl.pairs[sample, 1])
    maps = {}
    checked = 0
    for k, f in enumerate(sample):
        i, j = wl.pairs[f]
        if j not in maps:
            maps[j] = O.build_voxelmap(wl.scans[j], wl.scan_covs[j], wl.resolution)
        sel = wl.source_index[i]
        try:
            ref = O.linearize(wl.scans[i][sel], wl.scan_covs[i][sel], maps[j], R[k], t[k])
        except ValueError:
            assert host[f][91] < 10
            continue
        assert_lin(RG.unpack_record(host[f], False), ref, False)
        checked += 1
    assert checked >= 12


def test_assemble_records_device_equals_assemble_poses(small_graph):
    """K6 alone over finalize_device's records (what each rank runs in the sharded step) gives
    the same system as the one-call assemble_poses."""
    import torch

    poses, est, scans, covs, maps, srcs, pairs = small_graph
    clouds = [_lib.DeviceCloud(s, c) for s, c in srcs]
    dmaps = [_lib.DeviceMap.build(_lib.DeviceCloud(s, c), 1.0) for s, c in zip(scans, covs)]
    F, V = len(pairs), len(est)
    table = np.array([G.pose_row(p) for p in est])
    b = _lib.DeviceBatch([clouds[i] for i, _ in pairs], [dmaps[j] for _, j in pairs],
                         [False] * F, [10] * F, pairs[:, 0], pairs[:, 1])
    b.assemble_setup(V)
    ref = b.assemble_poses(table, unpack=False)
    tp = torch.from_numpy(table).cuda()
    rec = torch.zeros((F, 92), dtype=torch.float64, device="cuda")
    ne = torch.zeros(b.asm_size, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    b.compose_device(tp.data_ptr(), V)
    b.accumulate_device(_lib.MODE_LINEARIZE)
    b.finalize_device(_lib.MODE_LINEARIZE, rec.data_ptr())
    b.assemble_records_device(rec.data_ptr(), ne.data_ptr())
    b.ctx.synchronize()
    assert np.array_equal(ne.cpu().numpy(), ref)


@pytest.mark.parametrize("wide", [False, True])
def test_hash_stress_every_cell_and_misses(wide):
    """A 150k-cell map (many overflowing 16 B buckets, and an int64-key map when `wide`):
    every occupied cell's centre finds its reference row, and random points match the
    oracle's binary search, including misses."""
    rng = np.random.default_rng(77)
    cells = np.unique(rng.integers(0, 200, (160000, 3)) * [1, 1, 1], axis=0)
    if wide:
        cells = np.vstack([cells, [[5000, 3, 3]]])
    pts = (cells + 0.5) * 0.25
    covs = np.broadcast_to(np.eye(3) * 0.01, (len(pts), 3, 3)).copy()
    ref = O.build_voxelmap(pts, covs, 0.25)
    vm = RG.build_voxelmap(make_frame(pts, covs), 0.25)
    assert np.array_equal(vm.keys, ref[1])
    rows = vm.lookup(pts)
    assert np.array_equal(rows, O.lookup(ref, pts)) and np.all(rows >= 0)
    q = rng.uniform(-1, 52, (200000, 3))
    assert np.array_equal(vm.lookup(q), O.lookup(ref, q))


@pytest.mark.parametrize("name", ["odometry_window", "local_mapping"])
def test_configs_3_and_4_full_size_sample_vs_oracle(name):
    """BASELINE configs 3 (69 factors of 16,384-point frames at 0.5/1.0/2.0 m, 15 unary) and
    4 (4,950 factors of 8,192-point frames at 0.5 m) at full size: the batch path's records
    for a seeded sample of factors match the oracle (bit-exact inliers, blocks within
    1e-4 rel / 1e-6 abs), and the host and device paths agree bit for bit."""
    import torch

    from paper_2202_00242_b200 import workloads

    wl = getattr(workloads, name)()
    batch = wl.batch()
    table = wl.pose_table
    F = len(wl.clouds)
    host = batch.linearize_poses(table)
    dev = torch.zeros((F, 92), dtype=torch.float64, device="cuda")
    poses = torch.from_numpy(table).cuda()
    torch.cuda.synchronize()
    batch.linearize_poses_device(poses.data_ptr(), len(table), _lib.MODE_LINEARIZE, dev.data_ptr())
    batch.ctx.synchronize()
    assert np.array_equal(host, dev.cpu().numpy())
    rng = np.random.default_rng(66)
    gated_in = np.flatnonzero(host[:, 91] >= 10)
    sample = np.unique(np.concatenate([rng.choice(gated_in, min(len(gated_in), 10), replace=False),
                                       rng.choice(F, min(F, 4), replace=False)]))
    R, t = O.relative_transforms(table, wl.var_source[sample], wl.var_target[sample])
    checked = 0
    for k, f in enumerate(sample):
        pts, covs = wl.host_sources[f]
        tp, tc, res = wl.host_targets[f]
        vmap = O.build_voxelmap(tp, tc, res)
        try:
            ref = O.linearize(pts, covs, vmap, R[k], t[k], target_fixed=bool(wl.unary[f]))
        except ValueError:
            assert host[f][91] < 10
            continue
        assert_lin(RG.unpack_record(host[f], bool(wl.unary[f])), ref, bool(wl.unary[f]))
        checked += 1
    assert checked >= 7


# ---- round 2: ADVICE regressions ------------------------------------------------------------

def test_empty_source_inside_a_batch(small_graph):
    """A factor whose source cloud has no points gets no work item (its point arrays are never
    read): zero record, and its neighbours in the batch are unaffected — also when the empty
    factor is the last one (K-compose must not write a header past the item table)."""
    poses, est, scans, covs, maps, srcs, pairs = small_graph
    empty = _lib.DeviceCloud(np.zeros((0, 3)), np.zeros((0, 3, 3)))
    clouds = [_lib.DeviceCloud(s, c) for s, c in srcs[:3]]
    dmaps = [_lib.DeviceMap.build(_lib.DeviceCloud(s, c), 1.0) for s, c in zip(scans[:3], covs[:3])]
    table = np.array([G.pose_row(p) for p in est[:3]])
    solo = _lib.DeviceBatch([clouds[0], clouds[1]], [dmaps[1], dmaps[0]], [False] * 2, [10] * 2,
                            [0, 1], [1, 0]).linearize_poses(table)
    for order in ([empty, clouds[0], clouds[1]], [clouds[0], clouds[1], empty]):
        maps_ = [dmaps[2] if c is empty else (dmaps[1] if c is clouds[0] else dmaps[0])
                 for c in order]
        vs = [2 if c is empty else (0 if c is clouds[0] else 1) for c in order]
        vt = [0 if c is empty else (1 if c is clouds[0] else 0) for c in order]
        b = _lib.DeviceBatch(order, maps_, [False] * 3, [10] * 3, vs, vt)
        for mode in (_lib.MODE_LINEARIZE, _lib.MODE_COST, _lib.MODE_INLIERS):
            out = b.linearize_poses(table, mode)
            k = [i for i, c in enumerate(order) if c is empty][0]
            assert np.all(out[k] == 0.0)
            if mode == _lib.MODE_LINEARIZE:
                rest = [i for i in range(3) if i != k]
                assert np.array_equal(out[rest], solo)
        rows, inl = b.lookup_rows(table)
        assert inl[[i for i, c in enumerate(order) if c is empty][0]] == 0


def test_small_host_graph_survives_pose_table_growth(small_graph):
    """The small-batch host path replays a graph with the batch's pose buffer baked in; a call
    with a larger pose table reallocates that buffer and must retire the graph."""
    poses, est, scans, covs, maps, srcs, pairs = small_graph
    clouds = [_lib.DeviceCloud(s, c) for s, c in srcs[:2]]
    dmaps = [_lib.DeviceMap.build(_lib.DeviceCloud(s, c), 1.0) for s, c in zip(scans[:2], covs[:2])]
    b = _lib.DeviceBatch(clouds, [dmaps[1], dmaps[0]], [False] * 2, [10] * 2, [0, 1], [1, 0])
    small = np.array([G.pose_row(p) for p in est[:2]])
    first = b.linearize_poses(small)            # captures the host graph at V = 2
    big = np.vstack([small, np.array([G.pose_row(p) for p in est[2:12]])])
    rows_big, _ = b.lookup_rows(big)             # V = 12: reallocates the pose buffer
    junk = torch_junk_allocations()
    again = b.linearize_poses(small)             # must not replay against the freed buffer
    assert np.array_equal(first, again)
    del junk


def torch_junk_allocations():
    """Device allocations that would land in a freed pool block (makes a stale-pointer replay
    read garbage instead of stale-but-equal data)."""
    import torch

    return [torch.full((4096,), float("nan"), dtype=torch.float64, device="cuda")
            for _ in range(8)]


def test_d2d_error_matches_reference_formula_anywhere():
    """d2d_error (registration.py:101-110) returns (error, d, W) for any input — points on a
    voxel face, far-away points (|x| >= 2^20 m would wrap a 1 m key) — matching the reference's
    np.linalg.inv formula within the parity bar."""
    rng = np.random.default_rng(5)
    cases = [np.array([0.0, 0.0, 0.0]), np.array([1.0, -2.0, 3.0]), np.array([0.5, 0.25, -7.0]),
             np.array([2.0 ** 21 + 0.5, 3.0, -1.0]), rng.normal(size=3) * 100]
    for mean in cases:
        cov_p = np.diag(rng.uniform(0.01, 0.1, 3))
        cov_v = np.diag(rng.uniform(0.01, 0.1, 3))
        for tij in (G.Se3Pose.identity(), G.Se3Pose(G.so3_exp([0.1, -0.2, 0.3]), [0.25, 0.5, 0.0])):
            p = G.Gaussian3(mean, cov_p)
            v = G.Gaussian3(tij.rotation.matrix() @ mean + tij.translation + [0.01, -0.02, 0.03],
                            cov_v)
            err, d, w = RG.d2d_error(p, v, tij)
            R = tij.rotation.matrix()
            d_ref = v.mean - (R @ mean + tij.translation)
            w_ref = np.linalg.inv(cov_v + R @ cov_p @ R.T)
            assert_tol(d, d_ref, "d")
            assert_tol(w, w_ref, "W")
            assert_tol(err, d_ref @ w_ref @ d_ref, "error")


# ---- round 2: the headline workload's correspondences, every factor -------------------------

def _oracle_rows_by_target(wl, R, t):
    """Vectorised oracle lookup (registration.py:47-55,149: searchsorted over the sorted packed
    keys of np.unique) for every factor of the workload, grouped by target submap; returns
    the concatenated rows in factor order and the count of points whose transformed
    coordinate lies within 1e-12 (relative, in cells) of a voxel face."""
    F = len(wl.pairs)
    n = np.array([len(wl.source_index[i]) for i in wl.pairs[:, 0]])
    off = np.concatenate([[0], np.cumsum(n)])
    rows = np.empty(off[-1], np.int64)
    near = 0
    res = wl.resolution
    by_target = np.argsort(wl.pairs[:, 1], kind="stable")
    bounds = np.flatnonzero(np.r_[True, np.diff(wl.pairs[by_target, 1]) != 0, True])
    for a, b in zip(bounds[:-1], bounds[1:]):
        fids = by_target[a:b]
        j = wl.pairs[fids[0], 1]
        keys = np.unique(O.pack_voxel_keys(wl.scans[j], res))
        pts = [wl.scans[i][wl.source_index[i]] for i in wl.pairs[fids, 0]]
        owner = np.repeat(np.arange(len(fids)), [len(p) for p in pts])
        P = np.concatenate(pts)
        moved = np.einsum("nij,nj->ni", R[fids][owner], P) + t[fids][owner]
        q = moved / res
        frac = q - np.floor(q)
        near += int(np.sum((frac < 1e-12 * np.maximum(1.0, np.abs(q))) |
                           (1.0 - frac < 1e-12 * np.maximum(1.0, np.abs(q)))))
        qk = O.pack_voxel_keys(moved, res)
        pos = np.minimum(np.searchsorted(keys, qk), len(keys) - 1)
        r = np.where(keys[pos] == qk, pos, -1)
        start = 0
        for f, p in zip(fids, pts):
            rows[off[f]:off[f + 1]] = r[start:start + len(p)]
            start += len(p)
        assert start == len(P)
    return rows, off, near


def test_config5_every_factor_rows_and_inliers_bit_exact(config5):
    """north_star: correspondence indices and inlier counts bit-exact at the size the headline
    is quoted on — all 50,000 factors, 19.9M correspondences, straight from the K4a hit lists
    K4b consumes (vg_batch_lookup_rows) — plus the linearization records' inlier counts."""
    wl = config5
    batch = wl.batch()
    table = wl.pose_table
    rows, inl = batch.lookup_rows(table)
    R, t = O.relative_transforms(table, wl.pairs[:, 0], wl.pairs[:, 1])
    ref_rows, off, near = _oracle_rows_by_target(wl, R, t)
    print(f"config 5: {len(ref_rows)} correspondences, {int((ref_rows >= 0).sum())} hits, "
          f"{near} near a voxel face")
    assert near == 0
    assert len(rows) == len(ref_rows) == wl.num_points
    assert np.array_equal(rows, ref_rows)
    ref_inl = np.add.reduceat((ref_rows >= 0).astype(np.int64), off[:-1])
    assert np.array_equal(inl, ref_inl)
    rec = batch.linearize_poses(table)
    assert np.array_equal(rec[:, 91].astype(np.int64), ref_inl)
    cost = batch.linearize_poses(table, _lib.MODE_COST)
    assert np.array_equal(cost[:, 1].astype(np.int64), ref_inl)
    # cost mode (K4c: lookup + cost fused, no hit compaction) against the linearization's
    # cost (K4a + K4b): the same per-hit terms, summed in another order
    live = ref_inl >= 10
    assert np.allclose(cost[live, 0], rec[live, 90], rtol=1e-12, atol=0.0)


def test_config5_blocks_of_600_factors_vs_oracle(config5):
    """H/b/cost of every factor of 12 seeded target submaps (~600 factors of the headline
    workload) within 1e-4 rel / 1e-6 abs of the fp64 oracle; gated factors gate in both."""
    wl = config5
    batch = wl.batch()
    table = wl.pose_table
    host = batch.linearize_poses(table)
    rng = np.random.default_rng(56)
    targets = rng.choice(wl.n_submaps, 12, replace=False)
    fids = np.flatnonzero(np.isin(wl.pairs[:, 1], targets))
    R, t = O.relative_transforms(table, wl.pairs[fids, 0], wl.pairs[fids, 1])
    maps = {int(j): O.build_voxelmap(wl.scans[j], wl.scan_covs[j], wl.resolution) for j in targets}
    r32 = batch.linearize_poses_f32(table)
    c32, i32 = _lib.record_cost_inliers_f32(r32)
    gated = 0
    for k, f in enumerate(fids):
        i, j = wl.pairs[f]
        sel = wl.source_index[i]
        try:
            ref = O.linearize(wl.scans[i][sel], wl.scan_covs[i][sel], maps[int(j)], R[k], t[k])
        except ValueError:
            assert host[f][91] < 10 and np.all(host[f][:90] == 0)
            gated += 1
            continue
        assert_lin(RG.unpack_record(host[f], False), ref, False)
        # the compact fp32 record (what the factor shim and the e2e bench consume)
        rec = np.concatenate([r32[f, :90].astype(np.float64), [c32[f], i32[f]]])
        assert_lin(RG.unpack_record(rec, False), ref, False)
    assert len(fids) >= 500 and gated < len(fids) // 4


def test_f32_records_are_the_rounded_fp64_records(small_graph, config5):
    """vg_batch_linearize_poses_f32 = K5's fp64 records rounded per element (blocks), with the
    fp64 cost and the inlier count carried exactly — on the small graph (graph-replayed host
    path) and on config 5 (the 8-stage pipelined host path), and with explicit transforms."""
    poses, est, scans, covs, maps, srcs, pairs = small_graph
    clouds = [_lib.DeviceCloud(s, c) for s, c in srcs]
    dmaps = [_lib.DeviceMap.build(_lib.DeviceCloud(s, c), 1.0) for s, c in zip(scans, covs)]
    F = len(pairs)
    small = _lib.DeviceBatch([clouds[i] for i, _ in pairs], [dmaps[j] for _, j in pairs],
                             [(f % 5) == 2 for f in range(F)], [10] * F, pairs[:, 0], pairs[:, 1])
    table = np.array([G.pose_row(p) for p in est])
    R, t = O.relative_transforms(table, pairs[:, 0], pairs[:, 1])
    T = np.concatenate([R.reshape(F, 9), t], axis=1)
    cases = [(small.linearize_poses(table), small.linearize_poses_f32(table)),
             (small.linearize(T), small.linearize_f32(T))]
    wl = config5
    big = wl.batch()
    cases.append((big.linearize_poses(wl.pose_table), big.linearize_poses_f32(wl.pose_table)))
    for r64, r32 in cases:
        assert r32.dtype == np.float32 and r32.shape == (len(r64), _lib.REC_LINEARIZE_F32)
        assert np.array_equal(r32[:, :90], r64[:, :90].astype(np.float32))
        cost, inl = _lib.record_cost_inliers_f32(r32)
        assert np.array_equal(cost, r64[:, 90]) and np.array_equal(inl, r64[:, 91].astype(np.int64))
        assert np.all(r32[:, 93] == 0)


def test_linearize_from_terms_accepts_foreign_match_terms(golden):
    """linearize_from_terms with a MatchTerms that carries no voxel map (the reference's own
    match_terms makes those: registration.py:133-157) linearizes the explicit per-point
    weights on the GPU (vg_linearize_terms) — the same blocks as the map-carrying path and the
    oracle, within the parity bar; binary and unary."""
    from dataclasses import dataclass

    @dataclass
    class ForeignTerms:  # the reference MatchTerms' fields, nothing else
        hit: np.ndarray
        moved: np.ndarray
        d: np.ndarray
        weight: np.ndarray
        wd: np.ndarray
        cost: float
        inliers: int

    g = golden("registration")
    src = make_frame(g["src_points"], g["src_covs"])
    _, k, mu, c, n = golden_map(g)
    vm = RG.GaussianVoxelMap(0.5, k, mu, c, n)
    for case in range(6):
        R, t = g[f"case{case}_R"], g[f"case{case}_t"]
        unary = bool(g[f"case{case}_unary"])
        terms = RG.match_terms(src, vm, _TPose(R, t))
        if terms.inliers < 10:
            continue
        foreign = ForeignTerms(terms.hit, terms.moved, terms.d, terms.weight, terms.wd,
                               terms.cost, terms.inliers)
        ref = {k: (g[f"case{case}_{k}"] if f"case{case}_{k}" in g.files else None)
               for k in NAMES + ("cost", "inliers")}
        ref["inliers"] = int(ref["inliers"])
        lin = RG.linearize_from_terms(src, foreign, _TPose(R, t), target_fixed=unary)
        assert_lin(lin, ref, unary)
        mine = RG.linearize_from_terms(src, terms, _TPose(R, t), target_fixed=unary)
        for name in NAMES:
            if getattr(mine, name) is not None:
                assert_tol(getattr(lin, name), getattr(mine, name), name)
    with pytest.raises(DegenerateConstraint):
        RG.linearize_from_terms(src, ForeignTerms(terms.hit, terms.moved, terms.d, terms.weight,
                                                  terms.wd, terms.cost, 3), _TPose(R, t))

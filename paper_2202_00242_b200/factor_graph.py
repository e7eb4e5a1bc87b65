"""Drop-in MatchingCostFactor with a batching shim, plus the host-side LM that calls it.

``MatchingCostFactor`` keeps the reference's per-factor interface (factor_graph.py:102-126,
209-308): ``keys``, ``unary``, ``grounding``, ``kind``, ``cost(values)``,
``linearize(values) -> FactorLinearization``.  The reference ``FactorGraph`` calls it one
factor at a time (total_cost :472-474, _assemble_dense :522-536).  Behind that unchanged
interface, the first factor that misses its cache for a given set of values triggers ONE
batched GPU evaluation of every live matching factor whose variables are in ``values``;
each factor then serves its own record from an identity-keyed cache, exactly as the
reference's ``_terms_cache`` does for one factor (:253-269).  Values are immutable, so
identity of (v_i, v_j) is a safe key.

``integrate.patch(limapper)`` swaps in this MatchingCostFactor and replaces the FactorGraph
methods whose host work dominates at global-mapping scale — ``total_cost`` (:472-474: one
batched cost launch for all of the graph's matching factors), ``_assemble_dense`` (:522-536:
the normal equations summed on the device, K6, and scattered into the reference's dense H/g),
and, above the reference's dense threshold, ``optimize_lm`` / ``marginal_covariance``
(:546-612, :703-722: H kept on the device, each damped solve a device factorization; the
reference's control flow, and its own method below the threshold).
"""

from __future__ import annotations

import itertools
import sys
import weakref
from collections import OrderedDict
from dataclasses import dataclass

import numpy as np
import scipy.sparse
import scipy.sparse.csgraph

from . import _lib
from .geometry import pose_row
from .preprocess import device_cloud
from .registration import _as_device_map, unpack_sym6

VARIABLE_DIMS = {"frame-state": 15, "submap-pose": 6, "endpoint-state": 15}


@dataclass(frozen=True, order=True)
class Key:
    kind: str
    index: int

    @property
    def dim(self) -> int:
        return VARIABLE_DIMS[self.kind]

    def __repr__(self) -> str:
        return f"{self.kind}:{self.index}"


def frame_key(index: int) -> Key:
    return Key("frame-state", index)


def submap_key(index: int) -> Key:
    return Key("submap-pose", index)


class FactorLinearization:
    """Gradient/Hessian blocks of one factor (factor_graph.py:102-111)."""

    __slots__ = ("keys", "g", "h", "cost")

    def __init__(self, keys, g, h, cost):
        self.keys = keys
        self.g = g
        self.h = h
        self.cost = cost


class Factor:
    keys: tuple
    grounding = False

    def cost(self, values) -> float:
        raise NotImplementedError

    def linearize(self, values) -> FactorLinearization:
        raise NotImplementedError


# ---- the batching shim ---------------------------------------------------------------------


class _PoseTable:
    """The (V + fixed, 8) pose table of a batch's variables at given values (the C-ABI layout,
    geometry.pose_row).  When `values` holds the same key objects in the same order as the
    last call — the LM's candidate dicts are built from the graph's own keys
    (factor_graph.py:539-544) — the per-key dict lookups are skipped."""

    def __init__(self, var_keys, fixed):
        self.var_keys = var_keys
        self.fixed = fixed
        self.submap = [k.kind == "submap-pose" for k in var_keys]
        self._order = None  # (the key objects of values, index of each variable among them)

    def build(self, values) -> np.ndarray:
        keys = self.var_keys
        order = self._order
        if (order is not None and len(values) == len(order[0])
                and all(a is b for a, b in zip(values, order[0]))):
            listed = list(values.values())
            vals = [listed[i] for i in order[1]]
        else:
            vals = [values[k] for k in keys]
            # positions by key equality (factors often hold equal but distinct Key objects),
            # remembered for dicts holding these same key objects in this order
            pos = {k: i for i, k in enumerate(values)}
            self._order = (tuple(values), [pos[k] for k in keys])
        poses = [v if sub else v.pose for v, sub in zip(vals, self.submap)]
        n = len(keys)
        table = np.empty((n + self.fixed.shape[0], 8))
        if n:
            table[:n, :4] = [p.rotation.quat for p in poses]
            table[:n, 4:7] = [p.translation for p in poses]
            table[:n, 7] = 0.0
        table[n:] = self.fixed
        return table


class _Batcher:
    """Registry of live GPU matching factors and the cache of flattened device batches."""

    def __init__(self):
        self._live: "weakref.WeakValueDictionary[int, MatchingCostFactor]" = \
            weakref.WeakValueDictionary()
        self._serial = itertools.count()
        self._batches: "OrderedDict[tuple, tuple]" = OrderedDict()
        self.evaluations = 0

    def register(self, f: "MatchingCostFactor") -> None:
        f._serial = next(self._serial)
        self._live[f._serial] = f

    def _remember(self, sig, entry):
        self._batches[sig] = entry
        while len(self._batches) > 8:
            self._batches.popitem(last=False)

    def _batch_for(self, group, sig=None):
        """(device batch, pose table builder, gate thresholds) of exactly `group`."""
        sig = tuple(f._serial for f in group) if sig is None else sig
        hit = self._batches.get(sig)
        if hit is not None:
            self._batches.move_to_end(sig)
            return hit
        var_index: dict = {}
        for f in group:
            for k in f.keys:
                var_index.setdefault(k, len(var_index))
        var_keys = list(var_index)
        fixed_rows = []
        vs, vt = [], []
        for f in group:
            vs.append(var_index[f.keys[0]])
            if f.unary:
                vt.append(len(var_keys) + len(fixed_rows))
                fixed_rows.append(pose_row(f.fixed_target_pose))
            else:
                vt.append(var_index[f.keys[1]])
        mins = [f.min_inliers for f in group]
        batch = _lib.DeviceBatch([device_cloud(f.source) for f in group],
                                 [_as_device_map(f.target_map) for f in group],
                                 [f.unary for f in group], mins, vs, vt)
        table = _PoseTable(var_keys, np.array(fixed_rows).reshape(-1, 8))
        entry = (batch, table, np.asarray(mins, dtype=np.float64), [weakref.ref(f) for f in group])
        self._remember(sig, entry)
        return entry

    def evaluate(self, values, mode: int, requester: "MatchingCostFactor") -> None:
        # factors added to a FactorGraph (graph_add_factor) batch with their own graph only:
        # another graph reusing the same keys neither joins the batch nor can fail it
        owner = requester._graph
        group = []
        for serial in sorted(self._live.keys()):
            f = self._live.get(serial)
            if f is None or f._empty or f._graph is not owner:
                continue
            if any(k not in values for k in f.keys):
                continue
            if f._cached(values, mode) is not None:
                continue
            group.append(f)
        if requester not in group:
            group.append(requester)
        # factors sharing a target map adjacent: the batch's item order is then target-major
        # (map reuse in L2) and its pipelined host copy moves contiguous record ranges
        group.sort(key=lambda f: id(f.target_map))
        batch, table, _, _ = self._batch_for(group)
        # fp64 records into pinned memory (the staged copies overlap the compute); the compact
        # fp32 record (linearize_poses_f32) halves the PCIe bytes for callers that take fp32
        # blocks, but here the per-factor Python unpacking dominates either way
        out = batch.linearize_poses(table.build(values), mode)
        self.evaluations += 1
        for f, rec in zip(group, out):
            f._store(values, mode, rec)

    def gated_costs(self, group, values, sig=None) -> np.ndarray:
        """Per-factor gated cost of `group` at `values` (MatchingCostFactor.cost, factor order)
        from ONE cost-mode launch over exactly these factors."""
        batch, table, mins, _ = self._batch_for(group, sig)
        rec = batch.linearize_poses(table.build(values), _lib.MODE_COST)
        self.evaluations += 1
        return np.where(rec[:, 1] >= mins, rec[:, 0], 0.0)

    def assemble(self, group, values, var_keys) -> "_lib.NormalEquations":
        """Device-assembled normal equations of `group` over the graph variables `var_keys`
        (FactorGraph._assemble_dense, factor_graph.py:522-536)."""
        batch, poses = self.assembly_batch(group, values, var_keys)
        return batch.assemble_poses(poses)

    def assembly_batch(self, group, values, var_keys, sig=None):
        """(device batch set up to assemble `group` over `var_keys`, its pose table at
        `values`) — one evaluation of the normal equations follows."""
        sig = ("asm", tuple(f._serial for f in group) if sig is None else sig, tuple(var_keys))
        hit = self._batches.get(sig)
        if hit is None:
            index = {k: i for i, k in enumerate(var_keys)}
            fixed_rows, vs, vt = [], [], []
            for f in group:
                vs.append(index[f.keys[0]])
                if f.unary:
                    vt.append(len(var_keys) + len(fixed_rows))
                    fixed_rows.append(pose_row(f.fixed_target_pose))
                else:
                    vt.append(index[f.keys[1]])
            batch = _lib.DeviceBatch([device_cloud(f.source) for f in group],
                                     [_as_device_map(f.target_map) for f in group],
                                     [f.unary for f in group], [f.min_inliers for f in group],
                                     vs, vt)
            batch.assemble_setup(len(var_keys))
            hit = (batch, _PoseTable(list(var_keys), np.array(fixed_rows).reshape(-1, 8)),
                   [weakref.ref(f) for f in group])
            self._remember(sig, hit)
        self._batches.move_to_end(sig)
        batch, table, _ = hit
        self.evaluations += 1
        return batch, table.build(values)


_BATCHER = _Batcher()


class MatchingCostFactor(Factor):
    """Voxelized registration constraint between a source frame and a target voxel map;
    unary when the target pose is fixed (factor_graph.py:209-308).  GPU-evaluated."""

    def __init__(self, key_source: Key, source, target_map, key_target: Key | None = None,
                 fixed_target_pose=None, min_inliers: int = 10):
        if (key_target is None) == (fixed_target_pose is None):
            raise ValueError("exactly one of key_target / fixed_target_pose")
        self.keys = (key_source,) if key_target is None else (key_source, key_target)
        self.source = source
        self.target_map = target_map
        self.fixed_target_pose = fixed_target_pose
        self.min_inliers = min_inliers
        self._empty = (len(source) == 0 or len(target_map) == 0
                       or getattr(source, "covs", None) is None)
        self._cache = None  # (v_i, v_j, mode, record)
        self._graph_ref = None  # the FactorGraph it was added to (graph_add_factor), weak
        _BATCHER.register(self)

    @property
    def _graph(self):
        return self._graph_ref() if self._graph_ref is not None else None

    @property
    def unary(self) -> bool:
        return self.fixed_target_pose is not None

    @property
    def grounding(self) -> bool:
        return self.unary

    @property
    def kind(self) -> str:
        return "matching-cost-unary" if self.unary else "matching-cost-binary"

    def _vals(self, values):
        return values[self.keys[0]], (None if self.unary else values[self.keys[1]])

    def _cached(self, values, mode):
        c = self._cache
        if c is None:
            return None
        v_i, v_j = self._vals(values)
        if c[0] is v_i and c[1] is v_j and (c[2] == _lib.MODE_LINEARIZE or mode == c[2]):
            return c
        return None

    def _store(self, values, mode, rec) -> None:
        v_i, v_j = self._vals(values)
        self._cache = (v_i, v_j, mode, rec)

    def _record(self, values, mode):
        c = self._cached(values, mode)
        if c is None:
            _BATCHER.evaluate(values, mode, self)
            c = self._cache
        return c[2], c[3]

    def cost(self, values) -> float:
        if self._empty:
            return 0.0
        mode, rec = self._record(values, _lib.MODE_COST)
        cost, inl = (rec[0], rec[1]) if mode == _lib.MODE_COST else (rec[90], rec[91])
        return 0.0 if inl < self.min_inliers else float(cost)

    def linearize(self, values) -> FactorLinearization:
        zeros = [np.zeros(k.dim) for k in self.keys]
        if not self._empty:
            _, rec = self._record(values, _lib.MODE_LINEARIZE)
            cost, inl = float(rec[90]), rec[91]
        if self._empty or inl < self.min_inliers:  # DegenerateConstraint -> no-op
            h = {(a, a): np.zeros((k.dim, k.dim)) for a, k in enumerate(self.keys)}
            return FactorLinearization(self.keys, zeros, h, 0.0)
        di = self.keys[0].dim
        g_i = np.zeros(di)
        g_i[:6] = rec[78:84]
        h_ii = np.zeros((di, di))
        h_ii[:6, :6] = unpack_sym6(rec[0:21])
        if self.unary:
            return FactorLinearization(self.keys, [g_i], {(0, 0): h_ii}, cost)
        dj = self.keys[1].dim
        g_j = np.zeros(dj)
        g_j[:6] = rec[84:90]
        h_jj = np.zeros((dj, dj))
        h_jj[:6, :6] = unpack_sym6(rec[57:78])
        h_ij = np.zeros((di, dj))
        h_ij[:6, :6] = rec[21:57].reshape(6, 6)
        return FactorLinearization(self.keys, [g_i, g_j],
                                   {(0, 0): h_ii, (0, 1): h_ij, (1, 1): h_jj}, cost)


# ---- FactorGraph methods replaced by integrate.patch (factor_graph.py:472-474, 522-536) ------

class _Split:
    """A graph's GPU matching factors and the rest, their positions in graph.factors, and the
    GPU group's batch signature (built once, not per evaluation)."""

    __slots__ = ("key", "gpu", "rest", "gpos", "rpos", "serials")

    def __init__(self, key, facs):
        self.key = key
        self.gpu, self.rest, gpos, self.rpos = [], [], [], []
        for i, f in enumerate(facs):
            if isinstance(f, MatchingCostFactor) and not f._empty:
                self.gpu.append(f)
                gpos.append(i)
            else:
                self.rest.append(f)
                self.rpos.append(i)
        self.gpos = np.array(gpos, dtype=np.int64)
        self.serials = tuple(f._serial for f in self.gpu)


def _split(graph) -> _Split:
    """The graph's _Split, cached while its factor list is unchanged (the reference only
    appends to it or replaces it: factor_graph.py:465, 701)."""
    facs = graph.factors
    key = (id(facs), len(facs), id(facs[-1]) if facs else 0)
    sp = graph.__dict__.get("_vgicp_split")
    if sp is None or sp.key != key:
        sp = _Split(key, facs)
        graph.__dict__["_vgicp_split"] = sp
    return sp


def _split_factors(graph):
    """(GPU matching factors, the rest) of a graph."""
    sp = _split(graph)
    return sp.gpu, sp.rest


#: (patched reference class, method name) -> the reference's own function (integrate.patch)
_ORIGINALS: dict = {}


def _original(graph, name):
    for cls in type(graph).__mro__:
        fn = _ORIGINALS.get((cls, name))
        if fn is not None:
            return fn
    raise TypeError(f"{type(graph).__name__}.{name} was not patched by integrate.patch")


def graph_add_factor(self, factor) -> None:
    """FactorGraph.add_factor (factor_graph.py:460-467) that also tags a MatchingCostFactor with
    its graph, so the per-factor batching shim groups a graph's own factors only."""
    _original(self, "add_factor")(self, factor)
    if isinstance(factor, MatchingCostFactor):
        factor._graph_ref = weakref.ref(self)


def graph_total_cost(self, values=None) -> float:
    """FactorGraph.total_cost (factor_graph.py:472-474): the graph's matching factors in one
    batched cost launch, the others per factor, and the per-factor costs summed as the
    reference sums them — Python's sum() over the factor-ordered list (same terms, same
    order, same summation, so the same float)."""
    values = self.values if values is None else values
    sp = _split(self)
    if not sp.gpu:
        return float(sum(f.cost(values) for f in self.factors))
    costs = np.empty(len(self.factors))
    costs[sp.gpos] = _BATCHER.gated_costs(sp.gpu, values, sp.serials)
    for i, f in zip(sp.rpos, sp.rest):
        costs[i] = f.cost(values)
    return float(sum(costs.tolist()))


def graph_assemble_dense(self, values, slices, dim):
    """FactorGraph._assemble_dense (factor_graph.py:522-536): the matching factors' blocks
    summed into the block-sparse normal equations on the device (K6, factor order per block)
    and scattered into the dense H/g the reference's solver takes (6-dof blocks top-left of
    15-dof frame-state slices, :292-308); the other factors per factor as the reference does."""
    h = np.zeros((dim, dim))
    g = np.zeros(dim)
    cost = 0.0
    gpu, rest = _split_factors(self)
    if gpu:
        keys = list(self.values)
        ne = _BATCHER.assemble(gpu, values, keys)
        hd, gd = ne.dense([slices[k].start for k in keys], dim)
        h += hd
        g += gd
        cost += ne.cost
    for f in rest:
        lin = f.linearize(values)
        cost += lin.cost
        sls = [slices[k] for k in lin.keys]
        for a, ga in enumerate(lin.g):
            g[sls[a]] += ga
        for (a, b), blk in lin.h.items():
            h[sls[a], sls[b]] += blk
            if a != b:
                h[sls[b], sls[a]] += blk.T
    return h, g, cost


# ---- the LM's linear solve on the device ----------------------------------
#
# For graphs above the reference's dense_threshold its LM factors a CSC copy of the dense
# damped H with splu on every damping attempt (factor_graph.py:565-576); at global-mapping
# size that is a 6,000 x 6,000 system assembled and factored on the host.  Here H and g never
# leave the device: the matching factors' normal equations go from K6 straight into the dense
# device H (vg_solver_add_batch), the other factors' host blocks are added by one upload, and
# each damping attempt is a device Cholesky (LU when not positive definite: splu's semantics)
# returning only the dim-sized step.  The LM control flow is the reference's (:546-612); the
# small dense branch (dim <= dense_threshold) stays the reference's own code.


#: the dense device system (H and its damped copy, 16 * dim^2 bytes: 14.4 GB at 30,000) is used
#: up to this tangent dimension; larger graphs keep the reference's sparse host solve
DEVICE_SOLVE_MAX_DIM = 30000


def _ref_module(graph):
    """The module defining the reference FactorGraph (LmSettings, OptimizeResult, errors)."""
    for cls in type(graph).__mro__:
        mod = sys.modules.get(cls.__module__)
        if mod is not None and hasattr(mod, "LmSettings") and hasattr(mod, "OptimizeResult"):
            return mod
    raise TypeError(f"{type(graph).__name__} is not a reference FactorGraph")


class DeviceNormalEquations:
    """A graph's H, g on the device at given values (the device side of _assemble_dense,
    factor_graph.py:522-536) and the damped solves of its LM."""

    def __init__(self, graph, slices, dim):
        self.graph, self.slices, self.dim = graph, slices, dim
        self.solver = _lib.DeviceSolver(dim)

    @classmethod
    def of(cls, graph, slices, dim) -> "DeviceNormalEquations":
        """The graph's solver (kept on the graph while its dimension is unchanged)."""
        ne = graph.__dict__.get("_vgicp_normal")
        if ne is None or ne.dim != dim:
            graph.__dict__.pop("_vgicp_normal", None)
            ne = cls(graph, slices, dim)
            graph.__dict__["_vgicp_normal"] = ne
        ne.slices = slices
        return ne

    def assemble(self, values) -> float:
        """H, g := the normal equations at `values`; returns the total cost (:522-536)."""
        s = self.solver
        s.reset()
        sp = _split(self.graph)
        gpu, rest = sp.gpu, sp.rest
        cost = 0.0
        if gpu:
            keys = list(self.graph.values)
            batch, poses = _BATCHER.assembly_batch(gpu, values, keys, sp.serials)
            cost += s.add_batch(batch, poses, [self.slices[k].start for k in keys])
        if rest:
            blocks: dict = {}
            g = np.zeros(self.dim)
            for f in rest:
                lin = f.linearize(values)
                cost += lin.cost
                sls = [self.slices[k] for k in lin.keys]
                for a, ga in enumerate(lin.g):
                    g[sls[a]] += ga
                for (a, b), blk in lin.h.items():
                    _add_block(blocks, sls[a].start, sls[b].start, blk)
                    if a != b:
                        _add_block(blocks, sls[b].start, sls[a].start, blk.T)
            s.add_blocks([(r, c, blk) for (r, c), blk in blocks.items()], g)
        return float(cost)

    def damped_step(self, lam: float):
        """delta solving (H + lam diag(H)) delta = -g, or None where the reference's solve
        raises (singular system, non-finite update: :574-578)."""
        if self.solver.factor(lam, 0.0, _lib.SOLVE_CHOLESKY_LU):
            return None
        delta = self.solver.solve()
        return delta if np.all(np.isfinite(delta)) else None


def _add_block(blocks, r, c, blk):
    cur = blocks.get((r, c))
    blocks[(r, c)] = np.array(blk, dtype=np.float64) if cur is None else cur + blk


def graph_check_structure(self) -> None:
    """FactorGraph.check_structure (factor_graph.py:478-510) over integer variable indices:
    the same loose-variable and anchoring checks, exceptions and messages, with the
    components from one connected-components pass instead of a Python union-find over
    hashed keys (≈0.1-0.4 s per LM call at 50,000 factors), and skipped while the graph's
    structure is the one last checked."""
    keys = list(self.values)
    facs = self.factors
    sig = (tuple(map(id, keys)), id(facs), len(facs), id(facs[-1]) if facs else 0)
    if self.__dict__.get("_vgicp_checked") == sig:
        return
    try:  # plain (kind, index) tuples hash in C; Key's dataclass __hash__ / __eq__ do not
        index = {(k.kind, k.index): i for i, k in enumerate(keys)}
        ids_of = [[index[(k.kind, k.index)] for k in f.keys] for f in facs]
    except (AttributeError, KeyError):  # foreign keys, or a factor on a removed variable:
        return _original(self, "check_structure")(self)  # the reference's own behaviour
    touched = np.zeros(len(keys), dtype=bool)
    touched[list(itertools.chain.from_iterable(ids_of))] = True
    edges = [(ids[j], ids[j + 1]) for ids in ids_of for j in range(len(ids) - 1)]
    roots = [ids[0] for f, ids in zip(facs, ids_of) if f.grounding]
    ref = _ref_module(self)
    loose = [k for k, t in zip(keys, touched) if not t]
    if loose:
        raise ref.UnderConstrainedGraph(f"variables without factors: {loose}")
    n = len(keys)
    e = np.array(edges, dtype=np.int64).reshape(-1, 2)
    adj = scipy.sparse.coo_matrix((np.ones(len(e)), (e[:, 0], e[:, 1])), shape=(n, n))
    _, label = scipy.sparse.csgraph.connected_components(adj, directed=False)
    grounded = np.zeros(n, dtype=bool)
    grounded[np.unique(label[roots]) if roots else []] = True
    bad = np.flatnonzero(~grounded[label])
    if len(bad):
        raise ref.UnderConstrainedGraph(
            f"component containing {keys[bad[0]]} has no anchoring factor")
    self.__dict__["_vgicp_checked"] = sig


def graph_optimize_lm(self, settings=None):
    """FactorGraph.optimize_lm (factor_graph.py:546-612) with the damped solve on the device
    above the dense threshold; the reference's own method at or below it."""
    ref = _ref_module(self)
    settings = settings or ref.LmSettings()
    slices, dim = self._slices()
    if dim <= settings.dense_threshold or dim > DEVICE_SOLVE_MAX_DIM:
        return _original(self, "optimize_lm")(self, settings)
    self.check_structure()
    values = dict(self.values)
    cost = self.total_cost(values)
    lam = settings.lambda_init
    ne = DeviceNormalEquations.of(self, slices, dim)
    iterations = 0

    def give_up(message):
        self.values = values
        self._cached_normal = None
        raise ref.NotConverged(message, estimates=values, cost=cost)

    for _ in range(settings.max_iterations):
        cost = ne.assemble(values)
        iterations += 1
        converged = False
        while True:  # damping attempts (:568-600)
            delta = ne.damped_step(lam)
            if delta is None:
                lam *= settings.lambda_up
                if lam > settings.lambda_max:
                    give_up("damping exhausted on singular system")
                continue
            if np.max(np.abs(delta)) < settings.update_tol:
                converged = True
                break
            candidate = self._retract_all(values, slices, delta)
            new_cost = self.total_cost(candidate)
            if np.isfinite(new_cost) and new_cost < cost:
                break
            lam *= settings.lambda_up
            if lam > settings.lambda_max:
                give_up("no cost-reducing step found")
        if converged:
            break
        values = candidate  # accepted (:590-594)
        lam = max(lam * settings.lambda_down, 1e-12)
        small = (cost - new_cost) <= settings.rel_cost_tol * max(cost, 1e-30)
        cost = new_cost
        if small:
            break
    self.values = values
    final = ne.assemble(values)
    # H is not copied back: marginal_covariance re-assembles it on the device (:705-709)
    self._cached_normal = None
    return ref.OptimizeResult(values, final, iterations)


def graph_marginal_covariance(self, key):
    """FactorGraph.marginal_covariance (factor_graph.py:703-722) with the factorization on the
    device above the dense threshold (same jitter retry); the reference's method below it."""
    ref = _ref_module(self)
    slices, dim = self._slices()
    if dim <= ref.LmSettings().dense_threshold or dim > DEVICE_SOLVE_MAX_DIM:
        return _original(self, "marginal_covariance")(self, key)
    ne = DeviceNormalEquations.of(self, slices, dim)
    ne.assemble(self.values)
    sl = slices[key]
    rhs = np.zeros((dim, key.dim))
    rhs[sl] = np.eye(key.dim)
    if ne.solver.factor(0.0, 0.0, _lib.SOLVE_CHOLESKY):
        jitter = 1e-9 * max(1.0, float(np.max(np.abs(ne.solver.diagonal()))))
        if ne.solver.factor(0.0, jitter, _lib.SOLVE_CHOLESKY):
            raise np.linalg.LinAlgError("marginal covariance: H + jitter I is not positive definite")
    return ne.solver.solve(rhs)[sl]

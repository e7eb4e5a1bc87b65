"""Swap the reference package's VGICP path for this one, in place.

    import limapper, paper_2202_00242_b200.integrate as vg
    undo = vg.patch(limapper)      # limapper.* now run on the B200 through libvgicp
    ...
    undo()

Every replaced name keeps the reference's signature, argument meaning and exceptions
(registration.py:29-269, preprocess.py:68-164, factor_graph.py:209-308); the keyframe overlap
matrix of OdometryEstimator (odometry.py:396-403) becomes one batched lookup launch, and
FactorGraph.total_cost / _assemble_dense (factor_graph.py:472-474, 522-536) batch the graph's
matching factors (one cost launch; device-assembled normal equations).  Modules that
imported a name with ``from .registration import ...`` (factor_graph.py:49-55,
odometry.py:21-46) get their module-level binding replaced too.  Above the reference's dense
threshold (600 tangent dims) optimize_lm and marginal_covariance keep H on the device and
factor it there (factor_graph.py:546-612, 703-722; the reference's control flow); IMU factors
and odometry logic are untouched and call the drop-in through the unchanged Factor protocol.  patch() is idempotent (a second call changes nothing).
"""

from __future__ import annotations

import importlib
import sys

from . import factor_graph as _fg
from . import preprocess as _pp
from . import registration as _rg

REPLACEMENTS = {
    "registration": {
        "GaussianVoxelMap": _rg.GaussianVoxelMap,
        "build_voxelmap": _rg.build_voxelmap,
        "d2d_error": _rg.d2d_error,
        "match_terms": _rg.match_terms,
        "matching_cost": _rg.matching_cost,
        "overlap_rate": _rg.overlap_rate,
        "linearize_from_terms": _rg.linearize_from_terms,
        "linearize_matching_cost": _rg.linearize_matching_cost,
        "MatchTerms": _rg.MatchTerms,
        "MatchingCostLinearization": _rg.MatchingCostLinearization,
    },
    "preprocess": {
        "pack_voxel_keys": _pp.pack_voxel_keys,
        "voxel_downsample": _pp.voxel_downsample,
        "knn_search": _pp.knn_search,
        "estimate_covariances": _pp.estimate_covariances,
    },
    "factor_graph": {
        "MatchingCostFactor": _fg.MatchingCostFactor,
        "GaussianVoxelMap": _rg.GaussianVoxelMap,
        "match_terms": _rg.match_terms,
        "linearize_from_terms": _rg.linearize_from_terms,
    },
    "odometry": {
        "MatchingCostFactor": _fg.MatchingCostFactor,
        "GaussianVoxelMap": _rg.GaussianVoxelMap,
        "build_voxelmap": _rg.build_voxelmap,
        "overlap_rate": _rg.overlap_rate,
        "voxel_downsample": _pp.voxel_downsample,
        "knn_search": _pp.knn_search,
        "estimate_covariances": _pp.estimate_covariances,
    },
}


def _overlap_matrix(self):
    """OdometryEstimator._overlap_matrix (odometry.py:396-403) as one batched launch."""
    kfs = self.keyframes
    return _rg.overlap_matrix([kf.frame for kf in kfs], [kf.voxelmap for kf in kfs],
                              [kf.pose() for kf in kfs])


# methods of reference classes whose per-factor / per-pair loops become batched GPU calls
METHOD_REPLACEMENTS = {
    "odometry": {"OdometryEstimator": {"_overlap_matrix": _overlap_matrix}},
    # FactorGraph.total_cost (factor_graph.py:472-474): one batched cost launch for the
    # graph's matching factors; _assemble_dense (:522-536): their normal equations summed on
    # the device (K6) and scattered into the dense H/g the reference's LM solves
    # optimize_lm / marginal_covariance (:546-612, :703-722): above the dense threshold the
    # damped solves run on the device against a device-resident H
    "factor_graph": {"FactorGraph": {"total_cost": _fg.graph_total_cost,
                                     "_assemble_dense": _fg.graph_assemble_dense,
                                     "add_factor": _fg.graph_add_factor,
                                     "check_structure": _fg.graph_check_structure,
                                     "optimize_lm": _fg.graph_optimize_lm,
                                     "marginal_covariance": _fg.graph_marginal_covariance}},
}

#: (class, method name) -> the reference's own function, for callers that compare against it
ORIGINALS: dict = {}


def _module(pkg, sub):
    if isinstance(pkg, str):
        name = f"{pkg}.{sub}"
    else:
        name = f"{pkg.__name__}.{sub}"
    if name in sys.modules:
        return sys.modules[name]
    try:
        return importlib.import_module(name)
    except ImportError:
        return None


def patch(pkg="limapper"):
    """Replace the reference's VGICP path inside package `pkg`; returns an undo callable."""
    saved = []
    for sub, names in REPLACEMENTS.items():
        mod = _module(pkg, sub) if not hasattr(pkg, sub) else getattr(pkg, sub)
        if mod is None:
            continue
        for name, obj in names.items():
            if hasattr(mod, name) and getattr(mod, name) is not obj:
                saved.append((mod, name, getattr(mod, name)))
                setattr(mod, name, obj)
    for sub, classes in METHOD_REPLACEMENTS.items():
        mod = _module(pkg, sub) if not hasattr(pkg, sub) else getattr(pkg, sub)
        for cname, methods in classes.items():
            cls = getattr(mod, cname, None) if mod is not None else None
            if cls is None:
                continue
            for name, fn in methods.items():
                if name in vars(cls) and vars(cls)[name] is not fn:
                    saved.append((cls, name, vars(cls)[name]))
                    ORIGINALS.setdefault((cls, name), vars(cls)[name])
                    _fg._ORIGINALS.setdefault((cls, name), vars(cls)[name])
                    setattr(cls, name, fn)

    # deskew keeps the reference's host IMU integration (taken from its preprocess module) and
    # moves the per-point work to the GPU (preprocess.py:181-232)
    prep = _module(pkg, "preprocess") if not hasattr(pkg, "preprocess") else pkg.preprocess
    if prep is not None and hasattr(prep, "deskew") and hasattr(prep, "integration_nodes"):
        dk = _pp.make_deskew(prep)
        for sub in ("preprocess", "odometry"):
            mod = _module(pkg, sub) if not hasattr(pkg, sub) else getattr(pkg, sub)
            if mod is not None and hasattr(mod, "deskew"):
                saved.append((mod, "deskew", getattr(mod, "deskew")))
                setattr(mod, "deskew", dk)

    def undo():
        for mod, name, obj in reversed(saved):
            setattr(mod, name, obj)

    return undo

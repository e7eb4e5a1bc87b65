#!/usr/bin/env python
"""The device damped solve alone (vg_solver_*) on a dense SPD system of --dim (default 6,000,
config 5's tangent dimension): wall-clock ms of factor (copy H -> A, damp, Cholesky) and solve
(A x = -g, 48 KB back), median of --reps, next to scipy's host cho_factor / cho_solve and
splu on the same matrix (the reference's dense and sparse branches, factor_graph.py:570-576)."""
import argparse
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2202_00242_b200 import _lib  # noqa: E402


def med(fn, reps):
    ts = []
    for _ in range(reps):
        a = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - a)
    return statistics.median(ts) * 1e3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dim", type=int, default=6000)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--no-host", action="store_true")
    a = ap.parse_args()
    rng = np.random.default_rng(0)
    n = a.dim
    J = rng.normal(size=(n + 64, n))
    H = J.T @ J
    g = rng.normal(size=n)
    s = _lib.DeviceSolver(n)
    t = 64
    s.add_blocks([(r, c, H[r:r + t, c:c + t]) for r in range(0, n, t) for c in range(0, n, t)], g)
    s.factor(1e-6)
    s.solve()
    out = {"dim": n,
           "device_factor_ms": med(lambda: s.factor(1e-6, 0.0, _lib.SOLVE_CHOLESKY_LU), a.reps),
           "device_solve_ms": med(lambda: s.solve(), a.reps)}
    if not a.no_host:
        import scipy.linalg
        import scipy.sparse
        import scipy.sparse.linalg

        A = H + np.diag(1e-6 * np.diag(H))
        out["host_cho_ms"] = med(lambda: scipy.linalg.cho_solve(
            scipy.linalg.cho_factor(A, lower=True), -g), 1)
        out["host_splu_ms"] = med(lambda: scipy.sparse.linalg.splu(
            scipy.sparse.csc_matrix(A)).solve(-g), 1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

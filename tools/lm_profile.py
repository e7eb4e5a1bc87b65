#!/usr/bin/env python
"""Where one config-5 LM iteration with the device solve spends its time (wall clock per
part, median of 5): device assembly (pose table + K-compose..K6 + scatter into the dense
device H), damped factorization, solve, the reference's retraction, the batched cost."""
import json
import statistics
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tools"))

import lm_workloads  # noqa: E402

from paper_2202_00242_b200 import _lib  # noqa: E402
from paper_2202_00242_b200 import factor_graph as vfg  # noqa: E402
from paper_2202_00242_b200 import workloads as W  # noqa: E402


def med(fn, n=5):
    ts = []
    for _ in range(n):
        a = time.perf_counter()
        out = fn()
        ts.append(time.perf_counter() - a)
    return statistics.median(ts) * 1e3, out


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    wl = W.global_mapping(n_submaps=n, neighbors=50)
    g, fg, _ = lm_workloads.global_mapping_lm(wl)
    slices, dim = g._slices()
    ne = vfg.DeviceNormalEquations.of(g, slices, dim)
    ne.assemble(g.values)
    out = {"submaps": n, "dim": dim}
    out["assemble_ms"], _ = med(lambda: ne.assemble(g.values))
    out["factor_ms"], _ = med(lambda: ne.solver.factor(1e-6, 0.0, _lib.SOLVE_CHOLESKY_LU))
    out["solve_ms"], delta = med(lambda: ne.solver.solve())
    out["retract_ms"], cand = med(lambda: g._retract_all(g.values, slices, delta))
    out["total_cost_ms"], _ = med(lambda: g.total_cost(cand))
    out["optimize_lm_1_iteration_ms"], _ = med(
        lambda: g.optimize_lm(fg.LmSettings(max_iterations=1)), 3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()

#!/bin/bash
# K4b time attribution: K4 with VGICP_K4B_DEBUG = 0 (full), 1 (no gathers),
# 2 (no math), 3 (neither), 4 (no lane-own point/covariance gathers); K4b = K4 - K4a.
# Profiling only: the results of the debug modes are wrong.
for d in 0 1 2 3 4; do
  VGICP_K4B_DEBUG=$d timeout 300 python tools/kernel_timing.py --reps 20 > gpurun_out/kt_dbg$d.json 2>&1
  echo "dbg=$d $(tail -1 gpurun_out/kt_dbg$d.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('K4a', round(d['k4_inliers_flush_ms'],4), 'K4', round(d['k4_linearize_flush_ms'],4), 'K4b', round(d['k4_linearize_flush_ms']-d['k4_inliers_flush_ms'],4))")"
done

for d in 0 3; do
  VGICP_K4B_DEBUG=$d timeout 300 python tools/kernel_timing.py --reps 20 > gpurun_out/kt_dbg$d.json 2>&1
  echo "dbg=$d $(python -c "import json; d=json.load(open('gpurun_out/kt_dbg$d.json')); print(round(d['k4_inliers_flush_ms'],4), round(d['k4_linearize_flush_ms'],4), round(d['k4_linearize_flush_ms']-d['k4_inliers_flush_ms'],4))")"
done

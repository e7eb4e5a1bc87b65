for v in 0 9; do
  VGICP_ACC_VARIANT=$v timeout 300 python tools/kernel_timing.py --reps 20 > gpurun_out/kt_v$v.json 2>&1
  echo "variant=$v $(python -c "import json; d=json.load(open('gpurun_out/kt_v$v.json')); print(round(d['k4_inliers_flush_ms'],4), round(d['k4_linearize_flush_ms'],4), round(d['k4_linearize_flush_ms']-d['k4_inliers_flush_ms'],4))")"
done

for cfg in "0 3" "1 3" "1 4"; do
  set -- $cfg
  VGICP_LOOKUP_FAST=$1 VGICP_LOOKUP_BLOCKS=$2 timeout 300 python tools/kernel_timing.py --reps 20 > gpurun_out/kt_$1_$2.json 2>&1
  echo "fast=$1 B=$2 $(python -c "import json; d=json.load(open('gpurun_out/kt_$1_$2.json')); print(round(d['k4_inliers_flush_ms'],4), round(d['k4_linearize_flush_ms'],4), round(d['k4_cost_flush_ms'],4))")"
done

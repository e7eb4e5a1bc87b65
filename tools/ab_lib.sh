#!/bin/bash
# A/B timing of library variants (VGICP_LIB) with tools/kernel_timing.py, interleaved.
# usage: tools/ab_lib.sh libA libB ... (names under paper_2202_00242_b200/lib, no .so)
L=paper_2202_00242_b200/lib
for i in 1 2; do
  for v in "$@"; do
    VGICP_LIB=$PWD/$L/$v.so timeout 300 python tools/kernel_timing.py --reps 20 > gpurun_out/ab_${v}_$i.json 2>&1
    echo "$v $i $(tail -1 gpurun_out/ab_${v}_$i.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(v, 4) for k, v in d.items() if k.endswith('ms')})")"
  done
done

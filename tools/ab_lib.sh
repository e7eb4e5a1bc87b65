set -x
L=paper_2202_00242_b200/lib
for i in 1 2; do
for v in libvgicp libvgicp_r8; do
  VGICP_LIB=$PWD/$L/$v.so timeout 300 python tools/kernel_timing.py --reps 20 > gpurun_out/ab_${v}_$i.json 2>&1
  echo "$v $i $(tail -1 gpurun_out/ab_${v}_$i.json)"
done
done
VGICP_LIB=$PWD/$L/libvgicp_r8.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -m gpu 2>&1 | tail -3

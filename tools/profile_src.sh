#!/bin/bash
# Source-level ncu capture of the given kernels on one workload (run under gpurun):
#   tools/profile_src.sh <tag> <workload> <kernel regex> [...]
# Leaves gpurun_out/<tag>_<kernel>.ncu-rep (+ .src.csv / .raw.csv exports made on the box).
tag=$1; wl=$2; shift 2
cmd="python bench.py --steps 2 --warmup 3 --no-cpu --no-also --workload $wl"
for k in "$@"; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -f -o gpurun_out/${tag}_$k $cmd > gpurun_out/${tag}_ncu_$k.log 2>&1
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page source --csv > gpurun_out/${tag}_$k.src.csv 2>/dev/null
  ncu -i gpurun_out/${tag}_$k.ncu-rep --page raw --csv > gpurun_out/${tag}_$k.raw.csv 2>/dev/null
done
ls -la gpurun_out/${tag}_*

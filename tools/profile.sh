#!/bin/bash
# Profile pass on the GPU box (run under gpurun):  tools/profile.sh <tag> [workload]
# Writes gpurun_out/<tag>_launches.csv (launch list of a whole bench.py run) and one
# `ncu --set full` capture per hot kernel; summarise here with profiles/summarize_ncu.py.
tag=${1:-rX}; wl=${2:-c2}
cmd="python bench.py --steps 2 --warmup 3 --no-cpu --workload $wl"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${tag}_launches.csv $cmd > gpurun_out/${tag}_ncu_b.log 2>&1
for k in k_blend2 k_preprocess k_place k_tile_sort_medium k_tile_sort_large k_scan_tiles k_tile_order; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -f -o gpurun_out/${tag}_$k $cmd > gpurun_out/${tag}_ncu_$k.log 2>&1
done
ls -la gpurun_out/${tag}_*

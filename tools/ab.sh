#!/bin/bash
# A/B of tuning variants on the GPU box (run under gpurun):  tools/ab.sh "<workloads>" <variant> [...]
# "main" = the in-tree library; other names = _lib/variants/<name> (python -m paper_2408_07967_b200.build --variant).
wls=$1; shift
for rep in 1 2; do
for v in "$@"; do
  lib=""; [ "$v" != main ] && lib=$PWD/paper_2408_07967_b200/_lib/variants/$v/libflashgs_b200.so
  for w in $wls; do
    FGS_LIB=$lib python bench.py --no-cpu --workload $w --steps 64 > gpurun_out/ab_${v}_${w}_$rep.json 2>> gpurun_out/ab.err
  done
done
done
python tools/benchsum.py gpurun_out/ab_*.json

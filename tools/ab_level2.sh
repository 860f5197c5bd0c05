for v in main redo4; do
  lib=""; [ "$v" != main ] && lib=$PWD/paper_2408_07967_b200/_lib/variants/$v/libflashgs_b200.so
  FGS_LIB=$lib python bench.py --no-cpu --no-also --workload c4-4k --steps 64 --lazy-level 2 > gpurun_out/ab_${v}_l2.json 2>> gpurun_out/ab.err
done
python tools/benchsum.py gpurun_out/ab_*_l2.json

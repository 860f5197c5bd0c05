bash tools/profile.sh r01_v9 c2 2>&1 | tail -2
tag=r01_v9_c44k; cmd="python bench.py --steps 2 --warmup 3 --no-cpu --workload c4-4k"
for k in k_preprocess k_place k_tile_sort_large k_blend2; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -f -o gpurun_out/${tag}_$k $cmd > gpurun_out/${tag}_ncu_$k.log 2>&1
done
ls gpurun_out/*.ncu-rep | wc -l

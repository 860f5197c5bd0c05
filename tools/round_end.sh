#!/bin/bash
# Everything a round's profiles/ needs, in one gpurun call:  tools/round_end.sh <tag>
# (GPU tests, every bench line, launch list + `ncu --set full` of the hot kernels on the
# north-star frame and on C2, the torchrun launches at world size 1)
tag=${1:-rX}
python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python bench.py > gpurun_out/${tag}_bench_c4-4k.json 2> gpurun_out/${tag}_bench.err
python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2>> gpurun_out/${tag}_bench.err
for w in c1 c2 c2-dense c3 c4 c5; do
  python bench.py --no-cpu --no-also --workload $w --steps 64 > gpurun_out/${tag}_bench_$w.json 2>> gpurun_out/${tag}_bench.err
done
python tools/benchsum.py gpurun_out/${tag}_bench_c*.json
cmd="python bench.py --steps 2 --warmup 3 --no-cpu --no-also --workload c4-4k"
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/${tag}_launches.csv $cmd > gpurun_out/${tag}_ncu_b.log 2>&1
for k in k_preprocess k_scan_tiles k_tile_order k_scatter_runs k_tile_sort_medium k_tile_front k_blend2; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -f -o gpurun_out/${tag}_c44k_$k $cmd > gpurun_out/${tag}_ncu_$k.log 2>&1
done
cmd="python bench.py --steps 2 --warmup 3 --no-cpu --no-also --workload c2"
for k in k_preprocess k_scatter_runs k_tile_sort_medium k_blend2; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -f -o gpurun_out/${tag}_c2_$k $cmd > gpurun_out/${tag}_ncu_c2_$k.log 2>&1
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu --no-also > gpurun_out/${tag}_torchrun_views.json 2> gpurun_out/torchrun.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu --no-also --mode bands --workload c4 > gpurun_out/${tag}_bench_bands_c4.json 2>> gpurun_out/torchrun.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/${tag}_torchrun_ref.json 2>> gpurun_out/torchrun.err
tail -3 gpurun_out/torchrun.err; cut -c1-300 gpurun_out/${tag}_torchrun_views.json gpurun_out/${tag}_bench_bands_c4.json gpurun_out/${tag}_torchrun_ref.json
ls gpurun_out/${tag}_*.ncu-rep | wc -l

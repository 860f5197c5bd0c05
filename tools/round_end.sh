python -m pytest tests -m gpu -x -q 2>&1 | tail -2
bash tools/bench_all.sh r01_v9 2>&1 | tail -12
bash tools/profile.sh r01_v9 c2 2>&1 | tail -3
tag=r01_v9_c44k; cmd="python bench.py --steps 2 --warmup 3 --no-cpu --workload c4-4k"
for k in k_preprocess k_place k_tile_sort_large k_blend2; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 8 -c 1 -f -o gpurun_out/${tag}_$k $cmd > gpurun_out/${tag}_ncu_$k.log 2>&1
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 50 --warmup 3 --no-cpu > gpurun_out/r01_v9_torchrun_views.json 2> gpurun_out/torchrun.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu --mode bands --workload c3 > gpurun_out/r01_v9_bench_bands_c3.json 2>> gpurun_out/torchrun.err
python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 1 --steps 3 --warmup 1 > gpurun_out/r01_v9_torchrun_ref.json 2>> gpurun_out/torchrun.err
tail -3 gpurun_out/torchrun.err; cut -c1-300 gpurun_out/r01_v9_torchrun_views.json gpurun_out/r01_v9_bench_bands_c3.json gpurun_out/r01_v9_torchrun_ref.json

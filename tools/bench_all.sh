#!/bin/bash
# All bench lines of a round (run under gpurun):  tools/bench_all.sh <tag>
tag=${1:-rX}
python bench.py > gpurun_out/${tag}_bench_c2.json 2> gpurun_out/${tag}_bench.err
python bench.py --impl reference > gpurun_out/${tag}_bench_ref.json 2>> gpurun_out/${tag}_bench.err
python bench.py --no-cpu --streams 1 > gpurun_out/${tag}_bench_c2_s1.json 2>> gpurun_out/${tag}_bench.err
for w in c1 c2-dense c3 c4-4k c4 c5; do
  python bench.py --no-cpu --workload $w --steps 64 > gpurun_out/${tag}_bench_$w.json 2>> gpurun_out/${tag}_bench.err
done
python tools/benchsum.py gpurun_out/${tag}_bench_*.json

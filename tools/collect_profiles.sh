#!/bin/bash
# gpurun_out/<tag>_* (tools/round_end.sh) -> the tracked summaries under profiles/:  tools/collect_profiles.sh <tag>
tag=$1
python profiles/summarize_ncu.py $tag gpurun_out/${tag}_launches.csv gpurun_out/${tag}_c44k_*.ncu-rep gpurun_out/${tag}_c2_*.ncu-rep > profiles/${tag}_ncu.md
python profiles/extract_traffic.py $tag c4-4k gpurun_out/${tag}_c44k_*.ncu-rep > profiles/${tag}_c4-4k_traffic.json
python profiles/extract_traffic.py $tag c2 gpurun_out/${tag}_c2_*.ncu-rep > profiles/${tag}_c2_traffic.json
cp gpurun_out/${tag}_launches.csv profiles/${tag}_launches.csv
for f in gpurun_out/${tag}_bench_*.json gpurun_out/${tag}_torchrun_*.json; do cp $f profiles/; done
# SASS evidence: opcode counts of the shipped library + the blend's packed-FP32 loop
python profiles/sass_summary.py > profiles/${tag}_sass.txt
ls -la profiles/${tag}_*

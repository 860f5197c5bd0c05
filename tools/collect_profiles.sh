#!/bin/bash
# gpurun_out/<tag>_* (tools/round_end.sh) -> the tracked summaries under profiles/:  tools/collect_profiles.sh <tag>
tag=$1
python profiles/summarize_ncu.py $tag gpurun_out/${tag}_launches.csv gpurun_out/${tag}_c44k_*.ncu-rep gpurun_out/${tag}_c2_*.ncu-rep > profiles/${tag}_ncu.md
python profiles/extract_traffic.py $tag c4-4k gpurun_out/${tag}_c44k_*.ncu-rep > profiles/${tag}_c4-4k_traffic.json
python profiles/extract_traffic.py $tag c2 gpurun_out/${tag}_c2_*.ncu-rep > profiles/${tag}_c2_traffic.json
cp gpurun_out/${tag}_launches.csv profiles/${tag}_launches.csv
for f in gpurun_out/${tag}_bench_*.json gpurun_out/${tag}_torchrun_*.json; do cp $f profiles/; done
# SASS evidence: opcode counts of the shipped library + the hot loops' packed-FP32 / cp.async lines
lib=paper_2408_07967_b200/_lib/libflashgs_b200.so
{
  echo "# cuobjdump -sass $lib (sm_100a), opcode counts per kernel family"
  cuobjdump -sass $lib | awk '
    /Function :/ { fn=$3; sub(/^_Z[0-9]+/, "", fn); sub(/I.*$/, "", fn) }
    /^\s+\/\*[0-9a-f]+\*\// { op=$2; sub(/\..*$/, "", op); sub(/;$/, "", op); if (op ~ /^@/) { op=$3; sub(/\..*$/, "", op); sub(/;$/, "", op) } c[fn" "op]++ }
    END { for (k in c) print k, c[k] }' | sort | awk '$2 ~ /^(FFMA2|FMUL2|FADD2|LDGSTS|MUFU|UTMALDG|UTMASTG|UTCHMMA|LDTM|STTM|ATOMS|ATOMG|RED|REDUX|SHFL|MATCH|BAR|ACQBULK|SYNCS)$/'
  echo
  echo "# first packed-FP32 and LDGSTS instructions of k_blend2 (CONTRIB, no extras)"
  cuobjdump -sass -fun '_Z8k_blend2ILb1ELb0EEvPKfS1_PKjS3_PKiS3_iiiiffffPfS6_S6_PhP9fgs_stats' $lib | grep -E "FFMA2|FMUL2|FADD2|LDGSTS|MUFU.EX2" | head -24
} > profiles/${tag}_sass.txt
ls -la profiles/${tag}_*

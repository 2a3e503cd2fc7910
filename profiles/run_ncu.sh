#!/bin/bash
# ncu evidence for the bench's kernels (run under gpurun on ONE GPU).
# 1) launch list (per-launch device time, cold cache, serialised)
# 2) one --set full capture of the two hot launches (bcast, reduce), exported
#    as CSV (raw metrics + per-instruction source page) next to the report.
# usage: bash profiles/run_ncu.sh <outdir> <tag>
set -e
OUT=${1:-gpurun_out}
TAG=${2:-r1}
mkdir -p $OUT
CMD="python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD > $OUT/plain_$TAG.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launches_$TAG.log 2>&1
CMD2="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
$CMD2 > $OUT/plain2_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:segments_kernel -s 6 -c 2 -o /tmp/prof_$TAG $CMD2 > $OUT/ncu_full_$TAG.log 2>&1
ncu -i /tmp/prof_$TAG.ncu-rep --page raw --csv > $OUT/prof_${TAG}_raw.csv
ncu -i /tmp/prof_$TAG.ncu-rep --page details --csv > $OUT/prof_${TAG}_details.csv
echo done

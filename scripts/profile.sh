#!/bin/bash
# Run on the GPU box (via gpurun). Plain run first; ncu only if it exited 0.
#   scripts/profile.sh <tag> <kernel-regex> [extra bench args]
set -u
TAG=$1; KREGEX=$2; shift 2
OUT=gpurun_out
mkdir -p $OUT
CMD="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 $*"
$CMD > $OUT/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $CMD > $OUT/${TAG}_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$KREGEX -s 1 -c 1 -o $OUT/${TAG}_prof $CMD > $OUT/${TAG}_ncu_full.log 2>&1
echo "exit=$?"
tail -3 $OUT/${TAG}_ncu_full.log

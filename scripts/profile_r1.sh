#!/bin/bash
# Round-1 evidence: bench line, launch list, full ncu of the two tensor-core kernels.
set -u
OUT=gpurun_out; mkdir -p $OUT
python bench.py --steps 200 --warmup 10 > $OUT/r1_bench.json 2> $OUT/r1_bench.err
echo "bench exit=$?"
CMD="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0"
$CMD > $OUT/r1_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r1_launches.csv $CMD > $OUT/r1_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bwd_tc|k_fwd_tc|k_adam|k_sample|k_composite" -s 5 -c 5 -o $OUT/r1_full $CMD > $OUT/r1_ncu_full.log 2>&1
echo "ncu exit=$?"

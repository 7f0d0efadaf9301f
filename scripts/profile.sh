#!/bin/bash
# Evidence capture on the GPU box (run through gpurun; one GPU):
#   scripts/profile.sh <tag> [bench args, e.g. --mlp bf16x3 --workload cfg2]
# 1. the bench line (plain run, no profiler);
# 2. the launch list of the same command (ncu gpu__time_duration.sum, cold and serialised);
# 3. one `ncu --set full` capture of each step kernel (after the plain run exited 0),
#    with source pages and the raw metric CSV of the tensor-core kernels.
# Outputs: gpurun_out/<tag>_*; summarise with scripts/ncu_summary.py into profiles/.
set -u
TAG=$1; shift
OUT=gpurun_out; mkdir -p $OUT
python bench.py --steps 200 --warmup 10 "$@" > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench exit=$?"
CMD="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 --steady-steps 0 $*"
$CMD > $OUT/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/${TAG}_launches.csv $CMD > $OUT/${TAG}_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bwd_tc|k_fwd_wx|k_fwd_ws|k_fwd_ts|k_fwd_tc|k_adam|k_sample|k_composite|k_mlp_grad_reduce" -s 6 -c 7 -o $OUT/${TAG}_full $CMD > $OUT/${TAG}_ncu_full.log 2>&1
echo "ncu exit=$?"
for k in k_bwd_tc k_fwd_wx; do
  ncu -i $OUT/${TAG}_full.ncu-rep -k regex:$k --page source --csv --print-source cuda,sass > $OUT/${TAG}_src_$k.csv 2>/dev/null
done
ncu -i $OUT/${TAG}_full.ncu-rep --page raw --csv > $OUT/${TAG}_raw.csv 2>/dev/null
ncu -i $OUT/${TAG}_full.ncu-rep --page details > $OUT/${TAG}_details.txt 2>/dev/null
ls -la $OUT | grep $TAG

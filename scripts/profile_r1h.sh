#!/bin/bash
# Round-1 (latest state: TMEM slot, forward carve-out + TMA feature store, 64-register compositing) evidence on the current code: bench line, launch
# list, full ncu of the step's kernels (one launch each), source pages.
set -u
OUT=gpurun_out; mkdir -p $OUT
python bench.py --steps 200 --warmup 10 > $OUT/r1h_bench.json 2> $OUT/r1h_bench.err
echo "bench exit=$?"
CMD="python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0"
$CMD > $OUT/r1h_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r1h_launches.csv $CMD > $OUT/r1h_ncu_launch.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_bwd_tc|k_fwd_tc|k_adam|k_sample|k_composite" -s 5 -c 5 -o $OUT/r1h_full $CMD > $OUT/r1h_ncu_full.log 2>&1
echo "ncu exit=$?"
for k in k_bwd_tc k_fwd_tc; do
  ncu -i $OUT/r1h_full.ncu-rep -k regex:$k --page source --csv --print-source cuda,sass > $OUT/r1h_src_$k.csv 2>/dev/null
done
ncu -i $OUT/r1h_full.ncu-rep --page raw --csv > $OUT/r1h_raw.csv 2>/dev/null
ncu -i $OUT/r1h_full.ncu-rep --page details > $OUT/r1h_details.txt 2>/dev/null
ls -la $OUT
# the other BASELINE workloads and the fp32-MLP mode, on the same code
mkdir -p $OUT/r1h_workloads
for w in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w > $OUT/r1h_workloads/$w.json 2> $OUT/r1h_workloads/$w.err
  echo "$w exit=$?"
done
timeout 600 python bench.py --mlp fp32 > $OUT/r1h_workloads/cfg2_fp32.json 2> $OUT/r1h_workloads/cfg2_fp32.err
echo "fp32 exit=$?"

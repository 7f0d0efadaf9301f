#!/bin/bash
# Final evidence of a round on one GPU box (run through gpurun):
#   bash scripts/gpu_session.sh <tag>
# full GPU test suite; the headline capture (scripts/profile.sh: 200-step bench line with CPU
# baseline, launch list, ncu --set full); the other workloads / MLP modes; the reference arm;
# the backward phase trace. Outputs gpurun_out/<tag>_*; summarised into profiles/.
set -x
T=${1:-r2f}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_gputests.log 2>&1
bash scripts/profile.sh ${T} --mlp bf16x3
for w in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w --steps 50 --warmup 5 > gpurun_out/${T}_wl_$w.json 2> gpurun_out/${T}_wl_$w.err
done
timeout 900 python bench.py --mlp bf16 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/${T}_wl_cfg2_bf16.json 2> gpurun_out/${T}_wl_cfg2_bf16.err
timeout 900 python bench.py --mlp fp32 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/${T}_wl_cfg2_fp32.json 2> gpurun_out/${T}_wl_cfg2_fp32.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${T}_reference.json 2> gpurun_out/${T}_reference.err
python scripts/bwd_trace.py bf16x3 gpurun_out/${T}_trace_x3.json > gpurun_out/${T}_trace.log 2>&1
echo done

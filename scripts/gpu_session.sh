set -x
mkdir -p gpurun_out
T=r2i
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --steady-steps 0"
PRENOM_FWDS_TS=2 timeout 300 python -m pytest tests/test_split_bf16.py -x -q -m gpu -k "forward or first_step" > gpurun_out/${T}_tests_ws.log 2>&1
PRENOM_FWDS_TS=2 $B --mlp bf16x3 > gpurun_out/${T}_x3_ws.log 2>&1
PRENOM_FWDS_TS=2 PRENOM_FWDS_CARVEOUT=44 $B --mlp bf16x3 > gpurun_out/${T}_x3_ws44.log 2>&1
PRENOM_FWDS_TS=2 PRENOM_FWDS_CTAS=1 PRENOM_FWDS_CARVEOUT=30 $B --mlp bf16x3 > gpurun_out/${T}_x3_ws1.log 2>&1
PRENOM_FWD_TS=2 $B --mlp bf16 > gpurun_out/${T}_bf16_ws.log 2>&1
python scripts/bwd_trace.py bf16x3 gpurun_out/${T}_trace_x3.json > gpurun_out/${T}_trace.log 2>&1
python scripts/bwd_trace.py bf16 gpurun_out/${T}_trace_bf16.json >> gpurun_out/${T}_trace.log 2>&1
echo done

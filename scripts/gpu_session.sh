set -x
mkdir -p gpurun_out
T=r2t
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --steady-steps 0"
PRENOM_FWDS_TS=3 PRENOM_FWD_TS=3 timeout 600 python -m pytest tests/test_split_bf16.py tests/test_gpu_parity.py -x -q -m gpu -k "not 200_steps" > gpurun_out/${T}_tests.log 2>&1
for i in 1 2; do
  $B --mlp bf16x3 > gpurun_out/${T}_x3_ws_$i.log 2>&1
  PRENOM_FWDS_TS=3 $B --mlp bf16x3 > gpurun_out/${T}_x3_wx_$i.log 2>&1
  PRENOM_FWDS_TS=3 PRENOM_FWDS_CARVEOUT=30 $B --mlp bf16x3 > gpurun_out/${T}_x3_wx30_$i.log 2>&1
done
PRENOM_FWD_TS=3 PRENOM_FWD_CARVEOUT=30 $B --mlp bf16 > gpurun_out/${T}_bf16_wx30.log 2>&1
$B --mlp bf16 > gpurun_out/${T}_bf16_ws.log 2>&1
echo done

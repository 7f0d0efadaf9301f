set -x
mkdir -p gpurun_out
T=r2s
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --steady-steps 0 --mlp bf16x3"
PRENOM_FWDS_TS=6 timeout 300 python -m pytest tests/test_split_bf16.py -x -q -m gpu -k "forward or first_step" > gpurun_out/${T}_tests.log 2>&1
for i in 1 2; do
  $B > gpurun_out/${T}_ws2_$i.log 2>&1
  PRENOM_FWDS_TS=6 $B > gpurun_out/${T}_ws6_$i.log 2>&1
done
echo done

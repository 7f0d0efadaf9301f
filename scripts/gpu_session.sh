set -x
mkdir -p gpurun_out
T=r2h
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --steady-steps 0"
timeout 900 python -m pytest tests/test_split_bf16.py -x -q -m gpu -k "not 200_steps" > gpurun_out/${T}_tests.log 2>&1
$B --mlp bf16x3 > gpurun_out/${T}_x3.log 2>&1
PRENOM_SPLIT_MASK=23 $B --mlp bf16x3 > gpurun_out/${T}_x3_m23.log 2>&1
PRENOM_SPLIT_MASK=39 $B --mlp bf16x3 > gpurun_out/${T}_x3_m39.log 2>&1
timeout 900 python scripts/loss_parity.py cfg1 200 --oracle-cache profiles/loss_parity_cfg1.json --modes x3m23,x3m39,x3m7 --repeats 2 --tag ${T} > gpurun_out/${T}_lp_cfg1.log 2>&1
timeout 900 python scripts/loss_parity.py cfg2 200 --oracle-cache profiles/loss_parity_cfg2.json --modes x3m23,x3m39 --repeats 2 --tag ${T} > gpurun_out/${T}_lp_cfg2.log 2>&1
cp profiles/loss_parity_*_${T}.json gpurun_out/
echo done

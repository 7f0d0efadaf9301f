set -x
mkdir -p gpurun_out
T=r2l
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --steady-steps 0"
timeout 600 python -m pytest tests/test_split_bf16.py tests/test_full_size.py -x -q -m gpu -k "not 200_steps" > gpurun_out/${T}_tests.log 2>&1
$B --mlp bf16x3 > gpurun_out/${T}_x3.log 2>&1
$B --mlp bf16 > gpurun_out/${T}_bf16.log 2>&1
timeout 1500 bash scripts/profile.sh ${T} --mlp bf16x3 > gpurun_out/${T}_profile.log 2>&1
echo done

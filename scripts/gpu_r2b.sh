set -x
mkdir -p gpurun_out
T=r2b
timeout 900 python -m pytest tests/test_split_bf16.py -x -q -m gpu -k "not 200_steps" > gpurun_out/${T}_split_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_meta_multi.py -x -q -m gpu > gpurun_out/${T}_meta_tests.log 2>&1
for cfg in "512 2" "256 2" "256 3" "512 1"; do set -- $cfg
  PRENOM_FWDS_THREADS=$1 PRENOM_FWDS_CTAS=$2 timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --mlp bf16x3 > gpurun_out/${T}_bench_x3_t$1_c$2.log 2>&1
done
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --mlp bf16 > gpurun_out/${T}_bench_bf16.log 2>&1
timeout 600 python scripts/loss_parity.py cfg2 200 --oracle-cache profiles/loss_parity_cfg2.json --modes bf16x3 --repeats 3 --tag ${T} > gpurun_out/${T}_lp_cfg2.log 2>&1
timeout 600 python scripts/loss_parity.py cfg1 200 --oracle-cache profiles/loss_parity_cfg1.json --modes bf16x3 --repeats 3 --tag ${T} > gpurun_out/${T}_lp_cfg1.log 2>&1
cp profiles/loss_parity_*_${T}.json gpurun_out/
echo done

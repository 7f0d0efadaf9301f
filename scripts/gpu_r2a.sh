set -x
mkdir -p gpurun_out
nproc > gpurun_out/r2a_nproc.txt
timeout 900 python -m pytest tests/test_split_bf16.py -x -q -m gpu -k "not 200_steps" > gpurun_out/r2a_split_tests.log 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "bf16 or tile or tcgen05" > gpurun_out/r2a_parity.log 2>&1
for m in bf16 bf16x3; do
  timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 --mlp $m > gpurun_out/r2a_bench_$m.log 2>&1
done
for t in 512 256; do for c in 2 1; do
  PRENOM_FWDS_THREADS=$t PRENOM_FWDS_CTAS=$c timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --mlp bf16x3 > gpurun_out/r2a_bench_x3_t${t}_c${c}.log 2>&1
done; done
timeout 1200 python scripts/loss_parity.py cfg2 200 --oracle-cache profiles/loss_parity_cfg2.json --modes bf16,bf16x3,x3m1,x3m2,x3m4,x3m3,fp32 --tag r2a > gpurun_out/r2a_lp_cfg2.log 2>&1
timeout 600 python scripts/loss_parity.py cfg1 200 --oracle-cache profiles/loss_parity_cfg1.json --modes bf16,bf16x3,x3m1,x3m2,x3m4,x3m3 --tag r2a > gpurun_out/r2a_lp_cfg1.log 2>&1
cp profiles/loss_parity_*_r2a.json gpurun_out/
timeout 1500 python -m pytest tests/test_split_bf16.py -x -q -m gpu -k "200_steps" -s > gpurun_out/r2a_split_200.log 2>&1
echo done

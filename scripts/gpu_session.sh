set -x
mkdir -p gpurun_out
T=r2z
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --steady-steps 0"
V=paper_2503_01582_b200/_lib/variants/libprenom_one.so
timeout 600 python -m pytest tests/test_split_bf16.py tests/test_gpu_parity.py -x -q -m gpu -k "not 200_steps" > gpurun_out/${T}_tests.log 2>&1
for i in 1 2; do
  $B --mlp bf16x3 > gpurun_out/${T}_x3_two_$i.log 2>&1
  PRENOM_LIB=$V $B --mlp bf16x3 > gpurun_out/${T}_x3_one_$i.log 2>&1
done
$B --mlp bf16 > gpurun_out/${T}_bf16_two.log 2>&1
PRENOM_LIB=$V $B --mlp bf16 > gpurun_out/${T}_bf16_one.log 2>&1
python scripts/bwd_trace.py bf16x3 gpurun_out/${T}_trace_x3.json > gpurun_out/${T}_trace.log 2>&1
echo done

set -x
mkdir -p gpurun_out
T=r2n
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --steady-steps 0 --mlp bf16x3"
timeout 1200 python -m pytest tests/test_split_bf16.py tests/test_gpu_meta_multi.py -x -q -m gpu > gpurun_out/${T}_tests.log 2>&1
for i in 1 2; do
  $B > gpurun_out/${T}_x3_pipe_$i.log 2>&1
  PRENOM_LIB=paper_2503_01582_b200/_lib/variants/libprenom_nopipe.so $B > gpurun_out/${T}_x3_nopipe_$i.log 2>&1
done
python scripts/bwd_trace.py bf16x3 gpurun_out/${T}_trace_x3.json > gpurun_out/${T}_trace.log 2>&1
echo done

# round-2 final evidence: headline profile, workloads, full GPU suite, smoke, reference arm
set -x
mkdir -p gpurun_out
T=${T:-r2v}
timeout 1500 bash scripts/profile.sh ${T} --mlp bf16x3 > gpurun_out/${T}_profile.log 2>&1
python scripts/bwd_trace.py bf16x3 gpurun_out/${T}_trace_x3.json > gpurun_out/${T}_trace.log 2>&1
mkdir -p gpurun_out/${T}_workloads
for w in cfg1 cfg3 cfg4 cfg5; do
  timeout 900 python bench.py --workload $w --steps 50 --warmup 5 > gpurun_out/${T}_workloads/$w.json 2> gpurun_out/${T}_workloads/$w.err
done
timeout 600 python bench.py --mlp bf16 --steps 200 --warmup 10 --no-cpu-baseline > gpurun_out/${T}_workloads/cfg2_bf16.json 2> gpurun_out/${T}_workloads/cfg2_bf16.err
timeout 600 python bench.py --mlp fp32 --steps 50 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${T}_workloads/cfg2_fp32.json 2> gpurun_out/${T}_workloads/cfg2_fp32.err
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${T}_gputests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${T}_reference.json 2> gpurun_out/${T}_reference.err
echo done

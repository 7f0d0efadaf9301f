# final-state validation: the driver's commands (GPU test suite, smoke, default bench, reference arm)
set -x
mkdir -p gpurun_out
T=${T:-r2o}
timeout 2400 python -m pytest tests -q -m gpu > gpurun_out/${T}_gputests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/${T}_bench_default.json 2> gpurun_out/${T}_bench_default.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/${T}_reference.json 2> gpurun_out/${T}_reference.err
echo done

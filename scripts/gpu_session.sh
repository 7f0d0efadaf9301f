set -x
mkdir -p gpurun_out
T=r2p
timeout 900 python bench.py > gpurun_out/${T}_bench_default_1.json 2> gpurun_out/${T}_bench_default_1.err
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/${T}_bench_default_2.json 2> gpurun_out/${T}_bench_default_2.err
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --steady-steps 0 --mlp bf16x3"
$B > gpurun_out/${T}_ws2.log 2>&1
PRENOM_FWDS_TS=3 PRENOM_FWDS_CTAS=1 PRENOM_FWDS_CARVEOUT=30 $B > gpurun_out/${T}_ws3.log 2>&1
PRENOM_FWDS_TS=4 PRENOM_FWDS_CTAS=2 PRENOM_FWDS_CARVEOUT=58 $B > gpurun_out/${T}_ws4.log 2>&1
PRENOM_FWDS_TS=5 PRENOM_FWDS_CTAS=1 PRENOM_FWDS_CARVEOUT=30 $B > gpurun_out/${T}_ws5.log 2>&1
PRENOM_FWDS_TS=3 PRENOM_FWDS_CTAS=1 PRENOM_FWDS_CARVEOUT=44 $B > gpurun_out/${T}_ws3b.log 2>&1
echo done

# one gpurun session of round-2 checks (tag r2d)
set -x
mkdir -p gpurun_out
T=r2d
B="timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0"
timeout 900 python -m pytest tests/test_split_bf16.py tests/test_integration.py -x -q -m gpu -k "not 200_steps" > gpurun_out/${T}_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "bf16 or tile or tcgen05" > gpurun_out/${T}_tests_bf16.log 2>&1
$B --mlp bf16x3 > gpurun_out/${T}_x3_default.log 2>&1
PRENOM_FWDS_TS=0 $B --mlp bf16x3 > gpurun_out/${T}_x3_nots.log 2>&1
PRENOM_FWDS_THREADS=256 PRENOM_FWDS_CTAS=3 PRENOM_FWDS_CARVEOUT=72 $B --mlp bf16x3 > gpurun_out/${T}_x3_ts256c3.log 2>&1
PRENOM_FWDS_THREADS=512 PRENOM_FWDS_CTAS=3 PRENOM_FWDS_CARVEOUT=72 $B --mlp bf16x3 > gpurun_out/${T}_x3_ts512c3.log 2>&1
PRENOM_FWDS_THREADS=256 PRENOM_FWDS_CTAS=4 PRENOM_FWDS_CARVEOUT=86 $B --mlp bf16x3 > gpurun_out/${T}_x3_ts256c4.log 2>&1
PRENOM_FWDS_THREADS=256 PRENOM_FWDS_CTAS=2 PRENOM_FWDS_CARVEOUT=44 $B --mlp bf16x3 > gpurun_out/${T}_x3_ts256c2.log 2>&1
for w in 1 2 3; do PRENOM_BWD_WAIT=$w $B --mlp bf16x3 > gpurun_out/${T}_x3_wait$w.log 2>&1; done
$B --mlp bf16 > gpurun_out/${T}_bf16.log 2>&1
PRENOM_FWD_TS=1 $B --mlp bf16 > gpurun_out/${T}_bf16_ts.log 2>&1
PRENOM_FWD_TS=1 PRENOM_FWD_CTAS=4 PRENOM_FWD_CARVEOUT=44 $B --mlp bf16 > gpurun_out/${T}_bf16_ts4.log 2>&1
timeout 600 python scripts/loss_parity.py cfg2 200 --oracle-cache profiles/loss_parity_cfg2.json --modes bf16x3 --repeats 2 --tag ${T} > gpurun_out/${T}_lp_cfg2.log 2>&1
timeout 600 python scripts/loss_parity.py cfg1 200 --oracle-cache profiles/loss_parity_cfg1.json --modes bf16x3 --repeats 2 --tag ${T} > gpurun_out/${T}_lp_cfg1.log 2>&1
cp profiles/loss_parity_*_${T}.json gpurun_out/
echo done

# loss after 200 steps at BASELINE cfg1 / cfg2 full size on the final code
set -x
mkdir -p gpurun_out
T=${T:-r2w}
timeout 1200 python scripts/loss_parity.py cfg2 200 --oracle-cache profiles/r1/loss_parity_cfg2.json --modes bf16x3,bf16,fp32 --repeats 2 --tag ${T} > gpurun_out/${T}_lp_cfg2.log 2>&1
timeout 1200 python scripts/loss_parity.py cfg1 200 --oracle-cache profiles/r1/loss_parity_cfg1.json --modes bf16x3,bf16,fp32 --repeats 2 --tag ${T} > gpurun_out/${T}_lp_cfg1.log 2>&1
cp profiles/loss_parity_*_${T}.json gpurun_out/
echo done

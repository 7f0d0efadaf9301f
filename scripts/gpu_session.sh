set -x
mkdir -p gpurun_out
T=r2q
B="timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 --steady-steps 0"
for w in cfg3 cfg5; do
  for mt in 8 16 32; do for ln in 8 16; do
    PRENOM_MIN_TILES_PER_CTA=$mt PRENOM_LANES=$ln $B --workload $w > gpurun_out/${T}_${w}_mt${mt}_l${ln}.log 2>&1
  done; done
done
for tpg in 4 8; do for mt in 8 16; do
  PRENOM_MIN_TILES_PER_CTA=$mt $B --workload cfg4 --tasks-per-gpu $tpg > gpurun_out/${T}_cfg4_t${tpg}_mt${mt}.log 2>&1
done; done
echo done

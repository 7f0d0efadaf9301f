#!/bin/bash
# launch-shape sweep for the step kernels (cfg2): env knobs of kernels_tc.cu
run() { env "$@" timeout 120 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | python scripts/summ.py "$*"; }
run PRENOM_X=default
run PRENOM_BWD_SMEM_KB=79 PRENOM_BWD_CARVEOUT=72
run PRENOM_BWD_SMEM_KB=70 PRENOM_BWD_CARVEOUT=72
run PRENOM_FWD_THREADS=512 PRENOM_FWD_CTAS=2 PRENOM_FWD_SMEM_KB=40 PRENOM_FWD_CARVEOUT=44
run PRENOM_FWD_CTAS=3 PRENOM_FWD_SMEM_KB=40 PRENOM_FWD_CARVEOUT=72
run PRENOM_FWD_CTAS=4 PRENOM_FWD_SMEM_KB=40 PRENOM_FWD_CARVEOUT=72
run PRENOM_X=default

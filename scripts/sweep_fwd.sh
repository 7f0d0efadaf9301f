#!/bin/bash
# usage: sweep_fwd.sh "ctas:smem_kb" ...
for cfg in "$@"; do
  c=${cfg%%:*}; k=${cfg##*:}
  PRENOM_FWD_CTAS=$c PRENOM_FWD_SMEM_KB=$k python bench.py --steps 100 --warmup 5 --mlp bf16 --no-cpu-baseline --e2e-steps 0 2>&1 | python scripts/summ.py "ctas=$c smem=$k"
done

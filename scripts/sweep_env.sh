#!/bin/bash
# usage: sweep_env.sh "VAR=a VAR2=b" "VAR=c" ...   (cfg2 bench per env set)
for cfg in "$@"; do
  env $cfg python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 2>&1 | python scripts/summ.py "$cfg"
done

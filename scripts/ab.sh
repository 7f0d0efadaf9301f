#!/bin/bash
# A/B the libraries in exp/*.so on the cfg2 bench (interleaved, 2 rounds).
for rnd in 1 2; do
  for lib in exp/*.so; do
    PRENOM_LIB=$PWD/$lib python bench.py --steps 100 --warmup 5 --no-cpu-baseline --e2e-steps 0 "$@" 2>&1 | python scripts/summ.py "$(basename $lib)"
  done
done

#!/bin/bash
# A/B the libraries in exp/*.so on the multi-object and Reptile workloads (one round each).
for w in "$@"; do
  for lib in exp/*.so; do
    PRENOM_LIB=$PWD/$lib timeout 600 python bench.py --workload $w --no-cpu-baseline 2>&1 | python scripts/summ.py "$w $(basename $lib)"
  done
done

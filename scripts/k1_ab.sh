#!/bin/bash
# A/B of K1 variants on the configs (timing only); correctness via k1_variants.py
for v in default deep; do
  if [ "$v" = deep ]; then export IPI_K1_DEEP=1; else unset IPI_K1_DEEP; fi
  echo "== $v"
  timeout 300 python scripts/config_sweep.py --k1-only --configs ${1:-1,2} > gpurun_out/ab_$v.log 2>&1
  python scripts/show_sweep.py gpurun_out/ab_$v.log
done

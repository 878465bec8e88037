#!/bin/bash
# C4 K1 (generic rows) A/B: loads per lane (IPI_K1_GEN_U) x CTAs per SM for the
# windowed plan (IPI_K1_GEN_CTAS).  Timing only (correctness: test_gpu_k1_variants).
for cfg in ${C4_SHAPES:-"8 2" "8 3" "8 4" "8 6" "8 8" "4 6"}; do
  set -- $cfg
  echo "== U=$1 ctas/SM=$2"
  IPI_K1_GEN_U=$1 IPI_K1_GEN_CTAS=$2 timeout 300 python scripts/config_sweep.py --k1-only --configs 4 2>&1 | python scripts/show_sweep.py /dev/stdin
done

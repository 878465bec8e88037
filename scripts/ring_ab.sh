#!/bin/bash
# A/B of the flat-row K1 kernels on C3 (timing only; correctness: tests/test_gpu_k1_variants.py)
for v in ${RING_SHAPES:-reg 4x18 4x16 6x12}; do
  unset IPI_RING_STAGES IPI_RING_WARPS
  case $v in
    reg) export IPI_K1_RING=0 ;;
    *) export IPI_K1_RING=1 IPI_RING_STAGES=${v%x*} IPI_RING_WARPS=${v#*x} ;;
  esac
  echo "== $v"
  timeout 300 python scripts/config_sweep.py --k1-only --configs ${1:-3} > gpurun_out/ring_$v.log 2>&1
  python scripts/show_sweep.py gpurun_out/ring_$v.log
done

#!/bin/bash
# A/B of the uniform-row K1 kernels (K = 64) on C2 (timing only; correctness:
# tests/test_gpu_k1_variants.py).  Shapes are warps x stages x waves.
for v in ${URING_SHAPES:-reg 8x4x1 8x4x2 10x3x1 12x4x2 16x4x2 8x3x1}; do
  unset IPI_URING_WARPS IPI_URING_STAGES IPI_URING_WAVES
  case $v in
    reg) export IPI_K1_URING=0 ;;
    *) IFS=x read -r w s q <<< "$v"
       export IPI_K1_URING=1 IPI_URING_WARPS=$w IPI_URING_STAGES=$s IPI_URING_WAVES=$q ;;
  esac
  echo "== $v"
  timeout 300 python scripts/config_sweep.py --k1-only --configs ${1:-2} > gpurun_out/uring_$v.log 2>&1
  python scripts/show_sweep.py gpurun_out/uring_$v.log
done

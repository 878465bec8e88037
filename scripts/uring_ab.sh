#!/bin/bash
# A/B of the uniform-row K1 kernels (K = 64) on C2 (timing only; correctness:
# tests/test_gpu_k1_variants.py).  Shapes: warps x stages x waves x lookahead;
# WIN_ASYNC="0 1" also toggles the cp.async V-window staging.
for v in ${URING_SHAPES:-reg 12x3x4x1 10x3x2x1 10x4x4x2 8x5x2x2 12x4x6x2}; do
  for wa in ${WIN_ASYNC:-1}; do
    unset IPI_URING_WARPS IPI_URING_STAGES IPI_URING_WAVES IPI_URING_AHEAD
    export IPI_K1_WIN_ASYNC=$wa IPI_K1_INTERLEAVE=${INTERLEAVE:-1} IPI_K1_ROTATE=${ROTATE:-1}
    case $v in
      reg) export IPI_K1_URING=0 ;;
      *) IFS=x read -r w s q d <<< "$v"
         export IPI_K1_URING=1 IPI_URING_WARPS=$w IPI_URING_STAGES=$s IPI_URING_WAVES=$q IPI_URING_AHEAD=${d:-1} ;;
    esac
    echo "== $v win_async=$wa interleave=${INTERLEAVE:-1} rotate=${ROTATE:-1}"
    timeout 300 python scripts/config_sweep.py --k1-only --configs ${1:-2} > gpurun_out/uring_$v.log 2>&1
    python scripts/show_sweep.py gpurun_out/uring_$v.log
  done
done

#!/bin/bash
# C5 per-rank proxy (R = 8, rank 0) A/B over K1 kernels / ring shapes (timing only).
#   variants: reg (register-pipelined uniform kernel), deep, or WxSxQxD ring shapes;
#   INTERLEAVE / ROTATE env as in uring_ab.sh
for v in ${C5_SHAPES:-reg deep 12x3x8x1 12x3x4x1}; do
  unset IPI_URING_WARPS IPI_URING_STAGES IPI_URING_WAVES IPI_URING_AHEAD IPI_K1_URING IPI_K1_DEEP
  export IPI_K1_INTERLEAVE=${INTERLEAVE:-1} IPI_K1_ROTATE=${ROTATE:-1}
  case $v in
    reg) export IPI_K1_URING=0 ;;
    deep) export IPI_K1_URING=0 IPI_K1_DEEP=1 ;;
    *) IFS=x read -r w s q d <<< "$v"
       export IPI_URING_WARPS=$w IPI_URING_STAGES=$s IPI_URING_WAVES=$q IPI_URING_AHEAD=$d ;;
  esac
  echo "== $v interleave=${INTERLEAVE:-1} rotate=${ROTATE:-1}"
  timeout 300 python scripts/c5_shard_proxy.py --world ${WORLD:-8} --reps 5 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3f ms frac %.3f blocks %d threads %d variant %d halo %d' % (d['k1_ms'], d['k1_frac'], d['plan']['k1_blocks'], d['plan']['k1_threads'], d['plan']['k1_variant'], d['plan']['halo']))"
done

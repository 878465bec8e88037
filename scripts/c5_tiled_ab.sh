#!/bin/bash
# C5 rank proxy: register-deep (IPI_K1_TILED=0) vs column-tiled (=1) K1; timing only.
for i in 1 2; do
  for t in 0 1; do
    echo "== tiled=$t"
    IPI_K1_TILED=$t timeout 600 python scripts/c5_shard_proxy.py --world ${WORLD:-8} --reps 5 | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.3f ms frac %.3f variant %d build %.2f s' % (d['k1_ms'], d['k1_frac'], d['plan']['k1_variant'], d['build_s']))"
  done
done

#!/bin/bash
# A/B compile-time variants of the tiled K1 (paper_2507_22538_b200/var_*.so.bin,
# built locally with -DIPI_TILED_*): parity spot check + C5 rank-block timing each.
cd ${GRAFT_REPO_ROOT:-.}
cp paper_2507_22538_b200/libipi_b200.so /tmp/orig.so
for v in ${VARS:-4_4}; do
  cp paper_2507_22538_b200/var_$v.so.bin paper_2507_22538_b200/libipi_b200.so
  p=$(timeout 300 python scripts/tiled_pipe_check.py 2>&1 | tail -1)
  r=$(IPI_K1_TILED=1 timeout 300 python scripts/c5_shard_proxy.py --world 8 --reps 5 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.3f ms frac %.3f v%d' % (d['k1_ms'], d['k1_frac'], d['plan']['k1_variant']))")
  echo "variant=$v $r | $p"
done
cp /tmp/orig.so paper_2507_22538_b200/libipi_b200.so

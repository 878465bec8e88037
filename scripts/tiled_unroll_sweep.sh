cd $GRAFT_REPO_ROOT
cp paper_2507_22538_b200/libipi_b200.so /tmp/orig.so
for v in ${VARS:-4_4 8_4 8_8 12_8}; do
  cp paper_2507_22538_b200/var_$v.so.bin paper_2507_22538_b200/libipi_b200.so
  r=$(IPI_K1_TILED=1 timeout 300 python scripts/c5_shard_proxy.py --world 8 --reps 5 | tail -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print('%.3f ms frac %.3f v%d' % (d['k1_ms'], d['k1_frac'], d['plan']['k1_variant']))")
  echo "UN_UF=$v $r"
done
cp /tmp/orig.so paper_2507_22538_b200/libipi_b200.so

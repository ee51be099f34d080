# A/B: L1::no_allocate on the 128-bit streaming loads (WD_L1_NOALLOC) vs default __ldg
for v in paper_1505_03851_b200/_lib/libwarpdraw_b200.so paper_1505_03851_b200/_lib/var/libwd_l1na.so; do
  echo "== $v"
  WARPDRAW_B200_LIB=$v timeout 300 python tools/exp_tiles.py 1000000 1024 41 2>&1 | grep tile
  WARPDRAW_B200_LIB=$v timeout 300 python tools/exp_tiles.py 500000 2048 41 2>&1 | grep tile
  WARPDRAW_B200_LIB=$v timeout 300 python tools/quick_perf.py 256,1024,4096 rows 2>&1 | grep -v Warn | cut -c1-160
done

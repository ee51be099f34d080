for v in paper_1505_03851_b200/_lib/var/libwd_c4.so paper_1505_03851_b200/_lib/var/libwd_c5.so paper_1505_03851_b200/_lib/var/libwd_c6.so; do echo "== $v"; WARPDRAW_B200_LIB=$v python tools/exp_tiles.py 500000 2048 41 2>&1 | grep tile; WARPDRAW_B200_LIB=$v python tools/exp_tiles.py 300000 4096 41 2>&1 | grep tile; done
python tools/exp_tiles.py 1000000 1024 41 2>&1 | grep tile

# A/B the LDA draw across library variants (WARPDRAW_B200_LIB)
for v in "$@"; do echo "== $v"; WARPDRAW_B200_LIB=$v timeout 300 python tools/exp_tiles.py 1000000 2>&1 | grep -E "41MB|32MB"; done
echo "== mb5 PIPE4"; WD_PIPE_LDA=4 WARPDRAW_B200_LIB=paper_1505_03851_b200/_lib/var/libwd_mb5.so timeout 300 python tools/exp_tiles.py 1000000 2>&1 | grep -E "41MB|32MB"

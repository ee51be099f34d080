for v in 1 5 6; do echo "== PIPE_LDA=$v"; WD_PIPE_LDA=$v timeout 300 python tools/exp_tiles.py 1000000 2>&1 | grep -E "41MB|20MB"; done
for v in 2 5 6; do echo "== PIPE_ROWS=$v"; WD_PIPE_ROWS=$v timeout 300 python tools/quick_perf.py 256,1024,2048 rows 2>&1 | grep -v Warn | cut -c1-100; done

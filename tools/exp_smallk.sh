for v in 0 1 2 4; do echo "== PIPE_ROWS=$v"; WD_PIPE_ROWS=$v timeout 600 python tools/sweep.py --out /tmp/sw_$v --ks 16,32,48,64,80,112 --lda-ks 16 > /dev/null 2>&1; sed -n 5,12p /tmp/sw_$v.md; done

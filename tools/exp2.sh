for v in 2 4; do echo "ROWS pipe=$v"; WD_PIPE_ROWS=$v timeout 120 python tools/quick_perf.py 256,1024,2048 rows 2>&1 | grep -v Warn | cut -c1-120; done
for v in 1 4; do echo "LDA pipe=$v"; WD_PIPE_LDA=$v timeout 120 python tools/exp_vsweep.py 1024 2>&1 | grep -v Warn; done
for h in "1 2" "1 0"; do set -- $h; echo "LDA pipe=4 l2x=$1 l2t=$2"; WD_PIPE_LDA=4 WD_L2_X=$1 WD_L2_T=$2 timeout 120 python tools/exp_vsweep.py 1024 2>&1 | grep -v Warn; done

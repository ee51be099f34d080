for h in "0 0" "1 2" "1 0" "0 2" "2 2"; do set -- $h; echo "== L2_X=$1 L2_T=$2"; WD_L2_X=$1 WD_L2_T=$2 python tools/exp_tiles.py 1000000 1024 27,41 2>&1 | grep tile; done

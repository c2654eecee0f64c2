cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for d in _w_5141a60 _w_cdf0e87 .; do echo "== $d"; (cd $d && timeout 300 python $GRAFT_REPO_ROOT/scripts/bnb_time.py); done > gpurun_out/bnbcmp.txt 2>&1

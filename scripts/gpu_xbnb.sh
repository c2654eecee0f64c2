cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_xlayout.py -x -q -p no:cacheprovider --timeout 600 -k bnb --durations=5 > gpurun_out/xbnb_test.txt 2>&1; echo "rc=$?" >> gpurun_out/xbnb_test.txt
tail -n 12 gpurun_out/xbnb_test.txt

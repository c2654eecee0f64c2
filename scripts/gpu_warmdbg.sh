cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_warm.py -q -x -p no:cacheprovider > gpurun_out/wd_pytest.txt 2>&1; tail -n 30 gpurun_out/wd_pytest.txt
timeout 300 python scripts/bnb_run.py --family taib --n 20 --sb 1 --iters 30 --warm --budget-s 120 --chunk 1000 > gpurun_out/wd_run.txt 2>&1; tail -n 12 gpurun_out/wd_run.txt | cut -c1-400

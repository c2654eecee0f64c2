# quick validation of the current LAP, then the budgeted tai35b-shaped B&B with the N <= 30
# settings and UB0 = the incumbent of the first run + 1
cd $GRAFT_REPO_ROOT
bash scripts/gpu_iter.sh i2
timeout 2400 python scripts/bnb_run.py --family taib --n 35 --sb 1 --iters 60 --K 1e-4 --warm --batch 8 --ub0 1109441 --budget-s 1800 --chunk 100 --out gpurun_out/j1c_taib35.jsonl > gpurun_out/j1c_taib35.log 2>&1
tail -n 2 gpurun_out/j1c_taib35.log | cut -c1-900

# usage: bash scripts/gpu_j1.sh <tag> <budget_s> : bench lines at N = 20, 35, 40, then the budgeted
# tai35b-shaped B&B (J1)
cd $GRAFT_REPO_ROOT
TAG=${1:-j1}
B=${2:-1500}
mkdir -p gpurun_out
bash scripts/gpu_sizes.sh ${TAG}
timeout $((B + 600)) python scripts/bnb_run.py --family taib --n 35 --iters 10 --sb 1 --batch 8 --budget-s $B --chunk 100 --out gpurun_out/${TAG}_taib35.jsonl > gpurun_out/${TAG}_taib35.log 2>&1
tail -n 2 gpurun_out/${TAG}_taib35.log | cut -c1-900

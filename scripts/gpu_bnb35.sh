# usage: bash scripts/gpu_bnb35.sh <tag> <budget_s> : budgeted B&B of a tai35b-shaped instance (J1)
cd $GRAFT_REPO_ROOT
TAG=${1:-b35}
B=${2:-1500}
mkdir -p gpurun_out
timeout $((B + 600)) python scripts/bnb_run.py --family taib --n 35 --iters 10 --sb 1 --budget-s $B --chunk 200 --out gpurun_out/${TAG}_taib35.jsonl > gpurun_out/${TAG}_taib35.log 2>&1
tail -n 1 gpurun_out/${TAG}_taib35.jsonl | cut -c1-700

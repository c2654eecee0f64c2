# usage: bash scripts/gpu_bnb20.sh <tag> : B&B at N = 20 (tai20b- and nug20-shaped), budgeted
cd $GRAFT_REPO_ROOT
TAG=${1:-b20}
mkdir -p gpurun_out
timeout 700 python scripts/bnb_run.py --family taib --n 20 --iters 10 --sb 1 --budget-s 300 --chunk 100 --out gpurun_out/${TAG}_taib20.jsonl > gpurun_out/${TAG}_taib20.log 2>&1
tail -n 1 gpurun_out/${TAG}_taib20.jsonl | cut -c1-600
timeout 700 python scripts/bnb_run.py --family nug --n 20 --iters 10 --sb 1 --budget-s 240 --chunk 100 --out gpurun_out/${TAG}_nug20.jsonl > gpurun_out/${TAG}_nug20.log 2>&1
tail -n 1 gpurun_out/${TAG}_nug20.jsonl | cut -c1-600

# usage: bash scripts/gpu_j1b.sh <tag> : full solves at N = 20 (warm, T = 60, K = 1e-4) and the
# tai25b- / tai30b-shaped instances, then the budgeted tai35b-shaped run with the same settings
cd $GRAFT_REPO_ROOT
TAG=${1:-j1b}
mkdir -p gpurun_out
for fam in taib nug; do
  timeout 400 python scripts/bnb_run.py --family $fam --n 20 --sb 1 --iters 60 --K 1e-4 --warm --budget-s 300 --chunk 1000 --out gpurun_out/${TAG}_${fam}20.jsonl > /dev/null 2>&1
  tail -n 1 gpurun_out/${TAG}_${fam}20.jsonl | cut -c1-300
done
timeout 900 python scripts/bnb_run.py --family taib --n 25 --sb 1 --iters 60 --K 1e-4 --warm --budget-s 600 --chunk 500 --out gpurun_out/${TAG}_taib25.jsonl > gpurun_out/${TAG}_taib25.log 2>&1
tail -n 1 gpurun_out/${TAG}_taib25.jsonl | cut -c1-300
timeout 1500 python scripts/bnb_run.py --family taib --n 30 --sb 1 --iters 60 --K 1e-4 --warm --batch 12 --budget-s 1200 --chunk 200 --out gpurun_out/${TAG}_taib30.jsonl > gpurun_out/${TAG}_taib30.log 2>&1
tail -n 1 gpurun_out/${TAG}_taib30.jsonl | cut -c1-300

# usage: bash scripts/gpu_bnbstudy.sh <tag> : B&B configuration study at N = 20 (iterations per
# node, K stop, warm children) — full solves, one line each
cd $GRAFT_REPO_ROOT
TAG=${1:-bs}
mkdir -p gpurun_out
for fam in taib nug; do
for cfg in "--iters 10" "--iters 30" "--iters 60 --K 1e-4" "--iters 30 --warm" "--iters 100 --K 1e-4"; do
  timeout 400 python scripts/bnb_run.py --family $fam --n 20 --sb 1 $cfg --budget-s 240 --chunk 1000 --out gpurun_out/${TAG}.jsonl > /dev/null 2>&1
  echo "$fam $cfg: $(tail -n 1 gpurun_out/${TAG}.jsonl | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d.get("complete"), d.get("opt"), d.get("bounded"), round(d.get("seconds",0),1), round(d.get("nodes_per_s",0)))')"
done
done

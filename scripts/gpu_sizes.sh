# usage: bash scripts/gpu_sizes.sh <tag> : bench lines at N = 20, 35, 40 (BASELINE configs 3-5 on one GPU)
cd $GRAFT_REPO_ROOT
TAG=${1:-sz}
mkdir -p gpurun_out
for n in 20 35 40; do
  timeout 900 python bench.py --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_n$n.txt 2>&1
  echo "n=$n $(grep -o '"value": [0-9.]*' gpurun_out/${TAG}_n$n.txt | head -1)"
done

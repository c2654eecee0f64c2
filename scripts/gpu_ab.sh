# usage: bash scripts/gpu_ab.sh <tag> : A/B bench on one box (block layout (default) vs class layout, twice each)
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
mkdir -p gpurun_out
for r in 1 2; do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench_x$r.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb --class-layout > gpurun_out/${TAG}_bench_c$r.txt 2>&1
done

# usage: bash scripts/gpu_x6.sh <tag> : fused-kernel sweep of the transfer-preferring warp fraction
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
mkdir -p gpurun_out
for tm in 1 3 7 15 31 1023; do
  QAP_FUSED_TMASK=$tm timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb --fused > gpurun_out/${TAG}_benchf_$tm.txt 2>&1
  echo "tmask=$tm $(grep -o '"value": [0-9.]*' gpurun_out/${TAG}_benchf_$tm.txt | head -1)"
done

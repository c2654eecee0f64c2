# usage: bash scripts/gpu_promo.sh <tag> : transfer DRAM bytes / duration for each L2 promotion
cd $GRAFT_REPO_ROOT
TAG=${1:-pr}
mkdir -p gpurun_out
for v in 256 128 64 0; do
  QAP_TMA_L2_PROMO=$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_transfer -s 1 -c 2 --csv python scripts/profile_one.py 30 3 0 0 > gpurun_out/${TAG}_promo$v.csv 2>&1
  echo "promo $v"; grep -h "dram__bytes\|gpu__time" gpurun_out/${TAG}_promo$v.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  QAP_TMA_L2_PROMO=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench$v.txt 2>&1
  grep -o '"value": [0-9.]*\|"transfer": {[^}]*}' gpurun_out/${TAG}_bench$v.txt | head -3
done

# usage: VAR=NAME VALS="a b" bash scripts/gpu_ab2.sh <tag> : A/B of an environment knob on one box
# (selected parity tests, transfer/lap ncu metrics, bench without B&B)
cd $GRAFT_REPO_ROOT
TAG=${1:-ab}
mkdir -p gpurun_out
for v in $VALS; do
  export $VAR=$v
  timeout 900 python -m pytest tests/test_gpu_transfer.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "${K:-transfer or config4 or phase or stop}" > gpurun_out/${TAG}_pytest$v.txt 2>&1; echo "$VAR=$v: $(tail -n 1 gpurun_out/${TAG}_pytest$v.txt)"
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_transfer -s 1 -c 1 --csv python scripts/profile_one.py 30 3 0 0 > gpurun_out/${TAG}_ncu$v.csv 2>&1
  grep -h "dram__bytes\|gpu__time" gpurun_out/${TAG}_ncu$v.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench$v.txt 2>&1
  grep -o '"value": [0-9.]*\|"transfer": {[^}]*}\|"lap2": {[^}]*}' gpurun_out/${TAG}_bench$v.txt | head -4
done

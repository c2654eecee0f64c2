# usage: bash scripts/gpu_pipe.sh <tag> : transfer variants (QAP_TRANSFER_PIPE = 0 / 128 / 256):
# parity subset, bench, ncu duration + DRAM bytes of the transfer
cd $GRAFT_REPO_ROOT
TAG=${1:-tp}
mkdir -p gpurun_out
for v in ${VARIANTS:-128 256 0}; do
  QAP_TRANSFER_PIPE=$v timeout 900 python -m pytest tests/test_gpu_transfer.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "transfer or config4 or phase or bound_larger or wide or fixed" > gpurun_out/${TAG}_pytest$v.txt 2>&1; echo "pipe $v: $(tail -n 1 gpurun_out/${TAG}_pytest$v.txt)"
  QAP_TRANSFER_PIPE=$v timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none -k regex:k_transfer -s 1 -c 1 --csv python scripts/profile_one.py 30 3 0 0 > gpurun_out/${TAG}_ncu$v.csv 2>&1
  grep -h "dram__bytes\|gpu__time\|inst_exec" gpurun_out/${TAG}_ncu$v.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
  QAP_TRANSFER_PIPE=$v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench$v.txt 2>&1
  grep -o '"value": [0-9.]*\|"transfer": {[^}]*}\|"lap2": {[^}]*}' gpurun_out/${TAG}_bench$v.txt | head -4
done

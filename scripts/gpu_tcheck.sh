# usage: bash scripts/gpu_tcheck.sh <tag> : transfer + parity GPU tests, bench, transfer ncu duration
cd $GRAFT_REPO_ROOT
TAG=${1:-tc}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_transfer.py tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_test.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_test.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench.txt 2>&1
timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_transfer -s 1 -c 1 --csv python scripts/profile_one.py 30 2 0 4 > gpurun_out/${TAG}_tr.csv 2>&1
tail -n 2 gpurun_out/${TAG}_test.txt
grep -E "inst_executed|gpu__time|dram__bytes" gpurun_out/${TAG}_tr.csv | awk -F'","' '{print $(NF-2), $NF}'

# usage: bash scripts/gpu_lapcheck.sh <tag> : LAP/parity GPU tests, bench, lap2 instruction count (iteration 1)
cd $GRAFT_REPO_ROOT
TAG=${1:-lc}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_test.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_test.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench.txt 2>&1
timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:k_lap -s 2 -c 1 --csv python scripts/profile_one.py 30 1 0 4 > gpurun_out/${TAG}_lap2.csv 2>&1
tail -n 2 gpurun_out/${TAG}_test.txt
grep -o '"value": [0-9.]*' gpurun_out/${TAG}_bench.txt | head -1
grep -E "inst_executed|gpu__time" gpurun_out/${TAG}_lap2.csv | awk -F'","' '{print $(NF-2), $NF}'

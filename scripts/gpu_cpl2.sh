# usage: bash scripts/gpu_cpl2.sh <tag> [notest] : two-columns-per-lane LAP parity tests + N=35 bench
cd $GRAFT_REPO_ROOT
TAG=${1:-c2}
mkdir -p gpurun_out
if [ "$2" != "notest" ]; then
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider --timeout 600 -k "lap_kernel or wide_columns" > gpurun_out/${TAG}_test.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_test.txt
tail -n 2 gpurun_out/${TAG}_test.txt
fi
timeout 600 python bench.py --n 35 --steps 3 --warmup 2 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench35.txt 2>&1
grep -o '"value": [0-9.]*' gpurun_out/${TAG}_bench35.txt | head -1

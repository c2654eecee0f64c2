# usage: bash scripts/gpu_x7.sh <tag> : class-layout tests, A/B bench (class vs block layout, twice), ncu lap2
cd $GRAFT_REPO_ROOT
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_xlayout.py tests/test_gpu_transfer.py -x -q -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_xtest.txt 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_xtest.txt
for r in 1 2; do
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench_x$r.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb --block-layout > gpurun_out/${TAG}_bench_b$r.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lap -s 2 -c 1 -o gpurun_out/${TAG}_lap2 python scripts/profile_one.py 30 1 0 4 > gpurun_out/${TAG}_lap2.txt 2>&1
tail -n 2 gpurun_out/${TAG}_xtest.txt

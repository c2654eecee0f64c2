# usage: bash scripts/gpu_iter.sh <tag> [pytest -k expr] : quick iteration loop — selected GPU
# parity tests, the N=30 bench without B&B, lap2 instruction count at iteration 1
cd $GRAFT_REPO_ROOT
TAG=${1:-it}
K=${2:-"lap_kernel or config4 or phase or bound_larger or wide"}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "$K" > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:k_lap -s 2 -c 1 --csv python scripts/profile_one.py 30 1 0 0 > gpurun_out/${TAG}_lap2_it1.csv 2>&1
tail -n 2 gpurun_out/${TAG}_pytest.txt
grep -o '"value": [0-9.]*\|"lap2": {[^}]*}\|"transfer": {[^}]*}' gpurun_out/${TAG}_bench.txt | head -4
grep -h "inst_executed\|gpu__time" gpurun_out/${TAG}_lap2_it1.csv | awk -F'","' '{print $(NF-2), $NF}'

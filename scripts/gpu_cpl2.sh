# usage: bash scripts/gpu_cpl2.sh <tag> : two-columns-per-lane LAP: parity tests (LAP batches
# m = 33..64, N = 33..35 wide-column iterations, N = 40 one iteration) + bench lines N = 35, 40
cd $GRAFT_REPO_ROOT
TAG=${1:-c2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "lap_kernel or wide or n35 or n40 or config5" > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
tail -n 3 gpurun_out/${TAG}_pytest.txt
for n in 35 40 30; do
  timeout 900 python bench.py --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_n$n.txt 2>&1
  echo "n=$n $(grep -o '"value": [0-9.]*' gpurun_out/${TAG}_n$n.txt | head -1) $(grep -o '"lap2": {[^}]*}' gpurun_out/${TAG}_n$n.txt | head -1)"
done

# usage: bash scripts/gpu_check.sh <tag> : smoke + full GPU suite + N=30 bench (no B&B) + N = 20/35/40 lines
cd $GRAFT_REPO_ROOT
TAG=${1:-ck}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
tail -n 2 gpurun_out/${TAG}_pytest.txt; tail -n 1 gpurun_out/${TAG}_smoke.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
grep -o '"value": [0-9.]*\|"lap2": {[^}]*}\|"transfer": {[^}]*}' gpurun_out/${TAG}_bench.txt | head -3
for n in ${SIZES:-20 35 40}; do
  timeout 900 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_n$n.txt 2>&1
  echo "n=$n $(grep -o '"value": [0-9.]*' gpurun_out/${TAG}_n$n.txt | head -1) $(grep -o '"transfer": {[^}]*}' gpurun_out/${TAG}_n$n.txt | head -1 | cut -c1-60)"
done

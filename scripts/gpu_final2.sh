# usage: bash scripts/gpu_final2.sh <tag> : end-of-round check on one box — smoke, full GPU suite,
# bench (N = 30, every key, default flags), reference arm, bench lines at N = 20 / 35 / 40
cd $GRAFT_REPO_ROOT
TAG=${1:-h}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
tail -n 2 gpurun_out/${TAG}_pytest.txt; tail -n 2 gpurun_out/${TAG}_smoke.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_reference.txt 2>&1; echo "ref rc=$?" >> gpurun_out/${TAG}_reference.txt
for n in 20 35 40; do
  timeout 900 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_n$n.txt 2>&1
done
grep -o '"value": [0-9.]*' gpurun_out/${TAG}_bench.txt gpurun_out/${TAG}_n*.txt gpurun_out/${TAG}_reference.txt | head

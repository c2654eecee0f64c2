# usage: bash scripts/gpu_quick.sh <tag> : GPU tests + bench (no profiles)
cd $GRAFT_REPO_ROOT
TAG=${1:-r}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
tail -n 3 gpurun_out/${TAG}_pytest.txt
tail -n 2 gpurun_out/${TAG}_bench.txt | cut -c1-300

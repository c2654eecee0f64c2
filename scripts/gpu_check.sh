cd $GRAFT_REPO_ROOT
TAG=${1:-r}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -x > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
timeout 300 python scripts/sweep_lap.py 30 > gpurun_out/${TAG}_sweep.txt 2>&1
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
tail -n 3 gpurun_out/${TAG}_smoke.txt gpurun_out/${TAG}_pytest.txt gpurun_out/${TAG}_sweep.txt gpurun_out/${TAG}_bench.txt

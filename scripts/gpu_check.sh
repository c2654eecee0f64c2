cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r1_smi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r1_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/r1_smoke.txt
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 400 -x > gpurun_out/r1_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/r1_pytest.txt
timeout 400 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r1_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/r1_bench.txt
tail -3 gpurun_out/r1_smoke.txt gpurun_out/r1_pytest.txt gpurun_out/r1_bench.txt

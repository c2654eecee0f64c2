# usage: bash scripts/gpu_r2.sh <tag> : GPU tests, bench (N=30), lap2 instruction counts at
# iterations 1, 5, 20 (ncu metrics pass)
cd $GRAFT_REPO_ROOT
TAG=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider --timeout 900 > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
for t in 1 5 20; do
  s=$((2 + 3 * (t - 1)))
  timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_lap -s $s -c 1 --csv python scripts/profile_one.py 30 $t 0 0 > gpurun_out/${TAG}_lap2_it$t.csv 2>&1
done
tail -n 3 gpurun_out/${TAG}_pytest.txt
tail -n 2 gpurun_out/${TAG}_bench.txt | cut -c1-300

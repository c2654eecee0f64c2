# usage: bash scripts/gpu_round2_final.sh <tag> : the round's evidence on one box — smoke, full GPU
# suite, bench (N=30, all keys), reference arm, launch list, ncu --set full of lap2 (iteration 1)
# and the transfer, lap2 instruction counts at iterations 1/5/10/20, bench lines at N=20/35/40,
# (compute-sanitizer is closed on this pool: scripts/gpu_sanitize.sh for pools where it is not)
cd $GRAFT_REPO_ROOT
TAG=${1:-f}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 900 > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
tail -n 2 gpurun_out/${TAG}_pytest.txt
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.txt 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_bench.txt
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${TAG}_reference.txt 2>&1; echo "ref rc=$?" >> gpurun_out/${TAG}_reference.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_launches_stdout.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lap -s 2 -c 1 -o gpurun_out/${TAG}_lap2 python scripts/profile_one.py 30 1 0 0 > gpurun_out/${TAG}_ncu_lap2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_transfer -s 1 -c 1 -o gpurun_out/${TAG}_transfer python scripts/profile_one.py 30 2 0 0 > gpurun_out/${TAG}_ncu_transfer.txt 2>&1
for t in 1 5 10 20; do
  s=$((2 + 3 * (t - 1)))
  timeout 600 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_lap -s $s -c 1 --csv python scripts/profile_one.py 30 $t 0 0 > gpurun_out/${TAG}_lap2_it$t.csv 2>&1
done
for n in 20 35 40; do
  timeout 900 python bench.py --n $n --steps 3 --warmup 2 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_n$n.txt 2>&1
done
tail -n 2 gpurun_out/${TAG}_bench.txt | cut -c1-300

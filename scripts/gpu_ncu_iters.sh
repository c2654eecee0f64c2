# usage: bash scripts/gpu_ncu_iters.sh <tag> : lap2 instruction counts at iterations 1, 5, 10, 20 of a T=20 bound
# (k_lap launches: 2 in iteration 0, then lap2, lap1, lap0 per iteration -> iteration t's lap2 = index 2 + 3 (t - 1))
cd $GRAFT_REPO_ROOT
TAG=${1:-it}
mkdir -p gpurun_out
for t in 1 5 10 20; do
  s=$((2 + 3 * (t - 1)))
  timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_lap -s $s -c 1 --csv python scripts/profile_one.py 30 $t 0 4 > gpurun_out/${TAG}_lap2_it$t.csv 2>&1
done
tail -n 5 gpurun_out/${TAG}_lap2_it20.csv

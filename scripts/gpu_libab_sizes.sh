# usage: VARS="A B" SIZES="30 20" bash scripts/gpu_libab_sizes.sh <tag> : same-box A/B of prebuilt libraries over sizes
cd $GRAFT_REPO_ROOT
TAG=${1:-lab}
mkdir -p gpurun_out
cp paper_1510_02065_b200/libqaprlt2.so /tmp/lib_orig.so
for n in ${SIZES:-30 20 34 35}; do
for v in ${VARS:-A B A B}; do
  cp ablib/lib$v.so paper_1510_02065_b200/libqaprlt2.so
  timeout 600 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_${n}_$v.txt 2>&1
  echo "n=$n $v: $(grep -o '"value": [0-9.]*' gpurun_out/${TAG}_${n}_$v.txt | head -1) $(grep -o '"lap2": {[^}]*}' gpurun_out/${TAG}_${n}_$v.txt | head -1 | cut -c1-60) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/${TAG}_${n}_$v.txt)"
done
done
cp /tmp/lib_orig.so paper_1510_02065_b200/libqaprlt2.so

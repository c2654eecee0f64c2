# usage: VARS="A B A B" bash scripts/gpu_libab.sh <tag> [n] : same-box A/B of prebuilt libraries
# ablib/lib<V>.so (bench without B&B / oracle)
cd $GRAFT_REPO_ROOT
TAG=${1:-lab}
N=${2:-30}
mkdir -p gpurun_out
cp paper_1510_02065_b200/libqaprlt2.so /tmp/lib_orig.so
for v in ${VARS:-A B A B}; do
  cp ablib/lib$v.so paper_1510_02065_b200/libqaprlt2.so
  timeout 600 python bench.py --n $N --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_$v.txt 2>&1
  echo "$v: $(grep -o '"value": [0-9.]*' gpurun_out/${TAG}_$v.txt | head -1) $(grep -o '"lap2": {[^}]*}' gpurun_out/${TAG}_$v.txt | head -1 | cut -c1-60) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/${TAG}_$v.txt)"
done
cp /tmp/lib_orig.so paper_1510_02065_b200/libqaprlt2.so

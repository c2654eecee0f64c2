# usage: bash scripts/gpu_tm.sh <tag> : TMEM LAP warps — parity subset, then bench A/B (QAP_LAP_TMEM=0/1) at N = 30, 20, 34, 35, 40
cd $GRAFT_REPO_ROOT
TAG=${1:-tm}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "${K:-level2_full or lap_kernel or config4_n30_full or phase or bound_larger or golden or wide or config5 or largest}" > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
tail -n 3 gpurun_out/${TAG}_pytest.txt
for n in ${SIZES:-30 20 34 35 40}; do
for v in 0 1 0 1; do
  QAP_LAP_TMEM=$v timeout 600 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_n${n}_$v.txt 2>&1
  echo "n=$n tmem=$v $(grep -o '"value": [0-9.]*' gpurun_out/${TAG}_n${n}_$v.txt | head -1) $(grep -o '"lap2": {[^}]*}' gpurun_out/${TAG}_n${n}_$v.txt | head -1 | cut -c1-60) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/${TAG}_n${n}_$v.txt)"
done
done

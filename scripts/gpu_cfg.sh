# usage: bash scripts/gpu_cfg.sh <tag> : parity subset + bench lines at N = 30, 20, 34, 35, 40 (current build)
cd $GRAFT_REPO_ROOT
TAG=${1:-cf}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "${K:-level2_full or lap_kernel or config4 or phase or bound_larger or wide or config5 or largest or bnb_config2}" > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
tail -n 3 gpurun_out/${TAG}_pytest.txt
for n in ${SIZES:-30 20 34 35 40}; do
  timeout 600 python bench.py --n $n --steps 3 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_n${n}.txt 2>&1
  echo "n=$n $(grep -o '"value": [0-9.]*' gpurun_out/${TAG}_n${n}.txt | head -1) $(grep -o '"lap2": {[^}]*}' gpurun_out/${TAG}_n${n}.txt | head -1 | cut -c1-60) $(grep -o '"frac": [0-9.]*' gpurun_out/${TAG}_n${n}.txt | head -1) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/${TAG}_n${n}.txt)"
done

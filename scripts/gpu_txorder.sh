# usage: bash scripts/gpu_txorder.sh <tag> : A/B of the TMA transfer's dispatch order on one box
# (QAP_TX_CUBE = triple-cube edge, 0 = lexicographic; QAP_TX_G = ntile^G tile groups)
cd $GRAFT_REPO_ROOT
TAG=${1:-tx}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_transfer.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "transfer or config4 or phase" > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
tail -n 2 gpurun_out/${TAG}_pytest.txt
for cfg in ${CFGS:-"0:0" "4:0" "0:1" "4:1" "3:1" "6:1" "4:2" "0:0" "4:1"}; do
  export QAP_TX_CUBE=${cfg%%:*} QAP_TX_G=${cfg##*:}
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/${TAG}_b_${cfg/:/_}.txt 2>&1
  echo "cube=$QAP_TX_CUBE G=$QAP_TX_G $(grep -o '"value": [0-9.]*' gpurun_out/${TAG}_b_${cfg/:/_}.txt | head -1) $(grep -o '"transfer": {[^}]*}' gpurun_out/${TAG}_b_${cfg/:/_}.txt | head -1 | cut -c1-60)"
done
export QAP_TX_CUBE=${NCU_CUBE:-4} QAP_TX_G=0
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_transfer -s 1 -c 1 --csv python scripts/profile_one.py 30 3 0 0 > gpurun_out/${TAG}_ncu41.csv 2>&1
grep -h "dram__bytes\|gpu__time" gpurun_out/${TAG}_ncu41.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'

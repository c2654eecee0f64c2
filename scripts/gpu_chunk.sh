# A/B of the level-2 LAP work-queue grab size (QAP_LAP_CHUNK) at N = 30 and N = 20
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for n in 30 20; do
for c in 4 1 2 4 1 2; do
  QAP_LAP_CHUNK=$c timeout 600 python bench.py --n $n --steps 5 --warmup 3 --no-cpu-baseline --no-bnb > gpurun_out/ch_${n}_$c.txt 2>&1
  echo "n=$n chunk=$c $(grep -o '"value": [0-9.]*' gpurun_out/ch_${n}_$c.txt | head -1) $(grep -o '"lap2": {[^}]*}' gpurun_out/ch_${n}_$c.txt | head -1 | cut -c1-60) $(grep -o '"sm_mhz": [0-9.]*' gpurun_out/ch_${n}_$c.txt)"
done
done

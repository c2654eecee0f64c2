# J1 segment: tai35b-shaped B&B, resumable; the checkpoint lives in profiles/r02/bnb/j1_ckpt/ (it
# travels with the snapshot) and is copied back through gpurun_out/
cd $GRAFT_REPO_ROOT
TAG=${1:-j1d}
B=${2:-3200}
mkdir -p gpurun_out/j1_ckpt
cp profiles/r02/bnb/j1_ckpt/* gpurun_out/j1_ckpt/ 2>/dev/null
R=""; [ -f gpurun_out/j1_ckpt/taib35.ckpt ] && R="--resume"
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "largest_sizes or depth_counters" > gpurun_out/${TAG}_pytest.txt 2>&1; tail -n 2 gpurun_out/${TAG}_pytest.txt
timeout $((B + 900)) python scripts/bnb_run.py --family taib --n 35 --sb 1 --iters 60 --K 1e-4 --warm --batch 8 --ub0 990211 --budget-s $B --chunk 100 --ckpt gpurun_out/j1_ckpt/taib35.ckpt $R --out gpurun_out/${TAG}_taib35.jsonl > gpurun_out/${TAG}_taib35.log 2>&1
tail -n 2 gpurun_out/${TAG}_taib35.log | cut -c1-700

# usage: bash scripts/gpu_final.sh <tag> : smoke + full GPU suite + bench lines at N = 20, 35, 40
cd $GRAFT_REPO_ROOT
TAG=${1:-fin}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
bash scripts/gpu_sizes.sh ${TAG}
tail -n 2 gpurun_out/${TAG}_pytest.txt

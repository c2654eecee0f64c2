# usage: bash scripts/gpu_full.sh <tag> : smoke + full GPU suite + round profile (bench, launch list, ncu)
cd $GRAFT_REPO_ROOT
TAG=${1:-r}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --timeout 600 > gpurun_out/${TAG}_pytest.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.txt
bash scripts/gpu_round_profile.sh ${TAG}

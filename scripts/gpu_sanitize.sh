cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  if [ $tool = synccheck ]; then extra="--num-cuda-barriers 65536"; fi
  timeout 1200 compute-sanitizer --tool $tool $extra --error-exitcode 9 python scripts/sanitize_one.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_$tool.txt
  tail -n 4 gpurun_out/sanitize_$tool.txt
done

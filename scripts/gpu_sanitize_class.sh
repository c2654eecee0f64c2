cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  extra=""
  if [ $tool = synccheck ]; then extra="--num-cuda-barriers 65536"; fi
  timeout 1500 compute-sanitizer --tool $tool $extra --error-exitcode 9 python scripts/sanitize_class.py > gpurun_out/sanitize_class_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_class_$tool.txt
  tail -n 3 gpurun_out/sanitize_class_$tool.txt
done

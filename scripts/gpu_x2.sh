cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_lap -s 2 -c 1 -o gpurun_out/x2_lap2 python scripts/profile_one.py 30 1 0 4 > gpurun_out/x2_lap2.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_transfer -s 1 -c 1 -o gpurun_out/x2_transfer python scripts/profile_one.py 30 2 0 4 > gpurun_out/x2_transfer.txt 2>&1
tail -2 gpurun_out/x2_lap2.txt gpurun_out/x2_transfer.txt

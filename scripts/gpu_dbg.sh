cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 300 ncu --metrics $M --clock-control none -k regex:k_lap --csv python scripts/profile_one.py 30 2 0 4 > gpurun_out/dbg_nograph.txt 2>&1; echo "rc=$?" >> gpurun_out/dbg_nograph.txt
cd _head
timeout 300 ncu --metrics $M --clock-control none -k regex:k_lap --csv python scripts/profile_one.py 30 2 0 > ../gpurun_out/dbg_head.txt 2>&1; echo "rc=$?" >> ../gpurun_out/dbg_head.txt

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 4 -c 1 -o gpurun_out/full_c2 python scripts/prof_c2.py > gpurun_out/prof_c2.log 2>&1; tail -2 gpurun_out/prof_c2.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 5 -c 1 -o gpurun_out/full_c4 python scripts/prof_c4.py > gpurun_out/prof_c4.log 2>&1; tail -2 gpurun_out/prof_c4.log

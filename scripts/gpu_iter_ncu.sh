cd $GRAFT_REPO_ROOT
bash scripts/gpu_iter.sh
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 4 -c 1 -o gpurun_out/full_c2 python scripts/prof_c2.py > gpurun_out/prof_c2.log 2>&1; tail -1 gpurun_out/prof_c2.log

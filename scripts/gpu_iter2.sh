cd $GRAFT_REPO_ROOT
bash scripts/gpu_iter.sh
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 30 -c 1 -o gpurun_out/full_c4x python scripts/prof_c4x.py > gpurun_out/prof_c4x.log 2>&1; tail -2 gpurun_out/prof_c4x.log

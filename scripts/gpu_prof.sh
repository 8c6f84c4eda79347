cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 1 -c 1 -o gpurun_out/prof_c2 python scripts/prof_replay.py c2 2>&1 | tail -5

cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
./scripts/micro/stream_bench > gpurun_out/micro.txt 2>&1; cat gpurun_out/micro.txt
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 5 -c 1 -o gpurun_out/full_c4 python scripts/prof_c4.py > gpurun_out/prof_c4.log 2>&1; tail -3 gpurun_out/prof_c4.log
ls -la gpurun_out

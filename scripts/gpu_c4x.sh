cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python bench.py --workload c4x --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c4x.json 2> gpurun_out/bench_c4x.err; tail -1 gpurun_out/bench_c4x.json; tail -3 gpurun_out/bench_c4x.err

# round-end measurement: parity tests, smoke, bench lines (c5 default with cpu_baseline; c4,
# c4x, c2), launch lists and ncu --set full captures of k_replay (c5 bench step, c4, c4x)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3 > gpurun_out/final_tests.log; cat gpurun_out/final_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/final_c5.json 2> gpurun_out/final_c5.err; tail -1 gpurun_out/final_c5.json
timeout 900 python bench.py --workload c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_c4.json 2> gpurun_out/final_c4.err; tail -1 gpurun_out/final_c4.json
timeout 1500 python bench.py --workload c4x --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_c4x.json 2> gpurun_out/final_c4x.err; tail -1 gpurun_out/final_c4x.json
timeout 900 python bench.py --workload c2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/final_c2.json 2> gpurun_out/final_c2.err; tail -1 gpurun_out/final_c2.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 3 -c 1 -o gpurun_out/full_c5 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4.csv python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 5 -c 1 -o gpurun_out/full_c4 python scripts/prof_c4.py > gpurun_out/prof_c4.log 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 30 -c 1 -o gpurun_out/full_c4x python scripts/prof_c4x.py > gpurun_out/prof_c4x.log 2>&1
ls -la gpurun_out | head -40

cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 900 python bench.py --steps 5 --warmup 3 --cpu-seconds 5 2>&1 | tail -2
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -2

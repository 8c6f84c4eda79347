set -x
cd $GRAFT_REPO_ROOT
timeout 900 python bench.py --steps 5 --warmup 3 2>&1 | tail -5
timeout 900 python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -5

cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
VARS="t4096" WLS="c4x c4" bash scripts/gpu_btile.sh

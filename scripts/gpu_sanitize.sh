cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for t in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize.py > gpurun_out/san_$t.log 2>&1
  echo "== $t"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|hazard|ok" gpurun_out/san_$t.log | head -12
done

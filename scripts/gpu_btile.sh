cd $GRAFT_REPO_ROOT
for v in ${VARS:-t1024 t2048}; do
  cp scratch_so/libsae_$v.so paper_2605_18825_b200/libsae.so
  for w in ${WLS:-c4x c4}; do
    timeout 1500 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bt_$w.json 2> gpurun_out/bt_$w.err
    python -c "
import json; d=json.loads(open('gpurun_out/bt_$w.json').read().strip().splitlines()[-1]); p=d['score_select_phase']
print('$v $w', round(d['value'],1), 'frac', round(d['roofline']['frac'],4), 'scan_us', round(p['scan_ns_per_pass']/1e3,2), 'GBps', round(p.get('streamed_GBps',0)))" || tail -3 gpurun_out/bt_$w.err
  done
done
cp scratch_so/libsae_t2048.so paper_2605_18825_b200/libsae.so

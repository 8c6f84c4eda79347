# threshold-policy sweep: CFGS="trim_at,trim_to:slack ..." over workloads WL
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for cfg in ${CFGS:-8,4:32}; do t=${cfg%%:*}; sl=${cfg##*:}; for w in ${WL:-c4 c5 c2}; do
  SAE_TRIM=$t SAE_SLACK=$sl timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sw_$w.json 2> gpurun_out/sw_$w.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/sw_$w.json').read().strip().splitlines()[-1])
p=d.get('score_select_phase')
print('cfg $cfg $w', round(d['value'],1), 'frac', round(d['roofline']['frac'],4), 'passes', round(p['passes_per_request'],3), 'cands', round(p['cands_per_pass']), 'raw', round(p['raw_cands_per_pass']), 'scan_us', round(p['scan_ns_per_pass']/1e3,1), 'ph', p['phase_ms_per_step'])" || tail -5 gpurun_out/sw_$w.err
done; done

# build-measure iteration: GPU parity tests, then the three bench workloads
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu ${TESTSEL:-} 2>&1 | tail -15 > gpurun_out/gpu_tests.log; cat gpurun_out/gpu_tests.log
for w in ${WL:-c4 c5 c2}; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  python -c "
import json,sys; d=json.loads(open('gpurun_out/bench_$w.json').read().strip().splitlines()[-1])
print('$w', round(d['value'],1), d['unit'], 'frac', round(d['roofline']['frac'],4), 'e2e', round(d['e2e']['value'],1), json.dumps(d.get('score_select_phase')))" || tail -5 gpurun_out/bench_$w.err
done

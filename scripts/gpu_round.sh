#!/usr/bin/env bash
# One documented entry point for the GPU-box work of a round (run under gpurun):
#
#   gpurun --timeout 1800 -- 'bash scripts/gpu_round.sh <step> [<step> ...]'
#
# Steps (each writes under gpurun_out/, which gpurun copies back):
#   info        host cores / GPU / clocks of the box
#   tests       pytest -m gpu (parity through the C ABI) + smoke()
#   bench       default bench line (C5, cpu_baseline) -> gpurun_out/bench_c5.json
#   bench_all   bench lines of c2, c3, c4, c4x, predictor (no cpu baseline) + the reference arm
#   ncu_c5      launch list + ncu --set full --import-source on of the timed C5 k_replay
#   ncu_c4      launch list + full capture of a C4 200-request k_replay launch
#   ncu_c4x     full capture of a C4x 200-request k_replay launch
#   ncu_select  full capture of one 10-pass sae_select launch on the full 2^24-block pool
#   sanitize    compute-sanitizer memcheck / racecheck / synccheck on small replays (closed on
#               the GPU pool since round 2: it left GPUs needing a reset)
#   sass        cuobjdump -sass of libsae.so -> per-kernel counts of the TMA / mbarrier / tcgen05
#               mnemonics (gpurun_out/sass_summary.txt)
#   ablation    scripts/ablation.py on the balanced, multi-turn- and single-turn-dominant mixes
#   sweep       C5 bench lines over the select's SAE_SLACK / SAE_TRIM knobs
#   variants    C5 bench lines of the v256 / v256g replay variants over SAE_TRIM
#   characterize  scripts/characterize.py (unbounded-cache reuse structure of the three mixes)
# Summaries worth keeping are copied into profiles/ by hand (scripts/profile_summary.py).
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
O=gpurun_out
# gpurun copies gpurun_out/ back only when it stays under 64 MiB: each ncu report is reduced
# on the box to its raw-metrics CSV, the hot-source-lines text and a gzipped source page.
shrink_rep() {   # $1 = report path without .ncu-rep
  ncu -i $1.ncu-rep --page raw --csv > $1_raw.csv 2>/dev/null
  python scripts/ncu_hot_lines.py $1.ncu-rep 60 > $1_hot.txt 2>&1
  ncu -i $1.ncu-rep --page source --csv --print-source cuda,sass 2>/dev/null | gzip -9 > $1_source.csv.gz
  [ -n "${KEEP_REP:-}" ] || rm -f $1.ncu-rep
  ls -la $1_*
}
for step in "$@"; do
  echo "== $step"
  case "$step" in
    info)
      (nproc; lscpu | grep -E 'Model name|Socket|Thread|Core' ; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv) > $O/box_info.txt 2>&1
      cat $O/box_info.txt ;;
    tests)
      timeout 1500 python -m pytest tests -q -m gpu -x 2>&1 | tail -15 | tee $O/gpu_tests.log
      timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2 | tee $O/smoke.log ;;
    bench)
      timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err; tail -1 $O/bench_c5.json ;;
    bench_all)
      for w in c2 c3 c4 c4x predictor; do
        timeout 1200 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline --no-predictor --no-score-select > $O/bench_$w.json 2> $O/bench_$w.err
        tail -c 400 $O/bench_$w.json
      done
      timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
      tail -c 400 $O/bench_reference.json ;;
    ncu_c5)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5.csv \
        python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-score-select --no-predictor > /dev/null 2>&1
      timeout 1200 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 3 -c 1 -f -o $O/full_c5 \
        python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-score-select --no-predictor > /dev/null 2>&1
      shrink_rep $O/full_c5 ;;
    ncu_c4)
      timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
        python bench.py --workload c4 --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
      timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 5 -c 1 -f -o $O/full_c4 \
        python scripts/prof_c4.py > $O/prof_c4.log 2>&1
      shrink_rep $O/full_c4 ;;
    ncu_c4x)
      timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_replay -s 30 -c 1 -f -o $O/full_c4x \
        python scripts/prof_c4x.py > $O/prof_c4x.log 2>&1
      shrink_rep $O/full_c4x ;;
    ncu_select)
      timeout 1500 ncu --set full --import-source on --clock-control none -k regex:k_select -s 2 -c 1 -f -o $O/full_select \
        python scripts/prof_select.py > $O/prof_select.log 2>&1
      shrink_rep $O/full_select ;;
    sanitize)
      for tool in memcheck racecheck synccheck; do
        timeout 900 compute-sanitizer --tool $tool python scripts/sanitize.py > $O/sanitize_$tool.log 2>&1
        tail -3 $O/sanitize_$tool.log
      done ;;
    sass)
      cuobjdump -sass paper_2605_18825_b200/libsae.so > /tmp/sass_all.txt 2>&1
      python scripts/sass_summary.py /tmp/sass_all.txt > $O/sass_summary.txt
      cat $O/sass_summary.txt | head -30 ;;
    ablation)
      for w in c5 c2 c4s; do
        timeout 900 python scripts/ablation.py --workload $w --out $O/ablation_$w > $O/ablation_$w.log 2>&1
        tail -14 $O/ablation_$w.log
      done ;;
    sweep)
      for sl in 16 8 4; do for tr in 8,4 4,2 3,2; do
        SAE_SLACK=$sl SAE_TRIM=$tr timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $O/sweep_${sl}_${tr}.json 2>/dev/null
        python -c "import json,sys; d=json.loads(open('$O/sweep_${sl}_${tr}.json').read().strip().splitlines()[-1]); print('slack $sl trim $tr', round(d['value']), d['score_select_phase']['passes_per_request'], round(d['score_select_phase']['cands_per_pass']))"
      done; done ;;
    variants)
      for v in 256 257; do for tr in 8,4 4,2 3,2; do
        SAE_VARIANT=$v SAE_TRIM=$tr timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-score-select > $O/var_${v}_${tr}.json 2>/dev/null
        python -c "import json,sys; d=json.loads(open('$O/var_${v}_${tr}.json').read().strip().splitlines()[-1]); print('variant $v trim $tr', round(d['value']), d['score_select_phase']['passes_per_request'], round(d['score_select_phase']['cands_per_pass']), d['score_select_phase']['phase_ms_per_step'])"
      done; done ;;
    characterize)
      timeout 900 python scripts/characterize.py $O/characterize 200000 > $O/characterize.log 2>&1; tail -40 $O/characterize.log ;;
    *) echo "unknown step $step" ;;
  esac
done

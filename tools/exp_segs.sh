# A/B of the planner's trailing-segment trim (TQD_PLAN_SEG_KEEP, TQD_PLAN_SEG_MIN_GATES)
for cfg in "3 6" "3 8" "2 8" "2 10"; do
  set -- $cfg
  TQD_PLAN_SEG_KEEP=$1 TQD_PLAN_SEG_MIN_GATES=$2 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp_seg_$1_$2.log 2>&1
  echo "== keep $1 min_gates $2"; python tools/bench_brief.py gpurun_out/exp_seg_$1_$2.log | sed -n 1,3p
done

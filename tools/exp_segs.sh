# A/B of the planner's trailing-segment trim (TQD_PLAN_SEG_MIN_GATES)
for mg in 0 4 6; do
  TQD_PLAN_SEG_MIN_GATES=$mg python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/exp_segmin$mg.log 2>&1
  echo "== min_gates $mg"; python tools/bench_brief.py gpurun_out/exp_segmin$mg.log | sed -n 1,3p
done

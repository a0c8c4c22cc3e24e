# A/B of sweep-kernel variant bits (TQD_EXPERIMENT_FLAGS), full bench and data-movement skeleton
mkdir -p gpurun_out
for f in ${FLAGS:-0 1}; do
  TQD_EXPERIMENT_FLAGS=$f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/flags_$f.log 2>&1
  echo "flags=$f"; python tools/bench_brief.py gpurun_out/flags_$f.log | sed -n 1,3p
  TQD_EXPERIMENT_SKIP_OPS=1 TQD_EXPERIMENT_FLAGS=$f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/flags_skel_$f.log 2>&1
  echo "skeleton flags=$f"; python tools/bench_brief.py gpurun_out/flags_skel_$f.log | sed -n 2,3p
done

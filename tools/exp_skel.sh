# data-movement skeleton: sweeps with all gate ops removed (TQD_EXPERIMENT_SKIP_OPS), varying pinned low bits and tile size
mkdir -p gpurun_out
for c in 4 5; do for k in 12 10; do
  TQD_EXPERIMENT_SKIP_OPS=1 TQD_C_LOW=$c python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --tile $k > gpurun_out/skel_c${c}_k${k}.log 2>&1
  echo "C=$c k=$k"; python tools/bench_brief.py gpurun_out/skel_c${c}_k${k}.log | sed -n 2,3p
done; done
for c in 4 5; do
  TQD_C_LOW=$c python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/full_c${c}.log 2>&1
  echo "full C=$c"; python tools/bench_brief.py gpurun_out/full_c${c}.log | sed -n 1,3p
done

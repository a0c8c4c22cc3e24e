# occupancy experiment: R=3 register bits, 256-thread CTAs (k=11), 4 CTAs/SM
mkdir -p gpurun_out
TQD_NVCC_EXTRA="-DTQD_SWEEP_R=3 -DTQD_LB_THREADS=256 -DTQD_LB_MINB_F32_BWD=4 -DTQD_LB_MINB_F32_FWD=4" \
  python -c "import paper_2511_19291_b200.build as b; b.build(force=True, verbose=True)" 2>&1 | grep -A2 "sweep_kernelIf" | grep -E "registers|stack"
for k in 11 12; do
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --tile $k > gpurun_out/r3k$k.log 2>&1
echo "R=3 k=$k"; python tools/bench_brief.py gpurun_out/r3k$k.log | sed -n 1,3p
done

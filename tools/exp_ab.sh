# A/B timing of build-time kernel knobs: tools/exp_ab.sh "<nvcc extra A>" "<nvcc extra B>"
# (each variant rebuilt in place, bench run twice, alternating; brief lines printed)
mkdir -p gpurun_out
for rep in 1 2; do
  for v in A B; do
    if [ $v = A ]; then X="$1"; else X="$2"; fi
    TQD_NVCC_EXTRA="$X" python -c "import paper_2511_19291_b200.build as b; b.build(force=True)" > /dev/null 2>&1
    python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ab_${v}_$rep.log 2>&1
    echo "variant $v ($X) rep $rep"; python tools/bench_brief.py gpurun_out/ab_${v}_$rep.log | head -3
  done
done
python -c "import paper_2511_19291_b200.build as b; b.build(force=True)" > /dev/null 2>&1

# launch-bound / tile-size experiments (each rebuilds the library on the box)
mkdir -p gpurun_out
run() { # name extra-nvcc bench-args
  TQD_NVCC_EXTRA="$2" python -c "import paper_2511_19291_b200.build as b; b.build(force=True)" > /dev/null 2>&1
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e $3 > gpurun_out/lb_$1.log 2>&1
  echo "== $1"; python tools/bench_brief.py gpurun_out/lb_$1.log | sed -n 1,3p
}
run k11 "" "--tile 11"
run fwd2 "-DTQD_LB_MINB_F32_FWD=2" ""
run bwd1 "-DTQD_LB_MINB_F32_BWD=1" ""
run base "" ""

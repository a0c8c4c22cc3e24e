# A/B of TMA-staged sweeps (TQD_SWEEP_TMA bit 0 = forward, bit 1 = adjoint)
run() { name=$1; shift; env "$@" python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e $BARGS > gpurun_out/exp_$name.log 2>&1; echo "== $name"; python tools/bench_brief.py gpurun_out/exp_$name.log | sed -n 2,3p; }
TQD_SWEEP_TMA=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_emulated_world.py -m gpu -q -p no:cacheprovider -x -k "sweep_path or adjoint_random or hea_sweep or diagonal_blocks or world_adjoint or random_22q or cfg1" 2>&1 | tail -2
run tma0 TQD_SWEEP_TMA=0
run tma2 TQD_SWEEP_TMA=2
run skel_tma2 TQD_SWEEP_TMA=2 TQD_EXPERIMENT_SKIP_OPS=1
BARGS="--tile 11" run tma2_k11 TQD_SWEEP_TMA=2
BARGS="--tile 11" run skel_tma2_k11 TQD_SWEEP_TMA=2 TQD_EXPERIMENT_SKIP_OPS=1

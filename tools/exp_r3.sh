set -x
mkdir -p gpurun_out
TQD_EXPERIMENT_SMEM_KB=110 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r4_110.log 2>&1
python tools/bench_brief.py gpurun_out/r4_110.log | head -3
TQD_NVCC_EXTRA="-DTQD_SWEEP_R=3" python -c "import paper_2511_19291_b200.build as b; b.build(force=True, verbose=True)" 2>&1 | grep -A2 "sweep_kernelIf" | grep -E "registers|stack"
TQD_EXPERIMENT_SMEM_KB=110 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r3_110.log 2>&1
python tools/bench_brief.py gpurun_out/r3_110.log | head -3
TQD_EXPERIMENT_SMEM_KB=110 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "adjoint or sweep" 2>&1 | tail -2

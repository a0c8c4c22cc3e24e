# Round measurement set: GPU tests, smoke, bench (+cpu baseline, e2e), reference arm,
# ncu launch list of the bench command, ncu --set full of one fwd + one adjoint sweep.
TAG=${1:-cur}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
python bench.py > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
python tools/bench_brief.py gpurun_out/bench_$TAG.log
python bench.py --impl reference > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/bench_ref_$TAG.log | cut -c1-300
python tools/bench_configs.py --ksweep 9,10,11,12 > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; echo "configs rc=$?"
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_short_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
bash tools/ncu_capture.sh $TAG; echo "ncu full rc=$?"

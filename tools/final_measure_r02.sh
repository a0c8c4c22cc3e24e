# Round-2 measurement set (one GPU): tests, smoke, bench (headline + forward + e2e + cpu
# baseline), reference arm, configs 2 / 4 through bench.py, per-config table, ncu launch
# list of the bench command, ncu --set full of one forward + one adjoint sweep.
TAG=${1:-r02}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/gpu_tests_$TAG.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/gpu_tests_$TAG.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.log 2>&1; echo "bench rc=$?"
python tools/bench_brief.py gpurun_out/bench_$TAG.log
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "ref rc=$?"
python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg2_$TAG.log 2>&1; echo "cfg2 rc=$?"
python tools/bench_brief.py gpurun_out/bench_cfg2_$TAG.log | head -3
python bench.py --config 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_$TAG.log 2>&1; echo "cfg4 rc=$?"
python tools/bench_brief.py gpurun_out/bench_cfg4_$TAG.log | head -3
python tools/bench_configs.py --cases cfg1,cfg2,cfg5_8,cfg5_8_sweep > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err; echo "configs rc=$?"
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_short_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv --log-file gpurun_out/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch list rc=$?"
bash tools/ncu_capture.sh $TAG; echo "ncu full rc=$?"

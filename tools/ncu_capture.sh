#!/bin/bash
# ncu --set full capture of one forward and one adjoint sweep launch of the
# 30q bench workload (tools/prof_sweep.py); run on the GPU box after the same
# command exited 0 without ncu.  usage: tools/ncu_capture.sh TAG
set -e
TAG=${1:-cur}
mkdir -p gpurun_out
python tools/prof_sweep.py > gpurun_out/prof_plain.log 2>&1
# launches: 66 forward sweeps, then 66 adjoint sweeps (see prof_plain.log): adjoint #14, forward #11
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel --launch-skip 79 -c 1 \
    -o gpurun_out/prof_bwd_$TAG -f python tools/prof_sweep.py > gpurun_out/ncu_bwd.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel --launch-skip 10 -c 1 \
    -o gpurun_out/prof_fwd_$TAG -f python tools/prof_sweep.py > gpurun_out/ncu_fwd.log 2>&1

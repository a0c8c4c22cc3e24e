#!/bin/bash
# Build a kernel-experiment variant of libtqd.so: the float sweep kernels recompiled
# with extra nvcc flags, linked with the default build's other objects.
#   tools/build_variant.sh NAME "-DTQD_LB_MINB_TP_FWD=3 ..."
# -> paper_2511_19291_b200/variants/libtqd_NAME.so (load with TQD_LIB=<path>)
set -e
NAME=$1; FLAGS=$2
ROOT=$(cd "$(dirname "$0")/.." && pwd)
PKG=$ROOT/paper_2511_19291_b200
OBJ=$PKG/build; OUT=$PKG/variants/$NAME; mkdir -p $OUT
NCCL=$(python -c "import nvidia.nccl as m, os; print(list(m.__path__)[0])")
COMMON="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC,-O3 -I$NCCL/include $FLAGS"
for f in sweep_f32_fwd sweep_f32_bwd; do
  (cd $PKG/csrc && nvcc $COMMON -c $f.cu -o $OUT/$f.o) &
done
wait
objs=""
for f in kernels sweep_f64_fwd sweep_f64_bwd dense_tc plan comm abi; do objs="$objs $OBJ/$f.o"; done
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $PKG/variants/libtqd_$NAME.so $objs $OUT/sweep_f32_fwd.o $OUT/sweep_f32_bwd.o \
  -L$NCCL/lib -l:$(basename $(ls $NCCL/lib/libnccl.so* | head -1)) -Xlinker -rpath,$NCCL/lib
echo $PKG/variants/libtqd_$NAME.so

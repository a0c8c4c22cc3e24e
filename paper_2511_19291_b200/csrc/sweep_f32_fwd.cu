// sweep_f32_fwd.cu -- instantiation of the fused sweep kernel (float, adjoint=false).
#include "sweep.cuh"
TQD_INSTANTIATE_SWEEP(float, false, f32_fwd)

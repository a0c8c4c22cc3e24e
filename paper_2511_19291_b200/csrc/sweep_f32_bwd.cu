// sweep_f32_bwd.cu -- instantiation of the fused sweep kernel (float, adjoint=true).
#include "sweep.cuh"
TQD_INSTANTIATE_SWEEP(float, true, f32_bwd)

// sweep_f64_bwd.cu -- instantiation of the fused sweep kernel (double, adjoint=true).
#include "sweep.cuh"
TQD_INSTANTIATE_SWEEP(double, true, f64_bwd)

// sweep_f64_fwd.cu -- instantiation of the fused sweep kernel (double, adjoint=false).
#include "sweep.cuh"
TQD_INSTANTIATE_SWEEP(double, false, f64_fwd)

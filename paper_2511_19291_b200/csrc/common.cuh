// common.cuh -- complex helpers shared by the sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tqd {

template <typename Real> struct CT;
template <> struct CT<float> { typedef float2 C; };
template <> struct CT<double> { typedef double2 C; };

template <typename C> __device__ __forceinline__ C mk(decltype(C::x) x, decltype(C::x) y) {
    C r;
    r.x = x;
    r.y = y;
    return r;
}
template <typename C> __device__ __forceinline__ C cmul(C a, C b) {
    return mk<C>(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// a*x + b*y (complex)
template <typename C> __device__ __forceinline__ C cmul2(C a, C x, C b, C y) {
    return mk<C>(a.x * x.x - a.y * x.y + b.x * y.x - b.y * y.y, a.x * x.y + a.y * x.x + b.x * y.y + b.y * y.x);
}
// Re(conj(a) b), Im(conj(a) b)
template <typename C> __device__ __forceinline__ decltype(C::x) re_cj(C a, C b) { return a.x * b.x + a.y * b.y; }
template <typename C> __device__ __forceinline__ decltype(C::x) im_cj(C a, C b) { return a.x * b.y - a.y * b.x; }

template <typename C> __device__ __forceinline__ C ldc(const double *m, int i) {
    return mk<C>((decltype(C::x))m[2 * i], (decltype(C::x))m[2 * i + 1]);
}

template <typename Real> __device__ __forceinline__ Real warp_sum(Real v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// block-wide sum; the result is valid in thread 0.  red: >= 32 slots of shared memory.
template <typename Real> __device__ __forceinline__ Real block_sum(Real v, Real *red) {
    v = warp_sum(v);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    Real t = 0;
    if (threadIdx.x < 32) {
        t = (threadIdx.x < (blockDim.x >> 5)) ? red[threadIdx.x] : (Real)0;
        t = warp_sum(t);
    }
    return t;
}

}  // namespace tqd

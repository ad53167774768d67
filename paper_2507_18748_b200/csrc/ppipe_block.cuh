// Block-wide scans for the kernels of this library (warp shuffles + one shared
// array of per-warp totals). Hand-written replacements of library block scans.
#pragma once
#include <cuda_runtime.h>

namespace ppipe {

// Inclusive scan of v over the CTA (blockDim.x == NT, a multiple of 32) under the
// associative op with identity id; *total receives the CTA-wide result. sh must hold
// NT / 32 elements. Contains __syncthreads(): every thread of the CTA must call it.
template <int NT, class T, class Op>
__device__ __forceinline__ T block_inclusive_scan(T v, T id, Op op, T* total, T* sh) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x = op(y, x);
  }
  if (lane == 31) sh[warp] = x;
  __syncthreads();
  T before = id, all = id;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    if (w < warp) before = op(before, sh[w]);
    all = op(all, sh[w]);
  }
  __syncthreads();
  *total = all;
  return op(before, x);
}

// Exclusive form: the op-combination of every earlier thread's value (id for thread 0).
template <int NT, class T, class Op>
__device__ __forceinline__ T block_exclusive_scan(T v, T id, Op op, T* sh) {
  constexpr int NW = NT / 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const T y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= d) x = op(y, x);
  }
  if (lane == 31) sh[warp] = x;
  T ex = __shfl_up_sync(0xffffffffu, x, 1);
  if (lane == 0) ex = id;
  __syncthreads();
  T before = id;
#pragma unroll
  for (int w = 0; w < NW; ++w)
    if (w < warp) before = op(before, sh[w]);
  __syncthreads();
  return op(before, ex);
}

struct OpSum {
  template <class T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a + b; }
};
struct OpMax {
  template <class T>
  __device__ __forceinline__ T operator()(T a, T b) const { return a > b ? a : b; }
};

}  // namespace ppipe

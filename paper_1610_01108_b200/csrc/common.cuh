// Shared helpers for the sm_100a decoder kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <stdexcept>
#include <string>

namespace amun {

struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string &m) : std::runtime_error(m), code(c) {}
};

#define AMUN_CUDA(call)                                                                     \
  do {                                                                                      \
    cudaError_t e_ = (call);                                                                \
    if (e_ != cudaSuccess) {                                                                \
      int code_ = (e_ == cudaErrorMemoryAllocation) ? 3 : 2;                                \
      throw ::amun::Error(code_, std::string(#call) + ": " + cudaGetErrorString(e_) + " at " + \
                                     __FILE__ + ":" + std::to_string(__LINE__));           \
    }                                                                                       \
  } while (0)

#define AMUN_CHECK_LAUNCH() AMUN_CUDA(cudaGetLastError())

__host__ __device__ inline int ceil_div(int a, int b) { return (a + b - 1) / b; }

// Accurate transcendentals (SURVEY §7 hard part (f)): full-precision expf /
// tanhf, never the .approx forms.
__device__ __forceinline__ float sigmoid_acc(float x) { return 1.0f / (1.0f + expf(-x)); }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Candidate ordering used everywhere in selection: value desc, then token
// asc, then parent asc (search.py:75-91).  `better(a, b)` is a strict total
// order on distinct (tok, par) pairs.
struct Key {
  double v;
  int tok;
  int par;
};
__device__ __forceinline__ bool key_better(double va, int ta, int pa, double vb, int tb, int pb) {
  if (va != vb) return va > vb;
  if (ta != tb) return ta < tb;
  return pa < pb;
}
__device__ __forceinline__ Key warp_best(Key k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Key q;
    q.v = __shfl_xor_sync(0xffffffffu, k.v, o);
    q.tok = __shfl_xor_sync(0xffffffffu, k.tok, o);
    q.par = __shfl_xor_sync(0xffffffffu, k.par, o);
    if (key_better(q.v, q.tok, q.par, k.v, k.tok, k.par)) k = q;
  }
  return k;
}

constexpr int kMaxRowCand = 16;

// 3xTF32 operand split: hi = tf32-exact (low 13 mantissa bits cleared),
// lo = x - hi (exact).  Writes both when `hi` is non-null.
__device__ __forceinline__ void store_split(float *hi, float *lo, long long off, float x) {
  if (hi) {
    const float h = __uint_as_float(__float_as_uint(x) & 0xFFFFE000u);
    hi[off] = h;
    lo[off] = x - h;
  }
}  // fused logit epilogue keeps <= 16 per row/tile

}  // namespace amun

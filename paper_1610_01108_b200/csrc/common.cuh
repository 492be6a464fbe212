// Shared helpers for the sm_100a decoder kernels.
#pragma once

#include <cuda_fp16.h>
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

// CTAs of the most recent tensor-core launch on this host thread (profiling:
// the decode driver attributes them to the launch's kernel class)
inline int &last_launch_ctas() {
  static thread_local int n = 0;
  return n;
}

// In-situ CTA-time accounting (bench.py roofline in the timed multi-lane
// graph-replay mode): a kernel whose args carry kt != nullptr adds, per CTA,
// (globaltimer at exit - at entry) to kt[0] and 1 to kt[1].  The decode
// driver points kt at its kernel class's slot (ktime_ptr(), set around every
// launch by Ctx::run); nullptr (the default) costs one predicate per CTA.
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct CtaClock {
  unsigned long long *kt;
  unsigned long long t0;
  __device__ __forceinline__ explicit CtaClock(unsigned long long *p) : kt(p), t0(p && threadIdx.x == 0 ? gtimer() : 0ull) {}
  // thread 0, after the CTA's last barrier
  __device__ __forceinline__ void done() const {
    if (kt && threadIdx.x == 0) {
      atomicAdd(kt, gtimer() - t0);
      atomicAdd(kt + 1, 1ull);
    }
  }
};
inline unsigned long long *&ktime_ptr() {
  static thread_local unsigned long long *p = nullptr;
  return p;
}

// Accurate transcendentals (SURVEY §7 hard part (f)): full-precision expf /
// tanhf, never the .approx forms.
// acc += w * h on four lanes as two packed FFMA2 (fma.rn.f32x2: the same
// correctly rounded fma per element as four scalar fmaf, half the issue slots)
__device__ __forceinline__ void fma4x2(float w, const float4 &h, float4 &acc) {
  const float2 ww = make_float2(w, w);
  const float2 lo = __ffma2_rn(ww, make_float2(h.x, h.y), make_float2(acc.x, acc.y));
  const float2 hi = __ffma2_rn(ww, make_float2(h.z, h.w), make_float2(acc.z, acc.w));
  acc = make_float4(lo.x, lo.y, hi.x, hi.y);
}

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

// 3xFP16 operand split for the tensor-core GEMMs (kind::f16, fp32
// accumulate): activations are scaled by 2^kXShift (exact), then
// hi = fp16(x'), lo = fp16(x' - hi) (x' - hi is exact in fp32), so hi + lo
// carries ~22 significant bits, like the 3xTF32 split, at twice the MMA rate
// and half the bytes.  The scale keeps lo out of the fp16 subnormal range for
// |x| >= 2^-13; decoder activations are bounded by max(1, max|E_trg|) and the
// model loader only enables the tensor-core path when that is <= 2^(15 -
// kXShift).  The GEMM epilogues multiply the accumulator by
// 2^-(kXShift + weight shift).
constexpr int kXShift = 10;
constexpr float kXScale = 1024.f;
__device__ __forceinline__ void split_h(float x, __half &h, __half &l) {
  const float xs = x * kXScale;
  h = __float2half_rn(xs);
  l = __float2half_rn(xs - __half2float(h));
}
__device__ __forceinline__ void store_split(__half *hi, __half *lo, long long off, float x) {
  if (hi) {
    __half h, l;
    split_h(x, h, l);
    hi[off] = h;
    lo[off] = l;
  }
}  // fused logit epilogue keeps <= 16 per row/tile

}  // namespace amun

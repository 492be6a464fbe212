// FP32 CUDA-core GEMM with fused epilogues (the exact-FP32 baseline path and
// the path for shapes the tensor-core kernel does not take: tiny test
// models, the encoder recurrence at small batch, the hooks).
//
//   C[M, N] = A[M, K] * B[K, N]     (B row-major, N contiguous)
//
// A may be given as two row-major segments concatenated along K
// ([a0 | a1], e.g. [y ; c ; s] and s' for the deep output), and segment 0 may
// be row-gathered through an index array (embedding lookup fused into the
// GEMM A-load, nnet.py:113 / :155).  blockIdx.z selects one of several
// independent problems (the two encoder directions) via element strides.
#pragma once

#include "common.cuh"

namespace amun {

struct GemmArgs {
  int M, N;
  const float *a0;
  int lda0, k0;
  const int *rows0;  // optional row gather for segment 0
  const float *a1;
  int lda1, k1;
  const float *B;
  int ldb;
  int n_split, k_limit;        // tiles with n0 >= n_split only use K <= k_limit
  long long a_zs, b_zs;        // per-problem element strides of a0 and B
  int splits, kchunk;          // split-K: blockIdx.z = problem * splits + split
};

constexpr int kBM = 64, kBN = 128, kBK = 16, kThreads = 256;
constexpr int kApad = 4;
constexpr int kSmemFloats =
    (2 * kBK * (kBM + kApad) + 2 * kBK * kBN) > (kBM * (kBN + 1)) ? (2 * kBK * (kBM + kApad) + 2 * kBK * kBN)
                                                                   : (kBM * (kBN + 1));

// Elementwise epilogue interface: operator()(m, n, acc, z) for m < M, n < N.
// Tile epilogues (kTile == true) instead get the full BM x BN tile staged in
// shared memory (row stride kBN + 1) and run with all 256 threads.

template <class Epi>
__global__ void __launch_bounds__(kThreads) gemm_simt_kernel(GemmArgs g, Epi epi) {
  __shared__ __align__(16) float smem[kSmemFloats];
  float *As = smem;                               // [2][BK][BM + pad]
  float *Bs = smem + 2 * kBK * (kBM + kApad);     // [2][BK][BN]
  const int tid = threadIdx.x;
  const int z = blockIdx.z;
  const int zp = z / g.splits, zs = z % g.splits;
  const float *a0 = g.a0 + zp * g.a_zs;
  const float *Bp = g.B + zp * g.b_zs;
  const int m0 = blockIdx.y * kBM, n0 = blockIdx.x * kBN;
  int K = g.k0 + g.k1;
  if (n0 >= g.n_split && g.k_limit < K) K = g.k_limit;
  const int kbeg = zs * g.kchunk;
  const int kend = min(K, kbeg + g.kchunk);
  const int nk = kend > kbeg ? ceil_div(kend - kbeg, kBK) : 0;

  // Per-thread A rows (4 rows, fixed over k): pointer bases for segment 0/1.
  const float *arow0[4];
  const float *arow1[4];
  bool arow_ok[4];
  const int a_kk = tid % kBK;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int r = tid / kBK + i * (kThreads / kBK);
    int m = m0 + r;
    arow_ok[i] = m < g.M;
    int src = arow_ok[i] ? (g.rows0 ? g.rows0[m] : m) : 0;
    arow0[i] = a0 + (long long)src * g.lda0;
    arow1[i] = g.a1 ? g.a1 + (long long)(arow_ok[i] ? m : 0) * g.lda1 : nullptr;
  }
  const int b_n = tid % kBN;
  const bool b_ok = (n0 + b_n) < g.N;

  float ra[4], rb[8];
  auto load = [&](int kt) {
    const int kbase = kbeg + kt * kBK;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int k = kbase + a_kk;
      float v = 0.f;
      if (arow_ok[i] && k < kend) v = (k < g.k0) ? arow0[i][k] : arow1[i][k - g.k0];
      ra[i] = v;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      int k = kbase + tid / kBN + i * (kThreads / kBN);
      rb[i] = (b_ok && k < kend) ? Bp[(long long)k * g.ldb + n0 + b_n] : 0.f;
    }
  };
  auto store = [&](int buf) {
    float *as = As + buf * kBK * (kBM + kApad);
    float *bs = Bs + buf * kBK * kBN;
#pragma unroll
    for (int i = 0; i < 4; ++i) as[a_kk * (kBM + kApad) + tid / kBK + i * (kThreads / kBK)] = ra[i];
#pragma unroll
    for (int i = 0; i < 8; ++i) bs[(tid / kBN + i * (kThreads / kBN)) * kBN + b_n] = rb[i];
  };

  const int ty = tid / 16, tx = tid % 16;
  float acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.f;

  if (nk > 0) {
    load(0);
    store(0);
  }
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    if (kt + 1 < nk) load(kt + 1);
    const float *as = As + (kt & 1) * kBK * (kBM + kApad);
    const float *bs = Bs + (kt & 1) * kBK * kBN;
#pragma unroll
    for (int kk = 0; kk < kBK; ++kk) {
      float4 a = *reinterpret_cast<const float4 *>(as + kk * (kBM + kApad) + ty * 4);
      float4 b0 = *reinterpret_cast<const float4 *>(bs + kk * kBN + tx * 4);
      float4 b1 = *reinterpret_cast<const float4 *>(bs + kk * kBN + 64 + tx * 4);
      float av[4] = {a.x, a.y, a.z, a.w};
      float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) store((kt + 1) & 1);
    __syncthreads();
  }

  if constexpr (Epi::kTile) {
    float *Ct = smem;  // [BM][BN + 1]; all threads passed the last barrier
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int c = (j < 4) ? tx * 4 + j : 64 + tx * 4 + (j - 4);
        Ct[(ty * 4 + i) * (kBN + 1) + c] = acc[i][j];
      }
    __syncthreads();
    epi.tile(Ct, m0, n0, g.M, g.N, z);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int m = m0 + ty * 4 + i;
      if (m >= g.M) continue;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        int n = n0 + ((j < 4) ? tx * 4 + j : 64 + tx * 4 + (j - 4));
        if (n < g.N) epi(m, n, acc[i][j], z);
      }
    }
  }
}

// Split-K partial store: P[(problem * splits + split)][M][N].
struct EpiPartial {
  static constexpr bool kTile = false;
  float *P;
  int M, N;
  __device__ void operator()(int m, int n, float v, int z) const { P[((long long)z * M + m) * N + n] = v; }
};

// Sum the split partials in a fixed order (deterministic), then apply the
// elementwise epilogue.
template <class Epi>
__global__ void splitk_reduce_kernel(const float *P, int M, int N, int splits, long long total, Epi epi) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const long long mn = (long long)M * N;
  const int p = (int)(i / mn);
  const long long rem = i - p * mn;
  const int m = (int)(rem / N), n = (int)(rem % N);
  const float *src = P + (long long)p * splits * mn + rem;
  float v = 0.f;
  for (int s = 0; s < splits; ++s) v += src[s * mn];
  epi(m, n, v, p);
}

// Split count depends only on (N, K, problems) — never on M — so a row's
// result is independent of how many rows share the launch (batch
// invariance: identical output for any bucket size or GPU count).
inline int choose_splits(int N, int K, int nz) {
  const int tiles_n = ceil_div(N, kBN) * nz;
  int s = ceil_div(128, tiles_n);
  s = std::min(s, std::max(1, K / 128));
  return std::max(1, s);
}

inline int effective_splits(int K, int splits) {
  if (splits <= 1) return 1;
  int kchunk = ceil_div(ceil_div(K, splits), kBK) * kBK;
  return ceil_div(K, kchunk);
}

// Returns the number of kernel launches issued.  `splits` > 1 needs a
// workspace of effective_splits(K, splits) * nz * M * N floats.
template <class Epi>
inline int launch_gemm_simt(GemmArgs g, const Epi &epi, int nz, int splits, cudaStream_t st, float *ws) {
  if (g.M <= 0 || g.N <= 0) return 0;
  const int Kfull = g.k0 + g.k1;
  if (Epi::kTile) splits = 1;
  int kchunk = splits > 1 ? ceil_div(ceil_div(Kfull, splits), kBK) * kBK : Kfull + kBK;
  if (splits > 1) splits = ceil_div(Kfull, kchunk);
  g.splits = splits;
  g.kchunk = kchunk;
  dim3 grid(ceil_div(g.N, kBN), ceil_div(g.M, kBM), nz * splits);
  if (splits == 1) {
    gemm_simt_kernel<Epi><<<grid, kThreads, 0, st>>>(g, epi);
    AMUN_CHECK_LAUNCH();
    return 1;
  }
  if constexpr (!Epi::kTile) {
    gemm_simt_kernel<EpiPartial><<<grid, kThreads, 0, st>>>(g, EpiPartial{ws, g.M, g.N});
    AMUN_CHECK_LAUNCH();
    long long total = (long long)nz * g.M * g.N;
    splitk_reduce_kernel<Epi><<<(unsigned)((total + 255) / 256), 256, 0, st>>>(ws, g.M, g.N, splits, total, epi);
    AMUN_CHECK_LAUNCH();
  }
  return 2;
}

// 4 consecutive columns (n % 4 == 0, 16-byte aligned rows): fp16 split copies
__device__ __forceinline__ void store_split4(__half *hi, __half *lo, long long off, float4 v) {
  if (!hi) return;
  __half h[4], l[4];
  split_h(v.x, h[0], l[0]);
  split_h(v.y, h[1], l[1]);
  split_h(v.z, h[2], l[2]);
  split_h(v.w, h[3], l[3]);
  *reinterpret_cast<uint2 *>(hi + off) = *reinterpret_cast<const uint2 *>(h);
  *reinterpret_cast<uint2 *>(lo + off) = *reinterpret_cast<const uint2 *>(l);
}

// ------------------------------------------------------------------ epilogues

// C = act(acc + bias)    act: 0 identity, 1 tanh
struct EpiStore {
  static constexpr bool kTile = false;
  float *C;
  int ldc;
  const float *bias;
  int act;
  long long c_zs;
  __half *hi = nullptr, *lo = nullptr;  // optional 3xFP16 split copies (row pitch ldh, no z)
  int ldh = 0;
  float *ex2 = nullptr;  // optional e^{2v} (attention query rows: factored tanh, kernels.cu)
  // optional per-row term: v += rowadd[rowtok[m] * ldadd + n] (a table row
  // per token), or rowadd[m * ldadd + n] without rowtok
  const float *rowadd = nullptr;
  const int *rowtok = nullptr;
  int ldadd = 0;
  __device__ void operator()(int m, int n, float v, int z) const {
    if (rowadd) v += rowadd[(long long)(rowtok ? rowtok[m] : m) * ldadd + n];
    if (bias) v += bias[n];
    if (act == 1) v = tanhf(v);
    if (C) C[z * c_zs + (long long)m * ldc + n] = v;
    if (ex2) {
      float y;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v * 2.8853900817779268f));
      ex2[(long long)m * ldc + n] = y;
    }
    store_split(hi, lo, (long long)m * ldh + n, v);
  }
  // two-phase 4-column form for the tensor-core reduction (gemm_sk.cuh):
  // every load of a batch of items is issued before any of its stores
  struct Pre {
    float4 b, r;
  };
  __device__ __forceinline__ Pre load4(int m, int n) const {
    Pre p;
    p.b = bias ? *reinterpret_cast<const float4 *>(bias + n) : make_float4(0.f, 0.f, 0.f, 0.f);
    p.r = rowadd ? *reinterpret_cast<const float4 *>(rowadd + (long long)(rowtok ? rowtok[m] : m) * ldadd + n)
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    return p;
  }
  __device__ __forceinline__ void store4(int m, int n, float4 v, const Pre &p) const {
    v.x += p.r.x;
    v.y += p.r.y;
    v.z += p.r.z;
    v.w += p.r.w;
    v.x += p.b.x;
    v.y += p.b.y;
    v.z += p.b.z;
    v.w += p.b.w;
    if (act == 1) {
      v.x = tanhf(v.x);
      v.y = tanhf(v.y);
      v.z = tanhf(v.z);
      v.w = tanhf(v.w);
    }
    if (C) *reinterpret_cast<float4 *>(C + (long long)m * ldc + n) = v;
    if (ex2) {
      float4 y;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.x) : "f"(v.x * 2.8853900817779268f));
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.y) : "f"(v.y * 2.8853900817779268f));
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.z) : "f"(v.z * 2.8853900817779268f));
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.w) : "f"(v.w * 2.8853900817779268f));
      *reinterpret_cast<float4 *>(ex2 + (long long)m * ldc + n) = y;
    }
    store_split4(hi, lo, (long long)m * ldh + n, v);
  }
};

// Projected-context step, first GEMM: s [W_att_s | U_z | U_r].  Columns
// [0, da) are the attention query (stored with e^{2q}, as EpiStore.ex2);
// columns [da, da + 2dh) the state's gate products s U_{z,r}, which the
// attention kernel completes (kernels.cu attn_sent_kernel, PROJ).
struct EpiQS {
  static constexpr bool kTile = false;
  float *Q, *EQ;  // [M, da]
  float *SU;      // [M, 2dh]
  int da, dh2;
  __device__ void operator()(int m, int n, float v, int) const {
    if (n < da) {
      Q[(long long)m * da + n] = v;
      float y;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(v * 2.8853900817779268f));
      EQ[(long long)m * da + n] = y;
    } else {
      SU[(long long)m * dh2 + n - da] = v;
    }
  }
  struct Pre {};
  __device__ __forceinline__ Pre load4(int, int) const { return Pre{}; }
  __device__ __forceinline__ void store4(int m, int n, float4 v, const Pre &) const {
    if (n < da) {
      *reinterpret_cast<float4 *>(Q + (long long)m * da + n) = v;
      float4 y;
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.x) : "f"(v.x * 2.8853900817779268f));
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.y) : "f"(v.y * 2.8853900817779268f));
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.z) : "f"(v.z * 2.8853900817779268f));
      asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y.w) : "f"(v.w * 2.8853900817779268f));
      *reinterpret_cast<float4 *>(EQ + (long long)m * da + n) = y;
    } else {
      *reinterpret_cast<float4 *>(SU + (long long)m * dh2 + n - da) = v;
    }
  }
};

// Projected-context step with the query folded forward: s' [W_o^s | 0 |
// W_att_s | U_z | U_r].  Columns [0, de): the deep output t = tanh(acc + CO
// row + b_out) (3xFP16 split for the logits); [q0, ...): the NEXT step's
// query, e^{2q} and s' U_{z,r} for this row (the next step's rows read them
// through the select's parent index).
struct EpiDQ {
  static constexpr bool kTile = false;
  const float *CO;  // [M, ldco] context + y term of the deep output (attention epilogue)
  int ldco;
  const float *bias;  // b_out [de]
  __half *hi, *lo;    // t split [M, ldh]
  int ldh, de, q0;
  EpiQS qs;
  __device__ void operator()(int m, int n, float v, int z) const {
    if (n < de) {
      v = tanhf(v + CO[(long long)m * ldco + n] + bias[n]);
      store_split(hi, lo, (long long)m * ldh + n, v);
    } else if (n >= q0) {
      qs(m, n - q0, v, z);
    }
  }
  struct Pre {
    float4 b, r;
  };
  __device__ __forceinline__ Pre load4(int m, int n) const {
    Pre p;
    if (n < de) {
      p.r = *reinterpret_cast<const float4 *>(CO + (long long)m * ldco + n);
      p.b = *reinterpret_cast<const float4 *>(bias + n);
    }
    return p;
  }
  __device__ __forceinline__ void store4(int m, int n, float4 v, const Pre &p) const {
    if (n < de) {
      v.x = tanhf(v.x + p.r.x + p.b.x);
      v.y = tanhf(v.y + p.r.y + p.b.y);
      v.z = tanhf(v.z + p.r.z + p.b.z);
      v.w = tanhf(v.w + p.r.w + p.b.w);
      store_split4(hi, lo, (long long)m * ldh + n, v);
    } else if (n >= q0) {
      qs.store4(m, n - q0, v, EpiQS::Pre{});
    }
  }
};

// A bucket's annotation products in one GEMM over h (split): columns
// [0, da) precomp_att P = h W_att_h (nnet.py:126), then the projected
// annotations HX = h [C_z | C_r | C_h | W_o^c] (row pitch ldx, nx columns used).
struct EpiPH {
  static constexpr bool kTile = false;
  float *P, *HX;
  int da, ldx, nx;
  __device__ void operator()(int m, int n, float v, int) const {
    if (n < da)
      P[(long long)m * da + n] = v;
    else if (n - da < nx)
      HX[(long long)m * ldx + n - da] = v;
  }
  struct Pre {};
  __device__ __forceinline__ Pre load4(int, int) const { return Pre{}; }
  __device__ __forceinline__ void store4(int m, int n, float4 v, const Pre &) const {
    if (n < da)
      *reinterpret_cast<float4 *>(P + (long long)m * da + n) = v;
    else if (n - da < nx)
      *reinterpret_cast<float4 *>(HX + (long long)m * ldx + n - da) = v;
  }
};

// Decoder GRU phase A (nnet.py:66-69): columns [0,dh) -> z, [dh,2dh) -> r
// (stored as r*h), [2dh,3dh) -> x W_h + b_h (the input half of h~).
struct EpiGruA {
  static constexpr bool kTile = false;
  const float *bias;  // [3 dh]
  const float *S;     // current state rows, stride lds
  int lds, dh;
  float *Z, *RH, *XH;  // [M, dh] each
  __half *RHh = nullptr, *RHl = nullptr;  // optional 3xFP16 split of r*s
  // optional per-row table term (the y rows' contribution, amun_model YWg)
  const float *rowadd = nullptr;
  const int *rowtok = nullptr;
  int ldadd = 0;
  __device__ void operator()(int m, int n, float v, int) const {
    if (rowadd) v += rowadd[(long long)rowtok[m] * ldadd + n];
    v += bias[n];
    if (n < dh) {
      Z[(long long)m * dh + n] = sigmoid_acc(v);
    } else if (n < 2 * dh) {
      int j = n - dh;
      const float rh = sigmoid_acc(v) * S[(long long)m * lds + j];
      RH[(long long)m * dh + j] = rh;
      store_split(RHh, RHl, (long long)m * dh + j, rh);
    } else {
      XH[(long long)m * dh + n - 2 * dh] = v;
    }
  }
  struct Pre {
    float4 b, s, r;
  };
  __device__ __forceinline__ Pre load4(int m, int n) const {
    Pre p;
    p.b = *reinterpret_cast<const float4 *>(bias + n);
    p.r = rowadd ? *reinterpret_cast<const float4 *>(rowadd + (long long)rowtok[m] * ldadd + n)
                 : make_float4(0.f, 0.f, 0.f, 0.f);
    p.s = (n >= dh && n < 2 * dh) ? *reinterpret_cast<const float4 *>(S + (long long)m * lds + n - dh)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
    return p;
  }
  __device__ __forceinline__ void store4(int m, int n, float4 v, const Pre &p) const {
    v.x += p.r.x;
    v.y += p.r.y;
    v.z += p.r.z;
    v.w += p.r.w;
    v.x += p.b.x;
    v.y += p.b.y;
    v.z += p.b.z;
    v.w += p.b.w;
    if (n < dh) {
      *reinterpret_cast<float4 *>(Z + (long long)m * dh + n) =
          make_float4(sigmoid_acc(v.x), sigmoid_acc(v.y), sigmoid_acc(v.z), sigmoid_acc(v.w));
    } else if (n < 2 * dh) {
      const long long o = (long long)m * dh + n - dh;
      const float4 rh = make_float4(sigmoid_acc(v.x) * p.s.x, sigmoid_acc(v.y) * p.s.y, sigmoid_acc(v.z) * p.s.z,
                                    sigmoid_acc(v.w) * p.s.w);
      *reinterpret_cast<float4 *>(RH + o) = rh;
      store_split4(RHh, RHl, o, rh);
    } else {
      *reinterpret_cast<float4 *>(XH + (long long)m * dh + n - 2 * dh) = v;
    }
  }
};

// Decoder GRU phase B (nnet.py:69-70): h~ = tanh(xW_h + b_h + (r*h)U_h),
// s' = (1-z) s + z h~.
struct EpiGruB {
  static constexpr bool kTile = false;
  const float *S;
  int lds, dh;
  const float *Z, *XH;
  float *Sn;
  __half *Snh = nullptr, *Snl = nullptr;  // optional 3xFP16 split of s'
  __device__ void operator()(int m, int n, float v, int) const {
    long long o = (long long)m * dh + n;
    float ht = tanhf(v + XH[o]);
    float zz = Z[o];
    float s = S[(long long)m * lds + n];
    const float sn = (1.0f - zz) * s + zz * ht;
    Sn[o] = sn;
    store_split(Snh, Snl, o, sn);
  }
  struct Pre {
    float4 xh, z, s;
  };
  __device__ __forceinline__ Pre load4(int m, int n) const {
    const long long o = (long long)m * dh + n;
    Pre p;
    p.xh = *reinterpret_cast<const float4 *>(XH + o);
    p.z = *reinterpret_cast<const float4 *>(Z + o);
    p.s = *reinterpret_cast<const float4 *>(S + (long long)m * lds + n);
    return p;
  }
  __device__ __forceinline__ void store4(int m, int n, float4 v, const Pre &p) const {
    const long long o = (long long)m * dh + n;
    float4 sn;
    sn.x = (1.0f - p.z.x) * p.s.x + p.z.x * tanhf(v.x + p.xh.x);
    sn.y = (1.0f - p.z.y) * p.s.y + p.z.y * tanhf(v.y + p.xh.y);
    sn.z = (1.0f - p.z.z) * p.s.z + p.z.z * tanhf(v.z + p.xh.z);
    sn.w = (1.0f - p.z.w) * p.s.w + p.z.w * tanhf(v.w + p.xh.w);
    *reinterpret_cast<float4 *>(Sn + o) = sn;
    store_split4(Snh, Snl, o, sn);
  }
};

// Encoder recurrence phase A, both directions (blockIdx.z = dir).
// XP holds x W + b for all positions: [B*Jmax, 6 dh] = [fwd z r h | bwd z r h].
struct EpiEncA {
  static constexpr bool kTile = false;
  const float *XP;
  const float *Hs;  // [2][B][dh] states
  const int *len;
  int jmax, dh, t, B;
  float *Z, *RH;  // [2][B][dh]
  __device__ void operator()(int b, int n, float v, int dir) const {
    int L = len[b];
    if (t >= L) return;
    int pos = dir == 0 ? t : L - 1 - t;
    v += XP[((long long)b * jmax + pos) * 6 * dh + dir * 3 * dh + n];
    long long o = ((long long)dir * B + b) * dh;
    if (n < dh) {
      Z[o + n] = sigmoid_acc(v);
    } else {
      int j = n - dh;
      RH[o + j] = sigmoid_acc(v) * Hs[o + j];
    }
  }
};

struct EpiEncB {
  static constexpr bool kTile = false;
  const float *XP;
  float *Hs;
  const int *len;
  int jmax, dh, t, B;
  const float *Z;
  float *Hann;  // [B][jmax][2 dh]
  __device__ void operator()(int b, int n, float v, int dir) const {
    int L = len[b];
    if (t >= L) return;
    int pos = dir == 0 ? t : L - 1 - t;
    long long o = ((long long)dir * B + b) * dh + n;
    float ht = tanhf(v + XP[((long long)b * jmax + pos) * 6 * dh + dir * 3 * dh + 2 * dh + n]);
    float zz = Z[o];
    float h = (1.0f - zz) * Hs[o] + zz * ht;
    Hs[o] = h;
    Hann[((long long)b * jmax + pos) * 2 * dh + dir * dh + n] = h;
  }
};

// Logit epilogue, fused mode: per (row, N-tile) partial log-sum-exp and the
// tile's top-kk (logit desc, token asc).  Full logits never reach HBM.
//   pmax/psum: [M][ntiles]   cval/ctok: [M][ntiles][kk]
// Tensor-core encoder recurrence (gemm_sk.cuh, decode.cu encode_bucket):
// both directions in one GEMM over 2B rows m = dir * B + b, with block rows
// [h_fwd | 0] / [0 | h_bwd] against K-stacked weights [U_fwd ; U_bwd].  Same
// arithmetic as EpiEncA / EpiEncB per (b, n, dir); additionally keeps the
// 3xFP16 splits of r*h (phase-B input) and of h (next step's phase-A input,
// and the annotation rows for precomp_att).
struct EpiEncA2 {
  const float *XP;
  const float *Hs;  // [2B][dh]
  const int *len;
  int jmax, dh, t, B;
  float *Z, *RH;            // [2B][dh]
  __half *RRh, *RRl;        // [2B][2dh] block rows
  struct Pre {
    float4 xp, hs;
    int L;
  };
  __device__ __forceinline__ Pre load4(int m, int n) const {
    Pre p;
    const int dir = m >= B, b = m - dir * B;
    p.L = len[b];
    if (t < p.L) {
      const int pos = dir == 0 ? t : p.L - 1 - t;
      p.xp = *reinterpret_cast<const float4 *>(XP + ((long long)b * jmax + pos) * 6 * dh + dir * 3 * dh + n);
      p.hs = n >= dh ? *reinterpret_cast<const float4 *>(Hs + (long long)m * dh + n - dh) : make_float4(0, 0, 0, 0);
    }
    return p;
  }
  __device__ __forceinline__ void store4(int m, int n, float4 v, const Pre &p) const {
    if (t >= p.L) return;
    const int dir = m >= B;
    v.x += p.xp.x;
    v.y += p.xp.y;
    v.z += p.xp.z;
    v.w += p.xp.w;
    const long long o = (long long)m * dh;
    if (n < dh) {
      *reinterpret_cast<float4 *>(Z + o + n) =
          make_float4(sigmoid_acc(v.x), sigmoid_acc(v.y), sigmoid_acc(v.z), sigmoid_acc(v.w));
    } else {
      const int j = n - dh;
      const float4 rh = make_float4(sigmoid_acc(v.x) * p.hs.x, sigmoid_acc(v.y) * p.hs.y, sigmoid_acc(v.z) * p.hs.z,
                                    sigmoid_acc(v.w) * p.hs.w);
      *reinterpret_cast<float4 *>(RH + o + j) = rh;
      store_split4(RRh, RRl, (long long)m * 2 * dh + dir * dh + j, rh);
    }
  }
};
struct EpiEncB2 {
  const float *XP;
  float *Hs;
  const int *len;
  int jmax, dh, t, B;
  const float *Z;
  float *Hann;               // [B][jmax][2dh]
  __half *HHh, *HHl;         // [2B][2dh] block rows (next phase-A input)
  __half *Hah, *Hal;         // [B][jmax][2dh] split annotations (precomp_att input)
  struct Pre {
    float4 xp, z, hs;
    int L;
  };
  __device__ __forceinline__ Pre load4(int m, int n) const {
    Pre p;
    const int dir = m >= B, b = m - dir * B;
    p.L = len[b];
    if (t < p.L) {
      const int pos = dir == 0 ? t : p.L - 1 - t;
      const long long o = (long long)m * dh + n;
      p.xp = *reinterpret_cast<const float4 *>(XP + ((long long)b * jmax + pos) * 6 * dh + dir * 3 * dh + 2 * dh + n);
      p.z = *reinterpret_cast<const float4 *>(Z + o);
      p.hs = *reinterpret_cast<const float4 *>(Hs + o);
    }
    return p;
  }
  __device__ __forceinline__ void store4(int m, int n, float4 v, const Pre &p) const {
    if (t >= p.L) return;
    const int dir = m >= B, b = m - dir * B;
    const int pos = dir == 0 ? t : p.L - 1 - t;
    const long long o = (long long)m * dh + n;
    float4 h;
    h.x = (1.0f - p.z.x) * p.hs.x + p.z.x * tanhf(v.x + p.xp.x);
    h.y = (1.0f - p.z.y) * p.hs.y + p.z.y * tanhf(v.y + p.xp.y);
    h.z = (1.0f - p.z.z) * p.hs.z + p.z.z * tanhf(v.z + p.xp.z);
    h.w = (1.0f - p.z.w) * p.hs.w + p.z.w * tanhf(v.w + p.xp.w);
    *reinterpret_cast<float4 *>(Hs + o) = h;
    const long long ao = ((long long)b * jmax + pos) * 2 * dh + dir * dh + n;
    *reinterpret_cast<float4 *>(Hann + ao) = h;
    store_split4(HHh, HHl, (long long)m * 2 * dh + dir * dh + n, h);
    store_split4(Hah, Hal, ao, h);
  }
};

struct EpiLogitTopK {
  static constexpr bool kTile = true;
  const float *bias;
  int kk, ntiles;
  float *pmax, *psum, *cval;
  int *ctok;
  __device__ void tile(const float *Ct, int m0, int n0, int M, int N, int) const {
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const int nt = n0 / kBN;
    for (int r = warp; r < kBM; r += kThreads / 32) {
      int m = m0 + r;
      if (m >= M) break;
      float v[4];
      bool ok[4];
      float mx = -INFINITY;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        int c = lane + 32 * q;
        ok[q] = (n0 + c) < N;
        v[q] = ok[q] ? Ct[r * (kBN + 1) + c] + bias[n0 + c] : -INFINITY;
        mx = fmaxf(mx, v[q]);
      }
      mx = warp_max(mx);
      float se = 0.f;
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (ok[q]) se += expf(v[q] - mx);
      se = warp_sum(se);
      if (lane == 0) {
        pmax[(long long)m * ntiles + nt] = mx;
        psum[(long long)m * ntiles + nt] = se;
      }
      // kk passes of "best key strictly below the previous pick"
      double lv = INFINITY;
      int lt = -1;
      long long base = ((long long)m * ntiles + nt) * kk;
      for (int p = 0; p < kk; ++p) {
        Key best{-INFINITY, 0x7fffffff, 0};
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          if (!ok[q]) continue;
          int tok = n0 + lane + 32 * q;
          double x = v[q];
          bool below = (x < lv) || (x == lv && tok > lt);
          if (below && key_better(x, tok, 0, best.v, best.tok, 0)) best = Key{x, tok, 0};
        }
        best = warp_best(best);
        if (lane == 0) {
          cval[base + p] = best.tok == 0x7fffffff ? -INFINITY : (float)best.v;
          ctok[base + p] = best.tok == 0x7fffffff ? -1 : best.tok;
        }
        lv = best.v;
        lt = best.tok;
      }
    }
  }
};

// ---- encode-ahead recurrence (decode.cu encode_ahead), tensor-core only.
// Rows m are encoder rows (sentences in descending length order, all active
// at this step); the accumulator holds h U, and the input projection plus
// bias, x_t W + b, is one gathered row of the model's per-source-token table
// (amun_model::XWenc, built at load).  nnet.py:66-70, 110-126.
// Phase A: z = sigmoid(acc + xw_z) -> Z;  r = sigmoid(acc + xw_r), r * h -> split RH.
struct EpiEncFA {
  static constexpr bool kTile = false;
  const float *xw;    // [Vs][ldx] per-token input projection + bias, this direction's (z | r) columns
  const int *tok;     // [n] the step's source token per row
  int ldx;
  const float *H;     // [n][dh] state
  float *Z;           // [n][dh]
  __half *RHh, *RHl;  // [n][dh]
  int dh;
  __device__ void operator()(int, int, float, int) const {}
  struct Pre {
    float4 b, hs;
  };
  __device__ __forceinline__ Pre load4(int m, int n) const {
    Pre p;
    p.b = *reinterpret_cast<const float4 *>(xw + (long long)tok[m] * ldx + n);
    p.hs = n >= dh ? *reinterpret_cast<const float4 *>(H + (long long)m * dh + n - dh) : make_float4(0, 0, 0, 0);
    return p;
  }
  __device__ __forceinline__ void store4(int m, int n, float4 v, const Pre &p) const {
    v.x += p.b.x;
    v.y += p.b.y;
    v.z += p.b.z;
    v.w += p.b.w;
    if (n < dh) {
      *reinterpret_cast<float4 *>(Z + (long long)m * dh + n) =
          make_float4(sigmoid_acc(v.x), sigmoid_acc(v.y), sigmoid_acc(v.z), sigmoid_acc(v.w));
    } else {
      const float4 rh = make_float4(sigmoid_acc(v.x) * p.hs.x, sigmoid_acc(v.y) * p.hs.y,
                                    sigmoid_acc(v.z) * p.hs.z, sigmoid_acc(v.w) * p.hs.w);
      store_split4(RHh, RHl, (long long)m * dh + n - dh, rh);
    }
  }
};
// Phase B: h~ = tanh(acc + xw_h), h' = (1 - z) h + z h~ -> state (fp32 and
// split), the annotation store row of (sentence, position) at column
// dir*dh + n (fp32 and split, the precomp_att input), and the running sum
// over positions for the initial-state mean (nnet.py:129).
struct EpiEncFB {
  static constexpr bool kTile = false;
  const float *xw;    // [Vs][ldx] per-token input projection + bias, this direction's h columns
  const int *tok;     // [n]
  int ldx;
  float *H;           // [n][dh]
  const float *Z;
  __half *Hh, *Hl;    // [n][dh] next phase-A operand
  float *Hann;        // store [rows][2dh] fp32 (nullptr: only the split copy is kept)
  __half *Hah, *Hal;
  float *Hsum;        // [n][2dh]
  const int *len;            // [n]
  const long long *ann_row;  // [n] store row of position 0
  int dh, t, dir;
  __device__ void operator()(int, int, float, int) const {}
  struct Pre {
    float4 b, z, hs, sum;
    int L;
    long long ar;
  };
  __device__ __forceinline__ Pre load4(int m, int n) const {
    Pre p;
    const long long o = (long long)m * dh + n;
    p.b = *reinterpret_cast<const float4 *>(xw + (long long)tok[m] * ldx + n);
    p.z = *reinterpret_cast<const float4 *>(Z + o);
    p.hs = *reinterpret_cast<const float4 *>(H + o);
    p.sum = t ? *reinterpret_cast<const float4 *>(Hsum + (long long)m * 2 * dh + dir * dh + n)
              : make_float4(0, 0, 0, 0);
    p.L = len[m];
    p.ar = ann_row[m];
    return p;
  }
  __device__ __forceinline__ void store4(int m, int n, float4 v, const Pre &p) const {
    const long long o = (long long)m * dh + n;
    float4 h;
    h.x = (1.0f - p.z.x) * p.hs.x + p.z.x * tanhf(v.x + p.b.x);
    h.y = (1.0f - p.z.y) * p.hs.y + p.z.y * tanhf(v.y + p.b.y);
    h.z = (1.0f - p.z.z) * p.hs.z + p.z.z * tanhf(v.z + p.b.z);
    h.w = (1.0f - p.z.w) * p.hs.w + p.z.w * tanhf(v.w + p.b.w);
    *reinterpret_cast<float4 *>(H + o) = h;
    store_split4(Hh, Hl, o, h);
    const int pos = dir ? p.L - 1 - t : t;
    const long long ao = (p.ar + pos) * 2 * dh + dir * dh + n;
    if (Hann) *reinterpret_cast<float4 *>(Hann + ao) = h;
    store_split4(Hah, Hal, ao, h);
    *reinterpret_cast<float4 *>(Hsum + (long long)m * 2 * dh + dir * dh + n) =
        make_float4(p.sum.x + h.x, p.sum.y + h.y, p.sum.z + h.z, p.sum.w + h.w);
  }
};

}  // namespace amun

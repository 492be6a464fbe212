// Non-GEMM kernels of the decode path (see kernels.cuh).
#include <cooperative_groups.h>
#include <mutex>
#include <set>
#include <utility>

#include "kernels.cuh"
#include "tc_common.cuh"

namespace amun {

// Opt a kernel into the device's full dynamic shared memory, once per
// (kernel, device).  The attribute is only an upper bound, so one value
// serves every launch size -- and host threads decoding concurrently on one
// device (Engine workers) never lower it under each other's launches, which
// setting it to each launch's own size would.
static void smem_optin(const void *kern) {
  static std::mutex mu;
  static std::set<std::pair<const void *, int>> done;
  int dev = 0;
  AMUN_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> g(mu);
  if (done.insert({kern, dev}).second) {
    int optin = 0;
    AMUN_CUDA(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa{};
    AMUN_CUDA(cudaFuncGetAttributes(&fa, kern));
    AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   optin - (int)fa.sharedSizeBytes));
  }
}


// ================================================================ attention

// tanh(x) = 1 - 2 / (exp(2x) + 1) with the ex2-based exponential and a fast
// reciprocal: ~1e-7 absolute error (saturates exactly to +-1), far below the
// fp32 rounding of the 1024-term energy sum it feeds.
__device__ __forceinline__ float tanh_attn(float x) { return 1.0f - __fdividef(2.0f, __expf(2.0f * x) + 1.0f); }

__device__ __forceinline__ float tc_rcp(float x) {  // rcp.approx (SFU), as __fdividef
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ float tc_exp2(float x) {  // ex2.approx (SFU)
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(256) attention_kernel(AttnArgs a) {
  extern __shared__ float sm[];
  float *q = sm;              // [da]
  float *vv = sm + a.da;      // [da]
  float *e = sm + 2 * a.da;   // [jmax]
  __shared__ float s_red[2];
  const int r = blockIdx.x;
  const int b = r / a.rows_per_sent;
  if (a.n_act) {
    int slot = r % a.rows_per_sent;
    if (a.done[b] || slot >= a.n_act[b]) return;
  }
  const int J = a.len[b];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  for (int i = threadIdx.x; i < a.da; i += blockDim.x) {
    q[i] = a.Q[(long long)r * a.ldq + i];
    vv[i] = a.v[i];
  }
  __syncthreads();
  const float *Pb = a.P + (long long)b * a.jmax * a.da;
  // energies: warp per source position, 4 independent accumulators per lane
  for (int j = warp; j < J; j += nw) {
    const float *pj = Pb + (long long)j * a.da;
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    for (int i0 = lane; i0 < a.da; i0 += 128) {
      float p[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) p[u] = (i0 + 32 * u < a.da) ? __ldg(pj + i0 + 32 * u) : 0.f;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = i0 + 32 * u;
        if (i < a.da) acc[u] = fmaf(vv[i], tanh_attn(p[u] + q[i]), acc[u]);
      }
    }
    float s = warp_sum((acc[0] + acc[1]) + (acc[2] + acc[3]));
    if (lane == 0) e[j] = s;
  }
  __syncthreads();
  if (warp == 0) {
    float mx = -INFINITY;
    for (int j = lane; j < J; j += 32) mx = fmaxf(mx, e[j]);
    mx = warp_max(mx);
    float s = 0.f;
    for (int j = lane; j < J; j += 32) {
      float w = expf(e[j] - mx);
      e[j] = w;
      s += w;
    }
    s = warp_sum(s);
    if (lane == 0) s_red[0] = s;
  }
  __syncthreads();
  const float inv = 1.0f / s_red[0];
  for (int j = threadIdx.x; j < J; j += blockDim.x) {
    float al = e[j] * inv;
    e[j] = al;
    if (a.alpha) a.alpha[(long long)r * a.jmax + j] = al;
  }
  __syncthreads();
  // context: 8 independent column accumulators per thread, coalesced H rows
  const float *Hb = a.H + (long long)b * a.jmax * a.dh2;
  for (int c0 = threadIdx.x; c0 < a.dh2; c0 += 8 * blockDim.x) {
    float acc[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) acc[u] = 0.f;
    for (int j = 0; j < J; ++j) {
      const float w = e[j];
      const float *hj = Hb + (long long)j * a.dh2;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int c = c0 + u * blockDim.x;
        if (c < a.dh2) acc[u] = fmaf(w, __ldg(hj + c), acc[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int c = c0 + u * blockDim.x;
      if (c < a.dh2) {
        a.ctx[(long long)r * a.ldctx + c] = acc[u];
        store_split(a.ctx_hi, a.ctx_lo, (long long)r * a.ldctx_h + c, acc[u]);
      }
    }
  }
}

// Two-phase attention for beam rows grouped by sentence (rows_per_sent = k
// rows of sentence b share P_b / H_b):
//   attn_energy_kernel: warp per (sentence b, source position j); the lane
//     keeps 32 elements of P_bj and v in registers and computes
//     e[r, j] = v . tanh(P_bj + q_r) for every active row r of the sentence
//     (P_bj read once per sentence, 32 independent tanh chains per lane).
//   attn_context_kernel: CTA per (sentence, 256 columns of 2 d_h): masked
//     softmax of the sentence's energy rows in shared memory, then
//     thread = column, ctx[r, c] = sum_j alpha[r, j] H_bj[c] over the rows.
// Energies and context sums run in a fixed order, independent of which other
// sentences share the launch.
constexpr int kEnergyWarps = 8;  // warps per energy CTA
constexpr int kEnergyPos = 8;    // source positions per energy CTA (one per warp)
constexpr float kTwoLog2e = 2.8853900817779268f;  // 2 / ln 2: e^{2x} = 2^{x kTwoLog2e}
constexpr float kFactorSafe = 20.f;  // |p|, |q| below this: e^{2p} e^{2q} cannot overflow
// per-sentence kernel, paired reciprocals: (1 + e^{2p} e^{2q}) <= e^44, so the
// product of two such terms stays below the fp32 maximum (e^88.7)
constexpr float kPairSafe = 11.f;

// tanh(p + q) = 1 - 2 / (1 + e^{2p} e^{2q}): e^{2p} is computed once per
// (position, element) and shared by the beam rows, e^{2q} once per (row,
// element) and shared by all positions, leaving one SFU op (rcp) per tanh
// instead of two.  Rows or positions with a factor outside +-kFactorSafe take
// the direct formula (warp-uniform branch).
template <int KA>
__global__ void __launch_bounds__(32 * kEnergyWarps, 3) attn_energy_kernel(AttnArgs a) {
  extern __shared__ float vs[];  // [da] v, then [k] "large query row" flags
  const int b = blockIdx.y;
  if (a.n_act && a.done[b]) return;
  const int J = a.len[b];
  const int j0 = blockIdx.x * kEnergyPos;
  if (j0 >= J) return;
  const int k = a.rows_per_sent;
  const int na = a.n_act ? a.n_act[b] : k;
  int *qbig = reinterpret_cast<int *>(vs + a.da);
  const int lane = threadIdx.x % 32, warp = threadIdx.x / 32;
  const int j = j0 + warp;
  // this warp's P row first: its latency overlaps the prologue below
  const float *pj = a.P + ((long long)b * a.jmax + min(j, J - 1)) * a.da;
  float ep[32];
#pragma unroll
  for (int u = 0; u < 32; ++u) {
    const int i = lane + 32 * u;
    ep[u] = i < a.da ? __ldg(pj + i) : 0.f;
  }
  for (int i = threadIdx.x; i < a.da; i += blockDim.x) vs[i] = __ldg(a.v + i);
  for (int r = warp; r < na; r += kEnergyWarps) {
    const float *qr = a.Q + (long long)(b * k + r) * a.ldq;
    float m = 0.f;
    for (int c = lane; c < a.da; c += 32) m = fmaxf(m, fabsf(__ldg(qr + c)));
    m = warp_max(m);
    if (lane == 0) qbig[r] = m > kFactorSafe;
  }
  __syncthreads();
  if (j >= J) return;
  int anybig = 0;
  for (int r = 0; r < na; ++r) anybig |= qbig[r];
  float pm = 0.f;
#pragma unroll
  for (int u = 0; u < 32; ++u) {
    pm = fmaxf(pm, fabsf(ep[u]));
    ep[u] = tc_exp2(ep[u] * kTwoLog2e);
  }
  const bool pbig = warp_max(pm) > kFactorSafe;
  if (!pbig && !anybig && na == KA && a.da == 1024) {
    // exact row count, full-width rows: KA independent accumulation chains
    // per lane; e^{2q} rows come from the query GEMM epilogue (L1-resident)
    const float *eqr[KA];
#pragma unroll
    for (int r = 0; r < KA; ++r) eqr[r] = a.EQ + (long long)(b * k + r) * a.ldq + lane;
    float acc[KA];
#pragma unroll
    for (int r = 0; r < KA; ++r) acc[r] = 0.f;
#pragma unroll
    for (int u = 0; u < 32; ++u) {
      const float vi = vs[lane + 32 * u];
#pragma unroll
      for (int r = 0; r < KA; ++r)
        acc[r] = fmaf(vi, fmaf(-2.0f, tc_rcp(fmaf(ep[u], __ldg(eqr[r] + 32 * u), 1.0f)), 1.0f), acc[r]);
    }
#pragma unroll
    for (int r = 0; r < KA; ++r) {
      const float sum = warp_sum(acc[r]);
      if (lane == 0) a.energy[(long long)(b * k + r) * a.jmax + j] = sum;
    }
  } else {
    for (int r = 0; r < na; ++r) {
      float s0 = 0.f;
      const float *qr = a.Q + (long long)(b * k + r) * a.ldq;
      const float *er = a.EQ + (long long)(b * k + r) * a.ldq;
      const bool direct = pbig || qbig[r];
      for (int u = 0; u < 32; ++u) {
        const int i = lane + 32 * u;
        if (i < a.da)
          s0 = fmaf(vs[i],
                    direct ? tanh_attn(__ldg(pj + i) + __ldg(qr + i))
                           : 1.0f - __fdividef(2.0f, fmaf(ep[u], __ldg(er + i), 1.0f)),
                    s0);
      }
      const float sum = warp_sum(s0);
      if (lane == 0) a.energy[(long long)(b * k + r) * a.jmax + j] = sum;
    }
  }
}

constexpr int kCtxCols = 128;    // threads per J-group: thread = 4 consecutive columns (float4)
constexpr int kCtxGroups = 2;    // J-groups: group g sums positions j = g, g + 2, ... (then fixed-order add)
constexpr int kCtxRows = 8;      // row accumulators per pass
constexpr int kCtxUnroll = 8;    // independent 16-byte loads in flight per thread

__global__ void __launch_bounds__(kCtxCols * kCtxGroups) attn_context_kernel(AttnArgs a) {
  extern __shared__ float al[];  // [k][jmax] alpha, then [kCtxRows][kCtxCols] float4 partials of group 1
  const int b = blockIdx.x;
  if (a.n_act && a.done[b]) return;
  const int k = a.rows_per_sent;
  const int na = a.n_act ? a.n_act[b] : k;
  const int J = a.len[b];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, nw = blockDim.x / 32;
  float4 *part = reinterpret_cast<float4 *>(al + ((k * a.jmax + 3) & ~3));
  // masked softmax over j < J, one warp per row (nnet.py:137-139)
  for (int r = warp; r < na; r += nw) {
    const float *er = a.energy + (long long)(b * k + r) * a.jmax;
    float *e = al + r * a.jmax;
    float mx = -INFINITY;
    for (int j = lane; j < J; j += 32) {
      e[j] = er[j];
      mx = fmaxf(mx, e[j]);
    }
    mx = warp_max(mx);
    float s = 0.f;
    for (int j = lane; j < J; j += 32) {
      const float x = expf(e[j] - mx);
      e[j] = x;
      s += x;
    }
    s = warp_sum(s);
    const float inv = 1.0f / s;
    for (int j = lane; j < J; j += 32) {
      const float x = e[j] * inv;
      e[j] = x;
      if (a.alpha && blockIdx.y == 0) a.alpha[(long long)(b * k + r) * a.jmax + j] = x;
    }
  }
  __syncthreads();
  const int grp = tid / kCtxCols, ct = tid % kCtxCols;
  const int c = (blockIdx.y * kCtxCols + ct) * 4;
  const bool live = c < a.dh2;
  const float4 *Hb = reinterpret_cast<const float4 *>(a.H + (long long)b * a.jmax * a.dh2 + (live ? c : 0));
  const int hs = a.dh2 / 4;  // float4 stride between positions
  for (int r0 = 0; r0 < na; r0 += kCtxRows) {
    float4 acc[kCtxRows];
#pragma unroll
    for (int r = 0; r < kCtxRows; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (live) {
      int j = grp;
      for (; j + kCtxGroups * (kCtxUnroll - 1) < J; j += kCtxGroups * kCtxUnroll) {
        float4 h[kCtxUnroll];
#pragma unroll
        for (int jj = 0; jj < kCtxUnroll; ++jj) h[jj] = __ldg(Hb + (long long)(j + kCtxGroups * jj) * hs);
#pragma unroll
        for (int jj = 0; jj < kCtxUnroll; ++jj)
#pragma unroll
          for (int r = 0; r < kCtxRows; ++r)
            if (r0 + r < na) {
              const float w = al[(r0 + r) * a.jmax + j + kCtxGroups * jj];
              acc[r].x = fmaf(w, h[jj].x, acc[r].x);
              acc[r].y = fmaf(w, h[jj].y, acc[r].y);
              acc[r].z = fmaf(w, h[jj].z, acc[r].z);
              acc[r].w = fmaf(w, h[jj].w, acc[r].w);
            }
      }
      for (; j < J; j += kCtxGroups) {
        const float4 h = __ldg(Hb + (long long)j * hs);
#pragma unroll
        for (int r = 0; r < kCtxRows; ++r)
          if (r0 + r < na) {
            const float w = al[(r0 + r) * a.jmax + j];
            acc[r].x = fmaf(w, h.x, acc[r].x);
            acc[r].y = fmaf(w, h.y, acc[r].y);
            acc[r].z = fmaf(w, h.z, acc[r].z);
            acc[r].w = fmaf(w, h.w, acc[r].w);
          }
      }
    }
    // fixed-order combine of the two J-groups: ctx = sum(even j) + sum(odd j)
    if (grp == 1) {
#pragma unroll
      for (int r = 0; r < kCtxRows; ++r) part[r * kCtxCols + ct] = acc[r];
    }
    __syncthreads();
    if (grp == 0 && live) {
#pragma unroll
      for (int r = 0; r < kCtxRows; ++r) {
        if (r0 + r >= na) break;
        const float4 o4 = part[r * kCtxCols + ct];
        const float vals[4] = {acc[r].x + o4.x, acc[r].y + o4.y, acc[r].z + o4.z, acc[r].w + o4.w};
        const long long o = (long long)(b * k + r0 + r) * a.ldctx + c;
        const long long oh = (long long)(b * k + r0 + r) * a.ldctx_h + c;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          a.ctx[o + u] = vals[u];
          store_split(a.ctx_hi, a.ctx_lo, oh + u, vals[u]);
        }
      }
    }
    __syncthreads();
  }
}

// Fused per-sentence attention (one CTA of 512 threads per sentence):
// the energies of every position for every beam row (factored tanh as in
// attn_energy_kernel), the masked softmax in shared memory, and the context
// (thread = 4 consecutive columns, all rows, positions summed in order).  One
// launch and 64 CTAs per bucket step instead of two launches of 256 CTAs:
// fewer, longer-lived CTAs leave the SMs to the tensor-core kernels of the
// other bucket lanes (the step is throughput-bound with 16 lanes in flight).
// Two CTAs per SM for beams <= 8 (<= 64 registers: P rows in chunks of 8,
// e^{2q} rows staged in shared memory), so a step's 64 sentence CTAs share
// the SMs left by the other lanes' tensor-core kernels.
// PROJ (projected-context mode, AttnArgs.su): one thread per 4 columns of
// the 3 dh + de wide projected rows (1024 threads; 512 threads with two
// quads each above beam 8, where 64 registers would spill), and the gate
// epilogue.
// projected-context annotation staging: kProjNB buffers of kProjHP positions
#ifndef AMUN_PROJ_HP
#define AMUN_PROJ_HP 4
#endif
#ifndef AMUN_PROJ_NB
#define AMUN_PROJ_NB 3
#endif
// P values per lane per energies chunk (the next chunk loads during this one)
#ifndef AMUN_ENERGY_CHUNK
#define AMUN_ENERGY_CHUNK 8
#endif
constexpr int kEC = AMUN_ENERGY_CHUNK;
// beams above 12 (e^{2q} rows of 16 beams: 64 KB) keep five 2-position buffers
constexpr int proj_hp(int ka) { return ka <= 12 ? AMUN_PROJ_HP : 2; }
constexpr int proj_nb(int ka) { return ka <= 12 ? AMUN_PROJ_NB : 5; }
// the attn_sent_kernel instantiation a beam width runs (launch_attention's switch)
constexpr int attn_ka(int k) { return (k <= 6 || k == 8 || k == 10 || k == 12) ? k : 16; }
template <int KA>
constexpr int attn_threads(bool proj) { return proj && KA <= 8 ? 1024 : 512; }
template <int KA, bool PROJ>
__global__ void __launch_bounds__(attn_threads<KA>(PROJ), (KA <= 8 && !PROJ) ? 2 : 1) attn_sent_kernel(AttnArgs a) {
  const CtaClock clk(a.kt);
  extern __shared__ float sm[];
  const int b = blockIdx.x;
  if (a.n_act && a.done[b]) return;
  const int k = a.rows_per_sent;
  const int na = a.n_act ? a.n_act[b] : k;
  const int J = a.len[b];
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32, nw = blockDim.x / 32;
  float *vs = sm;                                    // [da]
  float *al = vs + a.da;                             // [k][jmax]
  const int k4 = (k + 3) & ~3;
  int *qrs = reinterpret_cast<int *>(al + (size_t)k * a.jmax);  // [k] row whose query (Q, EQ) and s U_zr row r uses
  int *toks = qrs + k4;                                          // [k] row r's previous token (PROJ epilogue)
  unsigned *wmask = reinterpret_cast<unsigned *>(toks + k4);     // [32] per-warp masks of rows with |q| > kPairSafe
  float *eqs = reinterpret_cast<float *>((reinterpret_cast<uintptr_t>(wmask + 32) + 15) & ~uintptr_t(15));  // [KA][1024] e^{2q} (fast path)
  // H of the sentence streamed into shared memory in chunks of kHP
  // positions by bulk copies, two buffers, issued now and consumed by the
  // context phase: the annotation reads overlap the energies instead of
  // stalling the context loop (one thread per 4 columns: dh2 == 4 x threads)
  // PROJ rows are 14 KB per position: three 4-position buffers keep twelve
  // positions in flight with one CTA barrier per 4 positions (same-box A/B:
  // 4x3 and 6x2 ~1.3% faster than 2x5, 3x3 in between; 171 KB; beams above
  // 12 keep 2x5, 143 KB, next to their 64 KB of e^{2q} rows)
  constexpr int kHP = PROJ ? proj_hp(KA) : 4, kNB = PROJ ? proj_nb(KA) : 2;
  const bool hsmem = PROJ || a.dh2 == 4 * (int)blockDim.x;
  float *hbuf = reinterpret_cast<float *>(
      (reinterpret_cast<uintptr_t>(eqs + (a.da == 1024 ? k * 1024 : 0)) + 127) & ~uintptr_t(127));
  uint64_t *hbar = reinterpret_cast<uint64_t *>(hbuf + kNB * kHP * a.dh2);
  const int nch = (J + kHP - 1) / kHP;
  const float *Hsent = a.H + (long long)b * a.jmax * a.dh2;
  auto issue_chunk = [&](int c) {  // thread 0
    const uint32_t bytes = (uint32_t)(min(kHP, J - c * kHP) * a.dh2 * 4);
    tc::mbar_arrive_expect_tx(&hbar[c % kNB], bytes);
    tc::bulk_load_1d(hbuf + (c % kNB) * kHP * a.dh2, Hsent + (long long)c * kHP * a.dh2, bytes, &hbar[c % kNB]);
  };
  if (hsmem && tid == 0) {
    for (int i = 0; i < kNB; ++i) tc::mbar_init(&hbar[i], 1);
    tc::fence_barrier_init();
    for (int c = 0; c < kNB && c < nch; ++c) issue_chunk(c);
  }
  for (int i = tid; i < a.da; i += blockDim.x) vs[i] = __ldg(a.v + i);
  const bool fast_shape = na == KA && a.da == 1024;
  // the first P chunk of this warp's first position is loaded before the
  // prologue's dependent index loads and barriers (consumed by the energies)
  float nx0[kEC];
  if (fast_shape && warp < J) {
#pragma unroll
    for (int u = 0; u < kEC; ++u) nx0[u] = __ldg(a.P + ((long long)b * a.jmax + warp) * a.da + lane + 32 * u);
  }
  // per-row indices staged once: the query row (the select's parent row in
  // the query-folded step) and the previous token
  if (tid < k) qrs[tid] = a.qrow ? a.qrow[b * k + tid] : b * k + tid;
  else if (PROJ && tid - k < k) toks[tid - k] = a.tok[b * k + tid - k];
  __syncthreads();
  // e^{2q} rows into shared memory and the |q| check of every row in one
  // pass of independent loads (column-parallel over the CTA)
  unsigned qm = 0;
  for (int i = tid; i < a.da; i += blockDim.x) {
#pragma unroll 4
    for (int r = 0; r < na; ++r) {
      const long long qo = (long long)qrs[r] * a.ldq + i;
      if (fabsf(__ldg(a.Q + qo)) > kPairSafe) qm |= 1u << r;
      // rows 2p, 2p+1 interleaved as float2 pairs (one 64-bit load per
      // pair in the energies); an odd last row after the pairs
      if (fast_shape) eqs[r < (KA & ~1) ? ((r >> 1) * 1024 + i) * 2 + (r & 1) : (KA / 2) * 2048 + i] = __ldg(a.EQ + qo);
    }
  }
  qm = __reduce_or_sync(0xffffffffu, qm);
  if (lane == 0) wmask[warp] = qm;
  __syncthreads();
  unsigned qbigm = 0;
  for (int w = 0; w < nw; ++w) qbigm |= wmask[w];
  const int anybig = qbigm != 0;
  // ---- energies: warp per source position (nnet.py:135-136)
  for (int j = warp; j < J; j += nw) {
    const float *pj = a.P + ((long long)b * a.jmax + j) * a.da;
    bool done = false;
    if (fast_shape && !anybig) {
      // factored tanh over the P row in chunks of 8 values per lane (same
      // per-lane order as one pass), |p| tracked for the safety check
      float2 accp[KA / 2 + 1];  // (row 2p+1, row 2p) per pair p; the odd last row in .x of [KA / 2]
#pragma unroll
      for (int p = 0; p <= KA / 2; ++p) accp[p] = make_float2(0.f, 0.f);
      const float2 *eqs2 = reinterpret_cast<const float2 *>(eqs);
      float pm = 0.f;
      // the next chunk's P values are loaded while this chunk is computed
      // (one load latency per position instead of four)
      float nx[kEC];
      if (j == warp) {
#pragma unroll
        for (int u = 0; u < kEC; ++u) nx[u] = nx0[u];
      } else {
#pragma unroll
        for (int u = 0; u < kEC; ++u) nx[u] = __ldg(pj + lane + 32 * u);
      }
#pragma unroll 1
      for (int u0 = 0; u0 < 32; u0 += kEC) {
        float ep[kEC];
#pragma unroll
        for (int u = 0; u < kEC; ++u) ep[u] = nx[u];
        if (u0 + kEC < 32) {
#pragma unroll
          for (int u = 0; u < kEC; ++u) nx[u] = __ldg(pj + lane + 32 * (u0 + kEC + u));
        }
#pragma unroll
        for (int u = 0; u < kEC; ++u) {
          pm = fmaxf(pm, fabsf(ep[u]));
          ep[u] = tc_exp2(ep[u] * kTwoLog2e);
        }
#pragma unroll
        for (int u = 0; u < kEC; ++u) {
          const int i = lane + 32 * (u0 + u);
          const float vi = vs[i];
          // two rows per SFU reciprocal: 1/a = b / (ab), 1/b = a / (ab)
          // (|p|, |q| <= kPairSafe keeps ab finite), the pair's arithmetic
          // as packed f32x2 (the same rounded fma/mul per element as the
          // scalar form: tanh(p + q_r) = 1 - 2 / a_r)
          const float2 epp = make_float2(ep[u], ep[u]), one2 = make_float2(1.0f, 1.0f);
#pragma unroll
          for (int p = 0; p < KA / 2; ++p) {
            const float2 a2 = __ffma2_rn(epp, eqs2[p * 1024 + i], one2);  // (a_2p, a_2p+1)
            const float inv = tc_rcp(a2.x * a2.y);
            const float2 t = __fmul2_rn(a2, make_float2(inv, inv));  // (1 / a_2p+1, 1 / a_2p)
            accp[p] = __ffma2_rn(make_float2(vi, vi), __ffma2_rn(make_float2(-2.0f, -2.0f), t, one2), accp[p]);
          }
          if constexpr (KA % 2 == 1)
            accp[KA / 2].x = fmaf(vi, fmaf(-2.0f, tc_rcp(fmaf(ep[u], eqs[(KA / 2) * 2048 + i], 1.0f)), 1.0f),
                                  accp[KA / 2].x);
        }
      }
      if (!(warp_max(pm) > kPairSafe)) {
#pragma unroll
        for (int r = 0; r < KA; ++r) {
          const float2 ap = accp[r / 2];
          const float sum = warp_sum(r == KA - 1 && KA % 2 == 1 ? ap.x : (r & 1) ? ap.x : ap.y);
          if (lane == 0) al[r * a.jmax + j] = sum;
        }
        done = true;
      }
    }
    if (!done) {
      float pm = 0.f;
      for (int u = 0; u < 32; ++u) {
        const int i = lane + 32 * u;
        if (i < a.da) pm = fmaxf(pm, fabsf(__ldg(pj + i)));
      }
      const bool pbig = warp_max(pm) > kFactorSafe;
      for (int r = 0; r < na; ++r) {
        float s0 = 0.f;
        const float *qr = a.Q + (long long)qrs[r] * a.ldq;
        const float *er = a.EQ + (long long)qrs[r] * a.ldq;
        const bool direct = pbig || ((qbigm >> r) & 1u);
        for (int u = 0; u < 32; ++u) {
          const int i = lane + 32 * u;
          if (i < a.da)
            s0 = fmaf(vs[i],
                      direct ? tanh_attn(__ldg(pj + i) + __ldg(qr + i))
                             : 1.0f - __fdividef(2.0f, fmaf(tc_exp2(__ldg(pj + i) * kTwoLog2e), __ldg(er + i), 1.0f)),
                      s0);
        }
        const float sum = warp_sum(s0);
        if (lane == 0) al[r * a.jmax + j] = sum;
      }
    }
  }
  __syncthreads();
  // ---- masked softmax over j < J, warp per row (nnet.py:137-139)
  for (int r = warp; r < na; r += nw) {
    float *e = al + r * a.jmax;
    float mx = -INFINITY;
    for (int j = lane; j < J; j += 32) mx = fmaxf(mx, e[j]);
    mx = warp_max(mx);
    float s = 0.f;
    for (int j = lane; j < J; j += 32) {
      const float x = expf(e[j] - mx);
      e[j] = x;
      s += x;
    }
    s = warp_sum(s);
    const float inv = 1.0f / s;
    for (int j = lane; j < J; j += 32) {
      const float x = e[j] * inv;
      e[j] = x;
      if (a.alpha) a.alpha[(long long)(b * k + r) * a.jmax + j] = x;
    }
  }
  __syncthreads();
  // ---- context (nnet.py:141): thread = 4 consecutive columns, every row
  const int hs = a.dh2 / 4;
  const float4 *Hb = reinterpret_cast<const float4 *>(a.H + (long long)b * a.jmax * a.dh2);
  if (hsmem) {
    // thread = column quads tid (+ blockDim for the 512-thread PROJ variant)
    constexpr int kQ = PROJ && KA > 8 ? 2 : 1;
    int cq[kQ];
    bool live[kQ];  // PROJ: threads past the row's columns only join the barriers
    float4 acc[kQ][KA];
#pragma unroll
    for (int i = 0; i < kQ; ++i) {
      cq[i] = tid + i * (int)blockDim.x;
      live[i] = !PROJ || cq[i] < hs;
#pragma unroll
      for (int r = 0; r < KA; ++r) acc[i][r] = make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int c = 0; c < nch; ++c) {
      tc::mbar_wait(&hbar[c % kNB], (c / kNB) & 1);
      const float4 *hb = reinterpret_cast<const float4 *>(hbuf + (c % kNB) * kHP * a.dh2);
      const int j0 = c * kHP;
#pragma unroll
      for (int jj = 0; jj < kHP; ++jj) {
        if (j0 + jj >= J || !live[0]) break;
        float4 h[kQ];
#pragma unroll
        for (int i = 0; i < kQ; ++i) h[i] = live[i] ? hb[jj * hs + cq[i]] : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int r = 0; r < KA; ++r)
          if (r < na) {  // positions summed in order, as the global-memory loop below
            const float w = al[r * a.jmax + j0 + jj];
#pragma unroll
            for (int i = 0; i < kQ; ++i) fma4x2(w, h[i], acc[i][r]);
          }
      }
      if (c + kNB < nch) {
        __syncthreads();  // every thread is done with this buffer
        if (tid == 0) {
          tc::fence_proxy_async();
          issue_chunk(c + kNB);
        }
      }
    }
    if constexpr (PROJ) {
      // gate epilogue, columns n .. n + 3 of every row (a quad never
      // straddles two blocks: dh and de are multiples of 4)
#pragma unroll
      for (int i = 0; i < kQ; ++i) {
      const int n = 4 * cq[i], dh = a.dh;
      if (live[i] && n < 3 * dh + a.de) {
        // operands of row r + 1 are loaded (read-only path) while row r is
        // finished and stored: one load latency for the epilogue instead of
        // one per row (the stores would otherwise order the next loads)
        const int reg = n < dh ? 0 : n < 2 * dh ? 1 : n < 3 * dh ? 2 : 3;  // Z | r*s | h~ input | deep output
        const float4 f0 = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 bb = reg < 3 ? __ldg(reinterpret_cast<const float4 *>(a.bg + n)) : f0;
        auto load = [&](int r, float4 &y, float4 &su, float4 &sv) {
          const long long t = toks[r];
          y = reg < 3 ? __ldg(reinterpret_cast<const float4 *>(a.ywg + t * 3 * dh + n))
                      : __ldg(reinterpret_cast<const float4 *>(a.ywo + t * a.de + n - 3 * dh));
          su = reg < 2 ? __ldg(reinterpret_cast<const float4 *>(a.su + (long long)qrs[r] * 2 * dh + n)) : f0;
          sv = reg == 1 ? __ldg(reinterpret_cast<const float4 *>(a.S + ((long long)b * k + r) * a.lds + n - dh)) : f0;
        };
#pragma unroll
        for (int r = 0; r < KA; ++r) {
          if (r >= na) break;
          float4 y, su, sv;
          load(r, y, su, sv);
          const long long gr = (long long)b * k + r;
          const float4 cx = acc[i][r];
          if (reg < 3) {
            float4 v = reg < 2 ? make_float4(cx.x + su.x, cx.y + su.y, cx.z + su.z, cx.w + su.w) : cx;
            v = make_float4(v.x + y.x + bb.x, v.y + y.y + bb.y, v.z + y.z + bb.z, v.w + y.w + bb.w);
            if (reg == 0) {
              *reinterpret_cast<float4 *>(a.Z + gr * dh + n) =
                  make_float4(sigmoid_acc(v.x), sigmoid_acc(v.y), sigmoid_acc(v.z), sigmoid_acc(v.w));
            } else if (reg == 1) {
              const long long o = gr * dh + n - dh;
              store_split(a.RHh, a.RHl, o + 0, sigmoid_acc(v.x) * sv.x);
              store_split(a.RHh, a.RHl, o + 1, sigmoid_acc(v.y) * sv.y);
              store_split(a.RHh, a.RHl, o + 2, sigmoid_acc(v.z) * sv.z);
              store_split(a.RHh, a.RHl, o + 3, sigmoid_acc(v.w) * sv.w);
            } else {
              *reinterpret_cast<float4 *>(a.XH + gr * dh + n - 2 * dh) = v;
            }
          } else {
            *reinterpret_cast<float4 *>(a.CO + gr * a.ldco + n - 3 * dh) =
                make_float4(cx.x + y.x, cx.y + y.y, cx.z + y.z, cx.w + y.w);
          }
        }
      }
      }
    } else {
    const int c4 = tid;
#pragma unroll
    for (int r = 0; r < KA; ++r) {
      if (r >= na) break;
      const long long o = (long long)(b * k + r) * a.ldctx + 4 * c4;
      *reinterpret_cast<float4 *>(a.ctx + o) = acc[0][r];
      const long long oh = (long long)(b * k + r) * a.ldctx_h + 4 * c4;
      store_split(a.ctx_hi, a.ctx_lo, oh + 0, acc[0][r].x);
      store_split(a.ctx_hi, a.ctx_lo, oh + 1, acc[0][r].y);
      store_split(a.ctx_hi, a.ctx_lo, oh + 2, acc[0][r].z);
      store_split(a.ctx_hi, a.ctx_lo, oh + 3, acc[0][r].w);
    }
    }
  }
  for (int c4 = hsmem ? hs : tid; c4 < hs; c4 += blockDim.x) {
    float4 acc[KA];
#pragma unroll
    for (int r = 0; r < KA; ++r) acc[r] = make_float4(0.f, 0.f, 0.f, 0.f);
    constexpr int kHB = KA <= 8 ? 4 : 8;  // H rows in flight per thread
    for (int j0 = 0; j0 < J; j0 += kHB) {
      float4 h[kHB];
#pragma unroll
      for (int jj = 0; jj < kHB; ++jj)
        h[jj] = j0 + jj < J ? __ldg(Hb + (long long)(j0 + jj) * hs + c4) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
      for (int jj = 0; jj < kHB; ++jj) {
        if (j0 + jj >= J) break;
#pragma unroll
        for (int r = 0; r < KA; ++r)
          if (r < na) {
            const float w = al[r * a.jmax + j0 + jj];
            acc[r].x = fmaf(w, h[jj].x, acc[r].x);
            acc[r].y = fmaf(w, h[jj].y, acc[r].y);
            acc[r].z = fmaf(w, h[jj].z, acc[r].z);
            acc[r].w = fmaf(w, h[jj].w, acc[r].w);
          }
      }
    }
#pragma unroll
    for (int r = 0; r < KA; ++r) {
      if (r >= na) break;
      const long long o = (long long)(b * k + r) * a.ldctx + 4 * c4;
      *reinterpret_cast<float4 *>(a.ctx + o) = acc[r];
      const long long oh = (long long)(b * k + r) * a.ldctx_h + 4 * c4;
      store_split(a.ctx_hi, a.ctx_lo, oh + 0, acc[r].x);
      store_split(a.ctx_hi, a.ctx_lo, oh + 1, acc[r].y);
      store_split(a.ctx_hi, a.ctx_lo, oh + 2, acc[r].z);
      store_split(a.ctx_hi, a.ctx_lo, oh + 3, acc[r].w);
    }
  }
  if (a.kt) {
    __syncthreads();
    clk.done();
  }
}

template <int KA>
static void launch_sent(const AttnArgs &a, int B, size_t smem, cudaStream_t st) {
  AttnArgs ak = a;
  ak.kt = ktime_ptr();
  if (a.su) {
    auto kern = attn_sent_kernel<KA, true>;
    if (smem > 48 * 1024) smem_optin(reinterpret_cast<const void *>(kern));
    kern<<<B, attn_threads<KA>(true), smem, st>>>(ak);
  } else {
    auto kern = attn_sent_kernel<KA, false>;
    if (smem > 48 * 1024) smem_optin(reinterpret_cast<const void *>(kern));
    kern<<<B, 512, smem, st>>>(ak);
  }
}

template <int KA>
static void launch_energy(const AttnArgs &a, dim3 grid, size_t smem, cudaStream_t st) {
  auto kern = attn_energy_kernel<KA>;
  static size_t attr_q[64] = {};
  int dev = 0;
  AMUN_CUDA(cudaGetDevice(&dev));
  if (smem > 48 * 1024 && (dev >= 64 || attr_q[dev] < smem)) {
    AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    if (dev < 64) attr_q[dev] = smem;
  }
  kern<<<grid, 32 * kEnergyWarps, smem, st>>>(a);
}

int launch_attention(const AttnArgs &a, int R, cudaStream_t st) {
  if (R <= 0) return 0;
  const int k = a.rows_per_sent;
  const size_t smem = sizeof(float) * (size_t)k * a.jmax;
  const size_t smem_ctx = sizeof(float) * (((size_t)k * a.jmax + 3) & ~size_t(3)) + sizeof(float4) * kCtxRows * kCtxCols;
  const size_t smem_q = sizeof(float) * (size_t)a.da + sizeof(int) * (size_t)k;
  static const bool fused = [] {
    const char *e = getenv("AMUN_ATTN_FUSED");  // 0: two-phase kernels
    return !(e && e[0] == '0');
  }();
  const size_t smem_s = sizeof(float) * ((size_t)a.da + (size_t)k * a.jmax) + sizeof(int) * (size_t)(2 * ((k + 3) & ~3) + 32) + 16 +
                        (a.da == 1024 ? sizeof(float) * (size_t)k * 1024 : 0) +
                        (a.su ? 128 + sizeof(float) * proj_nb(attn_ka(k)) * proj_hp(attn_ka(k)) * (size_t)a.dh2 + proj_nb(attn_ka(k)) * sizeof(uint64_t)
                              : a.dh2 == 4 * 512 ? 128 + sizeof(float) * 2 * 4 * (size_t)a.dh2 + 2 * sizeof(uint64_t) : 0);
  // The kernel is chosen from per-call constants only (beam width, model
  // layout), never from the bucket's longest sentence: the fused and the
  // two-phase kernels sum in different orders, and a sentence's result must
  // not depend on its batch-mates.  A bucket too long for the fused kernel's
  // shared-memory energies is refused instead of silently switching paths.
  const bool fused_ok = fused && a.EQ && a.da <= 1024 && a.dh2 % 4 == 0 && R % k == 0 && k <= 16 &&
                        (a.su || ((size_t)a.ldctx % 4 == 0 && reinterpret_cast<uintptr_t>(a.ctx) % 16 == 0));
  if (a.su && (!fused_ok || a.dh2 > 4 * 1024))
    throw Error(4, "projected-context attention: unsupported shape");
  const size_t smem_lim = 227 * 1024, smem_fixed = smem_s - sizeof(float) * (size_t)k * a.jmax;
  if (fused_ok && smem_s > smem_lim)
    throw Error(4, "source sentence of " + std::to_string(a.jmax) + " tokens exceeds the device attention limit (" +
                       std::to_string(smem_fixed < smem_lim ? (smem_lim - smem_fixed) / (sizeof(float) * k) : 0) +
                       " at beam " + std::to_string(k) + ")");
  if (fused_ok) {
    const int B = R / k;
    switch (k) {  // exact beam width: no predicated-off rows in the inner loops
      case 1: launch_sent<1>(a, B, smem_s, st); break;
      case 2: launch_sent<2>(a, B, smem_s, st); break;
      case 3: launch_sent<3>(a, B, smem_s, st); break;
      case 4: launch_sent<4>(a, B, smem_s, st); break;
      case 5: launch_sent<5>(a, B, smem_s, st); break;
      case 6: launch_sent<6>(a, B, smem_s, st); break;
      case 8: launch_sent<8>(a, B, smem_s, st); break;
      case 10: launch_sent<10>(a, B, smem_s, st); break;
      case 12: launch_sent<12>(a, B, smem_s, st); break;
      default: launch_sent<16>(a, B, smem_s, st); break;
    }
    AMUN_CHECK_LAUNCH();
    return 1;
  }
  if (a.energy && a.EQ && a.da <= 1024 && a.dh2 % 4 == 0 && R % k == 0 && smem_ctx <= 200 * 1024 && smem_q <= 200 * 1024) {
    const int B = R / k;
    const dim3 eg(ceil_div(a.jmax, kEnergyPos), B);
    switch (k) {  // exact beam width: no predicated-off rows in the inner loop
      case 1: launch_energy<1>(a, eg, smem_q, st); break;
      case 2: launch_energy<2>(a, eg, smem_q, st); break;
      case 3: launch_energy<3>(a, eg, smem_q, st); break;
      case 4: launch_energy<4>(a, eg, smem_q, st); break;
      case 5: launch_energy<5>(a, eg, smem_q, st); break;
      case 6: launch_energy<6>(a, eg, smem_q, st); break;
      case 8: launch_energy<8>(a, eg, smem_q, st); break;
      case 10: launch_energy<10>(a, eg, smem_q, st); break;
      case 12: launch_energy<12>(a, eg, smem_q, st); break;
      default: launch_energy<16>(a, eg, smem_q, st); break;
    }
    AMUN_CHECK_LAUNCH();
    if (smem_ctx > 48 * 1024) {
      static size_t attr_set[64] = {};
      int dev = 0;
      AMUN_CUDA(cudaGetDevice(&dev));
      if (dev >= 64 || attr_set[dev] < smem_ctx) {
        AMUN_CUDA(cudaFuncSetAttribute(attn_context_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        if (dev < 64) attr_set[dev] = smem_ctx;
      }
    }
    attn_context_kernel<<<dim3(B, ceil_div(a.dh2, 4 * kCtxCols)), kCtxCols * kCtxGroups, smem_ctx, st>>>(a);
    AMUN_CHECK_LAUNCH();
    return 2;
  }
  size_t smem1 = sizeof(float) * (2 * a.da + a.jmax);
  if (smem1 > 48 * 1024) smem_optin(reinterpret_cast<const void *>(attention_kernel));
  attention_kernel<<<R, 256, smem1, st>>>(a);
  AMUN_CHECK_LAUNCH();
  return 1;
}

// ================================================================ encoder

__global__ void masked_mean_kernel(const float *Hann, const int *len, int jmax, int dh2, float *out) {
  const int b = blockIdx.x;
  const int L = len[b];
  const float *Hb = Hann + (long long)b * jmax * dh2;
  for (int c = threadIdx.x; c < dh2; c += blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < L; ++j) s += Hb[(long long)j * dh2 + c];
    out[(long long)b * dh2 + c] = s / (float)L;
  }
}

void launch_masked_mean(const float *Hann, const int *len, int B, int jmax, int dh2, float *out,
                        cudaStream_t st) {
  masked_mean_kernel<<<B, 256, 0, st>>>(Hann, len, jmax, dh2, out);
  AMUN_CHECK_LAUNCH();
}

// ================================================================ beam init

__global__ void init_beam_kernel(BeamState bs, ModelRows mr, const float *const *S0) {
  const int b = blockIdx.x;
  const int k = bs.k;
  if (threadIdx.x == 0) {
    bs.n_act[b] = 1;
    bs.done[b] = 0;
    bs.steps[b] = 0;
    bs.fin_n[b] = 0;
    bs.best_fin[b] = -INFINITY;
    for (int i = 0; i < k; ++i) {
      bs.score[b * k + i] = 0.0;
      bs.tok[b * k + i] = 0;
      if (bs.qrow) bs.qrow[b * k + i] = b * k + i;
    }
    if (b == 0) *bs.n_done = 0;
  }
  for (int m = 0; m < mr.n_models; ++m) {
    float *XS = mr.XS[m];
    __half *XSh = mr.XSh ? mr.XSh[m] : nullptr;
    __half *XSl = mr.XSl ? mr.XSl[m] : nullptr;
    const float *E = mr.E_trg[m];
    const RowDims md = mr.dim[m];
    for (int i = 0; i < k; ++i) {
      const long long ro = (long long)(b * k + i) * md.ldxs;
      const long long roh = (long long)(b * k + i) * md.ldxh;
      for (int c = threadIdx.x; c < md.ldxs; c += blockDim.x) {
        float v = 0.f;
        if (i == 0) {
          if (c < md.de) v = E[c];  // E_trg[EOS_ID]
          else if (c >= md.s_off && c < md.s_off + md.dh) v = S0[m][(long long)b * md.dh + (c - md.s_off)];
        }
        XS[ro + c] = v;
        store_split(XSh, XSl, roh + c + (c >= md.de ? md.hpad : 0), v);
      }
    }
  }
}

void launch_init_beam(const BeamState &bs, const ModelRows &mr, const float *const *S0, cudaStream_t st) {
  init_beam_kernel<<<bs.B, 256, 0, st>>>(bs, mr, S0);
  AMUN_CHECK_LAUNCH();
}

// ================================================================ select

__device__ __forceinline__ double combine_models(double l0, const double *lm, int n) {
  // search.py:67-72 mean about the first member: first + mean(stack - first)
  if (n == 1) return l0;
  double acc = 0.0;
  for (int m = 0; m < n; ++m) acc += (lm[m] - l0);
  return l0 + acc / (double)n;
}

constexpr int kNoTok = 0x7fffffff;

// A lane's sorted (best-first) list of up to KMAX candidate keys.
template <int KMAX>
struct LaneList {
  double v[KMAX];
  int t[KMAX], p[KMAX];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {
      v[i] = -INFINITY;
      t[i] = kNoTok;
      p[i] = kNoTok;
    }
  }
  // insertion by compare-exchange down the list (registers only)
  __device__ __forceinline__ void push(Key c, int kk) {
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {
      if (i < kk && key_better(c.v, c.tok, c.par, v[i], t[i], p[i])) {
        double tv = v[i];
        int tt = t[i], tp = p[i];
        v[i] = c.v;
        t[i] = c.tok;
        p[i] = c.par;
        c = Key{tv, tt, tp};
      }
    }
  }
  __device__ __forceinline__ Key get(int h) const {
    Key k{-INFINITY, kNoTok, kNoTok};
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i == h) k = Key{v[i], t[i], p[i]};
    return k;
  }
};

// kk best keys of the union of the warp's lane lists, in order; out(j, key)
// is called by every lane with the warp-uniform j-th key.
template <int KMAX, class Out>
__device__ __forceinline__ void warp_merge(const LaneList<KMAX> &L, int kk, Out out) {
  int h = 0;
  __syncwarp();  // lanes reconverge after the lane-divergent scans: plain shuffles below
  for (int j = 0; j < kk; ++j) {
    Key mine = L.get(h);
    Key best = warp_best(mine);
    if (best.tok != kNoTok && mine.tok == best.tok && mine.par == best.par) ++h;
    out(j, best);
  }
}

// Warp-cooperative exact top-kk of candidates get(0..n-1) (entries with
// tok < 0 are skipped) in (value desc, tok asc, par asc) order; out(j, key)
// is called by every lane with the warp-uniform j-th key (tok == kNoTok when
// fewer than kk candidates exist).  (tok, par) pairs must be unique.
// KMAX > 0: per-lane register lists (kk <= KMAX) then a kk-round warp merge;
// KMAX == 0: general kk-pass scan (any kk).
template <int KMAX, class Get, class Out>
__device__ __forceinline__ void warp_topk(int n, int kk, Get get, Out out) {
  const int lane = threadIdx.x % 32;
  if constexpr (KMAX > 0) {
    LaneList<KMAX> L;
    L.init();
    Key worst{-INFINITY, kNoTok, kNoTok};
    // fetch 8 candidates per lane before inserting any: the loads are
    // independent, so their latency overlaps instead of serialising.  The
    // insertion loop stays rolled (code size: this kernel runs once per step
    // and would otherwise thrash the instruction cache).
    for (int e0 = lane; e0 < n; e0 += 32 * 8) {
      Key c[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int e = e0 + 32 * u;
        c[u] = e < n ? get(e) : Key{-INFINITY, -1, -1};
      }
#pragma unroll 1
      for (int u = 0; u < 8; ++u) {
        const Key cu = c[u];
        if (cu.tok >= 0 && key_better(cu.v, cu.tok, cu.par, worst.v, worst.tok, worst.par)) {
          L.push(cu, kk);
          worst = L.get(kk - 1);
        }
      }
    }
    int h = 0;
    __syncwarp();
    for (int j = 0; j < kk; ++j) {
      Key mine = L.get(h);
      Key best = warp_best(mine);
      if (best.tok != kNoTok && mine.tok == best.tok && mine.par == best.par) ++h;
      out(j, best);
    }
  } else {
    Key last{INFINITY, -1, -1};
    for (int j = 0; j < kk; ++j) {
      Key best{-INFINITY, kNoTok, kNoTok};
      for (int e = lane; e < n; e += 32) {
        Key c = get(e);
        if (c.tok < 0) continue;
        if (key_better(last.v, last.tok, last.par, c.v, c.tok, c.par) &&
            key_better(c.v, c.tok, c.par, best.v, best.tok, best.par))
          best = c;
      }
      best = warp_best(best);
      out(j, best);
      last = best;
    }
  }
}

template <int KMAX, bool FUSED>
__global__ void __launch_bounds__(256) select_kernel(SelectArgs sa, BeamState bs, ModelRows mr) {
  extern __shared__ unsigned char smraw[];
  const int k = bs.k;
  double *ch_v = reinterpret_cast<double *>(smraw);     // [k]
  int *ch_tok = reinterpret_cast<int *>(ch_v + k);      // [k]
  int *ch_par = ch_tok + k;                             // [k]
  int *fin_par = ch_par + k;                            // [k] finished this step: parent
  int *fin_idx = fin_par + k;                           // [k]
  // phase-1 row candidates [k][kk] (log-prob, token), consumed by phase 2
  double *c_lp = reinterpret_cast<double *>(smraw + (((size_t)k * (sizeof(double) + 4 * sizeof(int)) + 15) & ~size_t(15)));
  int *c_tok = reinterpret_cast<int *>(c_lp + (size_t)k * sa.kk);
  // the beam's scores, staged during the row phase for the sentence top-k
  double *s_sc = reinterpret_cast<double *>((reinterpret_cast<uintptr_t>(c_tok + (size_t)k * sa.kk) + 7) & ~uintptr_t(7));
  __shared__ int s_nch, s_newna, s_nfin;

  const CtaClock kclk(sa.kt);
  long long clk0 = clock64();
  const int b = blockIdx.x;
  if (bs.done[b]) return;
  const int t = bs.steps[b];  // this sentence's step index (graph-replay safe: no host-side t)
  // the update phase's per-sentence scalars, read now (their latency overlaps
  // the row phase instead of serialising thread 0's update)
  int fin_n0 = 0, cap0 = 0;
  double best_fin0 = 0.0;
  if (threadIdx.x == 0) {
    fin_n0 = bs.fin_n[b];
    best_fin0 = bs.best_fin[b];
    cap0 = bs.cap[b];
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  const int na = bs.n_act[b];
  const int kk = sa.kk;
  for (int i = threadIdx.x; i < na; i += blockDim.x) s_sc[i] = bs.score[b * k + i];
  const int n_models = mr.n_models;

  // ---- phase 1: per active row, log-sum-exp and top-kk candidates
  for (int i = warp; i < na; i += nw) {
    const int r = b * k + i;
    double *out_lp = c_lp + (size_t)i * kk;
    int *out_tok = c_tok + (size_t)i * kk;
    if constexpr (FUSED) {
      // per-tile partial (max, sum) pairs, kept in registers (<= 8 per lane);
      // ensembles fused in the logit kernel: one set per member, and the
      // candidates carry the member sum of the logits, so the ensemble
      // log-prob mean_m(logit_m - lse_m) (search.py:67-72) is
      // (sum_m logit_m - sum_m lse_m) / nm
      constexpr int kPT = 8;
      const int n = sa.ntiles * kk;
      const float *cv = sa.cval + (long long)r * n;
      const int *ct = sa.ctok + (long long)r * n;
      // tile maxima (each tile list is sorted best-first) are loaded with the
      // first member's partials: independent loads, one round trip
      float tmax[kPT];
#pragma unroll
      for (int u = 0; u < kPT; ++u) {
        const int tt = lane + 32 * u;
        tmax[u] = tt < sa.ntiles ? __ldg(cv + tt * kk) : -INFINITY;
      }
      double lse = 0.0;
      for (int mi = 0; mi < sa.nm_fused; ++mi) {
        const float *pmax = sa.pmax + mi * sa.pm_stride, *psum = sa.psum + mi * sa.pm_stride;
        float pm[kPT], ps[kPT];
        float mx = -INFINITY;
#pragma unroll
        for (int u = 0; u < kPT; ++u) {
          const int tt = lane + 32 * u;
          const bool ok = tt < sa.ntiles;
          pm[u] = ok ? __ldg(pmax + (long long)r * sa.ntiles + tt) : -INFINITY;
          ps[u] = ok ? __ldg(psum + (long long)r * sa.ntiles + tt) : 0.f;
        }
        for (int tt = lane + 32 * kPT; tt < sa.ntiles; tt += 32) mx = fmaxf(mx, pmax[(long long)r * sa.ntiles + tt]);
#pragma unroll
        for (int u = 0; u < kPT; ++u) mx = fmaxf(mx, pm[u]);
        mx = warp_max(mx);
        // exp(pm - mx) <= 1 in fp32 (1-ulp expf), products summed in f64
        double s = 0.0;
#pragma unroll
        for (int u = 0; u < kPT; ++u) s += (double)(ps[u] * expf(pm[u] - mx));
        for (int tt = lane + 32 * kPT; tt < sa.ntiles; tt += 32) {
          long long o = (long long)r * sa.ntiles + tt;
          s += (double)(psum[o] * expf(pmax[o] - mx));
        }
        s = warp_sum_d(s);
        lse += (double)mx + log(s);
      }
      auto emit = [&](int j, const Key &bk) {
        if (lane == 0) {
          bool none = bk.tok == kNoTok;
          // ordering by logit == by logit - lse
          out_lp[j] = none ? -INFINITY : (sa.nm_fused == 1 ? bk.v - lse : (bk.v - lse) / sa.nm_fused);
          out_tok[j] = none ? -1 : bk.tok;
        }
      };
      if constexpr (KMAX > 0) {
        if (sa.ntiles <= 32 * kPT) {
          // Threshold filter: every tile list is sorted best-first, so the
          // kk-th best tile maximum (thr) is a lower bound on the row's kk-th
          // best logit; only tile prefixes >= thr can hold the row's top-kk.
          float lv = INFINITY;
          int lt = -1;
          for (int p = 0; p < kk; ++p) {
            float bv = -INFINITY;
            int bt = 0x7fffffff;
#pragma unroll
            for (int u = 0; u < kPT; ++u) {
              const int tt = lane + 32 * u;
              const float x = tmax[u];
              const bool below = (x < lv) || (x == lv && tt > lt);
              if (below && (x > bv || (x == bv && tt < bt))) {
                bv = x;
                bt = tt;
              }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
              const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
              const int ot = __shfl_xor_sync(0xffffffffu, bt, o);
              if (ov > bv || (ov == bv && ot < bt)) {
                bv = ov;
                bt = ot;
              }
            }
            lv = bv;
            lt = bt;
          }
          const float thr = lv;  // -inf when fewer than kk tiles have candidates
          LaneList<KMAX> L;
          L.init();
          unsigned scan = 0;  // tiles of this lane whose maximum reaches thr
#pragma unroll
          for (int u = 0; u < kPT; ++u)
            if (lane + 32 * u < sa.ntiles && tmax[u] >= thr) scan |= 1u << u;
#pragma unroll 1
          for (; scan; scan &= scan - 1) {  // rolled: keeps the kernel small
            const int tt = lane + 32 * (__ffs(scan) - 1);
            // the tile's list in batches of independent loads (the whole
            // list for beams <= 8, 4 at a time above: whole lists cost more
            // than they save at beam 12), the prefix >= thr inserted (was:
            // one dependent load per candidate)
            constexpr int kB = KMAX <= 8 ? KMAX : 4;
            for (int j0 = 0; j0 < kk; j0 += kB) {
              float xs[kB];
              int ts[kB];
#pragma unroll
              for (int u = 0; u < kB; ++u) {
                xs[u] = j0 + u < kk ? __ldg(cv + tt * kk + j0 + u) : -INFINITY;
                ts[u] = j0 + u < kk ? __ldg(ct + tt * kk + j0 + u) : -1;
              }
              bool more = true;
#pragma unroll
              for (int u = 0; u < kB; ++u) {
                if (!more || ts[u] < 0 || xs[u] < thr) {
                  more = false;
                } else {
                  L.push(Key{(double)xs[u], ts[u], 0}, kk);
                }
              }
              if (!more) break;
            }
          }
          warp_merge<KMAX>(L, kk, emit);
        } else {
          warp_topk<KMAX>(n, kk, [&](int e) { return Key{(double)cv[e], ct[e], 0}; }, emit);
        }
      } else {
        warp_topk<KMAX>(n, kk, [&](int e) { return Key{(double)cv[e], ct[e], 0}; }, emit);
      }
    } else {
      const int *ids = sa.sl_ids ? sa.sl_ids + sa.sl_off[b] : nullptr;
      const int ncols = sa.sl_ids ? sa.sl_len[b] : sa.V;
      double lse[kMaxModels];
      for (int m = 0; m < n_models; ++m) {
        const float *Lr = sa.L[m] + (long long)r * sa.ldl;
        float mx = -INFINITY;
        for (int c = lane; c < ncols; c += 32) mx = fmaxf(mx, Lr[ids ? ids[c] : c]);
        mx = warp_max(mx);
        double s = 0.0;
        for (int c = lane; c < ncols; c += 32) s += exp((double)Lr[ids ? ids[c] : c] - (double)mx);
        s = warp_sum_d(s);
        lse[m] = (double)mx + log(s);
      }
      warp_topk<KMAX>(
          ncols, kk,
          [&](int c) {
            int g = ids ? ids[c] : c;
            double lm[kMaxModels];
            for (int m = 0; m < n_models; ++m) lm[m] = (double)sa.L[m][(long long)r * sa.ldl + g] - lse[m];
            return Key{combine_models(lm[0], lm, n_models), g, 0};
          },
          [&](int j, const Key &bk) {
            if (lane == 0) {
              bool none = bk.tok == kNoTok;
              out_lp[j] = none ? -INFINITY : bk.v;
              out_tok[j] = none ? -1 : bk.tok;
            }
          });
    }
  }
  __syncthreads();
  if (sa.dbg && threadIdx.x == 0) { const long long c = clock64(); atomicAdd(sa.dbg + 0, (unsigned long long)(c - clk0)); clk0 = c; }

  // ---- phase 2: sentence top-k over na*kk candidates, key (score desc,
  // token asc, parent asc) with f64 scores (search.py:169-170, :75-91)
  if (warp == 0 && na * kk <= 32) {
    // one candidate per lane: its rank is the number of candidates that beat
    // it in the total (score desc, token asc, parent asc) order; ranks < k
    // are the selection, in order (no lists, no divergent shuffles)
    const int n = na * kk;
    Key me{-INFINITY, -1, -1};
    if (lane < n) {
      const int par = lane / kk;
      me = Key{s_sc[par] + c_lp[lane], c_tok[lane], par};
    }
    const bool valid = lane < n && me.tok >= 0;
    int rank = 0, nvalid = 0;
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const double ov = __shfl_sync(0xffffffffu, me.v, j);
      const int ot = __shfl_sync(0xffffffffu, me.tok, j);
      const int op = __shfl_sync(0xffffffffu, me.par, j);
      if (j < n && ot >= 0) {
        ++nvalid;
        rank += key_better(ov, ot, op, me.v, me.tok, me.par);
      }
    }
    if (valid && rank < k) {
      ch_v[rank] = me.v;
      ch_tok[rank] = me.tok;
      ch_par[rank] = me.par;
    }
    if (lane == 0) s_nch = min(k, nvalid);
  } else if (warp == 0) {
    const int n = na * kk;
    const double *clp = c_lp;
    const int *ctk = c_tok;
    int nch = 0;
    warp_topk<KMAX>(
        n, k,
        [&](int e) {
          int par = e / kk;
          return Key{s_sc[par] + clp[e], ctk[e], par};
        },
        [&](int j, const Key &bk) {
          if (bk.tok == kNoTok) return;
          if (lane == 0) {
            ch_v[j] = bk.v;
            ch_tok[j] = bk.tok;
            ch_par[j] = bk.par;
          }
          nch = j + 1;
        });
    if (lane == 0) s_nch = nch;
  }
  __syncthreads();
  if (sa.dbg && threadIdx.x == 0) { const long long c = clock64(); atomicAdd(sa.dbg + 1, (unsigned long long)(c - clk0)); clk0 = c; }

  // ---- phase 3: beam update (search.py:172-198)
  if (threadIdx.x == 0) {
    const int nch = s_nch;
    int newna = 0, nfin = 0;
    double best_new = -INFINITY;
    const int rowbase = (b * bs.cap_max + t) * k;
    for (int j = 0; j < nch; ++j) {
      if (ch_tok[j] == 0) {  // EOS_ID -> finished list (unbounded in the reference)
        const int idx = fin_n0++;
        long long fo = (long long)b * bs.fin_cap + idx;
        bs.fin_score[fo] = ch_v[j];
        bs.fin_t[fo] = t;
        bs.fin_par[fo] = ch_par[j];
        if (ch_v[j] > best_fin0) best_fin0 = ch_v[j];
        fin_par[nfin] = ch_par[j];
        fin_idx[nfin] = idx;
        ++nfin;
      } else {
        int slot = newna++;
        bs.bp_tok[rowbase + slot] = ch_tok[j];
        bs.bp_par[rowbase + slot] = ch_par[j];
        if (ch_v[j] > best_new) best_new = ch_v[j];
        // reuse ch_* arrays in place: slot <= j always
        ch_v[slot] = ch_v[j];
        ch_tok[slot] = ch_tok[j];
        ch_par[slot] = ch_par[j];
      }
    }
    if (nfin > 0) {
      bs.fin_n[b] = fin_n0;
      bs.best_fin[b] = best_fin0;
    }
    bs.steps[b] = t + 1;
    int done = 0;
    if (newna == 0) {
      done = 1;  // search.py:186-187 (beam left as it was)
    } else {
      bs.n_act[b] = newna;
      for (int i = 0; i < newna; ++i) {
        bs.score[b * k + i] = ch_v[i];
        bs.tok[b * k + i] = ch_tok[i];
        if (bs.qrow) bs.qrow[b * k + i] = b * k + ch_par[i];
      }
      if (fin_n0 > 0 && best_new <= best_fin0) done = 1;  // search.py:195-198
    }
    if (t + 1 >= cap0) done = 1;
    if (done) {
      bs.done[b] = 1;
      atomicAdd(bs.n_done, 1);
    }
    s_newna = newna;
    s_nfin = nfin;
  }
  __syncthreads();
  if (sa.dbg && threadIdx.x == 0) { const long long c = clock64(); atomicAdd(sa.dbg + 2, (unsigned long long)(c - clk0)); clk0 = c; }

  // ---- phase 4: gather next-step decoder rows [E_trg[y] | . | s'_parent]
  // (float4 granules, 8 independent loads in flight per thread)
  const int newna = s_newna, nfin = s_nfin;
  for (int m = 0; m < n_models; ++m) {
    const RowDims md = mr.dim[m];
    const bool vec = (md.de % 4 == 0) && (md.dh % 4 == 0) && (md.ldxs % 4 == 0) && (md.s_off % 4 == 0);
    float *XS = mr.XS[m];
    __half *XSh = mr.XSh ? mr.XSh[m] : nullptr;
    __half *XSl = mr.XSl ? mr.XSl[m] : nullptr;
    const float *Sn = mr.Sn[m];
    const float *E = mr.E_trg[m];
    if (vec) {
      // granules [0, qe) are y's, [qe, qrow) the state's; without y rows the
      // loop starts at the state (y0 = qe granules skipped per row)
      const int qe = md.de / 4, y0 = md.y ? 0 : qe, qrow = (md.de + md.dh) / 4 - y0;
      const int total = newna * qrow;
      for (int base = threadIdx.x; base < total; base += 8 * blockDim.x) {
        float4 v[8];
        long long dst[8], dsth[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int idx = base + u * blockDim.x;
          dst[u] = -1;
          if (idx < total) {
            const int i = idx / qrow, c4 = idx - i * qrow + y0;
            const long long ro = (long long)(b * k + i) * md.ldxs;
            const long long roh = (long long)(b * k + i) * md.ldxh;
            if (c4 < qe) {
              v[u] = __ldg(reinterpret_cast<const float4 *>(E + (long long)ch_tok[i] * md.de) + c4);
              dst[u] = ro + 4 * c4;
              dsth[u] = roh + 4 * c4;
            } else {
              v[u] = __ldg(reinterpret_cast<const float4 *>(Sn + (long long)(b * k + ch_par[i]) * md.dh) + (c4 - qe));
              dst[u] = ro + md.s_off + 4 * (c4 - qe);
              dsth[u] = roh + md.s_off + md.hpad + 4 * (c4 - qe);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (dst[u] < 0) continue;
          *reinterpret_cast<float4 *>(XS + dst[u]) = v[u];
          if (XSh && md.split) {  // 4 halves = 8 bytes (ldxh, hpad and s_off are multiples of 4)
            __half h4[4], l4[4];
            split_h(v[u].x, h4[0], l4[0]);
            split_h(v[u].y, h4[1], l4[1]);
            split_h(v[u].z, h4[2], l4[2]);
            split_h(v[u].w, h4[3], l4[3]);
            *reinterpret_cast<uint2 *>(XSh + dsth[u]) = *reinterpret_cast<const uint2 *>(h4);
            *reinterpret_cast<uint2 *>(XSl + dsth[u]) = *reinterpret_cast<const uint2 *>(l4);
          }
        }
      }
    } else {
      for (int i = 0; i < newna; ++i) {
        const long long ro = (long long)(b * k + i) * md.ldxs;
        const long long roh = (long long)(b * k + i) * md.ldxh;
        const float *ey = E + (long long)ch_tok[i] * md.de;
        const float *sp = Sn + (long long)(b * k + ch_par[i]) * md.dh;
        for (int c = threadIdx.x; c < (md.y ? md.de : 0); c += blockDim.x) {
          XS[ro + c] = ey[c];
          store_split(XSh, XSl, roh + c, ey[c]);
        }
        for (int c = threadIdx.x; c < md.dh; c += blockDim.x) {
          XS[ro + md.s_off + c] = sp[c];
          store_split(XSh, XSl, roh + md.s_off + md.hpad + c, sp[c]);
        }
      }
    }
    if (mr.fin_states) {
      for (int i = 0; i < nfin; ++i) {
        float *dst = mr.fin_states[m] + ((long long)b * bs.fin_cap + fin_idx[i]) * md.dh;
        const float *sp = Sn + (long long)(b * k + fin_par[i]) * md.dh;
        for (int c = threadIdx.x; c < md.dh; c += blockDim.x) dst[c] = sp[c];
      }
    }
  }
  __syncthreads();
  if (sa.dbg && threadIdx.x == 0) { atomicAdd(sa.dbg + 3, (unsigned long long)(clock64() - clk0)); atomicAdd(sa.dbg + 4, 1ull); }
  kclk.done();
}

template <int KMAX, bool FUSED>
static void launch_select_t(const SelectArgs &sa, const BeamState &bs, const ModelRows &mr, size_t smem,
                            cudaStream_t st) {
  auto kern = select_kernel<KMAX, FUSED>;
  if (smem > 48 * 1024) smem_optin(reinterpret_cast<const void *>(kern));
  SelectArgs sk = sa;
  sk.kt = ktime_ptr();
  // one warp per beam row in the row phase: beams <= 8 run 5..8-warp CTAs
  // (k = 5: 160 threads, so three CTAs share an SM); AMUN_SELECT_THREADS overrides
  static const int forced = [] {
    const char *e = getenv("AMUN_SELECT_THREADS");
    return e ? atoi(e) : 0;
  }();
  const int threads = forced > 0 ? std::min(256, std::max(32, forced / 32 * 32))
                                 : (bs.k <= 8 ? 32 * std::max(4, bs.k) : 256);
  kern<<<bs.B, threads, smem, st>>>(sk, bs, mr);
  AMUN_CHECK_LAUNCH();
}

void launch_select(const SelectArgs &sa, const BeamState &bs, const ModelRows &mr, cudaStream_t st) {
  if (mr.n_models > kMaxModels) throw Error(4, "at most 8 ensemble members are supported on the device path");
  size_t smem = (((size_t)bs.k * (sizeof(double) + 4 * sizeof(int)) + 15) & ~size_t(15)) +
                (size_t)bs.k * sa.kk * (sizeof(double) + sizeof(int)) + 8 + (size_t)bs.k * sizeof(double);
  const int need = std::max(bs.k, sa.kk);  // list sizes used in phases 1 and 2
  if (sa.fused) {
    if (need <= 1) launch_select_t<1, true>(sa, bs, mr, smem, st);
    else if (need <= 4) launch_select_t<4, true>(sa, bs, mr, smem, st);
    else if (need <= 5) launch_select_t<5, true>(sa, bs, mr, smem, st);
    else if (need <= 8) launch_select_t<8, true>(sa, bs, mr, smem, st);
    else if (need <= 12) launch_select_t<12, true>(sa, bs, mr, smem, st);
    else launch_select_t<16, true>(sa, bs, mr, smem, st);
  } else {
    if (need <= 8) launch_select_t<8, false>(sa, bs, mr, smem, st);
    else if (need <= 16) launch_select_t<16, false>(sa, bs, mr, smem, st);
    else launch_select_t<0, false>(sa, bs, mr, smem, st);
  }
}

// ================================================================ hook logp

__global__ void logp_rows_kernel(const float *L, int ldl, int V, const int *sl, int n_sl, double *logp) {
  const int r = blockIdx.x;
  const int n = sl ? n_sl : V;
  const float *Lr = L + (long long)r * ldl;
  __shared__ float s_mx[32];
  __shared__ double s_sum[32];
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nw = blockDim.x / 32;
  float mx = -INFINITY;
  for (int c = threadIdx.x; c < n; c += blockDim.x) mx = fmaxf(mx, Lr[sl ? sl[c] : c]);
  mx = warp_max(mx);
  if (lane == 0) s_mx[warp] = mx;
  __syncthreads();
  mx = -INFINITY;
  for (int w = 0; w < nw; ++w) mx = fmaxf(mx, s_mx[w]);
  double s = 0.0;
  for (int c = threadIdx.x; c < n; c += blockDim.x) s += exp((double)Lr[sl ? sl[c] : c] - (double)mx);
  s = warp_sum_d(s);
  if (lane == 0) s_sum[warp] = s;
  __syncthreads();
  s = 0.0;
  for (int w = 0; w < nw; ++w) s += s_sum[w];
  const double lse = (double)mx + log(s);
  for (int c = threadIdx.x; c < n; c += blockDim.x) logp[(long long)r * n + c] = (double)Lr[sl ? sl[c] : c] - lse;
}

void launch_logp_rows(const float *L, int ldl, int R, int V, const int *sl, int n_sl, double *logp,
                      cudaStream_t st) {
  logp_rows_kernel<<<R, 256, 0, st>>>(L, ldl, V, sl, n_sl, logp);
  AMUN_CHECK_LAUNCH();
}

}  // namespace amun

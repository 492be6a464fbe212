// Logit projection, rows layout: the hypothesis rows are the MMA's M (one
// TMEM lane per row), the vocabulary its N (256 logits per work unit), so
// every epilogue thread owns ONE row and reads its logits straight out of
// TMEM with tcgen05.ld -- no transpose through shared memory, no barriers
// between epilogue warps, no cross-thread merges.  Fused like the swap-AB
// kernel (logits_tc.cu): nnet.py:161 logits + tensor.py:79-92 log-softmax
// partials + search.py:169-170 per-row top-k; full logits never reach HBM.
//
// Per work unit (128-row tile, 256-vocab tile) a thread keeps a running
// (max, sum exp) and a register top-KK list over its row's 256 logits and
// writes one partial per (row, 256-vocab tile) -- the layout the select
// kernel merges (kernels.cu select phase 1).
//
// Precision: 3xFP16 (hi*hi + hi*lo + lo*hi, fp32 accumulation in TMEM) on
// tcgen05.mma kind::f16, cta_group::1, M = 128, N = 256, exactly as the other
// tensor-core kernels (see logits_tc.cu).
//
// Clusters: the C CTAs of a cluster take the C row tiles of the same vocab
// tile in lockstep and share its weight tile through TMA multicast (each CTA
// fetches 1/C of the 32-row weight boxes for everyone), so the weights cross
// L2 once per vocab tile instead of once per row tile.  Stage reuse is
// cluster-wide: every CTA's MMA commit arrives on the empty barrier of every
// CTA (multicast commit), so a stage is refilled only after all C CTAs have
// consumed it.
#include "common.cuh"
#include "logits_tc.cuh"
#include "tc_common.cuh"

namespace amun {

namespace {

constexpr int rBK = 32;                           // fp16 K elements per 64-byte swizzled row (SWIZZLE_64B)
constexpr int rRowB = rBK * 2;
#ifndef AMUN_ROWS_STAGES
#define AMUN_ROWS_STAGES 3
#endif
#ifndef AMUN_ROWS_EPI
#define AMUN_ROWS_EPI 4
#endif
constexpr int rStages = AMUN_ROWS_STAGES;
constexpr int rTM = 128;                          // rows per CTA tile (TMEM lanes)
constexpr int rTN = 256;                          // vocabulary entries per unit (MMA N)
constexpr int rBoxV = 32;                         // vocabulary rows per (multicast) weight box
constexpr int rAB = rTM * rRowB;                  // 8 KB: one of hi / lo activation tiles
constexpr int rBB = rTN * rRowB;                  // 16 KB: one of hi / lo weight tiles
constexpr int rStageB = 2 * rAB + 2 * rBB;        // 48 KB
constexpr int rEpiGroups = AMUN_ROWS_EPI;         // epilogue warpgroups (2: one per accumulator buffer; 4: one per buffer half)
constexpr int rBufGroups = rEpiGroups / 2;        // warpgroups draining one accumulator buffer
constexpr int rTile = rTN / 2;                    // vocabulary per partial (one warpgroup's half of a unit)
constexpr int rStash = 32;                        // floats per thread in the candidate stash (rotated by 4 lane)
constexpr int rSmem = rStages * rStageB + rEpiGroups * rTM * rStash * 4 + rEpiGroups * 4 * 32 * 4 + 1024 + 256;
constexpr int rThreads = 64 + 128 * rEpiGroups;   // warp 0 TMA, warp 1 MMA, then the epilogue warpgroups
static_assert(rSmem <= 232448, "shared memory per CTA");
constexpr float kLog2e = 1.4426950408889634f;

// Register-resident top-KK list ordered by (logit desc, token asc).
template <int KK>
struct Top {
  float v[KK];
  int t[KK];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < KK; ++i) {
      v[i] = -INFINITY;
      t[i] = 0x7fffffff;
    }
  }
  // Insertion of (x, n) where n is larger than every token in the list (a
  // thread scans its columns in increasing order): x enters before the
  // first entry it strictly exceeds, so an equal value keeps the earlier
  // token first.  Every slot's update depends only on the old list (one
  // compare per slot, then selects): no serial chain through the slots.
  __device__ __forceinline__ void insert(float x, int n) {
    bool gt[KK];
#pragma unroll
    for (int i = 0; i < KK; ++i) gt[i] = x > v[i];
#pragma unroll
    for (int i = KK - 1; i > 0; --i) {
      v[i] = gt[i - 1] ? v[i - 1] : (gt[i] ? x : v[i]);
      t[i] = gt[i - 1] ? t[i - 1] : (gt[i] ? n : t[i]);
    }
    v[0] = gt[0] ? x : v[0];
    t[0] = gt[0] ? n : t[0];
  }
};

// Lower bound on the KK-th largest of x[0..31]: the KK-th largest of G group
// maxima (G = 8 groups of 4 for KK <= 8, 16 groups of 2 above) -- distinct
// elements, so at least KK elements reach it.
template <int KK>
__device__ __forceinline__ float first_chunk_bound(const float (&x)[32]) {
  constexpr int G = KK <= 8 ? 8 : 16;
  constexpr int W = 32 / G;
  float g[G];
#pragma unroll
  for (int j = 0; j < G; ++j) {
    g[j] = x[W * j];
#pragma unroll
    for (int i = 1; i < W; ++i) g[j] = fmaxf(g[j], x[W * j + i]);
  }
  // KK bubble passes float the KK largest to the front, in order
#pragma unroll
  for (int p = 0; p < KK; ++p)
#pragma unroll
    for (int j = G - 1; j > p; --j) {
      const float hi = fmaxf(g[j - 1], g[j]), lo = fminf(g[j - 1], g[j]);
      g[j - 1] = hi;
      g[j] = lo;
    }
  return g[KK - 1];
}

template <int KK>
__global__ void __launch_bounds__(rThreads, 1)
    logits_rows_kernel(const __grid_constant__ CUtensorMap tA_hi, const __grid_constant__ CUtensorMap tA_lo,
                       const __grid_constant__ CUtensorMap tB_hi, const __grid_constant__ CUtensorMap tB_lo,
                       LogitTcArgs a, int C) {
  const CtaClock clk(a.kt);
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = tc::align_smem<1024>(smem_raw);
  float *stash = reinterpret_cast<float *>(smem + rStages * rStageB);
  float *bias_s = stash + rEpiGroups * rTM * rStash;  // [epilogue warp][32] the chunk's biases
  uint64_t *full = reinterpret_cast<uint64_t *>(bias_s + rEpiGroups * 4 * 32);
  uint64_t *empty = full + rStages;
  uint64_t *tfull = empty + rStages;  // [2] accumulator buffers
  uint64_t *tempty = tfull + 2;       // [2]
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int crank = C > 1 ? (int)tc::cluster_rank() : 0;
  const int cl = blockIdx.x / C, ncl = gridDim.x / C;
  const int nvt = (a.N + rTN - 1) / rTN;
  const int nrt = (a.M + rTM - 1) / rTM;
  const int G = (nrt + C - 1) / C;  // row-tile groups of C
  const int units = nvt * G;
  const int upc = (units + ncl - 1) / ncl;  // contiguous units per cluster
  const int u_begin = cl * upc, u_end = min(units, u_begin + upc);
  const int nk = (a.K + rBK - 1) / rBK;
  const uint16_t cmask = (uint16_t)((1u << C) - 1u);
  // microbenchmark: per-unit clock64 stamps of CTA 0 (slot 8 u + k)
  auto stamp = [&](int u, int k) {
    if (a.debug_clock && blockIdx.x == 0 && u - u_begin < 64) a.debug_clock[(u - u_begin) * 8 + k] = clock64();
  };

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < rStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], C);  // one MMA commit from every CTA of the cluster
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 4 * rBufGroups);  // the epilogue warps draining this buffer
    }
    tc::fence_barrier_init();
    tc::tma_prefetch(&tA_hi);
    tc::tma_prefetch(&tA_lo);
    tc::tma_prefetch(&tB_hi);
    tc::tma_prefetch(&tB_lo);
  }
  if (warp == 1) tc::tmem_alloc<512>(tslot);
  tc::tc_fence_before();
  __syncthreads();
  if (C > 1) tc::cluster_sync();  // peers' barriers initialised before any multicast lands
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ---------------- TMA producer: own activation rows + 1/C of the weight boxes for the whole cluster
    if (lane == 0) {
      int it = 0;
      for (int u = u_begin; u < u_end; ++u) {
        const int vt = u / G, rt = (u % G) * C + crank;
        const int v0 = vt * rTN, r0 = rt * rTM;
        stamp(u, 4);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % rStages;
          if (it >= rStages) tc::mbar_wait(&empty[s], ((it / rStages) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&full[s], rStageB);
          uint8_t *st = smem + s * rStageB;
          const int kx = kb * rBK;
          tc::tma_load_2d(st, &tA_hi, &full[s], kx, r0);
          tc::tma_load_2d(st + rAB, &tA_lo, &full[s], kx, r0);
          for (int j = crank; j < rTN / rBoxV; j += C) {
            uint8_t *bh = st + 2 * rAB + j * rBoxV * rRowB;
            if (C > 1) {
              tc::tma_load_2d_mc(bh, &tB_hi, &full[s], kx, v0 + j * rBoxV, cmask);
              tc::tma_load_2d_mc(bh + rBB, &tB_lo, &full[s], kx, v0 + j * rBoxV, cmask);
            } else {
              tc::tma_load_2d(bh, &tB_hi, &full[s], kx, v0 + j * rBoxV);
              tc::tma_load_2d(bh + rBB, &tB_lo, &full[s], kx, v0 + j * rBoxV);
            }
          }
        }
        stamp(u, 5);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread): two TMEM accumulator buffers
    // so the epilogue of unit t overlaps the mainloop of unit t + 1
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_f16(rTM, rTN);
      int it = 0, ti = 0;
      for (int u = u_begin; u < u_end; ++u, ++ti) {
        const int buf = ti & 1;
        const uint32_t acc = tmem + buf * rTN;
        if (ti >= 2) {
          tc::mbar_wait(&tempty[buf], ((ti >> 1) - 1) & 1);
          tc::tc_fence_after();
        }
        stamp(u, 0);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % rStages;
          tc::mbar_wait(&full[s], (it / rStages) & 1);
          tc::tc_fence_after();
          const uint32_t base = tc::smem_u32(smem + s * rStageB);
#pragma unroll
          for (int k2 = 0; k2 < rBK / 16; ++k2) {
            const uint32_t koff = k2 * 32;
            const uint64_t ah = tc::desc_kmajor_sw64(base + koff);
            const uint64_t al = tc::desc_kmajor_sw64(base + rAB + koff);
            const uint64_t bh = tc::desc_kmajor_sw64(base + 2 * rAB + koff);
            const uint64_t bl = tc::desc_kmajor_sw64(base + 2 * rAB + rBB + koff);
            const uint32_t acc0 = (kb | k2) != 0;
            tc::mma_f16(acc, ah, bh, idesc, acc0);
            tc::mma_f16(acc, ah, bl, idesc, 1);
            tc::mma_f16(acc, al, bh, idesc, 1);
          }
          if (C > 1)
            tc::mma_commit_mc(&empty[s], cmask);
          else
            tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(&tfull[buf]);
        stamp(u, 1);
      }
    }
  } else {
    // ---------------- epilogue: thread = one hypothesis row of the tile;
    // warpgroup eg drains accumulator buffer eg / 2 (every other unit) and
    // vocabulary half eg % 2 of it (4 warps per SM sub-partition hide the
    // latencies of the per-row reductions)
    const int eg = (warp - 2) / 4;
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    const int lrow = q * 32 + lane;
    const int bsel = eg / rBufGroups, h0 = eg % rBufGroups;
    float *my = stash + (eg * rTM + lrow) * rStash;
    const int rot = 4 * lane;  // stash element i of this thread lives at (i + rot) & 31: conflict-free STS.128
    int ti = 0;
    for (int u = u_begin; u < u_end; ++u, ++ti) {
      const int buf = ti & 1;
      if (buf != bsel) continue;
      for (int half = h0; half < 2; half += rBufGroups) {
      const int vt = u / G, rt = (u % G) * C + crank;
      const int v0 = vt * rTN + half * rTile;
      const int nt = vt * 2 + half;  // partial tile index (rTile-wide)
      const int m = rt * rTM + lrow;
      const bool live = m < a.M;
      // biases: lane j holds column vc + j of the coming chunk (prefetched a
      // chunk ahead), staged through a 32-float per-warp slot for broadcast
      float *bs = bias_s + (warp - 2) * 32;
      float breg = v0 + lane < a.N ? __ldg(a.bias + v0 + lane) : -INFINITY;
      const uint32_t *mrow = a.vmask ? a.vmask + (long long)(m / a.rows_per_sent) * a.mask_words : nullptr;
      if (half == h0) {
        tc::mbar_wait(&tfull[buf], (ti >> 1) & 1);
        tc::tc_fence_after();
      }
      if (lrow == 0 && half == 0) stamp(u, 2);
      float mx = -INFINITY, se = 0.f;
      Top<KK> top;
      top.init();
#pragma unroll 1
      for (int c = 0; c < rTile / 32; ++c) {
        const int vc = v0 + c * 32;
        // the row's shortlist word for these 32 columns (issued before the TMEM read)
        const uint32_t allow = mrow ? ((live && vc < a.N) ? __ldg(mrow + (vc >> 5)) : 0u) : ~0u;
        __syncwarp();  // the previous chunk's reads of the slot are done
        bs[lane] = breg;
        __syncwarp();
        if (c + 1 < rTile / 32) breg = vc + 32 + lane < a.N ? __ldg(a.bias + vc + 32 + lane) : -INFINITY;
        float x[32];
        tc::tmem_ld_32x32(tmem + buf * rTN + ((uint32_t)(q * 32) << 16) + half * rTile + c * 32, x);
        if (!live) {  // rows past the batch: nothing to reduce
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = -INFINITY;
        }
        if (c == rTile / 32 - 1 && half + rBufGroups >= 2) {  // this warp's TMEM reads done: hand the buffer back
          tc::tc_fence_before();
          __syncwarp();
          if (lane == 0) tc::mbar_arrive(&tempty[buf]);
        }
        {  // bias (smem broadcast; -inf past the vocabulary)
          const float4 *b4 = reinterpret_cast<const float4 *>(bs);
#pragma unroll
          for (int i4 = 0; i4 < 8; ++i4) {
            const float4 b = b4[i4];
            x[4 * i4] = fmaf(x[4 * i4], a.unscale, b.x);
            x[4 * i4 + 1] = fmaf(x[4 * i4 + 1], a.unscale, b.y);
            x[4 * i4 + 2] = fmaf(x[4 * i4 + 2], a.unscale, b.z);
            x[4 * i4 + 3] = fmaf(x[4 * i4 + 3], a.unscale, b.w);
          }
        }
        // shortlist (nnet.py:160-163): columns outside the row's sentence list do not exist
        if (mrow) {
#pragma unroll
          for (int i = 0; i < 32; ++i) x[i] = (allow >> i) & 1u ? x[i] : -INFINITY;
        }
        // running (max, sum exp(x - max)), ex2-based
        float cmx[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) cmx[j] = fmaxf(fmaxf(x[4 * j], x[4 * j + 1]), fmaxf(x[4 * j + 2], x[4 * j + 3]));
        const float cm = fmaxf(fmaxf(fmaxf(cmx[0], cmx[1]), fmaxf(cmx[2], cmx[3])),
                               fmaxf(fmaxf(cmx[4], cmx[5]), fmaxf(cmx[6], cmx[7])));
        if (cm > mx) {
          if (mx != -INFINITY) se *= tc::exp2f_approx((mx - cm) * kLog2e);
          mx = cm;
        }
        if (mx != -INFINITY) {
          const float ml = mx * kLog2e;
          float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
          for (int i = 0; i < 32; ++i) s4[i & 3] += tc::exp2f_approx(fmaf(x[i], kLog2e, -ml));
          se += (s4[0] + s4[1]) + (s4[2] + s4[3]);
        }
        // top-KK: only logits strictly above the running KK-th best can
        // enter (an equal value has a larger token); the first chunk uses a
        // lower bound on its own KK-th largest instead
        unsigned cand = 0;
        if (c == 0) {
          const float thr = first_chunk_bound<KK>(x);
#pragma unroll
          for (int i = 0; i < 32; ++i) cand |= (x[i] >= thr && x[i] != -INFINITY ? 1u : 0u) << i;
        } else {
          const float thr = top.v[KK - 1];
#pragma unroll
          for (int i = 0; i < 32; ++i) cand |= (x[i] > thr ? 1u : 0u) << i;
        }
        if (__any_sync(0xffffffffu, cand != 0)) {
#pragma unroll
          for (int i4 = 0; i4 < 8; ++i4)
            *reinterpret_cast<float4 *>(my + ((4 * i4 + rot) & 31)) =
                make_float4(x[4 * i4], x[4 * i4 + 1], x[4 * i4 + 2], x[4 * i4 + 3]);
#pragma unroll 1
          while (cand) {  // two candidates per trip: both stash loads in flight together
            const int i0 = __ffs(cand) - 1;
            cand &= cand - 1;
            const int i1 = cand ? __ffs(cand) - 1 : -1;
            cand &= cand - 1;
            const float x0 = my[(i0 + rot) & 31], x1 = my[((i1 < 0 ? i0 : i1) + rot) & 31];
            top.insert(x0, vc + i0);
            if (i1 >= 0) top.insert(x1, vc + i1);
          }
        }
      }
      if (lrow == 0 && half == 0) stamp(u, 3);
      if (live && nt < a.ntiles && !(a.debug_flags & 64)) {
        const long long o = (long long)m * a.ntiles + nt;
        a.pmax[o] = mx;
        a.psum[o] = se;
        const long long base = o * a.kk;
#pragma unroll
        for (int i = 0; i < KK; ++i)
          if (i < a.kk) {
            const bool ok = top.v[i] != -INFINITY;
            a.cval[base + i] = ok ? top.v[i] : -INFINITY;
            a.ctok[base + i] = ok ? (a.vid ? __ldg(a.vid + top.t[i]) : top.t[i]) : -1;
          }
      }
      }
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if (C > 1) tc::cluster_sync();  // no CTA leaves while a peer may still multicast into it
  clk.done();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc<512>(tmem);
}

// CTAs per launch: env AMUN_LOGIT_ROWS_CTAS (default 48) caps the CTAs; the
// units (vocab tiles x row-tile groups) are spread evenly over the clusters
int rows_target_ctas() {
  static int v = [] {
    const char *e = getenv("AMUN_LOGIT_ROWS_CTAS");
    return e ? std::max(1, atoi(e)) : 48;
  }();
  return v;
}

template <int KK>
void launch_t(const LogitTcMaps &maps, const LogitTcArgs &a, cudaStream_t st) {
  auto kern = logits_rows_kernel<KK>;
  static bool attr[64] = {};
  int dev = 0;
  AMUN_CUDA(cudaGetDevice(&dev));
  if (dev >= 64 || !attr[dev]) {
    AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, rSmem));
    AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    if (dev < 64) attr[dev] = true;
  }
  const int nrt = ceil_div(a.M, rTM);
  static const int cmax = [] {  // env AMUN_LOGIT_ROWS_CMAX caps the cluster size (weight-tile sharing)
    const char *e = getenv("AMUN_LOGIT_ROWS_CMAX");
    return e ? std::min(8, std::max(1, atoi(e))) : 8;
  }();
  const int C = std::min(cmax, nrt);
  const int units = ceil_div(a.N, rTN) * ceil_div(nrt, C);
  const int target = std::max(1, rows_target_ctas() / C);
  const int per = ceil_div(units, std::min(target, units));
  const int clusters = ceil_div(units, per);
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(clusters * C);
  cfg.blockDim = dim3(rThreads);
  cfg.dynamicSmemBytes = rSmem;
  cfg.stream = st;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = C;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  last_launch_ctas() = (int)cfg.gridDim.x;
  LogitTcArgs ak = a;
  ak.kt = ktime_ptr();
  AMUN_CUDA(cudaLaunchKernelEx(&cfg, kern, maps.a_hi, maps.a_lo, maps.b_hi, maps.b_lo, ak, C));
}

}  // namespace

LogitTcMaps make_logit_rows_maps(const __half *t_hi, const __half *t_lo, int R, int K, int ldt, const __half *w_hi,
                                 const __half *w_lo, int ldw, int V) {
  LogitTcMaps m;
  m.a_hi = make_tma_2d_f16(t_hi, K, R, ldt, rBK, rTM);
  m.a_lo = make_tma_2d_f16(t_lo, K, R, ldt, rBK, rTM);
  m.b_hi = make_tma_2d_f16(w_hi, K, V, ldw, rBK, rBoxV);
  m.b_lo = make_tma_2d_f16(w_lo, K, V, ldw, rBK, rBoxV);
  return m;
}

void launch_logits_rows(const LogitTcMaps &maps, const LogitTcArgs &a, cudaStream_t st) {
  if (a.nm != 1) throw Error(4, "launch_logits_rows: single-member launch");
  switch (a.kk) {
    case 1: launch_t<1>(maps, a, st); break;
    case 2: launch_t<2>(maps, a, st); break;
    case 3: launch_t<3>(maps, a, st); break;
    case 4: launch_t<4>(maps, a, st); break;
    case 5: launch_t<5>(maps, a, st); break;
    case 6: launch_t<6>(maps, a, st); break;
    case 7: case 8: launch_t<8>(maps, a, st); break;
    case 9: case 10: launch_t<10>(maps, a, st); break;
    case 11: case 12: launch_t<12>(maps, a, st); break;
    case 13: case 14: case 15: case 16: launch_t<16>(maps, a, st); break;
    default: throw Error(4, "tensor-core logit path supports beam <= 16");
  }
}

}  // namespace amun

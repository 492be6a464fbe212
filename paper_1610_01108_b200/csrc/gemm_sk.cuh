// Decoder-step GEMMs on the 5th-gen tensor cores: swap-AB, cluster split-K
// with a deterministic DSMEM reduction and the elementwise epilogue fused in.
//
//   C[R, N] = X[R, K] * W[K, N]   (+ epilogue: GRU gates / state update /
//                                    tanh / 3xTF32 re-split of the output)
//
// The decoder step has few rows (R = bucket x beam = 320) and wide weights
// (N = 3 d_h for GRU phase A, K = d_e + 3 d_h), so the weight is the MMA's
// A operand (M = 128 output features per CTA, one TMEM lane per feature)
// and the hypothesis rows are the MMA's N dimension (up to 320 rows held in
// TMEM columns, as one or two MMAs of N <= 256).  Every weight byte is read
// once per launch; the activation K-slice is re-read once per 128 features.
//
// Precision: 3xFP16 (W_hi X_hi + W_hi X_lo + W_lo X_hi on kind::f16, fp32
// accumulate in TMEM) over power-of-two scaled operands (common.cuh
// split_h), the FP32-equivalent scheme of logits_tc.cu; the reduction
// multiplies by the inverse scale before the epilogue.
//
// Grid (S, N/128) with clusters of (S, 1, 1): the S CTAs of a cluster split
// K and each holds a 128 x R fp32 partial in TMEM.  After the mainloop each
// CTA stages its partial in its own shared memory (reusing the pipeline
// buffers); CTA c of the cluster then sums rows [c R/S, (c+1) R/S) over the
// S partials in split order 0..S-1 through distributed shared memory and
// applies the epilogue.  The split count depends only on (N, K), never on R,
// so a row's result does not depend on its batch-mates, and the fixed
// summation order makes every launch bit-reproducible.  Nothing but the
// epilogue's outputs is written to global memory and there is no second
// launch.
#pragma once

#include <cuda.h>

#include "common.cuh"
#include "gemm_simt.cuh"  // epilogue functors
#include "logits_tc.cuh"  // make_tma_2d_f32
#include "tc_common.cuh"

namespace amun {

// Tile configuration: BK fp16 K elements per swizzled smem row (32 -> 64 B
// rows / SWIZZLE_64B, 64 -> 128 B rows / SWIZZLE_128B), pipeline depth, rows
// per pass (TMEM columns; the smem reduction buffer is PR x 512 B) and CG,
// the CTA group: 1 = one CTA per 128 features, 2 = a CTA pair per 256
// features (tcgen05 cta_group::2: M = 256, each CTA stages its 128 weight
// rows and HALF of the activation rows, the pair's tensor cores share both).
template <int BK_, int STAGES_, int PR_ = 320, int CG_ = 1>
struct SkCfg {
  static constexpr int kBK = BK_;
  static constexpr int kCG = CG_;
  static constexpr int kRowBytes = BK_ * 2;
  static constexpr int kPR = PR_;
  static constexpr int kBoxR = 16;  // activation rows per TMA box
  static constexpr int kStages = STAGES_;
  static constexpr int kThreads = 384;  // warp 0 TMA, warp 1 MMA, warps 2-5 TMEM drain; all 12 reduce
  static constexpr int kWBytes = 128 * kRowBytes;            // one of hi/lo weight tiles
  static constexpr int kXBytes = (kPR / CG_) * kRowBytes;    // one of hi/lo activation tiles (this CTA's rows)
  static constexpr int kStageBytes = 2 * kWBytes + 2 * kXBytes;
  static constexpr int kSmem = kStages * kStageBytes + 1024 + 256;
  static constexpr int kMaxSplits = 8;
  static_assert(kPR * 128 * 4 <= kStages * kStageBytes, "reduction buffer must fit in the pipeline buffers");
  static_assert(kPR % (16 * CG_) == 0, "pass rows");
  static_assert(kSmem <= 232448, "shared memory per CTA");
};
using SkDefault = SkCfg<64, 3, 320, 2>;

struct SkMaps {
  CUtensorMap wh, wl, x1h, x1l, x2h, x2l;
  int N, k1, k2;
  float unscale;
  // features >= n_klim only need the first k_lim K elements (their weight
  // rows beyond are zero: the h-gate block of the decoder state rows)
  int n_klim = 1 << 30, k_lim = 0;
};

struct SkArgs {
  int M, N;
  int nk1, nk2;  // BK-wide K blocks of activation segment 1 / 2
  int k_off2;    // weight K coordinate where segment 2 starts
  int kb_per_split;
  int splits;
  float unscale;  // 2^-(activation shift + weight shift)
  int n_klim, nk_lim;  // CTA pairs at features >= n_klim run only the first nk_lim K blocks
  int debug;  // microbenchmark knobs: 1 skip weight loads, 2 skip activation loads, 4 skip MMA, 8 skip reduction
  int row_off1;  // first activation row of segment 1 (segment 2 and the epilogue rows start at 0)
  unsigned long long *kt;  // optional CTA-time accounting (common.cuh CtaClock)
};

// Row layout of one pass: one MMA of N0 columns, or two (N0 + N1) when the
// pass has more than 256 rows.  Each CTA of a group holds N_j / CG rows of
// sub-MMA j (the leader the first half); TMEM column = row of the pass.
struct SkPass {
  int n[2], nsub, h[2], rows_cta;
  __device__ __forceinline__ SkPass(int nr, int cg) {
    const int q = 16 * cg;
    const int np = (nr + q - 1) / q * q;
    nsub = np > 256 ? 2 : 1;
    n[0] = nsub == 1 ? np : (np / 2 + q - 1) / q * q;
    n[1] = np - n[0];
    h[0] = n[0] / cg;
    h[1] = n[1] / cg;
    rows_cta = h[0] + h[1];
  }
};

template <class C, class Epi>
__global__ void __launch_bounds__(C::kThreads, 1)
    gemm_sk_kernel(const __grid_constant__ CUtensorMap wh, const __grid_constant__ CUtensorMap wl,
                   const __grid_constant__ CUtensorMap x1h, const __grid_constant__ CUtensorMap x1l,
                   const __grid_constant__ CUtensorMap x2h, const __grid_constant__ CUtensorMap x2l, SkArgs a,
                   Epi epi) {
  constexpr int CG = C::kCG;
  const CtaClock clk(a.kt);
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = tc::align_smem<1024>(smem_raw);  // stays in the shared address space (LDS/STS)
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + C::kStages * C::kStageBytes);
  uint64_t *empty = full + C::kStages;
  uint64_t *tfull = empty + C::kStages;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tfull + 1);
  float *red = reinterpret_cast<float *>(smem);  // [kPR][128] partial sums, aliases the stages

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = tc::cluster_rank();
  const int member = (int)crank % CG;  // 0 = leader of the CTA pair
  const uint32_t leader = crank - member;
  const int split = (int)crank / CG;
  const int S = a.splits;
  const int n0 = blockIdx.y * 128 * CG + member * 128;  // this CTA's 128 features (TMEM lanes)
  const int nk = (blockIdx.y * 128 * CG >= a.n_klim) ? min(a.nk1 + a.nk2, a.nk_lim) : a.nk1 + a.nk2;
  const int kb0 = split * a.kb_per_split;
  const int kb1 = min(nk, kb0 + a.kb_per_split);
  const int nkb = max(0, kb1 - kb0);
  const int npass = (a.M + C::kPR - 1) / C::kPR;
  constexpr uint16_t kPairMask = CG == 2 ? 3 : 1;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < C::kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tfull, 1);
    tc::fence_barrier_init();
    tc::tma_prefetch(&wh);
    tc::tma_prefetch(&wl);
    tc::tma_prefetch(&x1h);
    tc::tma_prefetch(&x1l);
  }
  if (warp == 1) {
    if constexpr (CG == 2)
      tc::tmem_alloc_pair<512>(tslot);
    else
      tc::tmem_alloc<512>(tslot);
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();  // barrier inits visible to the pair before any remote arrive
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  // row passes of this cluster: blockIdx.z, blockIdx.z + gridDim.z, ...
  // (gridDim.z > 1 spreads the passes of a large-M launch over clusters)
  int lp = 0;  // passes done by this CTA (ring and barrier phases)
  for (int pass = blockIdx.z; pass < npass; pass += gridDim.z, ++lp) {
    const int row0 = pass * C::kPR;
    const int nr = min(C::kPR, a.M - row0);
    const SkPass ps(nr, CG);
    const int it0 = lp * nkb;  // ring position of this pass's first k-block
    if (warp == 0) {
      if (lane == 0) {
        tc::fence_proxy_async();  // generic-proxy use of the buffers (reduction) before TMA refills them
        const bool lw = !(a.debug & 1), lx = !(a.debug & 2);
        const uint32_t bytes = (lw ? 2 * C::kWBytes : 0) + (lx ? 2 * ps.rows_cta * C::kRowBytes : 0);
        for (int i = 0; i < nkb; ++i) {
          const int it = it0 + i;
          const int s = it % C::kStages;
          if (it >= C::kStages) tc::mbar_wait(&empty[s], ((it / C::kStages) & 1) ^ 1);
          if (member == 0) tc::mbar_arrive_expect_tx(&full[s], CG * bytes);
          const uint32_t bar = tc::mapa_shared(tc::smem_u32(&full[s]), leader);
          uint8_t *st = smem + s * C::kStageBytes;
          const int kb = kb0 + i;
          const bool seg2 = kb >= a.nk1;
          const int ka = seg2 ? (kb - a.nk1) * C::kBK : kb * C::kBK;  // K coordinate inside the activation segment
          const int kw = seg2 ? a.k_off2 + ka : ka;                   // K coordinate inside the weight
          auto load = [&](void *dst, const CUtensorMap *m, int x, int y) {
            if constexpr (CG == 2)
              tc::tma_load_2d_pair(dst, m, bar, x, y);
            else
              tc::tma_load_2d(dst, m, &full[s], x, y);
          };
          if (lw) {
            load(st, &wh, kw, n0);
            load(st + C::kWBytes, &wl, kw, n0);
          }
          if (lx) {
            const CUtensorMap *mh = seg2 ? &x2h : &x1h;
            const CUtensorMap *ml = seg2 ? &x2l : &x1l;
            int srow = 0;
            for (int j = 0; j < ps.nsub; ++j) {
              const int g = row0 + (j ? ps.n[0] : 0) + member * ps.h[j];
              for (int r = 0; r < ps.h[j]; r += C::kBoxR, srow += C::kBoxR) {
                const int gr = g + r + (seg2 ? 0 : a.row_off1);
                load(st + 2 * C::kWBytes + srow * C::kRowBytes, mh, ka, gr);
                load(st + 2 * C::kWBytes + C::kXBytes + srow * C::kRowBytes, ml, ka, gr);
              }
            }
          }
        }
      }
    } else if (warp == 1) {
      if (lane == 0 && member == 0) {
        const uint32_t id0 = tc::idesc_f16(128 * CG, ps.n[0]);
        const uint32_t id1 = tc::idesc_f16(128 * CG, ps.nsub == 2 ? ps.n[1] : 16 * CG);
        auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
          if constexpr (CG == 2)
            tc::mma_f16_pair(d, ad, bd, id, acc);
          else
            tc::mma_f16(d, ad, bd, id, acc);
        };
        for (int i = 0; i < nkb; ++i) {
          const int it = it0 + i;
          const int s = it % C::kStages;
          tc::mbar_wait(&full[s], (it / C::kStages) & 1);
          tc::tc_fence_after();
          const uint32_t base = tc::smem_u32(smem + s * C::kStageBytes);
#pragma unroll
          for (int k2 = 0; k2 < ((a.debug & 4) ? 0 : C::kBK / 16); ++k2) {
            const uint32_t koff = k2 * 32;  // 16 fp16 = 32 bytes along K (inside the swizzle row)
            const uint64_t awh = tc::desc_kmajor<C::kRowBytes>(base + koff);
            const uint64_t awl = tc::desc_kmajor<C::kRowBytes>(base + C::kWBytes + koff);
            const uint32_t xb = base + 2 * C::kWBytes + koff;
            const uint32_t acc0 = (i | k2) != 0;
            {
              const uint64_t bxh = tc::desc_kmajor<C::kRowBytes>(xb);
              const uint64_t bxl = tc::desc_kmajor<C::kRowBytes>(xb + C::kXBytes);
              mma(tmem, awh, bxh, id0, acc0);
              mma(tmem, awh, bxl, id0, 1);
              mma(tmem, awl, bxh, id0, 1);
            }
            if (ps.nsub == 2) {
              const uint32_t xo = ps.h[0] * C::kRowBytes;
              const uint64_t bxh = tc::desc_kmajor<C::kRowBytes>(xb + xo);
              const uint64_t bxl = tc::desc_kmajor<C::kRowBytes>(xb + C::kXBytes + xo);
              mma(tmem + ps.n[0], awh, bxh, id1, acc0);
              mma(tmem + ps.n[0], awh, bxl, id1, 1);
              mma(tmem + ps.n[0], awl, bxh, id1, 1);
            }
          }
          // stage free (in every CTA of the group) once these MMAs have read it
          if constexpr (CG == 2)
            tc::mma_commit_pair_mc(&empty[s], (uint16_t)(kPairMask << leader));
          else
            tc::mma_commit(&empty[s]);
        }
        if constexpr (CG == 2)
          tc::mma_commit_pair_mc(tfull, (uint16_t)(kPairMask << leader));
        else
          tc::mma_commit(tfull);  // this pass's partial is complete in TMEM
      }
    } else if (warp < 6) {
      // drain TMEM -> red[row][feature]; thread = feature (TMEM lane)
      const int lg = warp & 3;
      const int f = lg * 32 + lane;
      if (nkb > 0) {
        tc::mbar_wait(tfull, lp & 1);
        tc::tc_fence_after();
      }
      const int ncol = ps.n[0] + ps.n[1];
#pragma unroll 1
      for (int c0 = 0; c0 < ncol; c0 += 32) {
        float v[32];
        if (nkb > 0) {
          tc::tmem_ld_32x32(tmem + ((uint32_t)(lg * 32) << 16) + c0, v);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
#pragma unroll
        for (int i = 0; i < 32; ++i) red[(c0 + i) * 128 + f] = v[i];
      }
      tc::tc_fence_before();
    }
    __syncwarp();
    tc::cluster_sync();  // every CTA's partial is staged (release/acquire at cluster scope)
    tc::tc_fence_after();

    // deterministic reduction of this CTA's row slice over the S partials of
    // its 128 features (cluster ranks member + CG * s)
    const int per = (nr + S - 1) / S;
    const int rb = split * per;
    const int re = min(nr, rb + per);
    const int items = max(0, re - rb) * 32;
    const uint32_t red_base = tc::smem_u32(red);
    // items of (row, 4 features); kU items per thread per batch: all DSMEM
    // and epilogue loads of a batch are issued before its stores
    constexpr int kU = 2;
    for (int base = threadIdx.x; base < ((a.debug & 8) ? 0 : items); base += kU * C::kThreads) {
      float4 acc[kU];
      bool ok[kU];
      int mm[kU], nn[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int idx = base + u * C::kThreads;
        const int r = rb + idx / 32;
        const int q = idx % 32;
        nn[u] = n0 + 4 * q;
        mm[u] = row0 + r;
        ok[u] = idx < items && nn[u] < a.N;
        acc[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (idx < items) {
          const uint32_t off = red_base + (uint32_t)(r * 128 + 4 * q) * 4u;
          float4 p[C::kMaxSplits];
#pragma unroll
          for (int s = 0; s < C::kMaxSplits; ++s)
            if (s < S) p[s] = tc::ld_dsmem_v4(tc::mapa_shared(off, (uint32_t)(member + CG * s)));
#pragma unroll
          for (int s = 0; s < C::kMaxSplits; ++s)
            if (s < S) {
              acc[u].x += p[s].x;
              acc[u].y += p[s].y;
              acc[u].z += p[s].z;
              acc[u].w += p[s].w;
            }
          acc[u].x *= a.unscale;
          acc[u].y *= a.unscale;
          acc[u].z *= a.unscale;
          acc[u].w *= a.unscale;
        }
      }
      typename Epi::Pre pre[kU];
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ok[u]) pre[u] = epi.load4(mm[u], nn[u]);
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ok[u]) epi.store4(mm[u], nn[u], acc[u], pre[u]);
    }
    tc::fence_proxy_async();
    tc::tc_fence_before();
    __syncwarp();
    tc::cluster_sync();  // peers are done reading this CTA's buffer
    tc::tc_fence_after();
  }
  if (warp == 1) {
    if constexpr (CG == 2)
      tc::tmem_dealloc_pair<512>(tmem);
    else
      tc::tmem_dealloc<512>(tmem);
  }
  clk.done();  // every thread passed the final cluster barrier
}

// Activation segment s: hi/lo [rows, k_s] with row pitch lda_s (elements),
// Rmax rows allocated; weight hi/lo: [N, Kb = k1 + k2] K-major.
template <class C = SkDefault>
SkMaps make_sk_maps(const __half *x1h, const __half *x1l, int k1, int lda1, const __half *x2h, const __half *x2l,
                    int k2, int lda2, int Rmax, const __half *wh, const __half *wl, int N, int Kb, float unscale,
                    int Rmax2 = -1, int ldw = 0) {  // ldw: weight row pitch (default Kb)
  SkMaps m;
  m.x1h = make_tma_2d_f16(x1h, k1, Rmax, lda1, C::kBK, C::kBoxR);
  m.x1l = make_tma_2d_f16(x1l, k1, Rmax, lda1, C::kBK, C::kBoxR);
  if (x2h) {
    if (Rmax2 < 0) Rmax2 = Rmax;
    m.x2h = make_tma_2d_f16(x2h, k2, Rmax2, lda2, C::kBK, C::kBoxR);
    m.x2l = make_tma_2d_f16(x2l, k2, Rmax2, lda2, C::kBK, C::kBoxR);
  } else {
    m.x2h = m.x1h;
    m.x2l = m.x1l;
  }
  m.wh = make_tma_2d_f16(wh, Kb, N, ldw ? ldw : Kb, C::kBK, 128);
  m.wl = make_tma_2d_f16(wl, Kb, N, ldw ? ldw : Kb, C::kBK, 128);
  m.unscale = unscale;
  m.N = N;
  m.k1 = k1;
  m.k2 = x2h ? k2 : 0;
  return m;
}

// Split count from (N, K) only: about `target_ctas` CTAs per launch, at most
// kMaxSplits (portable cluster size), every split non-empty.
template <class C = SkDefault>
int sk_splits(const SkMaps &m, int target_ctas) {
  const int nt = ceil_div(m.N, 128 * C::kCG) * C::kCG;
  const int nk = ceil_div(m.k1, C::kBK) + ceil_div(m.k2, C::kBK);
  int s = std::max(1, std::min(C::kMaxSplits, target_ctas / nt));
  s = std::min(s, nk);
  const int kps = ceil_div(nk, s);
  return ceil_div(nk, kps);
}

template <class C = SkDefault, class Epi>
void launch_gemm_sk(const SkMaps &maps, int M, int splits, const Epi &epi, cudaStream_t st, int debug = 0,
                    int row_off1 = 0, int zgrid = 1) {
  if (M <= 0) return;
  SkArgs a{};
  a.M = M;
  a.N = maps.N;
  a.nk1 = ceil_div(maps.k1, C::kBK);
  a.nk2 = ceil_div(maps.k2, C::kBK);
  a.k_off2 = maps.k1;
  a.kb_per_split = ceil_div(a.nk1 + a.nk2, splits);
  a.splits = splits;
  a.unscale = maps.unscale;
  a.n_klim = maps.n_klim;
  a.nk_lim = maps.k_lim > 0 ? ceil_div(maps.k_lim, C::kBK) : a.nk1 + a.nk2;
  a.debug = debug;
  a.row_off1 = row_off1;
  a.kt = ktime_ptr();
  zgrid = std::max(1, std::min(zgrid, ceil_div(M, C::kPR)));
  auto kern = gemm_sk_kernel<C, Epi>;
  static bool attr[64] = {};
  int dev = 0;
  AMUN_CUDA(cudaGetDevice(&dev));
  if (dev >= 64 || !attr[dev]) {
    AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
    AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    if (dev < 64) attr[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C::kCG * splits, ceil_div(maps.N, 128 * C::kCG), zgrid);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = C::kCG * splits;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  last_launch_ctas() = (int)(cfg.gridDim.x * cfg.gridDim.y * cfg.gridDim.z);
  AMUN_CUDA(cudaLaunchKernelEx(&cfg, kern, maps.wh, maps.wl, maps.x1h, maps.x1l, maps.x2h, maps.x2l, a, epi));
}

// Clusters of `splits` CTAs of this kernel that fit on the device at once.
template <class C = SkDefault, class Epi>
int sk_max_active_clusters(int splits) {
  auto kern = gemm_sk_kernel<C, Epi>;
  AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem));
  AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(C::kCG * splits, 1);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = C::kCG * splits;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  int n = 0;
  AMUN_CUDA(cudaOccupancyMaxActiveClusters(&n, kern, &cfg));
  return n;
}

// Split count for one launch: the largest S <= kMaxSplits with at most
// `max_ctas` CTAs whose N/128 clusters of S CTAs are co-resident on the
// device (one wave).  Depends only on (N, K) and the device, never on R.
template <class C = SkDefault>
int sk_fit_splits(const SkMaps &m, int max_ctas) {
  const int nt = ceil_div(m.N, 128 * C::kCG) * C::kCG;
  const int nk = ceil_div(m.k1, C::kBK) + ceil_div(m.k2, C::kBK);
  static int maxc[64][C::kMaxSplits + 1] = {};
  int dev = 0;
  AMUN_CUDA(cudaGetDevice(&dev));
  for (int s = std::min(C::kMaxSplits, nk); s > 1; --s) {
    if (C::kCG * s > 16) continue;  // cluster size limit (non-portable 16)
    if (nt * s > max_ctas) continue;
    if (ceil_div(nk, ceil_div(nk, s)) != s) continue;  // every split non-empty
    int &mc = maxc[dev & 63][s];
    if (!mc) mc = std::max(1, sk_max_active_clusters<C, EpiStore>(s));
    if (nt / C::kCG <= mc) return s;
  }
  return 1;
}

}  // namespace amun

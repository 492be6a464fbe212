// Split-K tensor-core GEMM (tcgen05.mma kind::tf32, 3xTF32) producing fp32
// partial sums; the split partials are then reduced in a fixed order by
// splitk_reduce_kernel<Epi>, which applies the fused epilogue (GRU gates,
// state update, tanh, ...).  Used for the decoder-step GEMMs whose N is too
// small to fill 148 SMs with output tiles alone:
//   query  s W_att_s            (N = d_att, K = d_h)
//   GRU-A  [y c s] Wg           (N = 3 d_h, K = d_e + 3 d_h)
//   GRU-B  (r*s) U_h            (N = d_h,   K = d_h)
//   out    [y c | s'] W_out     (N = d_e,   K = d_e + 3 d_h, two A segments)
//
// CTA (blockIdx.x = N tile, blockIdx.y = K split) computes a BN-wide tile
// for all rows (MB x 128 per pass) over its K range.  Operands are hi/lo
// fp32 pairs (tf32-exact hi + residual lo) so hi*hi + hi*lo + lo*hi gives
// FP32-equivalent products.  A may be two K segments with separate tensor
// maps (segment 2's K coordinates continue at k_off2 in B).  Pairs of CTAs
// with the same split form a cluster and TMA-multicast the A tiles.
#include "common.cuh"
#include "gemm_tc.cuh"
#include "tc_common.cuh"

namespace amun {

namespace {

constexpr int kBK = 16;

template <int BN, int MB, int STAGES, int CS>
__global__ void __launch_bounds__(64 + 128 * MB, 1)
    gemm_tc_partial_kernel(const __grid_constant__ CUtensorMap a1h, const __grid_constant__ CUtensorMap a1l,
                           const __grid_constant__ CUtensorMap a2h, const __grid_constant__ CUtensorMap a2l,
                           const __grid_constant__ CUtensorMap bh, const __grid_constant__ CUtensorMap bl,
                           GemmTcArgs a) {
  constexpr int A_BYTES = MB * 128 * kBK * 4;
  constexpr int B_BYTES = BN * kBK * 4;
  constexpr int STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  constexpr uint32_t TMEM_COLS = (MB * BN <= 128) ? 128 : (MB * BN <= 256) ? 256 : 512;
  static_assert(MB * BN <= 512, "accumulators exceed TMEM");
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + STAGES;
  uint64_t *tempty = tfull + 1;
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n0 = blockIdx.x * BN;
  const int split = blockIdx.y;
  const int nk = a.nk1 + a.nk2;
  const int kb0 = split * a.kb_per_split;
  const int kb1 = min(nk, kb0 + a.kb_per_split);
  const int nkb = max(0, kb1 - kb0);
  const int nchunks = (a.M + MB * 128 - 1) / (MB * 128);
  const uint32_t crank = CS > 1 ? tc::cluster_rank() : 0;
  constexpr uint16_t kAll = (uint16_t)((1u << CS) - 1);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], CS);
    }
    tc::mbar_init(tfull, 1);
    tc::mbar_init(tempty, 4 * MB);
    tc::fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc<TMEM_COLS>(tslot);
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (CS > 1) tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (lane == 0 && nkb > 0) {
      int it = 0;
      for (int ch = 0; ch < nchunks; ++ch) {
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) tc::mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          tc::mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
          uint8_t *st = smem + s * STAGE_BYTES;
          const bool seg2 = kb >= a.nk1;
          const int ka = seg2 ? (kb - a.nk1) * kBK : kb * kBK;  // coordinate inside the A segment
          const int kbq = seg2 ? a.k_off2 + ka : ka;            // coordinate inside B's K
          const CUtensorMap *mh = seg2 ? &a2h : &a1h;
          const CUtensorMap *ml = seg2 ? &a2l : &a1l;
#pragma unroll
          for (int j = 0; j < 2 * MB; ++j) {
            if (j % CS != (int)crank) continue;
            const int mb = j >> 1;
            uint8_t *dst = st + (j & 1) * A_BYTES + mb * 128 * kBK * 4;
            const int row = (ch * MB + mb) * 128;
            if constexpr (CS > 1)
              tc::tma_load_2d_mc(dst, (j & 1) ? ml : mh, &full[s], ka, row, kAll);
            else
              tc::tma_load_2d(dst, (j & 1) ? ml : mh, &full[s], ka, row);
          }
          tc::tma_load_2d(st + 2 * A_BYTES, &bh, &full[s], kbq, n0);
          tc::tma_load_2d(st + 2 * A_BYTES + B_BYTES, &bl, &full[s], kbq, n0);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && nkb > 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(128, BN);
      int it = 0;
      for (int ch = 0; ch < nchunks; ++ch) {
        if (ch > 0) {
          tc::mbar_wait(tempty, (ch - 1) & 1);
          tc::tc_fence_after();
        }
        for (int i = 0; i < nkb; ++i, ++it) {
          const int s = it % STAGES;
          tc::mbar_wait(&full[s], (it / STAGES) & 1);
          tc::tc_fence_after();
          const uint32_t base = tc::smem_u32(smem + s * STAGE_BYTES);
#pragma unroll
          for (int k2 = 0; k2 < kBK / 8; ++k2) {
            const uint32_t koff = k2 * 32;
            const uint64_t dbh = tc::desc_kmajor_sw64(base + 2 * A_BYTES + koff);
            const uint64_t dbl = tc::desc_kmajor_sw64(base + 2 * A_BYTES + B_BYTES + koff);
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
              const uint64_t dah = tc::desc_kmajor_sw64(base + mb * 128 * kBK * 4 + koff);
              const uint64_t dal = tc::desc_kmajor_sw64(base + A_BYTES + mb * 128 * kBK * 4 + koff);
              const uint32_t d = tmem + mb * BN;
              tc::mma_tf32(d, dah, dbh, idesc, (i | k2) != 0);
              tc::mma_tf32(d, dah, dbl, idesc, 1);
              tc::mma_tf32(d, dal, dbh, idesc, 1);
            }
          }
          if constexpr (CS > 1)
            tc::mma_commit_mc(&empty[s], kAll);
          else
            tc::mma_commit(&empty[s]);
        }
        tc::mma_commit(tfull);
      }
    }
  } else {
    // epilogue: warp group mb stores its M-block's raw partial sums
    const int lg = warp & 3;
    const int mb = (warp - 2) >> 2;
    float *outp = a.out + (long long)split * a.M * a.N;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int m = (ch * MB + mb) * 128 + lg * 32 + lane;
      if (nkb > 0) {
        tc::mbar_wait(tfull, ch & 1);
        tc::tc_fence_after();
      }
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        if (nkb > 0) {
          tc::tmem_ld_32x32(tmem + ((uint32_t)(lg * 32) << 16) + mb * BN + c0, v);
        } else {
#pragma unroll
          for (int i = 0; i < 32; ++i) v[i] = 0.f;
        }
        if (m < a.M) {
          float *dst = outp + (long long)m * a.N + n0 + c0;
          const int lim = a.N - (n0 + c0);
          if (lim >= 32 && (a.N & 3) == 0) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4 *>(dst + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (i < lim) dst[i] = v[i];
          }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0 && nkb > 0) tc::mbar_arrive(tempty);
    }
  }
  __syncthreads();
  if constexpr (CS > 1) tc::cluster_sync();
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<TMEM_COLS>(tmem);
  }
}

constexpr int kBN = 128, kMB = 3, kCS = 2;

}  // namespace

int gemm_tc_tile_n() { return kBN; }

GemmTcMaps make_gemm_tc_maps(const float *a1h, const float *a1l, int k1, int lda1, const float *a2h,
                             const float *a2l, int k2, int lda2, int M, const float *bh, const float *bl, int N,
                             int Kb) {
  GemmTcMaps m;
  m.a1h = make_tma_2d_f32(a1h, k1, M, lda1, kBK, 128);
  m.a1l = make_tma_2d_f32(a1l, k1, M, lda1, kBK, 128);
  if (a2h) {
    m.a2h = make_tma_2d_f32(a2h, k2, M, lda2, kBK, 128);
    m.a2l = make_tma_2d_f32(a2l, k2, M, lda2, kBK, 128);
  } else {
    m.a2h = m.a1h;
    m.a2l = m.a1l;
  }
  m.bh = make_tma_2d_f32(bh, Kb, N, Kb, kBK, kBN);
  m.bl = make_tma_2d_f32(bl, Kb, N, Kb, kBK, kBN);
  m.k1 = k1;
  m.k2 = a2h ? k2 : 0;
  m.N = N;
  return m;
}

int gemm_tc_splits(const GemmTcMaps &maps, int target_ctas) {
  const int nt = ceil_div(ceil_div(maps.N, kBN), kCS) * kCS;
  const int nk = ceil_div(maps.k1, kBK) + ceil_div(maps.k2, kBK);
  int s = std::max(1, target_ctas / nt);
  s = std::min(s, nk);
  const int kps = ceil_div(nk, s);
  return ceil_div(nk, kps);
}

template <int kStages>
void launch_partial_s(const GemmTcMaps &maps, int M, int splits, float *out, cudaStream_t st);

void launch_gemm_tc_partial(const GemmTcMaps &maps, int M, int splits, float *out, cudaStream_t st) {
  static int stages = [] {
    const char *e = getenv("AMUN_TC_STAGES");
    return (e && e[0] == '2') ? 2 : 3;
  }();
  if (stages == 2)
    launch_partial_s<2>(maps, M, splits, out, st);
  else
    launch_partial_s<3>(maps, M, splits, out, st);
}

template <int kStages>
void launch_partial_s(const GemmTcMaps &maps, int M, int splits, float *out, cudaStream_t st) {
  GemmTcArgs a{};
  a.M = M;
  a.N = maps.N;
  a.nk1 = ceil_div(maps.k1, kBK);
  a.nk2 = ceil_div(maps.k2, kBK);
  a.k_off2 = maps.k1;
  a.kb_per_split = ceil_div(a.nk1 + a.nk2, splits);
  a.out = out;
  auto kern = gemm_tc_partial_kernel<kBN, kMB, kStages, kCS>;
  constexpr int stage = 2 * kMB * 128 * kBK * 4 + 2 * kBN * kBK * 4;
  const int smem = kStages * stage + 1024 + 256;
  static bool attr[64] = {};
  int dev = 0;
  AMUN_CUDA(cudaGetDevice(&dev));
  if (dev >= 64 || !attr[dev]) {
    AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (dev < 64) attr[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ceil_div(ceil_div(maps.N, kBN), kCS) * kCS, splits);
  cfg.blockDim = dim3(64 + 128 * kMB);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = kCS;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  AMUN_CUDA(cudaLaunchKernelEx(&cfg, kern, maps.a1h, maps.a1l, maps.a2h, maps.a2l, maps.bh, maps.bl, a));
}

}  // namespace amun

// Logit projection on the 5th-gen tensor cores, fused with the log-softmax
// partials and the per-row top-k (nnet.py:161 + tensor.py:79-92 +
// search.py:169-170): full logits never reach HBM.
//
//   logits[R, V] = t[R, K] * W_logit[K, V] + b_logit,  K = d_emb
//
// Precision: 3xTF32 on tcgen05.mma kind::tf32.  Both operands are split into
// tf32-exact hi and residual lo parts (t by the deep-output epilogue, the
// weights once at model load) and the CTA accumulates hi*hi + hi*lo + lo*hi
// in fp32 in TMEM — FP32-equivalent accuracy (BF16/TF32 flip the
// beam set in 1-4% of steps, FP32 and 3xTF32 in none).
//
// CTA = one BN-wide vocabulary tile for ALL hypothesis rows (up to MB*128 per
// pass; TMEM holds MB accumulators of 128 x BN fp32), so every weight byte is
// read from HBM exactly once per launch.  Warp roles: warp 0 issues TMA
// (SWIZZLE_64B K-major tiles, 3-stage mbarrier ring), warp 1 allocates TMEM
// and issues the MMAs from one thread, warps 2-5 run the epilogue: thread =
// one row (TMEM lane), tcgen05.ld 32 columns at a time, bias add, running
// max / top-kk insertion, then a second TMEM pass for sum(exp(x - max)).
#include "common.cuh"
#include "logits_tc.cuh"
#include "tc_common.cuh"

namespace amun {

namespace {

constexpr int kBK = 16;  // fp32 elements per 64-byte swizzled row

// Register-resident sorted top-KK list of one row (KK is a compile-time
// size >= kk so every index is static and nothing spills to local memory).
template <int KK>
struct RowTop {
  float v[KK];
  int t[KK];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < KK; ++i) {
      v[i] = -INFINITY;
      t[i] = -1;
    }
  }
  __device__ __forceinline__ float worst() const { return v[KK - 1]; }
  // caller guarantees x > worst().  Columns arrive in ascending token order,
  // so an equal value loses the tie (token asc): strict > is exact.
  __device__ __forceinline__ void insert(float x, int n) {
#pragma unroll
    for (int i = 0; i < KK; ++i) {
      if (x > v[i]) {
        float tv = v[i];
        int tt = t[i];
        v[i] = x;
        t[i] = n;
        x = tv;
        n = tt;
      }
    }
  }
};

template <int BN, int MB, int STAGES, int KK, int CS>
__global__ void __launch_bounds__(64 + 128 * MB, 1)
    logits_tc_kernel(const __grid_constant__ CUtensorMap tA_hi, const __grid_constant__ CUtensorMap tA_lo,
                     const __grid_constant__ CUtensorMap tB_hi, const __grid_constant__ CUtensorMap tB_lo,
                     LogitTcArgs a) {
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
  float *sbias = reinterpret_cast<float *>(tempty + 2);  // [BN] bias tile, -inf past the vocabulary

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n0 = blockIdx.x * BN;
  // CS CTAs of a cluster work on adjacent vocabulary tiles and share the
  // activation tiles: each CTA TMA-multicasts 1/CS of them to the cluster.
  const uint32_t crank = CS > 1 ? tc::cluster_rank() : 0;
  constexpr uint16_t kAll = (uint16_t)((1u << CS) - 1);
  const int nk = (a.K + kBK - 1) / kBK;
  const int nchunks = (a.M + MB * 128 - 1) / (MB * 128);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], CS);  // released by every CTA of the cluster
    }
    tc::mbar_init(tfull, 1);
    tc::mbar_init(tempty, 4 * MB);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tA_hi);
    tc::tma_prefetch(&tA_lo);
    tc::tma_prefetch(&tB_hi);
    tc::tma_prefetch(&tB_lo);
  }
  if (warp == 1) tc::tmem_alloc<TMEM_COLS>(tslot);
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (CS > 1) tc::cluster_sync();  // peers' barriers initialised before any multicast
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ---------------- TMA producer
    if (lane == 0) {
      int it = 0;
      for (int ch = 0; ch < nchunks; ++ch) {
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          if (it >= STAGES) tc::mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          const bool la = !(a.debug_flags & 1), lb = !(a.debug_flags & 2);
          tc::mbar_arrive_expect_tx(&full[s], (la ? 2 * A_BYTES : 0) + (lb ? 2 * B_BYTES : 0));
          uint8_t *st = smem + s * STAGE_BYTES;
          const int kx = kb * kBK;
          if (la) {
#pragma unroll
            for (int j = 0; j < 2 * MB; ++j) {
              if (j % CS != (int)crank) continue;
              const int mb = j >> 1;
              const int row = (ch * MB + mb) * 128;
              uint8_t *dst = st + (j & 1) * A_BYTES + mb * 128 * kBK * 4;
              const CUtensorMap *map = (j & 1) ? &tA_lo : &tA_hi;
              if constexpr (CS > 1)
                tc::tma_load_2d_mc(dst, map, &full[s], kx, row, kAll);
              else
                tc::tma_load_2d(dst, map, &full[s], kx, row);
            }
          }
          if (lb) {
            tc::tma_load_2d(st + 2 * A_BYTES, &tB_hi, &full[s], kx, n0);
            tc::tma_load_2d(st + 2 * A_BYTES + B_BYTES, &tB_lo, &full[s], kx, n0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread)
    if (lane == 0) {
      constexpr uint32_t idesc = tc::idesc_tf32(128, BN);
      int it = 0;
      for (int ch = 0; ch < nchunks; ++ch) {
        if (ch > 0) {
          tc::mbar_wait(tempty, (ch - 1) & 1);
          tc::tc_fence_after();
        }
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % STAGES;
          tc::mbar_wait(&full[s], (it / STAGES) & 1);
          tc::tc_fence_after();
          const uint32_t base = tc::smem_u32(smem + s * STAGE_BYTES);
#pragma unroll
          for (int k2 = 0; k2 < ((a.debug_flags & 4) ? 0 : kBK / 8); ++k2) {
            const uint32_t koff = k2 * 32;  // 8 tf32 = 32 bytes along K
            const uint64_t bh = tc::desc_kmajor_sw64(base + 2 * A_BYTES + koff);
            const uint64_t bl = tc::desc_kmajor_sw64(base + 2 * A_BYTES + B_BYTES + koff);
#pragma unroll
            for (int mb = 0; mb < MB; ++mb) {
              const uint64_t ah = tc::desc_kmajor_sw64(base + mb * 128 * kBK * 4 + koff);
              const uint64_t al = tc::desc_kmajor_sw64(base + A_BYTES + mb * 128 * kBK * 4 + koff);
              const uint32_t d = tmem + mb * BN;
              tc::mma_tf32(d, ah, bh, idesc, (kb | k2) != 0);  // hi * hi
              tc::mma_tf32(d, ah, bl, idesc, 1);               // hi * lo
              tc::mma_tf32(d, al, bh, idesc, 1);               // lo * hi
            }
          }
          if constexpr (CS > 1)
            tc::mma_commit_mc(&empty[s], kAll);  // slot free in every CTA's ring
          else
            tc::mma_commit(&empty[s]);  // smem stage free once these MMAs drain
        }
        tc::mma_commit(tfull);  // accumulators of this chunk complete
      }
    }
  } else {
    // ---------------- epilogue: 4*MB warps; warp group mb drains M-block mb,
    // thread = one row (TMEM lane) of the tile
    const int lg = warp & 3;  // TMEM lane quarter this warp may access
    const int mb = (warp - 2) >> 2;
    const int nt = blockIdx.x;
    for (int c = threadIdx.x - 64; c < BN; c += 128 * MB)
      sbias[c] = (n0 + c < a.N) ? __ldg(a.bias + n0 + c) : -INFINITY;
    asm volatile("bar.sync 1, %0;" ::"n"(128 * MB) : "memory");  // epilogue warps only
    for (int ch = 0; ch < nchunks; ++ch) {
      tc::mbar_wait(tfull, ch & 1);
      tc::tc_fence_after();
      if (!(a.debug_flags & 8)) {
        const int m = (ch * MB + mb) * 128 + lg * 32 + lane;
        const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + mb * BN;
        RowTop<KK> top;
        top.init();
        float mx = -INFINITY;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tc::tmem_ld_32x32(tb + c0, v);
          float cm = -INFINITY;
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v[i] += sbias[c0 + i];
            cm = fmaxf(cm, v[i]);
          }
          mx = fmaxf(mx, cm);
          if (cm > top.worst() && !(a.debug_flags & 16)) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (v[i] > top.worst()) top.insert(v[i], n0 + c0 + i);
          }
        }
        float se = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < ((a.debug_flags & 32) ? 0 : BN); c0 += 32) {
          float v[32];
          tc::tmem_ld_32x32(tb + c0, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) se += expf(v[i] + sbias[c0 + i] - mx);
        }
        if (m < a.M && nt < a.ntiles && !(a.debug_flags & 64)) {
          a.pmax[(long long)nt * a.M + m] = mx;
          a.psum[(long long)nt * a.M + m] = se;
          const long long base = ((long long)m * a.ntiles + nt) * a.kk;
#pragma unroll
          for (int i = 0; i < KK; ++i)
            if (i < a.kk) {
              a.cval[base + i] = top.v[i];
              a.ctok[base + i] = top.t[i];
            }
        }
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(tempty);
    }
  }
  __syncthreads();
  if constexpr (CS > 1) tc::cluster_sync();  // no CTA leaves while peers may still signal it
  if (warp == 1) {
    tc::tc_fence_after();
    tc::tmem_dealloc<TMEM_COLS>(tmem);
  }
}

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    AMUN_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw Error(2, "cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

constexpr int kTcBN = 128, kTcMB = 3, kTcCluster = 2;

// pipeline depth (env AMUN_TC_STAGES=2 trades latency hiding for 64 KB of
// shared memory that concurrent kernels of other lanes can use)
int tc_stages() {
  static int v = [] {
    const char *e = getenv("AMUN_TC_STAGES");
    return (e && e[0] == '2') ? 2 : 3;
  }();
  return v;
}

template <int KK, int kTcStages>
void launch_t_s(const LogitTcMaps &maps, const LogitTcArgs &a, cudaStream_t st) {
  auto kern = logits_tc_kernel<kTcBN, kTcMB, kTcStages, KK, kTcCluster>;
  constexpr int stage = 2 * kTcMB * 128 * kBK * 4 + 2 * kTcBN * kBK * 4;
  const int smem = kTcStages * stage + 1024 + 256 + kTcBN * 4;
  static bool attr[64] = {};
  int dev = 0;
  AMUN_CUDA(cudaGetDevice(&dev));
  if (dev >= 64 || !attr[dev]) {
    AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (dev < 64) attr[dev] = true;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(ceil_div(ceil_div(a.N, kTcBN), kTcCluster) * kTcCluster);
  cfg.blockDim = dim3(64 + 128 * kTcMB);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = kTcCluster;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  AMUN_CUDA(cudaLaunchKernelEx(&cfg, kern, maps.a_hi, maps.a_lo, maps.b_hi, maps.b_lo, a));
}

}  // namespace

int logits_tc_tile_n() { return kTcBN; }

CUtensorMap make_tma_2d_f32(const float *ptr, int inner, int outer, int row_stride_elems, int box_inner,
                            int box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)row_stride_elems * 4};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(ptr), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           box_inner * 4 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(2, "cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  return m;
}

LogitTcMaps make_logit_maps(const float *t_hi, const float *t_lo, int R, int K, int ldt, const float *w_hi,
                            const float *w_lo, int V) {
  LogitTcMaps m;
  m.a_hi = make_tma_2d_f32(t_hi, K, R, ldt, kBK, 128);
  m.a_lo = make_tma_2d_f32(t_lo, K, R, ldt, kBK, 128);
  m.b_hi = make_tma_2d_f32(w_hi, K, V, K, kBK, kTcBN);
  m.b_lo = make_tma_2d_f32(w_lo, K, V, K, kBK, kTcBN);
  return m;
}

template <int KK>
void launch_t(const LogitTcMaps &maps, const LogitTcArgs &a, cudaStream_t st) {
  if (tc_stages() == 2)
    launch_t_s<KK, 2>(maps, a, st);
  else
    launch_t_s<KK, 3>(maps, a, st);
}

void launch_logits_tc(const LogitTcMaps &maps, const LogitTcArgs &a, cudaStream_t st) {
  // list size >= kk (a sorted top-KK list contains the top-kk as its prefix)
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

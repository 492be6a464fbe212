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

template <int KMAX>
struct RowTop {
  float v[KMAX];
  int t[KMAX];
  float worst;
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {
      v[i] = -INFINITY;
      t[i] = -1;
    }
    worst = -INFINITY;
  }
  // columns arrive in ascending token order, so an equal value loses the
  // tie (token asc) and strict > is the exact reference order.
  __device__ __forceinline__ void push(float x, int n, int kk) {
    if (!(x > worst)) return;
#pragma unroll
    for (int i = 0; i < KMAX; ++i) {
      if (i < kk && x > v[i]) {
        float tv = v[i];
        int tt = t[i];
        v[i] = x;
        t[i] = n;
        x = tv;
        n = tt;
      }
    }
#pragma unroll
    for (int i = 0; i < KMAX; ++i)
      if (i == kk - 1) worst = v[i];
  }
};

template <int BN, int MB, int STAGES, int KMAX>
__global__ void __launch_bounds__(192, 1)
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

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n0 = blockIdx.x * BN;
  const int nk = (a.K + kBK - 1) / kBK;
  const int nchunks = (a.M + MB * 128 - 1) / (MB * 128);

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(tfull, 1);
    tc::mbar_init(tempty, 4);
    tc::fence_barrier_init();
    tc::tma_prefetch(&tA_hi);
    tc::tma_prefetch(&tA_lo);
    tc::tma_prefetch(&tB_hi);
    tc::tma_prefetch(&tB_lo);
  }
  if (warp == 1) tc::tmem_alloc<TMEM_COLS>(tslot);
  tc::tc_fence_before();
  __syncthreads();
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
          tc::mbar_arrive_expect_tx(&full[s], STAGE_BYTES);
          uint8_t *st = smem + s * STAGE_BYTES;
          const int kx = kb * kBK;
#pragma unroll
          for (int mb = 0; mb < MB; ++mb) {
            const int row = (ch * MB + mb) * 128;
            tc::tma_load_2d(st + mb * 128 * kBK * 4, &tA_hi, &full[s], kx, row);
            tc::tma_load_2d(st + A_BYTES + mb * 128 * kBK * 4, &tA_lo, &full[s], kx, row);
          }
          tc::tma_load_2d(st + 2 * A_BYTES, &tB_hi, &full[s], kx, n0);
          tc::tma_load_2d(st + 2 * A_BYTES + B_BYTES, &tB_lo, &full[s], kx, n0);
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
          for (int k2 = 0; k2 < kBK / 8; ++k2) {
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
          tc::mma_commit(&empty[s]);  // smem stage free once these MMAs drain
        }
        tc::mma_commit(tfull);  // accumulators of this chunk complete
      }
    }
  } else {
    // ---------------- epilogue: warps 2..5, thread = one row of the tile
    const int lg = warp & 3;  // TMEM lane quarter this warp may access
    const int nt = blockIdx.x;
    for (int ch = 0; ch < nchunks; ++ch) {
      tc::mbar_wait(tfull, ch & 1);
      tc::tc_fence_after();
#pragma unroll 1
      for (int mb = 0; mb < MB; ++mb) {
        const int m = (ch * MB + mb) * 128 + lg * 32 + lane;
        const uint32_t tb = tmem + ((uint32_t)(lg * 32) << 16) + mb * BN;
        RowTop<KMAX> top;
        top.init();
        float mx = -INFINITY;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tc::tmem_ld_32x32(tb + c0, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int n = n0 + c0 + i;
            if (n < a.N) {
              const float x = v[i] + __ldg(a.bias + n);
              mx = fmaxf(mx, x);
              top.push(x, n, a.kk);
            }
          }
        }
        float se = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tc::tmem_ld_32x32(tb + c0, v);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const int n = n0 + c0 + i;
            if (n < a.N) se += expf(v[i] + __ldg(a.bias + n) - mx);
          }
        }
        if (m < a.M) {
          a.pmax[(long long)nt * a.M + m] = mx;
          a.psum[(long long)nt * a.M + m] = se;
          const long long base = ((long long)m * a.ntiles + nt) * a.kk;
#pragma unroll
          for (int i = 0; i < KMAX; ++i)
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

constexpr int kTcBN = 128, kTcMB = 3, kTcStages = 3;

template <int KMAX>
void launch_t(const LogitTcMaps &maps, const LogitTcArgs &a, cudaStream_t st) {
  auto kern = logits_tc_kernel<kTcBN, kTcMB, kTcStages, KMAX>;
  constexpr int stage = 2 * kTcMB * 128 * kBK * 4 + 2 * kTcBN * kBK * 4;
  const int smem = kTcStages * stage + 1024 + 256;
  static bool attr[64] = {};
  int dev = 0;
  AMUN_CUDA(cudaGetDevice(&dev));
  if (dev >= 64 || !attr[dev]) {
    AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    if (dev < 64) attr[dev] = true;
  }
  kern<<<ceil_div(a.N, kTcBN), 192, smem, st>>>(maps.a_hi, maps.a_lo, maps.b_hi, maps.b_lo, a);
  AMUN_CHECK_LAUNCH();
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
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
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

void launch_logits_tc(const LogitTcMaps &maps, const LogitTcArgs &a, cudaStream_t st) {
  if (a.kk <= 1) launch_t<1>(maps, a, st);
  else if (a.kk <= 4) launch_t<4>(maps, a, st);
  else if (a.kk <= 8) launch_t<8>(maps, a, st);
  else if (a.kk <= 16) launch_t<16>(maps, a, st);
  else throw Error(4, "tensor-core logit path supports beam <= 16");
}

}  // namespace amun

// Logit projection on the 5th-gen tensor cores, fused with the log-softmax
// partials and the per-row top-k (nnet.py:161 + tensor.py:79-92 +
// search.py:169-170): full logits never reach HBM.
//
//   logits[R, V] = t[R, K] * W_logit[K, V] + b_logit,  K = d_emb
//
// Precision: 3xFP16 on tcgen05.mma kind::f16.  Both operands are scaled by a
// power of two and split into fp16 hi and residual lo parts (t by the
// deep-output epilogue, common.cuh split_h; the weights once at model load)
// and the MMAs accumulate hi*hi + hi*lo + lo*hi in fp32 in TMEM — ~22
// significant bits per operand like 3xTF32, FP32-equivalent accuracy (SURVEY
// §0.4: BF16/TF32 flip the beam set in 1-4% of steps, FP32 and 3xTF32 in
// none), at twice the tf32 MMA rate and half its operand bytes.  The epilogue
// multiplies by the inverse scale.
//
// Swap-AB on CTA pairs (tcgen05 cta_group::2): the vocabulary is the MMA's
// M dimension (256 logit rows per pair, 128 per CTA = one TMEM lane each)
// and the hypothesis rows are its N dimension (up to 160 per work unit; each
// CTA stages half of them and the pair's tensor cores share the halves,
// halving activation traffic and shared-memory reads).  Persistent: a pair
// loops over contiguous (256-vocab tile, 160-row block) work units with two
// TMEM accumulator buffers, so the epilogue of one unit overlaps the
// mainloop of the next.
//
// Epilogue (4 warps, both CTAs): tcgen05.ld 32 rows x 128 vocab at a time,
// bias add, transpose through shared memory, then thread = (row, quarter of
// the vocab): max, sum exp(x - max) and a register top-kk over 32 logits,
// merged across the 4 quarters with warp shuffles.  Per (row, 128-vocab
// tile) it writes (max, sum) and the tile's top-kk — the partial layout the
// select kernel consumes.
#include "common.cuh"
#include "logits_tc.cuh"
#include "tc_common.cuh"

namespace amun {

namespace {

constexpr int kBK = 64;                     // fp16 K elements per 128-byte swizzled row
constexpr int kRowB = kBK * 2;
#ifndef AMUN_LOGIT_STAGES
#define AMUN_LOGIT_STAGES 3
#endif
constexpr int kStages = AMUN_LOGIT_STAGES;
#ifndef AMUN_LOGIT_UNIT_ROWS
#define AMUN_LOGIT_UNIT_ROWS 160
#endif
constexpr int kUnitRows = AMUN_LOGIT_UNIT_ROWS;              // hypothesis rows per work unit (one MMA, N <= 160)
constexpr int kUnitRowsBig = 192;           // units of launches with >= 512 rows (balanced 6-chunk epilogue)
constexpr int kXRows = kUnitRowsBig / 2;    // rows staged by each CTA of the pair (largest unit)
constexpr int kBoxR = 16;                   // activation rows per TMA box
constexpr int kWB = 128 * kRowB;            // one of hi/lo weight tiles
constexpr int kXB = kXRows * kRowB;         // one of hi/lo activation tiles
constexpr int kStageB = 2 * kWB + 2 * kXB;  // 52 KB
constexpr int kAccCols = 256;               // TMEM column offset of accumulator buffer 1
constexpr int kTrQ = 36;                    // floats per vocabulary quarter in a transposed row (32 + pad)
constexpr int kTrRow = 4 * kTrQ;            // floats per transposed row (128 vocab + pad)
constexpr int kTrB = 32 * kTrRow * 4;       // one transpose buffer (32 rows x 128 vocab)
#ifndef AMUN_LOGIT_EPI
#define AMUN_LOGIT_EPI 3
#endif
constexpr int kEpiGroups = AMUN_LOGIT_EPI;               // epilogue warp groups (4 warps each) working on alternate chunks
constexpr int kSmem = kStages * kStageB + kEpiGroups * kTrB + 1024 + 256;
constexpr int kThreads = 64 + 128 * kEpiGroups;  // warp 0 TMA, warp 1 MMA (leader), then the epilogue groups
static_assert(kSmem <= 232448, "shared memory per CTA");

// Register-resident top-KK list ordered by (logit desc, token asc).
template <int KK>
struct RowTop {
  float v[KK];
  int t[KK];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int i = 0; i < KK; ++i) {
      v[i] = -INFINITY;
      t[i] = 0x7fffffff;
    }
  }
  __device__ __forceinline__ bool beats(float x, int n, int i) const {
    return x > v[i] || (x == v[i] && n < t[i]);
  }
  // Insertion of (x, n) where n is larger than every token in the list (a
  // thread inserts its candidates in increasing column order): x enters
  // before the first entry it strictly exceeds, so an equal value keeps the
  // earlier token first.  Every slot's update depends only on the old list
  // (one compare per slot, then selects): no serial chain through the slots.
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

__device__ __forceinline__ bool key_beats(float va, int ta, float vb, int tb) {
  return va > vb || (va == vb && ta < tb);
}

// top.{v,t} <- best KK of (top U partner lane's top), both sorted best-first:
// elementwise best of A[i] and B[P-1-i] is the union's top P as a bitonic
// sequence, which log2(P) half-cleaner stages sort (all steps independent
// compare-exchanges: short dependency chains, no divergence).
template <int KK>
__device__ __forceinline__ void merge_partner(RowTop<KK> &top, int lane_xor) {
  constexpr int P = KK <= 1 ? 1 : KK <= 2 ? 2 : KK <= 4 ? 4 : KK <= 8 ? 8 : 16;
  float ov[KK];
  int ot[KK];
#pragma unroll
  for (int i = 0; i < KK; ++i) {
    ov[i] = __shfl_xor_sync(0xffffffffu, top.v[i], lane_xor);
    ot[i] = __shfl_xor_sync(0xffffffffu, top.t[i], lane_xor);
  }
  float cv[P];
  int ct[P];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const float av = i < KK ? top.v[i] : -INFINITY;
    const int at = i < KK ? top.t[i] : 0x7fffffff;
    const int j = P - 1 - i;
    const float bv = j < KK ? ov[j] : -INFINITY;
    const int bt = j < KK ? ot[j] : 0x7fffffff;
    const bool ta = key_beats(av, at, bv, bt);
    cv[i] = ta ? av : bv;
    ct[i] = ta ? at : bt;
  }
#pragma unroll
  for (int d = P / 2; d >= 1; d /= 2)
#pragma unroll
    for (int i = 0; i < P; ++i)
      if ((i & d) == 0) {
        const int j = i + d;
        const bool sw = key_beats(cv[j], ct[j], cv[i], ct[i]);
        const float vi = cv[i], vj = cv[j];
        const int ti = ct[i], tj = ct[j];
        cv[i] = sw ? vj : vi;
        ct[i] = sw ? tj : ti;
        cv[j] = sw ? vi : vj;
        ct[j] = sw ? ti : tj;
      }
#pragma unroll
  for (int i = 0; i < KK; ++i) {
    top.v[i] = cv[i];
    top.t[i] = ct[i];
  }
}

// Hypothesis rows per work unit: the nm members' accumulators of one unit
// share a 256-column TMEM buffer (member m at column m * rows).
// Launches of >= 512 rows use 192-row units (6 chunks: every epilogue group
// drains two); the unit size only regroups rows, a row's logits and
// partials are the same in any unit.
__host__ __device__ constexpr int unit_rows(int nm, int M) {
  return nm <= 1 ? (M >= 512 ? kUnitRowsBig : kUnitRows) : nm == 2 ? 128 : 64;
}

// Work unit u of a launch: 256-vocab tile vt, rows [row0, row0 + nr); the
// pair's MMA has N = nr rounded up to 32, each CTA stages N / 2 of the rows.
struct Unit {
  int vt, row0, nr, n, h;
  __device__ __forceinline__ Unit(int u, int npass, int M, int ur) {
    vt = u / npass;
    row0 = (u % npass) * ur;
    nr = min(ur, M - row0);
    n = (nr + 31) / 32 * 32;
    h = n / 2;
  }
};

// activation / weight tensor maps of the NMX members of one launch
template <int NMX>
struct MapSet {
  LogitTcMaps m[NMX];
};

template <int KK, int NMX>
__global__ void __launch_bounds__(kThreads, 1)
    logits_pair_kernel(const __grid_constant__ MapSet<NMX> mp, LogitTcArgs a) {
  const CtaClock clk(a.kt);
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = tc::align_smem<1024>(smem_raw);  // stays in the shared address space (LDS/STS)
  float *tr = reinterpret_cast<float *>(smem + kStages * kStageB);  // [group][32][kTrRow]
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + kStages * kStageB + kEpiGroups * kTrB);
  uint64_t *empty = full + kStages;
  uint64_t *tfull = empty + kStages;  // [2] accumulator buffers
  uint64_t *tempty = tfull + 2;       // [2]
  uint32_t *tslot = reinterpret_cast<uint32_t *>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = tc::cluster_rank();
  const int member = (int)(crank & 1);
  const uint32_t leader = crank & ~1u;
  const int pair = blockIdx.x / 2, npairs = gridDim.x / 2;
  const int nm = NMX == 1 ? 1 : a.nm;
  const int ur = unit_rows(nm, a.M);
  const int nvt = (a.N + 255) / 256;
  const int npass = (a.M + ur - 1) / ur;
  const int units = nvt * npass;
  // contiguous units per pair: the two row halves of a vocabulary tile run
  // back to back on the same pair, so the second weight read hits L2
  const int upp = (units + npairs - 1) / npairs;
  const int u_begin = pair * upp, u_end = min(units, u_begin + upp);
  auto nk_of = [&](int mi) { return ((mi == 0 ? a.K : a.K_x[mi - 1]) + kBK - 1) / kBK; };
  constexpr uint16_t kMask = 3;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&tfull[b], 1);
      tc::mbar_init(&tempty[b], 2 * 4 * kEpiGroups);  // every epilogue warp of both CTAs of the pair
    }
    tc::fence_barrier_init();
    for (int mi = 0; mi < nm; ++mi) {
      tc::tma_prefetch(&mp.m[mi].a_hi);
      tc::tma_prefetch(&mp.m[mi].a_lo);
      tc::tma_prefetch(&mp.m[mi].b_hi);
      tc::tma_prefetch(&mp.m[mi].b_lo);
    }
  }
  if (warp == 1) tc::tmem_alloc_pair<512>(tslot);
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    // ---------------- TMA producer (both CTAs; bytes complete on the leader's barrier)
    if (lane == 0) {
      const bool lw = !(a.debug_flags & 1), lx = !(a.debug_flags & 2);
      int it = 0;
      for (int u = u_begin; u < u_end; ++u) {
        const Unit un(u, npass, a.M, ur);
        const int v0 = un.vt * 256 + member * 128;
        const int g = un.row0 + member * un.h;
        const uint32_t bytes = (lw ? 2 * kWB : 0) + (lx ? 2 * un.h * kRowB : 0);
        for (int mi = 0; mi < nm; ++mi) {
        const CUtensorMap *tW_hi = &mp.m[mi].b_hi, *tW_lo = &mp.m[mi].b_lo;
        const CUtensorMap *tX_hi = &mp.m[mi].a_hi, *tX_lo = &mp.m[mi].a_lo;
        const int nk = nk_of(mi);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages;
          if (it >= kStages) tc::mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          if (member == 0) tc::mbar_arrive_expect_tx(&full[s], 2 * bytes);
          const uint32_t bar = tc::mapa_shared(tc::smem_u32(&full[s]), leader);
          uint8_t *st = smem + s * kStageB;
          const int kx = kb * kBK;
          if (lw) {
            tc::tma_load_2d_pair(st, tW_hi, bar, kx, v0);
            tc::tma_load_2d_pair(st + kWB, tW_lo, bar, kx, v0);
          }
          if (lx) {
            for (int r = 0; r < un.h; r += kBoxR) {
              tc::tma_load_2d_pair(st + 2 * kWB + r * kRowB, tX_hi, bar, kx, g + r);
              tc::tma_load_2d_pair(st + 2 * kWB + kXB + r * kRowB, tX_lo, bar, kx, g + r);
            }
          }
        }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (leader CTA, one thread); accumulators
    // alternate between two TMEM buffers so the epilogue of unit t overlaps
    // the mainloop of unit t + 1
    if (lane == 0 && member == 0) {
      int it = 0, ti = 0;
      for (int u = u_begin; u < u_end; ++u, ++ti) {
        const Unit un(u, npass, a.M, ur);
        const int buf = ti & 1;
        const uint32_t idesc = tc::idesc_f16(256, un.n);
        if (ti >= 2) {
          tc::mbar_wait(&tempty[buf], ((ti >> 1) - 1) & 1);  // both epilogues drained this buffer
          tc::tc_fence_after();
        }
        for (int mi = 0; mi < nm; ++mi) {
        const uint32_t acc = tmem + buf * kAccCols + mi * ur;
        const int nk = nk_of(mi);
        for (int kb = 0; kb < nk; ++kb, ++it) {
          const int s = it % kStages;
          tc::mbar_wait(&full[s], (it / kStages) & 1);
          tc::tc_fence_after();
          const uint32_t base = tc::smem_u32(smem + s * kStageB);
#pragma unroll
          for (int k2 = 0; k2 < ((a.debug_flags & 4) ? 0 : kBK / 16); ++k2) {
            const uint32_t koff = k2 * 32;
            const uint64_t awh = tc::desc_kmajor_sw128(base + koff);
            const uint64_t awl = tc::desc_kmajor_sw128(base + kWB + koff);
            const uint64_t bh = tc::desc_kmajor_sw128(base + 2 * kWB + koff);
            const uint64_t bl = tc::desc_kmajor_sw128(base + 2 * kWB + kXB + koff);
            const uint32_t acc0 = (kb | k2) != 0;
            tc::mma_f16_pair(acc, awh, bh, idesc, acc0);
            tc::mma_f16_pair(acc, awh, bl, idesc, 1);
            tc::mma_f16_pair(acc, awl, bh, idesc, 1);
          }
          tc::mma_commit_pair_mc(&empty[s], (uint16_t)(kMask << leader));
        }
        }
        tc::mma_commit_pair_mc(&tfull[buf], (uint16_t)(kMask << leader));
      }
    }
  } else {
    // ---------------- epilogue (both CTAs): group g drains and reduces the
    // 32-row chunks g, g + kEpiGroups, ... of each unit
    const int lg = warp & 3;        // TMEM lane quarter this warp may access
    const int f = lg * 32 + lane;   // vocabulary lane of this thread while draining
    const int g = (warp - 2) / 4;
    const int et = threadIdx.x - 64 - 128 * g;
    const int ri = et >> 2, q = et & 3;  // (row, vocabulary quarter) while reducing
    float *buf = tr + g * (32 * kTrRow);
    int ti = 0, dchunk = 0;
    // per-phase clock stamps (tools/bench_logits_tc.cu) only in builds with
    // AMUN_LOGIT_STAMPS: predicated-off stamps still cost ~6% of the
    // epilogue's issue slots
#ifdef AMUN_LOGIT_STAMPS
    const bool dstamp = a.debug_clock && blockIdx.x == 0 && et == 0 && g == 0;
#else
    constexpr bool dstamp = false;
#endif
    auto stamp = [&](int pt) {
      if (dstamp && dchunk < 64) a.debug_clock[dchunk * 16 + pt] = clock64();
    };
    for (int u = u_begin; u < u_end; ++u, ++ti) {
      const Unit un(u, npass, a.M, ur);
      const int ab = ti & 1;
      const int v0 = un.vt * 256 + member * 128;
      const int nt = un.vt * 2 + member;  // 128-vocab tile index of the partial outputs
      float bias_f[NMX];
#pragma unroll
      for (int mi = 0; mi < NMX; ++mi) {
        const float *bp = mi == 0 ? a.bias : a.bias_x[mi - 1];
        bias_f[mi] = (mi < nm && v0 + f < a.N) ? __ldg(bp + v0 + f) : -INFINITY;
      }
      if (dstamp && dchunk < 64) a.debug_clock[dchunk * 16 + 11] = clock64();
      tc::mbar_wait(&tfull[ab], (ti >> 1) & 1);
      tc::tc_fence_after();
      if (dstamp && dchunk < 64) a.debug_clock[dchunk * 16 + 12] = clock64();
#pragma unroll 1
      // the chunk -> group assignment rotates from unit to unit, so a unit
      // whose chunk count is not a multiple of the group count (160 rows:
      // 5 chunks for 3 groups) does not always leave the same group idle
      for (int c0 = 32 * ((g + ti) % kEpiGroups); c0 < un.n; c0 += 32 * kEpiGroups, ++dchunk) {
        const int m = un.row0 + c0 + ri;
        const bool wr = q == 0 && c0 + ri < un.nr && nt < a.ntiles && !(a.debug_flags & 64);
        // thread (ri, q): logits of row c0 + ri for vocab v0 + 32 q + [0, 32);
        // the quarter pad makes each 8-lane LDS.128 phase hit 8 bank groups
        float *src = buf + ri * kTrRow + q * kTrQ;
        float x[32];   // this member's logits; after the member loop, the member sum
        float g8[4];   // 8-wide group maxima of x
        float mx = -INFINITY, se = 0.f;
        uint32_t allow = ~0u;
        // shortlist (nnet.py:160-163): columns outside the row's sentence
        // list do not exist; the thread's 32 columns are one mask word
        if (a.vmask) {
          const int vq = v0 + q * 32;
          allow = (m < a.M && vq < a.N)
                      ? __ldg(a.vmask + (long long)(m / a.rows_per_sent) * a.mask_words + (vq >> 5))
                      : 0u;
        }
        float xs[NMX > 1 ? 32 : 1];
#pragma unroll 1
        for (int mi = 0; mi < nm; ++mi) {
          if (mi) asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");  // buffer free
          stamp(0);
          {
            float v[32];
            tc::tmem_ld_32x32(tmem + ab * kAccCols + mi * ur + ((uint32_t)(lg * 32) << 16) + c0, v);
            float *dst = buf + lg * kTrQ + lane;
            const float us = mi == 0 ? a.unscale : a.unscale_x[mi - 1];
            float bf = bias_f[0];
#pragma unroll
            for (int j = 1; j < NMX; ++j) bf = mi == j ? bias_f[j] : bf;
#pragma unroll
            for (int i = 0; i < 32; ++i) dst[i * kTrRow] = fmaf(v[i], us, bf);
          }
          stamp(1);
          asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");
          stamp(2);
          if (a.debug_flags & 8) continue;
#pragma unroll
          for (int u4 = 0; u4 < 8; ++u4) {
            const float4 t4 = *reinterpret_cast<const float4 *>(src + 4 * u4);
            x[4 * u4] = t4.x;
            x[4 * u4 + 1] = t4.y;
            x[4 * u4 + 2] = t4.z;
            x[4 * u4 + 3] = t4.w;
          }
          if (a.vmask) {
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = (allow >> i) & 1u ? x[i] : -INFINITY;
          }
          // four 8-wide group maxima, the quarter max, and sum exp(x - max)
          // (ex2-based: x log2 e - max log2 e, one FFMA + MUFU per logit)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            g8[j] = x[8 * j];
#pragma unroll
            for (int i = 1; i < 8; ++i) g8[j] = fmaxf(g8[j], x[8 * j + i]);
          }
          mx = fmaxf(fmaxf(g8[0], g8[1]), fmaxf(g8[2], g8[3]));
          stamp(3);
          se = 0.f;
          if (mx != -INFINITY) {
            const float mxl = mx * 1.4426950408889634f;
#pragma unroll
            for (int i = 0; i < 32; ++i) se += tc::exp2f_approx(fmaf(x[i], 1.4426950408889634f, -mxl));
          }
          // merge (max, sum) over the four quarters of the row (lanes 4 ri .. 4 ri + 3)
#pragma unroll
          for (int o = 1; o <= 2; o <<= 1) {
            const float omx = __shfl_xor_sync(0xffffffffu, mx, o);
            const float ose = __shfl_xor_sync(0xffffffffu, se, o);
            const float nmx = fmaxf(mx, omx);
            // ex2.approx like the per-logit terms (rel. error ~2^-22)
            const float a0 = (mx == -INFINITY) ? 0.f : se * tc::exp2f_approx((mx - nmx) * 1.4426950408889634f);
            const float a1 = (omx == -INFINITY) ? 0.f : ose * tc::exp2f_approx((omx - nmx) * 1.4426950408889634f);
            se = (q & o) ? a1 + a0 : a0 + a1;  // same operand order in both partners
            mx = nmx;
          }
          if (wr) {
            const long long o = (long long)mi * a.pm_stride + (long long)m * a.ntiles + nt;
            a.pmax[o] = mx;
            a.psum[o] = se;
          }
          if constexpr (NMX > 1) {
#pragma unroll
            for (int i = 0; i < 32; ++i) xs[i] = mi == 0 ? x[i] : xs[i] + x[i];
          }
        }
        if (!(a.debug_flags & 8)) {
          if constexpr (NMX > 1) {
            // ensemble: the candidates rank the member sum of the logits
            // (search.py:67-72: mean_m(logit_m - lse_m) orders like sum_m
            // logit_m); the sum replaces this thread's own smem quarter row
#pragma unroll
            for (int i = 0; i < 32; ++i) x[i] = xs[i];
#pragma unroll
            for (int u4 = 0; u4 < 8; ++u4)
              *reinterpret_cast<float4 *>(src + 4 * u4) = make_float4(x[4 * u4], x[4 * u4 + 1], x[4 * u4 + 2], x[4 * u4 + 3]);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              g8[j] = x[8 * j];
#pragma unroll
              for (int i = 1; i < 8; ++i) g8[j] = fmaxf(g8[j], x[8 * j + i]);
            }
          }
          const float h0 = fmaxf(g8[0], g8[1]), h1 = fmaxf(g8[2], g8[3]);
          // Threshold: the KK-th largest of the row's 8 half maxima (16 group
          // maxima for KK > 8) is a lower bound on the row's KK-th largest
          // logit (those maxima are distinct logits), so only logits >= thr
          // can be in the tile's top-KK.
          stamp(4);
          float thr = -INFINITY;
          if constexpr (KK <= 8) {
            float hm[8];
            const int lb = lane & ~3;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              hm[2 * j] = __shfl_sync(0xffffffffu, h0, lb + j);
              hm[2 * j + 1] = __shfl_sync(0xffffffffu, h1, lb + j);
            }
            // optimal 19-comparator sorting network for 8 (descending); only
            // position KK - 1 is read, so the compiler drops the comparator
            // outputs that do not feed it
            constexpr int kNet[19][2] = {{0, 2}, {1, 3}, {4, 6}, {5, 7}, {0, 4}, {1, 5}, {2, 6},
                                         {3, 7}, {0, 1}, {2, 3}, {4, 5}, {6, 7}, {2, 4}, {3, 5},
                                         {1, 4}, {3, 6}, {1, 2}, {3, 4}, {5, 6}};
#pragma unroll
            for (int c = 0; c < 19; ++c) {
              const float hi = fmaxf(hm[kNet[c][0]], hm[kNet[c][1]]), lo = fminf(hm[kNet[c][0]], hm[kNet[c][1]]);
              hm[kNet[c][0]] = hi;
              hm[kNet[c][1]] = lo;
            }
            thr = hm[KK - 1];
          } else {
            // KK > 8 (beam 9..16): the KK-th largest of the row's 16 group
            // maxima (16 distinct logits) bounds the tile's KK-th largest
            // logit from below; 17 - KK bubble passes sink the smallest
            // maxima to the end, leaving the KK-th largest at KK - 1
            float hm[16];
            const int lb = lane & ~3;
#pragma unroll
            for (int j = 0; j < 4; ++j)
#pragma unroll
              for (int u = 0; u < 4; ++u) hm[4 * j + u] = __shfl_sync(0xffffffffu, g8[u], lb + j);
#pragma unroll
            for (int p = 0; p < 17 - KK; ++p)
#pragma unroll
              for (int j = 0; j < 15 - p; ++j) {
                const float hi = fmaxf(hm[j], hm[j + 1]), lo = fminf(hm[j], hm[j + 1]);
                hm[j] = hi;
                hm[j + 1] = lo;
              }
            thr = hm[KK - 1];
          }
          stamp(5);
          unsigned cand = 0;
#pragma unroll
          for (int i = 0; i < 32; ++i) cand |= (x[i] >= thr ? 1u : 0u) << i;
          cand &= allow;  // masked columns are -inf here but not in the smem copy
          stamp(6);
          RowTop<KK> top;
          top.init();
          const int tbase = v0 + q * 32;
#pragma unroll 1
          while (cand) {  // few candidates per quarter; two per trip (both loads in flight)
            const int i0 = __ffs(cand) - 1;
            cand &= cand - 1;
            const int i1 = cand ? __ffs(cand) - 1 : -1;
            cand &= cand - 1;
            const float x0 = src[i0], x1 = src[i1 < 0 ? i0 : i1];
            top.insert(x0, tbase + i0);
            if (i1 >= 0) top.insert(x1, tbase + i1);
          }
          stamp(7);
          // merge the four quarters' lists of the row
#pragma unroll
          for (int o = 1; o <= 2; o <<= 1) merge_partner(top, o);
          stamp(8);
          if (wr) {
            const long long base = ((long long)m * a.ntiles + nt) * a.kk;
#pragma unroll
            for (int i = 0; i < KK; ++i)
              if (i < a.kk) {
                const bool ok = top.v[i] != -INFINITY;
                a.cval[base + i] = ok ? top.v[i] : -INFINITY;
                a.ctok[base + i] = ok ? (a.vid ? __ldg(a.vid + top.t[i]) : top.t[i]) : -1;
              }
          }
        }
        stamp(9);
        asm volatile("bar.sync %0, 128;" ::"r"(1 + g) : "memory");  // buffer free for the next chunk
        stamp(10);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_remote(&tempty[ab], leader);
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::cluster_sync();  // no CTA leaves while its pair may still signal it
  clk.done();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc_pair<512>(tmem);
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

// work units per pair: (256-vocab tiles x row passes) spread evenly, about
// AMUN_LOGIT_UNITS (default 9, swept: cfg2 / cfg5 / cfg1) per pair -- long
// enough persistent loops that the epilogue of one unit hides behind the
// next unit's MMAs -- and at most AMUN_LOGIT_PAIRS (default 40) pairs.
int logit_pairs(int units) {
  static int cap = [] {
    const char *e = getenv("AMUN_LOGIT_PAIRS");
    return e ? std::max(1, atoi(e)) : 40;
  }();
  static int upp = [] {
    const char *e = getenv("AMUN_LOGIT_UNITS");
    return e ? std::max(1, atoi(e)) : 9;
  }();
  const int pairs = std::max(1, std::min({cap, 74, ceil_div(units, upp)}));
  const int per = ceil_div(units, pairs);
  return ceil_div(units, per);
}

template <int KK, int NMX>
void launch_t(const LogitTcMaps *maps, const LogitTcArgs &a, cudaStream_t st) {
  auto kern = logits_pair_kernel<KK, NMX>;
  MapSet<NMX> mp;
  for (int i = 0; i < NMX; ++i) mp.m[i] = maps[i < a.nm ? i : 0];
  static bool attr[64] = {};
  int dev = 0;
  AMUN_CUDA(cudaGetDevice(&dev));
  if (dev >= 64 || !attr[dev]) {
    AMUN_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmem));
    if (dev < 64) attr[dev] = true;
  }
  const int units = ceil_div(a.N, 256) * ceil_div(a.M, unit_rows(NMX == 1 ? 1 : a.nm, a.M));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2 * logit_pairs(units));
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = 2;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  last_launch_ctas() = (int)cfg.gridDim.x;
  LogitTcArgs ak = a;
  ak.kt = ktime_ptr();
  AMUN_CUDA(cudaLaunchKernelEx(&cfg, kern, mp, ak));
}

}  // namespace

int logits_tc_tile_n() { return 128; }

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

CUtensorMap make_tma_2d_f16(const __half *ptr, int inner, int outer, int row_stride_elems, int box_inner,
                            int box_outer) {
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)inner, (cuuint64_t)outer};
  cuuint64_t strides[1] = {(cuuint64_t)row_stride_elems * 2};
  cuuint32_t box[2] = {(cuuint32_t)box_inner, (cuuint32_t)box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<__half *>(ptr), dims, strides, box,
                           estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           box_inner * 2 == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw Error(2, "cuTensorMapEncodeTiled (f16) failed: " + std::to_string((int)r));
  return m;
}

LogitTcMaps make_logit_maps(const __half *t_hi, const __half *t_lo, int R, int K, int ldt, const __half *w_hi,
                            const __half *w_lo, int ldw, int V) {
  LogitTcMaps m;
  m.a_hi = make_tma_2d_f16(t_hi, K, R, ldt, kBK, kBoxR);
  m.a_lo = make_tma_2d_f16(t_lo, K, R, ldt, kBK, kBoxR);
  m.b_hi = make_tma_2d_f16(w_hi, K, V, ldw, kBK, 128);
  m.b_lo = make_tma_2d_f16(w_lo, K, V, ldw, kBK, 128);
  return m;
}

template <int NMX>
void launch_kk(const LogitTcMaps *maps, const LogitTcArgs &a, cudaStream_t st) {
  // list size >= kk (a sorted top-KK list contains the top-kk as its prefix)
  switch (a.kk) {
    case 1: launch_t<1, NMX>(maps, a, st); break;
    case 2: launch_t<2, NMX>(maps, a, st); break;
    case 3: launch_t<3, NMX>(maps, a, st); break;
    case 4: launch_t<4, NMX>(maps, a, st); break;
    case 5: launch_t<5, NMX>(maps, a, st); break;
    case 6: launch_t<6, NMX>(maps, a, st); break;
    case 7: case 8: launch_t<8, NMX>(maps, a, st); break;
    case 9: case 10: launch_t<10, NMX>(maps, a, st); break;
    case 11: case 12: launch_t<12, NMX>(maps, a, st); break;
    case 13: case 14: case 15: case 16: launch_t<16, NMX>(maps, a, st); break;
    default: throw Error(4, "tensor-core logit path supports beam <= 16");
  }
}

void launch_logits_tc(const LogitTcMaps &maps, const LogitTcArgs &a, cudaStream_t st) {
  if (a.nm != 1) throw Error(4, "launch_logits_tc: single-member launch");
  launch_kk<1>(&maps, a, st);
}

void launch_logits_tc_ens(const LogitTcMaps *maps, const LogitTcArgs &a, cudaStream_t st) {
  if (a.nm < 2 || a.nm > kLogitMembers) throw Error(4, "tensor-core logit ensembles take 2..4 members");
  launch_kk<kLogitMembers>(maps, a, st);
}

}  // namespace amun

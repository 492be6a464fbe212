// Tensor-core (tcgen05, 3xFP16) logit projection with fused log-softmax
// partials and per-row top-k; see logits_tc.cu.
#pragma once

#include <cuda.h>
#include <cuda_fp16.h>

namespace amun {

struct LogitTcArgs {
  int M, N, K;         // rows (hypotheses), vocabulary, d_emb
  const float *bias;   // b_logit [N]
  int kk, ntiles;      // candidates kept per (row, tile); ceil(N / tile_n)
  float unscale;       // 2^-(activation shift + weight shift) of the 3xFP16 operands
  float *pmax, *psum;  // [M][ntiles]
  float *cval;         // [M][ntiles][kk]
  int *ctok;
  // optional per-sentence vocabulary masks (shortlists, nnet.py:160-163):
  // bit v of vmask[(row / rows_per_sent) * mask_words + v / 32] allows token v
  const uint32_t *vmask = nullptr;
  int mask_words = 0, rows_per_sent = 1;
  // optional column -> vocabulary id map (gathered shortlist columns, strictly
  // ascending): candidate tokens are reported as vid[column]
  const int *vid = nullptr;
  // ensembles (search.py:56-72) fused in one launch: members 1 .. nm-1 run
  // their own logit GEMM (K_x, bias_x, unscale_x, their own tensor maps);
  // per member the (max, sum) partials go to pmax/psum + m * pm_stride and
  // the candidates are the row's top-kk of the member SUM of logits (the
  // ensemble log-prob mean_m(logit_m - lse_m) orders like that sum)
  int nm = 1;
  int K_x[3] = {0, 0, 0};
  const float *bias_x[3] = {nullptr, nullptr, nullptr};
  float unscale_x[3] = {0.f, 0.f, 0.f};
  long long pm_stride = 0;
  unsigned long long *kt = nullptr;  // optional CTA-time accounting (common.cuh CtaClock)
  int debug_flags = 0;  // microbenchmark knobs: 1 skip A loads, 2 skip B loads, 4 skip MMA, 8 skip epilogue
  long long *debug_clock = nullptr;  // microbenchmark: per-chunk clock64 stamps of CTA 0
};

struct LogitTcMaps {
  CUtensorMap a_hi, a_lo, b_hi, b_lo;
};
constexpr int kLogitMembers = 4;  // ensemble members of one fused logit launch

int logits_tc_tile_n();
// fp32 2D tensor map; the swizzle follows the box row width (64 B -> SW64,
// 128 B -> SW128)
CUtensorMap make_tma_2d_f32(const float *ptr, int inner, int outer, int row_stride_elems, int box_inner,
                            int box_outer);
// fp16 2D tensor map (row pitch must be a multiple of 8 elements)
CUtensorMap make_tma_2d_f16(const __half *ptr, int inner, int outer, int row_stride_elems, int box_inner,
                            int box_outer);
// t_hi/t_lo: [R, ldt] (first K columns used); w_hi/w_lo: [V, ldw] (logit rows)
LogitTcMaps make_logit_maps(const __half *t_hi, const __half *t_lo, int R, int K, int ldt, const __half *w_hi,
                            const __half *w_lo, int ldw, int V);
void launch_logits_tc(const LogitTcMaps &maps, const LogitTcArgs &a, cudaStream_t st);
// Rows layout (logits_rows.cu): hypothesis rows are the MMA's M, one epilogue
// thread per row, partials per (row, 128-vocab tile); single member.
constexpr int kLogitRowsTileN = 128;
LogitTcMaps make_logit_rows_maps(const __half *t_hi, const __half *t_lo, int R, int K, int ldt, const __half *w_hi,
                                 const __half *w_lo, int ldw, int V);
void launch_logits_rows(const LogitTcMaps &maps, const LogitTcArgs &a, cudaStream_t st);
// a.nm members (2 .. kLogitMembers), maps[m] = member m's activation / weight maps
void launch_logits_tc_ens(const LogitTcMaps *maps, const LogitTcArgs &a, cudaStream_t st);

}  // namespace amun

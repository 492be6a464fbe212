// Split-K tensor-core GEMM producing fp32 partials (see gemm_tc.cu).
#pragma once

#include <cuda.h>

#include "logits_tc.cuh"  // make_tma_2d_f32

namespace amun {

struct GemmTcArgs {
  int M, N;
  int nk1, nk2;       // 16-wide K blocks in A segment 1 / 2
  int k_off2;         // B's K coordinate where segment 2 starts
  int kb_per_split;
  float *out;         // partials [splits][M][N]
};

struct GemmTcMaps {
  CUtensorMap a1h, a1l, a2h, a2l, bh, bl;
  int k1, k2, N;
};

int gemm_tc_tile_n();
// A segment s: hi/lo [M rows, k_s columns] with row pitch lda_s (elements);
// B: hi/lo [N rows, Kb = k1 + k2 columns] (K-major weights).
GemmTcMaps make_gemm_tc_maps(const float *a1h, const float *a1l, int k1, int lda1, const float *a2h,
                             const float *a2l, int k2, int lda2, int M, const float *bh, const float *bl, int N,
                             int Kb);
int gemm_tc_splits(const GemmTcMaps &maps, int target_ctas);
void launch_gemm_tc_partial(const GemmTcMaps &maps, int M, int splits, float *out, cudaStream_t st);

}  // namespace amun

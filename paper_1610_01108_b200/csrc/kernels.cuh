// Non-GEMM kernels of the decode path: MLP attention, encoder helpers,
// beam initialisation, and the fused select / beam-update / state-gather.
#pragma once

#include "common.cuh"

namespace amun {

// ---------------------------------------------------------------- attention
// nnet.py:132-141 for a batch of hypothesis rows (sentence b = r /
// rows_per_sent): e_j = v . tanh(P_bj + q_r), masked softmax over j < len[b],
// ctx = sum_j a_j H_bj written straight into the decoder input buffer.  With
// an energy scratch buffer: one launch computing the energies of every
// (sentence, position) pair and one computing softmax + context per
// (sentence, column block); without: one CTA per row.
struct AttnArgs {
  const float *Q;  // [R, ldq]
  int ldq;
  const float *P;  // [B][jmax][da]
  const float *H;  // [B][jmax][2 dh]
  const float *v;  // [da]
  const int *len;
  int jmax, da, dh2, rows_per_sent;
  const int *n_act, *done;  // optional beam masks
  float *ctx;
  int ldctx;
  float *alpha;  // optional [R][jmax]
  __half *ctx_hi = nullptr, *ctx_lo = nullptr;  // optional 3xFP16 split (row pitch ldctx_h)
  int ldctx_h = 0;
  float *energy = nullptr;  // scratch [R][jmax]: enables the two-phase sentence kernels
  const float *EQ = nullptr;  // e^{2q} rows (same layout as Q), from the query GEMM epilogue
  unsigned long long *kt = nullptr;  // optional CTA-time accounting (common.cuh CtaClock)
  // Projected-context mode (su != nullptr; decode.cu step_rows): H rows are
  // the annotations' products with the decoder's context weights,
  // [h C_z | h C_r | h C_h | h W_o^c] (row pitch dh2, 3 dh + de used), so the
  // attention-weighted sum is the context's contribution to every gate and
  // to the deep output, and the kernel ends with the GRU gate math
  // (nnet.py:66-69): z -> Z, r * s -> RH split, the input half of h~ -> XH,
  // and the deep output's context + y term -> CO.
  const float *su = nullptr;   // [R][2dh] s U_{z,r} (EpiQS)
  const int *qrow = nullptr;   // optional [R]: row of Q / EQ / su to use (the parent's, when the
                               // previous step's deep-output GEMM computed them from s')
  const float *S = nullptr;    // state rows (pitch lds)
  int lds = 0;
  const int *tok = nullptr;    // [R] previous token
  const float *ywg = nullptr;  // [V][3dh] E_trg W^y_{z,r,h}
  const float *ywo = nullptr;  // [V][de] E_trg W_o^y
  const float *bg = nullptr;   // [3dh]
  float *Z = nullptr, *XH = nullptr;  // [R][dh]
  __half *RHh = nullptr, *RHl = nullptr;  // [R][dh]
  float *CO = nullptr;         // [R][ldco]
  int dh = 0, de = 0, ldco = 0;
};
// returns the number of kernels launched
int launch_attention(const AttnArgs &a, int R, cudaStream_t st);

// ---------------------------------------------------------------- encoder
// masked mean over real positions: out[b] = sum_{j < len_b} Hann[b, j] / len_b
void launch_masked_mean(const float *Hann, const int *len, int B, int jmax, int dh2, float *out,
                        cudaStream_t st);

// ---------------------------------------------------------------- beam state
struct BeamState {
  int B, k, cap_max, fin_cap;
  int *n_act;        // [B]
  double *score;     // [B*k]
  int *tok;          // [B*k] last emitted token per slot
  int *done;         // [B]
  int *steps;        // [B]
  const int *cap;    // [B]
  int *fin_n;        // [B]
  double *fin_score; // [B*fin_cap]
  int *fin_t, *fin_par;
  double *best_fin;  // [B]
  int *bp_tok, *bp_par;  // [B][cap_max][k]
  int *n_done;       // [1] sentences finished so far
  int *qrow = nullptr;  // [B*k] optional: row of the previous step each row continues (its parent)
};

constexpr int kMaxModels = 8;  // ensemble members on the device path

// Row layout of one ensemble member's decoder buffers.  Members may differ
// in d_emb / d_h / d_att (the reference runs one Forward per model,
// search.py:150-152), so every stride is per member.
struct RowDims {
  int ldxs, de, dh, s_off;  // XS = [y | c | s] row pitch and offsets
  // 3xFP16 split copies of XS in the padded layout: row pitch ldxh, XS
  // column c at c + (c >= de ? hpad : 0)
  int ldxh, hpad;
  int y = 1;  // 0: the step reads y only through per-token tables (projected context): no y gather
  int split = 1;  // 0: nothing reads the gathered rows' fp16 splits (query folded forward): fp32 only
};

struct ModelRows {  // per-model decoder row buffers (device arrays of pointers)
  float *const *XS;       // [R][ldxs] = [y | c | s]
  const float *const *Sn; // [R][dh]   s' of this step
  const float *const *E_trg;
  float *const *fin_states;  // optional [B][fin_cap][dh]
  int n_models;
  __half *const *XSh = nullptr;  // optional split copies (per model)
  __half *const *XSl = nullptr;
  RowDims dim[kMaxModels];
};

// XS rows of every sentence: slot 0 <- [E_trg[EOS] | 0 | s0_b], others 0;
// beam: one hypothesis, score 0, prev token EOS (search.py:153-158).
void launch_init_beam(const BeamState &bs, const ModelRows &mr, const float *const *S0, cudaStream_t st);

struct SelectArgs {
  int kk, fused, V;
  // fused-mode inputs (single model): per (row, N-tile) partial lse + top-kk
  const float *pmax, *psum, *cval;
  const int *ctok;
  int ntiles, M;
  // ensembles fused in the logit kernel: members' (max, sum) partial sets at
  // pmax / psum + m * pm_stride; cval holds the member sum of the logits
  int nm_fused = 1;
  long long pm_stride = 0;
  // full-mode inputs: logits per model [R][ldl]
  const float *const *L;
  int ldl;
  const int *sl_ids, *sl_off, *sl_len;  // optional per-sentence shortlists
  double *cand_lp;  // scratch [B*k*kk]
  int *cand_tok;
  unsigned long long *dbg = nullptr;  // profiling: summed clock64 per phase [6] (env AMUN_DEBUG_SELECT)
  unsigned long long *kt = nullptr;   // optional CTA-time accounting (common.cuh CtaClock)
};
// search.py:161-198 for one step of every sentence of the bucket.
void launch_select(const SelectArgs &sa, const BeamState &bs, const ModelRows &mr, cudaStream_t st);

// hook helpers (full logits): lse over (optionally shortlisted) columns and
// logp[r, i] = L[r, id_i] - lse_r
void launch_logp_rows(const float *L, int ldl, int R, int V, const int *sl, int n_sl, double *logp,
                      cudaStream_t st);

}  // namespace amun

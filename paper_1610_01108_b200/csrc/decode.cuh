// Device model handle and the decode / hook drivers behind the C ABI.
#pragma once

#include <vector>

#include "../../include/amun_b200.h"
#include "common.cuh"

// Device-resident model in the fused layouts the kernels consume.  All
// fp32, row-major, K rows x N cols ("B" operands of C = A * B).
struct amun_model {
  int device = 0;
  amun_dims d{};
  int xs_w = 0;  // decoder row width [y | c | s] = d_emb + 3 d_h
  float *E_src = nullptr, *E_trg = nullptr;
  float *Wenc = nullptr, *benc = nullptr;  // [de, 6dh], [6dh]  (fwd z r h | bwd z r h)
  float *Uzr = nullptr, *Uh = nullptr;     // [2][dh][2dh], [2][dh][dh]
  float *W_att_h = nullptr, *W_init = nullptr, *b_init = nullptr, *W_att_s = nullptr, *v_att = nullptr;
  float *Wg = nullptr, *bg = nullptr;      // [de+3dh, 3dh], [3dh]
  float *Uh_dec = nullptr;                 // [dh, dh]
  float *Wout = nullptr, *b_out = nullptr; // [de+3dh, de], [de]
  float *W_logit = nullptr, *b_logit = nullptr;  // [de, V], [V]
  // tensor-core (3xFP16, common.cuh split_h) copies, K-major [N, Kpitch]
  // fp16 hi/lo, with the epilogue inverse scales us_*; the decoder-row
  // weights use the padded row layout [y | pad to dep | c | s] (pitch xsp)
  bool tc_ok = false;    // dims / activation range allow the tensor-core path
  bool tc_gemm = false;  // decoder-step GEMMs on tensor cores
  int dep = 0, xsp = 0;  // d_emb rounded up to 8; padded decoder-row pitch
  __half *Wl_hi = nullptr, *Wl_lo = nullptr;    // W_logit^T [V, dep]
  __half *Wq_hi = nullptr, *Wq_lo = nullptr;    // W_att_s^T [da, dh]
  // [W_att_s | U_z | U_r]^T [da + 2dh, dh]: the attention query and the
  // state's gate products in one GEMM (projected-context step, decode.cu)
  __half *Wqs_hi = nullptr, *Wqs_lo = nullptr;
  float us_qs = 1.f;
  // [W_o^s | 0 | W_att_s | U_z | U_r]^T [dep + da + 2dh, dh]: the deep output
  // and the NEXT step's query + gate products of s' in one GEMM (columns
  // [0, d_e) deep output, [dep, ...) the Wqs block)
  __half *Wdq_hi = nullptr, *Wdq_lo = nullptr;
  float us_dq = 1.f;
  // [W_att_h | C_z | C_r | C_h | W_o^c | 0]^T [da + 3dh + dep, 2dh]: precomp_att
  // and the projected annotations HX of a bucket in one GEMM over the split annotations
  __half *Wph_hi = nullptr, *Wph_lo = nullptr;
  float us_ph = 1.f;
  __half *Wg_hi = nullptr, *Wg_lo = nullptr;    // Wg^T      [3dh, xsp]
  __half *Uhd_hi = nullptr, *Uhd_lo = nullptr;  // U_h^T     [dh, dh]
  __half *Wo_hi = nullptr, *Wo_lo = nullptr;    // Wout^T    [de, xsp]
  float us_l = 1.f, us_q = 1.f, us_g = 1.f, us_u = 1.f, us_o = 1.f;
  // embedding rows through the decoder's y weights, per target token (tensor-
  // core path): the step GEMMs then run over [c | s] only and the epilogues
  // add the gathered row (y = E_trg[previous token] is a table lookup)
  float *XWenc = nullptr;  // [Vs, 6 dh] = E_src [W_{z,r,h} fwd | bwd] + b (encode-ahead)
  float *YWg = nullptr;  // [V, 3 dh] = E_trg W_{z,r,h}^y
  float *YWo = nullptr;  // [V, de]   = E_trg W_out_y
  // encoder: recurrent weights of both directions stacked along K (the
  // recurrence runs both directions as one block-structured GEMM, rows
  // [fwd sentences ; bwd sentences]) and W_att_h^T for precomp_att
  __half *Uzr_hi = nullptr, *Uzr_lo = nullptr;      // [2dh, 2dh]  (N = z|r, K = fwd|bwd state)
  __half *Uh_hi = nullptr, *Uh_lo = nullptr;        // [dh, 2dh]
  __half *Watth_hi = nullptr, *Watth_lo = nullptr;  // [da, 2dh]
  __half *Wenc_hi = nullptr, *Wenc_lo = nullptr;    // [6dh, dep] input projection, both directions
  float us_ea = 1.f, us_eb = 1.f, us_p = 1.f, us_x = 1.f;
  // encode-ahead recurrence (decode.cu encode_ahead): per direction the input
  // projection fused into the recurrent GEMMs, K-major over the padded row
  // [x (dep) | state (dh)]: phase A [W_z W_r ; U_z U_r] -> [2dh, dep + dh],
  // phase B [W_h ; U_h] -> [dh, dep + dh]
  __half *Efa_hi[2] = {}, *Efa_lo[2] = {}, *Efb_hi[2] = {}, *Efb_lo[2] = {};
  float us_efa[2] = {1.f, 1.f}, us_efb[2] = {1.f, 1.f};
  int64_t bytes = 0;
  bool live = false;  // counted in the device's live-handle count (api.cu)
  std::vector<void *> allocs;
  cudaStream_t stream = nullptr;
};

namespace amun {

amun_result *decode_run(const std::vector<amun_model *> &ms, const int32_t *src_ids, const int32_t *src_len,
                        int n_sent, const int32_t *sl_ids, const int32_t *sl_len, const amun_decode_opts &o,
                        amun_bucket_done_fn on_bucket = nullptr, void *user = nullptr);

// free the pooled decode lanes of a device (last model handle destroyed)
void release_device_lanes(int dev);

void hook_encode(amun_model *m, const int32_t *ids, int J, float *h_out, float *p_out, float *s0_out);

void hook_init_state(amun_model *m, const float *h, int J, float *s0_out);

void hook_gru_cell(int device, int d_in, int d_h, const float *const *W, const float *const *U,
                   const float *const *b, int R, const float *x, const float *h, float *h_out);

// y_prev == nullptr -> attention only (alpha_out, ctx_out)
void hook_step(amun_model *m, const float *s, const int32_t *y_prev, int R, const float *h, const float *p,
               int J, const int32_t *sl, int n_sl, float *s_out, double *logp_out, float *alpha_out,
               float *ctx_out);

// production-kernel parity hooks (the tensor-core kernels amun_decode runs)
void hook_step_tc(amun_model *m, int B, int k, const float *s, const int32_t *y_prev, const float *h,
                  const float *p, const int32_t *lens, int jmax, int kk, float *s_out, float *pmax_out,
                  float *psum_out, float *cval_out, int32_t *ctok_out, float *alpha_out);
void hook_encode_batch(amun_model *m, const int32_t *ids, const int32_t *lens, int B, int jmax, bool production,
                       float *h_out, float *p_out, float *s0_out);

}  // namespace amun

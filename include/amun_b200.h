/*
 * amun_b200.h — C ABI of the B200-native beam-search decoder.
 *
 * The reference (`beamnmt`, pure Python/numpy, /root/reference/pkg/src) has no
 * FFI: its compute seams are Python calls.  Each entry point below names the
 * reference interface it replaces; `paper_1610_01108_b200/_lib.py` binds them
 * with ctypes exactly as a maintainer would bind them into the reference
 * (see INTEGRATION.md).
 *
 * Conventions
 *   - plain C types only: host pointers, sizes, status codes; no torch types.
 *   - every function returns AMUN_OK (0) or an AMUN_ERR_* code; the message of
 *     the last failure on the calling thread is amun_last_error().
 *   - AMUN_ERR_INVALID maps to the reference's ValueError, everything else to
 *     RuntimeError on the Python side.
 *   - float tensors are row-major float32; log-probabilities and beam scores
 *     are float64 like the reference.
 *   - a model handle is bound to one device and is used by one host thread at
 *     a time (the caller serialises); different handles/devices run
 *     concurrently.
 */
#ifndef AMUN_B200_H_
#define AMUN_B200_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AMUN_OK 0
#define AMUN_ERR_INVALID 1     /* bad arguments  -> ValueError   */
#define AMUN_ERR_CUDA 2        /* CUDA failure   -> RuntimeError */
#define AMUN_ERR_OOM 3         /* device OOM     -> RuntimeError */
#define AMUN_ERR_UNSUPPORTED 4 /* outside limits -> RuntimeError */

typedef struct amun_model amun_model;

/* ModelConfig (model.py:45-63): d_att already resolved (never 0). */
typedef struct {
  int32_t v_src, v_trg, d_emb, d_h, d_att;
} amun_dims;

/* DecodeOptions (search.py:44-53) plus device batching controls. */
typedef struct {
  int32_t beam_size;        /* >= 1 */
  int32_t max_len_factor;   /* cap = factor * J + offset, must be >= 1 */
  int32_t max_len_offset;
  int32_t length_normalize; /* rank by score/len (final ranking only) */
  int32_t n_best;           /* >= 1 */
  int32_t want_states;      /* also return Hypothesis.states rows */
  int32_t max_batch;        /* sentences per length bucket (0 -> 64) */
  int32_t force_full_logits;/* 1: materialise logits (debug/parity path) */
  int32_t profile;          /* bitmask of AMUN_K_* classes whose launches are CUDA-event timed */
} amun_decode_opts;

/* kernel classes timed when amun_decode_opts.profile is set */
#define AMUN_K_ENCODER 0  /* input projection, recurrence, precomp, init */
#define AMUN_K_QUERY 1    /* s W_att_s */
#define AMUN_K_ATTN 2     /* MLP attention + context */
#define AMUN_K_GRU_A 3    /* [y c s] x [W_zr|W_h ; U_zr] + gates */
#define AMUN_K_GRU_B 4    /* (r*s) U_h + state update */
#define AMUN_K_OUT 5      /* deep output */
#define AMUN_K_LOGIT 6    /* logits + log-softmax partials + top-k */
#define AMUN_K_SELECT 7   /* beam select / update / gather */
#define AMUN_K_CLASSES 8
/* amun_decode_opts.profile flag: device CTA-time accounting in the normal
 * (multi-lane, graph-replay) mode -- kernel_ms[c] = summed CTA lifetimes
 * (globaltimer, ms) and kernel_ctas[c] = CTAs of the class's tensor-core,
 * attention and select kernels; no per-launch events, no single-lane mode */
#define AMUN_PROFILE_CTA_TIME 0x40000000

/* Result of amun_decode: per sentence up to n_best hypotheses, already
 * ranked by (-rank_score, tokens) like search.py:215. */
typedef struct {
  int32_t n_sent, n_models, d_h;
  int64_t n_hyp;
  int32_t *hyp_offsets;  /* [n_sent + 1] */
  double *scores;        /* [n_hyp] */
  int32_t *finished;     /* [n_hyp] */
  int64_t *tok_offsets;  /* [n_hyp + 1] */
  int32_t *tokens;       /* [tok_offsets[n_hyp]] */
  float *states;         /* [n_hyp * n_models * d_h] or NULL */
  /* run statistics */
  int64_t decoder_steps;    /* bucket-steps executed on the device */
  int64_t kernel_launches;  /* kernels launched by this call */
  double device_ms;         /* device time of the decode (CUDA events) */
  int64_t h2d_bytes, d2h_bytes;  /* host<->device bytes moved by the call */
  double kernel_ms[AMUN_K_CLASSES];     /* profile: summed launch durations */
  int64_t kernel_count[AMUN_K_CLASSES]; /* profile: launches per class */
  double host_setup_ms;     /* host time before the first device event (buckets, lanes, workspace) */
  double host_post_ms;      /* host time after the last device event (result assembly) */
  int64_t kernel_ctas[AMUN_K_CLASSES];  /* profile: tensor-core CTAs launched per class */
} amun_result;

/* ---- library / device ------------------------------------------------ */
const char *amun_last_error(void);
int amun_version(void);
int amun_device_count(int32_t *n);

/* ---- model handle: replaces Forward.for_params (nnet.py:102-108) ------
 * tensors: n_tensors == 40 host float32 pointers in schema order
 * (model.py:94-117), each contiguous with the schema's rows x cols.  The
 * library COPIES them to the device (the caller's arrays stay read-only,
 * model.py:156) and builds its own fused/padded layouts. */
int amun_model_create(int32_t device, const amun_dims *dims, const float *const *tensors,
                      int32_t n_tensors, amun_model **out);
int amun_model_destroy(amun_model *m);
int amun_model_device_bytes(const amun_model *m, int64_t *bytes);

/* ---- batched decode: replaces beam_search (search.py:116-216) as called
 * by Engine.translate_corpus (engine.py:181-221) -----------------------
 * models: n_models handles on the same device (ensemble, search.py:56-72).
 * src_ids: concatenated source ids (host), src_len[n_sent] >= 1 each.
 * shortlist_ids/shortlist_len: optional per-sentence ascending global ids
 * (shortlist.py:27-59), NULL for the full vocabulary. */
int amun_decode(amun_model *const *models, int32_t n_models, const int32_t *src_ids,
                const int32_t *src_len, int32_t n_sent, const int32_t *shortlist_ids,
                const int32_t *shortlist_len, const amun_decode_opts *opts, amun_result **out);
int amun_result_free(amun_result *r);
/* Streaming variant: as amun_decode, and after each length bucket finishes
 * (while later buckets still decode) calls on_bucket(user, partial, idx):
 * `partial` holds the final hypotheses of partial->n_sent sentences whose
 * input positions are idx[0 .. n_sent); it and idx are valid during the
 * call only.  Lets the caller post-process (detokenise) while the device
 * works; the callback runs on the calling thread and should be short. */
typedef void (*amun_bucket_done_fn)(void *user, const amun_result *partial, const int32_t *idx);
int amun_decode_stream(amun_model *const *models, int32_t n_models, const int32_t *src_ids,
                       const int32_t *src_len, int32_t n_sent, const int32_t *shortlist_ids,
                       const int32_t *shortlist_len, const amun_decode_opts *opts, amun_bucket_done_fn on_bucket,
                       void *user, amun_result **out);

/* ---- per-step parity hooks (host pointers) ---------------------------- */
/* Forward.encode + init_state_row (nnet.py:110-130):
 * h_out [J, 2*d_h], p_out [J, d_att], s0_out [d_h]. */
int amun_encode(amun_model *m, const int32_t *ids, int32_t J, float *h_out, float *p_out,
                float *s0_out);
/* Forward.init_state_row (nnet.py:128-130): h [J, 2 d_h] -> s0 [d_h]. */
int amun_init_state(amun_model *m, const float *h, int32_t J, float *s0_out);
/* gru_step (nnet.py:177-185 / _GruWeights.step_rows nnet.py:66-70) for a
 * standalone cell on `device`: W[3] = {W_z, W_r, W_h} [d_in, d_h],
 * U[3] = {U_z, U_r, U_h} [d_h, d_h], b[3] [d_h]; x [R, d_in], h [R, d_h]
 * -> h_out [R, d_h]. */
int amun_gru_cell(int32_t device, int32_t d_in, int32_t d_h, const float *const *W, const float *const *U,
                  const float *const *b, int32_t R, const float *x, const float *h, float *h_out);
/* Forward.attention_rows (nnet.py:132-141): s [R, d_h], h [J, 2 d_h],
 * p [J, d_att] -> alpha [R, J], ctx [R, 2 d_h]. */
int amun_attention(amun_model *m, const float *s, int32_t R, const float *h, const float *p,
                   int32_t J, float *alpha_out, float *ctx_out);
/* Forward.step_rows (nnet.py:143-164): s [R, d_h], y_prev [R] ->
 * s_out [R, d_h], logp_out [R, n] (n = n_sl or v_trg), alpha_out [R, J]. */
int amun_decoder_step(amun_model *m, const float *s, const int32_t *y_prev, int32_t R,
                      const float *h, const float *p, int32_t J, const int32_t *shortlist,
                      int32_t n_sl, float *s_out, double *logp_out, float *alpha_out);

/* ---- production-kernel parity hooks -----------------------------------
 * The hooks above run FP32 CUDA-core kernels; these two run exactly the
 * kernels amun_decode runs (tcgen05 3xFP16 GEMMs, fused attention, fused
 * tensor-core logits), so the per-step gates test the shipped code. */
/* Forward.encode + init_state_row (nnet.py:110-130) for B padded sentences:
 * ids [B, jmax] (entries past lens[b] ignored), lens [B] in [1, jmax].
 * production = 1: tensor-core encoder (input projection, bi-GRU recurrence,
 * precomp_att), 0: FP32 CUDA-core encoder.  h_out [B, jmax, 2 d_h] (zero
 * rows past each length), p_out [B, jmax, d_att], s0_out [B, d_h]. */
int amun_encode_batch(amun_model *m, const int32_t *ids, const int32_t *lens, int32_t B, int32_t jmax,
                      int32_t production, float *h_out, float *p_out, float *s0_out);
/* Forward.step_rows (nnet.py:143-164) + log_softmax_rows (tensor.py:79-92) +
 * the per-row candidate stage of _select_top (search.py:169) for B
 * sentences x k rows (row r belongs to sentence r / k), on the production
 * kernels.  s [B*k, d_h], y_prev [B*k], h [B, jmax, 2 d_h], p [B, jmax,
 * d_att], lens [B].  Outputs the fused logit kernel's partials per (row r,
 * 128-wide vocabulary tile t), nt = ceil(v_trg / 128):
 *   pmax/psum [B*k, nt]: max_t and sum_t exp(logit - max_t) of the tile;
 *   cval/ctok [B*k, nt, kk]: the tile's kk best (logit, token), ordered by
 *   (logit desc, token asc); token -1 marks an empty slot.
 * log p(v | row) = logit_v - (M + log sum_t psum_t exp(pmax_t - M)).
 * s_out [B*k, d_h], alpha_out [B*k, jmax] (either may be NULL). */
int amun_decoder_step_fused(amun_model *m, int32_t B, int32_t k, const float *s, const int32_t *y_prev,
                            const float *h, const float *p, const int32_t *lens, int32_t jmax, int32_t kk,
                            float *s_out, float *pmax_out, float *psum_out, float *cval_out, int32_t *ctok_out,
                            float *alpha_out);

/* ---- host text front-end: replaces the per-line source_tokens ->
 * Vocabulary.ids_and_oov loop of Engine.translate_corpus (engine.py:144-164,
 * model.py Vocabulary: <unk> for unknown tokens, OOV counted) -------------
 * A vocabulary handle holds token i = bytes[offsets[i], offsets[i+1]) (UTF-8,
 * no duplicates).  amun_vocab_encode splits each line of `text` (line l =
 * bytes [line_off[l], line_off[l+1])) exactly like Python's str.split() (all
 * Unicode whitespace) -- the caller applies the preprocessing's lowercasing
 * first -- and writes the ids of all lines back to back (unk_id for tokens
 * outside the vocabulary; ids_cap entries available), the token count and
 * OOV count of every line, and the total in *n_ids. */
typedef struct amun_vocab amun_vocab;
int amun_vocab_create(const char *bytes, const int64_t *offsets, int32_t n_tokens, amun_vocab **out);
int amun_vocab_destroy(amun_vocab *v);
int amun_vocab_encode(const amun_vocab *v, const char *text, const int64_t *line_off, int32_t n_lines,
                      int32_t unk_id, int32_t *ids, int64_t ids_cap, int32_t *lens, int32_t *oov, int64_t *n_ids);

#ifdef __cplusplus
}
#endif
#endif /* AMUN_B200_H_ */

// Decode driver: length buckets -> batched encoder -> device-resident beam
// search loop (all bookkeeping on the device) -> host back-pointer walk and
// final ranking.  Mirrors search.py:116-216 for a batch of sentences, the
// way engine.py:181-221 fans sentences out — but as one device batch.
#include <algorithm>
#include <chrono>
#include <climits>
#include <deque>
#include <memory>
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "decode.cuh"
#include "gemm_simt.cuh"
#include "kernels.cuh"
#include "gemm_sk.cuh"
#include "logits_tc.cuh"

namespace amun {

namespace {

struct Carver {  // bump allocator; base == nullptr -> sizing pass
  char *base = nullptr;
  size_t off = 0;
  template <class T>
  T *take(size_t n) {
    size_t a = (off + 255) & ~size_t(255);
    off = a + n * sizeof(T);
    return base ? reinterpret_cast<T *>(base + a) : nullptr;
  }
};

struct DevMem {  // owning stream-ordered device allocation
  void *p = nullptr;
  cudaStream_t st = nullptr;
  DevMem() = default;
  DevMem(const DevMem &) = delete;
  DevMem &operator=(const DevMem &) = delete;
  void alloc(size_t n, cudaStream_t s) {
    st = s;
    AMUN_CUDA(cudaMallocAsync(&p, std::max<size_t>(n, 256), s));
  }
  ~DevMem() {
    if (p) cudaFreeAsync(p, st);
  }
};

// Per-device pool of decode-lane resources reused across amun_decode calls:
// stream, workspace (grown on demand), pinned probe ring and probe events.
// Creating them per call (pinned allocation, stream-ordered workspace
// allocation, event creation) cost tens of ms of host time per call.
struct LaneRes {
  cudaStream_t st = nullptr;
  void *mem = nullptr;
  size_t cap = 0;
  int *h_probe = nullptr;
  std::vector<cudaEvent_t> ev;
  cudaGraphExec_t gexec = nullptr;  // step graph, updated in place per bucket
  std::vector<uintptr_t> gkey;      // what the graph was captured for (models, options)
  float *ws = nullptr;              // SIMT split-K partials
  size_t ws_floats = 0;
  int high = 0;                     // stream created with the device's greatest priority
};
constexpr int kProbeSlots = 64;
std::mutex g_lane_mu;
std::vector<LaneRes *> g_lane_pool[64][2];  // [device][high priority]
cudaMemPool_t g_ws_pool[64] = {};             // private workspace pool per device

// Private stream-ordered pool for the lane workspaces: freed memory stays
// mapped across calls (stream syncs must not trim it) without changing the
// release threshold of the device's default pool, which other users share.
cudaMemPool_t ws_pool(int dev) {
  std::lock_guard<std::mutex> g(g_lane_mu);
  cudaMemPool_t &p = g_ws_pool[dev & 63];
  if (!p) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = dev;
    AMUN_CUDA(cudaMemPoolCreate(&p, &props));
    uint64_t thr = UINT64_MAX;
    AMUN_CUDA(cudaMemPoolSetAttribute(p, cudaMemPoolAttrReleaseThreshold, &thr));
  }
  return p;
}

LaneRes *lane_acquire(int dev, int high) {
  {
    std::lock_guard<std::mutex> g(g_lane_mu);
    auto &v = g_lane_pool[dev & 63][high ? 1 : 0];
    if (!v.empty()) {
      LaneRes *r = v.back();
      v.pop_back();
      return r;
    }
  }
  std::unique_ptr<LaneRes> r(new LaneRes());
  {
    int least = 0, greatest = 0;
    AMUN_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    r->high = high ? 1 : 0;
    AMUN_CUDA(cudaStreamCreateWithPriority(&r->st, cudaStreamNonBlocking, high ? greatest : least));
  }
  AMUN_CUDA(cudaMallocHost(&r->h_probe, sizeof(int) * kProbeSlots));
  r->ev.resize(kProbeSlots);
  for (auto &e : r->ev) AMUN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return r.release();
}
void lane_release(int dev, LaneRes *r) {
  std::lock_guard<std::mutex> g(g_lane_mu);
  g_lane_pool[dev & 63][r->high].push_back(r);
}

// the last n lanes run on high-priority streams: the dispatch hands the
// longest buckets to the highest lanes first, and the longest bucket's
// serial step chain bounds the pass
int high_priority_lanes() {
  static int v = [] {
    const char *e = getenv("AMUN_HIGH_LANES");
    return e ? std::max(0, atoi(e)) : 0;  // swept: no measurable effect on cfg2
  }();
  return v;
}
// workspace of at least n bytes on the lane's stream
void *lane_mem(LaneRes *r, size_t n, cudaMemPool_t pool) {
  n = std::max<size_t>(n, 256);
  if (r->cap < n) {
    if (r->mem) AMUN_CUDA(cudaFreeAsync(r->mem, r->st));
    r->mem = nullptr;
    r->cap = 0;
    AMUN_CUDA(cudaMallocFromPoolAsync(&r->mem, n, pool, r->st));
    r->cap = n;
  }
  return r->mem;
}

// Launch context: stream, launch counter, byte counters, and (when
// profiling) CUDA-event pairs around every launch, bucketed by kernel class.
struct Ctx {
  cudaStream_t st;
  int64_t launches = 0;
  int64_t h2d = 0, d2h = 0;
  uint32_t prof = 0;  // bitmask of kernel classes to time with events
  int cls = AMUN_K_ENCODER;
  std::vector<cudaEvent_t> pool;
  std::vector<int> rec_cls;
  size_t used = 0;
  double kms[AMUN_K_CLASSES] = {0};
  int64_t kcount[AMUN_K_CLASSES] = {0};
  int64_t kctas[AMUN_K_CLASSES] = {0};  // tensor-core CTAs launched per class (profiling)
  float *ws = nullptr;  // split-K partials (stream-ordered, grown on demand)
  size_t ws_floats = 0;
  float **ws_keep = nullptr;  // when set, the buffer outlives the Ctx (pooled lane)
  size_t *ws_keep_n = nullptr;
  cudaMemPool_t ws_pool = nullptr;  // allocation pool of ws (nullptr: the device default)
  unsigned long long *kt = nullptr;  // CTA-time accounting slots [class][2] (AMUN_PROFILE_CTA_TIME)
  explicit Ctx(cudaStream_t s) : st(s) {}
  ~Ctx() {
    for (auto e : pool) cudaEventDestroy(e);
    if (ws_keep) {
      *ws_keep = ws;
      *ws_keep_n = ws_floats;
    } else if (ws) {
      cudaFreeAsync(ws, st);
    }
  }
  void ensure_ws(size_t n) {
    if (n <= ws_floats) return;
    if (ws) AMUN_CUDA(cudaFreeAsync(ws, st));
    ws = nullptr;
    if (ws_pool)
      AMUN_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void **>(&ws), n * sizeof(float), ws_pool, st));
    else
      AMUN_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&ws), n * sizeof(float), st));
    ws_floats = n;
  }
  cudaEvent_t next_event() {
    if (used == pool.size()) {
      cudaEvent_t e;
      AMUN_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[used++];
  }
  // profiling ablation only (AMUN_ABLATE_CLASSES bitmask): outputs are garbage
  static unsigned ablated() {
    static const unsigned skip = [] {
      const char *e = getenv("AMUN_ABLATE_CLASSES");
      return e ? (unsigned)strtoul(e, nullptr, 0) : 0u;
    }();
    return skip;
  }
  template <class F>
  void run(int k, F &&f) {
    if (ablated() & (1u << k)) return;
    ++launches;
    struct KtScope {  // kernels launched inside f() account their CTA time to class k
      unsigned long long *prev;
      KtScope(unsigned long long *p) : prev(ktime_ptr()) { ktime_ptr() = p; }
      ~KtScope() { ktime_ptr() = prev; }
    } kts(kt ? kt + 2 * k : nullptr);
    if (!(prof & (1u << k))) {
      f();
      return;
    }
    AMUN_CUDA(cudaEventRecord(next_event(), st));
    last_launch_ctas() = 0;
    f();
    kctas[k] += last_launch_ctas();
    AMUN_CUDA(cudaEventRecord(next_event(), st));
    rec_cls.push_back(k);
  }
  // call after the stream is synchronised: fold recorded pairs into totals
  void collect() {
    for (size_t i = 0; i < rec_cls.size(); ++i) {
      float ms = 0.f;
      AMUN_CUDA(cudaEventElapsedTime(&ms, pool[2 * i], pool[2 * i + 1]));
      kms[rec_cls[i]] += ms;
      kcount[rec_cls[i]] += 1;
    }
    rec_cls.clear();
    used = 0;
  }
};

template <class T>
void h2d(Ctx &c, T *dst, const T *src, size_t n) {
  if (n) AMUN_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyHostToDevice, c.st));
  c.h2d += (int64_t)(n * sizeof(T));
}
template <class T>
void d2h(Ctx &c, T *dst, const T *src, size_t n) {
  if (n) AMUN_CUDA(cudaMemcpyAsync(dst, src, n * sizeof(T), cudaMemcpyDeviceToHost, c.st));
  c.d2h += (int64_t)(n * sizeof(T));
}

GemmArgs ga(int M, int N, const float *a0, int lda0, int k0, const float *B, int ldb) {
  GemmArgs g{};
  g.M = M;
  g.N = N;
  g.a0 = a0;
  g.lda0 = lda0;
  g.k0 = k0;
  g.rows0 = nullptr;
  g.a1 = nullptr;
  g.lda1 = 0;
  g.k1 = 0;
  g.B = B;
  g.ldb = ldb;
  g.n_split = INT_MAX;
  g.k_limit = INT_MAX;
  g.a_zs = 0;
  g.b_zs = 0;
  g.splits = 1;
  g.kchunk = 0;
  return g;
}

// GEMM with split-K when the output has too few tiles to fill 148 SMs.
// allow_split = false for the large-M encoder GEMMs (enough tiles already).
template <class Epi>
void gemm(Ctx &c, const GemmArgs &g, const Epi &e, int nz = 1, bool allow_split = true) {
  const int K = g.k0 + g.k1;
  int splits = (allow_split && !Epi::kTile) ? effective_splits(K, choose_splits(g.N, K, nz)) : 1;
  if (splits > 1) c.ensure_ws((size_t)splits * nz * g.M * g.N);
  int n = 1;
  c.run(c.cls, [&] { n = launch_gemm_simt(g, e, nz, splits, c.st, c.ws); });
  c.launches += n - 1;
}

// Encoder buffers of one model for a bucket of B sentences, jmax positions.
struct EncBufs {
  float *XP, *Hann, *P, *Hs, *Zs, *RHs, *Hmean, *S0;
  float *HX = nullptr;  // projected annotations [B*jmax][proj_ldhx] (projected-context step)
  // tensor-core encoder (3xFP16 splits): block rows [2B][2dh] of the states
  // (HH) and of r*h (RR), and the split annotations [B*jmax][2dh] (Ha)
  __half *HHh = nullptr, *HHl = nullptr, *RRh = nullptr, *RRl = nullptr, *Hah = nullptr, *Hal = nullptr;
  __half *Xh = nullptr, *Xl = nullptr;  // gathered source embeddings [B*jmax][dep] (input projection)
};
// Decoder row buffers of one model for R hypothesis rows.
struct DecBufs {
  float *XS, *Sn, *Q, *Z, *RH, *XH, *T, *L;
  float *SU = nullptr, *CO = nullptr;  // projected-context step: s U_{z,r} [R][2dh], deep-output row terms [R][dep]
  float *En = nullptr;  // attention energies [R][jmax]
  float *EQ = nullptr;  // e^{2q} of the attention query rows [R][da]
  __half *T_hi = nullptr, *T_lo = nullptr;  // 3xFP16 split of t [R][dep] (tensor-core logits)
  // 3xFP16 splits of the tensor-core GEMM activation operands; XSh/XSl use
  // the padded row layout [y | pad | c | s] (pitch xsp, pad columns zero)
  __half *XSh = nullptr, *XSl = nullptr, *RHh = nullptr, *RHl = nullptr, *Snh = nullptr, *Snl = nullptr;
};

void carve_enc(Carver &cv, EncBufs &e, const amun_model *m, int B, int jmax) {
  const int dh = m->d.d_h, da = m->d.d_att;
  e.XP = cv.take<float>((size_t)B * jmax * 6 * dh);
  e.Hann = cv.take<float>((size_t)B * jmax * 2 * dh);
  e.P = cv.take<float>((size_t)B * jmax * da);
  e.Hs = cv.take<float>((size_t)2 * B * dh);
  e.Zs = cv.take<float>((size_t)2 * B * dh);
  e.RHs = cv.take<float>((size_t)2 * B * dh);
  e.Hmean = cv.take<float>((size_t)B * 2 * dh);
  e.S0 = cv.take<float>((size_t)B * dh);
}

void carve_enc_tc(Carver &cv, EncBufs &e, const amun_model *m, int B, int jmax) {
  const int dh = m->d.d_h;
  e.HHh = cv.take<__half>((size_t)2 * B * 2 * dh);
  e.HHl = cv.take<__half>((size_t)2 * B * 2 * dh);
  e.RRh = cv.take<__half>((size_t)2 * B * 2 * dh);
  e.RRl = cv.take<__half>((size_t)2 * B * 2 * dh);
  e.Hah = cv.take<__half>((size_t)B * jmax * 2 * dh);
  e.Hal = cv.take<__half>((size_t)B * jmax * 2 * dh);
  e.Xh = cv.take<__half>((size_t)B * jmax * m->dep);
  e.Xl = cv.take<__half>((size_t)B * jmax * m->dep);
}

// 3xFP16 split of the gathered source embeddings E_src[ids] (nnet.py:113,
// 167-174), zero pad columns [de, dep): the input-projection A operand.
__global__ void gather_split_kernel(const float *__restrict__ E, const int *__restrict__ ids, int de, int dep,
                                    __half *xh, __half *xl) {
  const long long r = blockIdx.x;
  const float *src = E + (long long)ids[r] * de;
  for (int c = threadIdx.x; c < dep; c += blockDim.x) {
    __half h = __float2half_rn(0.f), l = h;
    if (c < de) split_h(__ldg(src + c), h, l);
    xh[r * dep + c] = h;
    xl[r * dep + c] = l;
  }
}

// Gathered shortlist columns: W_logit rows (fp16 hi/lo, K-major) and biases
// of the bucket's shortlist union U (nnet.py:163 logit_rows[sl_ids]).
__global__ void gather_logit_rows_kernel(const __half *__restrict__ whi, const __half *__restrict__ wlo,
                                         const float *__restrict__ bias, int dep, const int *__restrict__ U,
                                         __half *ghi, __half *glo, float *gb) {
  const int j = blockIdx.x;
  const long long src = (long long)U[j] * dep, dst = (long long)j * dep;
  for (int c = threadIdx.x; c < dep; c += blockDim.x) {
    ghi[dst + c] = whi[src + c];
    glo[dst + c] = wlo[src + c];
  }
  if (threadIdx.x == 0) gb[j] = bias[U[j]];
}

// Tensor-core encoder GEMMs of one model: recurrence phase A / B over the
// 2B block rows, and precomp_att over the split annotations; split counts
// from (N, K) only.
struct TcEnc {
  SkMaps x, a, b, p;
  int sx = 1, sa = 1, sb = 1, sp = 1;
};

int enc_target_ctas() {
  static int v = [] {
    const char *e = getenv("AMUN_ENC_CTAS");
    return e ? std::max(1, atoi(e)) : 32;
  }();
  return v;
}

void tc_enc_maps(const amun_model *m, const EncBufs &e, int Bmax, int jmax, TcEnc &te) {
  const int dh = m->d.d_h, da = m->d.d_att;
  te.a = make_sk_maps(e.HHh, e.HHl, 2 * dh, 2 * dh, nullptr, nullptr, 0, 0, 2 * Bmax, m->Uzr_hi, m->Uzr_lo, 2 * dh,
                      2 * dh, m->us_ea);
  te.b = make_sk_maps(e.RRh, e.RRl, 2 * dh, 2 * dh, nullptr, nullptr, 0, 0, 2 * Bmax, m->Uh_hi, m->Uh_lo, dh, 2 * dh,
                      m->us_eb);
  te.p = make_sk_maps(e.Hah, e.Hal, 2 * dh, 2 * dh, nullptr, nullptr, 0, 0, Bmax * jmax, m->Watth_hi, m->Watth_lo,
                      da, 2 * dh, m->us_p);
  te.x = make_sk_maps(e.Xh, e.Xl, m->dep, m->dep, nullptr, nullptr, 0, 0, Bmax * jmax, m->Wenc_hi, m->Wenc_lo,
                      6 * dh, m->dep, m->us_x);
  const int t = enc_target_ctas();
  te.sx = sk_fit_splits(te.x, t);
  te.sa = sk_fit_splits(te.a, t);
  te.sb = sk_fit_splits(te.b, t);
  te.sp = sk_fit_splits(te.p, t);
}

void carve_dec(Carver &cv, DecBufs &d, const amun_model *m, int R, int jmax, bool full_logits) {
  const int dh = m->d.d_h, da = m->d.d_att, de = m->d.d_emb;
  d.En = cv.take<float>((size_t)R * jmax);
  d.EQ = cv.take<float>((size_t)R * da);
  d.XS = cv.take<float>((size_t)R * m->xs_w);
  d.Sn = cv.take<float>((size_t)R * dh);
  d.Q = cv.take<float>((size_t)R * da);
  d.Z = cv.take<float>((size_t)R * dh);
  d.RH = cv.take<float>((size_t)R * dh);
  d.XH = cv.take<float>((size_t)R * dh);
  d.T = cv.take<float>((size_t)R * de);
  d.L = full_logits ? cv.take<float>((size_t)R * m->d.v_trg) : nullptr;
  if (!full_logits && m->Wl_hi) {
    d.T_hi = cv.take<__half>((size_t)R * m->dep);
    d.T_lo = cv.take<__half>((size_t)R * m->dep);
  }
}

// Projected-context step (tensor-core path): the decoder's context weights
// act on the annotations once, at encode time -- HX = h [C_z | C_r | C_h |
// W_o^c] per source position -- instead of on the context every step:
// c C = (sum_j alpha_j h_j) C = sum_j alpha_j (h_j C).  The step is then
// s [W_att_s | U_z | U_r] (one GEMM), the attention summing HX rows and
// finishing the gates, (r*s) U_h, and s' W_o^s: the per-row MMA work outside
// the logits drops from 12.1M to 4.7M MACs.  Env
// AMUN_NO_PROJ_CTX=1 keeps the GRU-A step (A/B runs).
int proj_ldhx(const amun_model *m) { return 3 * m->d.d_h + m->dep; }
// the next step's query + s U_zr computed by the deep-output GEMM from s'
// (one launch per step fewer; AMUN_NO_FOLD_QUERY=1 keeps a separate launch)
bool fold_query() {
  static const bool off = [] {
    const char *e = getenv("AMUN_NO_FOLD_QUERY");
    return e && e[0] == '1';
  }();
  return !off;
}
bool proj_ok(const amun_model *m) {
  static const bool off = [] {
    const char *e = getenv("AMUN_NO_PROJ_CTX");
    return e && e[0] == '1';
  }();
  return !off && m->tc_gemm && m->Wqs_hi && m->YWg && m->YWo && proj_ldhx(m) <= 4 * 1024 &&
         (3 * m->d.d_h + m->d.d_emb) % 4 == 0;
}

void compute_hx(Ctx &c, const amun_model *m, const __half *Hah, const __half *Hal, long long store_rows,
                long long row0, int M, float *HX, int target);

void carve_dec_tc(Carver &cv, DecBufs &d, const amun_model *m, int R) {
  const int dh = m->d.d_h;
  if (proj_ok(m)) {
    d.SU = cv.take<float>((size_t)R * 2 * dh);
    d.CO = cv.take<float>((size_t)R * m->dep);
  }
  d.XSh = cv.take<__half>((size_t)R * m->xsp);
  d.XSl = cv.take<__half>((size_t)R * m->xsp);
  d.RHh = cv.take<__half>((size_t)R * dh);
  d.RHl = cv.take<__half>((size_t)R * dh);
  d.Snh = cv.take<__half>((size_t)R * dh);
  d.Snl = cv.take<__half>((size_t)R * dh);
}

// nnet.py:110-130 for B padded sentences: input projection (embedding
// gather fused into the A-load), the bi-GRU recurrence (both directions per
// launch), precomp_att, masked mean and the initial decoder state.
void encode_bucket(Ctx &c, const amun_model *m, const EncBufs &e, const int *d_ids, const int *d_len, int B,
                   int jmax, const TcEnc *te = nullptr) {
  const int de = m->d.d_emb, dh = m->d.d_h, da = m->d.d_att;
  c.cls = AMUN_K_ENCODER;
  if (te) {  // input projection on tensor cores (embedding gather + split first)
    c.run(AMUN_K_ENCODER, [&] {
      gather_split_kernel<<<B * jmax, 128, 0, c.st>>>(m->E_src, d_ids, de, m->dep, e.Xh, e.Xl);
      AMUN_CHECK_LAUNCH();
    });
    EpiStore ex{e.XP, 6 * dh, m->benc, 0, 0};
    c.run(AMUN_K_ENCODER, [&] { launch_gemm_sk(te->x, B * jmax, te->sx, ex, c.st); });
  } else {
    GemmArgs g = ga(B * jmax, 6 * dh, m->E_src, de, de, m->Wenc, 6 * dh);
    g.rows0 = d_ids;
    gemm(c, g, EpiStore{e.XP, 6 * dh, m->benc, 0, 0}, 1, false);
  }
  AMUN_CUDA(cudaMemsetAsync(e.Hs, 0, sizeof(float) * 2 * B * dh, c.st));
  AMUN_CUDA(cudaMemsetAsync(e.Hann, 0, sizeof(float) * (size_t)B * jmax * 2 * dh, c.st));
  if (te) {
    // block rows start as zeros (h0 = 0; the off-diagonal halves stay zero)
    const size_t blk = sizeof(__half) * (size_t)2 * B * 2 * dh, ann = sizeof(__half) * (size_t)B * jmax * 2 * dh;
    AMUN_CUDA(cudaMemsetAsync(e.HHh, 0, blk, c.st));
    AMUN_CUDA(cudaMemsetAsync(e.HHl, 0, blk, c.st));
    AMUN_CUDA(cudaMemsetAsync(e.RRh, 0, blk, c.st));
    AMUN_CUDA(cudaMemsetAsync(e.RRl, 0, blk, c.st));
    AMUN_CUDA(cudaMemsetAsync(e.Hah, 0, ann, c.st));
    AMUN_CUDA(cudaMemsetAsync(e.Hal, 0, ann, c.st));
    for (int t = 0; t < jmax; ++t) {
      EpiEncA2 ea{e.XP, e.Hs, d_len, jmax, dh, t, B, e.Zs, e.RHs, e.RRh, e.RRl};
      c.run(AMUN_K_ENCODER, [&] { launch_gemm_sk(te->a, 2 * B, te->sa, ea, c.st); });
      EpiEncB2 eb{e.XP, e.Hs, d_len, jmax, dh, t, B, e.Zs, e.Hann, e.HHh, e.HHl, e.Hah, e.Hal};
      c.run(AMUN_K_ENCODER, [&] { launch_gemm_sk(te->b, 2 * B, te->sb, eb, c.st); });
    }
    EpiStore ep{e.P, da, nullptr, 0, 0};
    c.run(AMUN_K_ENCODER, [&] { launch_gemm_sk(te->p, B * jmax, te->sp, ep, c.st); });
    c.run(AMUN_K_ENCODER, [&] { launch_masked_mean(e.Hann, d_len, B, jmax, 2 * dh, e.Hmean, c.st); });
    gemm(c, ga(B, dh, e.Hmean, 2 * dh, 2 * dh, m->W_init, dh), EpiStore{e.S0, dh, m->b_init, 1, 0});
    return;
  }
  for (int t = 0; t < jmax; ++t) {
    GemmArgs a = ga(B, 2 * dh, e.Hs, dh, dh, m->Uzr, 2 * dh);
    a.a_zs = (long long)B * dh;
    a.b_zs = (long long)dh * 2 * dh;
    gemm(c, a, EpiEncA{e.XP, e.Hs, d_len, jmax, dh, t, B, e.Zs, e.RHs}, 2);
    GemmArgs b = ga(B, dh, e.RHs, dh, dh, m->Uh, dh);
    b.a_zs = (long long)B * dh;
    b.b_zs = (long long)dh * dh;
    gemm(c, b, EpiEncB{e.XP, e.Hs, d_len, jmax, dh, t, B, e.Zs, e.Hann}, 2);
  }
  gemm(c, ga(B * jmax, da, e.Hann, 2 * dh, 2 * dh, m->W_att_h, da), EpiStore{e.P, da, nullptr, 0, 0}, 1, false);
  c.run(AMUN_K_ENCODER, [&] { launch_masked_mean(e.Hann, d_len, B, jmax, 2 * dh, e.Hmean, c.st); });
  gemm(c, ga(B, dh, e.Hmean, 2 * dh, 2 * dh, m->W_init, dh), EpiStore{e.S0, dh, m->b_init, 1, 0});
}

// ================================================================ encode-ahead
//
// The encoder of a whole chunk of sentences (nnet.py:110-130), run before the
// decode lanes start instead of per length bucket: the bi-GRU recurrence is
// one GEMM pair per time step and direction over EVERY sentence still active
// at that step (sentences in descending length order, so the active set is a
// prefix), with the input projection fused into the recurrent GEMMs (the
// activation row is [x_t | state], the weight [W ; U]).  At the headline
// workload a step's GEMM has up to 4000 rows instead of 64: the tensor cores
// run full tiles, the weights are read once per step for all sentences, and
// the encoder costs ~2 x max-length launches per direction for the whole
// call instead of 2 x J launches per bucket.  Forward and backward run
// concurrently on two streams.  Results land in an annotation store laid out
// per length bucket ([B][jmax] rows), which the decode lanes read in place.

struct AheadIn {
  int n;                       // sentences
  const int32_t *ids;          // host, sentence i at ids + off[i]
  const long long *off;        // host [n]
  const int32_t *len;          // host [n]
  const long long *ann_row;    // host [n]: store row of (sentence i, position 0)
  long long store_rows;
};
struct AheadOut {
  float *Hann, *P, *S0;  // store [rows][2dh], [rows][da]; S0 [n][dh] indexed by sentence i
  __half *Hah, *Hal;     // store [rows][2dh] split annotations
  float *HX = nullptr;   // optional store [rows][proj_ldhx] projected annotations
};

// Hmean[i] = Hsum[e(i)] / len[e(i)] for sentences i0 .. i0 + gridDim.x - 1
__global__ void enc_mean_kernel(const float *__restrict__ Hsum, const int *__restrict__ len_e,
                                const int *__restrict__ e_of_i, int i0, int w, float *__restrict__ out) {
  const int i = i0 + blockIdx.x, e = e_of_i[i];
  const float inv = 1.0f / (float)len_e[e];
  const float *src = Hsum + (long long)e * w;
  float *dst = out + (long long)i * w;
  for (int c = threadIdx.x; c < w; c += blockDim.x) dst[c] = src[c] * inv;
}

int ahead_target_ctas() {
  static int v = [] {
    const char *e = getenv("AMUN_AHEAD_CTAS");
    return e ? std::max(2, atoi(e)) : 148;
  }();
  return v;
}

// (splits, z-grid) of one encode-ahead GEMM launch.  The split count comes
// from (N, K) only (about 32 CTAs per row pass), never from the row count, so
// a sentence's encoder result does not depend on which other sentences share
// the call, chunk or device; the z-grid spreads the row passes.
template <class C = SkDefault>
std::pair<int, int> ahead_grid(const SkMaps &mp, int M, int target) {
  static const int split_ctas = [] {  // CTAs per row pass the split count aims at
    const char *e = getenv("AMUN_AHEAD_SPLIT_CTAS");
    return e ? std::max(1, atoi(e)) : 32;
  }();
  const int per_pass = ceil_div(mp.N, 128 * C::kCG) * C::kCG;
  const int s = sk_fit_splits<C>(mp, split_ctas);
  const int npass = ceil_div(M, C::kPR);
  return {s, std::max(1, std::min(npass, target / (per_pass * s)))};
}

// run(): the recurrence of every sentence (both directions, two streams);
// an event per time step marks which sentences are complete (a sentence of
// length L is final after step L - 1 in both directions).  prepare(): on a
// decode lane's stream, once a bucket's sentences are complete, its
// precomp_att rows (nnet.py:126) and initial states tanh(mean_j h_j W_init +
// b_init) (nnet.py:128-130) -- so the lanes start decoding short buckets
// while the encoder still runs the long sentences' tail steps.
class AheadEncoder {
 public:
  AheadEncoder(const amun_model *m, const AheadIn &in, const AheadOut &out, cudaMemPool_t pool)
      : m_(m), in_(in), out_(out), pool_(pool) {}
  AheadEncoder(const AheadEncoder &) = delete;
  AheadEncoder &operator=(const AheadEncoder &) = delete;
  ~AheadEncoder() = default;

  void run(Ctx &cf, Ctx &cb) {
    const amun_model *m = m_;
    const int n = in_.n, de = m->d.d_emb, dh = m->d.d_h, dep = m->dep;
    std::vector<int> ord(n);  // encoder row e -> sentence, descending length (stable)
    std::iota(ord.begin(), ord.end(), 0);
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return in_.len[a] > in_.len[b]; });
    T_ = in_.len[ord[0]];
    std::vector<int> nact(T_, 0);
    for (int e = 0; e < n; ++e)
      for (int t = 0; t < in_.len[ord[e]]; ++t) ++nact[t];
    std::vector<long long> offt(T_ + 1, 0);
    for (int t = 0; t < T_; ++t) offt[t + 1] = offt[t] + nact[t];
    const long long total = offt[T_];
    std::vector<int> tokf(total), tokb(total), len_e(n), e_of_i(n);
    std::vector<long long> arow(n);
    std::vector<char> need(T_, 0);  // some sentence completes at step t
    for (int e = 0; e < n; ++e) {
      const int i = ord[e];
      len_e[e] = in_.len[i];
      e_of_i[i] = e;
      arow[e] = in_.ann_row[i];
      need[in_.len[i] - 1] = 1;
    }
    for (int t = 0; t < T_; ++t)
      for (int e = 0; e < nact[t]; ++e) {
        const int i = ord[e];
        tokf[offt[t] + e] = in_.ids[in_.off[i] + t];
        tokb[offt[t] + e] = in_.ids[in_.off[i] + in_.len[i] - 1 - t];
      }
    int *d_tok[2];
    __half *Hh[2], *Hl[2], *RHh[2], *RHl[2];
    float *H[2], *Z[2];
    for (int pass = 0; pass < 2; ++pass) {
      Carver cv;
      cv.base = static_cast<char *>(mem_);
      for (int d = 0; d < 2; ++d) {
        d_tok[d] = cv.take<int>(total);
        Hh[d] = cv.take<__half>((size_t)n * dh);
        Hl[d] = cv.take<__half>((size_t)n * dh);
        RHh[d] = cv.take<__half>((size_t)n * dh);
        RHl[d] = cv.take<__half>((size_t)n * dh);
        H[d] = cv.take<float>((size_t)n * dh);
        Z[d] = cv.take<float>((size_t)n * dh);
      }
      d_len_ = cv.take<int>(n);
      d_e_of_i_ = cv.take<int>(n);
      d_arow_ = cv.take<long long>(n);
      Hsum_ = cv.take<float>((size_t)n * 2 * dh);
      Hmean_ = cv.take<float>((size_t)n * 2 * dh);
      if (!pass) AMUN_CUDA(cudaMallocFromPoolAsync(&mem_, std::max<size_t>(cv.off, 256), pool_, cf.st));
    }
    h2d(cf, d_tok[0], tokf.data(), total);
    h2d(cf, d_tok[1], tokb.data(), total);
    h2d(cf, d_len_, len_e.data(), n);
    h2d(cf, d_e_of_i_, e_of_i.data(), n);
    h2d(cf, d_arow_, arow.data(), n);
    // store: padded positions must read as zero (attention masks them, the
    // precomp GEMM reads them); P and S0 are fully written by prepare()
    const size_t ann = (size_t)in_.store_rows * 2 * dh;
    if (out_.Hann) AMUN_CUDA(cudaMemsetAsync(out_.Hann, 0, ann * sizeof(float), cf.st));
    AMUN_CUDA(cudaMemsetAsync(out_.Hah, 0, ann * sizeof(__half), cf.st));
    AMUN_CUDA(cudaMemsetAsync(out_.Hal, 0, ann * sizeof(__half), cf.st));
    if (Ctx::ablated() & (1u << AMUN_K_ENCODER)) {  // encoder ablated: finite inputs for the decoder
      AMUN_CUDA(cudaMemsetAsync(out_.P, 0, sizeof(float) * (size_t)in_.store_rows * m->d.d_att, cf.st));
      AMUN_CUDA(cudaMemsetAsync(out_.S0, 0, sizeof(float) * (size_t)n * dh, cf.st));
    }
    for (int d = 0; d < 2; ++d) {
      AMUN_CUDA(cudaMemsetAsync(H[d], 0, sizeof(float) * (size_t)n * dh, cf.st));
      AMUN_CUDA(cudaMemsetAsync(Hh[d], 0, sizeof(__half) * (size_t)n * dh, cf.st));
      AMUN_CUDA(cudaMemsetAsync(Hl[d], 0, sizeof(__half) * (size_t)n * dh, cf.st));
    }
    const bool two = cb.st != cf.st;
    cudaEvent_t ev0 = new_event();
    AMUN_CUDA(cudaEventRecord(ev0, cf.st));
    if (two) AMUN_CUDA(cudaStreamWaitEvent(cb.st, ev0, 0));
    // state-only GEMMs: the U rows of the [W ; U] weights (K offset dep)
    SkMaps fa[2], fb[2];
    for (int d = 0; d < 2; ++d) {
      fa[d] = make_sk_maps(Hh[d], Hl[d], dh, dh, nullptr, nullptr, 0, 0, n, m->Efa_hi[d] + dep, m->Efa_lo[d] + dep,
                           2 * dh, dh, m->us_efa[d], -1, dep + dh);
      fb[d] = make_sk_maps(RHh[d], RHl[d], dh, dh, nullptr, nullptr, 0, 0, n, m->Efb_hi[d] + dep,
                           m->Efb_lo[d] + dep, dh, dh, m->us_efb[d], -1, dep + dh);
    }
    const int target = ahead_target_ctas() / (two ? 2 : 1);
    evf_.assign(T_, nullptr);
    evb_.assign(T_, nullptr);
    for (int t = 0; t < T_; ++t) {
      for (int d = 0; d < 2; ++d) {
        Ctx &c = d ? cb : cf;
        const int M = nact[t];
        const float *xw = m->XWenc + d * 3 * dh;
        const int *tok = d_tok[d] + offt[t];
        EpiEncFA ea{xw, tok, 6 * dh, H[d], Z[d], RHh[d], RHl[d], dh};
        const auto ga_ = ahead_grid(fa[d], M, target);
        c.run(AMUN_K_ENCODER, [&] { launch_gemm_sk(fa[d], M, ga_.first, ea, c.st, 0, 0, ga_.second); });
        EpiEncFB eb{xw + 2 * dh, tok, 6 * dh, H[d], Z[d], Hh[d], Hl[d], out_.Hann, out_.Hah, out_.Hal, Hsum_,
                    d_len_, d_arow_, dh, t, d};
        const auto gb_ = ahead_grid(fb[d], M, target);
        c.run(AMUN_K_ENCODER, [&] { launch_gemm_sk(fb[d], M, gb_.first, eb, c.st, 0, 0, gb_.second); });
      }
      if (need[t]) {
        evf_[t] = new_event();
        AMUN_CUDA(cudaEventRecord(evf_[t], cf.st));
        if (two) {
          evb_[t] = new_event();
          AMUN_CUDA(cudaEventRecord(evb_[t], cb.st));
        }
      }
    }
    if (two) {  // the temporaries are freed on cf: order cb's work before that
      cudaEvent_t e = new_event();
      AMUN_CUDA(cudaEventRecord(e, cb.st));
      AMUN_CUDA(cudaStreamWaitEvent(cf.st, e, 0));
    }
  }

  // Sentences [i0, i0 + cnt) (max length jmax) whose store rows are
  // [row0, row0 + nrows): precomp_att and initial states on c's stream.
  void prepare(Ctx &c, int i0, int cnt, long long row0, long long nrows, int jmax) {
    const amun_model *m = m_;
    const int dh = m->d.d_h, da = m->d.d_att;
    if (jmax < 1 || jmax > T_ || !evf_[jmax - 1]) throw Error(AMUN_ERR_CUDA, "encode-ahead: bucket not tracked");
    AMUN_CUDA(cudaStreamWaitEvent(c.st, evf_[jmax - 1], 0));
    if (evb_[jmax - 1]) AMUN_CUDA(cudaStreamWaitEvent(c.st, evb_[jmax - 1], 0));
    const int M = (int)nrows;
    const int cls = c.cls;
    c.cls = AMUN_K_ENCODER;
    if (out_.HX && m->Wph_hi) {  // P and HX in one GEMM (one read of the annotations)
      const int ld = proj_ldhx(m);
      const SkMaps pm = make_sk_maps(out_.Hah, out_.Hal, 2 * dh, 2 * dh, nullptr, nullptr, 0, 0,
                                     (int)in_.store_rows, m->Wph_hi, m->Wph_lo, da + ld, 2 * dh, m->us_ph);
      const auto gp = ahead_grid(pm, M, std::max(32, prep_ctas_));
      EpiPH ep{out_.P + row0 * da, out_.HX + row0 * ld, da, ld, 3 * dh + m->d.d_emb};
      c.run(AMUN_K_ENCODER, [&] { launch_gemm_sk(pm, M, gp.first, ep, c.st, 0, (int)row0, gp.second); });
    } else {
      const SkMaps pm = make_sk_maps(out_.Hah, out_.Hal, 2 * dh, 2 * dh, nullptr, nullptr, 0, 0,
                                     (int)in_.store_rows, m->Watth_hi, m->Watth_lo, da, 2 * dh, m->us_p);
      const auto gp = ahead_grid(pm, M, std::max(32, prep_ctas_));
      EpiStore ep{out_.P + row0 * da, da, nullptr, 0, 0};
      c.run(AMUN_K_ENCODER, [&] { launch_gemm_sk(pm, M, gp.first, ep, c.st, 0, (int)row0, gp.second); });
      if (out_.HX) compute_hx(c, m, out_.Hah, out_.Hal, in_.store_rows, row0, M, out_.HX, std::max(32, prep_ctas_));
    }
    c.run(AMUN_K_ENCODER, [&] {
      enc_mean_kernel<<<cnt, 256, 0, c.st>>>(Hsum_, d_len_, d_e_of_i_, i0, 2 * dh, Hmean_);
      AMUN_CHECK_LAUNCH();
    });
    gemm(c, ga(cnt, dh, Hmean_ + (long long)i0 * 2 * dh, 2 * dh, 2 * dh, m->W_init, dh),
         EpiStore{out_.S0 + (long long)i0 * dh, dh, m->b_init, 1, 0});
    c.cls = cls;
  }

  // after every prepare() and every consumer of the prepared rows on c
  void release(Ctx &c) {
    if (mem_) AMUN_CUDA(cudaFreeAsync(mem_, c.st));
    mem_ = nullptr;
  }
  void set_prep_ctas(int n) { prep_ctas_ = n; }

 private:
  cudaEvent_t new_event() {
    cudaEvent_t e;
    AMUN_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    owned_.push_back(e);
    return e;
  }
  const amun_model *m_;
  AheadIn in_;
  AheadOut out_;
  cudaMemPool_t pool_;
  void *mem_ = nullptr;
  int T_ = 0, prep_ctas_ = 148;
  int *d_len_ = nullptr, *d_e_of_i_ = nullptr;
  long long *d_arow_ = nullptr;
  float *Hsum_ = nullptr, *Hmean_ = nullptr;
  std::vector<cudaEvent_t> evf_, evb_;
  struct Owned {
    std::vector<cudaEvent_t> v;
    void push_back(cudaEvent_t e) { v.push_back(e); }
    ~Owned() {
      for (auto e : v) cudaEventDestroy(e);
    }
  } owned_;
};

// nnet.py:143-161 for R rows: query, attention (-> ctx into XS), GRU phase
// A/B, deep output, logits (fused top-k partials or full logits).
struct LogitOut {
  bool fused;
  int kk, ntiles;
  float *pmax, *psum, *cval;
  int *ctok;
  const LogitTcMaps *tc = nullptr;  // tensor-core path when set
  bool rows = false;                // tc maps are rows-layout maps (logits_rows.cu)
  const uint32_t *vmask = nullptr;  // per-sentence shortlist masks (tensor-core path)
  int mask_words = 0;
  // gathered shortlist columns (tensor-core path): the bucket's union U of
  // shortlist ids, its W_logit rows and biases; 0 / nullptr = full vocabulary
  int n_vocab = 0;
  const int *vid = nullptr;
  const float *bias = nullptr;
};

// Tensor-core (3xTF32, swap-AB cluster split-K, gemm_sk.cuh) versions of the
// four decoder-step GEMMs of one model: tensor maps over the hi/lo row
// buffers and split counts fixed by (N, K) only.
struct TcStep {
  SkMaps q, g, u, o;
  int sq = 1, sg = 1, su = 1, so = 1;
  bool proj = false;  // projected-context maps below are valid
  SkMaps qs, os;      // s [W_att_s | U_zr]; s' W_o^s
  int sqs = 1, sos = 1;
  bool dq_ok = false;  // s' [W_o^s | 0 | W_att_s | U_zr] (deep output + next query) is valid
  SkMaps dq;
  int sdq = 1;
};

// target CTAs per decoder-step GEMM launch (env AMUN_TC_CTAS overrides)
int tc_target_ctas() {
  static int v = [] {
    const char *e = getenv("AMUN_TC_CTAS");
    // AMUN_TC_CTAS caps CTAs per GEMM launch; the default (12, swept) keeps every
    // decoder GEMM at one K split: each launch is SM-efficient and the
    // concurrent bucket lanes fill the machine
    return e ? std::max(1, atoi(e)) : 12;
  }();
  return v;
}

void tc_step_maps(const amun_model *m, const DecBufs &d, int Rmax, TcStep &ts) {
  const int de = m->d.d_emb, dh = m->d.d_h, da = m->d.d_att, xp = m->xsp, dep = m->dep;
  const int s_off = dep + 2 * dh;  // padded fp16 row layout
  ts.q = make_sk_maps(d.XSh + s_off, d.XSl + s_off, dh, xp, nullptr, nullptr, 0, 0, Rmax, m->Wq_hi, m->Wq_lo, da,
                      dh, m->us_q);
  // with the per-token y tables (m->YWg / YWo) the GRU-A and deep-output
  // GEMMs run over [c | s] only: their A rows and weight rows start at
  // column dep (the epilogues add the y rows' products from the tables)
  const int y0 = m->YWg ? dep : 0;
  ts.g = make_sk_maps(d.XSh + y0, d.XSl + y0, xp - y0, xp, nullptr, nullptr, 0, 0, Rmax, m->Wg_hi + y0,
                      m->Wg_lo + y0, 3 * dh, xp - y0, m->us_g, -1, xp);
  if ((2 * dh) % 256 == 0) {  // h-gate features: the state rows' weights are zero
    ts.g.n_klim = 2 * dh;
    ts.g.k_lim = dep - y0 + 2 * dh;
  }
  ts.u = make_sk_maps(d.RHh, d.RHl, dh, dh, nullptr, nullptr, 0, 0, Rmax, m->Uhd_hi, m->Uhd_lo, dh, dh, m->us_u);
  ts.o = make_sk_maps(d.XSh + y0, d.XSl + y0, s_off - y0, xp, d.Snh, d.Snl, dh, dh, Rmax, m->Wo_hi + y0,
                      m->Wo_lo + y0, de, xp - y0, m->us_o, -1, xp);
  const int t = tc_target_ctas();
  ts.sq = sk_fit_splits(ts.q, t);
  ts.sg = sk_fit_splits(ts.g, t);
  ts.su = sk_fit_splits(ts.u, t);
  ts.so = sk_fit_splits(ts.o, t);
  ts.proj = proj_ok(m) && d.SU;
  if (ts.proj) {
    ts.qs = make_sk_maps(d.XSh + s_off, d.XSl + s_off, dh, xp, nullptr, nullptr, 0, 0, Rmax, m->Wqs_hi, m->Wqs_lo,
                         da + 2 * dh, dh, m->us_qs);
    ts.os = make_sk_maps(d.Snh, d.Snl, dh, dh, nullptr, nullptr, 0, 0, Rmax, m->Wo_hi + s_off, m->Wo_lo + s_off, de,
                         dh, m->us_o, -1, xp);
    ts.sqs = sk_fit_splits(ts.qs, t);
    ts.sos = sk_fit_splits(ts.os, t);
    ts.dq_ok = m->Wdq_hi != nullptr && fold_query();
    if (ts.dq_ok) {
      ts.dq = make_sk_maps(d.Snh, d.Snl, dh, dh, nullptr, nullptr, 0, 0, Rmax, m->Wdq_hi, m->Wdq_lo,
                           dep + da + 2 * dh, dh, m->us_dq);
      ts.sdq = sk_fit_splits(ts.dq, t);
    }
  }
}


// HX rows [row0, row0 + M) of a store whose split annotations are Hah/Hal
// ([rows][2dh]): h [C_z | C_r | C_h] (the c rows of the gate weights) and
// h W_o^c (the c rows of the deep output), both views of the step weights.
void compute_hx(Ctx &c, const amun_model *m, const __half *Hah, const __half *Hal, long long store_rows,
                long long row0, int M, float *HX, int target) {
  const int dh = m->d.d_h, de = m->d.d_emb, xp = m->xsp, dep = m->dep, ld = proj_ldhx(m);
  const SkMaps mg = make_sk_maps(Hah, Hal, 2 * dh, 2 * dh, nullptr, nullptr, 0, 0, (int)store_rows, m->Wg_hi + dep,
                                 m->Wg_lo + dep, 3 * dh, 2 * dh, m->us_g, -1, xp);
  const SkMaps mo = make_sk_maps(Hah, Hal, 2 * dh, 2 * dh, nullptr, nullptr, 0, 0, (int)store_rows, m->Wo_hi + dep,
                                 m->Wo_lo + dep, de, 2 * dh, m->us_o, -1, xp);
  const auto gg = ahead_grid(mg, M, target);
  const auto go = ahead_grid(mo, M, target);
  EpiStore eg{HX + row0 * ld, ld, nullptr, 0, 0};
  EpiStore eo{HX + row0 * ld + 3 * dh, ld, nullptr, 0, 0};
  c.run(AMUN_K_ENCODER, [&] { launch_gemm_sk(mg, M, gg.first, eg, c.st, 0, (int)row0, gg.second); });
  c.run(AMUN_K_ENCODER, [&] { launch_gemm_sk(mo, M, go.first, eo, c.st, 0, (int)row0, go.second); });
}

// one launch: tensor-core partials, DSMEM split reduction, fused epilogue
// profiling knobs (outputs invalid): AMUN_DEBUG_SK_FLAGS / AMUN_DEBUG_LOGIT_FLAGS
// skip parts of the decoder-step tensor-core kernels (gemm_sk.cuh SkArgs.debug,
// logits_tc.cu debug_flags) to attribute the pass time
int debug_env(const char *name) {
  const char *e = getenv(name);
  return e ? (int)strtol(e, nullptr, 0) : 0;
}
template <class Epi>
void gemm_tc(Ctx &c, const SkMaps &maps, int M, int splits, const Epi &epi) {
  static const int dbg = debug_env("AMUN_DEBUG_SK_FLAGS");
  c.run(c.cls, [&] { launch_gemm_sk(maps, M, splits, epi, c.st, dbg); });
}

// Projected-context step, query folded forward: Q, e^{2q} and s U_zr of the
// rows' current states (a bucket's first step, the parity hook); later steps
// get them from the previous step's deep-output GEMM (EpiDQ).
void qs_prologue(Ctx &c, const amun_model *m, const DecBufs &d, const TcStep &ts, int R) {
  const int cls = c.cls;
  c.cls = AMUN_K_QUERY;
  gemm_tc(c, ts.qs, R, ts.sqs, EpiQS{d.Q, d.EQ, d.SU, m->d.d_att, 2 * m->d.d_h});
  c.cls = cls;
}

void step_rows(Ctx &c, const amun_model *m, const DecBufs &d, const EncBufs &e, const int *d_len, int jmax,
               int R, int rows_per_sent, const int *n_act, const int *done, float *alpha, const LogitOut &lo,
               const TcStep *ts = nullptr, bool do_logits = true, const int *tok = nullptr,
               const int *qrow = nullptr) {
  const int de = m->d.d_emb, dh = m->d.d_h, da = m->d.d_att, V = m->d.v_trg, xs = m->xs_w;
  const int s_off = de + 2 * dh;
  const bool proj = ts && ts->proj && e.HX;
  // folded query: Q / EQ / s U_zr of each row's parent come from the previous
  // step's deep-output GEMM (or qs_prologue), indexed through qrow
  const bool fold = proj && qrow && ts->dq_ok && lo.tc;
  if (proj) {  // projected-context step (proj_ok): query + s U_zr, attention with the gate math
    if (!tok) throw Error(AMUN_ERR_CUDA, "step_rows: previous tokens required with the y tables");
    c.cls = AMUN_K_QUERY;
    if (!fold) gemm_tc(c, ts->qs, R, ts->sqs, EpiQS{d.Q, d.EQ, d.SU, da, 2 * dh});
    AttnArgs aa{d.Q, da, e.P, e.HX, m->v_att, d_len, jmax, da, proj_ldhx(m), rows_per_sent, n_act, done,
                nullptr, 0, alpha};
    aa.energy = d.En;
    aa.EQ = d.EQ;
    aa.su = d.SU;
    aa.S = d.XS + s_off;
    aa.lds = xs;
    aa.tok = tok;
    aa.ywg = m->YWg;
    aa.ywo = m->YWo;
    aa.bg = m->bg;
    aa.Z = d.Z;
    aa.XH = d.XH;
    aa.RHh = d.RHh;
    aa.RHl = d.RHl;
    aa.CO = d.CO;
    aa.dh = dh;
    aa.de = de;
    aa.ldco = m->dep;
    if (fold) aa.qrow = qrow;
    int na_launch = 1;
    c.run(AMUN_K_ATTN, [&] { na_launch = launch_attention(aa, R, c.st); });
    c.launches += na_launch - 1;
  } else {
  c.cls = AMUN_K_QUERY;
  {
    EpiStore eq{d.Q, da, nullptr, 0, 0};
    eq.ex2 = d.EQ;
    if (ts)
      gemm_tc(c, ts->q, R, ts->sq, eq);
    else
      gemm(c, ga(R, da, d.XS + s_off, xs, dh, m->W_att_s, da), eq);
  }
  AttnArgs aa{d.Q, da, e.P, e.Hann, m->v_att, d_len, jmax, da, 2 * dh, rows_per_sent, n_act, done,
              d.XS + de, xs, alpha};
  aa.energy = d.En;
  aa.EQ = d.EQ;
  if (ts) {
    aa.ctx_hi = d.XSh + m->dep;
    aa.ctx_lo = d.XSl + m->dep;
    aa.ldctx_h = m->xsp;
  }
  int na_launch = 1;
  c.run(AMUN_K_ATTN, [&] { na_launch = launch_attention(aa, R, c.st); });
  c.launches += na_launch - 1;
  c.cls = AMUN_K_GRU_A;
  {
    EpiGruA ea{m->bg, d.XS + s_off, xs, dh, d.Z, d.RH, d.XH};
    if (ts) {
      ea.RHh = d.RHh;
      ea.RHl = d.RHl;
      if (m->YWg) {  // y rows' products from the per-token table (tc_step_maps)
        if (!tok) throw Error(AMUN_ERR_CUDA, "step_rows: previous tokens required with the y tables");
        ea.rowadd = m->YWg;
        ea.rowtok = tok;
        ea.ldadd = 3 * dh;
      }
      gemm_tc(c, ts->g, R, ts->sg, ea);
    } else {
      GemmArgs g = ga(R, 3 * dh, d.XS, xs, xs, m->Wg, 3 * dh);
      g.n_split = 2 * dh;
      g.k_limit = de + 2 * dh;
      gemm(c, g, ea);
    }
  }
  }  // GRU-A step
  c.cls = AMUN_K_GRU_B;
  {
    EpiGruB eb{d.XS + s_off, xs, dh, d.Z, d.XH, d.Sn};
    if (ts) {
      eb.Snh = d.Snh;
      eb.Snl = d.Snl;
      gemm_tc(c, ts->u, R, ts->su, eb);
    } else {
      gemm(c, ga(R, dh, d.RH, dh, dh, m->Uh_dec, dh), eb);
    }
  }
  c.cls = AMUN_K_OUT;
  {
    EpiStore e{lo.tc ? nullptr : d.T, de, m->b_out, 1, 0};
    if (lo.tc) {
      e.hi = d.T_hi;
      e.lo = d.T_lo;
      e.ldh = m->dep;
    }
    if (fold) {  // s' [W_o^s | 0 | W_att_s | U_zr]: deep output + the next step's query
      EpiDQ eq{d.CO, m->dep, m->b_out, d.T_hi, d.T_lo, m->dep, de, m->dep, EpiQS{d.Q, d.EQ, d.SU, da, 2 * dh}};
      gemm_tc(c, ts->dq, R, ts->sdq, eq);
    } else if (proj) {  // s' W_o^s + (context + y term from the attention kernel)
      e.rowadd = d.CO;
      e.ldadd = m->dep;
      gemm_tc(c, ts->os, R, ts->sos, e);
    } else if (ts) {
      if (m->YWo) {
        e.rowadd = m->YWo;
        e.rowtok = tok;
        e.ldadd = de;
      }
      gemm_tc(c, ts->o, R, ts->so, e);
    } else {
      GemmArgs g = ga(R, de, d.XS, xs, de + 2 * dh, m->Wout, de);
      g.a1 = d.Sn;
      g.lda1 = dh;
      g.k1 = dh;
      gemm(c, g, e);
    }
  }
  if (!do_logits) return;  // ensemble members: one fused logit launch for all of them
  c.cls = AMUN_K_LOGIT;
  if (lo.tc) {
    LogitTcArgs ta{R, lo.n_vocab ? lo.n_vocab : V, de, lo.bias ? lo.bias : m->b_logit, lo.kk, lo.ntiles, m->us_l,
                   lo.pmax, lo.psum, lo.cval, lo.ctok};
    ta.vid = lo.vid;
    ta.vmask = lo.vmask;
    ta.mask_words = lo.mask_words;
    ta.rows_per_sent = rows_per_sent;
    static const int ldbg = debug_env("AMUN_DEBUG_LOGIT_FLAGS");
    ta.debug_flags = ldbg;
    if (lo.rows)
      c.run(AMUN_K_LOGIT, [&] { launch_logits_rows(*lo.tc, ta, c.st); });
    else
      c.run(AMUN_K_LOGIT, [&] { launch_logits_tc(*lo.tc, ta, c.st); });
    return;
  }
  GemmArgs g = ga(R, V, d.T, de, de, m->W_logit, V);
  if (lo.fused)
    gemm(c, g, EpiLogitTopK{m->b_logit, lo.kk, lo.ntiles, lo.pmax, lo.psum, lo.cval, lo.ctok});
  else
    gemm(c, g, EpiStore{d.L, V, m->b_logit, 0, 0});
}

__global__ void split_rows_kernel(const float *__restrict__ x, long long n, __half *hi, __half *lo) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) store_split(hi, lo, i, x[i]);
}

__global__ void build_rows_kernel(float *XS, int ldxs, const float *E, const int *y, const float *s, int de, int dh,
                                  int s_off) {
  const int r = blockIdx.x;
  float *row = XS + (long long)r * ldxs;
  for (int c = threadIdx.x; c < de; c += blockDim.x) row[c] = y ? E[(long long)y[r] * de + c] : 0.f;
  for (int c = threadIdx.x; c < dh; c += blockDim.x) row[s_off + c] = s[(long long)r * dh + c];
}

struct HostHyp {
  double score;
  int finished;
  std::vector<int> toks;
  std::vector<float> state;  // n_models * dh (optional)
};

// Flat amun_result over the sentences `sel` (in that order) of out_hyps.
// States: per hypothesis the members' final state rows concatenated
// (width sw = sum of the members' d_h; d_h reports member 0's).
amun_result *flatten_hyps(const std::vector<std::vector<HostHyp>> &out_hyps, const int *sel, int n, int n_models,
                          int dh, int sw, bool want_states) {
  amun_result *r = static_cast<amun_result *>(calloc(1, sizeof(amun_result)));
  r->n_sent = n;
  r->n_models = n_models;
  r->d_h = dh;
  int64_t nh = 0, nt = 0;
  for (int i = 0; i < n; ++i)
    for (auto &h : out_hyps[sel[i]]) {
      ++nh;
      nt += (int64_t)h.toks.size();
    }
  r->n_hyp = nh;
  r->hyp_offsets = static_cast<int32_t *>(malloc(sizeof(int32_t) * (n + 1)));
  r->scores = static_cast<double *>(malloc(sizeof(double) * std::max<int64_t>(nh, 1)));
  r->finished = static_cast<int32_t *>(malloc(sizeof(int32_t) * std::max<int64_t>(nh, 1)));
  r->tok_offsets = static_cast<int64_t *>(malloc(sizeof(int64_t) * (nh + 1)));
  r->tokens = static_cast<int32_t *>(malloc(sizeof(int32_t) * std::max<int64_t>(nt, 1)));
  r->states = want_states ? static_cast<float *>(malloc(sizeof(float) * std::max<int64_t>(nh * sw, 1)))
                          : nullptr;
  int64_t hi = 0, ti = 0;
  r->tok_offsets[0] = 0;
  for (int i = 0; i < n; ++i) {
    r->hyp_offsets[i] = (int32_t)hi;
    for (auto &h : out_hyps[sel[i]]) {
      r->scores[hi] = h.score;
      r->finished[hi] = h.finished;
      std::copy(h.toks.begin(), h.toks.end(), r->tokens + ti);
      ti += (int64_t)h.toks.size();
      r->tok_offsets[hi + 1] = ti;
      if (r->states) std::copy(h.state.begin(), h.state.end(), r->states + hi * sw);
      ++hi;
    }
  }
  r->hyp_offsets[n] = (int32_t)hi;
  return r;
}


}  // namespace

// ====================================================================== decode

amun_result *decode_run(const std::vector<amun_model *> &ms, const int32_t *src_ids, const int32_t *src_len,
                        int n_sent, const int32_t *sl_ids, const int32_t *sl_len, const amun_decode_opts &o,
                        amun_bucket_done_fn on_bucket, void *user) {
  const auto t_enter = std::chrono::steady_clock::now();
  amun_model *m0 = ms[0];
  AMUN_CUDA(cudaSetDevice(m0->device));
  const int n_models = (int)ms.size();
  const int k = o.beam_size;
  if (k < 1) throw Error(AMUN_ERR_INVALID, "beam_size must be >= 1, got " + std::to_string(k));
  if (o.n_best < 1) throw Error(AMUN_ERR_INVALID, "n_best must be >= 1, got " + std::to_string(o.n_best));
  const int V = m0->d.v_trg, Vs = m0->d.v_src, dh = m0->d.d_h;
  if (n_models > kMaxModels)
    throw Error(AMUN_ERR_UNSUPPORTED, "at most " + std::to_string(kMaxModels) + " ensemble members are supported");
  int state_w = 0;  // concatenated final-state width of all members
  for (auto *m : ms) state_w += m->d.d_h;
  std::vector<long long> off(n_sent + 1, 0), sl_offs(n_sent + 1, 0);
  for (int i = 0; i < n_sent; ++i) {
    if (src_len[i] < 1) throw Error(AMUN_ERR_INVALID, "cannot decode an empty source sentence");
    long long cap = (long long)o.max_len_factor * src_len[i] + o.max_len_offset;
    if (cap < 1) throw Error(AMUN_ERR_INVALID, "length cap " + std::to_string(cap) + " must be >= 1");
    off[i + 1] = off[i] + src_len[i];
    if (sl_ids) {
      if (sl_len[i] < 1) throw Error(AMUN_ERR_INVALID, "shortlist must be non-empty");
      sl_offs[i + 1] = sl_offs[i] + sl_len[i];
    }
  }
  for (long long j = 0; j < off[n_sent]; ++j)
    if (src_ids[j] < 0 || src_ids[j] >= Vs)
      throw Error(AMUN_ERR_INVALID, "source id " + std::to_string(src_ids[j]) + " out of range for v_src=" +
                                        std::to_string(Vs));
  if (sl_ids)
    for (long long j = 0; j < sl_offs[n_sent]; ++j)
      if (sl_ids[j] < 0 || sl_ids[j] >= V)
        throw Error(AMUN_ERR_INVALID, "shortlist id " + std::to_string(sl_ids[j]) + " out of range for v_trg=" +
                                          std::to_string(V));

  if (n_sent == 0) {  // nothing to decode: no lanes, no tensor maps
    amun_result *r = flatten_hyps({}, nullptr, 0, n_models, dh, state_w, o.want_states);
    r->host_setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_enter).count();
    return r;
  }
  const int Bmax_opt = o.max_batch > 0 ? o.max_batch : 64;
  const char *no_tc = getenv("AMUN_NO_TC");
  const bool tc_logits = m0->Wl_hi && !(no_tc && no_tc[0] == '1');
  // shortlists ride the fused tensor-core logit kernel as per-sentence
  // vocabulary masks; the CUDA-core fused kernel has no mask (full logits)
  // ensembles of up to kLogitMembers tensor-core members run one fused
  // logit launch for all members (member-sum candidates + per-member
  // log-softmax partials); larger ensembles take the full-logit path
  bool ens_tc = n_models > 1 && n_models <= kLogitMembers && tc_logits;
  for (auto *m : ms) ens_tc = ens_tc && m->Wl_hi;
  const bool fused = (n_models == 1 || ens_tc) && (!sl_ids || tc_logits) && k <= kMaxRowCand && !o.force_full_logits;
  const bool ens_fused = fused && n_models > 1;
  const bool use_tc = fused && tc_logits;
  // AMUN_LOGIT_ROWS=1 / 0 forces the rows-layout / swap-AB logit kernel
  const char *rows_env = getenv("AMUN_LOGIT_ROWS");
  // beams >= 8: the rows-layout kernel (one row per epilogue thread) wins
  // over the swap-AB kernel (cfg4: +25%); smaller beams keep swap-AB.  The
  // choice depends on per-call constants only (the beam), never on a
  // bucket's size, so a sentence's result never depends on its batch-mates.
  const bool use_rows = use_tc && n_models == 1 &&
                        (rows_env ? rows_env[0] == '1' : k >= 8);
  const int tile_n = use_rows ? kLogitRowsTileN : kBN;
  const bool use_mask = fused && sl_ids != nullptr;
  const int mask_words = ceil_div(V, 32);
  // shortlist buckets whose union of ids is at most gather_cap wide run their
  // logits over the gathered union (fewer weight bytes and MMAs per step);
  // wider unions keep the full-vocabulary masked kernel
  const char *gfe = getenv("AMUN_SL_GATHER_FRAC");
  const double gfrac = gfe ? atof(gfe) : 0.9;
  const int gather_cap = (use_mask && use_tc && gfrac > 0 && n_models == 1) ? std::min(V, (int)(gfrac * V)) : 0;
  std::vector<int> gstamp(gather_cap > 0 ? V : 0, -1), gpos(gather_cap > 0 ? V : 0, 0);
  const char *no_tcg = getenv("AMUN_NO_TC_GEMM");
  bool use_tcg = !(no_tc && no_tc[0] == '1') && !(no_tcg && no_tcg[0] == '1');
  for (auto *m : ms) use_tcg = use_tcg && m->tc_gemm;
  const char *no_tce = getenv("AMUN_NO_TC_ENC");
  bool use_tce = !(no_tc && no_tc[0] == '1') && !(no_tce && no_tce[0] == '1');
  for (auto *m : ms) use_tce = use_tce && m->Uzr_hi;
  // encode-ahead: the whole chunk's encoder before its buckets decode
  // (tensor-core models); AMUN_NO_AHEAD=1 encodes per bucket in the lanes
  const char *no_ahead = getenv("AMUN_NO_AHEAD");
  bool ahead = use_tce && !(no_ahead && no_ahead[0] == '1');
  for (auto *m : ms) ahead = ahead && m->Efa_hi[0];
  const int kk = std::min(k, V);
  const int ntiles = ceil_div(V, kBN);

  // length buckets: stable sort by source length, cut every Bmax sentences
  std::vector<int> order(n_sent);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return src_len[a] < src_len[b]; });
  struct Bucket {
    int first, count, jmax, cap_max;
  };
  std::vector<Bucket> buckets;
  int Bmax = 0, jmax_all = 0, cap_all = 0, sl_max = 0;
  for (int s = 0; s < n_sent; s += Bmax_opt) {
    Bucket bk{s, std::min(Bmax_opt, n_sent - s), 0, 0};
    for (int i = bk.first; i < bk.first + bk.count; ++i) {
      int L = src_len[order[i]];
      bk.jmax = std::max(bk.jmax, L);
      bk.cap_max = std::max(bk.cap_max, o.max_len_factor * L + o.max_len_offset);
    }
    Bmax = std::max(Bmax, bk.count);
    jmax_all = std::max(jmax_all, bk.jmax);
    cap_all = std::max(cap_all, bk.cap_max);
    if (sl_ids) {
      int tot = 0;
      for (int i = bk.first; i < bk.first + bk.count; ++i) tot += sl_len[order[i]];
      sl_max = std::max(sl_max, tot);
    }
    buckets.push_back(bk);
  }
  const int Rmax = Bmax * k;
  const int fin_cap = k * cap_all;
  const int de = m0->d.d_emb;

  // ---- lanes: each lane = stream + workspace + captured step graph and
  // decodes one length bucket at a time; lanes run concurrently so that
  // small kernels of one bucket overlap with another bucket's GEMMs (every
  // bucket is still one batch of <= max_batch sentences).
  const char *lanes_env = getenv("AMUN_LANES");
  int n_lanes = lanes_env ? std::max(1, atoi(lanes_env)) : 24;
  const uint32_t prof_ev = (uint32_t)o.profile & 0xFFu;  // classes timed with per-launch events
  const bool cta_time = (o.profile & AMUN_PROFILE_CTA_TIME) != 0;
  if (prof_ev) n_lanes = 1;  // per-launch event timing wants one ordered stream
  n_lanes = std::max(1, std::min<int>(n_lanes, (int)buckets.size()));
  const char *no_graph = getenv("AMUN_NO_GRAPH");
  const bool graphs_ok = prof_ev == 0 && !(no_graph && no_graph[0] == '1');
  struct KtBuf {  // device CTA-time accumulators [class][ns, CTAs]
    unsigned long long *p = nullptr;
    ~KtBuf() {
      if (p) cudaFree(p);
    }
  } ktb;
  if (cta_time) {
    AMUN_CUDA(cudaMalloc(&ktb.p, sizeof(unsigned long long) * 2 * AMUN_K_CLASSES));
    AMUN_CUDA(cudaMemset(ktb.p, 0, sizeof(unsigned long long) * 2 * AMUN_K_CLASSES));
  }
  constexpr int kProbeEvery = 8, kMaxAhead = 16;

  struct Lane {
    cudaStream_t st = nullptr;
    std::unique_ptr<Ctx> c;
    std::vector<EncBufs> eb;
    std::vector<DecBufs> db;
    std::vector<float *> fin_states;
    std::vector<TcStep> tsteps;
    std::vector<TcEnc> tencs;
    int *d_ids, *d_len, *d_cap, *d_sl, *d_sl_off, *d_sl_len;
    uint32_t *d_vmask = nullptr;  // [Bmax][mask_words] shortlist masks (fused path)
    // gathered shortlist columns (buckets whose union U fits gather_cap)
    int *d_U = nullptr;
    __half *Wg_hi = nullptr, *Wg_lo = nullptr;
    float *bg = nullptr;
    uint32_t *d_vmask_g = nullptr;  // [Bmax][ceil(gather_cap / 32)] masks over U
    LogitTcMaps tc_maps_g{};
    float *pmax, *psum, *cval;
    int *ctok, *cand_tok;
    double *cand_lp;
    BeamState bs{};
    float **p_XS;
    const float **p_Sn, **p_E, **p_S0, **p_L;
    float **p_fin;
    __half **p_XSh, **p_XSl;
    LogitTcMaps tc_maps{};
    std::vector<LogitTcMaps> tc_maps_ens;  // fused ensemble logits: one map set per member
    LaneRes *res = nullptr;  // pooled stream / workspace / probe ring
    int dev = 0;
    void *mem = nullptr;
    int *h_probe = nullptr;  // pinned ring of n_done probes
    cudaEvent_t *probe_ev = nullptr;
    std::deque<std::pair<int, int>> pending;  // (step, slot)
    int probe_next = 0;
    // current bucket
    bool active = false, stop = false;
    int bucket = -1, B = 0, jmax = 0, capm = 0, R = 0, t = 0;
    ModelRows mr{};
    LogitOut lo{};
    SelectArgs sa{};
    cudaGraphExec_t gexec = nullptr;
    bool gstale = false;
    int64_t step_launches = 0;
    ~Lane() {
      static const bool dbg = getenv("AMUN_DEBUG_TEARDOWN") != nullptr;
      auto t0 = std::chrono::steady_clock::now();
      if (res) res->gexec = gexec;  // kept (stale) for the next call to update
      c.reset();
      auto t1 = std::chrono::steady_clock::now();
      if (res) {  // back to the pool once this call's work on the stream is done
        cudaStreamSynchronize(st);
        lane_release(dev, res);
      }
      auto t2 = std::chrono::steady_clock::now();
      if (dbg)
        fprintf(stderr, "lane teardown: ctx %.2f ms, sync+release %.2f ms\n",
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(t2 - t1).count());
    }
  };
  std::vector<std::unique_ptr<Lane>> lanes;
  for (int li = 0; li < n_lanes; ++li) {
    lanes.emplace_back(new Lane());
    Lane &L = *lanes.back();
    L.dev = m0->device;
    L.res = lane_acquire(L.dev, li >= n_lanes - high_priority_lanes());
    L.st = L.res->st;
    L.h_probe = L.res->h_probe;
    L.probe_ev = L.res->ev.data();
    // a pooled step graph is only updated in place for the same models and
    // options (same kernels and cluster shapes; buckets differ in arguments
    // and grid sizes only); otherwise it is rebuilt
    {
      std::vector<uintptr_t> key;
      for (auto *m : ms) key.push_back(reinterpret_cast<uintptr_t>(m));
      for (int v : {k, (int)use_tc, (int)use_tcg, (int)fused, (int)(sl_ids != nullptr), (int)o.want_states, Bmax,
                    jmax_all, cap_all})
        key.push_back((uintptr_t)(unsigned)v);
      if (L.res->gexec && L.res->gkey != key) {
        cudaGraphExecDestroy(L.res->gexec);
        L.res->gexec = nullptr;
      }
      L.res->gkey = key;
    }
    L.gexec = L.res->gexec;
    L.gstale = true;
    L.c.reset(new Ctx(L.st));
    L.c->ws = L.res->ws;
    L.c->ws_floats = L.res->ws_floats;
    L.c->ws_keep = &L.res->ws;
    L.c->ws_keep_n = &L.res->ws_floats;
    L.c->ws_pool = ws_pool(L.dev);
    L.c->prof = prof_ev;
    L.c->kt = ktb.p;
    L.eb.resize(n_models);
    L.db.resize(n_models);
    L.fin_states.assign(n_models, nullptr);
    L.tsteps.resize(n_models);
    L.tencs.resize(n_models);
    for (int pass = 0; pass < 2; ++pass) {
      Carver cv;
      cv.base = pass ? static_cast<char *>(L.mem) : nullptr;
      for (int m = 0; m < n_models; ++m) {
        if (!ahead) {
          carve_enc(cv, L.eb[m], ms[m], Bmax, jmax_all);
          if (use_tce) carve_enc_tc(cv, L.eb[m], ms[m], Bmax, jmax_all);
        }
        carve_dec(cv, L.db[m], ms[m], Rmax, jmax_all, !fused);
        if (!use_tc) L.db[m].T_hi = L.db[m].T_lo = nullptr;
        if (use_tcg) {
          carve_dec_tc(cv, L.db[m], ms[m], Rmax);
        }
        L.fin_states[m] = o.want_states ? cv.take<float>((size_t)Bmax * fin_cap * ms[m]->d.d_h) : nullptr;
      }
      L.d_ids = cv.take<int>((size_t)Bmax * jmax_all);
      L.d_len = cv.take<int>(Bmax);
      L.d_cap = cv.take<int>(Bmax);
      L.d_sl = cv.take<int>(std::max(sl_max, 1));
      L.d_vmask = cv.take<uint32_t>(use_mask ? (size_t)Bmax * mask_words : 1);
      if (gather_cap > 0) {
        L.d_U = cv.take<int>(gather_cap);
        L.Wg_hi = cv.take<__half>((size_t)gather_cap * m0->dep);
        L.Wg_lo = cv.take<__half>((size_t)gather_cap * m0->dep);
        L.bg = cv.take<float>(gather_cap);
        L.d_vmask_g = cv.take<uint32_t>((size_t)Bmax * ceil_div(gather_cap, 32));
      }
      L.d_sl_off = cv.take<int>(Bmax);
      L.d_sl_len = cv.take<int>(Bmax);
      L.pmax = cv.take<float>(fused ? (size_t)ntiles * Rmax * n_models : 1);
      L.psum = cv.take<float>(fused ? (size_t)ntiles * Rmax * n_models : 1);
      L.cval = cv.take<float>(fused ? (size_t)Rmax * ntiles * kk : 1);
      L.ctok = cv.take<int>(fused ? (size_t)Rmax * ntiles * kk : 1);
      L.cand_lp = cv.take<double>((size_t)Rmax * kk);
      L.cand_tok = cv.take<int>((size_t)Rmax * kk);
      BeamState &bs = L.bs;
      bs.n_act = cv.take<int>(Bmax);
      bs.score = cv.take<double>(Rmax);
      bs.tok = cv.take<int>(Rmax);
      bs.qrow = cv.take<int>(Rmax);
      bs.done = cv.take<int>(Bmax);
      bs.steps = cv.take<int>(Bmax);
      bs.cap = L.d_cap;
      bs.fin_n = cv.take<int>(Bmax);
      bs.fin_score = cv.take<double>((size_t)Bmax * fin_cap);
      bs.fin_t = cv.take<int>((size_t)Bmax * fin_cap);
      bs.fin_par = cv.take<int>((size_t)Bmax * fin_cap);
      bs.best_fin = cv.take<double>(Bmax);
      bs.bp_tok = cv.take<int>((size_t)Bmax * cap_all * k);
      bs.bp_par = cv.take<int>((size_t)Bmax * cap_all * k);
      bs.n_done = cv.take<int>(1);
      L.p_XS = cv.take<float *>(n_models);
      L.p_Sn = cv.take<const float *>(n_models);
      L.p_E = cv.take<const float *>(n_models);
      L.p_S0 = cv.take<const float *>(n_models);
      L.p_L = cv.take<const float *>(n_models);
      L.p_fin = cv.take<float *>(n_models);
      L.p_XSh = cv.take<__half *>(n_models);
      L.p_XSl = cv.take<__half *>(n_models);
      if (!pass) L.mem = lane_mem(L.res, cv.off, ws_pool(L.dev));
    }
    if (use_tc) {
      static_assert(kBN == 128, "fused-logit tile width shared by SIMT and tensor-core paths");
      if (logits_tc_tile_n() != kBN) throw Error(AMUN_ERR_UNSUPPORTED, "logit tile width mismatch");
      L.tc_maps = use_rows ? make_logit_rows_maps(L.db[0].T_hi, L.db[0].T_lo, Rmax, de, m0->dep, m0->Wl_hi,
                                                  m0->Wl_lo, m0->dep, V)
                           : make_logit_maps(L.db[0].T_hi, L.db[0].T_lo, Rmax, de, m0->dep, m0->Wl_hi, m0->Wl_lo,
                                             m0->dep, V);
      if (ens_fused) {
        L.tc_maps_ens.resize(n_models);
        for (int m = 0; m < n_models; ++m)
          L.tc_maps_ens[m] = make_logit_maps(L.db[m].T_hi, L.db[m].T_lo, Rmax, ms[m]->d.d_emb, ms[m]->dep,
                                             ms[m]->Wl_hi, ms[m]->Wl_lo, ms[m]->dep, V);
      }
    }
    if (use_tcg)
      for (int m = 0; m < n_models; ++m) tc_step_maps(ms[m], L.db[m], Rmax, L.tsteps[m]);
    if (use_tce && !ahead)
      for (int m = 0; m < n_models; ++m) tc_enc_maps(ms[m], L.eb[m], Bmax, jmax_all, L.tencs[m]);
    std::vector<const void *> hx(n_models), hs(n_models), he(n_models), h0(n_models), hl(n_models), hf(n_models),
        hxh(n_models), hxl(n_models);
    for (int m = 0; m < n_models; ++m) {
      hx[m] = L.db[m].XS;
      hs[m] = L.db[m].Sn;
      he[m] = ms[m]->E_trg;
      h0[m] = L.eb[m].S0;
      hl[m] = L.db[m].L;
      hf[m] = L.fin_states[m];
      hxh[m] = L.db[m].XSh;
      hxl[m] = L.db[m].XSl;
    }
    Ctx &c = *L.c;
    h2d(c, (const void **)L.p_XS, hx.data(), n_models);
    h2d(c, (const void **)L.p_Sn, hs.data(), n_models);
    h2d(c, (const void **)L.p_E, he.data(), n_models);
    h2d(c, (const void **)L.p_S0, h0.data(), n_models);
    h2d(c, (const void **)L.p_L, hl.data(), n_models);
    h2d(c, (const void **)L.p_fin, hf.data(), n_models);
    h2d(c, (const void **)L.p_XSh, hxh.data(), n_models);
    h2d(c, (const void **)L.p_XSl, hxl.data(), n_models);
    if (use_tcg)  // pad columns of the fp16 rows must read as zero
      for (int m = 0; m < n_models; ++m) {
        AMUN_CUDA(cudaMemsetAsync(L.db[m].XSh, 0, sizeof(__half) * (size_t)Rmax * ms[m]->xsp, L.st));
        AMUN_CUDA(cudaMemsetAsync(L.db[m].XSl, 0, sizeof(__half) * (size_t)Rmax * ms[m]->xsp, L.st));
      }
  }

  cudaEvent_t ev0, ev1;
  AMUN_CUDA(cudaEventCreate(&ev0));
  AMUN_CUDA(cudaEventCreate(&ev1));
  struct EvGuard {
    cudaEvent_t a, b;
    ~EvGuard() {
      cudaEventDestroy(a);
      cudaEventDestroy(b);
    }
  } evg{ev0, ev1};
  AMUN_CUDA(cudaEventRecord(ev0, lanes[0]->st));
  const auto t_ev0 = std::chrono::steady_clock::now();
  for (int li = 1; li < n_lanes; ++li) AMUN_CUDA(cudaStreamWaitEvent(lanes[li]->st, ev0, 0));

  std::vector<std::vector<HostHyp>> out_hyps(n_sent);
  long long host_launch_ns = 0, host_launch_n = 0;  // host time inside cudaGraphLaunch
  unsigned long long *sel_dbg = nullptr;  // AMUN_DEBUG_SELECT: select-kernel phase cycles
  if (getenv("AMUN_DEBUG_SELECT")) {
    AMUN_CUDA(cudaMalloc(&sel_dbg, 8 * sizeof(unsigned long long)));
    AMUN_CUDA(cudaMemset(sel_dbg, 0, 8 * sizeof(unsigned long long)));
  }
  int64_t total_steps = 0;
  size_t next_bucket = 0;
  // encode-ahead annotation stores of the current chunk (per model)
  struct Store {
    float *Hann = nullptr, *P = nullptr, *S0 = nullptr, *HX = nullptr;
    __half *Hah = nullptr, *Hal = nullptr;
    void *mem = nullptr;
  };
  // per chunk of the group in flight: stores, encoders, first sorted sentence
  std::vector<std::vector<Store>> gstores;
  std::vector<std::vector<std::unique_ptr<AheadEncoder>>> gencs;
  std::vector<int> gchunk_first;
  std::vector<int> chunk_of_bucket(buckets.size(), 0);  // chunk (within the group) of every bucket
  std::vector<long long> bucket_row(buckets.size(), 0);  // store row of (bucket's first sentence, position 0)
  // dispatch order: longest-running buckets first (step count x rows), so
  // the short ones fill the lanes at the end instead of a long bucket
  // running alone in the tail (bucket composition, hence every result, is
  // unchanged)
  std::vector<int> dispatch;
  // dispatch order inside a chunk: longest-running buckets first (step
  // count x rows), so the short ones fill the lanes at the end instead of a
  // long bucket running alone in the tail (bucket composition, hence every
  // result, is unchanged)
  auto lpt_order = [&](int b0, int b1) {
    std::vector<int> d(b1 - b0);
    std::iota(d.begin(), d.end(), b0);
    std::stable_sort(d.begin(), d.end(), [&](int x, int y) {
      const long long wx = (long long)buckets[x].cap_max * buckets[x].count * (buckets[x].jmax + 8);
      const long long wy = (long long)buckets[y].cap_max * buckets[y].count * (buckets[y].jmax + 8);
      return wx > wy;
    });
    return d;
  };

  auto launch_step = [&](Lane &L) {
    Ctx &c = *L.c;
    for (int m = 0; m < n_models; ++m)
      step_rows(c, ms[m], L.db[m], L.eb[m], L.d_len, L.jmax, L.R, k, L.bs.n_act, L.bs.done, nullptr, L.lo,
                use_tcg ? &L.tsteps[m] : nullptr, !ens_fused, L.bs.tok, L.bs.qrow);
    if (ens_fused) {  // every member's logits in one launch (search.py:56-72)
      LogitTcArgs ta{L.R, V, ms[0]->d.d_emb, ms[0]->b_logit, kk, ntiles, ms[0]->us_l,
                     L.pmax, L.psum, L.cval, L.ctok};
      ta.nm = n_models;
      for (int m = 1; m < n_models; ++m) {
        ta.K_x[m - 1] = ms[m]->d.d_emb;
        ta.bias_x[m - 1] = ms[m]->b_logit;
        ta.unscale_x[m - 1] = ms[m]->us_l;
      }
      ta.pm_stride = (long long)Rmax * ntiles;
      ta.vmask = L.lo.vmask;
      ta.mask_words = L.lo.mask_words;
      ta.rows_per_sent = k;
      c.cls = AMUN_K_LOGIT;
      c.run(AMUN_K_LOGIT, [&] { launch_logits_tc_ens(L.tc_maps_ens.data(), ta, L.st); });
    }
    c.run(AMUN_K_SELECT, [&] { launch_select(L.sa, L.bs, L.mr, L.st); });
  };

  // AMUN_DEBUG_SCHED: host-side (start, end) of every bucket, printed as a
  // lane-occupancy profile after the decode
  static const bool dbg_sched = getenv("AMUN_DEBUG_SCHED") != nullptr;
  std::vector<std::pair<double, double>> bucket_span(buckets.size(), {0.0, 0.0});
  auto now_ms = [&] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_enter).count(); };
  auto start_bucket = [&](Lane &L, int bi) {
    if (dbg_sched) bucket_span[bi].first = now_ms();
    Ctx &c = *L.c;
    const Bucket &bk = buckets[bi];
    L.bucket = bi;
    L.B = bk.count;
    L.jmax = bk.jmax;
    L.capm = bk.cap_max;
    L.R = L.B * k;
    L.t = 0;
    L.active = true;
    L.stop = false;
    L.pending.clear();
    L.gstale = true;  // the step graph is re-captured at step 1 and updated in place
    const int B = L.B, jmax = L.jmax;
    std::vector<int> ids((size_t)B * jmax, 0), lens(B), caps(B), slo(B), sll(B), slv;
    for (int i = 0; i < B; ++i) {
      int s = order[bk.first + i];
      lens[i] = src_len[s];
      caps[i] = o.max_len_factor * src_len[s] + o.max_len_offset;
      std::copy(src_ids + off[s], src_ids + off[s + 1], ids.begin() + (size_t)i * jmax);
      if (sl_ids) {
        slo[i] = (int)slv.size();
        sll[i] = sl_len[s];
        slv.insert(slv.end(), sl_ids + sl_offs[s], sl_ids + sl_offs[s + 1]);
      }
    }
    // pageable sources: cudaMemcpyAsync stages them before returning
    h2d(c, L.d_ids, ids.data(), ids.size());
    h2d(c, L.d_len, lens.data(), B);
    h2d(c, L.d_cap, caps.data(), B);
    int n_gath = 0;  // > 0: this bucket's logits run over its shortlist union only
    if (use_mask) {
      // union U of the bucket's shortlists (ascending); when it is small
      // enough, gather its W_logit rows once per bucket so every step's
      // logit GEMM has N = |U| instead of V (nnet.py:162-163 per sentence;
      // here per bucket, each sentence masked to its own list inside U)
      std::vector<int> U;
      if (gather_cap > 0) {
        for (int e = 0; e < (int)slv.size(); ++e) {
          const int v = slv[e];
          if (gstamp[v] != bi) {
            gstamp[v] = bi;
            U.push_back(v);
          }
        }
        if ((int)U.size() <= gather_cap) {
          std::sort(U.begin(), U.end());
          n_gath = (int)U.size();
        }
      }
      if (n_gath) {
        for (int j = 0; j < n_gath; ++j) gpos[U[j]] = j;
        const int words = ceil_div(n_gath, 32);
        std::vector<uint32_t> mask((size_t)B * words, 0u);
        for (int i = 0; i < B; ++i)
          for (int e = slo[i]; e < slo[i] + sll[i]; ++e) {
            const int v = gpos[slv[e]];
            mask[(size_t)i * words + v / 32] |= 1u << (v % 32);
          }
        h2d(c, L.d_vmask_g, mask.data(), mask.size());
        h2d(c, L.d_U, U.data(), U.size());
        c.run(AMUN_K_LOGIT, [&] {
          gather_logit_rows_kernel<<<n_gath, 128, 0, c.st>>>(m0->Wl_hi, m0->Wl_lo, m0->b_logit, m0->dep, L.d_U,
                                                              L.Wg_hi, L.Wg_lo, L.bg);
          AMUN_CHECK_LAUNCH();
        });
        L.tc_maps_g = use_rows ? make_logit_rows_maps(L.db[0].T_hi, L.db[0].T_lo, Rmax, de, m0->dep, L.Wg_hi,
                                                      L.Wg_lo, m0->dep, n_gath)
                               : make_logit_maps(L.db[0].T_hi, L.db[0].T_lo, Rmax, de, m0->dep, L.Wg_hi, L.Wg_lo,
                                                 m0->dep, n_gath);
      } else {
        std::vector<uint32_t> mask((size_t)B * mask_words, 0u);
        for (int i = 0; i < B; ++i)
          for (int e = slo[i]; e < slo[i] + sll[i]; ++e) {
            const int v = slv[e];
            mask[(size_t)i * mask_words + v / 32] |= 1u << (v % 32);
          }
        h2d(c, L.d_vmask, mask.data(), mask.size());
      }
    }
    if (sl_ids) {
      h2d(c, L.d_sl, slv.data(), slv.size());
      h2d(c, L.d_sl_off, slo.data(), B);
      h2d(c, L.d_sl_len, sll.data(), B);
    }
    if (ahead) {  // annotations and initial states from this chunk's store
      std::vector<const float *> s0p(n_models);
      const int ci = chunk_of_bucket[bi], chunk_first = gchunk_first[ci];
      auto &stores = gstores[ci];
      for (int m = 0; m < n_models; ++m) {
        gencs[ci][m]->prepare(c, bk.first - chunk_first, B, bucket_row[bi], (long long)B * jmax, jmax);
        const int dh_m = ms[m]->d.d_h, da_m = ms[m]->d.d_att;
        L.eb[m].Hann = stores[m].Hann ? stores[m].Hann + bucket_row[bi] * 2 * dh_m : nullptr;
        L.eb[m].P = stores[m].P + bucket_row[bi] * da_m;
        L.eb[m].HX = stores[m].HX ? stores[m].HX + bucket_row[bi] * proj_ldhx(ms[m]) : nullptr;
        s0p[m] = stores[m].S0 + (long long)(bk.first - chunk_first) * dh_m;
      }
      h2d(c, L.p_S0, s0p.data(), n_models);
    } else {
      for (int m = 0; m < n_models; ++m)
        encode_bucket(c, ms[m], L.eb[m], L.d_ids, L.d_len, B, jmax, use_tce ? &L.tencs[m] : nullptr);
    }
    L.bs.B = B;
    L.bs.k = k;
    L.bs.cap_max = L.capm;
    L.bs.fin_cap = fin_cap;
    L.mr = ModelRows{L.p_XS, L.p_Sn, L.p_E, o.want_states ? L.p_fin : nullptr, n_models};
    for (int m = 0; m < n_models; ++m) {
      const amun_model *mm = ms[m];
      const int de_m = mm->d.d_emb, dh_m = mm->d.d_h;
      L.mr.dim[m] = RowDims{mm->xs_w, de_m, dh_m, de_m + 2 * dh_m, use_tcg ? mm->xsp : 0,
                            use_tcg ? mm->dep - de_m : 0, (use_tcg && L.eb[m].HX) ? 0 : 1};
    }
    if (use_tcg) {
      L.mr.XSh = L.p_XSh;
      L.mr.XSl = L.p_XSl;
    }
    c.run(AMUN_K_SELECT, [&] { launch_init_beam(L.bs, L.mr, L.p_S0, L.st); });
    L.lo = LogitOut{fused, kk, ceil_div(V, tile_n), L.pmax, L.psum, L.cval, L.ctok};
    L.lo.rows = use_rows;
    if (use_mask) {
      L.lo.vmask = L.d_vmask;
      L.lo.mask_words = mask_words;
    }
    if (use_tc) L.lo.tc = &L.tc_maps;
    if (n_gath) {
      L.lo.tc = &L.tc_maps_g;
      L.lo.vmask = L.d_vmask_g;
      L.lo.mask_words = ceil_div(n_gath, 32);
      L.lo.n_vocab = n_gath;
      L.lo.vid = L.d_U;
      L.lo.bias = L.bg;
      L.lo.ntiles = ceil_div(n_gath, tile_n);
    }
    // folded query (step_rows): the bucket's first Q / EQ / s U_zr from the
    // initial rows; every later step's come from the deep-output GEMM
    for (int m = 0; m < n_models; ++m)
      if (use_tcg && L.tsteps[m].proj && L.tsteps[m].dq_ok && L.eb[m].HX && L.lo.tc) {
        qs_prologue(c, ms[m], L.db[m], L.tsteps[m], L.R);
        L.mr.dim[m].split = 0;  // the step reads the gathered rows in fp32 only (attention, GRU-B)
      } else {
        L.mr.dim[m].split = 1;
      }
    SelectArgs &sa = L.sa;
    sa = SelectArgs{};
    sa.kk = kk;
    sa.fused = fused;
    sa.V = V;
    sa.pmax = L.pmax;
    sa.psum = L.psum;
    sa.cval = L.cval;
    sa.ctok = L.ctok;
    sa.ntiles = L.lo.ntiles;
    sa.M = L.R;
    sa.nm_fused = ens_fused ? n_models : 1;
    sa.pm_stride = (long long)Rmax * ntiles;
    sa.L = L.p_L;
    sa.ldl = V;
    sa.sl_ids = sl_ids ? L.d_sl : nullptr;
    sa.sl_off = L.d_sl_off;
    sa.sl_len = L.d_sl_len;
    sa.cand_lp = L.cand_lp;
    sa.cand_tok = L.cand_tok;
    sa.dbg = sel_dbg;
  };

  // Enqueue one decoder step.  Step 0 runs eagerly (it also sizes lazily
  // grown workspaces); step 1 is captured as a CUDA graph that every later
  // step replays (identical launches: select reads each sentence's own step
  // counter).  Every kProbeEvery steps an async copy of the done-count is
  // queued; the host never runs more than kMaxAhead steps past the newest
  // probe it has read, so a bucket whose sentences all stopped early ends
  // without decoding to the cap.
  auto enqueue_step = [&](Lane &L) {
    Ctx &c = *L.c;
    if (graphs_ok && L.capm > 2 && L.t == 1 && (!L.gexec || L.gstale)) {
      const int64_t before = c.launches;
      cudaGraph_t graph = nullptr;
      AMUN_CUDA(cudaStreamBeginCapture(L.st, cudaStreamCaptureModeThreadLocal));
      try {
        launch_step(L);
      } catch (...) {
        cudaStreamEndCapture(L.st, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      AMUN_CUDA(cudaStreamEndCapture(L.st, &graph));
      L.step_launches = c.launches - before;
      c.launches = before;
      // same topology as the previous bucket's graph (only kernel arguments
      // differ): update the executable graph instead of re-instantiating
      bool updated = false;
      if (L.gexec) {
        cudaGraphExecUpdateResultInfo info{};
        updated = cudaGraphExecUpdate(L.gexec, graph, &info) == cudaSuccess;
        if (!updated) {
          (void)cudaGetLastError();
          cudaGraphExecDestroy(L.gexec);
          L.gexec = nullptr;
        }
      }
      cudaError_t ie = updated ? cudaSuccess : cudaGraphInstantiate(&L.gexec, graph, 0);
      cudaGraphDestroy(graph);
      AMUN_CUDA(ie);
      L.gstale = false;
    }
    if (L.gexec && !L.gstale) {
      const auto tg0 = std::chrono::steady_clock::now();
      AMUN_CUDA(cudaGraphLaunch(L.gexec, L.st));
      host_launch_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - tg0).count();
      ++host_launch_n;
      c.launches += L.step_launches;
    } else {
      launch_step(L);
    }
    ++L.t;
    ++total_steps;
    if (L.t % kProbeEvery == 0 && L.t < L.capm) {
      const int slot = L.probe_next++ % kProbeSlots;
      d2h(c, L.h_probe + slot, L.bs.n_done, 1);
      AMUN_CUDA(cudaEventRecord(L.probe_ev[slot], L.st));
      L.pending.emplace_back(L.t, slot);
    }
  };

  // read probes; `block` waits for the oldest one
  auto poll = [&](Lane &L, bool block) {
    while (!L.pending.empty()) {
      auto [step, slot] = L.pending.front();
      if (block) {
        AMUN_CUDA(cudaEventSynchronize(L.probe_ev[slot]));
        block = false;
      } else if (cudaEventQuery(L.probe_ev[slot]) != cudaSuccess) {
        break;
      }
      L.pending.pop_front();
      if (L.h_probe[slot] >= L.B) L.stop = true;
    }
  };

  auto finish_bucket = [&](Lane &L) {
    if (dbg_sched) bucket_span[L.bucket].second = now_ms();
    Ctx &c = *L.c;
    const Bucket &bk = buckets[L.bucket];
    const int B = L.B, capm = L.capm, R = L.R;
    BeamState &bs = L.bs;
    std::vector<int> n_act(B), steps(B), fin_n(B), fin_t((size_t)B * fin_cap), fin_par((size_t)B * fin_cap);
    std::vector<int> bp_tok((size_t)B * capm * k), bp_par((size_t)B * capm * k);
    std::vector<double> score(R), fin_score((size_t)B * fin_cap);
    d2h(c, n_act.data(), bs.n_act, B);
    d2h(c, steps.data(), bs.steps, B);
    d2h(c, fin_n.data(), bs.fin_n, B);
    d2h(c, score.data(), bs.score, R);
    AMUN_CUDA(cudaStreamSynchronize(L.st));
    // finished lists: only the used prefix of every sentence's row
    const int fmax = *std::max_element(fin_n.begin(), fin_n.end());
    if (fmax > 0) {
      auto rows2d = [&](void *dst, const void *src, size_t esz) {
        AMUN_CUDA(cudaMemcpy2DAsync(dst, fin_cap * esz, src, fin_cap * esz, fmax * esz, B, cudaMemcpyDeviceToHost,
                                    L.st));
        c.d2h += (int64_t)(fmax * esz * B);
      };
      rows2d(fin_score.data(), bs.fin_score, sizeof(double));
      rows2d(fin_t.data(), bs.fin_t, sizeof(int));
      rows2d(fin_par.data(), bs.fin_par, sizeof(int));
    }
    d2h(c, bp_tok.data(), bs.bp_tok, (size_t)B * capm * k);
    d2h(c, bp_par.data(), bs.bp_par, (size_t)B * capm * k);
    // per member m: active rows [R][dh_m] and finished rows [B][fin_cap][dh_m]
    std::vector<std::vector<float>> act_states(n_models), fin_st(n_models);
    if (o.want_states) {
      for (int m = 0; m < n_models; ++m) {
        const int de_m = ms[m]->d.d_emb, dh_m = ms[m]->d.d_h;
        act_states[m].resize((size_t)R * dh_m);
        fin_st[m].resize((size_t)B * fin_cap * dh_m);
        AMUN_CUDA(cudaMemcpy2DAsync(act_states[m].data(), dh_m * sizeof(float), L.db[m].XS + de_m + 2 * dh_m,
                                    ms[m]->xs_w * sizeof(float), dh_m * sizeof(float), R, cudaMemcpyDeviceToHost,
                                    L.st));
        d2h(c, fin_st[m].data(), L.fin_states[m], (size_t)B * fin_cap * dh_m);
      }
    }
    AMUN_CUDA(cudaStreamSynchronize(L.st));
    c.collect();
    L.pending.clear();
    L.active = false;
    auto walk = [&](int i, int tt, int slot) {
      std::vector<int> seq;
      for (; tt >= 0; --tt) {
        size_t o2 = ((size_t)i * capm + tt) * k + slot;
        seq.push_back(bp_tok[o2]);
        slot = bp_par[o2];
      }
      std::reverse(seq.begin(), seq.end());
      return seq;
    };
    for (int i = 0; i < B; ++i) {
      const int s = order[bk.first + i];
      std::vector<HostHyp> hyps;
      if (fin_n[i] > 0) {
        for (int f = 0; f < fin_n[i]; ++f) {
          size_t fo = (size_t)i * fin_cap + f;
          HostHyp h{fin_score[fo], 1, walk(i, fin_t[fo] - 1, fin_par[fo]), {}};
          h.toks.push_back(0);
          if (o.want_states)
            for (int m = 0; m < n_models; ++m) {
              const int dh_m = ms[m]->d.d_h;
              const float *p = fin_st[m].data() + fo * dh_m;
              h.state.insert(h.state.end(), p, p + dh_m);
            }
          hyps.push_back(std::move(h));
        }
      } else {
        for (int a = 0; a < n_act[i]; ++a) {
          HostHyp h{score[(size_t)i * k + a], 0, walk(i, steps[i] - 1, a), {}};
          if (o.want_states)
            for (int m = 0; m < n_models; ++m) {
              const int dh_m = ms[m]->d.d_h;
              const float *p = act_states[m].data() + ((size_t)i * k + a) * dh_m;
              h.state.insert(h.state.end(), p, p + dh_m);
            }
          hyps.push_back(std::move(h));
        }
      }
      auto rank = [&](const HostHyp &h) {
        return (o.length_normalize && !h.toks.empty()) ? h.score / (double)h.toks.size() : h.score;
      };
      std::stable_sort(hyps.begin(), hyps.end(), [&](const HostHyp &a, const HostHyp &b) {
        double ra = rank(a), rb = rank(b);
        if (ra != rb) return ra > rb;
        return a.toks < b.toks;
      });
      if ((int)hyps.size() > o.n_best) hyps.resize(o.n_best);
      out_hyps[s] = std::move(hyps);
    }
    if (on_bucket) {  // stream this bucket's final hypotheses to the caller
      const int *sel = order.data() + bk.first;
      amun_result *part = flatten_hyps(out_hyps, sel, B, n_models, dh, state_w, o.want_states);
      on_bucket(user, part, sel);
      amun_result_free(part);
    }
  };

  // chunks of whole buckets: with encode-ahead, a chunk's encoder runs
  // before its buckets decode (bounded annotation-store memory,
  // AMUN_ENC_CHUNK sentences per chunk, decoded one after the other)
  std::vector<std::pair<int, int>> chunks;
  {
    const char *ce = getenv("AMUN_ENC_CHUNK");  // read per call (tests vary it)
    const int cap = ce ? std::max(1, atoi(ce)) : 16384;
    const int nb = (int)buckets.size();
    for (int b = 0; b < nb;) {
      int e = b, cnt = 0;
      while (e < nb && (e == b || !ahead || cnt + buckets[e].count <= cap)) cnt += buckets[e++].count;
      chunks.emplace_back(b, e);
      b = e;
    }
  }
  // groups of chunks in flight together.  A single chunk is split in two:
  // its longest buckets (AMUN_ENC_LEAD sentences, default 8 buckets' worth)
  // are encoded first, on their own -- a short recurrence over few rows --
  // so the longest bucket, which bounds the pass, starts decoding after a
  // few milliseconds instead of after the whole corpus's encoder; the
  // rest's encoder follows on the encoder streams while those decode
  std::vector<std::vector<std::pair<int, int>>> groups;
  {
    const char *le = getenv("AMUN_ENC_LEAD");
    const int lead = le ? std::max(0, atoi(le)) : 8 * Bmax_opt;
    if (ahead && chunks.size() == 1 && lead > 0) {
      const int nb = (int)buckets.size();
      int b = nb, cnt = 0;
      while (b > 1 && cnt < lead) cnt += buckets[--b].count;
      if (b > 0 && b < nb)
        groups.push_back({{b, nb}, {0, b}});
      else
        groups.push_back(chunks);
    } else {
      for (const auto &ch : chunks) groups.push_back({ch});
    }
  }
  for (const auto &group : groups) {
  gstores.assign(group.size(), std::vector<Store>());
  gencs.clear();
  gencs.resize(group.size());
  gchunk_first.assign(group.size(), 0);
  dispatch.clear();
  for (size_t ci = 0; ci < group.size(); ++ci) {
  const auto &ch = group[ci];
  for (int bi = ch.first; bi < ch.second; ++bi) chunk_of_bucket[bi] = (int)ci;
  if (ahead) {
    auto &stores = gstores[ci];
    auto &encs = gencs[ci];
    stores.assign(n_models, Store{});
    encs.resize(n_models);
    // store rows per bucket ([B][jmax] each), the chunk's sentences in
    // sorted order, then the encoder of every model
    const int chunk_first = buckets[ch.first].first;
    gchunk_first[ci] = chunk_first;
    long long rows = 0;
    for (int bi = ch.first; bi < ch.second; ++bi) {
      bucket_row[bi] = rows;
      rows += (long long)buckets[bi].count * buckets[bi].jmax;
    }
    const int nc = buckets[ch.second - 1].first + buckets[ch.second - 1].count - chunk_first;
    std::vector<int32_t> cids;
    std::vector<long long> coff(nc), carow(nc);
    std::vector<int32_t> clen(nc);
    for (int bi = ch.first; bi < ch.second; ++bi)
      for (int j = 0; j < buckets[bi].count; ++j) {
        const int i = buckets[bi].first + j - chunk_first, s = order[buckets[bi].first + j];
        coff[i] = (long long)cids.size();
        clen[i] = src_len[s];
        carow[i] = bucket_row[bi] + (long long)j * buckets[bi].jmax;
        cids.insert(cids.end(), src_ids + off[s], src_ids + off[s + 1]);
      }
    // encoder streams: chunk ci of the group runs its forward / backward
    // recurrences on lanes 2 ci and 2 ci + 1 (when there are enough lanes),
    // so the lead chunk's long serial recurrence and the bulk chunk's big
    // one run concurrently instead of one after the other
    const int e0 = std::min(2 * (int)ci, n_lanes - 1), e1 = std::min(2 * (int)ci + 1, n_lanes - 1);
    Ctx &cf = *lanes[e0]->c;
    Ctx &cb = *lanes[e1]->c;
    for (int m = 0; m < n_models; ++m) {
      const int dh_m = ms[m]->d.d_h, da_m = ms[m]->d.d_att;
      Store &S = stores[m];
      Carver cv;
      for (int pass = 0; pass < 2; ++pass) {
        cv = Carver{};
        cv.base = static_cast<char *>(S.mem);
        const bool proj_m = use_tcg && proj_ok(ms[m]);  // the step reads HX, never fp32 H
        S.Hann = proj_m ? nullptr : cv.take<float>((size_t)rows * 2 * dh_m);
        S.P = cv.take<float>((size_t)rows * da_m);
        S.S0 = cv.take<float>((size_t)nc * dh_m);
        S.Hah = cv.take<__half>((size_t)rows * 2 * dh_m);
        S.Hal = cv.take<__half>((size_t)rows * 2 * dh_m);
        S.HX = use_tcg && proj_ok(ms[m]) ? cv.take<float>((size_t)rows * proj_ldhx(ms[m])) : nullptr;
        if (!pass) AMUN_CUDA(cudaMallocFromPoolAsync(&S.mem, cv.off, ws_pool(m0->device), cf.st));
      }
      AheadIn in{nc, cids.data(), coff.data(), clen.data(), carow.data(), rows};
      encs[m].reset(
          new AheadEncoder(ms[m], in, AheadOut{S.Hann, S.P, S.S0, S.Hah, S.Hal, S.HX}, ws_pool(m0->device)));
      encs[m]->set_prep_ctas(enc_target_ctas());
      encs[m]->run(cf, cb);
    }
  }
  {
    const std::vector<int> d = lpt_order(ch.first, ch.second);
    dispatch.insert(dispatch.end(), d.begin(), d.end());
  }
  }  // chunks of the group
  next_bucket = 0;
  // the longest buckets go to the highest lanes: lanes 0 and 1 also carry
  // the encoder streams
  for (int li = n_lanes - 1; li >= 0; --li)
    if (next_bucket < dispatch.size()) start_bucket(*lanes[li], dispatch[next_bucket++]);
  for (;;) {
    bool any = false;
    for (auto &Lp : lanes) {
      Lane &L = *Lp;
      if (!L.active) continue;
      any = true;
      poll(L, false);
      if (L.stop || L.t >= L.capm) {
        finish_bucket(L);
        if (next_bucket < dispatch.size()) start_bucket(L, dispatch[next_bucket++]);
        continue;
      }
      // bounded run-ahead past the newest probe the host has seen
      if (!L.pending.empty() && L.t - L.pending.front().first >= kMaxAhead) {
        poll(L, true);
        if (L.stop) continue;
      }
      enqueue_step(L);
    }
    if (!any) break;
  }
  if (ahead)  // every lane finished (and synchronised) this group's buckets
    for (size_t ci = 0; ci < group.size(); ++ci)
      for (int m = 0; m < n_models; ++m) {
        gencs[ci][m]->release(*lanes[0]->c);
        gencs[ci][m].reset();
        AMUN_CUDA(cudaFreeAsync(gstores[ci][m].mem, lanes[0]->st));
        gstores[ci][m] = Store{};
      }
  }  // groups

  for (int li = 1; li < n_lanes; ++li) {
    AMUN_CUDA(cudaEventRecord(lanes[li]->probe_ev[0], lanes[li]->st));
    AMUN_CUDA(cudaStreamWaitEvent(lanes[0]->st, lanes[li]->probe_ev[0], 0));
  }
  AMUN_CUDA(cudaEventRecord(ev1, lanes[0]->st));
  AMUN_CUDA(cudaEventSynchronize(ev1));
  const auto t_ev1 = std::chrono::steady_clock::now();
  if (dbg_sched) {
    double t_end = 0;
    for (auto &sp : bucket_span) t_end = std::max(t_end, sp.second);
    fprintf(stderr, "sched: %zu buckets, last finish %.1f ms; active lanes per 10%% of the run:", buckets.size(), t_end);
    for (int d = 0; d < 10; ++d) {
      const double t = t_end * (d + 0.5) / 10;
      int act = 0;
      for (auto &sp : bucket_span) act += sp.first <= t && t < sp.second;
      fprintf(stderr, " %d", act);
    }
    int longest = 0;
    for (size_t i = 0; i < buckets.size(); ++i)
      if (bucket_span[i].second - bucket_span[i].first > bucket_span[longest].second - bucket_span[longest].first) longest = (int)i;
    fprintf(stderr, "; longest bucket %d: %d steps in %.1f ms (%.2f ms/step)\n", longest, buckets[longest].cap_max,
            bucket_span[longest].second - bucket_span[longest].first,
            (bucket_span[longest].second - bucket_span[longest].first) / std::max(1, buckets[longest].cap_max));
  }
  if (getenv("AMUN_DEBUG_HOST"))
    fprintf(stderr, "host: %lld graph launches, %.1f ms inside cudaGraphLaunch, decode loop %.1f ms\n", host_launch_n,
            host_launch_ns / 1e6, std::chrono::duration<double, std::milli>(t_ev1 - t_ev0).count());
  if (sel_dbg) {
    unsigned long long h[8];
    AMUN_CUDA(cudaMemcpy(h, sel_dbg, sizeof(h), cudaMemcpyDeviceToHost));
    const double n = (double)std::max(1ull, h[4]);
    fprintf(stderr, "select phases (cycles per CTA): rows %.0f | sentence top-k %.0f | update %.0f | gather %.0f (%llu CTAs)\n",
            h[0] / n, h[1] / n, h[2] / n, h[3] / n, h[4]);
    cudaFree(sel_dbg);
  }
  float ms_elapsed = 0.f;
  AMUN_CUDA(cudaEventElapsedTime(&ms_elapsed, ev0, ev1));
  Ctx c(nullptr);  // totals over lanes
  for (auto &Lp : lanes) {
    c.launches += Lp->c->launches;
    c.h2d += Lp->c->h2d;
    c.d2h += Lp->c->d2h;
    for (int i = 0; i < AMUN_K_CLASSES; ++i) {
      c.kms[i] += Lp->c->kms[i];
      c.kcount[i] += Lp->c->kcount[i];
      c.kctas[i] += Lp->c->kctas[i];
    }
  }

  // ---- assemble the flat result
  std::vector<int> all(n_sent);
  std::iota(all.begin(), all.end(), 0);
  amun_result *r = flatten_hyps(out_hyps, all.data(), n_sent, n_models, dh, state_w, o.want_states);
  r->decoder_steps = total_steps;
  r->kernel_launches = c.launches;
  r->device_ms = ms_elapsed;
  r->h2d_bytes = c.h2d;
  r->d2h_bytes = c.d2h;
  for (int i = 0; i < AMUN_K_CLASSES; ++i) {
    r->kernel_ms[i] = c.kms[i];
    r->kernel_count[i] = c.kcount[i];
    r->kernel_ctas[i] = c.kctas[i];
  }
  if (ktb.p) {  // CTA-time accounting replaces the (absent) event totals
    unsigned long long h[2 * AMUN_K_CLASSES];
    AMUN_CUDA(cudaMemcpy(h, ktb.p, sizeof(h), cudaMemcpyDeviceToHost));
    for (int i = 0; i < AMUN_K_CLASSES; ++i) {
      r->kernel_ms[i] = (double)h[2 * i] * 1e-6;
      r->kernel_ctas[i] = (int64_t)h[2 * i + 1];
    }
  }
  using ms_d = std::chrono::duration<double, std::milli>;
  r->host_setup_ms = ms_d(t_ev0 - t_enter).count();
  lanes.clear();  // lane teardown (back to the pool) counts as host post-processing
  r->host_post_ms = ms_d(std::chrono::steady_clock::now() - t_ev1).count();
  return r;
}

// Frees the pooled lanes of a device (streams, workspaces, step graphs,
// pinned probe rings) and trims its workspace pool: called when the last
// model handle on the device is destroyed, so a long-running process does
// not keep its peak decode memory after the models are gone.
void release_device_lanes(int dev) {
  std::vector<LaneRes *> rs;
  cudaMemPool_t pool = nullptr;
  {
    std::lock_guard<std::mutex> g(g_lane_mu);
    for (auto &v : g_lane_pool[dev & 63]) {
      rs.insert(rs.end(), v.begin(), v.end());
      v.clear();
    }
    pool = g_ws_pool[dev & 63];
  }
  for (LaneRes *r : rs) {
    cudaStreamSynchronize(r->st);
    if (r->mem) cudaFreeAsync(r->mem, r->st);
    if (r->ws) cudaFreeAsync(r->ws, r->st);
    cudaStreamSynchronize(r->st);
    if (r->gexec) cudaGraphExecDestroy(r->gexec);
    for (auto e : r->ev) cudaEventDestroy(e);
    if (r->h_probe) cudaFreeHost(r->h_probe);
    cudaStreamDestroy(r->st);
    delete r;
  }
  if (pool) cudaMemPoolTrimTo(pool, 0);
}

// ====================================================================== hooks

void hook_encode(amun_model *m, const int32_t *ids, int J, float *h_out, float *p_out, float *s0_out) {
  AMUN_CUDA(cudaSetDevice(m->device));
  Ctx c(m->stream);
  EncBufs e{};
  int *d_ids, *d_len;
  DevMem mem;
  for (int pass = 0; pass < 2; ++pass) {
    Carver cv;
    cv.base = pass ? static_cast<char *>(mem.p) : nullptr;
    carve_enc(cv, e, m, 1, J);
    d_ids = cv.take<int>(J);
    d_len = cv.take<int>(1);
    if (!pass) mem.alloc(cv.off, c.st);
  }
  h2d(c, d_ids, ids, J);
  h2d(c, d_len, &J, 1);
  encode_bucket(c, m, e, d_ids, d_len, 1, J);
  const int dh = m->d.d_h, da = m->d.d_att;
  if (h_out) d2h(c, h_out, e.Hann, (size_t)J * 2 * dh);
  if (p_out) d2h(c, p_out, e.P, (size_t)J * da);
  if (s0_out) d2h(c, s0_out, e.S0, dh);
  AMUN_CUDA(cudaStreamSynchronize(c.st));
}

void hook_step(amun_model *m, const float *s, const int32_t *y_prev, int R, const float *h, const float *p, int J,
               const int32_t *sl, int n_sl, float *s_out, double *logp_out, float *alpha_out, float *ctx_out) {
  AMUN_CUDA(cudaSetDevice(m->device));
  Ctx c(m->stream);
  const int de = m->d.d_emb, dh = m->d.d_h, da = m->d.d_att, V = m->d.v_trg, xs = m->xs_w;
  EncBufs e{};
  DecBufs d{};
  int *d_len, *d_y, *d_sl;
  float *d_s, *d_alpha;
  double *d_logp;
  const int n_out = sl ? n_sl : V;
  DevMem mem;
  for (int pass = 0; pass < 2; ++pass) {
    Carver cv;
    cv.base = pass ? static_cast<char *>(mem.p) : nullptr;
    e.Hann = cv.take<float>((size_t)J * 2 * dh);
    e.P = cv.take<float>((size_t)J * da);
    carve_dec(cv, d, m, R, J, true);
    d_len = cv.take<int>(1);
    d_y = cv.take<int>(R);
    d_sl = cv.take<int>(std::max(n_sl, 1));
    d_s = cv.take<float>((size_t)R * dh);
    d_alpha = cv.take<float>((size_t)R * J);
    d_logp = cv.take<double>((size_t)R * n_out);
    if (!pass) mem.alloc(cv.off, c.st);
  }
  h2d(c, e.Hann, h, (size_t)J * 2 * dh);
  h2d(c, e.P, p, (size_t)J * da);
  h2d(c, d_len, &J, 1);
  h2d(c, d_s, s, (size_t)R * dh);
  if (y_prev) h2d(c, d_y, y_prev, R);
  if (sl) h2d(c, d_sl, sl, n_sl);
  AMUN_CUDA(cudaMemsetAsync(d.XS, 0, sizeof(float) * (size_t)R * xs, c.st));
  build_rows_kernel<<<R, 256, 0, c.st>>>(d.XS, xs, m->E_trg, y_prev ? d_y : nullptr, d_s, de, dh, de + 2 * dh);
  AMUN_CHECK_LAUNCH();
  if (!y_prev) {  // attention only (nnet.py:132-141)
    EpiStore eq{d.Q, da, nullptr, 0, 0};
    eq.ex2 = d.EQ;
    gemm(c, ga(R, da, d.XS + de + 2 * dh, xs, dh, m->W_att_s, da), eq);
    AttnArgs aa{d.Q, da, e.P, e.Hann, m->v_att, d_len, J, da, 2 * dh, R, nullptr, nullptr, d.XS + de, xs, d_alpha};
    aa.energy = d.En;
    aa.EQ = d.EQ;
    launch_attention(aa, R, c.st);
  } else {
    LogitOut lo{false, 0, 0, nullptr, nullptr, nullptr, nullptr};
    step_rows(c, m, d, e, d_len, J, R, R, nullptr, nullptr, d_alpha, lo);
    launch_logp_rows(d.L, V, R, V, sl ? d_sl : nullptr, n_sl, d_logp, c.st);
  }
  if (alpha_out) d2h(c, alpha_out, d_alpha, (size_t)R * J);
  if (ctx_out)
    AMUN_CUDA(cudaMemcpy2DAsync(ctx_out, 2 * dh * sizeof(float), d.XS + de, xs * sizeof(float),
                                2 * dh * sizeof(float), R, cudaMemcpyDeviceToHost, c.st));
  if (s_out) d2h(c, s_out, d.Sn, (size_t)R * dh);
  if (logp_out && y_prev) d2h(c, logp_out, d_logp, (size_t)R * n_out);
  AMUN_CUDA(cudaStreamSynchronize(c.st));
}

// fp16 split of the y and s parts of decoder rows in the padded layout
// [y | pad | c | s] (what select's next-row gather writes in production)
__global__ void build_rows_split_kernel(__half *XSh, __half *XSl, int ldh, const float *E, const int *y,
                                        const float *s, int de, int dh, int s_off_h) {
  const int r = blockIdx.x;
  const long long ro = (long long)r * ldh;
  for (int c = threadIdx.x; c < de; c += blockDim.x) store_split(XSh, XSl, ro + c, E[(long long)y[r] * de + c]);
  for (int c = threadIdx.x; c < dh; c += blockDim.x)
    store_split(XSh, XSl, ro + s_off_h + c, s[(long long)r * dh + c]);
}

// Production-kernel step hook: B sentences x k hypothesis rows through
// exactly the kernels amun_decode runs per step (tcgen05 query / GRU-A /
// GRU-B / deep-output GEMMs, fused attention writing the context split, and
// the fused tensor-core logit kernel), returning the logit kernel's raw
// per-(row, 128-vocab tile) partials: (max, sum exp) and the tile's top-kk
// (value, token).  nnet.py:143-164 + tensor.py:79-92 + search.py:169.
void hook_step_tc(amun_model *m, int B, int k, const float *s, const int32_t *y_prev, const float *h,
                  const float *p, const int32_t *lens, int jmax, int kk, float *s_out, float *pmax_out,
                  float *psum_out, float *cval_out, int32_t *ctok_out, float *alpha_out) {
  if (!m->tc_gemm || !m->Wl_hi)
    throw Error(AMUN_ERR_UNSUPPORTED, "model dimensions / embedding range are outside the tensor-core path");
  if (kk < 1 || kk > kMaxRowCand) throw Error(AMUN_ERR_UNSUPPORTED, "kk must be in [1, 16]");
  AMUN_CUDA(cudaSetDevice(m->device));
  Ctx c(m->stream);
  const int de = m->d.d_emb, dh = m->d.d_h, da = m->d.d_att, V = m->d.v_trg, xs = m->xs_w;
  const int R = B * k, ntiles = ceil_div(V, kBN);
  EncBufs e{};
  DecBufs d{};
  int *d_len, *d_y, *ctok, *d_qrow;
  float *d_s, *d_alpha, *pmax, *psum, *cval;
  DevMem mem;
  for (int pass = 0; pass < 2; ++pass) {
    Carver cv;
    cv.base = pass ? static_cast<char *>(mem.p) : nullptr;
    e.Hann = cv.take<float>((size_t)B * jmax * 2 * dh);
    e.P = cv.take<float>((size_t)B * jmax * da);
    d_qrow = cv.take<int>(R);
    if (proj_ok(m)) {  // the product's projected annotations, from the given h
      e.HX = cv.take<float>((size_t)B * jmax * proj_ldhx(m));
      e.Hah = cv.take<__half>((size_t)B * jmax * 2 * dh);
      e.Hal = cv.take<__half>((size_t)B * jmax * 2 * dh);
    }
    carve_dec(cv, d, m, R, jmax, false);
    carve_dec_tc(cv, d, m, R);
    d_len = cv.take<int>(B);
    d_y = cv.take<int>(R);
    d_s = cv.take<float>((size_t)R * dh);
    d_alpha = cv.take<float>((size_t)R * jmax);
    pmax = cv.take<float>((size_t)R * ntiles);
    psum = cv.take<float>((size_t)R * ntiles);
    cval = cv.take<float>((size_t)R * ntiles * kk);
    ctok = cv.take<int>((size_t)R * ntiles * kk);
    if (!pass) mem.alloc(cv.off, c.st);
  }
  h2d(c, e.Hann, h, (size_t)B * jmax * 2 * dh);
  h2d(c, e.P, p, (size_t)B * jmax * da);
  h2d(c, d_len, lens, B);
  h2d(c, d_s, s, (size_t)R * dh);
  h2d(c, d_y, y_prev, R);
  {
    std::vector<int> ident(R);
    std::iota(ident.begin(), ident.end(), 0);
    h2d(c, d_qrow, ident.data(), R);
  }
  if (e.HX) {
    const long long n = (long long)B * jmax * 2 * dh;
    split_rows_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, c.st>>>(e.Hann, n, e.Hah, e.Hal);
    AMUN_CHECK_LAUNCH();
    compute_hx(c, m, e.Hah, e.Hal, (long long)B * jmax, 0, B * jmax, e.HX, 148);
  }
  AMUN_CUDA(cudaMemsetAsync(d.XS, 0, sizeof(float) * (size_t)R * xs, c.st));
  AMUN_CUDA(cudaMemsetAsync(d.XSh, 0, sizeof(__half) * (size_t)R * m->xsp, c.st));
  AMUN_CUDA(cudaMemsetAsync(d.XSl, 0, sizeof(__half) * (size_t)R * m->xsp, c.st));
  build_rows_kernel<<<R, 256, 0, c.st>>>(d.XS, xs, m->E_trg, d_y, d_s, de, dh, de + 2 * dh);
  AMUN_CHECK_LAUNCH();
  build_rows_split_kernel<<<R, 256, 0, c.st>>>(d.XSh, d.XSl, m->xsp, m->E_trg, d_y, d_s, de, dh, m->dep + 2 * dh);
  AMUN_CHECK_LAUNCH();
  TcStep ts;
  tc_step_maps(m, d, R, ts);
  // the product's logit kernel for this beam (decode_run: rows layout for
  // beams >= 8, swap-AB below); the outputs keep the [R][ceil(V / 128)]
  // layout, tiles the kernel does not produce padded as empty partials
  const char *rows_env = getenv("AMUN_LOGIT_ROWS");
  const bool rows = rows_env ? rows_env[0] == '1' : k >= 8;
  const int nt_dev = ceil_div(V, rows ? kLogitRowsTileN : kBN);
  const LogitTcMaps lm = rows ? make_logit_rows_maps(d.T_hi, d.T_lo, R, de, m->dep, m->Wl_hi, m->Wl_lo, m->dep, V)
                              : make_logit_maps(d.T_hi, d.T_lo, R, de, m->dep, m->Wl_hi, m->Wl_lo, m->dep, V);
  LogitOut lo{true, kk, nt_dev, pmax, psum, cval, ctok};
  lo.tc = &lm;
  lo.rows = rows;
  // exactly a bucket's first step in amun_decode: the folded query's
  // prologue, then the step (whose deep-output GEMM also computes the next
  // query, unused here)
  if (ts.proj && ts.dq_ok && e.HX) qs_prologue(c, m, d, ts, R);
  step_rows(c, m, d, e, d_len, jmax, R, k, nullptr, nullptr, d_alpha, lo, &ts, true, d_y, d_qrow);
  std::vector<float> hpm((size_t)R * nt_dev), hps((size_t)R * nt_dev), hcv((size_t)R * nt_dev * kk);
  std::vector<int> hct((size_t)R * nt_dev * kk);
  if (s_out) d2h(c, s_out, d.Sn, (size_t)R * dh);
  d2h(c, hpm.data(), pmax, hpm.size());
  d2h(c, hps.data(), psum, hps.size());
  d2h(c, hcv.data(), cval, hcv.size());
  d2h(c, hct.data(), ctok, hct.size());
  if (alpha_out) d2h(c, alpha_out, d_alpha, (size_t)R * jmax);
  AMUN_CUDA(cudaStreamSynchronize(c.st));
  for (int r = 0; r < R; ++r)
    for (int t = 0; t < ntiles; ++t) {
      const bool have = t < nt_dev;
      const size_t o = (size_t)r * ntiles + t, od = (size_t)r * nt_dev + t;
      if (pmax_out) pmax_out[o] = have ? hpm[od] : -INFINITY;
      if (psum_out) psum_out[o] = have ? hps[od] : 0.f;
      for (int i = 0; i < kk; ++i) {
        if (cval_out) cval_out[o * kk + i] = have ? hcv[od * kk + i] : -INFINITY;
        if (ctok_out) ctok_out[o * kk + i] = have ? hct[od * kk + i] : -1;
      }
    }
}

// Batched encoder hook: B padded sentences (ids [B][jmax], lens[B]) through
// encode_bucket, on the production tensor-core kernels (input projection,
// bi-GRU recurrence, precomp_att) when `production`, else on the FP32
// CUDA-core kernels.  h_out [B][jmax][2 d_h] (zero past each length),
// p_out [B][jmax][d_att], s0_out [B][d_h].
void hook_encode_batch(amun_model *m, const int32_t *ids, const int32_t *lens, int B, int jmax, bool production,
                       float *h_out, float *p_out, float *s0_out) {
  if (production && !m->Efa_hi[0])
    throw Error(AMUN_ERR_UNSUPPORTED, "model dimensions / embedding range are outside the tensor-core path");
  AMUN_CUDA(cudaSetDevice(m->device));
  Ctx c(m->stream);
  EncBufs e{};
  int *d_ids, *d_len;
  DevMem mem;
  for (int pass = 0; pass < 2; ++pass) {
    Carver cv;
    cv.base = pass ? static_cast<char *>(mem.p) : nullptr;
    carve_enc(cv, e, m, B, jmax);
    if (production) carve_enc_tc(cv, e, m, B, jmax);
    d_ids = cv.take<int>((size_t)B * jmax);
    d_len = cv.take<int>(B);
    if (!pass) mem.alloc(cv.off, c.st);
  }
  if (production) {
    // the product path: encode-ahead over the B sentences (store = [B][jmax])
    c.ws_pool = ws_pool(m->device);
    std::vector<long long> off(B), arow(B);
    for (int b = 0; b < B; ++b) off[b] = arow[b] = (long long)b * jmax;
    AheadIn in{B, ids, off.data(), lens, arow.data(), (long long)B * jmax};
    AheadEncoder enc(m, in, AheadOut{e.Hann, e.P, e.S0, e.Hah, e.Hal}, ws_pool(m->device));
    enc.run(c, c);
    enc.prepare(c, 0, B, 0, (long long)B * jmax, *std::max_element(lens, lens + B));
    enc.release(c);
  } else {
    h2d(c, d_ids, ids, (size_t)B * jmax);
    h2d(c, d_len, lens, B);
    encode_bucket(c, m, e, d_ids, d_len, B, jmax, nullptr);
  }
  const int dh = m->d.d_h, da = m->d.d_att;
  if (h_out) d2h(c, h_out, e.Hann, (size_t)B * jmax * 2 * dh);
  if (p_out) d2h(c, p_out, e.P, (size_t)B * jmax * da);
  if (s0_out) d2h(c, s0_out, e.S0, (size_t)B * dh);
  AMUN_CUDA(cudaStreamSynchronize(c.st));
}

}  // namespace amun

namespace amun {

void hook_init_state(amun_model *m, const float *h, int J, float *s0_out) {
  AMUN_CUDA(cudaSetDevice(m->device));
  Ctx c(m->stream);
  const int dh = m->d.d_h;
  float *d_h, *d_mean, *d_s0;
  int *d_len;
  DevMem mem;
  for (int pass = 0; pass < 2; ++pass) {
    Carver cv;
    cv.base = pass ? static_cast<char *>(mem.p) : nullptr;
    d_h = cv.take<float>((size_t)J * 2 * dh);
    d_mean = cv.take<float>(2 * dh);
    d_s0 = cv.take<float>(dh);
    d_len = cv.take<int>(1);
    if (!pass) mem.alloc(cv.off, c.st);
  }
  h2d(c, d_h, h, (size_t)J * 2 * dh);
  h2d(c, d_len, &J, 1);
  launch_masked_mean(d_h, d_len, 1, J, 2 * dh, d_mean, c.st);
  gemm(c, ga(1, dh, d_mean, 2 * dh, 2 * dh, m->W_init, dh), EpiStore{d_s0, dh, m->b_init, 1, 0});
  d2h(c, s0_out, d_s0, dh);
  AMUN_CUDA(cudaStreamSynchronize(c.st));
}

// Standalone GRU cell (nnet.py:177-185): same phase A / phase B kernels as
// the decoder, with rows [x | h] and fused weights [[W_z W_r W_h];[U_z U_r 0]].
void hook_gru_cell(int device, int d_in, int dh, const float *const *W, const float *const *U,
                   const float *const *b, int R, const float *x, const float *h, float *h_out) {
  AMUN_CUDA(cudaSetDevice(device));
  cudaStream_t st;
  AMUN_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  } sg{st};
  Ctx c(st);
  const int w = d_in + dh;
  std::vector<float> Wg((size_t)w * 3 * dh, 0.f), bg(3 * dh), rows((size_t)R * w);
  for (int g = 0; g < 3; ++g) {
    for (int i = 0; i < d_in; ++i)
      std::memcpy(&Wg[(size_t)i * 3 * dh + g * dh], W[g] + (size_t)i * dh, dh * sizeof(float));
    if (g < 2)
      for (int i = 0; i < dh; ++i)
        std::memcpy(&Wg[(size_t)(d_in + i) * 3 * dh + g * dh], U[g] + (size_t)i * dh, dh * sizeof(float));
    std::memcpy(&bg[g * dh], b[g], dh * sizeof(float));
  }
  for (int r = 0; r < R; ++r) {
    std::memcpy(&rows[(size_t)r * w], x + (size_t)r * d_in, d_in * sizeof(float));
    std::memcpy(&rows[(size_t)r * w + d_in], h + (size_t)r * dh, dh * sizeof(float));
  }
  float *d_W, *d_b, *d_Uh, *d_rows, *d_Z, *d_RH, *d_XH, *d_out;
  DevMem mem;
  for (int pass = 0; pass < 2; ++pass) {
    Carver cv;
    cv.base = pass ? static_cast<char *>(mem.p) : nullptr;
    d_W = cv.take<float>(Wg.size());
    d_b = cv.take<float>(bg.size());
    d_Uh = cv.take<float>((size_t)dh * dh);
    d_rows = cv.take<float>(rows.size());
    d_Z = cv.take<float>((size_t)R * dh);
    d_RH = cv.take<float>((size_t)R * dh);
    d_XH = cv.take<float>((size_t)R * dh);
    d_out = cv.take<float>((size_t)R * dh);
    if (!pass) mem.alloc(cv.off, st);
  }
  h2d(c, d_W, Wg.data(), Wg.size());
  h2d(c, d_b, bg.data(), bg.size());
  h2d(c, d_Uh, U[2], (size_t)dh * dh);
  h2d(c, d_rows, rows.data(), rows.size());
  GemmArgs g = ga(R, 3 * dh, d_rows, w, w, d_W, 3 * dh);
  g.n_split = 2 * dh;
  g.k_limit = d_in;
  gemm(c, g, EpiGruA{d_b, d_rows + d_in, w, dh, d_Z, d_RH, d_XH});
  gemm(c, ga(R, dh, d_RH, dh, dh, d_Uh, dh), EpiGruB{d_rows + d_in, w, dh, d_Z, d_XH, d_out});
  d2h(c, h_out, d_out, (size_t)R * dh);
  AMUN_CUDA(cudaStreamSynchronize(st));
}

}  // namespace amun

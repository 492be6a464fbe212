// C-ABI of the B200 decoder (include/amun_b200.h): device model handle,
// length-bucketed batched beam-search decode, and the per-step parity hooks.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/amun_b200.h"
#include "common.cuh"
#include "decode.cuh"
#include "gemm_simt.cuh"
#include "kernels.cuh"

using namespace amun;

static thread_local std::string g_last_error;
// shared with the other C-ABI translation units (text.cu)
void amun_set_last_error(const std::string &m) { g_last_error = m; }
// live model handles per device: the pooled decode lanes of a device are
// released when its last handle is destroyed
static std::atomic<int> g_live_models[64];

#define AMUN_API_BEGIN try {
#define AMUN_API_END                                  \
  }                                                   \
  catch (const ::amun::Error &e) {                    \
    g_last_error = e.what();                          \
    return e.code;                                    \
  }                                                   \
  catch (const std::exception &e) {                   \
    g_last_error = e.what();                          \
    return AMUN_ERR_CUDA;                             \
  }                                                   \
  return AMUN_OK;

static void invalid(const std::string &m) { throw Error(AMUN_ERR_INVALID, m); }

extern "C" const char *amun_last_error(void) { return g_last_error.c_str(); }
extern "C" int amun_version(void) { return 1; }

extern "C" int amun_device_count(int32_t *n) {
  AMUN_API_BEGIN
  int c = 0;
  AMUN_CUDA(cudaGetDeviceCount(&c));
  *n = c;
  AMUN_API_END
}

// ------------------------------------------------------------------ model

namespace {

// schema order (model.py:94-117)
enum {
  T_E_SRC = 0, T_E_TRG = 1,
  T_ENC_FWD = 2, T_ENC_BWD = 11, T_DEC = 20,  // + {W_z W_r W_h U_z U_r U_h b_z b_r b_h}
  T_W_INIT = 29, T_B_INIT, T_W_ATT_S, T_W_ATT_H, T_V_ATT, T_W_OUT_S, T_W_OUT_Y, T_W_OUT_C, T_B_OUT,
  T_W_LOGIT, T_B_LOGIT, T_COUNT
};
enum { G_WZ = 0, G_WR, G_WH, G_UZ, G_UR, G_UH, G_BZ, G_BR, G_BH };

}  // namespace

static float *upload(amun_model *m, const std::vector<float> &h);

template <class T>
static T *upload_t(amun_model *m, const std::vector<T> &h) {
  T *d = nullptr;
  AMUN_CUDA(cudaMalloc(&d, h.size() * sizeof(T)));
  m->allocs.push_back(d);
  AMUN_CUDA(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  m->bytes += (int64_t)(h.size() * sizeof(T));
  return d;
}

// max |W| over n floats (non-negative float bits order like unsigned ints)
__global__ void absmax_kernel(const float *__restrict__ W, size_t n, unsigned *out) {
  float m = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    m = fmaxf(m, fabsf(W[i]));
  for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, __float_as_uint(m));
}

// W [K, N] row-major (device) -> hi/lo [N, Kp] K-major through 32 x 32
// shared-memory tiles (coalesced on both sides); source row k lands in
// column k < split ? k : k + pad
__global__ void kmajor_split_kernel(const float *__restrict__ W, int K, int N, int Kp, int split, int pad, float sc,
                                    __half *__restrict__ hi, __half *__restrict__ lo) {
  __shared__ float tile[32][33];
  const int n0 = blockIdx.x * 32, k0 = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int k = k0 + j, n = n0 + threadIdx.x;
    tile[j][threadIdx.x] = (k < K && n < N) ? W[(size_t)k * N + n] : 0.f;
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int n = n0 + j, k = k0 + threadIdx.x;
    if (n < N && k < K) {
      const float x = tile[threadIdx.x][j] * sc;
      const __half h = __float2half_rn(x);
      const size_t o = (size_t)n * Kp + (k < split ? k : k + pad);
      hi[o] = h;
      lo[o] = __float2half_rn(x - __half2float(h));
    }
  }
}

static float device_absmax(const float *d, size_t n);

// C[M, N] = A[M, K] B[K, N] in fp32 (row-major, pitches lda / ldb / N), 64 x 64
// tiles through shared memory, 4 x 4 outputs per thread: the per-token
// embedding tables E_trg W^y built once at model load
__global__ void table_gemm_kernel(const float *__restrict__ A, int lda, const float *__restrict__ B, int ldb, int M,
                                  int N, int K, const float *__restrict__ bias, float *__restrict__ C) {
  __shared__ float As[16][64 + 1], Bs[16][64];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int r = i / 16, kk = i % 16;
      As[kk][r] = (m0 + r < M && k0 + kk < K) ? A[(long long)(m0 + r) * lda + k0 + kk] : 0.f;
      const int kb = i / 64, c = i % 64;
      Bs[kb][c] = (k0 + kb < K && n0 + c < N) ? B[(long long)(k0 + kb) * ldb + n0 + c] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk)
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(As[kk][ty * 4 + i], Bs[kk][tx * 4 + j], acc[i][j]);
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty * 4 + i, n = n0 + tx * 4 + j;
      if (m < M && n < N) C[(long long)m * N + n] = bias ? acc[i][j] + bias[n] : acc[i][j];
    }
}

static float *device_table(amun_model *m, const float *A, int lda, const float *B, int ldb, int M, int N, int K,
                           const float *bias = nullptr) {
  float *d = nullptr;
  AMUN_CUDA(cudaMalloc(&d, (size_t)M * N * sizeof(float)));
  m->allocs.push_back(d);
  m->bytes += (int64_t)((size_t)M * N * sizeof(float));
  table_gemm_kernel<<<dim3(ceil_div(N, 64), ceil_div(M, 64)), 256>>>(A, lda, B, ldb, M, N, K, bias, d);
  AMUN_CHECK_LAUNCH();
  return d;
}

// [K, N] row-major DEVICE matrix -> device [N, Kp] (K-major, row pitch Kp)
// 3xFP16 hi/lo copies for the tensor-core GEMMs (common.cuh split_h), built
// on the device from the fp32 copy: the matrix is scaled by 2^sw with
// max|W| 2^sw < 2^14 (fp16 max 65504, and lo stays normal for |W| >=
// 2^-17 max|W|), hi = fp16(W'), lo = fp16(W' - hi).  Source row k lands in
// column k < split ? k : k + pad (the padded decoder-row layout); unused
// columns are zero.  Returns the epilogue's inverse scale 2^-(sw + kXShift).
static float split_kmajor_dev(amun_model *m, const float *dW, int K, int N, int Kp, int split, int pad,
                              __half **hi_out, __half **lo_out) {
  const size_t n = (size_t)N * Kp;
  __half *hi = nullptr, *lo = nullptr;
  AMUN_CUDA(cudaMalloc(&hi, n * sizeof(__half)));
  m->allocs.push_back(hi);
  AMUN_CUDA(cudaMalloc(&lo, n * sizeof(__half)));
  m->allocs.push_back(lo);
  m->bytes += (int64_t)(2 * n * sizeof(__half));
  AMUN_CUDA(cudaMemset(hi, 0, n * sizeof(__half)));
  AMUN_CUDA(cudaMemset(lo, 0, n * sizeof(__half)));
  const float mx = device_absmax(dW, (size_t)K * N);
  int e = 0;
  if (mx > 0.f) std::frexp(mx, &e);  // mx < 2^e
  const int sw = mx > 0.f ? 14 - e : 0;
  kmajor_split_kernel<<<dim3(ceil_div(N, 32), ceil_div(K, 32)), dim3(32, 8)>>>(dW, K, N, Kp, split, pad,
                                                                              std::ldexp(1.f, sw), hi, lo);
  AMUN_CHECK_LAUNCH();
  *hi_out = hi;
  *lo_out = lo;
  return std::ldexp(1.f, -(sw + kXShift));
}

// as split_kmajor_dev for a host matrix needed only in its split form
static float split_kmajor_host(amun_model *m, const float *W, int K, int N, int Kp, int split, int pad,
                               __half **hi_out, __half **lo_out) {
  float *d = nullptr;
  AMUN_CUDA(cudaMalloc(&d, (size_t)K * N * sizeof(float)));
  struct Free {
    float *p;
    ~Free() { cudaFree(p); }
  } f{d};
  AMUN_CUDA(cudaMemcpy(d, W, (size_t)K * N * sizeof(float), cudaMemcpyHostToDevice));
  const float us = split_kmajor_dev(m, d, K, N, Kp, split, pad, hi_out, lo_out);
  AMUN_CUDA(cudaDeviceSynchronize());
  return us;
}

static float *upload(amun_model *m, const std::vector<float> &h) { return upload_t(m, h); }

// n floats straight from the caller's (read-only) array: no host staging copy
static float *upload_ptr(amun_model *m, const float *h, size_t n) {
  float *d = nullptr;
  AMUN_CUDA(cudaMalloc(&d, n * sizeof(float)));
  m->allocs.push_back(d);
  AMUN_CUDA(cudaMemcpy(d, h, n * sizeof(float), cudaMemcpyHostToDevice));
  m->bytes += (int64_t)(n * sizeof(float));
  return d;
}

// max |x| of a device array (absmax_kernel), synchronous
static float device_absmax(const float *d, size_t n) {
  unsigned *dmax = nullptr, hmax = 0;
  AMUN_CUDA(cudaMalloc(&dmax, sizeof(unsigned)));
  AMUN_CUDA(cudaMemset(dmax, 0, sizeof(unsigned)));
  absmax_kernel<<<296, 256>>>(d, n, dmax);
  AMUN_CHECK_LAUNCH();
  AMUN_CUDA(cudaMemcpy(&hmax, dmax, sizeof(unsigned), cudaMemcpyDeviceToHost));
  cudaFree(dmax);
  float mx;
  std::memcpy(&mx, &hmax, sizeof(float));
  return mx;
}

extern "C" int amun_model_create(int32_t device, const amun_dims *dims, const float *const *t,
                                 int32_t n_tensors, amun_model **out) {
  amun_model *m = nullptr;
  AMUN_API_BEGIN
  if (!dims || !t || !out) invalid("null argument");
  if (n_tensors != T_COUNT) invalid("expected 40 tensors in schema order, got " + std::to_string(n_tensors));
  if (dims->d_emb < 1 || dims->d_h < 1 || dims->d_att < 1 || dims->v_src < 2 || dims->v_trg < 2)
    invalid("invalid model dimensions");
  for (int i = 0; i < T_COUNT; ++i)
    if (!t[i]) invalid("null tensor pointer " + std::to_string(i));
  int ndev = 0;
  AMUN_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) invalid("device " + std::to_string(device) + " out of range");
  AMUN_CUDA(cudaSetDevice(device));
  m = new amun_model();
  m->device = device;
  m->d = *dims;
  const int de = dims->d_emb, dh = dims->d_h, da = dims->d_att, V = dims->v_trg, Vs = dims->v_src;
  const int din = de + 2 * dh;  // decoder GRU input [y ; c]
  m->xs_w = de + 3 * dh;
  m->dep = (de + 7) / 8 * 8;
  m->xsp = m->dep + 3 * dh;
  // decoder-row column -> padded fp16 row column ([y | pad | c | s])
  const int pad = m->dep - de;
  auto cp = [&](int idx, size_t n) { return upload_ptr(m, t[idx], n); };
  m->E_src = cp(T_E_SRC, (size_t)Vs * de);
  m->E_trg = cp(T_E_TRG, (size_t)V * de);
  {  // tensor-core path: 16-byte fp16 row pitches and activations inside the
     // split's range (decoder rows |x| <= max(1, max|E_trg|) <= 2^(15 - kXShift);
     // encoder states and annotations are GRU outputs in (-1, 1))
    const float emax = std::max(device_absmax(m->E_trg, (size_t)V * de), device_absmax(m->E_src, (size_t)Vs * de));
    m->tc_ok = (de % 4 == 0) && (dh % 8 == 0) && (da % 8 == 0) && emax <= std::ldexp(1.f, 15 - kXShift);
  }

  {  // encoder input projection, both directions: [de, 6dh] = [fwd z r h | bwd z r h]
    std::vector<float> W((size_t)de * 6 * dh), b(6 * dh);
    for (int dir = 0; dir < 2; ++dir) {
      int base = dir ? T_ENC_BWD : T_ENC_FWD;
      for (int g = 0; g < 3; ++g) {
        const float *src = t[base + G_WZ + g];
        for (int i = 0; i < de; ++i)
          std::memcpy(&W[(size_t)i * 6 * dh + (dir * 3 + g) * dh], src + (size_t)i * dh, dh * sizeof(float));
        std::memcpy(&b[(dir * 3 + g) * dh], t[base + G_BZ + g], dh * sizeof(float));
      }
    }
    m->Wenc = upload(m, W);
    m->benc = upload(m, b);
    if (m->tc_ok) m->us_x = split_kmajor_dev(m, m->Wenc, de, 6 * dh, m->dep, de, 0, &m->Wenc_hi, &m->Wenc_lo);
    // per-source-token input projections E_src W + b (fp32, [Vs, 6dh]):
    // the encode-ahead recurrence then runs its GEMMs over the state only
    if (m->tc_ok) m->XWenc = device_table(m, m->E_src, de, m->Wenc, 6 * dh, Vs, 6 * dh, de, m->benc);
  }
  {  // encoder recurrent weights: Uzr [2][dh][2dh], Uh [2][dh][dh]
    std::vector<float> Uzr((size_t)2 * dh * 2 * dh), Uh((size_t)2 * dh * dh);
    for (int dir = 0; dir < 2; ++dir) {
      int base = dir ? T_ENC_BWD : T_ENC_FWD;
      for (int i = 0; i < dh; ++i) {
        std::memcpy(&Uzr[((size_t)dir * dh + i) * 2 * dh], t[base + G_UZ] + (size_t)i * dh, dh * sizeof(float));
        std::memcpy(&Uzr[((size_t)dir * dh + i) * 2 * dh + dh], t[base + G_UR] + (size_t)i * dh, dh * sizeof(float));
      }
      std::memcpy(&Uh[(size_t)dir * dh * dh], t[base + G_UH], (size_t)dh * dh * sizeof(float));
    }
    m->Uzr = upload(m, Uzr);
    m->Uh = upload(m, Uh);
    if (m->tc_ok) {  // both directions stacked along K: [2dh, 2dh] and [2dh, dh]
      m->us_ea = split_kmajor_dev(m, m->Uzr, 2 * dh, 2 * dh, 2 * dh, 2 * dh, 0, &m->Uzr_hi, &m->Uzr_lo);
      m->us_eb = split_kmajor_dev(m, m->Uh, 2 * dh, dh, 2 * dh, 2 * dh, 0, &m->Uh_hi, &m->Uh_lo);
    }
  }
  if (m->tc_ok) {  // encode-ahead recurrence weights: [x | state] rows (x padded to dep)
    for (int dir = 0; dir < 2; ++dir) {
      const int base = dir ? T_ENC_BWD : T_ENC_FWD;
      std::vector<float> A((size_t)(de + dh) * 2 * dh), Bm((size_t)(de + dh) * dh);
      for (int i = 0; i < de; ++i) {
        std::memcpy(&A[(size_t)i * 2 * dh], t[base + G_WZ] + (size_t)i * dh, dh * sizeof(float));
        std::memcpy(&A[(size_t)i * 2 * dh + dh], t[base + G_WR] + (size_t)i * dh, dh * sizeof(float));
        std::memcpy(&Bm[(size_t)i * dh], t[base + G_WH] + (size_t)i * dh, dh * sizeof(float));
      }
      for (int i = 0; i < dh; ++i) {
        std::memcpy(&A[(size_t)(de + i) * 2 * dh], t[base + G_UZ] + (size_t)i * dh, dh * sizeof(float));
        std::memcpy(&A[(size_t)(de + i) * 2 * dh + dh], t[base + G_UR] + (size_t)i * dh, dh * sizeof(float));
        std::memcpy(&Bm[(size_t)(de + i) * dh], t[base + G_UH] + (size_t)i * dh, dh * sizeof(float));
      }
      m->us_efa[dir] = split_kmajor_host(m, A.data(), de + dh, 2 * dh, m->dep + dh, de, pad, &m->Efa_hi[dir],
                                         &m->Efa_lo[dir]);
      m->us_efb[dir] = split_kmajor_host(m, Bm.data(), de + dh, dh, m->dep + dh, de, pad, &m->Efb_hi[dir],
                                         &m->Efb_lo[dir]);
    }
  }
  m->W_att_h = cp(T_W_ATT_H, (size_t)2 * dh * da);
  if (m->tc_ok)
    m->us_p = split_kmajor_dev(m, m->W_att_h, 2 * dh, da, 2 * dh, 2 * dh, 0, &m->Watth_hi, &m->Watth_lo);
  if (m->tc_ok) {  // [W_att_h | C_z | C_r | C_h | W_o^c | 0]: precomp_att + HX in one GEMM
    const int nph = da + 3 * dh + m->dep, din = de + 2 * dh;
    std::vector<float> Wph((size_t)2 * dh * nph, 0.f);
    for (int i = 0; i < 2 * dh; ++i) {
      float *row = &Wph[(size_t)i * nph];
      std::memcpy(row, t[T_W_ATT_H] + (size_t)i * da, da * sizeof(float));
      for (int g = 0; g < 3; ++g)  // the context rows (de + i) of the decoder's input weights
        std::memcpy(row + da + g * dh, t[T_DEC + G_WZ + g] + (size_t)(de + i) * dh, dh * sizeof(float));
      std::memcpy(row + da + 3 * dh, t[T_W_OUT_C] + (size_t)i * de, de * sizeof(float));
    }
    (void)din;
    float *dWph = nullptr;
    AMUN_CUDA(cudaMalloc(&dWph, Wph.size() * sizeof(float)));
    AMUN_CUDA(cudaMemcpy(dWph, Wph.data(), Wph.size() * sizeof(float), cudaMemcpyHostToDevice));
    m->us_ph = split_kmajor_dev(m, dWph, 2 * dh, nph, 2 * dh, 2 * dh, 0, &m->Wph_hi, &m->Wph_lo);
    AMUN_CUDA(cudaDeviceSynchronize());
    AMUN_CUDA(cudaFree(dWph));
  }
  m->W_init = cp(T_W_INIT, (size_t)2 * dh * dh);
  m->b_init = cp(T_B_INIT, dh);
  m->W_att_s = cp(T_W_ATT_S, (size_t)dh * da);
  m->v_att = cp(T_V_ATT, da);
  {  // decoder gates: rows [y ; c ; s] (= XS columns), cols [z | r | h];
     // the h block of the s rows is zero (reset-before-matmul: s enters h~
     // only through (r*s) U_h, applied in phase B).
    std::vector<float> Wg((size_t)(din + dh) * 3 * dh, 0.f), bg(3 * dh);
    for (int g = 0; g < 3; ++g) {
      const float *W = t[T_DEC + G_WZ + g];
      for (int i = 0; i < din; ++i)
        std::memcpy(&Wg[(size_t)i * 3 * dh + g * dh], W + (size_t)i * dh, dh * sizeof(float));
      if (g < 2) {
        const float *U = t[T_DEC + G_UZ + g];
        for (int i = 0; i < dh; ++i)
          std::memcpy(&Wg[(size_t)(din + i) * 3 * dh + g * dh], U + (size_t)i * dh, dh * sizeof(float));
      }
      std::memcpy(&bg[g * dh], t[T_DEC + G_BZ + g], dh * sizeof(float));
    }
    m->Wg = upload(m, Wg);
    m->bg = upload(m, bg);
    m->Uh_dec = cp(T_DEC + G_UH, (size_t)dh * dh);
    m->tc_gemm = m->tc_ok;
    if (m->tc_gemm) {
      m->us_g = split_kmajor_dev(m, m->Wg, din + dh, 3 * dh, m->xsp, de, pad, &m->Wg_hi, &m->Wg_lo);
      m->us_u = split_kmajor_dev(m, m->Uh_dec, dh, dh, dh, dh, 0, &m->Uhd_hi, &m->Uhd_lo);
      m->us_q = split_kmajor_dev(m, m->W_att_s, dh, da, dh, dh, 0, &m->Wq_hi, &m->Wq_lo);
      std::vector<float> Wqs((size_t)dh * (da + 2 * dh));
      for (int i = 0; i < dh; ++i) {
        std::memcpy(&Wqs[(size_t)i * (da + 2 * dh)], t[T_W_ATT_S] + (size_t)i * da, da * sizeof(float));
        for (int g = 0; g < 2; ++g)
          std::memcpy(&Wqs[(size_t)i * (da + 2 * dh) + da + g * dh], t[T_DEC + G_UZ + g] + (size_t)i * dh,
                      dh * sizeof(float));
      }
      float *dWqs = nullptr;
      AMUN_CUDA(cudaMalloc(&dWqs, Wqs.size() * sizeof(float)));
      AMUN_CUDA(cudaMemcpy(dWqs, Wqs.data(), Wqs.size() * sizeof(float), cudaMemcpyHostToDevice));
      m->us_qs = split_kmajor_dev(m, dWqs, dh, da + 2 * dh, dh, dh, 0, &m->Wqs_hi, &m->Wqs_lo);
      AMUN_CUDA(cudaDeviceSynchronize());
      AMUN_CUDA(cudaFree(dWqs));
      {  // [W_o^s | 0 | W_att_s | U_z | U_r]: deep output + next query in one GEMM
        const int nq = m->dep + da + 2 * dh;
        std::vector<float> Wdq((size_t)dh * nq, 0.f);
        for (int i = 0; i < dh; ++i) {
          std::memcpy(&Wdq[(size_t)i * nq], t[T_W_OUT_S] + (size_t)i * de, de * sizeof(float));
          std::memcpy(&Wdq[(size_t)i * nq + m->dep], &Wqs[(size_t)i * (da + 2 * dh)], (da + 2 * dh) * sizeof(float));
        }
        float *dWdq = nullptr;
        AMUN_CUDA(cudaMalloc(&dWdq, Wdq.size() * sizeof(float)));
        AMUN_CUDA(cudaMemcpy(dWdq, Wdq.data(), Wdq.size() * sizeof(float), cudaMemcpyHostToDevice));
        m->us_dq = split_kmajor_dev(m, dWdq, dh, nq, dh, dh, 0, &m->Wdq_hi, &m->Wdq_lo);
        AMUN_CUDA(cudaDeviceSynchronize());
        AMUN_CUDA(cudaFree(dWdq));
      }
    }
  }
  {  // deep output: rows [y ; c ; s'] = [W_out_y ; W_out_c ; W_out_s]
    std::vector<float> Wo((size_t)(de + 3 * dh) * de);
    std::memcpy(&Wo[0], t[T_W_OUT_Y], (size_t)de * de * sizeof(float));
    std::memcpy(&Wo[(size_t)de * de], t[T_W_OUT_C], (size_t)2 * dh * de * sizeof(float));
    std::memcpy(&Wo[(size_t)(de + 2 * dh) * de], t[T_W_OUT_S], (size_t)dh * de * sizeof(float));
    m->Wout = upload(m, Wo);
    m->b_out = cp(T_B_OUT, de);
    if (m->tc_gemm) m->us_o = split_kmajor_dev(m, m->Wout, de + 3 * dh, de, m->xsp, de, pad, &m->Wo_hi, &m->Wo_lo);
  }
  if (m->tc_gemm) {  // y = E_trg[previous token]: its products with the y weight rows, per token
    m->YWg = device_table(m, m->E_trg, de, m->Wg, 3 * dh, V, 3 * dh, de);
    m->YWo = device_table(m, m->E_trg, de, m->Wout, de, V, de, de);
  }
  m->W_logit = cp(T_W_LOGIT, (size_t)de * V);
  m->b_logit = cp(T_B_LOGIT, V);
  if (m->tc_ok)  // logit rows [V, dep] (K-major, padded to a 16-byte pitch)
    m->us_l = split_kmajor_dev(m, m->W_logit, de, V, m->dep, de, 0, &m->Wl_hi, &m->Wl_lo);
  AMUN_CUDA(cudaDeviceSynchronize());  // every layout kernel done before the handle is used
  AMUN_CUDA(cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking));
  m->live = true;
  g_live_models[m->device & 63].fetch_add(1);
  *out = m;
  m = nullptr;
  }
  catch (const ::amun::Error &e) {
    g_last_error = e.what();
    if (m) amun_model_destroy(m);
    return e.code;
  }
  catch (const std::exception &e) {
    g_last_error = e.what();
    if (m) amun_model_destroy(m);
    return AMUN_ERR_CUDA;
  }
  return AMUN_OK;
}

extern "C" int amun_model_destroy(amun_model *m) {
  if (!m) return AMUN_OK;
  cudaSetDevice(m->device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  for (void *p : m->allocs) cudaFree(p);
  if (m->stream) cudaStreamDestroy(m->stream);
  if (m->live && g_live_models[m->device & 63].fetch_sub(1) == 1) {
    try {
      release_device_lanes(m->device);
    } catch (...) {
    }
  }
  delete m;
  return AMUN_OK;
}

extern "C" int amun_model_device_bytes(const amun_model *m, int64_t *bytes) {
  AMUN_API_BEGIN
  if (!m || !bytes) invalid("null argument");
  *bytes = m->bytes;
  AMUN_API_END
}

// ------------------------------------------------------------------ decode

extern "C" int amun_decode(amun_model *const *models, int32_t n_models, const int32_t *src_ids,
                           const int32_t *src_len, int32_t n_sent, const int32_t *sl_ids,
                           const int32_t *sl_len, const amun_decode_opts *opts, amun_result **out) {
  AMUN_API_BEGIN
  if (!models || n_models < 1) invalid("at least one model is required");
  if (!opts || !out || (n_sent > 0 && (!src_ids || !src_len))) invalid("null argument");
  *out = nullptr;
  std::vector<amun_model *> ms(models, models + n_models);
  for (auto *m : ms) {
    if (!m) invalid("null model handle");
    if (m->device != ms[0]->device) invalid("ensemble members must live on the same device");
    if (m->d.v_src != ms[0]->d.v_src || m->d.v_trg != ms[0]->d.v_trg)
      invalid("model vocabulary mismatch");
  }
  *out = decode_run(ms, src_ids, src_len, n_sent, sl_ids, sl_len, *opts);
  AMUN_API_END
}

extern "C" int amun_decode_stream(amun_model *const *models, int32_t n_models, const int32_t *src_ids,
                                  const int32_t *src_len, int32_t n_sent, const int32_t *sl_ids,
                                  const int32_t *sl_len, const amun_decode_opts *opts,
                                  amun_bucket_done_fn on_bucket, void *user, amun_result **out) {
  AMUN_API_BEGIN
  if (!models || n_models < 1) invalid("at least one model is required");
  if (!opts || !out || (n_sent > 0 && (!src_ids || !src_len))) invalid("null argument");
  *out = nullptr;
  std::vector<amun_model *> ms(models, models + n_models);
  for (auto *m : ms) {
    if (!m) invalid("null model handle");
    if (m->device != ms[0]->device) invalid("ensemble members must live on the same device");
    if (m->d.v_src != ms[0]->d.v_src || m->d.v_trg != ms[0]->d.v_trg)
      invalid("model vocabulary mismatch");
  }
  *out = decode_run(ms, src_ids, src_len, n_sent, sl_ids, sl_len, *opts, on_bucket, user);
  AMUN_API_END
}

extern "C" int amun_result_free(amun_result *r) {
  if (!r) return AMUN_OK;
  free(r->hyp_offsets);
  free(r->scores);
  free(r->finished);
  free(r->tok_offsets);
  free(r->tokens);
  free(r->states);
  free(r);
  return AMUN_OK;
}

// ------------------------------------------------------------------ hooks

extern "C" int amun_encode(amun_model *m, const int32_t *ids, int32_t J, float *h_out, float *p_out,
                           float *s0_out) {
  AMUN_API_BEGIN
  if (!m || !ids) invalid("null argument");
  if (J < 1) invalid("cannot encode an empty source sentence");
  for (int j = 0; j < J; ++j)
    if (ids[j] < 0 || ids[j] >= m->d.v_src)
      invalid("source id " + std::to_string(ids[j]) + " at position " + std::to_string(j) +
              " out of range for v_src=" + std::to_string(m->d.v_src));
  hook_encode(m, ids, J, h_out, p_out, s0_out);
  AMUN_API_END
}

extern "C" int amun_attention(amun_model *m, const float *s, int32_t R, const float *h, const float *p,
                              int32_t J, float *alpha_out, float *ctx_out) {
  AMUN_API_BEGIN
  if (!m || !s || !h || !p) invalid("null argument");
  if (R < 1 || J < 1) invalid("attention needs at least one state row and one source position");
  hook_step(m, s, nullptr, R, h, p, J, nullptr, 0, nullptr, nullptr, alpha_out, ctx_out);
  AMUN_API_END
}

extern "C" int amun_decoder_step(amun_model *m, const float *s, const int32_t *y_prev, int32_t R,
                                 const float *h, const float *p, int32_t J, const int32_t *sl, int32_t n_sl,
                                 float *s_out, double *logp_out, float *alpha_out) {
  AMUN_API_BEGIN
  if (!m || !s || !y_prev || !h || !p) invalid("null argument");
  if (R < 1 || J < 1) invalid("decoder step needs at least one state row and one source position");
  for (int r = 0; r < R; ++r)
    if (y_prev[r] < 0 || y_prev[r] >= m->d.v_trg)
      invalid("previous token id " + std::to_string(y_prev[r]) + " out of range for v_trg=" +
              std::to_string(m->d.v_trg));
  if (sl) {
    if (n_sl < 1) invalid("shortlist must be non-empty");
    for (int i = 0; i < n_sl; ++i)
      if (sl[i] < 0 || sl[i] >= m->d.v_trg)
        invalid("shortlist id " + std::to_string(sl[i]) + " out of range for v_trg=" + std::to_string(m->d.v_trg));
  }
  hook_step(m, s, y_prev, R, h, p, J, sl, n_sl, s_out, logp_out, alpha_out, nullptr);
  AMUN_API_END
}

extern "C" int amun_init_state(amun_model *m, const float *h, int32_t J, float *s0_out) {
  AMUN_API_BEGIN
  if (!m || !h || !s0_out) invalid("null argument");
  if (J < 1) invalid("annotations must have at least one source position");
  hook_init_state(m, h, J, s0_out);
  AMUN_API_END
}

extern "C" int amun_gru_cell(int32_t device, int32_t d_in, int32_t d_h, const float *const *W,
                             const float *const *U, const float *const *b, int32_t R, const float *x,
                             const float *h, float *h_out) {
  AMUN_API_BEGIN
  if (!W || !U || !b || !x || !h || !h_out) invalid("null argument");
  for (int i = 0; i < 3; ++i)
    if (!W[i] || !U[i] || !b[i]) invalid("null weight pointer");
  if (d_in < 1 || d_h < 1 || R < 1) invalid("invalid GRU cell dimensions");
  hook_gru_cell(device, d_in, d_h, W, U, b, R, x, h, h_out);
  AMUN_API_END
}

extern "C" int amun_encode_batch(amun_model *m, const int32_t *ids, const int32_t *lens, int32_t B, int32_t jmax,
                                 int32_t production, float *h_out, float *p_out, float *s0_out) {
  AMUN_API_BEGIN
  if (!m || !ids || !lens) invalid("null argument");
  if (B < 1 || jmax < 1) invalid("encode needs at least one sentence and one position");
  for (int b = 0; b < B; ++b) {
    if (lens[b] < 1) invalid("cannot encode an empty source sentence");
    if (lens[b] > jmax) invalid("sentence length exceeds jmax");
    for (int j = 0; j < lens[b]; ++j) {
      const int32_t v = ids[(size_t)b * jmax + j];
      if (v < 0 || v >= m->d.v_src)
        invalid("source id " + std::to_string(v) + " at position " + std::to_string(j) +
                " out of range for v_src=" + std::to_string(m->d.v_src));
    }
  }
  // positions past a sentence's length are never read as ids of real
  // tokens, but the gather still indexes them: pass a sanitised copy
  std::vector<int32_t> safe(ids, ids + (size_t)B * jmax);
  for (int b = 0; b < B; ++b)
    for (int j = lens[b]; j < jmax; ++j) safe[(size_t)b * jmax + j] = 0;
  hook_encode_batch(m, safe.data(), lens, B, jmax, production != 0, h_out, p_out, s0_out);
  AMUN_API_END
}

extern "C" int amun_decoder_step_fused(amun_model *m, int32_t B, int32_t k, const float *s, const int32_t *y_prev,
                                       const float *h, const float *p, const int32_t *lens, int32_t jmax,
                                       int32_t kk, float *s_out, float *pmax_out, float *psum_out,
                                       float *cval_out, int32_t *ctok_out, float *alpha_out) {
  AMUN_API_BEGIN
  if (!m || !s || !y_prev || !h || !p || !lens) invalid("null argument");
  if (B < 1 || k < 1 || jmax < 1) invalid("decoder step needs at least one state row and one source position");
  for (int b = 0; b < B; ++b)
    if (lens[b] < 1 || lens[b] > jmax) invalid("source lengths must lie in [1, jmax]");
  for (int r = 0; r < B * k; ++r)
    if (y_prev[r] < 0 || y_prev[r] >= m->d.v_trg)
      invalid("previous token id " + std::to_string(y_prev[r]) + " out of range for v_trg=" +
              std::to_string(m->d.v_trg));
  hook_step_tc(m, B, k, s, y_prev, h, p, lens, jmax, kk, s_out, pmax_out, psum_out, cval_out, ctok_out, alpha_out);
  AMUN_API_END
}

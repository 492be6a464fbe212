// Microbenchmark of the decoder-step tensor-core GEMM (gemm_sk.cuh; not part
// of the product): the GRU phase-A / query / GRU phase-B / deep-output shapes
// at several split counts, L2 flushed before every launch, with the
// attribution knobs (debug: 1 skip weight loads, 2 skip activation loads,
// 4 skip MMA, 8 skip reduction + epilogue).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lcuda \
//     tools/bench_sk.cu paper_1610_01108_b200/csrc/logits_tc.cu -o build/bench_sk
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1610_01108_b200/csrc/gemm_simt.cuh"
#include "../paper_1610_01108_b200/csrc/gemm_sk.cuh"

using namespace amun;

struct Shape {
  const char *name;
  int N, k1, k2;
  bool grub;  // GRU phase-B epilogue instead of a plain store
};

static unsigned g_seed = 1;
static __half *dev_rand_h(size_t n) {
  std::vector<__half> h(n);
  srand(g_seed++);
  for (auto &x : h) x = __float2half_rn((rand() / (float)RAND_MAX - 0.5f) * 100.f);
  __half *d;
  cudaMalloc(&d, n * sizeof(__half));
  cudaMemcpy(d, h.data(), n * sizeof(__half), cudaMemcpyHostToDevice);
  return d;
}
static float *dev_zero(size_t n) {
  float *d;
  cudaMalloc(&d, n * sizeof(float));
  cudaMemset(d, 0, n * sizeof(float));
  return d;
}

template <class C>
void run(const char *cname, const Shape &sh, int R, float *flush, size_t flush_n, int debug) {
  const int K = sh.k1 + sh.k2;
  g_seed = 1;
  __half *xh = dev_rand_h((size_t)R * sh.k1), *xl = dev_rand_h((size_t)R * sh.k1);
  __half *x2h = sh.k2 ? dev_rand_h((size_t)R * sh.k2) : nullptr, *x2l = sh.k2 ? dev_rand_h((size_t)R * sh.k2) : nullptr;
  __half *wh = dev_rand_h((size_t)sh.N * K), *wl = dev_rand_h((size_t)sh.N * K);
  float *out = dev_zero((size_t)R * sh.N), *S = dev_zero((size_t)R * sh.N), *Z = dev_zero((size_t)R * sh.N),
        *XH = dev_zero((size_t)R * sh.N);
  __half *oh, *ol;
  cudaMalloc(&oh, sizeof(__half) * R * sh.N);
  cudaMalloc(&ol, sizeof(__half) * R * sh.N);
  SkMaps maps = make_sk_maps<C>(xh, xl, sh.k1, sh.k1, x2h, x2l, sh.k2, sh.k2, R, wh, wl, sh.N, K, 1.f / 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nt = ceil_div(sh.N, 128 * C::kCG) * C::kCG;
  for (int S_ : {1, 2, 3, 4, 6, 8}) {
    const int splits = sk_splits<C>(maps, S_ * nt);
    if (splits != S_) continue;
    if (C::kCG * splits > 16) continue;
    EpiStore epi{out, sh.N, nullptr, 0, 0};
    EpiGruB eb{S, sh.N, sh.N, Z, XH, out};
    eb.Snh = oh;
    eb.Snl = ol;
    auto launch = [&] {
      if (sh.grub)
        launch_gemm_sk<C>(maps, R, splits, eb, 0, debug);
      else
        launch_gemm_sk<C>(maps, R, splits, epi, 0, debug);
    };
    float tot = 0.f, warm = 0.f;
    const int it = 10;
    for (int i = 0; i < it + 2; ++i) {
      cudaMemsetAsync(flush, i, flush_n * sizeof(float));
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (i >= 2) tot += ms;
    }
    cudaEventRecord(e0);
    for (int i = 0; i < it; ++i) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&warm, e0, e1);
    cudaError_t err = cudaGetLastError();
    const double flops = 3.0 * 2.0 * R * (double)K * sh.N;
    const double wbytes = 4.0 * K * sh.N;
    const double us = 1000.0 * tot / it;
    printf("%-8s %-14s R=%d S=%d ctas=%3d dbg=%2d  cold %7.1f us (%5.0f TF/s issued f16, W %5.0f GB/s)  "
           "warm %7.1f us  %s\n",
           sh.name, cname, R, splits, splits * nt, debug, us, flops / us * 1e-6, wbytes / us * 1e-3,
           1000.0 * warm / it, cudaGetErrorString(err));
  }
  cudaFree(xh);
  cudaFree(xl);
  if (x2h) {
    cudaFree(x2h);
    cudaFree(x2l);
  }
  cudaFree(wh);
  cudaFree(wl);
  cudaFree(out);
  cudaFree(S);
  cudaFree(Z);
  cudaFree(XH);
  cudaFree(oh);
  cudaFree(ol);
}

int main(int argc, char **argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 320;
  const int debug = argc > 2 ? atoi(argv[2]) : 0;
  const size_t flush_n = 256u << 20 >> 2;
  float *flush;
  cudaMalloc(&flush, flush_n * sizeof(float));
  Shape shapes[] = {{"gru_a", 3072, 3576, 0, false},
                    {"query", 1024, 1024, 0, false},
                    {"gru_b", 1024, 1024, 0, true},
                    {"deep_out", 500, 2552, 1024, false}};
  for (auto &sh : shapes) run<SkDefault>("bk64 st3 cg2", sh, R, flush, flush_n, debug);
  return 0;
}

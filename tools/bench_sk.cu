// Microbenchmark of the decoder-step tensor-core GEMM (gemm_sk.cuh; not part
// of the product): sweeps tile configurations and split counts on the GRU
// phase-A / query / deep-output shapes, L2 flushed before every launch.
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
};

static unsigned g_seed = 1;
static float *dev_rand(size_t n) {
  std::vector<float> h(n);
  srand(g_seed++);
  for (auto &x : h) x = (rand() / (float)RAND_MAX - 0.5f) * 0.2f;
  float *d;
  cudaMalloc(&d, n * sizeof(float));
  cudaMemcpy(d, h.data(), n * sizeof(float), cudaMemcpyHostToDevice);
  return d;
}

static std::vector<float> g_ref;

template <class C>
void run(const char *cname, const Shape &sh, int R, float *flush, size_t flush_n, int debug) {
  const int K = sh.k1 + sh.k2;
  g_seed = 1;
  float *xh = dev_rand((size_t)R * sh.k1), *xl = dev_rand((size_t)R * sh.k1);
  float *x2h = sh.k2 ? dev_rand((size_t)R * sh.k2) : nullptr, *x2l = sh.k2 ? dev_rand((size_t)R * sh.k2) : nullptr;
  float *wh = dev_rand((size_t)sh.N * K), *wl = dev_rand((size_t)sh.N * K);
  float *out;
  cudaMalloc(&out, sizeof(float) * R * sh.N);
  SkMaps maps = make_sk_maps<C>(xh, xl, sh.k1, sh.k1, x2h, x2l, sh.k2, sh.k2, R, wh, wl, sh.N, K);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nt = ceil_div(sh.N, 128 * C::kCG) * C::kCG;
  for (int S : {1, 2, 3, 4, 5, 6, 8}) {
    const int splits = sk_splits<C>(maps, S * nt);
    if (splits != S) continue;
    if (C::kCG * splits > 16) continue;
    const int maxc = sk_max_active_clusters<C, EpiStore>(splits);
    EpiStore epi{out, sh.N, nullptr, 0, 0};
    float tot = 0.f, warm = 0.f;
    const int it = 10;
    for (int i = 0; i < it + 2; ++i) {
      cudaMemsetAsync(flush, i, flush_n * sizeof(float));
      cudaEventRecord(e0);
      launch_gemm_sk<C>(maps, R, splits, epi, 0, debug);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (i >= 2) tot += ms;
    }
    cudaEventRecord(e0);
    for (int i = 0; i < it; ++i) launch_gemm_sk<C>(maps, R, splits, epi, 0, debug);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&warm, e0, e1);
    cudaError_t err = cudaGetLastError();
    std::vector<float> got((size_t)R * sh.N);
    cudaMemcpy(got.data(), out, got.size() * sizeof(float), cudaMemcpyDeviceToHost);
    if (g_ref.empty()) g_ref = got;
    double md = 0;
    for (size_t i = 0; i < got.size(); ++i) md = std::max(md, (double)std::fabs(got[i] - g_ref[i]));
    const double flops = 3.0 * 2.0 * R * (double)K * sh.N;
    const double wbytes = 8.0 * K * sh.N;
    const double us = 1000.0 * tot / it;
    printf("%-8s %-14s R=%d S=%d ctas=%3d maxclusters=%3d dbg=%d  cold %7.1f us (%5.0f TF/s 3xTF32, W %5.0f GB/s)  "
           "warm %7.1f us  maxdiff %.2e %s\n",
           sh.name, cname, R, splits, splits * nt, maxc, debug, us, flops / us * 1e-6, wbytes / us * 1e-3,
           1000.0 * warm / it, md, cudaGetErrorString(err));
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
}

int main(int argc, char **argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 320;
  const int debug = argc > 2 ? atoi(argv[2]) : 0;
  const size_t flush_n = 256u << 20 >> 2;
  float *flush;
  cudaMalloc(&flush, flush_n * sizeof(float));
  Shape shapes[] = {{"gru_a", 3072, 3572, 0}, {"query", 1024, 1024, 0}, {"deep_out", 500, 2548, 1024}};
  for (auto &sh : shapes) {
    g_ref.clear();
    run<SkCfg<32, 2, 320, 1>>("bk32 st2 cg1", sh, R, flush, flush_n, debug);
    run<SkCfg<32, 3, 320, 2>>("bk32 st3 cg2", sh, R, flush, flush_n, debug);
    run<SkCfg<16, 5, 320, 2>>("bk16 st5 cg2", sh, R, flush, flush_n, debug);
  }
  return 0;
}

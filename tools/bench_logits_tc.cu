// Microbenchmark of the tensor-core logit kernel (not part of the product):
// times launch variants with pieces disabled to attribute the step time.
//   nvcc ... tools/bench_logits_tc.cu paper_1610_01108_b200/csrc/logits_tc.cu -o build/bench_logits_tc
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1610_01108_b200/csrc/common.cuh"
#include "../paper_1610_01108_b200/csrc/logits_tc.cuh"

using namespace amun;

int main(int argc, char **argv) {
  const int R = argc > 1 ? atoi(argv[1]) : 320, K = 500, V = 30000;
  const int kk = argc > 3 ? atoi(argv[3]) : 5;
  const bool rows = argc > 2 && argv[2][0] == 'r';  // rows-layout kernel (logits_rows.cu)
  const int ntiles = (V + 127) / 128;
  const int Kp = (K + 7) / 8 * 8;
  std::vector<__half> h((size_t)std::max(R, V) * Kp);
  for (auto &x : h) x = __float2half_rn((rand() / (float)RAND_MAX - 0.5f) * 100.f);
  __half *thi, *tlo, *whi, *wlo;
  float *bias, *pmax, *psum, *cval;
  int *ctok;
  cudaMalloc(&thi, sizeof(__half) * R * Kp);
  cudaMalloc(&tlo, sizeof(__half) * R * Kp);
  cudaMalloc(&whi, sizeof(__half) * (size_t)V * Kp);
  cudaMalloc(&wlo, sizeof(__half) * (size_t)V * Kp);
  cudaMalloc(&bias, sizeof(float) * V);
  cudaMalloc(&pmax, sizeof(float) * ntiles * R);
  cudaMalloc(&psum, sizeof(float) * ntiles * R);
  cudaMalloc(&cval, sizeof(float) * ntiles * R * kk);
  cudaMalloc(&ctok, sizeof(int) * ntiles * R * kk);
  cudaMemcpy(thi, h.data(), sizeof(__half) * R * Kp, cudaMemcpyHostToDevice);
  cudaMemcpy(tlo, h.data(), sizeof(__half) * R * Kp, cudaMemcpyHostToDevice);
  cudaMemcpy(whi, h.data(), sizeof(__half) * (size_t)V * Kp, cudaMemcpyHostToDevice);
  cudaMemcpy(wlo, h.data(), sizeof(__half) * (size_t)V * Kp, cudaMemcpyHostToDevice);
  cudaMemset(bias, 0, sizeof(float) * V);
  LogitTcMaps maps = rows ? make_logit_rows_maps(thi, tlo, R, K, Kp, whi, wlo, Kp, V)
                          : make_logit_maps(thi, tlo, R, K, Kp, whi, wlo, Kp, V);
  auto launch = [&](const LogitTcArgs &a) {
    if (rows)
      launch_logits_rows(maps, a, 0);
    else
      launch_logits_tc(maps, a, 0);
  };
  const char *names[] = {"full", "no A loads", "no B loads", "no A/B loads", "no MMA", "no epilogue",
                         "loads only (no MMA, no epi)", "MMA only (no loads, no epi)", "no top-k", "no sum pass",
                         "no stores", "no topk/sum/stores", "no merge", "no topk/sum/merge/stores"};
  const int flags[] = {0, 1, 2, 3, 4, 8, 12, 11, 16, 32, 64, 112, 128, 240};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int v = 0; v < (rows ? 1 : 14); ++v) {
    LogitTcArgs a{R, V, K, bias, kk, ntiles, 1.f / (1 << 20), pmax, psum, cval, ctok};
    a.debug_flags = flags[v];
    for (int i = 0; i < 3; ++i) launch(a);
    cudaEventRecord(e0);
    const int it = 20;
    for (int i = 0; i < it; ++i) launch(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("%s R=%d kk=%d %-30s %8.1f us  %s\n", rows ? "rows" : "swap", R, kk, names[v], 1000 * ms / it, cudaGetErrorString(err));
  }
  {
    long long *dclk;
    cudaMalloc(&dclk, sizeof(long long) * 64 * 16);
    cudaMemset(dclk, 0, sizeof(long long) * 64 * 16);
    LogitTcArgs a{R, V, K, bias, kk, ntiles, 1.f / (1 << 20), pmax, psum, cval, ctok};
    a.debug_clock = dclk;
    launch(a);
    cudaDeviceSynchronize();
    std::vector<long long> c(64 * 16);
    cudaMemcpy(c.data(), dclk, sizeof(long long) * 64 * 16, cudaMemcpyDeviceToHost);
    if (rows) {
      printf("unit: prod_start prod_end | mma_start mma_end | epi_start epi_end (cycles from unit 0 producer start)\n");
      const long long t0 = c[4];
      for (int u = 0; u < 8; ++u) {
        long long *r = &c[u * 8];
        if (!r[4]) break;
        printf("%2d: %8lld %8lld | %8lld %8lld | %8lld %8lld\n", u, r[4] - t0, r[5] - t0, r[0] - t0, r[1] - t0,
               r[2] - t0, r[3] - t0);
      }
    } else {
      printf("chunk: wait_tfull | drain | bar | ldmax | exp | thr | mask | cand | merge | store | bar2   (cycles)\n");
      for (int ch = 0; ch < 12; ++ch) {
        long long *r = &c[ch * 16];
        printf("%2d: %6lld | %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld %6lld\n", ch, r[12] ? r[12] - r[11] : 0,
               r[1] - r[0], r[2] - r[1], r[3] - r[2], r[4] - r[3], r[5] - r[4], r[6] - r[5], r[7] - r[6], r[8] - r[7],
               r[9] - r[8], r[10] - r[9]);
      }
    }
  }
  return 0;
}

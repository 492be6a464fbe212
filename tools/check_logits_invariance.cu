// Batch-invariance probe of the tensor-core logit kernel (not product code):
// the first R0 rows' partial outputs must be bit-identical for any R >= R0.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../paper_1610_01108_b200/csrc/common.cuh"
#include "../paper_1610_01108_b200/csrc/logits_tc.cuh"

using namespace amun;

int main() {
  const int K = 500, V = 30000, kk = 5, ntiles = (V + 127) / 128;
  const int Rs[] = {25, 32, 120, 320, 200, 640};
  const int Rmax = 640;
  std::vector<float> h((size_t)V * K);
  srand(3);
  for (auto &x : h) x = (rand() / (float)RAND_MAX - 0.5f) * 0.2f;
  const int Kp = (K + 7) / 8 * 8;  // 16-byte fp16 row pitch
  std::vector<__half> hh((size_t)V * Kp, __float2half_rn(0.f)), hl(hh.size(), __float2half_rn(0.f));
  for (int r = 0; r < V; ++r)  // 3xFP16 split of (x * 2^10), as the product does
    for (int c = 0; c < K; ++c) {
      const float x = h[(size_t)r * K + c] * 1024.f;
      const __half a = __float2half_rn(x);
      hh[(size_t)r * Kp + c] = a;
      hl[(size_t)r * Kp + c] = __float2half_rn(x - __half2float(a));
    }
  __half *thi, *tlo, *whi, *wlo;
  float *bias, *pmax, *psum, *cval;
  int *ctok;
  cudaMalloc(&thi, sizeof(__half) * Rmax * Kp);
  cudaMalloc(&tlo, sizeof(__half) * Rmax * Kp);
  cudaMalloc(&whi, sizeof(__half) * (size_t)V * Kp);
  cudaMalloc(&wlo, sizeof(__half) * (size_t)V * Kp);
  cudaMalloc(&bias, sizeof(float) * V);
  cudaMalloc(&pmax, sizeof(float) * ntiles * Rmax);
  cudaMalloc(&psum, sizeof(float) * ntiles * Rmax);
  cudaMalloc(&cval, sizeof(float) * ntiles * Rmax * kk);
  cudaMalloc(&ctok, sizeof(int) * ntiles * Rmax * kk);
  cudaMemcpy(thi, hh.data(), sizeof(__half) * Rmax * Kp, cudaMemcpyHostToDevice);
  cudaMemcpy(tlo, hl.data(), sizeof(__half) * Rmax * Kp, cudaMemcpyHostToDevice);
  cudaMemcpy(whi, hh.data(), sizeof(__half) * (size_t)V * Kp, cudaMemcpyHostToDevice);
  cudaMemcpy(wlo, hl.data(), sizeof(__half) * (size_t)V * Kp, cudaMemcpyHostToDevice);
  cudaMemcpy(bias, h.data(), sizeof(float) * V, cudaMemcpyHostToDevice);
  std::vector<float> ref_m, ref_s, ref_v;
  const int R0 = 25;
  for (int R : Rs) {
    LogitTcMaps maps = make_logit_maps(thi, tlo, R, K, Kp, whi, wlo, Kp, V);
    LogitTcArgs a{R, V, K, bias, kk, ntiles, 1.f / (1 << 20), pmax, psum, cval, ctok};
    launch_logits_tc(maps, a, 0);
    cudaDeviceSynchronize();
    std::vector<float> m((size_t)ntiles * R), s((size_t)ntiles * R), v((size_t)R * ntiles * kk);
    cudaMemcpy(m.data(), pmax, m.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(s.data(), psum, s.size() * 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(v.data(), cval, v.size() * 4, cudaMemcpyDeviceToHost);
    std::vector<float> m0, s0, v0;
    for (int t = 0; t < ntiles; ++t)
      for (int r = 0; r < R0; ++r) {
        m0.push_back(m[(size_t)r * ntiles + t]);
        s0.push_back(s[(size_t)r * ntiles + t]);
      }
    v0.assign(v.begin(), v.begin() + (size_t)R0 * ntiles * kk);
    if (ref_m.empty()) {
      ref_m = m0;
      ref_s = s0;
      ref_v = v0;
    }
    int dm = 0, ds = 0, dv = 0;
    for (size_t i = 0; i < m0.size(); ++i) {
      dm += m0[i] != ref_m[i];
      ds += s0[i] != ref_s[i];
    }
    for (size_t i = 0; i < v0.size(); ++i) dv += v0[i] != ref_v[i];
    printf("R=%3d  mismatches vs R=25: max %d  sum %d  topk %d  (%s)\n", R, dm, ds, dv,
           cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

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
  std::vector<float> hh(h.size()), hl(h.size());
  for (size_t i = 0; i < h.size(); ++i) {
    unsigned u;
    memcpy(&u, &h[i], 4);
    u &= 0xFFFFE000u;
    float t;
    memcpy(&t, &u, 4);
    hh[i] = t;
    hl[i] = h[i] - t;
  }
  float *thi, *tlo, *whi, *wlo, *bias, *pmax, *psum, *cval;
  int *ctok;
  cudaMalloc(&thi, sizeof(float) * Rmax * K);
  cudaMalloc(&tlo, sizeof(float) * Rmax * K);
  cudaMalloc(&whi, sizeof(float) * (size_t)V * K);
  cudaMalloc(&wlo, sizeof(float) * (size_t)V * K);
  cudaMalloc(&bias, sizeof(float) * V);
  cudaMalloc(&pmax, sizeof(float) * ntiles * Rmax);
  cudaMalloc(&psum, sizeof(float) * ntiles * Rmax);
  cudaMalloc(&cval, sizeof(float) * ntiles * Rmax * kk);
  cudaMalloc(&ctok, sizeof(int) * ntiles * Rmax * kk);
  cudaMemcpy(thi, hh.data(), sizeof(float) * Rmax * K, cudaMemcpyHostToDevice);
  cudaMemcpy(tlo, hl.data(), sizeof(float) * Rmax * K, cudaMemcpyHostToDevice);
  cudaMemcpy(whi, hh.data(), sizeof(float) * (size_t)V * K, cudaMemcpyHostToDevice);
  cudaMemcpy(wlo, hl.data(), sizeof(float) * (size_t)V * K, cudaMemcpyHostToDevice);
  cudaMemcpy(bias, h.data(), sizeof(float) * V, cudaMemcpyHostToDevice);
  std::vector<float> ref_m, ref_s, ref_v;
  const int R0 = 25;
  for (int R : Rs) {
    LogitTcMaps maps = make_logit_maps(thi, tlo, R, K, K, whi, wlo, V);
    LogitTcArgs a{R, V, K, bias, kk, ntiles, pmax, psum, cval, ctok};
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

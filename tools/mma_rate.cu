// Tensor-core issue-rate probe (not part of the product): one CTA (or CTA
// pair) per SM issues back-to-back tcgen05.mma on resident shared memory,
// no loads, and reports dense FLOP/s for kind::tf32 / kind::f16 at several
// N, with cta_group::1 (M = 128) and cta_group::2 (M = 256).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 tools/mma_rate.cu -o build/mma_rate
#include <cstdio>

#include "../paper_1610_01108_b200/csrc/tc_common.cuh"

using namespace amun;

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {  // bf16 x bf16 -> f32, K-major
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int KIND, int CG>  // KIND 0 tf32, 1 bf16; CG cta_group
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int N, int iters, unsigned long long *cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = tc::align_smem<1024>(smem_raw);  // stays in the shared address space (LDS/STS)
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const int warp = threadIdx.x / 32;
  const uint32_t rank = CG == 2 ? tc::cluster_rank() : 0;
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar, 1);
    tc::fence_barrier_init();
  }
  if (warp == 0) {
    if constexpr (CG == 1) {
      tc::tmem_alloc<512>(&tslot);
    } else {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(tc::smem_u32(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = tslot;
  if (warp == 1 && threadIdx.x % 32 == 0 && rank == 0) {
    const int M = 128 * CG;
    const uint32_t idesc = KIND == 0 ? tc::idesc_tf32(M, N) : idesc_f16(M, N);
    const uint32_t base = tc::smem_u32(smem);
    const uint64_t da = tc::desc_kmajor_sw128(base);
    const uint64_t db = tc::desc_kmajor_sw128(base + 65536);
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint32_t acc = (i | k) != 0;
        if constexpr (CG == 1) {
          if constexpr (KIND == 0)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
        } else {
          if constexpr (KIND == 0)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
          else
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                         "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                         "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"(acc));
        }
      }
    }
    if constexpr (CG == 1)
      tc::mma_commit(&bar);
    else
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              tc::smem_u32(&bar)),
          "h"((uint16_t)3)
          : "memory");
    tc::mbar_wait(&bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = (unsigned long long)(t1 - t0);
  }
  if constexpr (CG == 2) {
    if (rank == 1 && threadIdx.x == 0) tc::mbar_wait(&bar, 0);
  }
  tc::tc_fence_before();
  __syncthreads();
  if constexpr (CG == 2) tc::cluster_sync();
  tc::tc_fence_after();
  if (warp == 0) {
    if constexpr (CG == 1)
      tc::tmem_dealloc<512>(tmem);
    else
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

template <int KIND, int CG>
void run(int N) {
  auto kern = mma_rate_kernel<KIND, CG>;
  const int smem = 160 * 1024;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  unsigned long long *dcyc;
  cudaMalloc(&dcyc, 8);
  const int iters = 2000;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute la[1];
  la[0].id = cudaLaunchAttributeClusterDimension;
  la[0].val.clusterDim.x = CG;
  la[0].val.clusterDim.y = 1;
  la[0].val.clusterDim.z = 1;
  cfg.attrs = la;
  cfg.numAttrs = 1;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchKernelEx(&cfg, kern, N, iters, dcyc);
  cudaEventRecord(e0);
  cudaLaunchKernelEx(&cfg, kern, N, iters, dcyc);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long cyc;
  cudaMemcpy(&cyc, dcyc, 8, cudaMemcpyDeviceToHost);
  const int K = KIND == 0 ? 8 : 16;
  const double flop_per_mma = 2.0 * 128 * CG * N * K;
  const double mmas = 4.0 * iters;
  const double total = flop_per_mma * mmas * (148 / CG);
  printf("%s cta_group::%d M=%d N=%3d: %7.1f cyc/MMA, %6.0f flop/clk/SM, %7.1f TFLOP/s  %s\n", KIND ? "bf16" : "tf32", CG,
         128 * CG, N, cyc / mmas, flop_per_mma / (cyc / mmas) / CG, total / (ms * 1e-3) * 1e-12,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  for (int N : {64, 128, 160, 256}) run<0, 1>(N);
  for (int N : {64, 128, 160, 256}) run<1, 1>(N);
  for (int N : {64, 128, 160, 256}) run<0, 2>(N);
  for (int N : {64, 128, 160, 256}) run<1, 2>(N);
  return 0;
}

// Microbenchmark: tcgen05.mma issue throughput for the attention shapes (M=128, K=16 per
// instruction, N in {16, 64, 128, 256}; A from smem or TMEM; B K-major SW128 / MN-major / SW32).
// Operand contents are garbage (timing only).  Build + run on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_17633_b200/csrc \
//        tools/mma_bench.cu -o /tmp/mma_bench && /tmp/mma_bench
#include <cstdio>

#include "zs_common.cuh"

using namespace zs;

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .b32 %%rx;\n\t.reg .pred %%px;\n\t"
      "elect.sync %%rx|%%px, %1;\n\t"
      "@%%px mov.s32 %0, 1;\n\t}\n"
      : "+r"(pred)
      : "r"(0xffffffffu));
  return pred != 0;
}
__device__ __forceinline__ void umma_ss_e(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_ts_e(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}

// mode: 0 SS K-major SW128 (A 128x16, B Nx16); 1 TS (A tmem) + B MN-major SW128; 2 SS SW32 (tail);
//       3 TS + B MN-major SW32
__global__ void __launch_bounds__(128, 1) bench(int mode, int N, int iters, int nd, unsigned long long* out) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 0) {  // whole warp runs the loop (uniform registers), one elected lane issues
    uint32_t id;
    if (mode == 0 || mode == 2) id = idesc_bf16(128, N);
    else id = idesc_bf16(128, N, false, true);
    uint8_t* A = smem;
    uint8_t* B = smem + 65536;
    // descriptors hoisted; 8 MMAs per iteration with compile-time offsets (issue cost floor)
    const uint64_t a0 = (mode == 2) ? sdesc_k_sw32(A) : sdesc_k_sw128(A);
    const uint64_t b0 = (mode == 0) ? sdesc_k_sw128(B) : (mode == 1 ? sdesc_mn_sw128(B) : sdesc_k_sw32(B));
    const uint32_t D0 = tmem + 64;
    const unsigned long long t0 = clock64();
    if (mode == 0 || mode == 2) {
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          umma_ss_e(D0 + (nd == 2 ? (j & 1) * 192 : 0), a0 + 2 * (j & 3), b0 + 2 * (j & 3), id, 1);
      }
    } else {
      for (int i = 0; i < iters; i += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          umma_ts_e(D0 + (nd == 2 ? (j & 1) * 192 : 0), tmem + 8 * (j & 3), b0 + 128 * (j & 3), id, 1);
      }
    }
    if (elect_one()) umma_commit(&bar);
    mbar_wait(&bar, 0);
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 148 * sizeof(unsigned long long));
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const char* names[4] = {"SS K-major SW128", "TS + B MN SW128", "SS SW32 (tail)", "TS + B MN SW32"};
  const int iters = 4096;
  for (int mode = 0; mode < 4; ++mode) {
    for (int N : {16, 64, 128, 256}) {
      for (int nd : {1, 2}) {
        if (mode == 3 || (nd == 2 && N > 192)) continue;
        const int grid = 148;
        bench<<<grid, 128, 200 * 1024>>>(mode, N, iters, nd, d);
        unsigned long long h[148];
        cudaMemcpy(h, d, grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
        unsigned long long mx = 0;
        for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
        const double cyc = (double)mx / iters;
        const double macs = 128.0 * N * 16;
        printf("%-18s N=%3d nd=%d  %7.1f cycles/MMA  %6.0f MAC/clk/SM\n", names[mode], N, nd, cyc, macs / cyc);
      }
    }
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

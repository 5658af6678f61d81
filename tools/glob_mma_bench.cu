// Microbenchmark: tensor-core time of the global attention kernel's per-chunk MMA sequence
// (zs_attn_glob.cu), garbage operands, one CTA per SM, the MMA warp alone (no softmax):
//   S'  = 4 x (M128 N128 K16 bf16 SS SW128) + 1 x SW32 tail + 8 x (M128 N128 K16 fp16, A smem or TMEM)
//   PV  = 8 x (M128 N64 K16 TS MN-SW128 + N16 TS MN-SW32 tail + N16 ones)
// and each part alone, so the per-chunk tensor floor is measured rather than assumed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_17633_b200/csrc \
//        tools/glob_mma_bench.cu -o /tmp/glob_mma_bench && /tmp/glob_mma_bench
#include <cstdio>

#include "zs_common.cuh"

using namespace zs;

__host__ __device__ constexpr uint32_t idesc_f16_(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

// what: bit 0 QK, bit 1 bias (SS), bit 2 bias (TS), bit 3 PV main, bit 4 PV tail + ones, bit 5 bias K=64 only
__global__ void __launch_bounds__(128, 1) bench(int what, int iters, unsigned long long* out) {
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
  if (warp == 0) {
    constexpr uint32_t id_s = idesc_bf16(128, 128);
    constexpr uint32_t id_b = idesc_f16_(128, 128);
    constexpr uint32_t id_pv = idesc_bf16(128, 64, false, true);
    constexpr uint32_t id_pv2 = idesc_bf16(128, 16, false, true);
    const uint64_t dq = sdesc_k_sw128(smem), dqt = sdesc_k_sw32(smem + 16384);
    const uint64_t dk = sdesc_k_sw128(smem + 24576), dkt = sdesc_k_sw32(smem + 24576 + 16384);
    const uint64_t dbq = sdesc_k_sw128(smem + 49152), doh = sdesc_k_sw128(smem + 81920);
    const uint64_t dv = sdesc_mn_sw128(smem + 114688), dvt = sdesc_mn_sw32(smem + 114688 + 16384);
    const uint64_t dones = sdesc_mn_sw32(smem + 139264);
    constexpr uint32_t id_pv96 = idesc_bf16(128, 96, false, true);
    constexpr uint32_t id_pv32 = idesc_bf16(128, 32, false, true);
    const uint64_t dv96 = sdesc(smem + 114688, 4096, 256, 6);
    const uint64_t dv32 = sdesc(smem + 114688 + 16384, 4096, 256, 6);
    const uint64_t dv128 = sdesc(smem + 114688, 16384, 1024, 2);
    const uint32_t S0 = tmem, O0 = tmem + 256, BQ = tmem + 448;
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t d = S0 + (i & 1) * 128;
      if (what & 1) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) umma_ss(d, dq + 2 * ks, dk + 2 * ks, id_s, ks > 0);
        umma_ss(d, dqt, dkt, id_s, 1);
      }
      if (what & 2) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)
          umma_ss(d, dbq + (ks >> 2) * 1024 + 2 * (ks & 3), doh + (ks >> 2) * 1024 + 2 * (ks & 3), id_b, 1);
      }
      if (what & 4) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) umma_ts(d, BQ + 8 * ks, doh + (ks >> 2) * 1024 + 2 * (ks & 3), id_b, 1);
      }
      if (what & 32) {
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) umma_ts(d, BQ + 8 * ks, doh + 2 * ks, id_b, 1);
      }
      const uint32_t o = O0 + (i & 1) * 96;
      if (what & 8) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) umma_ts(o, d + 8 * ks, dv + ks * 128, id_pv, 1);
      }
      if (what & 64) {  // PV as one N=96 MMA per k-step: B = 6 MN-major SW32 atoms (16 cols x 128 keys), LBO 4096
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) umma_ts(o, d + 8 * ks, dv96 + ks * 32, id_pv96, 1);
      }
      if (what & 128) {  // PV as N=64 (SW128) + N=32 (two SW32 atoms, LBO 4096)
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          umma_ts(o, d + 8 * ks, dv + ks * 128, id_pv, 1);
          umma_ts(o + 64, d + 8 * ks, dv32 + ks * 32, id_pv32, 1);
        }
      }
      if (what & 256) {  // PV as one N=96 MMA, SW128 MN-major atoms (64 cols x 128 keys), LBO 16384
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) umma_ts(o, d + 8 * ks, dv128 + ks * 128, id_pv96, 1);
      }
      if (what & 16) {
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          umma_ts(o + 64, d + 8 * ks, dvt + ks * 32, id_pv2, 1);
          umma_ts(o + 80, d + 8 * ks, dones + ks * 32, id_pv2, 1);
        }
      }
    }
    umma_commit_elect(&bar);
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
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int iters = 2000;
  struct {
    int what;
    const char* name;
  } cases[] = {{1, "QK (4 SS SW128 + SW32 tail)"},
               {2, "bias K=128 SS"},
               {4, "bias K=128 TS"},
               {32, "bias K=64 TS"},
               {8, "PV main N=64 x8"},
               {16, "PV tail+ones N=16 x16"},
               {24, "PV all"},
               {1 | 2 | 24, "chunk tile A (SS bias)"},
               {1 | 4 | 24, "chunk tile B (TS bias)"},
               {1 | 32 | 24, "chunk, K=64 bias"},
               {1 | 8 | 4, "chunk, no tail/ones"},
               {64, "PV N=96 SW32 atoms"},
               {128, "PV N=64 + N=32"},
               {256, "PV N=96 SW128 atoms"},
               {1 | 32 | 64, "chunk K=64 bias, PV N=96"}};
  for (auto& c : cases) {
    bench<<<148, 128, 200 * 1024>>>(c.what, iters, d);
    bench<<<148, 128, 200 * 1024>>>(c.what, iters, d);
    cudaDeviceSynchronize();
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double s = 0;
    for (int i = 0; i < 148; ++i) s += h[i];
    printf("%-28s %7.1f cycles per chunk\n", c.name, s / 148 / iters);
  }
  printf("status: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

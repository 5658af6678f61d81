// Microbenchmark: one warp gathering 512 random 256-byte rows (L2-resident 2 MiB table) into
// shared memory with (0) cp.async 4 B, (1) cp.async 16 B, (2) LDG.128 + STS.128, (3) LDG.32 +
// STS.32; cycles per item (512 rows).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// -I paper_2605_17633_b200/csrc tools/copy_bench.cu -o /tmp/copy_bench && /tmp/copy_bench
#include <cstdio>

#include "zs_common.cuh"

using namespace zs;

__global__ void bench(const float* __restrict__ tab, const int* __restrict__ rows, int mode, int reps,
                      unsigned long long* out) {
  extern __shared__ float sm[];
  const int lane = threadIdx.x;
  unsigned long long t0 = clock64();
  for (int rep = 0; rep < reps; ++rep) {
    if (mode == 0) {
      for (int r = 0; r < 128; ++r) {
        const float* src = tab + (long long)rows[rep * 128 + r] * 64;
        for (int c = lane; c < 64; c += 32) {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sm + r * 65 + c)), "l"(src + c)
                       : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(sm + 8320 + r * 65 + c)),
                       "l"(src + 2097152 / 4 / 2 + c)
                       : "memory");
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (mode == 1) {
      for (int r = 0; r < 128; r += 2) {
        const int rr = r + (lane >> 4), c = (lane & 15) * 4;
        const float* src = tab + (long long)rows[rep * 128 + rr] * 64;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + rr * 68 + c)), "l"(src + c)
                     : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + 8704 + rr * 68 + c)),
                     "l"(src + 2097152 / 4 / 2 + c)
                     : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (mode == 2) {
#pragma unroll 1
      for (int r0 = 0; r0 < 128; r0 += 16) {
        float4 v[8], w[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int rr = r0 + 2 * q + (lane >> 4), c = (lane & 15) * 4;
          const float* src = tab + (long long)rows[rep * 128 + rr] * 64;
          v[q] = __ldg(reinterpret_cast<const float4*>(src + c));
          w[q] = __ldg(reinterpret_cast<const float4*>(src + 2097152 / 4 / 2 + c));
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int rr = r0 + 2 * q + (lane >> 4), c = (lane & 15) * 4;
          *reinterpret_cast<float4*>(sm + rr * 68 + c) = v[q];
          *reinterpret_cast<float4*>(sm + 8704 + rr * 68 + c) = w[q];
        }
      }
    } else {
#pragma unroll 1
      for (int r0 = 0; r0 < 128; r0 += 8) {
        float v[16], w[16];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const float* src = tab + (long long)rows[rep * 128 + r0 + q] * 64;
          v[2 * q] = __ldg(src + lane);
          v[2 * q + 1] = __ldg(src + 32 + lane);
          w[2 * q] = __ldg(src + 2097152 / 4 / 2 + lane);
          w[2 * q + 1] = __ldg(src + 2097152 / 4 / 2 + 32 + lane);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int rr = r0 + q;
          sm[lane * 129 + rr] = v[2 * q];  // transposed, padded: bT[j][r]
          sm[(lane + 32) * 129 + rr] = v[2 * q + 1];
          sm[8256 + lane * 129 + rr] = w[2 * q];
          sm[8256 + (lane + 32) * 129 + rr] = w[2 * q + 1];
        }
      }
    }
    __syncwarp();
  }
  unsigned long long t1 = clock64();
  if (lane == 0) out[blockIdx.x] = (t1 - t0) / reps;
}

int main() {
  float* tab;
  int* rows;
  unsigned long long* d;
  cudaMalloc(&tab, 4 << 20);
  cudaMemset(tab, 0, 4 << 20);
  const int reps = 64;
  int h[148 * 64 * 128];
  for (int i = 0; i < 148 * 64 * 128; ++i) h[i] = (i * 2654435761u >> 7) % 4096;
  cudaMalloc(&rows, sizeof(h));
  cudaMemcpy(rows, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMalloc(&d, 148 * 8);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const char* names[4] = {"cp.async 4B (stride 65)", "cp.async 16B (stride 68)", "LDG.128+STS (stride 68)",
                          "LDG.32+STS transposed (129)"};
  for (int mode = 0; mode < 4; ++mode) {
    for (int grid : {1, 148}) {
      bench<<<grid, 32, 100 * 1024>>>(tab, rows, mode, reps, d);
      unsigned long long o[148];
      cudaMemcpy(o, d, grid * 8, cudaMemcpyDeviceToHost);
      unsigned long long mx = 0;
      for (int i = 0; i < grid; ++i) mx = o[i] > mx ? o[i] : mx;
      printf("%-30s grid=%3d  %8llu cycles per 128-row item (bh+bw)\n", names[mode], grid, mx);
    }
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}

// Microbenchmark: per-SM issue throughput of the softmax instruction mix on B200 —
// MUFU.EX2 (fp32), FMNMX (2-input), 3-input max.f32, F2FP bf16x2 pack, FFMA2 (fma.rn.f32x2),
// and a degree-3 polynomial exp2 on the FMA pipe (FA4-style).  8 independent chains per thread,
// 8 warps per SM (2 per SMSP, as the attention softmax), one CTA per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2605_17633_b200/csrc \
//        tools/pipe_bench.cu -o /tmp/pipe_bench && /tmp/pipe_bench
#include <cstdio>

#include "zs_common.cuh"

// exp2_pair_bf16_ns on the FMA / ALU pipes (no MUFU): t = s * c + m2 (FFMA2), clamped at -127,
// split t = n + f with n = round(t) (magic-number add, FADD2) and f in [-0.5, 0.5], 2^f by a
// degree-3 polynomial with p(0) = 1 (Lawson minimax on [-0.5, 0.5], max relative error 1.0e-4,
// below the bf16 rounding of P: 2^-9), 2^n added to the exponent as an integer.  t = -inf or
// NaN gives 0.  Used for a fixed share of the softmax pairs so the exponentials of one warp
// overlap on two pipes (the MUFU alone issues one warp instruction per 8 cycles per SMSP).
namespace zs {
__device__ __forceinline__ uint32_t exp2_pair_bf16_poly(float s0, float s1, unsigned long long c2,
                                                        unsigned long long m2) {
  unsigned long long t, r, n, f, p;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(t) : "l"(f32x2(s0, s1)), "l"(c2), "l"(m2));
  float2 tt = unpack_f32x2(t);
  tt.x = fmaxf(tt.x, -127.f);
  tt.y = fmaxf(tt.y, -127.f);
  t = f32x2(tt.x, tt.y);
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(t), "l"(f32x2(12582912.f, 12582912.f)));   // 1.5 * 2^23
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(n) : "l"(r), "l"(f32x2(-12582912.f, -12582912.f)));  // round(t)
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(f) : "l"(n), "l"(f32x2(-1.f, -1.f)), "l"(t));    // t - n
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(f32x2(0.05500893f, 0.05500893f)), "l"(f),
      "l"(f32x2(0.24221098f, 0.24221098f)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(p), "l"(f), "l"(f32x2(0.6932829f, 0.6932829f)));
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(p), "l"(f), "l"(f32x2(1.f, 1.f)));
  const float2 pp = unpack_f32x2(p), rr = unpack_f32x2(r);
  const float e0 = __uint_as_float(__float_as_uint(pp.x) + (__float_as_uint(rr.x) << 23));
  const float e1 = __uint_as_float(__float_as_uint(pp.y) + (__float_as_uint(rr.y) << 23));
  uint32_t o;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(o) : "f"(e1), "f"(e0));
  return o;
}
}  // namespace zs

constexpr int ITERS = 4096;

template <int OP>
__global__ void bench(float* out, long long* cyc, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed * (threadIdx.x + i) * 1e-3f;
  uint32_t u[8] = {0};
  unsigned long long v2[8];
  const unsigned long long k2 = zs::f32x2(1.0001f, 0.9999f);
#pragma unroll
  for (int i = 0; i < 8; ++i) v2[i] = zs::f32x2(a[i], a[i] + 1.f);
  __syncthreads();
  const long long t0 = clock64();
#pragma unroll 4
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if constexpr (OP == 0) {  // MUFU ex2
        asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
      } else if constexpr (OP == 1) {  // FMNMX 2-input
        asm volatile("max.f32 %0, %0, %1;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]));
      } else if constexpr (OP == 2) {  // 3-input max
        asm volatile("max.f32 %0, %0, %1, %2;" : "+f"(a[i]) : "f"(a[(i + 1) & 7]), "f"(a[(i + 2) & 7]));
      } else if constexpr (OP == 3) {  // F2FP bf16x2 pack
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(__uint_as_float(u[i])));
      } else if constexpr (OP == 4) {  // FFMA2: 8 independent packed accumulators
        asm volatile("fma.rn.f32x2 %0, %0, %1, %1;" : "+l"(v2[i]) : "l"(k2));
      } else if constexpr (OP == 7) {  // FADD2
        asm volatile("add.rn.f32x2 %0, %0, %1;" : "+l"(v2[i]) : "l"(k2));
      } else if constexpr (OP == 8) {  // FMUL2
        asm volatile("mul.rn.f32x2 %0, %0, %1;" : "+l"(v2[i]) : "l"(k2));
      } else if constexpr (OP == 5) {  // FFMA
        asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i]));
      } else if constexpr (OP == 6) {  // cvt f32 -> f16x2 pack
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(u[i]) : "f"(a[i]), "f"(__uint_as_float(u[i])));
      }
    }
  }
  const long long t1 = clock64();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i] + __uint_as_float(u[i]) + zs::unpack_f32x2(v2[i]).x;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int OP>
void run(const char* name, int threads) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  bench<OP><<<148, threads>>>(out, cyc, 1.0f);
  bench<OP><<<148, threads>>>(out, cyc, 1.0f);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  const double ops = (double)threads * ITERS * 8;  // thread-ops per SM
  printf("%-14s threads %4d: %.2f thread-ops/clk/SM (%.1f cycles per warp-instr per SMSP)\n", name, threads,
         ops / c, c / (ops / 32 / 4));
  cudaFree(out);
  cudaFree(cyc);
}

int main1() {
  for (int t : {256, 512}) {
    run<0>("mufu.ex2", t);
    run<1>("fmnmx", t);
    run<2>("max3", t);
    run<3>("f2fp.bf16x2", t);
    run<4>("ffma2", t);
    run<5>("ffma", t);
    run<6>("f2fp.f16x2", t);
    run<7>("fadd2", t);
    run<8>("fmul2", t);
  }
  return 0;
}

// softmax numerator pattern (exp2_pair_bf16_ns): 64 pairs per thread per "chunk", 256 threads
template <int PM>  // pairs q with (q % 8) < PM use the polynomial exp2
__global__ void bench_softmax(float* out, long long* cyc, float seed, int chunks) {
  float s[128];
#pragma unroll
  for (int i = 0; i < 128; ++i) s[i] = seed * (threadIdx.x + i) * 1e-3f;
  uint32_t acc = 0;
  const unsigned long long c2 = zs::f32x2(1.3f, 1.3f), m2 = zs::f32x2(-2.f, -2.f);
  __syncthreads();
  const long long t0 = clock64();
  for (int c = 0; c < chunks; ++c) {
#pragma unroll
    for (int q = 0; q < 64; ++q) {
      const uint32_t p = (q % 8) < PM ? zs::exp2_pair_bf16_poly(s[2 * q], s[2 * q + 1], c2, m2)
                                      : zs::exp2_pair_bf16_ns(s[2 * q], s[2 * q + 1], c2, m2);
      acc ^= p;
      s[2 * q] = __uint_as_float(p & 0xffff0000u);
    }
  }
  const long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = __uint_as_float(acc) + s[5];
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int PM>
int main2() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  for (int threads : {128, 256}) {
    bench_softmax<PM><<<148, threads>>>(out, cyc, 1.0f, 64);
    bench_softmax<PM><<<148, threads>>>(out, cyc, 1.0f, 64);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double c = 0;
    for (int i = 0; i < 148; ++i) c += h[i];
    c /= 148;
    printf("poly %d/8: softmax pattern threads %d: %.1f cycles per 128x128 chunk-equivalent (%.2f elems/clk/SM)\n", threads,
           PM, c / 64 * (128.0 * 128 / (threads * 128.0)), threads * 128.0 * 64 / c);
  }
  return 0;
}
int main() {
  main1();
  return 0;
}

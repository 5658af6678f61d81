// zs_host.h — host-side helpers shared by the kernel translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/zstripe_b200.h"

namespace zs {

struct GemmEpi {
  const float* bias;               // [N] fp32 or nullptr
  void* out;                       // bf16 or fp32 [*, ld_out]
  long long ld_out;
  const float* res;                // fp32 residual (may alias out) or nullptr
  long long ld_res;
  const int* row_map;              // [M] output row per GEMM row, or nullptr
  const int* m_dev;                // optional device-side row count (min with M)
  const unsigned char* zero_rows;  // [M] 1 -> write zeros, or nullptr
  int res_mod;                     // >0: residual row = m % res_mod
};

int launch_layernorm(const float* x, long long ldx, const int* rows, const int* out_rows, long long n,
                     const int* n_dev, int C, const float* g, const float* b, float eps, void* out, long long ldo,
                     int out_f32, cudaStream_t st);

// Kernel launches issued by the calling thread (zs_launch_counter, for the host's launch accounting).
void count_launch();

// Cached SM count of the current device.
int num_sms();

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
int make_tmap_2d_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                      uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz);
int make_tmap_3d_bf16(CUtensorMap* m, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t ld1_elems,
                      uint64_t ld2_elems, uint32_t b0, uint32_t b1, uint32_t b2, CUtensorMapSwizzle swz);

int launch_gemm(int epi, const void* A, long long lda, const void* W, long long ldw, int M, int N, int K,
                const GemmEpi& ep, cudaStream_t stream, int max_ctas);

}  // namespace zs

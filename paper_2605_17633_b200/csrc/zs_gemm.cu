// zs_gemm.cu — persistent warp-specialised tcgen05 GEMM with fused SparseSAM epilogues.
//
//   D[m, n] = sum_k A[m, k] * W[n, k]          (bf16 in, fp32 accumulate in TMEM)
//
// A is row-major [M, K] bf16 (activations), W is nn.Linear-layout [N, K] bf16
// (both K-major).  The epilogue fuses the per-row work that surrounds every
// dense matmul on the reference hot path (encoder.py:290,307; mlp.py:82-83):
//
//   EPI_BF16       out_bf16[m, n] = D + bias[n]                   (QKV, neck)
//   EPI_BF16_GELU  out_bf16[m, n] = gelu_erf(D + bias[n])          (RC-MLP fc1)
//   EPI_F32_RESID  out_f32[row(m), n] = res[rrow(m), n] + D + bias[n]
//                  row(m)  = row_map ? row_map[m] : m              (RC-MLP fc2 scatter-add,
//                  rrow(m) = res_mod ? m % res_mod : row(m)         attention proj + residual,
//                  zero_rows[m] != 0 -> the output row is written 0  patch-embed + abs-pos)
//
// Roles (256 threads, one CTA per SM, persistent over output tiles):
//   warp 0      TMA producer   (one elected lane)  smem ring of kStages {A, W} tiles
//   warp 1      MMA issuer     (one lane)          tcgen05.mma 128 x 256 x 16
//   warp 2      TMEM allocator
//   warps 4..7  epilogue       tcgen05.ld -> bias/GELU/residual -> global
// TMEM holds two 128x256 fp32 accumulators so the epilogue of tile i overlaps
// the MMAs of tile i+1.
#include <cstdlib>

#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {

enum GemmEpiKind : int { EPI_BF16 = 0, EPI_BF16_GELU = 1, EPI_F32_RESID = 2 };


namespace gemm {
constexpr int BM = 128, BN = 256, BK = 64, UK = 16;
constexpr int kStages = 4;
constexpr int A_BYTES = BM * BK * 2;   // 16 KB
constexpr int B_BYTES = BN * BK * 2;   // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int SMEM_BYTES = kStages * STAGE_BYTES + 1024 /*align slack*/ + 256 /*barriers*/;
constexpr int kThreads = 256;
constexpr uint32_t kTmemCols = 2 * BN;  // 512
}  // namespace gemm

template <int EPI>
__global__ void __launch_bounds__(gemm::kThreads, 1)
    zs_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M,
                   int N, int K, GemmEpi ep) {
  using namespace gemm;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);  // stays in the shared space
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * STAGE_BYTES);
  uint64_t* full = bars;                  // [kStages]
  uint64_t* empty = bars + kStages;       // [kStages]
  uint64_t* tfull = bars + 2 * kStages;   // [2]
  uint64_t* tempty = bars + 2 * kStages + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 128);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (ep.m_dev) M = min(M, *ep.m_dev);
  const int m_tiles = (M + BM - 1) / BM;
  const int n_tiles = (N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int nk = K / BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        const int m0 = (t / n_tiles) * BM;
        const int n0 = (t % n_tiles) * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait_sleep(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          mbar_expect_tx(&full[stage], STAGE_BYTES);
          tma_load_2d(sa, &tmA, &full[stage], kb * BK, m0);
          tma_load_2d(sb, &tmB, &full[stage], kb * BK, n0);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = idesc_bf16(BM, BN);
    int stage = 0;
    uint32_t phase = 0;
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      mbar_wait_sleep(&tempty[as], aphase ^ 1);
      tc_fence_after();
      const uint32_t dtm = tmem_base + as * BN;
      for (int kb = 0; kb < nk; ++kb) {
        mbar_wait_sleep(&full[stage], phase);
        tc_fence_after();
        if (lane == 0) {
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          const uint64_t da = sdesc_k_sw128(sa);
          const uint64_t db = sdesc_k_sw128(sb);
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) {
            // advance 16 bf16 = 32 bytes along K inside the 128B swizzle atom
            umma_bf16(dtm, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          }
          umma_commit(&empty[stage]);
          if (kb == nk - 1) umma_commit(&tfull[as]);
        }
        __syncwarp();
        if (++stage == kStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp >= 4) {
    const int q = warp & 3;  // TMEM lane quarter owned by this warp
    int it = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x, ++it) {
      const int as = it & 1;
      const uint32_t aphase = (it >> 1) & 1;
      const int m0 = (t / n_tiles) * BM;
      const int n0 = (t % n_tiles) * BN;
      mbar_wait_sleep(&tfull[as], aphase);
      tc_fence_after();
      const int m = m0 + q * 32 + lane;
      const bool valid = m < M;
      long long orow = m, rrow = m;
      bool zero = false;
      if (valid) {
        if (ep.row_map) orow = ep.row_map[m];
        rrow = ep.res_mod > 0 ? (long long)(m % ep.res_mod) : orow;
        if (ep.zero_rows) zero = ep.zero_rows[m] != 0;
      }
      const uint32_t trow = tmem_base + as * BN + ((uint32_t)(q * 32) << 16);
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        __syncwarp();
        tmem_ld32(trow + c, r);
        tmem_ld_wait();
        const int nb = n0 + c;
        if (valid && nb < N) {
        float v[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
        if (ep.bias) {
          const float4* b4 = reinterpret_cast<const float4*>(ep.bias + nb);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float4 b = __ldg(b4 + j);
            v[4 * j] += b.x;
            v[4 * j + 1] += b.y;
            v[4 * j + 2] += b.z;
            v[4 * j + 3] += b.w;
          }
        }
        if constexpr (EPI == EPI_BF16 || EPI == EPI_BF16_GELU) {
          if constexpr (EPI == EPI_BF16_GELU) {
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = gelu_erf(v[j]);
          }
          uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(ep.out) + orow * ep.ld_out + nb);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 w;
            w.x = pack_bf16(v[8 * j + 0], v[8 * j + 1]);
            w.y = pack_bf16(v[8 * j + 2], v[8 * j + 3]);
            w.z = pack_bf16(v[8 * j + 4], v[8 * j + 5]);
            w.w = pack_bf16(v[8 * j + 6], v[8 * j + 7]);
            dst[j] = w;
          }
        } else {
          float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.out) + orow * ep.ld_out + nb);
          if (zero) {
#pragma unroll
            for (int j = 0; j < 8; ++j) dst[j] = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            if (ep.res) {
              const float4* src = reinterpret_cast<const float4*>(ep.res + rrow * ep.ld_res + nb);
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float4 x = src[j];
                v[4 * j] += x.x;
                v[4 * j + 1] += x.y;
                v[4 * j + 2] += x.z;
                v[4 * j + 3] += x.w;
              }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) dst[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
        }
        }  // valid
      }
      __syncwarp();
      tc_fence_before();
      mbar_arrive(&tempty[as]);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem_base, kTmemCols);
}

}  // namespace zs

// ------------------------------------------------------------------ host side

namespace zs {

int launch_gemm2(int epi, const void* A, long long lda, const void* W, long long ldw, int M, int N, int K,
                 const GemmEpi& ep, cudaStream_t stream);

int launch_gemm(int epi, const void* A, long long lda, const void* W, long long ldw, int M, int N, int K,
                const GemmEpi& ep, cudaStream_t stream, int max_ctas) {
  using namespace gemm;
  if (M <= 0) return 0;
  if (N <= 0 || K <= 0 || (K % BK) != 0 || (N % 32) != 0) return ZS_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(A) & 15) || (reinterpret_cast<uintptr_t>(W) & 15) || (lda % 8) || (ldw % 8))
    return ZS_ERR_ALIGN;
  if (epi < 0 || epi > 2) return ZS_ERR_ARG;
  // CTA-pair kernel for everything but tiny problems (ZS_GEMM_1CTA=1 forces the single-CTA kernel)
  static const bool force_1cta = getenv("ZS_GEMM_1CTA") != nullptr;
  if (!force_1cta && max_ctas <= 0 && M > 128) return launch_gemm2(epi, A, lda, W, ldw, M, N, K, ep, stream);
  CUtensorMap ta, tb;
  int rc = make_tmap_2d_bf16(&ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d_bf16(&tb, W, (uint64_t)K, (uint64_t)N, (uint64_t)ldw, BK, BN, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const int tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  int grid = num_sms();
  if (max_ctas > 0 && max_ctas < grid) grid = max_ctas;
  if (grid > tiles) grid = tiles;
  cudaError_t e;
  switch (epi) {
    case EPI_BF16:
      cudaFuncSetAttribute(zs_gemm_kernel<EPI_BF16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      { zs_gemm_kernel<EPI_BF16><<<grid, kThreads, SMEM_BYTES, stream>>>(ta, tb, M, N, K, ep); count_launch(); }
      break;
    case EPI_BF16_GELU:
      cudaFuncSetAttribute(zs_gemm_kernel<EPI_BF16_GELU>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      { zs_gemm_kernel<EPI_BF16_GELU><<<grid, kThreads, SMEM_BYTES, stream>>>(ta, tb, M, N, K, ep); count_launch(); }
      break;
    case EPI_F32_RESID:
      cudaFuncSetAttribute(zs_gemm_kernel<EPI_F32_RESID>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      { zs_gemm_kernel<EPI_F32_RESID><<<grid, kThreads, SMEM_BYTES, stream>>>(ta, tb, M, N, K, ep); count_launch(); }
      break;
    default:
      return ZS_ERR_ARG;
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

}  // namespace zs

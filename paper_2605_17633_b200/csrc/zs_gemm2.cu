// zs_gemm2.cu — CTA-pair (cta_group::2) tcgen05 GEMM: 256 x 256 output tile per SM pair.
//
// Same contract and fused epilogues as zs_gemm.cu.  The two CTAs of a cluster
// each own 128 output rows and load their own A rows plus HALF of the B tile
// (128 of its 256 rows); the leader issues tcgen05.mma.cta_group::2 with
// M = 256, so both SMs' tensor cores consume both B halves while each SM only
// streams 32 KB per 64-wide K step instead of 48 KB: one third less L2->SM
// traffic for the same FLOPs, which is what bounds the single-CTA kernel.
//   warp 0      TMA (both CTAs; 2-SM TMA signals the leader's full barrier)
//   warp 1      MMA issue (leader CTA only), commits multicast to both CTAs
//   warp 2      TMEM allocation (cta_group::2, both CTAs)
//   warps 4-11  epilogue: 8 warps, TMEM lane quarter = warp % 4, column half = (warp - 4) / 4
#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {

namespace gemm2 {
constexpr int BM = 128;          // rows per CTA (256 per pair)
constexpr int BN = 256;          // output columns per tile
constexpr int BNH = BN / 2;      // B rows loaded per CTA
constexpr int BK = 64, UK = 16;
constexpr int kStages = 5;
constexpr int A_BYTES = BM * BK * 2;    // 16 KB
constexpr int B_BYTES = BNH * BK * 2;   // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int XS = 36;                                   // padded row stride (floats) of the epilogue transpose
constexpr int EPI_SMEM = 8 * 32 * XS * 4;                // per epilogue warp: 32 rows x 32 fp32
constexpr int SMEM_BYTES = kStages * STAGE_BYTES + 256 + EPI_SMEM + 1024;
constexpr int kThreads = 384;
constexpr int kEpiThreads = 256;
constexpr uint32_t kTmemCols = 2 * BN;  // two accumulators

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t cluster_id_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%clusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t nclusters_x() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%nclusterid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.aligned;\nbarrier.cluster.wait.aligned;" ::: "memory");
}
// arrive on the barrier at the same smem offset in cluster CTA `cta`
__device__ __forceinline__ void mbar_arrive_remote(uint64_t* bar, uint32_t cta) {
  asm volatile(
      "{\n\t.reg .b32 ra;\n\t"
      "mapa.shared::cluster.u32 ra, %0, %1;\n\t"
      "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(smem_u32(bar)),
      "r"(cta)
      : "memory");
}
// 2-SM TMA load: data into this CTA's smem, completion bytes to the leader's barrier
__device__ __forceinline__ void tma_load_2d_pair(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1) {
  const uint32_t leader_bar = smem_u32(bar) & 0xFEFFFFFFu;
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_pair_elect(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t.reg .b32 rx;\n\t"
      "elect.sync rx|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}\n" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
// commit this thread's MMAs to the barrier at the same offset in both CTAs of the pair
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tmem_alloc_pair(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
}  // namespace gemm2

template <int EPI>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(gemm2::kThreads, 1)
    zs_gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int M, int N,
                    int K, GemmEpi ep) {
  using namespace gemm2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kStages * STAGE_BYTES);
  uint64_t* full = bars;                       // [kStages]  (leader: 2 arrivals + tx)
  uint64_t* empty = bars + kStages;            // [kStages]  (multicast commit)
  uint64_t* tfull = bars + 2 * kStages;        // [2]        (multicast commit)
  uint64_t* tempty = bars + 2 * kStages + 2;   // [2]        (leader: 2 x 256 epilogue threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kStages + 4);
  float* xstage = reinterpret_cast<float*>(smem + kStages * STAGE_BYTES + 256);  // [8 warps][32][XS]

  // warp index via shfl: provably warp-uniform, so role code can use uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 2);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 2 * kEpiThreads);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc_pair(tmem_slot, kTmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (ep.m_dev) M = min(M, *ep.m_dev);
  const int m_pairs = (M + 2 * BM - 1) / (2 * BM);
  const int n_tiles = (N + BN - 1) / BN;
  const int num_tiles = m_pairs * n_tiles;
  const int nk = K / BK;
  const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int t = cid; t < num_tiles; t += ncl) {
        const int m0 = (t / n_tiles) * 2 * BM + rank * BM;
        const int n0 = (t % n_tiles) * BN + rank * BNH;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait_sleep(&empty[stage], phase ^ 1);
          uint8_t* sa = smem + stage * STAGE_BYTES;
          uint8_t* sb = sa + A_BYTES;
          if (leader)
            mbar_expect_tx(&full[stage], 2 * STAGE_BYTES);
          else
            mbar_arrive_remote(&full[stage], 0);
          tma_load_2d_pair(sa, &tmA, &full[stage], kb * BK, m0);
          tma_load_2d_pair(sb, &tmB, &full[stage], kb * BK, n0);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // whole warp runs the loop (uniform registers, hoisted descriptors), one elected lane
      // issues: rebuilding descriptors per MMA in a lane-0 branch costs ~120+ cycles per
      // instruction (tools/mma_bench.cu), as much as a 256x256x16 MMA pair itself
      constexpr uint32_t idesc = idesc_bf16(2 * BM, BN);
      const uint64_t da0 = sdesc_k_sw128(smem), db0 = sdesc_k_sw128(smem + A_BYTES);
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int t = cid; t < num_tiles; t += ncl, ++it) {
        const int as = it & 1;
        mbar_wait(&tempty[as], ((it >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t dtm = tmem_base + as * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t da = da0 + (uint64_t)(stage * (STAGE_BYTES >> 4));
          const uint64_t db = db0 + (uint64_t)(stage * (STAGE_BYTES >> 4));
#pragma unroll
          for (int k = 0; k < BK / UK; ++k) umma_pair_elect(dtm, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0);
          umma_commit_pair_elect(&empty[stage]);
          if (kb == nk - 1) umma_commit_pair_elect(&tfull[as]);
          if (++stage == kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp >= 4) {
    const int ew = warp - 4;
    const int q = warp & 3;          // TMEM lane quarter
    const int chalf = ew >> 2;       // column half of the 256-wide tile
    int it = 0;
    // EPI 2: L2 prefetch of the residual rows this thread reads for a tile (one bulk prefetch of
    // its half row), issued one tile ahead so the epilogue's read-modify-write hits L2 instead of
    // waiting a DRAM round trip per 32-column chunk.  The row index is loaded at the top of the
    // previous tile (volatile: kept there) so its latency hides behind that tile's epilogue.
    auto res_row_of = [&](int tt, int& prow) -> bool {
      const int pm = (tt / n_tiles) * 2 * BM + rank * BM + q * 32 + lane;
      if (tt >= num_tiles || pm >= M || !ep.res) return false;
      const int pn0 = (tt % n_tiles) * BN + chalf * (BN / 2);
      if (pn0 >= N) return false;
      prow = pm;
      return true;
    };
    auto ld_row_v = [&](const int* p) {
      int v;
      asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
      return v;
    };
    auto prefetch_res = [&](int tt, int prow) {
      const int pn0 = (tt % n_tiles) * BN + chalf * (BN / 2);
      const int ncols = min(BN / 2, N - pn0);
      const float* src = ep.res + (long long)prow * ep.ld_res + pn0;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(ncols * 4) : "memory");
    };
    auto res_row_index = [&](int tt, int pm) -> int {  // residual row of GEMM row pm (volatile loads)
      if (ep.res_mod > 0) return pm % ep.res_mod;
      if (ep.row_map) return ld_row_v(ep.row_map + pm);
      return pm;
    };
    int pf_row = -1;  // residual row to prefetch for this cluster's next tile (-1: none)
    if constexpr (EPI == 2) {
      int pm;
      if (res_row_of(cid, pm)) prefetch_res(cid, res_row_index(cid, pm));
    }
    for (int t = cid; t < num_tiles; t += ncl, ++it) {
      const int as = it & 1;
      const int m0 = (t / n_tiles) * 2 * BM + rank * BM;
      const int n0 = (t % n_tiles) * BN;
      if constexpr (EPI == 2) {
        int pm;
        pf_row = -1;
        if (res_row_of(t + ncl, pm)) pf_row = res_row_index(t + ncl, pm);  // (zeroed rows: harmless)
      }
      mbar_wait_sleep(&tfull[as], (it >> 1) & 1);
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
      const uint32_t trow = tmem_base + as * BN + ((uint32_t)(q * 32) << 16) + chalf * (BN / 2);
      if constexpr (EPI == 2) {
        // fp32 residual epilogue through a per-warp smem transpose: each lane moves 16-byte pieces
        // so a warp instruction covers 4 full 128-byte row segments.  Rows are fixed per tile;
        // the residual of chunk c + 1 is loaded while chunk c is transposed, added and stored.
        float* xs = xstage + ew * 32 * XS;
        const int c4 = lane & 7;  // float4 column within the 32-wide chunk
        const int nbase = n0 + chalf * (BN / 2);
        int orow2[8], rrow2[8];
        bool live2[8], zero2[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rl = 4 * i + (lane >> 3);
          orow2[i] = __shfl_sync(0xffffffffu, (int)orow, rl);
          rrow2[i] = __shfl_sync(0xffffffffu, (int)rrow, rl);
          zero2[i] = __shfl_sync(0xffffffffu, (int)zero, rl) != 0;
          live2[i] = m0 + q * 32 + rl < M;
        }
        auto load_res = [&](int c, float4(&xr)[8]) {
          const int nb = nbase + c;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            xr[i] = make_float4(0.f, 0.f, 0.f, 0.f);
            if (live2[i] && !zero2[i] && ep.res && nb < N) {
              const float* src = ep.res + (long long)rrow2[i] * ep.ld_res + nb + 4 * c4;
              asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];"
                           : "=f"(xr[i].x), "=f"(xr[i].y), "=f"(xr[i].z), "=f"(xr[i].w)
                           : "l"(src)
                           : "memory");
            }
          }
        };
        float4 xa[8], xb[8];
        load_res(0, xa);
#pragma unroll 1
        for (int c = 0; c < BN / 2; c += 32) {
          if (c + 32 < BN / 2) load_res(c + 32, xb);
          uint32_t r[32];
          __syncwarp();
          tmem_ld32(trow + c, r);
          tmem_ld_wait();
          const int nb = nbase + c;
          {
            float v[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
            if (ep.bias && nb < N) {
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
            float4* xr = reinterpret_cast<float4*>(xs + lane * XS);
#pragma unroll
            for (int j = 0; j < 8; ++j) xr[j] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            if (!live2[i] || nb >= N) continue;
            const int rl = 4 * i + (lane >> 3);
            float4 a = *reinterpret_cast<const float4*>(xs + rl * XS + 4 * c4);
            if (zero2[i]) {
              a = make_float4(0.f, 0.f, 0.f, 0.f);
            } else {
              a.x += xa[i].x;
              a.y += xa[i].y;
              a.z += xa[i].z;
              a.w += xa[i].w;
            }
            reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.out) + (long long)orow2[i] * ep.ld_out + nb)[c4] = a;
          }
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) xa[i] = xb[i];
        }
      } else {
        // TMEM loads software-pipelined: chunk c + 1 is in flight while chunk c is converted
        // and stored (tcgen05.wait::ld then covers both)
        static_assert(BN / 2 == 128, "four 32-column chunks per warp");
        uint32_t ra[32], rb[32];
        __syncwarp();
        tmem_ld32(trow, ra);
        tmem_ld_wait();
        auto emit = [&](const uint32_t (&r)[32], int c) {
          const int nb = n0 + chalf * (BN / 2) + c;
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
            if constexpr (EPI == 1) {
#pragma unroll
              for (int j = 0; j < 16; ++j) gelu_erf_x2(v[2 * j], v[2 * j + 1]);
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
          }
        };
        tmem_ld32(trow + 32, rb);
        emit(ra, 0);
        tmem_ld_wait();
        tmem_ld32(trow + 64, ra);
        emit(rb, 32);
        tmem_ld_wait();
        tmem_ld32(trow + 96, rb);
        emit(ra, 64);
        tmem_ld_wait();
        emit(rb, 96);
      }
      __syncwarp();
      tc_fence_before();
      if (leader)
        mbar_arrive(&tempty[as]);
      else
        mbar_arrive_remote(&tempty[as], 0);
      if constexpr (EPI == 2) {
        if (pf_row >= 0) prefetch_res(t + ncl, pf_row);
      }
    }
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 2) tmem_dealloc_pair(tmem_base, kTmemCols);
}

int launch_gemm2(int epi, const void* A, long long lda, const void* W, long long ldw, int M, int N, int K,
                 const GemmEpi& ep, cudaStream_t stream) {
  using namespace gemm2;
  CUtensorMap ta, tb;
  int rc = make_tmap_2d_bf16(&ta, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda, BK, BM, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  rc = make_tmap_2d_bf16(&tb, W, (uint64_t)K, (uint64_t)N, (uint64_t)ldw, BK, BNH, CU_TENSOR_MAP_SWIZZLE_128B);
  if (rc) return rc;
  const int tiles = ((M + 2 * BM - 1) / (2 * BM)) * ((N + BN - 1) / BN);
  int grid = (num_sms() / 2) * 2;
  if (grid > 2 * tiles) grid = 2 * tiles;
  switch (epi) {
    case 0:
      cudaFuncSetAttribute(zs_gemm2_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      { zs_gemm2_kernel<0><<<grid, kThreads, SMEM_BYTES, stream>>>(ta, tb, M, N, K, ep); count_launch(); }
      break;
    case 1:
      cudaFuncSetAttribute(zs_gemm2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      { zs_gemm2_kernel<1><<<grid, kThreads, SMEM_BYTES, stream>>>(ta, tb, M, N, K, ep); count_launch(); }
      break;
    case 2:
      cudaFuncSetAttribute(zs_gemm2_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      { zs_gemm2_kernel<2><<<grid, kThreads, SMEM_BYTES, stream>>>(ta, tb, M, N, K, ep); count_launch(); }
      break;
    default:
      return ZS_ERR_ARG;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

}  // namespace zs

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
// EPI 3 (fp32 residual through TMA): per epilogue warp kRB buffers of one 32-row x 32-column
// fp32 chunk (4 KB, SW128), gathered / scattered four rows per TMA instruction
#ifndef ZS_G2_RB
#define ZS_G2_RB 2
#endif
constexpr int kRB = ZS_G2_RB;
constexpr int RB_BYTES = 32 * 32 * 4;
#ifndef ZS_G2_DEAD
#define ZS_G2_DEAD (1 << 30)
#endif
constexpr int kDeadRow = ZS_G2_DEAD;  // row coordinate of rows past M: out of the maps' bounds
#ifndef ZS_G2_STAGES3
#define ZS_G2_STAGES3 5
#endif
constexpr int kStages3 = ZS_G2_STAGES3;  // operand ring of the EPI 3 kernel (shares smem with the buffers)
constexpr int SMEM3_BYTES = kStages3 * STAGE_BYTES + 1024 + 8 * kRB * RB_BYTES + 1024;
static_assert(SMEM3_BYTES <= 232448, "EPI 3 shared memory");
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
    zs_gemm2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmO, int M, int N,
                    int K, GemmEpi ep) {
  using namespace gemm2;
  constexpr int NST = EPI == 3 ? kStages3 : kStages;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NST * STAGE_BYTES);
  uint64_t* full = bars;                       // [NST]  (leader: 2 arrivals + tx)
  uint64_t* empty = bars + NST;            // [NST]  (multicast commit)
  uint64_t* tfull = bars + 2 * NST;        // [2]        (multicast commit)
  uint64_t* tempty = bars + 2 * NST + 2;   // [2]        (leader: 2 x 256 epilogue threads)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NST + 4);
  float* xstage = reinterpret_cast<float*>(smem + NST * STAGE_BYTES + 256);  // [8 warps][32][XS]

  // warp index via shfl: provably warp-uniform, so role code can use uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if constexpr (EPI == 3) {
      tma_prefetch_desc(&tmR);
      tma_prefetch_desc(&tmO);
      for (int s = 0; s < 8 * kRB; ++s) mbar_init(bars + 16 + s, 1);
    }
    for (int s = 0; s < NST; ++s) {
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
          if (++stage == NST) {
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
          if (++stage == NST) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (EPI == 3 && warp >= 4) {
    // fp32 residual stream: out[orow] = acc + bias + res[rrow] with the rows moved by TMA.
    // Each warp owns 32 rows x one 128-column half of the tile, in four 32-column chunks that
    // rotate through kRB shared-memory buffers: gather4 loads (4 residual rows per instruction,
    // lanes 0-7 one group each) are issued as soon as a buffer's previous scatter4 store has
    // been read, and the first chunks of the next tile are gathered while this tile's last
    // chunks are stored, so residual reads run ahead of the accumulator instead of behind it.
    // Thread = row: lane r reads / writes its row's 16-byte pieces at (j ^ (r & 7)) (SW128),
    // conflict-free.  Rows past M use coordinate kDeadRow (TMA out of bounds: zero-filled loads,
    // skipped stores); zero_rows rows store zeros without loading.
    const int ew = warp - 4, q = warp & 3, chalf = ew >> 2;
    uint8_t* rb = smem + NST * STAGE_BYTES + 1024 + ew * kRB * RB_BYTES;
    uint64_t* rbar = bars + 16 + ew * kRB;
    uint32_t rphase = 0;  // bit b: parity of buffer b's next completion
    auto ld_row_v = [&](const int* p) {
      int v;
      asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
      return v;
    };
    auto rows_of = [&](int tt, int& lr, int& sr, int& z) {
      lr = sr = kDeadRow;
      z = 0;
      if (tt >= num_tiles) return;
      const int m = (tt / n_tiles) * 2 * BM + rank * BM + q * 32 + lane;
      if (m >= M) return;
      sr = ep.row_map ? ld_row_v(ep.row_map + m) : m;
      z = ep.zero_rows ? (int)ep.zero_rows[m] : 0;
      lr = z ? kDeadRow : (ep.res_mod > 0 ? m % ep.res_mod : sr);
    };
    auto gather = [&](int tt, int c, int lr, int b) {  // chunk c (column offset) of tile tt -> buffer b
      const int col = (tt % n_tiles) * BN + chalf * (BN / 2) + c, g = lane & 7;
      const int r0 = __shfl_sync(0xffffffffu, lr, 4 * g), r1 = __shfl_sync(0xffffffffu, lr, 4 * g + 1);
      const int r2 = __shfl_sync(0xffffffffu, lr, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, lr, 4 * g + 3);
      if (lane == 0) mbar_expect_tx(&rbar[b], RB_BYTES);
      __syncwarp();
      if (lane < 8)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(smem_u32(rb + b * RB_BYTES + g * 512)),
            "l"(reinterpret_cast<uint64_t>(&tmR)), "r"(smem_u32(&rbar[b])), "r"(col), "r"(r0), "r"(r1), "r"(r2),
            "r"(r3)
            : "memory");
    };
    auto scatter = [&](int tt, int c, int sr, int b) {  // buffer b -> chunk c of tile tt, then buffer free
      const int col = (tt % n_tiles) * BN + chalf * (BN / 2) + c, g = lane & 7;
      const int r0 = __shfl_sync(0xffffffffu, sr, 4 * g), r1 = __shfl_sync(0xffffffffu, sr, 4 * g + 1);
      const int r2 = __shfl_sync(0xffffffffu, sr, 4 * g + 2), r3 = __shfl_sync(0xffffffffu, sr, 4 * g + 3);
      fence_proxy_async_smem();
      __syncwarp();
      if (lane < 8) {
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile::scatter4.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];"
                     ::"l"(reinterpret_cast<uint64_t>(&tmO)), "r"(smem_u32(rb + b * RB_BYTES + g * 512)), "r"(col),
                     "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                     : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    };
    auto buffer_read = [&]() {  // this warp's stores have read their smem
      if (lane < 8) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
    };
    constexpr int NCH = (BN / 2) / 32;  // chunks per tile half
    static_assert(kRB >= 2 && kRB <= NCH, "EPI 3 buffer count");
    int lr, sr, z;
    rows_of(cid, lr, sr, z);
    int it = 0, gc = 0;  // gc: chunks completed by this warp (buffer gc % kRB)
    for (int c = 0; c < kRB; ++c) gather(cid, 32 * c, lr, c);
    for (int t = cid; t < num_tiles; t += ncl, ++it) {
      const int as = it & 1;
      int nlr, nsr, nz;
      rows_of(t + ncl, nlr, nsr, nz);
      if (nlr != kDeadRow) {  // L2 prefetch of the next tile's residual half row (the later chunks' gathers hit L2)
        const int pn0 = ((t + ncl) % n_tiles) * BN + chalf * (BN / 2);
        const int ncols = min(BN / 2, N - pn0);
        if (ncols > 0)
          asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(ep.res + (long long)nlr * ep.ld_res + pn0),
                       "r"(ncols * 4)
                       : "memory");
      }
      mbar_wait_sleep(&tfull[as], (it >> 1) & 1);
      tc_fence_after();
      const uint32_t trow = tmem_base + as * BN + ((uint32_t)(q * 32) << 16) + chalf * (BN / 2);
      const int nbase = (t % n_tiles) * BN + chalf * (BN / 2);
#pragma unroll 1
      for (int c = 0; c < NCH; ++c, ++gc) {
        const int b = gc % kRB;
        uint32_t r[32];
        __syncwarp();
        tmem_ld32(trow + 32 * c, r);
        tmem_ld_wait();
        if (c == NCH - 1) {  // accumulator drained: release it to the MMA warp
          tc_fence_before();
          if (leader)
            mbar_arrive(&tempty[as]);
          else
            mbar_arrive_remote(&tempty[as], 0);
        }
        mbar_wait(&rbar[b], (rphase >> b) & 1);
        rphase ^= 1u << b;
        const int nb = nbase + 32 * c;
        float4* row = reinterpret_cast<float4*>(rb + b * RB_BYTES + lane * 128);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          float4 bj = make_float4(0.f, 0.f, 0.f, 0.f);
          if (ep.bias && nb < N) bj = __ldg(reinterpret_cast<const float4*>(ep.bias + nb) + j);
          float4* p = row + (j ^ (lane & 7));
          float4 a = *p;
          if (z) {
            a = make_float4(0.f, 0.f, 0.f, 0.f);
          } else {
            a.x += __uint_as_float(r[4 * j]) + bj.x;
            a.y += __uint_as_float(r[4 * j + 1]) + bj.y;
            a.z += __uint_as_float(r[4 * j + 2]) + bj.z;
            a.w += __uint_as_float(r[4 * j + 3]) + bj.w;
          }
          *p = a;
        }
        scatter(t, 32 * c, sr, b);
        // refill: the buffer whose store has been read gets the chunk kRB after the one it held
        // (this tile's, or the next tile's first ones)
        const int tgt = c + kRB, fb = b;
        buffer_read();
        if (tgt < NCH)
          gather(t, 32 * tgt, lr, fb);
        else if (t + ncl < num_tiles)
          gather(t + ncl, 32 * (tgt - NCH), nlr, fb);
      }
      lr = nlr;
      sr = nsr;
      z = nz;
    }
    if (lane < 8) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
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
  // fp32 residual epilogue through TMA gather4 / scatter4 (EPI 3) for long-K GEMMs (fc2, K = 4C)
  // when both row arrays qualify (16-byte aligned base and row pitch).  Paired A/B on ViT-H
  // shapes (tools/gemm_ab.py): fc2 -3 to -8 %, but proj (K = C: a short mainloop per tile)
  // +9 to +32 % for every buffer / stage split tried, so short-K GEMMs keep the LSU epilogue.
  // Rows are addressed by coordinate, so the row extent is left open (2^30) and only
  // coordinates the kernel computes from row_map / M are ever touched.
  static const bool g2_lsu = getenv("ZS_G2_LSU") != nullptr;  // A/B: force the LSU residual epilogue
  static const bool g2_tma_all = getenv("ZS_G2_TMA_ALL") != nullptr;  // A/B: TMA epilogue at any K
  CUtensorMap tr = ta, to = ta;
  if (epi == 2 && (K >= 2560 || g2_tma_all) && ep.res && ep.out && !(reinterpret_cast<uintptr_t>(ep.res) & 15) &&
      !(reinterpret_cast<uintptr_t>(ep.out) & 15) && !(ep.ld_res & 3) && !(ep.ld_out & 3) && !g2_lsu &&
      make_tmap_2d_f32(&tr, ep.res, (uint64_t)N, 1ull << 30, (uint64_t)ep.ld_res, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B) == 0 &&
      make_tmap_2d_f32(&to, ep.out, (uint64_t)N, 1ull << 30, (uint64_t)ep.ld_out, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B) == 0)
    epi = 3;
  switch (epi) {
    case 0:
      cudaFuncSetAttribute(zs_gemm2_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      { zs_gemm2_kernel<0><<<grid, kThreads, SMEM_BYTES, stream>>>(ta, tb, tr, to, M, N, K, ep); count_launch(); }
      break;
    case 1:
      cudaFuncSetAttribute(zs_gemm2_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      { zs_gemm2_kernel<1><<<grid, kThreads, SMEM_BYTES, stream>>>(ta, tb, tr, to, M, N, K, ep); count_launch(); }
      break;
    case 2:
      cudaFuncSetAttribute(zs_gemm2_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
      { zs_gemm2_kernel<2><<<grid, kThreads, SMEM_BYTES, stream>>>(ta, tb, tr, to, M, N, K, ep); count_launch(); }
      break;
    case 3:
      cudaFuncSetAttribute(zs_gemm2_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM3_BYTES);
      { zs_gemm2_kernel<3><<<grid, kThreads, SMEM3_BYTES, stream>>>(ta, tb, tr, to, M, N, K, ep); count_launch(); }
      break;
    default:
      return ZS_ERR_ARG;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

}  // namespace zs

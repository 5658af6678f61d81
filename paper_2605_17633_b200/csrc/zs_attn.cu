// zs_attn.cu — static block-sparse stripe-sort ("A-shape") attention on tcgen05.
//
// Semantics (attention.py:88-104, :167-221): inputs are already in scan (σ)
// order; query tile i (b_row rows) visits key tiles
//     J_i = {0 .. prefix-1} ∪ {min(i, Tc-1)}
// and computes softmax(tau * q k^T + bh[σq(q), σk(k)/w] + bw[σq(q), σk(k)%w]) v
// over exactly those columns (columns past Sk are excluded).
//
// B200 mapping.  One CTA owns 128 query rows of one (unit, head) and streams
// 128-key chunks; a chunk is visited only if some (query tile, key tile) pair
// inside it is active, and the exact 32/128-granular pattern is applied as a
// -inf mask — the schedule is the closed form above, never a dense mask.
//   warp 0      TMA: Q once, then K/V chunks into a 2-stage ring (3-D tensor
//               maps [units, S, cols]; rows past S are zero-filled by TMA)
//   warp 1      tcgen05.mma issue:  S_t = Q K_t^T      (128x128xdh, TMEM, 2 buffers)
//                                    O  += P_t V_t      (128xdh x128, TMEM accumulator)
//   warp 2      TMEM allocation (512 columns)
//   warps 4..7  softmax: one query row per thread — tcgen05.ld of S, tau scale,
//               decomposed-bias gather from smem, static mask, online max /
//               rescale, P (bf16) to smem in the UMMA 128B-swizzled K-major
//               layout; when the running max moves, the O accumulator is
//               rescaled in TMEM (ld/scale/st) before the next PV MMA.
// dh = 80 (ViT-H) is handled as a 64-column 128B-swizzle slab plus a 16-column
// 32B-swizzle slab: QK^T runs 4+1 K-steps, PV runs an N=64 and an N=16 MMA
// against V consumed MN-major straight from its TMA layout.
#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {

namespace attn {
constexpr int BQ = 128;   // query rows per CTA (UMMA M)
constexpr int BKC = 128;  // keys per chunk (UMMA N of QK^T, K of PV)
constexpr int kThreads = 256;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t TM_S = 0;     // S buffers at columns [0,128) and [128,256)
constexpr uint32_t TM_O = 256;   // O accumulator at [256, 256+dh)

struct Params {
  int units, heads, sq, sk, bias_w;
  long long ldo, o_unit_stride;
  const float* bh;
  const float* bw;
  const int* q_sp;
  const int* k_sp;
  int b_row, b_col, prefix, tc;
  float tau;
  __nv_bfloat16* out;
};

template <int DH>
struct Layout {
  static constexpr bool kTail = DH == 80;
  static constexpr int MAIN = BQ * 128;                // 64 bf16 x 128 rows, SW128
  static constexpr int TAIL = kTail ? BQ * 32 : 0;     // 16 bf16 x 128 rows, SW32
  static constexpr int TILE = MAIN + TAIL;             // one Q / K / V tile
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + ((TILE + 1023) / 1024) * 1024;
  static constexpr int KV_STRIDE = ((TILE + 1023) / 1024) * 1024;
  static constexpr int OFF_V = OFF_K + 2 * KV_STRIDE;
  static constexpr int OFF_P = OFF_V + 2 * KV_STRIDE;  // 2 atoms x 128 rows x 128 B
  static constexpr int OFF_KINFO = OFF_P + 2 * BQ * 128;
  static constexpr int OFF_BAR = OFF_KINFO + 2 * BKC * 4;
  static constexpr int OFF_BIAS = OFF_BAR + 256;
  static constexpr int TX_Q = BQ * DH * 2;
  static constexpr int TX_KV = 2 * BKC * DH * 2;
  static size_t smem_bytes(int bias_w) { return 1024 + OFF_BIAS + (size_t)2 * BQ * (bias_w + 1) * 4; }
};

struct ChunkPlan {
  int nck, p, tc, bcol, dlo, dhi;
  __device__ __forceinline__ bool needed(int cj) const {
    const int kt_lo = (cj * BKC) / bcol;
    if (kt_lo < p) return true;
    int kt_hi = (cj * BKC + BKC - 1) / bcol;
    if (kt_hi > tc - 1) kt_hi = tc - 1;
    return !(dhi < kt_lo || dlo > kt_hi);
  }
};
}  // namespace attn

template <int DH>
__global__ void __launch_bounds__(attn::kThreads, 1)
    zs_attn_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tq2,
                   const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tk2,
                   const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tv2,
                   attn::Params P) {
  using namespace attn;
  using L = Layout<DH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bar + 0;
  uint64_t* kv_full = bar + 1;    // [2]
  uint64_t* kv_empty = bar + 3;   // [2]
  uint64_t* s_full = bar + 5;     // [2]
  uint64_t* s_empty = bar + 7;    // [2]
  uint64_t* p_full = bar + 9;
  uint64_t* pv_full = bar + 10;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 16);
  uint32_t* kinfo = reinterpret_cast<uint32_t*>(smem + L::OFF_KINFO);  // [2][BKC]
  float* bias_h = reinterpret_cast<float*>(smem + L::OFF_BIAS);
  const int W1 = P.bias_w + 1;
  float* bias_w = bias_h + BQ * W1;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid: x = query block, y = head, z = unit
  const int mb = blockIdx.x, h = blockIdx.y, u = blockIdx.z;
  const int row0 = mb * BQ;

  ChunkPlan plan;
  plan.nck = (P.sk + BKC - 1) / BKC;
  plan.p = P.prefix;
  plan.tc = P.tc;
  plan.bcol = P.b_col;
  {
    const int qt_lo = row0 / P.b_row;
    const int qt_hi = min(row0 + BQ - 1, P.sq - 1) / P.b_row;
    plan.dlo = min(qt_lo, P.tc - 1);
    plan.dhi = min(qt_hi, P.tc - 1);
  }

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    mbar_init(q_full, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], 128);
    }
    mbar_init(pv_full, 1);
    mbar_init(p_full, 128);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sP = smem + L::OFF_P;
  const int col = h * DH;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      mbar_expect_tx(q_full, L::TX_Q);
      tma_load_3d(sQ, &tq, q_full, col, row0, u);
      if constexpr (L::kTail) tma_load_3d(sQ + L::MAIN, &tq2, q_full, col + 64, row0, u);
      int t = 0;
      for (int cj = 0; cj < plan.nck; ++cj) {
        if (!plan.needed(cj)) continue;
        const int st = t & 1;
        mbar_wait(&kv_empty[st], ((t >> 1) & 1) ^ 1);
        mbar_expect_tx(&kv_full[st], L::TX_KV);
        uint8_t* k = sK + st * L::KV_STRIDE;
        uint8_t* v = sV + st * L::KV_STRIDE;
        tma_load_3d(k, &tk, &kv_full[st], col, cj * BKC, u);
        tma_load_3d(v, &tv, &kv_full[st], col, cj * BKC, u);
        if constexpr (L::kTail) {
          tma_load_3d(k + L::MAIN, &tk2, &kv_full[st], col + 64, cj * BKC, u);
          tma_load_3d(v + L::MAIN, &tv2, &kv_full[st], col + 64, cj * BKC, u);
        }
        ++t;
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t id_s = idesc_bf16(BQ, BKC);
    constexpr uint32_t id_pv = idesc_bf16(BQ, 64, false, true);
    constexpr uint32_t id_pv2 = idesc_bf16(BQ, 16, false, true);
    auto issue_pv = [&](int j) {
      const int sj = j & 1;
      mbar_wait(p_full, j & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t d = tmem + TM_O;
        uint8_t* v = sV + sj * L::KV_STRIDE;
#pragma unroll
        for (int ks = 0; ks < BKC / 16; ++ks) {
          const uint64_t a = sdesc_k_sw128(sP + (ks >> 2) * (BQ * 128)) + 2 * (ks & 3);
          const uint32_t acc = (j > 0 || ks > 0) ? 1u : 0u;
          umma_bf16(d, a, sdesc_mn_sw128(v + ks * 16 * 128), id_pv, acc);
          if constexpr (L::kTail) umma_bf16(d + 64, a, sdesc_mn_sw32(v + L::MAIN + ks * 16 * 32), id_pv2, acc);
        }
        umma_commit(pv_full);
        umma_commit(&kv_empty[sj]);
      }
      __syncwarp();
    };
    mbar_wait(q_full, 0);
    int t = 0;
    for (int cj = 0; cj < plan.nck; ++cj) {
      if (!plan.needed(cj)) continue;
      const int st = t & 1;
      mbar_wait(&kv_full[st], (t >> 1) & 1);
      mbar_wait(&s_empty[st], ((t >> 1) & 1) ^ 1);
      tc_fence_after();
      if (lane == 0) {
        uint8_t* k = sK + st * L::KV_STRIDE;
        const uint32_t d = tmem + TM_S + st * 128;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_bf16(d, sdesc_k_sw128(sQ) + 2 * ks, sdesc_k_sw128(k) + 2 * ks, id_s, ks > 0);
        if constexpr (L::kTail) umma_bf16(d, sdesc_k_sw32(sQ + L::MAIN), sdesc_k_sw32(k + L::MAIN), id_s, 1);
        umma_commit(&s_full[st]);
      }
      __syncwarp();
      if (t > 0) issue_pv(t - 1);
      ++t;
    }
    issue_pv(t - 1);
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;  // row within the CTA tile == TMEM lane
    const int row = row0 + r;
    const bool valid = row < P.sq;
    const long long qsp_base = (long long)u * P.sq;
    const int sp = P.q_sp[qsp_base + (valid ? row : P.sq - 1)];
    {
      const float* th = P.bh + ((long long)h * P.sq + sp) * P.bias_w;
      const float* tw = P.bw + ((long long)h * P.sq + sp) * P.bias_w;
      for (int k = 0; k < P.bias_w; ++k) {
        bias_h[r * W1 + k] = __ldg(th + k);
        bias_w[r * W1 + k] = __ldg(tw + k);
      }
    }
    const float* bh_row = bias_h + r * W1;
    const float* bw_row = bias_w + r * W1;
    const int diag = min(row / P.b_row, P.tc - 1);
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    constexpr float L2E = 1.4426950408889634f;

    const uint32_t o_addr = tmem + TM_O + lane_off;
    float m_run = -INFINITY, ell = 0.f;
    int t = 0;
    for (int cj = 0; cj < plan.nck; ++cj) {
      if (!plan.needed(cj)) continue;
      const int st = t & 1;
      // key metadata for this chunk (one column per thread)
      {
        const int kg = cj * BKC + r;
        uint32_t info = 0xFFFFu << 16;
        if (kg < P.sk) {
          const int ksp = P.k_sp[(long long)u * P.sk + kg];
          info = (uint32_t)(ksp / P.bias_w) | ((uint32_t)(ksp % P.bias_w) << 8) | ((uint32_t)(kg / P.b_col) << 16);
        }
        kinfo[st * BKC + r] = info;
      }
      named_bar_sync(1, 128);
      const uint32_t* ki = kinfo + st * BKC;

      mbar_wait(&s_full[st], (t >> 1) & 1);
      tc_fence_after();
      const uint32_t s_addr = tmem + TM_S + st * 128 + lane_off;
      // pass 1: logits = tau*s + bh + bw (masked), written back over S in TMEM; row max
      float mx = -INFINITY;
#pragma unroll 1
      for (int cc = 0; cc < BKC / 32; ++cc) {
        uint32_t sr[32];
        tmem_ld32(s_addr + cc * 32, sr);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          const uint32_t info = ki[cc * 32 + j];
          const int kt = (int)(info >> 16);
          const bool ok = (kt < plan.p) || (kt == diag);
          float x = __fmul_rn(P.tau, __uint_as_float(sr[j]));
          x = __fadd_rn(x, bh_row[info & 255u]);
          x = __fadd_rn(x, bw_row[(info >> 8) & 255u]);
          x = ok ? x : -INFINITY;
          mx = fmaxf(mx, x);
          sr[j] = __float_as_uint(x);
        }
        tmem_st32(s_addr + cc * 32, sr);
      }
      tmem_st_wait();

      const float m_new = fmaxf(m_run, mx);
      const float m_use = (m_new == -INFINITY) ? 0.f : m_new;
      const float alpha = exp2f((m_run - m_use) * L2E);  // m_run = -inf -> 0
      const float mb2 = m_use * L2E;
      if (t > 0) {
        // PV_{t-1} done: O is current and the P buffer is free
        mbar_wait(pv_full, (t - 1) & 1);
        tc_fence_after();
        if (__any_sync(0xffffffffu, alpha != 1.0f)) {
#pragma unroll
          for (int c0 = 0; c0 < 64; c0 += 32) {
            uint32_t pr[32];
            tmem_ld32(o_addr + c0, pr);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 32; ++j) pr[j] = __float_as_uint(__uint_as_float(pr[j]) * alpha);
            tmem_st32(o_addr + c0, pr);
          }
          if constexpr (DH == 80) {
            uint32_t pr[16];
            tmem_ld16(o_addr + 64, pr);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) pr[j] = __float_as_uint(__uint_as_float(pr[j]) * alpha);
            tmem_st16(o_addr + 64, pr);
          }
          tmem_st_wait();
        }
      }
      // pass 2: p = exp(logit - m), row sum, P (bf16) -> smem in the UMMA K-major
      // 128B-swizzled layout: atom a = key/64, 16-byte chunk (key%64)/8 ^ (row%8)
      float rs = 0.f;
#pragma unroll 1
      for (int cc = 0; cc < BKC / 32; ++cc) {
        uint32_t sr[32];
        tmem_ld32(s_addr + cc * 32, sr);
        tmem_ld_wait();
        float pj[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          pj[j] = exp2f(fmaf(__uint_as_float(sr[j]), L2E, -mb2));
          rs += pj[j];
        }
#pragma unroll
        for (int q8 = 0; q8 < 4; ++q8) {
          uint4 w;
          w.x = pack_bf16(pj[8 * q8 + 0], pj[8 * q8 + 1]);
          w.y = pack_bf16(pj[8 * q8 + 2], pj[8 * q8 + 3]);
          w.z = pack_bf16(pj[8 * q8 + 4], pj[8 * q8 + 5]);
          w.w = pack_bf16(pj[8 * q8 + 6], pj[8 * q8 + 7]);
          const int g8 = cc * 4 + q8;
          const int a = g8 >> 3, c16 = (g8 & 7) ^ (r & 7);
          *reinterpret_cast<uint4*>(sP + a * (BQ * 128) + r * 128 + c16 * 16) = w;
        }
      }
      tc_fence_before();
      mbar_arrive(&s_empty[st]);
      ell = ell * alpha + rs;
      m_run = m_new;
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(p_full);
      ++t;
    }
    // epilogue: O / ell -> bf16 -> global
    mbar_wait(pv_full, (t - 1) & 1);
    tc_fence_after();
    const float inv = 1.0f / ell;
    uint4* dst = reinterpret_cast<uint4*>(P.out + (long long)u * P.o_unit_stride + (long long)row * P.ldo + col);
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 32) {
      uint32_t pr[32];
      tmem_ld32(o_addr + c0, pr);
      tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(pr[8 * j + 0]) * inv, __uint_as_float(pr[8 * j + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(pr[8 * j + 2]) * inv, __uint_as_float(pr[8 * j + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(pr[8 * j + 4]) * inv, __uint_as_float(pr[8 * j + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(pr[8 * j + 6]) * inv, __uint_as_float(pr[8 * j + 7]) * inv);
          dst[c0 / 8 + j] = w;
        }
      }
    }
    if constexpr (DH == 80) {
      uint32_t pr[16];
      tmem_ld16(o_addr + 64, pr);
      tmem_ld_wait();
      if (valid) {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          uint4 w;
          w.x = pack_bf16(__uint_as_float(pr[8 * j + 0]) * inv, __uint_as_float(pr[8 * j + 1]) * inv);
          w.y = pack_bf16(__uint_as_float(pr[8 * j + 2]) * inv, __uint_as_float(pr[8 * j + 3]) * inv);
          w.z = pack_bf16(__uint_as_float(pr[8 * j + 4]) * inv, __uint_as_float(pr[8 * j + 5]) * inv);
          w.w = pack_bf16(__uint_as_float(pr[8 * j + 6]) * inv, __uint_as_float(pr[8 * j + 7]) * inv);
          dst[8 + j] = w;
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace zs

using namespace zs;

template <int DH>
static int launch_attn(const void* q, const void* k, const void* v, long long ldq, long long ldk, long long ldv,
                       long long qus, long long kvus, const attn::Params& p, cudaStream_t st) {
  using L = attn::Layout<DH>;
  CUtensorMap m[6];
  const uint64_t ncol = (uint64_t)p.heads * DH;
  int rc = 0;
  rc |= make_tmap_3d_bf16(&m[0], q, ncol, p.sq, p.units, ldq, qus, 64, attn::BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  rc |= make_tmap_3d_bf16(&m[2], k, ncol, p.sk, p.units, ldk, kvus, 64, attn::BKC, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  rc |= make_tmap_3d_bf16(&m[4], v, ncol, p.sk, p.units, ldv, kvus, 64, attn::BKC, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  if (L::kTail) {
    rc |= make_tmap_3d_bf16(&m[1], q, ncol, p.sq, p.units, ldq, qus, 16, attn::BQ, 1, CU_TENSOR_MAP_SWIZZLE_32B);
    rc |= make_tmap_3d_bf16(&m[3], k, ncol, p.sk, p.units, ldk, kvus, 16, attn::BKC, 1, CU_TENSOR_MAP_SWIZZLE_32B);
    rc |= make_tmap_3d_bf16(&m[5], v, ncol, p.sk, p.units, ldv, kvus, 16, attn::BKC, 1, CU_TENSOR_MAP_SWIZZLE_32B);
  } else {
    m[1] = m[0];
    m[3] = m[2];
    m[5] = m[4];
  }
  if (rc) return ZS_ERR_TMAP;
  const size_t smem = L::smem_bytes(p.bias_w);
  if (smem > 227 * 1024) return ZS_ERR_SHAPE;
  cudaFuncSetAttribute(zs_attn_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  dim3 grid((p.sq + attn::BQ - 1) / attn::BQ, p.heads, p.units);
  zs_attn_kernel<DH><<<grid, attn::kThreads, smem, st>>>(m[0], m[1], m[2], m[3], m[4], m[5], p);
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

extern "C" int zs_stripe_attn_fwd(const void* q, const void* k, const void* v, long long ldq, long long ldk,
                                  long long ldv, long long q_unit_stride, long long kv_unit_stride, int units,
                                  int heads, int sq, int sk, int dh, const float* bh, const float* bw, int bias_w,
                                  const int32_t* q_sp, const int32_t* k_sp, int b_row, int b_col,
                                  int prefix_tiles, float tau, void* out, long long ldo, long long o_unit_stride,
                                  zs_stream_t stream) {
  if (units <= 0 || heads <= 0) return 0;
  if (!q || !k || !v || !bh || !bw || !q_sp || !k_sp || !out) return ZS_ERR_ARG;
  if (sq <= 0 || sk <= 0 || b_row <= 0 || b_col <= 0 || bias_w <= 0 || bias_w > 255) return ZS_ERR_SHAPE;
  if (bias_w * bias_w != sk) return ZS_ERR_SHAPE;
  if (dh != 64 && dh != 80) return ZS_ERR_SHAPE;
  const int tc = (sk + b_col - 1) / b_col;
  if (prefix_tiles < 0 || prefix_tiles > tc || tc >= 65535) return ZS_ERR_SHAPE;
  if ((ldq | ldk | ldv | ldo | q_unit_stride | kv_unit_stride | o_unit_stride) & 7) return ZS_ERR_ALIGN;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
       reinterpret_cast<uintptr_t>(out)) & 15)
    return ZS_ERR_ALIGN;
  attn::Params p;
  p.units = units;
  p.heads = heads;
  p.sq = sq;
  p.sk = sk;
  p.bias_w = bias_w;
  p.ldo = ldo;
  p.o_unit_stride = o_unit_stride;
  p.bh = bh;
  p.bw = bw;
  p.q_sp = q_sp;
  p.k_sp = k_sp;
  p.b_row = b_row;
  p.b_col = b_col;
  p.prefix = prefix_tiles;
  p.tc = tc;
  p.tau = tau;
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (dh == 64) return launch_attn<64>(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, p, st);
  return launch_attn<80>(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, p, st);
}

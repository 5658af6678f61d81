// zs_attn_local.cu — stripe-sort attention for short sequences (S <= 256: SAM windows, 196 tokens).
//
// Same semantics as zs_attn.cu (attention.py:88-104, :167-221).  A work item is a
// whole (unit, head): query tile A = rows [0,128), tile B = rows [128, S).  Each
// tile has its own softmax warpgroup (one thread per query row, full 128-key
// chunks, no cross-thread exchange) and its own MMA-issuer warp, so the two
// tiles ping-pong: while one warpgroup waits on the tensor core the other
// computes.  K and V of the item live in two chunk slots each (keys [0,128) and
// [128,256)) shared by both tiles; a slot is refilled for the next item as soon
// as both tiles have consumed it.
//   warp 0       TMA: lane 0 streams K/V chunk slots, lanes 1/2 stream Q_A / Q_B
//   warp 1 / 2   tcgen05.mma issue for tile A / tile B (warp 2 also owns TMEM):
//                S_X = Q_X K_j^T (TMEM cols X*128), O_X += P_X V_j (TMEM cols 256+X*128)
//   warp 3       per item, byte offsets of bh[., σk/w] and bw[., σk%w] for every key
//   warps 4-7    softmax tile A        warps 8-11   softmax tile B
// Bias rows are staged per thread (its own row only), the next item's rows are
// prefetched right after the last pass 1 of the current item.  P goes through
// smem in the UMMA 128B-swizzled K-major layout; the O accumulator stays in TMEM
// with lazy (thresholded) rescaling.
#include <algorithm>

#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {
namespace attnl {

constexpr int BQ = 128, BKC = 128;
constexpr int kThreads = 384;
constexpr uint32_t kTmemCols = 512;

struct Params {
  int units, heads, sq, sk, bias_w;
  long long ldo, o_unit_stride;
  const int* o_rows;  // optional: output row of (unit, query row), -1 = not written
  const float* bh;
  long long bias_us;  // floats between the bh / bw tables of consecutive units (0: shared)
  const float* bw;
  const int* q_sp;
  const int* k_sp;
  int b_row, b_col, prefix, tc, items;
  float tau;
  unsigned mask[2];  // needed-chunk bitmask of tile A / tile B (bit j = key chunk j)
  int fast;          // b_row, b_col multiples of 32 -> per-32-key-group mask
  __nv_bfloat16* out;
};

template <int DH>
struct Layout {
  static constexpr bool kTail = DH == 80;
  static constexpr int MAIN = BQ * 128;
  static constexpr int TAIL = kTail ? BQ * 32 : 0;
  static constexpr int TILE = ((MAIN + TAIL + 1023) / 1024) * 1024;
  static constexpr int OFF_Q = 0;                       // [2 tiles]
  static constexpr int OFF_K = OFF_Q + 2 * TILE;        // [2 chunk slots]
  static constexpr int OFF_V = OFF_K + 2 * TILE;        // [2 chunk slots]
  static constexpr int OFF_P = OFF_V + 2 * TILE;        // [2 tiles] x 32 KB
  static constexpr int OFF_KOFF = OFF_P + 2 * BQ * 256; // [2 item parity][256 keys] int2
  static constexpr int OFF_BAR = OFF_KOFF + 2 * 256 * 8;
  static constexpr int OFF_BIAS = OFF_BAR + 512;        // [2 tiles][BQ rows][2 tables][w+1]
  static constexpr int TX_TILE = BQ * DH * 2;
  static size_t smem_bytes(int w) { return 1024 + OFF_BIAS + (size_t)2 * BQ * 2 * (w + 1) * 4; }
};

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ void wait_sleep(uint64_t* bar, uint32_t parity) { mbar_wait_sleep(bar, parity); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint4 scale_pack8(const uint32_t* v, float s) {
  uint4 w;
  w.x = pack_bf16(__uint_as_float(v[0]) * s, __uint_as_float(v[1]) * s);
  w.y = pack_bf16(__uint_as_float(v[2]) * s, __uint_as_float(v[3]) * s);
  w.z = pack_bf16(__uint_as_float(v[4]) * s, __uint_as_float(v[5]) * s);
  w.w = pack_bf16(__uint_as_float(v[6]) * s, __uint_as_float(v[7]) * s);
  return w;
}

}  // namespace attnl

template <int DH>
__global__ void __launch_bounds__(attnl::kThreads, 1)
    zs_attn_local_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tq2,
                         const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tk2,
                         const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tv2,
                         attnl::Params P) {
  using namespace attnl;
  using L = Layout<DH>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bar + 0;    // [tile]
  uint64_t* q_empty = bar + 2;   // [tile]
  uint64_t* k_full = bar + 4;    // [slot]
  uint64_t* k_empty = bar + 6;   // [slot]  (2 arrivals: both MMA warps)
  uint64_t* v_full = bar + 8;    // [slot]
  uint64_t* v_empty = bar + 10;  // [slot]  (2 arrivals)
  uint64_t* s_full = bar + 12;   // [tile]
  uint64_t* p_full = bar + 14;   // [tile]  (128 arrivals: the tile's softmax threads; also frees S_X)
  uint64_t* o_full = bar + 16;   // [tile]  (PV of the tile completed)
  uint64_t* ki_full = bar + 18;  // [item parity] (32 arrivals)
  uint64_t* ki_empty = bar + 20; // [item parity] (256 arrivals)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 24);

  // warp index via shfl: provably warp-uniform, so role code can use uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int nck = (P.sk + BKC - 1) / BKC;     // 1 or 2 key chunks
  const bool has_b = P.sq > BQ;
  const unsigned mask_a = P.mask[0], mask_b = has_b ? P.mask[1] : 0u;
  // tiles using key chunk slot j: the release barriers count exactly these (static plan)
  auto users = [&](int j) { return (int)((mask_a >> j) & 1u) + (int)((mask_b >> j) & 1u); };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], users(s) > 0 ? users(s) : 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], users(s) > 0 ? users(s) : 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[s], 128);
      mbar_init(&o_full[s], 1);
      mbar_init(&ki_full[s], 32);
      mbar_init(&ki_empty[s], 256);
    }
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
  int2* koff = reinterpret_cast<int2*>(smem + L::OFF_KOFF);

  if (warp == 0) {
    // ------------------------------------------------------------ TMA: lane 0 K/V, lanes 1-2 Q_A / Q_B
    if (lane == 0) {
      int k = 0;
      for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
        const int u = it / P.heads, h = it % P.heads, col = h * DH;
        for (int j = 0; j < nck; ++j) {
          if (users(j) == 0) continue;
          wait_sleep(&k_empty[j], (k & 1) ^ 1);
          mbar_expect_tx(&k_full[j], BKC * DH * 2);
          uint8_t* kk = sK + j * L::TILE;
          tma_load_3d(kk, &tk, &k_full[j], col, j * BKC, u);
          if constexpr (L::kTail) tma_load_3d(kk + L::MAIN, &tk2, &k_full[j], col + 64, j * BKC, u);
          wait_sleep(&v_empty[j], (k & 1) ^ 1);
          mbar_expect_tx(&v_full[j], BKC * DH * 2);
          uint8_t* vv = sV + j * L::TILE;
          tma_load_3d(vv, &tv, &v_full[j], col, j * BKC, u);
          if constexpr (L::kTail) tma_load_3d(vv + L::MAIN, &tv2, &v_full[j], col + 64, j * BKC, u);
        }
      }
    } else if (lane == 1 || (lane == 2 && has_b)) {
      const int X = lane - 1;
      int k = 0;
      for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
        const int u = it / P.heads, h = it % P.heads, col = h * DH;
        wait_sleep(&q_empty[X], (k & 1) ^ 1);
        mbar_expect_tx(&q_full[X], L::TX_TILE);
        uint8_t* q = sQ + X * L::TILE;
        tma_load_3d(q, &tq, &q_full[X], col, X * BQ, u);
        if constexpr (L::kTail) tma_load_3d(q + L::MAIN, &tq2, &q_full[X], col + 64, X * BQ, u);
      }
    }
  } else if (warp == 1 || warp == 2) {
    // ------------------------------------------------------------ MMA issue, tile X
    const int X = warp - 1;
    constexpr uint32_t id_s = idesc_bf16(BQ, BKC);
    constexpr uint32_t id_pv = idesc_bf16(BQ, 64, false, true);
    constexpr uint32_t id_pv2 = idesc_bf16(BQ, 16, false, true);
    const unsigned mask = X ? mask_b : mask_a;
    const int jlast = mask ? 31 - __clz(mask) : -1;
    const uint32_t dS = tmem + X * 128, dO = tmem + 256 + X * 128;
    uint8_t* q = sQ + X * L::TILE;
    uint8_t* p = sP + X * (BQ * 256);
    int k = 0, n = 0;  // n: chunks processed by this tile so far (phase of s_full / p_full / o_full)
    for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
      bool first = true;
      for (int j = 0; j < nck; ++j) {
        if (!((mask >> j) & 1u)) continue;  // slot release counts only the tiles that use it
        if (first) wait_sleep(&q_full[X], k & 1);
        wait_sleep(&k_full[j], k & 1);
        if (n > 0) wait_sleep(&p_full[X], (n - 1) & 1);  // softmax done with S of the previous chunk
        tc_fence_after();
        if (lane == 0) {
          uint8_t* kk = sK + j * L::TILE;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
            umma_bf16(dS, sdesc_k_sw128(q) + 2 * ks, sdesc_k_sw128(kk) + 2 * ks, id_s, ks > 0);
          if constexpr (L::kTail) umma_bf16(dS, sdesc_k_sw32(q + L::MAIN), sdesc_k_sw32(kk + L::MAIN), id_s, 1);
          umma_commit(&s_full[X]);
          umma_commit(&k_empty[j]);
          if (j == jlast) umma_commit(&q_empty[X]);
        }
        __syncwarp();
        // PV of this chunk once the softmax has written P
        wait_sleep(&p_full[X], n & 1);
        wait_sleep(&v_full[j], k & 1);
        tc_fence_after();
        if (lane == 0) {
          uint8_t* vv = sV + j * L::TILE;
#pragma unroll
          for (int ks = 0; ks < BKC / 16; ++ks) {
            const uint64_t a = sdesc_k_sw128(p + (ks >> 2) * (BQ * 128)) + 2 * (ks & 3);
            const uint32_t acc = (!first || ks > 0) ? 1u : 0u;
            umma_bf16(dO, a, sdesc_mn_sw128(vv + ks * 16 * 128), id_pv, acc);
            if constexpr (L::kTail) umma_bf16(dO + 64, a, sdesc_mn_sw32(vv + L::MAIN + ks * 16 * 32), id_pv2, acc);
          }
          umma_commit(&o_full[X]);
          umma_commit(&v_empty[j]);
        }
        __syncwarp();
        first = false;
        ++n;
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ key metadata (per item, all keys)
    int k = 0;
    for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
      const int u = it / P.heads;
      const int par = k & 1;
      int ksp[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int j = lane + 32 * i;
        ksp[i] = j < P.sk ? __ldg(P.k_sp + (long long)u * P.sk + j) : -1;
      }
      wait_sleep(&ki_empty[par], ((k >> 1) & 1) ^ 1);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        koff[par * 256 + lane + 32 * i] =
            ksp[i] >= 0 ? make_int2((ksp[i] / P.bias_w) * 4, (ksp[i] % P.bias_w) * 4) : make_int2(0, 0);
      mbar_arrive(&ki_full[par]);
    }
  } else {
    // ------------------------------------------------------------ softmax, tile X, one thread per row
    const int X = (warp - 4) >> 2;
    const int q4 = warp & 3;
    const int r = q4 * 32 + lane;
    const int row = X * BQ + r;  // row within the unit
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    const uint32_t s_addr = tmem + X * 128 + lane_off;
    const uint32_t o_addr = tmem + 256 + X * 128 + lane_off;
    uint8_t* p = sP + X * (BQ * 256);
    const int W1 = P.bias_w + 1;
    float* my_bias = reinterpret_cast<float*>(smem + L::OFF_BIAS) + (X * BQ + r) * 2 * W1;  // bh | bw
    const unsigned mask = X ? mask_b : mask_a;
    const int diag = min(min(row, P.sq - 1) / P.b_row, P.tc - 1);
    constexpr float L2E = 1.4426950408889634f;
    constexpr float kRescaleThr = 5.545177444479562f;  // ln 256

    auto stage_bias = [&](int it) {
      const int u = it / P.heads, h = it % P.heads;
      const int sp = P.q_sp[(long long)u * P.sq + min(row, P.sq - 1)];
      const long long bo = (long long)u * P.bias_us + ((long long)h * P.sq + sp) * P.bias_w;
      const float* sh = P.bh + bo;
      const float* sw = P.bw + bo;
      for (int j = 0; j < P.bias_w; ++j) {
        cp_async4(my_bias + j, sh + j);
        cp_async4(my_bias + W1 + j, sw + j);
      }
    };

    int k = 0, n = 0;
    if (mask && (int)blockIdx.x < P.items) stage_bias(blockIdx.x);
    for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
      const int par = k & 1;
      wait_sleep(&ki_full[par], (k >> 1) & 1);  // warps sleep while the other tile computes
      if (!mask) {
        mbar_arrive(&ki_empty[par]);
        continue;
      }
      const int u = it / P.heads, h = it % P.heads;
      cp_async_wait_all();
      const char* bh_row = reinterpret_cast<const char*>(my_bias);
      const char* bw_row = bh_row + W1 * 4;
      float m_ref = -INFINITY, ell = 0.f;
      bool first = true;
      int jl = 31 - __clz(mask);
      for (int j = 0; j < nck; ++j) {
        if (!((mask >> j) & 1u)) continue;
        const int2* ko = koff + par * 256 + j * BKC;
        mbar_wait(&s_full[X], n & 1);
        tc_fence_after();
        // pass 1: logits over the 128 keys of chunk j, written back to TMEM; row max
        float mx = -INFINITY;
        unsigned live = 0;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          const int c0 = j * BKC + g * 32;
          bool ok = c0 < P.sk;
          if (P.fast) {
            const int kt = c0 / P.b_col;
            ok = ok && ((kt < P.prefix) || (kt == diag));
          }
          if (__any_sync(0xffffffffu, ok)) {
            live |= 1u << g;
            uint32_t sr[32];
            tmem_ld32(s_addr + g * 32, sr);
            tmem_ld_wait();
            if (P.fast) {
#pragma unroll
              for (int jj = 0; jj < 32; jj += 2) {
                const int4 oo = *reinterpret_cast<const int4*>(ko + g * 32 + jj);
                float x0 = fmaf(P.tau, __uint_as_float(sr[jj]), *reinterpret_cast<const float*>(bh_row + oo.x));
                float x1 = fmaf(P.tau, __uint_as_float(sr[jj + 1]), *reinterpret_cast<const float*>(bh_row + oo.z));
                x0 += *reinterpret_cast<const float*>(bw_row + oo.y);
                x1 += *reinterpret_cast<const float*>(bw_row + oo.w);
                sr[jj] = __float_as_uint(x0);
                sr[jj + 1] = __float_as_uint(x1);
              }
              if (!ok || c0 + 32 > P.sk) {  // masked group (non-uniform rows) or ragged end
#pragma unroll
                for (int jj = 0; jj < 32; ++jj)
                  if (!ok || c0 + jj >= P.sk) sr[jj] = __float_as_uint(-INFINITY);
              }
            } else {
#pragma unroll
              for (int jj = 0; jj < 32; ++jj) {
                const int kg = c0 + jj;
                const int kt = kg / P.b_col;
                const bool okk = kg < P.sk && ((kt < P.prefix) || (kt == diag));
                const int2 oo = ko[g * 32 + jj];
                float x = fmaf(P.tau, __uint_as_float(sr[jj]), *reinterpret_cast<const float*>(bh_row + oo.x));
                x += *reinterpret_cast<const float*>(bw_row + oo.y);
                sr[jj] = __float_as_uint(okk ? x : -INFINITY);
              }
            }
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) mx = fmaxf(mx, __uint_as_float(sr[jj]));
            tmem_st32(s_addr + g * 32, sr);
          }
        }
        tmem_st_wait();
        if (j == jl) {  // bias of this item no longer needed: prefetch the next item's row
          const int nxt = it + gridDim.x;
          if (nxt < P.items) stage_bias(nxt);
        }
        // reference max moves only past the threshold (O rescaled once in TMEM)
        float alpha = 1.f;
        bool resc = false;
        if (mx > m_ref + kRescaleThr || (m_ref == -INFINITY && mx > -INFINITY)) {
          alpha = (m_ref == -INFINITY) ? 0.f : ex2((m_ref - mx) * L2E);
          resc = !first;
          m_ref = mx;
        }
        if (!first) {
          mbar_wait(&o_full[X], (n - 1) & 1);  // previous PV done: O current, P buffer free
          tc_fence_after();
        }
        if (__any_sync(0xffffffffu, resc)) {
#pragma unroll
          for (int c0 = 0; c0 < 64; c0 += 32) {
            uint32_t pr[32];
            tmem_ld32(o_addr + c0, pr);
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 32; ++jj) pr[jj] = __float_as_uint(__uint_as_float(pr[jj]) * alpha);
            tmem_st32(o_addr + c0, pr);
          }
          if constexpr (DH == 80) {
            uint32_t p16[16];
            tmem_ld16(o_addr + 64, p16);
            tmem_ld_wait();
#pragma unroll
            for (int jj = 0; jj < 16; ++jj) p16[jj] = __float_as_uint(__uint_as_float(p16[jj]) * alpha);
            tmem_st16(o_addr + 64, p16);
          }
          tmem_st_wait();
        }
        const float mb2 = (m_ref == -INFINITY) ? 0.f : m_ref * L2E;
        // pass 2: P = exp(logit - m_ref) (bf16) -> smem; row sum
        float rs = 0.f;
#pragma unroll
        for (int g = 0; g < 4; ++g) {
          uint4 w4[4];
          if (live & (1u << g)) {
            uint32_t sr[32];
            tmem_ld32(s_addr + g * 32, sr);
            tmem_ld_wait();
#pragma unroll
            for (int q8 = 0; q8 < 4; ++q8) {
              float pj[8];
#pragma unroll
              for (int jj = 0; jj < 8; ++jj) {
                pj[jj] = ex2(fmaf(__uint_as_float(sr[8 * q8 + jj]), L2E, -mb2));
                rs += pj[jj];
              }
              w4[q8].x = pack_bf16(pj[0], pj[1]);
              w4[q8].y = pack_bf16(pj[2], pj[3]);
              w4[q8].z = pack_bf16(pj[4], pj[5]);
              w4[q8].w = pack_bf16(pj[6], pj[7]);
            }
          } else {
#pragma unroll
            for (int q8 = 0; q8 < 4; ++q8) w4[q8] = make_uint4(0u, 0u, 0u, 0u);
          }
#pragma unroll
          for (int q8 = 0; q8 < 4; ++q8) {
            const int g8 = g * 4 + q8;  // 16-byte chunk along the 128 keys
            const int a = g8 >> 3, c16 = (g8 & 7) ^ (r & 7);
            *reinterpret_cast<uint4*>(p + a * (BQ * 128) + r * 128 + c16 * 16) = w4[q8];
          }
        }
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(&p_full[X]);
        ell = ell * alpha + rs;
        first = false;
        ++n;
      }
      mbar_arrive(&ki_empty[par]);
      // epilogue: O / ell -> bf16 -> global
      mbar_wait(&o_full[X], (n - 1) & 1);
      tc_fence_after();
      const float inv = 1.0f / ell;
      bool valid = row < P.sq;
      long long orow_off = (long long)u * P.o_unit_stride + (long long)row * P.ldo;
      if (valid && P.o_rows) {
        const int m = P.o_rows[(long long)u * P.sq + row];
        valid = m >= 0;
        orow_off = (long long)m * P.ldo;
      }
      __nv_bfloat16* dst = P.out + orow_off + h * DH;
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t pr[32];
        tmem_ld32(o_addr + c0, pr);
        tmem_ld_wait();
        if (valid) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + c0);
#pragma unroll
          for (int jj = 0; jj < 4; ++jj) d4[jj] = scale_pack8(pr + 8 * jj, inv);
        }
      }
      if constexpr (DH == 80) {
        uint32_t p16[16];
        tmem_ld16(o_addr + 64, p16);
        tmem_ld_wait();
        if (valid) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + 64);
          d4[0] = scale_pack8(p16, inv);
          d4[1] = scale_pack8(p16 + 8, inv);
        }
      }
      tc_fence_before();
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace zs

using namespace zs;

// Host launcher for S <= 256 (called by zs_stripe_attn_fwd in zs_attn.cu).
int launch_attn_local(const void* q, const void* k, const void* v, long long ldq, long long ldk, long long ldv,
                      long long qus, long long kvus, int units, int heads, int sq, int sk, int dh, const float* bh,
                      const float* bw, int bias_w, const int* q_sp, const int* k_sp, int b_row, int b_col,
                      int prefix, float tau, void* out, long long ldo, long long ous, const int* o_rows,
                      long long bias_us, cudaStream_t st) {
  attnl::Params p;
  p.bias_us = bias_us;
  p.units = units;
  p.heads = heads;
  p.sq = sq;
  p.sk = sk;
  p.bias_w = bias_w;
  p.ldo = ldo;
  p.o_unit_stride = ous;
  p.o_rows = o_rows;
  p.bh = bh;
  p.bw = bw;
  p.q_sp = q_sp;
  p.k_sp = k_sp;
  p.b_row = b_row;
  p.b_col = b_col;
  p.prefix = prefix;
  p.tc = (sk + b_col - 1) / b_col;
  p.items = units * heads;
  p.tau = tau;
  p.fast = (b_row % 32 == 0 && b_col % 32 == 0) ? 1 : 0;
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  // static chunk plan: chunk j is needed by tile X iff one of its (query tile, key tile) pairs is active
  const int nck = (sk + 127) / 128;
  for (int X = 0; X < 2; ++X) {
    unsigned m = 0;
    const int r0 = X * 128;
    if (r0 < sq) {
      const int qlo = r0 / b_row, qhi = std::min(r0 + 127, sq - 1) / b_row;
      const int dlo = std::min(qlo, p.tc - 1), dhi = std::min(qhi, p.tc - 1);
      for (int j = 0; j < nck; ++j) {
        const int klo = (j * 128) / b_col, khi = std::min((j * 128 + 127) / b_col, p.tc - 1);
        if (klo < prefix || !(dhi < klo || dlo > khi)) m |= 1u << j;
      }
    }
    p.mask[X] = m;
  }
  CUtensorMap m[6];
  const uint64_t ncol = (uint64_t)heads * dh;
  int rc = 0;
  rc |= make_tmap_3d_bf16(&m[0], q, ncol, sq, units, ldq, qus, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  rc |= make_tmap_3d_bf16(&m[2], k, ncol, sk, units, ldk, kvus, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  rc |= make_tmap_3d_bf16(&m[4], v, ncol, sk, units, ldv, kvus, 64, 128, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  if (dh == 80) {
    rc |= make_tmap_3d_bf16(&m[1], q, ncol, sq, units, ldq, qus, 16, 128, 1, CU_TENSOR_MAP_SWIZZLE_32B);
    rc |= make_tmap_3d_bf16(&m[3], k, ncol, sk, units, ldk, kvus, 16, 128, 1, CU_TENSOR_MAP_SWIZZLE_32B);
    rc |= make_tmap_3d_bf16(&m[5], v, ncol, sk, units, ldv, kvus, 16, 128, 1, CU_TENSOR_MAP_SWIZZLE_32B);
  } else {
    m[1] = m[0];
    m[3] = m[2];
    m[5] = m[4];
  }
  if (rc) return ZS_ERR_TMAP;
  int grid = num_sms();
  if (grid > p.items) grid = p.items;
  cudaError_t e;
  if (dh == 64) {
    const size_t smem = attnl::Layout<64>::smem_bytes(bias_w);
    if (smem > 227 * 1024) return ZS_ERR_SHAPE;
    cudaFuncSetAttribute(zs_attn_local_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    { zs_attn_local_kernel<64><<<grid, attnl::kThreads, smem, st>>>(m[0], m[1], m[2], m[3], m[4], m[5], p); count_launch(); }
  } else {
    const size_t smem = attnl::Layout<80>::smem_bytes(bias_w);
    if (smem > 227 * 1024) return ZS_ERR_SHAPE;
    cudaFuncSetAttribute(zs_attn_local_kernel<80>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    { zs_attn_local_kernel<80><<<grid, attnl::kThreads, smem, st>>>(m[0], m[1], m[2], m[3], m[4], m[5], p); count_launch(); }
  }
  e = cudaGetLastError();
  return e == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

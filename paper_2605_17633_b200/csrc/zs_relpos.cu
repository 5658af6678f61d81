// zs_relpos.cu — SAM decomposed relative-position bias computed from q.
//
// SAM (segment_anything image_encoder.py, add_decomposed_rel_pos) adds to the logits of query
// q at spatial (qy, qx) and key at (ky, kx) of a w x w grid
//     rel_h[q, ky] = q . rel_pos_h[qy - ky + w - 1],   rel_w[q, kx] = q . rel_pos_w[qx - kx + w - 1]
// with the UNSCALED q of each head; rel_pos_h / rel_pos_w are [2w - 1, dh] tables shared by
// the heads of a block.  In the reference's terms these are per-(unit, head) BiasTables
// (attention.py:28-55) bh[s, ky], bw[s, kx] indexed by the spatial position s = σq(row), which
// the reference only ever fills from static tables (parity unpinned: the fp32 torch twin in
// tests/test_gpu_relpos.py pins it).
//
// B200 design: the 2(2w-1) dot products of every (row, head) are ONE tcgen05 GEMM tile
// D[128 rows, NB] = Q[128, dh] . R^T with R = [rel_pos_h ; rel_pos_w] (bf16, K-major, resident
// in shared memory for the whole kernel), NB = 64 (w = 14) or 256 (w = 64) TMEM columns,
// one accumulator per epilogue warpgroup (4 for NB = 64, 2 otherwise).  The epilogue picks each row's w + w entries out of its 2(2w - 1)
// (a per-row shift by qy / qx: fp16 row staged in shared memory, read back at the row's
// offset) and writes
//   mode 0: the attention kernels' fp16 operand row  [bh/tau | 0 | bw/tau | 0]  (2 * ceil16(w)
//           halves) at btab[u * btab_us + (h * S + s) * W16]  (zs_attn_win.cu / zs_attn_glob.cu
//           consume it directly: no fp32 table round trip)
//   mode 1: fp32 bh, bw [units, heads, S, w] (reference BiasTables layout, unscaled)
// Roles: warp 0 TMA (Q tiles, 2-4 stage ring; R once), warp 1 MMA, warps 2.. epilogue
// warpgroups (TMEM lane quarter = warp % 4, one row per thread; WG e takes every NE-th tile).
#include <cuda_fp16.h>

#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {
namespace relpos {

constexpr int BM = 128;
// epilogue warpgroups (= TMEM accumulators; WG e takes the tiles k with k % NE == e) and
// Q-tile ring depth per accumulator width: the epilogue (row shift through shared memory)
// is the longer stage, so narrow tiles get more epilogue warpgroups
__host__ __device__ constexpr int n_epi(int nb) { return nb <= 64 ? 4 : 2; }
__host__ __device__ constexpr int n_stages(int nb) { return nb >= 256 ? 2 : 4; }
__host__ __device__ constexpr int n_threads(int nb) { return 64 + 128 * n_epi(nb); }
__host__ __device__ constexpr int tmem_cols(int nb) {
  return n_epi(nb) * nb <= 32 ? 32 : (n_epi(nb) * nb <= 64 ? 64 : (n_epi(nb) * nb <= 128 ? 128 : (n_epi(nb) * nb <= 256 ? 256 : 512)));
}

struct Params {
  int units, heads, S, w, nr, nrb, tiles;
  uint32_t w_magic;  // floor(2^32 / w) + 1: s / w == umulhi(s, w_magic) for s * w < 2^32
  const int* q_sp;
  float inv_tau;
  __half* btab;  // mode 0
  long long btab_us;
  int w16;       // halves per operand row (2 * ceil16(w))
  float* bh;     // mode 1
  float* bw;
  int off_b, off_bt, off_a, off_at, a_stage, off_stage, stage_words, off_bar;
  int tx_a, tx_b;
};

__global__ void relpos_table_kernel(const float* __restrict__ rh, const float* __restrict__ rw, int nr, int dh,
                                    int nb, __nv_bfloat16* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nb * dh) return;
  const int r = i / dh, c = i % dh;
  float v = 0.f;
  if (r < nr) v = rh[(long long)r * dh + c];
  else if (r < 2 * nr) v = rw[(long long)(r - nr) * dh + c];
  out[i] = __float2bfloat16_rn(v);
}

}  // namespace relpos

template <int DH, int NB, int MODE>
__global__ void __launch_bounds__(relpos::n_threads(NB), 1)
    zs_relpos_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tq_t,
                     const __grid_constant__ CUtensorMap tr, const __grid_constant__ CUtensorMap tr_t,
                     const relpos::Params P) {
  using namespace relpos;
  constexpr bool kTail = DH == 80;
  constexpr int NE = n_epi(NB), kStages = n_stages(NB), kCols = tmem_cols(NB);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + P.off_bar);
  uint64_t* a_full = bar;               // [kStages]
  uint64_t* a_empty = bar + kStages;    // [kStages]
  uint64_t* b_full = bar + 2 * kStages;
  uint64_t* acc_full = b_full + 1;        // [NE]
  uint64_t* acc_empty = b_full + 1 + NE;  // [NE]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(b_full + 1 + 2 * NE);
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&a_full[s], 1);
      mbar_init(&a_empty[s], 1);
    }
    mbar_init(b_full, 1);
    for (int s = 0; s < NE; ++s) {
      mbar_init(&acc_full[s], 1);
      mbar_init(&acc_empty[s], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(b_full, P.tx_b);
      tma_load_2d(smem + P.off_b, &tr, b_full, 0, 0);
      if constexpr (kTail) tma_load_2d(smem + P.off_bt, &tr_t, b_full, 64, 0);
      int k = 0;
      for (int t = blockIdx.x; t < P.tiles; t += gridDim.x, ++k) {
        const int h = t % P.heads, rb = (t / P.heads) % P.nrb, u = t / (P.heads * P.nrb);
        const int s = k % kStages;
        mbar_wait(&a_empty[s], ((k / kStages) & 1) ^ 1);
        mbar_expect_tx(&a_full[s], P.tx_a);
        uint8_t* a = smem + P.off_a + s * P.a_stage;
        tma_load_3d(a, &tq, &a_full[s], h * DH, rb * BM, u);
        if constexpr (kTail) tma_load_3d(a + (P.off_at - P.off_a), &tq_t, &a_full[s], h * DH + 64, rb * BM, u);
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t id = idesc_bf16(BM, NB);
    const uint64_t db = sdesc_k_sw128(smem + P.off_b), dbt = sdesc_k_sw32(smem + P.off_bt);
    const uint64_t da = sdesc_k_sw128(smem + P.off_a), dat = sdesc_k_sw32(smem + P.off_at);
    const uint32_t sd = (uint32_t)P.a_stage >> 4;
    mbar_wait(b_full, 0);
    int k = 0;
    for (int t = blockIdx.x; t < P.tiles; t += gridDim.x, ++k) {
      const int s = k % kStages, buf = k % NE;
      mbar_wait(&acc_empty[buf], ((k / NE) & 1) ^ 1);
      mbar_wait(&a_full[s], (k / kStages) & 1);
      tc_fence_after();
      const uint32_t d = tmem + buf * NB;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) umma_ss(d, da + s * sd + 2 * ks, db + 2 * ks, id, ks > 0);
      if constexpr (kTail) umma_ss(d, dat + s * sd, dbt, id, 1);
      umma_commit_elect(&a_empty[s]);
      umma_commit_elect(&acc_full[buf]);
    }
  } else {
    // ------------------------------------------------------------ epilogue: one row per thread
    const int qd = warp & 3, e = (warp - 2) >> 2;
    const uint32_t lane_off = (uint32_t)(qd * 32) << 16;
    uint32_t* stage = reinterpret_cast<uint32_t*>(smem + P.off_stage) + (e * BM + qd * 32 + lane) * P.stage_words;
    const __half* st16 = reinterpret_cast<const __half*>(stage);
    const int w = P.w, nr = P.nr;
    int j = 0;  // tiles taken by this warpgroup
    for (int t = blockIdx.x + e * gridDim.x; t < P.tiles; t += NE * gridDim.x, ++j) {
      const int h = t % P.heads, rb = (t / P.heads) % P.nrb, u = t / (P.heads * P.nrb);
      const int buf = e;
      const int row = rb * BM + qd * 32 + lane;
      const bool valid = row < P.S;
      const int s = valid ? __ldg(P.q_sp + (long long)u * P.S + row) : 0;
      const int qy = (int)__umulhi((uint32_t)s, P.w_magic), qx = s - qy * w;
      mbar_wait(&acc_full[buf], j & 1);
      tc_fence_after();
      const uint32_t acc = tmem + buf * NB + lane_off;
      if constexpr (MODE == 0) {
        // D row -> fp16 (scaled by 1/tau) in this thread's staging row
#pragma unroll
        for (int c = 0; c < NB / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(acc + c * 32, v);
          tmem_ld_wait();
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint4 o;
            __half2 h0 = __floats2half2_rn(__uint_as_float(v[8 * j]) * P.inv_tau, __uint_as_float(v[8 * j + 1]) * P.inv_tau);
            __half2 h1 = __floats2half2_rn(__uint_as_float(v[8 * j + 2]) * P.inv_tau, __uint_as_float(v[8 * j + 3]) * P.inv_tau);
            __half2 h2 = __floats2half2_rn(__uint_as_float(v[8 * j + 4]) * P.inv_tau, __uint_as_float(v[8 * j + 5]) * P.inv_tau);
            __half2 h3 = __floats2half2_rn(__uint_as_float(v[8 * j + 6]) * P.inv_tau, __uint_as_float(v[8 * j + 7]) * P.inv_tau);
            o.x = *reinterpret_cast<uint32_t*>(&h0);
            o.y = *reinterpret_cast<uint32_t*>(&h1);
            o.z = *reinterpret_cast<uint32_t*>(&h2);
            o.w = *reinterpret_cast<uint32_t*>(&h3);
            *reinterpret_cast<uint4*>(stage + c * 16 + 4 * j) = o;
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
        if (valid) {
          // operand row: [bh/tau (w) | 0 .. ceil16(w) | bw/tau (w) | 0 ..]; entry ky of bh is
          // D column qy - ky + w - 1, entry kx of bw is column nr + qx - kx + w - 1
          const int half16 = P.w16 >> 1;
          uint4* dst = reinterpret_cast<uint4*>(P.btab + (long long)u * P.btab_us + ((long long)h * P.S + s) * P.w16);
          for (int part = 0; part < 2; ++part) {
            const int base = part ? nr + qx + w - 1 : qy + w - 1;
            for (int j0 = 0; j0 < half16; j0 += 8) {
              uint32_t wv[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const int j = j0 + 2 * e;
                const __half a = j < w ? st16[base - j] : __float2half_rn(0.f);
                const __half b = j + 1 < w ? st16[base - j - 1] : __float2half_rn(0.f);
                __half2 hb = __halves2half2(a, b);
                wv[e] = *reinterpret_cast<uint32_t*>(&hb);
              }
              dst[(part * half16 + j0) >> 3] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            }
          }
        }
      } else {
        // fp32 reference-layout tables, unscaled: scatter each needed column straight out
        float* oh = P.bh + (((long long)u * P.heads + h) * P.S + s) * w;
        float* ow = P.bw + (((long long)u * P.heads + h) * P.S + s) * w;
#pragma unroll 1
        for (int c = 0; c < NB / 32; ++c) {
          uint32_t v[32];
          tmem_ld32(acc + c * 32, v);
          tmem_ld_wait();
          if (valid) {
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              const int col = c * 32 + j;
              const float x = __uint_as_float(v[j]);
              const int ky = qy + w - 1 - col;
              const int kx = qx + w - 1 - (col - nr);
              if (col < nr) {
                if (ky >= 0 && ky < w) oh[ky] = x;
              } else if (col < 2 * nr) {
                if (kx >= 0 && kx < w) ow[kx] = x;
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[buf]);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, kCols);
}

// Host launcher (internal).  mode 0 -> fp16 operand rows of w16 halves (bh/tau at [0, w),
// bw/tau at [w16/2, w16/2 + w)) into btab (unit stride btab_us halves); mode 1 -> fp32 bh / bw
// [units, heads, S, w].  ws: >= relpos_ws_r_bytes() bytes for
// the bf16 R table.  Returns 1 when the shape is outside the kernel (w > 64, dh not 64/80).
size_t relpos_r_bytes(int dh, int w) {
  const int nb = 2 * (2 * w - 1) <= 64 ? 64 : (2 * (2 * w - 1) <= 128 ? 128 : 256);
  return ((size_t)nb * dh * 2 + 255) & ~(size_t)255;
}

int launch_relpos(const void* q, long long ldq, long long qus, int units, int heads, int S, int dh, int w,
                  const float* rel_h, const float* rel_w, const int* q_sp, float tau, int mode, __half* btab,
                  long long btab_us, int w16, float* bh, float* bw, void* ws, cudaStream_t st) {
  using namespace relpos;
  if ((dh != 64 && dh != 80) || w < 1 || w > 64 || w * w != S || !(tau > 0.f)) return 1;
  if (mode == 0 && (w16 % 16 || w16 < 2 * ((w + 15) & ~15))) return 1;
  const int nr = 2 * w - 1;
  const int nb = 2 * nr <= 64 ? 64 : (2 * nr <= 128 ? 128 : 256);
  Params p{};
  p.units = units;
  p.heads = heads;
  p.S = S;
  p.w = w;
  p.nr = nr;
  p.nrb = (S + BM - 1) / BM;
  const long long tiles = (long long)units * heads * p.nrb;
  if (tiles > 0x7FFFFFFF) return ZS_ERR_SHAPE;
  p.tiles = (int)tiles;
  p.w_magic = (uint32_t)((1ull << 32) / (unsigned)w + 1ull);
  p.q_sp = q_sp;
  p.inv_tau = 1.0f / tau;
  p.btab = btab;
  p.btab_us = btab_us;
  p.w16 = w16;
  p.bh = bh;
  p.bw = bw;
  int off = 0;
  auto take = [&](int bytes, int align) {
    off = (off + align - 1) / align * align;
    const int o = off;
    off += bytes;
    return o;
  };
  p.off_b = take(nb * 128, 1024);
  p.off_bt = take(nb * 32, 1024);
  p.a_stage = (BM * 128 + BM * 32 + 1023) / 1024 * 1024;
  p.off_a = take(n_stages(nb) * p.a_stage, 1024);
  p.off_at = p.off_a + BM * 128;
  p.stage_words = mode == 0 ? nb / 2 + 4 : 0;
  p.off_stage = take(n_epi(nb) * BM * p.stage_words * 4, 16);
  p.off_bar = take(256, 8);
  const size_t smem = 1024 + (size_t)off;
  if (smem > 227 * 1024) return 1;
  p.tx_a = BM * dh * 2;
  p.tx_b = nb * dh * 2;
  __nv_bfloat16* R = reinterpret_cast<__nv_bfloat16*>(ws);
  { relpos_table_kernel<<<(nb * dh + 255) / 256, 256, 0, st>>>(rel_h, rel_w, nr, dh, nb, R); count_launch(); }
  CUtensorMap m[4];
  const uint64_t ncol = (uint64_t)heads * dh;
  int rc = 0;
  rc |= make_tmap_3d_bf16(&m[0], q, ncol, S, units, ldq, qus, 64, BM, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  rc |= make_tmap_2d_bf16(&m[2], R, dh, nb, dh, 64, nb, CU_TENSOR_MAP_SWIZZLE_128B);
  if (dh == 80) {
    rc |= make_tmap_3d_bf16(&m[1], q, ncol, S, units, ldq, qus, 16, BM, 1, CU_TENSOR_MAP_SWIZZLE_32B);
    rc |= make_tmap_2d_bf16(&m[3], R, dh, nb, dh, 16, nb, CU_TENSOR_MAP_SWIZZLE_32B);
  } else {
    m[1] = m[0];
    m[3] = m[2];
  }
  if (rc) return ZS_ERR_TMAP;
  int grid = num_sms();
  if (grid > p.tiles) grid = p.tiles;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    { kern<<<grid, n_threads(nb), smem, st>>>(m[0], m[1], m[2], m[3], p); count_launch(); }
  };
#define ZS_RELPOS_DISPATCH(D)                                                          \
  if (nb == 64) {                                                                      \
    if (mode == 0) launch(zs_relpos_kernel<D, 64, 0>);                                 \
    else launch(zs_relpos_kernel<D, 64, 1>);                                           \
  } else if (nb == 128) {                                                              \
    if (mode == 0) launch(zs_relpos_kernel<D, 128, 0>);                                \
    else launch(zs_relpos_kernel<D, 128, 1>);                                          \
  } else {                                                                             \
    if (mode == 0) launch(zs_relpos_kernel<D, 256, 0>);                                \
    else launch(zs_relpos_kernel<D, 256, 1>);                                          \
  }
  if (dh == 64) {
    ZS_RELPOS_DISPATCH(64)
  } else {
    ZS_RELPOS_DISPATCH(80)
  }
#undef ZS_RELPOS_DISPATCH
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

}  // namespace zs

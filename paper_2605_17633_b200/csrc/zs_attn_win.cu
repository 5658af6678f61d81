// zs_attn_win.cu — stripe-sort attention for SAM windows (S <= 256 tokens, e.g. 14x14 = 196).
//
// Same semantics as zs_attn.cu (attention.py:88-104 active set, :167-221 tiled softmax):
// query tile i (b_row rows) sees key tiles J_i = {0..p-1} ∪ {min(i, Tc-1)}, logits
// tau*q.k + bh[σq(q), σk(k)/w] + bw[σq(q), σk(k)%w], softmax over exactly those keys.
//
// B200 design (one persistent CTA per SM, work item = (unit, head)):
//  * Decomposed rel-pos bias on the tensor core.  Q is extended by 32 fp16 columns
//    [bh[σq(r)]/tau | bw[σq(r)]/tau] and K by the one-hot columns [e_ky | e_kx] of every key,
//    so one MMA chain produces S' = q.k + (bh + bw)/tau in fp32 and the softmax never gathers
//    bias values (logit = tau * S').  The bias columns are a separate fp16 MMA (kind::f16
//    accepts fp16 or bf16 per instruction), the q.k part stays bf16.
//  * A window has at most 256 rows = two 128-row MMA tiles (A: rows [0,128), B: [128,S)).
//    For every 32-row warp the static schedule gives the live 32-key groups (warp-uniform
//    when b_row, b_col are multiples of 32).  Each tile computes S only over the union of
//    its warps' live groups, packed into contiguous TMEM columns ("runs"), so a whole
//    softmax row sits in ONE S buffer: no online rescaling, one pass.
//  * P (bf16) is written back into the tile's own S columns with tcgen05.st and consumed
//    from TMEM as the A operand of the PV MMA (tcgen05.mma ... [d], [a_tmem], b_desc).
//  * Q/K and V of item k+1 stream (TMA, 3-D maps [units, S, cols], OOB rows zero) into the
//    second half of double-buffered slabs while item k computes.  Tile-B operands only
//    load the rows that exist (box ceil16(S-128)); the M=128 MMA over-reads the remaining
//    Q_B rows, which only produce discarded output rows.
//  * MMA issue order ping-pongs the two softmax warpgroups:
//      S_A(k) PV_B(k-1) S_B(k) PV_A(k) S_A(k+1) ...
//  * Bias operands off the MMA chain (BQT variant): each query row's Bq (32 fp16) is written into
//    TMEM by the row's own softmax thread for item k + 1 as soon as S'(k) completed (A operand of
//    TS bias MMAs); the one-hot key rows are double-buffered and gathered one item ahead; keys past
//    S carry a -30000 bias marker column instead of being masked per element.  When those 32 TMEM
//    columns do not fit (d ~ 0.55-0.75), Bq lives in shared-memory slabs (BQT = false).
//  * The kernel is instruction-cache sensitive: loops over runtime schedule sizes stay rolled.
// Roles: warp 0 TMA, warp 1 MMA, warps 2-3 one-hot key rows by 16-byte cp.async (BQT = false:
// warp 3 the Bq rows, warp 2 the key rows; warp 2 also owns the TMEM allocation), warps 4-7
// softmax tile A, warps 8-11 softmax tile B (one thread per row; exponentials on the packed fp32
// pipes, exp2_pair_bf16 in zs_common.cuh).
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {
namespace attnw {

constexpr int kThreads = 384;
constexpr uint32_t kTmemCols = 512;
constexpr int kMaxRuns = 4;

struct Params {
  int units, heads, S, bias_w, items, nt, nlw;
  long long ldo, o_unit_stride;
  const int* o_rows;  // optional: output row of (unit, query row), -1 = not written
  const __half* btab;  // [heads, S, 32] fp16: bh/tau (cols 0..15), bw/tau (16..31), zero padded
  long long btab_us;   // halves between the tables of consecutive units (0: one table for all)
  const __half* kb1;   // [S, 32] fp16 one-hot rows of every spatial key: e_{s/w} | e_{s%w}
  const int* q_sp;
  const int* k_sp;
  float tau;
  int rb;       // rows of the tile-B operands (ceil16(S-128)), 0 when nt == 1
  int seq;      // 1: tiles A and B share the S columns and run one after the other (dense-ish windows)
  int kv_rows;  // rows of the K/V slabs
  // smem layout (byte offsets from the 1024-aligned base; buffer b adds b * buf_bytes)
  int off_qa, off_k, off_qb, off_v, off_qa_t, off_k_t, off_qb_t, off_v_t, buf_bytes;
  int off_kb_h, off_kb_w, kb_buf, off_bar;  // one-hot key rows (TMEM-Bq variant: two buffers kb_buf bytes apart)
  int tx_qk, tx_v;
  // schedule
  unsigned char live[8];  // per softmax warp (tile*4 + w): bit g = key group g live
  unsigned char uni[2];   // per tile: union of its warps' live groups
  short gcol[2][8];       // per tile: S column of group g (valid when uni bit set)
  unsigned char gw[8];    // width (16 or 32) of group g in S columns
  int nrun[2];
  short run_k0[2][kMaxRuns], run_n[2][kMaxRuns], run_c0[2][kMaxRuns];  // key start, length, S column
  int s_col[2], o_col[2];                                               // TMEM column bases
  int tm_bq;                                                            // TMEM: Bq rows, 16 columns per tile (BQT)
  __nv_bfloat16* out;
  int trace;
  int off_bq_h, off_bq_w;  // Bq slabs (shared-memory Bq variant only)
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// fp16 x fp16 -> fp32 instruction descriptor (A/B K-major)
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// byte offset of 16-byte chunk c (0/1) of row r in a K-major tile with 32-byte rows, 32B swizzle
// (address bit 4 ^= bit 7), the layout TMA SWIZZLE_32B writes and sdesc_k_sw32 describes
__device__ __forceinline__ uint32_t sw32_off(int r, int c) { return (uint32_t)(r * 32 + ((c ^ ((r >> 2) & 1)) << 4)); }

__device__ __forceinline__ uint4 scale_pack8(const uint32_t* v, float s) {
  uint4 w;
  w.x = pack_bf16(__uint_as_float(v[0]) * s, __uint_as_float(v[1]) * s);
  w.y = pack_bf16(__uint_as_float(v[2]) * s, __uint_as_float(v[3]) * s);
  w.z = pack_bf16(__uint_as_float(v[4]) * s, __uint_as_float(v[5]) * s);
  w.w = pack_bf16(__uint_as_float(v[6]) * s, __uint_as_float(v[7]) * s);
  return w;
}
__device__ __forceinline__ void tmem_ld16p(uint32_t taddr, uint32_t* r) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
        "=r"(r[15])
      : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld_group(uint32_t taddr, uint32_t* r, bool w32) {
  tmem_ld16p(taddr, r);
  if (w32) tmem_ld16p(taddr + 16, r + 16);
}
// row max of one key group; W = width in S columns, vc = keys below S.  MASK: keys past S -> -inf
// first (without it, keys past S carry the -30000 bias marker, see the BQT key-row gather)
template <int W, bool MASK>
__device__ __forceinline__ float group_max(uint32_t* sr, int vc) {
  if (MASK && vc < W) {
#pragma unroll
    for (int j = 0; j < W; ++j)
      if (j >= vc) sr[j] = __float_as_uint(-INFINITY);
  }
  float m0 = __uint_as_float(sr[0]), m1 = __uint_as_float(sr[1]);
#pragma unroll
  for (int j = 2; j < W; j += 2) {
    m0 = fmaxf(m0, __uint_as_float(sr[j]));
    m1 = fmaxf(m1, __uint_as_float(sr[j + 1]));
  }
  return fmaxf(m0, m1);
}
// p = 2^(s*c - mc) for one group -> bf16 pairs stored to TMEM at pa; adds to rs.
template <int W>
__device__ __forceinline__ void group_emit(const uint32_t* sr, uint32_t pa, float c, float mc, float& rs) {
  uint32_t pk[W / 2];
  const unsigned long long c2 = f32x2(c, c), m2 = f32x2(-mc, -mc);
  unsigned long long acc = f32x2(0.f, 0.f);
#pragma unroll
  for (int j = 0; j < W / 2; ++j)
    pk[j] = exp2_pair_bf16(__uint_as_float(sr[2 * j]), __uint_as_float(sr[2 * j + 1]), c2, m2, acc);
  const float2 r2 = unpack_f32x2(acc);
  rs += r2.x + r2.y;
  if constexpr (W == 32) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(pa),
        "r"(pk[0]), "r"(pk[1]), "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7]), "r"(pk[8]),
        "r"(pk[9]), "r"(pk[10]), "r"(pk[11]), "r"(pk[12]), "r"(pk[13]), "r"(pk[14]), "r"(pk[15])
        : "memory");
  } else {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(pa), "r"(pk[0]), "r"(pk[1]),
        "r"(pk[2]), "r"(pk[3]), "r"(pk[4]), "r"(pk[5]), "r"(pk[6]), "r"(pk[7])
        : "memory");
  }
}
__device__ __forceinline__ void tmem_zero(uint32_t pa, bool w32) {
  if (w32) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(pa),
        "r"(0u)
        : "memory");
  } else {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"r"(pa), "r"(0u)
                 : "memory");
  }
}

// [heads*S, 32] fp16 bias operand rows (bh/tau, 0-pad to 16, bw/tau, 0-pad to 16), followed by
// the [S, 32] one-hot key rows (e_{s/w}, e_{s%w})
__global__ void win_bias_prep_kernel(const float* __restrict__ bh, const float* __restrict__ bw, long long rows,
                                     int S, int w, float inv_tau, __half* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long r = i >> 5;
  const int c = (int)(i & 31), j = c & 15;
  if (r < rows) {
    float v = 0.f;
    if (j < w) v = (c < 16 ? bh : bw)[(long long)r * w + j] * inv_tau;
    out[i] = __float2half_rn(v);
  } else if (r < rows + S) {
    const int sp = (int)(r - rows);
    out[i] = __float2half_rn(j == (c < 16 ? sp / w : sp % w) ? 1.f : 0.f);
  }
}

}  // namespace attnw

// Debug timeline: build with -DZS_KERNEL_TRACE and run with ZS_WIN_TRACE=1 to record clock64()
// stamps of CTA 0's first items (32 slots per item).  Compiled out by default.
__device__ unsigned long long g_win_trace[64 * 32];
#ifdef ZS_KERNEL_TRACE
#define ZS_TR(k, slot)                                                                      \
  do {                                                                                      \
    if (P.trace && blockIdx.x == 0 && (k) < 64) g_win_trace[(k) * 32 + (slot)] = clock64(); \
  } while (0)
#else
#define ZS_TR(k, slot) \
  do {             \
  } while (0)
#endif

// REG: all live groups of a row fit in registers (<= 3 groups of 32); otherwise S' is
// re-read from TMEM for the exp pass.
// BQT: the Bq rows live in TMEM (written by the softmax threads one item ahead) and the one-hot
// key rows are double-buffered, so neither gather sits on the MMA chain.  Without BQT (when the
// 32 TMEM columns do not fit next to S_A + S_B + O_A + O_B, e.g. d = 0.6 windows) warp 3 gathers
// the Bq rows into shared-memory slabs and the key rows are single-buffered.
template <int DH, bool REG, bool BQT>
__global__ void __launch_bounds__(attnw::kThreads, 1)
    zs_attn_win_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tq_t,
                       const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tk_t,
                       const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tv_t,
                       const __grid_constant__ CUtensorMap tq1, const __grid_constant__ CUtensorMap tq1_t,
                       const __grid_constant__ CUtensorMap tk1, const __grid_constant__ CUtensorMap tk1_t,
                       const __grid_constant__ CUtensorMap tv1, const __grid_constant__ CUtensorMap tv1_t,
                       const attnw::Params P) {
  using namespace attnw;
  constexpr bool kTail = DH == 80;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + P.off_bar);
  uint64_t* qk_full = bar + 0;    // [2]
  uint64_t* qk_empty = bar + 2;   // [2]
  uint64_t* v_full = bar + 4;     // [2]
  uint64_t* v_empty = bar + 6;    // [2]
  uint64_t* s_full = bar + 8;     // [tile]
  uint64_t* p_full = bar + 10;    // [tile]   live softmax warps: P written, O of the previous item read
  uint64_t* o_full = bar + 12;    // [tile]
  uint64_t* bk_full = bar + 14;   // [2] one-hot key rows of the item in smem buffer k & 1 (warps 2, 3)
  uint64_t* bk_empty = bar + 16;  // [2] S MMAs that read that buffer completed
  uint64_t* bq_full = bar + 18;   // [tile] live softmax warps: the item's Bq rows are in TMEM
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 20);

  // warp index via shfl: provably warp-uniform, so role code can use uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int nt = P.nt;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qk_full[s], 1);
      mbar_init(&qk_empty[s], 1);
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
      mbar_init(&s_full[s], 1);
      // live softmax warps of tile s (warps whose 32 rows start below S)
      mbar_init(&p_full[s], (uint32_t)max(1, min(4, (P.S - 128 * s + 31) / 32)));
      mbar_init(&o_full[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&bk_full[s], 2);
      mbar_init(&bk_empty[s], 1);
      mbar_init(&bq_full[s], (uint32_t)max(1, min(4, (P.S - 128 * s + 31) / 32)));
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // register budget: the single-lane producer / MMA / operand warpgroup gives registers to the
  // softmax warpgroups, whose rows live in registers (128*96 + 256*200 <= 384*168 at launch)
  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer
      if (lane == 0) {
        int k = 0;
        for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
          const int u = it / P.heads, col = (it % P.heads) * DH, b = k & 1, ph = ((k >> 1) & 1) ^ 1;
          uint8_t* base = smem + b * P.buf_bytes;
          mbar_wait_sleep(&qk_empty[b], ph);
          mbar_expect_tx(&qk_full[b], P.tx_qk);
          tma_load_3d(base + P.off_qa, &tq, &qk_full[b], col, 0, u);
          ZS_TR(k, 0);
          tma_load_3d(base + P.off_k, &tk, &qk_full[b], col, 0, u);
          if constexpr (kTail) {
            tma_load_3d(base + P.off_qa_t, &tq_t, &qk_full[b], col + 64, 0, u);
            tma_load_3d(base + P.off_k_t, &tk_t, &qk_full[b], col + 64, 0, u);
          }
          if (nt > 1) {
            tma_load_3d(base + P.off_qb, &tq1, &qk_full[b], col, 128, u);
            tma_load_3d(base + P.off_k + 128 * 128, &tk1, &qk_full[b], col, 128, u);
            if constexpr (kTail) {
              tma_load_3d(base + P.off_qb_t, &tq1_t, &qk_full[b], col + 64, 128, u);
              tma_load_3d(base + P.off_k_t + 128 * 32, &tk1_t, &qk_full[b], col + 64, 128, u);
            }
          }
          mbar_wait_sleep(&v_empty[b], ph);
          mbar_expect_tx(&v_full[b], P.tx_v);
          tma_load_3d(base + P.off_v, &tv, &v_full[b], col, 0, u);
          ZS_TR(k, 1);
          if constexpr (kTail) tma_load_3d(base + P.off_v_t, &tv_t, &v_full[b], col + 64, 0, u);
          if (nt > 1) {
            tma_load_3d(base + P.off_v + 128 * 128, &tv1, &v_full[b], col, 128, u);
            if constexpr (kTail) tma_load_3d(base + P.off_v_t + 128 * 32, &tv1_t, &v_full[b], col + 64, 128, u);
          }
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer (whole warp, elected lane)
      constexpr uint32_t id_pv = idesc_bf16(128, 64, false, true);
      constexpr uint32_t id_pv2 = idesc_bf16(128, 16, false, true);
      // descriptors of buffer 0 hoisted; buffer b / row offsets are added in 16-byte units
      const uint32_t bufd = (uint32_t)P.buf_bytes >> 4;
      const uint64_t dq[2] = {sdesc_k_sw128(smem + P.off_qa), sdesc_k_sw128(smem + P.off_qb)};
      const uint64_t dqt[2] = {sdesc_k_sw32(smem + P.off_qa_t), sdesc_k_sw32(smem + P.off_qb_t)};
      const uint64_t dk = sdesc_k_sw128(smem + P.off_k), dkt = sdesc_k_sw32(smem + P.off_k_t);
      const uint64_t dkh = sdesc_k_sw32(smem + P.off_kb_h), dkw = sdesc_k_sw32(smem + P.off_kb_w);
      const uint64_t dbh = sdesc_k_sw32(smem + P.off_bq_h), dbw = sdesc_k_sw32(smem + P.off_bq_w);
      const uint32_t kbd = BQT ? (uint32_t)P.kb_buf >> 4 : 0u;
      const uint64_t dv = sdesc_mn_sw128(smem + P.off_v), dvt = sdesc_mn_sw32(smem + P.off_v_t);
      auto issue_s = [&](int X, int b) {
        const uint64_t q = dq[X] + b * bufd, qt = dqt[X] + b * bufd;
        const uint64_t kk = dk + b * bufd, kt = dkt + b * bufd;
        const uint64_t kh = dkh + b * kbd, kw = dkw + b * kbd;
        const uint32_t bq = tmem + P.tm_bq + 16 * X;  // A operand: this tile's [bh | bw] rows (fp16)
        const uint32_t d0 = tmem + P.s_col[X];
#pragma unroll 1  // not unrolled: the kernel is instruction-cache bound
        for (int r = 0; r < P.nrun[X]; ++r) {
          const int k0 = P.run_k0[X][r], n = P.run_n[X][r];
          const uint32_t id = idesc_bf16(128, n), idh = idesc_f16(128, n);
          const uint32_t d = d0 + P.run_c0[X][r];
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) umma_ss(d, q + 2 * ks, kk + k0 * 8 + 2 * ks, id, ks > 0);
          if constexpr (kTail) umma_ss(d, qt, kt + k0 * 2, id, 1);
          if constexpr (BQT) {
            umma_ts(d, bq, kh + k0 * 2, idh, 1);      // + bh[σq, ky] / tau
            umma_ts(d, bq + 8, kw + k0 * 2, idh, 1);  // + bw[σq, kx] / tau
          } else {  // Bq slabs: tile B rows start at row 128 (x 32 B)
            umma_ss(d, dbh + X * 256, kh + k0 * 2, idh, 1);
            umma_ss(d, dbw + X * 256, kw + k0 * 2, idh, 1);
          }
        }
        umma_commit_elect(&s_full[X]);
      };
      auto issue_pv = [&](int X, int b) {
        const uint64_t vv = dv + b * bufd, vt = dvt + b * bufd;
        const uint32_t a0 = tmem + P.s_col[X];
        const uint32_t d = tmem + P.o_col[X];
        uint32_t acc = 0;
#pragma unroll 1  // not unrolled: the kernel is instruction-cache bound
        for (int r = 0; r < P.nrun[X]; ++r) {
          const int k0 = P.run_k0[X][r], n = P.run_n[X][r], c0 = P.run_c0[X][r];
          for (int s = 0; s < n / 16; ++s) {
            const uint32_t a = a0 + (uint32_t)((c0 >> 1) + 8 * s);
            const int kr = k0 + 16 * s;
            umma_ts(d, a, vv + kr * 8, id_pv, acc);
            if constexpr (kTail) umma_ts(d + 64, a, vt + kr * 2, id_pv2, acc);
            acc = 1;
          }
        }
        umma_commit_elect(&o_full[X]);
      };
      // bias operands of item k in place (key rows; BQT: tile X's Bq rows in TMEM)
      auto wait_bias = [&](int k_, int X) {
        if constexpr (BQT) {
          mbar_wait(&bk_full[k_ & 1], (k_ >> 1) & 1);
          mbar_wait(&bq_full[X], k_ & 1);
        } else {
          mbar_wait(bk_full, k_ & 1);
        }
      };
      int k = 0, pb = 0;
      if (P.seq) {
        // high densities (S_A + S_B + 2 O > 512 columns): the two tiles share the S columns and run
        // back to back — S_A, PV_A, S_B (issued after PV_A: in-order, so P_A is read before S_B
        // overwrites it), PV_B — with Q / K / V of the next item still double-buffered
        for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
          const int b = k & 1;
          mbar_wait(&qk_full[b], (k >> 1) & 1);
          wait_bias(k, 0);
          tc_fence_after();
          issue_s(0, b);
          mbar_wait_sleep(&p_full[0], k & 1);
          mbar_wait(&v_full[b], (k >> 1) & 1);
          tc_fence_after();
          issue_pv(0, b);
          if constexpr (BQT) mbar_wait(&bq_full[1], k & 1);
          tc_fence_after();
          issue_s(1, b);
          umma_commit_elect(&qk_empty[b]);
          umma_commit_elect(&bk_empty[BQT ? b : 0]);
          mbar_wait_sleep(&p_full[1], k & 1);
          tc_fence_after();
          issue_pv(1, b);
          umma_commit_elect(&v_empty[b]);
        }
      }
      for (int it = P.seq ? P.items : blockIdx.x; it < P.items; it += gridDim.x, ++k) {
        const int b = k & 1;
        mbar_wait(&qk_full[b], (k >> 1) & 1);
        wait_bias(k, 0);
        tc_fence_after();
        issue_s(0, b);
        if (lane == 0) ZS_TR(k, 2);
        if (nt > 1) {
          if (k > 0) {  // PV of tile B, previous item
            mbar_wait_sleep(&p_full[1], (k - 1) & 1);
            tc_fence_after();
            issue_pv(1, pb);
            umma_commit_elect(&v_empty[pb]);
            if (lane == 0) ZS_TR(k, 3);
          }
          if constexpr (BQT) mbar_wait(&bq_full[1], k & 1);
          tc_fence_after();
          issue_s(1, b);
          if (lane == 0) ZS_TR(k, 4);
        }
        umma_commit_elect(&qk_empty[b]);
        umma_commit_elect(&bk_empty[BQT ? b : 0]);
        mbar_wait_sleep(&p_full[0], k & 1);
        mbar_wait(&v_full[b], (k >> 1) & 1);
        tc_fence_after();
        issue_pv(0, b);
        if (lane == 0) ZS_TR(k, 5);
        if (nt == 1) umma_commit_elect(&v_empty[b]);
        pb = b;
      }
      if (nt > 1 && k > 0 && !P.seq) {
        mbar_wait(&p_full[1], (k - 1) & 1);
        tc_fence_after();
        issue_pv(1, pb);
        umma_commit_elect(&v_empty[pb]);
      }
    } else {
      if constexpr (BQT) {
      // ---------------------------------------------------------- one-hot key rows of each item
      // kb1[σk(j)] = e_{σk/w} | e_{σk%w} (two 16-column SW32 slabs), 64-byte-row gathers with
      // 16-byte cp.async (8 rows x 4 chunks per instruction); warp 2 rows [0, 128), warp 3 the
      // rest, into buffer k & 1 — the item ahead is gathered while this item's S' runs
      const int i0 = (warp - 2) * 4;
      const int nrows = P.kv_rows;
      const int c = lane & 3;
      // key rows past S get fp16 1.0 in bias column 15 (free when w < 16: one-hot columns are
      // ky, kx < w), which the Bq rows hold as -30000: S' of those keys is ~-30000 and their P
      // underflows to exactly 0, so the softmax needs no key-range masking.  (w = 16 means
      // S = 256: no keys past S.)
      const uint4 kmark = (c == 1 && P.bias_w < 16) ? make_uint4(0u, 0u, 0u, 0x3C000000u) : make_uint4(0u, 0u, 0u, 0u);
      int k = 0;
      for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
        const int u = it / P.heads, b = k & 1;
        const int* isrc = P.k_sp + (long long)u * P.S;
        uint8_t* slab = smem + ((c >> 1) ? P.off_kb_w : P.off_kb_h) + b * P.kb_buf;
        int idx[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int j = lane + 32 * (i0 + i);
          idx[i] = j < P.S ? __ldg(isrc + j) : -1;
        }
        mbar_wait_sleep(&bk_empty[b], ((k >> 1) & 1) ^ 1);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (32 * (i0 + i) >= nrows) break;
#pragma unroll
          for (int l = 0; l < 32; l += 8) {
            const int rl = l + (lane >> 2);
            const int r = 32 * (i0 + i) + rl;
            const int sp = __shfl_sync(0xffffffffu, idx[i], rl);
            if (r < nrows) {
              uint8_t* dst = slab + sw32_off(r, c & 1);
              if (sp >= 0)
                cp_async16(dst, P.kb1 + (long long)sp * 32 + c * 8);
              else
                *reinterpret_cast<uint4*>(dst) = kmark;  // key rows past S: the bias marker column
            }
          }
        }
        cp_async_wait_all();
        fence_proxy_async_smem();  // generic-proxy smem writes -> tensor core
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&bk_full[b]);
          if (warp == 2) ZS_TR(k, 8);
        }
      }
      } else {
      // Bq rows btab[h, σq(r)] (warp 3) and one-hot key rows kb1[σk(j)] (warp 2) into single
      // shared-memory buffers, 64-byte-row gathers with 16-byte cp.async
      const bool is_q = warp == 3;
      const int nrows = is_q ? P.S : P.kv_rows;
      const uint32_t off_h = is_q ? P.off_bq_h : P.off_kb_h, off_w = is_q ? P.off_bq_w : P.off_kb_w;
      const int c = lane & 3;
      uint8_t* slab = smem + ((c >> 1) ? off_w : off_h);
      int k = 0;
      for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
        const int u = it / P.heads, h = it % P.heads;
        const int* isrc = (is_q ? P.q_sp : P.k_sp) + (long long)u * P.S;
        int idx[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int j = lane + 32 * i;
          idx[i] = j < P.S ? __ldg(isrc + j) : -1;
        }
        const __half* tab = is_q ? P.btab + (long long)u * P.btab_us + (long long)h * P.S * 32 : P.kb1;
        mbar_wait_sleep(bk_empty, (k & 1) ^ 1);
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          if (32 * i >= nrows) break;
#pragma unroll
          for (int l = 0; l < 32; l += 8) {
            const int rl = l + (lane >> 2);
            const int r = 32 * i + rl;
            const int sp = __shfl_sync(0xffffffffu, idx[i], rl);
            if (r < nrows) {
              uint8_t* dst = slab + sw32_off(r, c & 1);
              if (sp >= 0)
                cp_async16(dst, tab + (long long)sp * 32 + c * 8);
              else
                *reinterpret_cast<uint4*>(dst) = make_uint4(0u, 0u, 0u, 0u);  // key rows past S
            }
          }
        }
        cp_async_wait_all();
        fence_proxy_async_smem();  // generic-proxy smem writes -> tensor core
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(bk_full);
          if (is_q) ZS_TR(k, 8);
        }
      }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    // ------------------------------------------------------------ softmax, one thread per row
    const int X = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int row = X * 128 + wq * 32 + lane;
    const bool warp_live = (X < nt) && (X * 128 + wq * 32 < P.S);
    const bool valid = row < P.S;
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t s_addr = tmem + P.s_col[X] + lane_off;
    const uint32_t o_addr = tmem + P.o_col[X] + lane_off;
    const unsigned live = warp_live ? P.live[X * 4 + wq] : 0u;
    const unsigned dead = warp_live ? (P.uni[X] & ~live) : 0u;
    const float cexp = P.tau * 1.4426950408889634f;  // logit = tau * S'; exp via 2^(S' tau log2e)

    // output row of (item, row): o_rows entry loaded when the item starts (om), consumed by its
    // epilogue one item later, so the load latency is off the epilogue's path
    auto out_row = [&](int it) -> int {
      return (valid && P.o_rows) ? __ldg(P.o_rows + (long long)(it / P.heads) * P.S + row) : 0;
    };
    auto epilogue = [&](int it, float inv, int om) {
      const int u = it / P.heads, h = it % P.heads;
      long long orow_off = (long long)u * P.o_unit_stride + (long long)row * P.ldo;
      bool ok = valid;
      if (ok && P.o_rows) {
        ok = om >= 0;
        orow_off = (long long)om * P.ldo;
      }
      __nv_bfloat16* dst = P.out + orow_off + h * DH;
      // 16-byte stores (measured faster here than 32-byte st.global.v8: tools/attn_ab.py)
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t pr[32];
        tmem_ld32(o_addr + c0, pr);
        tmem_ld_wait();
#ifdef ZS_WIN_NOSTORE
        if (ok && pr[0] == 0x7fffffffu) {
#else
        if (ok) {
#endif
          uint4* d4 = reinterpret_cast<uint4*>(dst + c0);
#pragma unroll
          for (int j = 0; j < 4; ++j) d4[j] = scale_pack8(pr + 8 * j, inv);
        }
      }
      if constexpr (DH == 80) {
        uint32_t p16[16];
        tmem_ld16(o_addr + 64, p16);
        tmem_ld_wait();
#ifdef ZS_WIN_NOSTORE
        if (ok && p16[0] == 0x7fffffffu) {
#else
        if (ok) {
#endif
          uint4* d4 = reinterpret_cast<uint4*>(dst + 64);
          d4[0] = scale_pack8(p16, inv);
          d4[1] = scale_pack8(p16 + 8, inv);
        }
      }
    };
    auto gmax = [&](int g, uint32_t* sr) -> float {
      const int vc = P.S - 32 * g;
      return P.gw[g] == 32 ? group_max<32, !BQT>(sr, vc) : group_max<16, !BQT>(sr, vc);
    };
    auto emit_p = [&](int g, const uint32_t* sr, float mc, float& rs) {
      const uint32_t pa = s_addr + (uint32_t)(P.gcol[X][g] >> 1);
      if (P.gw[g] == 32) group_emit<32>(sr, pa, cexp, mc, rs);
      else group_emit<16>(sr, pa, cexp, mc, rs);
    };

    // Bq rows (the A operand of the bias MMAs, 32 fp16 [bh | bw] / tau per query row) live in
    // TMEM, written by the row's own thread: for item k + 1 as soon as S'(k) has completed (its
    // last read of Bq(k)), from registers loaded one item ahead; the spatial index σq of the
    // row one item before that.  Rows past S write zeros (their S' rows are never used).
    const uint32_t bq_addr = tmem + P.tm_bq + 16 * X + lane_off;
    const int G = gridDim.x;
    auto load_sp = [&](int it2) -> int {
      int v = -1;
      if (valid && it2 < P.items)
        asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(P.q_sp + (long long)(it2 / P.heads) * P.S + row) : "memory");
      return v;
    };
    auto load_bq = [&](int it2, int sp, uint4 (&x)[4]) {
      const int u2 = it2 / P.heads, h2 = it2 % P.heads;
      const uint4* src = reinterpret_cast<const uint4*>(P.btab + (long long)u2 * P.btab_us + ((long long)h2 * P.S + sp) * 32);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        x[q] = make_uint4(0u, 0u, 0u, 0u);
        if (sp >= 0 && it2 < P.items)
          asm volatile("ld.global.nc.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x[q].x), "=r"(x[q].y), "=r"(x[q].z), "=r"(x[q].w)
                       : "l"(src + q)
                       : "memory");
      }
    };
    auto store_bq = [&](uint4 (&x)[4]) {
      if (P.bias_w < 16) x[1].w = (x[1].w & 0xffffu) | 0xF7530000u;  // column 15: fp16 -30000 (marker)
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
          "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(bq_addr),
          "r"(x[0].x), "r"(x[0].y), "r"(x[0].z), "r"(x[0].w), "r"(x[1].x), "r"(x[1].y), "r"(x[1].z), "r"(x[1].w),
          "r"(x[2].x), "r"(x[2].y), "r"(x[2].z), "r"(x[2].w), "r"(x[3].x), "r"(x[3].y), "r"(x[3].z), "r"(x[3].w)
          : "memory");
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bq_full[X]);
    };
    uint4 bqn[4];
    int spn = -1;
    if (BQT && warp_live && blockIdx.x < P.items) {
      load_bq(blockIdx.x, load_sp(blockIdx.x), bqn);
      store_bq(bqn);                                       // item 0
      load_bq(blockIdx.x + G, load_sp(blockIdx.x + G), bqn);  // item 1, in flight during item 0
      spn = load_sp(blockIdx.x + 2 * G);
    }
    int k = 0;
    int prev_it = -1, prev_om = 0;
    float prev_inv = 0.f;
    for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
      if (warp_live) {
        const int om = out_row(it);
        mbar_wait(&s_full[X], k & 1);
        tc_fence_after();
        if (BQT && it + G < P.items) {  // S'(k) done reading Bq(k): install Bq(k + 1)
          store_bq(bqn);
          load_bq(it + 2 * G, spn, bqn);
          spn = load_sp(it + 3 * G);
        }
        if (lane == 0) ZS_TR(k, 16 + 8 * X + 2);
        float mx = -INFINITY, rs = 0.f;
        if constexpr (REG) {
          // all live groups (<= 3) in registers
          uint32_t sr[3][32];
          const int n = __popc(live);
          const unsigned l1 = live & (live - 1u), l2 = l1 & (l1 - 1u);
          const int gl[3] = {__ffs(live) - 1, __ffs(l1) - 1, __ffs(l2) - 1};
#pragma unroll
          for (int i = 0; i < 3; ++i)
            if (i < n) tmem_ld_group(s_addr + P.gcol[X][gl[i]], sr[i], P.gw[gl[i]] == 32);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 3; ++i)
            if (i < n) mx = fmaxf(mx, gmax(gl[i], sr[i]));
          const float mc = (mx == -INFINITY) ? 0.f : mx * cexp;
#pragma unroll
          for (int i = 0; i < 3; ++i)
            if (i < n) emit_p(gl[i], sr[i], mc, rs);
        } else {
          // pass 1: row max over every live group
          for (int g = 0; g < 8; ++g) {
            if (!((live >> g) & 1u)) continue;
            uint32_t sr[32];
            tmem_ld_group(s_addr + P.gcol[X][g], sr, P.gw[g] == 32);
            tmem_ld_wait();
            mx = fmaxf(mx, gmax(g, sr));
          }
          const float mc = (mx == -INFINITY) ? 0.f : mx * cexp;
          // pass 2 (ascending columns: a group's P lands at or below columns already read)
          for (int g = 0; g < 8; ++g) {
            if (!((live >> g) & 1u)) continue;
            uint32_t sr[32];
            tmem_ld_group(s_addr + P.gcol[X][g], sr, P.gw[g] == 32);
            tmem_ld_wait();
            gmax(g, sr);  // re-apply the key-range mask
            emit_p(g, sr, mc, rs);
          }
        }
        if (lane == 0) ZS_TR(k, 16 + 8 * X + 3);
        // groups other warps of this tile need: P = 0 for this warp's rows
        for (int g = 0; g < 8; ++g)
          if ((dead >> g) & 1u) tmem_zero(s_addr + (uint32_t)(P.gcol[X][g] >> 1), P.gw[g] == 32);
        tmem_st_wait();
        // epilogue of the previous item (its PV had a whole softmax to complete)
        if (prev_it >= 0) {
          mbar_wait(&o_full[X], (k - 1) & 1);
          tc_fence_after();
          epilogue(prev_it, prev_inv, prev_om);
          if (lane == 0) ZS_TR(k, 16 + 8 * X + 4);
        }
        prev_it = it;
        prev_om = om;
        prev_inv = 1.0f / rs;
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&p_full[X]);
          ZS_TR(k, 16 + 8 * X + 5);
        }
      }
    }
    if (warp_live && prev_it >= 0) {
      mbar_wait(&o_full[X], (k - 1) & 1);
      tc_fence_after();
      epilogue(prev_it, prev_inv, prev_om);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace zs

using namespace zs;

static inline int ceil16(int x) { return (x + 15) & ~15; }

// Host launcher.  Returns 1 when the shape / schedule is outside this kernel's envelope
// (the caller then uses the generic window kernel), 0 on launch, negative on error.
int launch_attn_win(const void* q, const void* k, const void* v, long long ldq, long long ldk, long long ldv,
                    long long qus, long long kvus, int units, int heads, int S, int dh, const float* bh,
                    const float* bw, int bias_w, const int* q_sp, const int* k_sp, int b_row, int b_col, int prefix,
                    float tau, void* out, long long ldo, long long ous, const int* o_rows, long long bias_us,
                    const __half* btab_ext, long long btab_us, void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace attnw;
  if (S <= 0 || S > 256 || (b_row % 32) || (b_col % 32) || (dh != 64 && dh != 80)) return 1;
  if (bias_w > 16 || bias_w * bias_w != S || !(tau > 0.f)) return 1;
  Params p{};
  p.units = units;
  p.heads = heads;
  p.S = S;
  p.bias_w = bias_w;
  p.items = units * heads;
  p.nt = S > 128 ? 2 : 1;
  p.ldo = ldo;
  p.o_unit_stride = ous;
  p.o_rows = o_rows;
  p.q_sp = q_sp;
  p.k_sp = k_sp;
  p.tau = tau;
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.trace = getenv("ZS_WIN_TRACE") ? 1 : 0;
  const int tc = (S + b_col - 1) / b_col;
  const int ng = (S + 31) / 32;
  const int kvr = ceil16(S);
  p.rb = p.nt > 1 ? ceil16(S - 128) : 0;
  for (int g = 0; g < 8; ++g) p.gw[g] = (unsigned char)(g < ng ? std::min(32, kvr - 32 * g) : 0);
  // live groups per warp (b_row % 32 == 0: a warp's 32 rows lie in one query tile)
  int max_live = 0;
  for (int X = 0; X < 2; ++X) {
    unsigned uni = 0;
    for (int w = 0; w < 4; ++w) {
      const int r0 = X * 128 + w * 32;
      unsigned m = 0;
      if (X < p.nt && r0 < S) {
        const int qi = r0 / b_row;
        const int diag = std::min(qi, tc - 1);
        for (int g = 0; g < ng; ++g) {
          const int kt = (32 * g) / b_col;
          if (kt < prefix || kt == diag) m |= 1u << g;
        }
      }
      p.live[X * 4 + w] = (unsigned char)m;
      uni |= m;
      max_live = std::max(max_live, __builtin_popcount(m));
    }
    p.uni[X] = (unsigned char)uni;
    // runs of consecutive live groups -> contiguous S columns
    int col = 0, nr = 0;
    for (int g = 0; g < ng;) {
      if (!((uni >> g) & 1u)) {
        ++g;
        continue;
      }
      int e = g;
      while (e < ng && ((uni >> e) & 1u)) ++e;
      if (nr == kMaxRuns) return 1;
      int n = 0;
      for (int j = g; j < e; ++j) {
        p.gcol[X][j] = (short)(col + n);
        n += p.gw[j];
      }
      p.run_k0[X][nr] = (short)(32 * g);
      p.run_n[X][nr] = (short)n;
      p.run_c0[X][nr] = (short)col;
      col += n;
      ++nr;
      g = e;
    }
    p.nrun[X] = nr;
    if (col > 256) return 1;
    p.s_col[X] = col;  // width for now
  }
  const int wa = (p.s_col[0] + 31) & ~31, wb = p.s_col[1];
  p.seq = 0;
  // TMEM: S columns | Bq (2 x 16, BQT) | O_A | O_B (96 wide when they fit, else 80)
  bool bqt = true;
  if (wa + wb + 32 + 2 * 80 > (int)kTmemCols) {
    if (wa + wb + 2 * 80 <= (int)kTmemCols) {
      bqt = false;  // Bq rows in shared memory instead
    } else {
      // high density: tiles A and B one after the other over shared S columns
      if (p.nt < 2 || std::max(wa, wb) + 32 + 2 * 80 > (int)kTmemCols || getenv("ZS_WIN_NO_SEQ")) return 1;
      p.seq = 1;
    }
  }
  p.s_col[0] = 0;
  p.s_col[1] = p.seq ? 0 : wa;
  const int s_cols = p.seq ? std::max(wa, wb) : wa + wb;
  if (s_cols + (bqt ? 32 : 0) <= (int)kTmemCols - 2 * 96) {  // O accumulators 32-column aligned when they fit
    p.o_col[0] = (int)kTmemCols - 2 * 96;
    p.o_col[1] = (int)kTmemCols - 96;
  } else {
    p.o_col[0] = (int)kTmemCols - 2 * 80;
    p.o_col[1] = (int)kTmemCols - 80;
  }
  p.tm_bq = p.o_col[0] - 32;
  if (p.nrun[1] == 0) p.nt = 1;
  if (p.nt == 1) p.seq = 0;
  p.nlw = 0;
  for (int X = 0; X < p.nt; ++X)
    for (int w = 0; w < 4; ++w) p.nlw += (X * 128 + w * 32 < S) ? 1 : 0;
  // shared memory: [buf0 | buf1] (SW128 slabs then SW32 slabs) | Bq | Kb | barriers
  const bool tail = dh == 80;
  int off = 0;
  auto take = [&](int bytes, int align) {
    off = (off + align - 1) / align * align;
    const int o = off;
    off += bytes;
    return o;
  };
  const int rb = p.nt > 1 ? p.rb : 0;
  const int kvs = p.nt > 1 ? kvr : 128;  // chunk 0 is always a 128-row box
  p.kv_rows = kvs;
  p.off_qa = take(128 * 128, 1024);
  p.off_k = take(kvs * 128, 1024);
  p.off_qb = take(std::max(rb, 16) * 128, 1024);
  p.off_v = take(kvs * 128, 1024);
  if (tail) {
    p.off_qa_t = take(128 * 32, 1024);
    p.off_k_t = take(kvs * 32, 256);
    p.off_qb_t = take(std::max(rb, 16) * 32, 256);
    p.off_v_t = take(kvs * 32, 256);
  } else {
    p.off_qa_t = p.off_k_t = p.off_qb_t = p.off_v_t = 0;
  }
  // the M=128 MMA over-reads Q_B up to 128 rows: keep those bytes inside the buffer
  off = std::max(off, p.off_qb + 128 * 128);
  if (tail) off = std::max(off, p.off_qb_t + 128 * 32);
  p.buf_bytes = (off + 1023) / 1024 * 1024;
  off = 2 * p.buf_bytes;
  if (bqt) {
    // one-hot key rows, two buffers: [kb_h | kb_w] of buffer 0, then of buffer 1
    p.off_bq_h = p.off_bq_w = 0;
    p.off_kb_h = take(kvs * 32, 1024);
    p.off_kb_w = take(kvs * 32, 256);
    p.kb_buf = (off - p.off_kb_h + 1023) / 1024 * 1024;
    off = p.off_kb_h + 2 * p.kb_buf;
  } else {
    // Bq slabs: tile A rows [0,128) then tile B rows (the MMA reads 128 rows from 128*32); one
    // key-row buffer
    p.off_bq_h = take(256 * 32, 1024);
    p.off_bq_w = take(256 * 32, 1024);
    p.off_kb_h = take(kvs * 32, 256);
    p.off_kb_w = take(kvs * 32, 256);
    p.kb_buf = 0;
  }
  p.off_bar = take(256, 8);
  const size_t smem = 1024 + (size_t)off;
  if (smem > 227 * 1024) return 1;
  const int row_b = dh * 2;  // TMA boxes count their OOB (zero-filled) rows too
  p.tx_qk = (p.nt > 1 ? 128 + rb + 128 + rb : 128 + 128) * row_b;
  p.tx_v = (p.nt > 1 ? 128 + rb : 128) * row_b;
  // fp16 bias operand rows (bh, bw scaled by 1/tau): [heads, S, 32], or [units, heads, S, 32]
  // for per-unit fp32 tables (contiguous, bias_us == heads * S * w), or the caller's btab_ext;
  // followed by the [S, 32] one-hot key rows
  if (bias_us && !btab_ext && bias_us != (long long)heads * S * bias_w) return 1;
  const long long trows = btab_ext ? 0 : (long long)heads * S * (bias_us ? units : 1);
  // caller-owned workspace (zs_stripe_attn_ws_bytes): fp16 operand rows + one-hot key rows
  if (!ws || ws_bytes < (size_t)(trows + S) * 32 * sizeof(__half)) return ZS_ERR_WORKSPACE;
  if (reinterpret_cast<uintptr_t>(ws) & 255) return ZS_ERR_ALIGN;
  __half* btab = reinterpret_cast<__half*>(ws);
  {
    const long long n = (trows + S) * 32;
    { win_bias_prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(bh, bw, trows, S, bias_w, 1.0f / tau, btab); count_launch(); }
  }
  p.btab = btab_ext ? btab_ext : btab;
  p.btab_us = btab_ext ? btab_us : (bias_us ? (long long)heads * S * 32 : 0);
  p.kb1 = btab + trows * 32;
  CUtensorMap m[12];
  const uint64_t ncol = (uint64_t)heads * dh;
  int rc = 0;
  const CUtensorMapSwizzle S128 = CU_TENSOR_MAP_SWIZZLE_128B, S32 = CU_TENSOR_MAP_SWIZZLE_32B;
  rc |= make_tmap_3d_bf16(&m[0], q, ncol, S, units, ldq, qus, 64, 128, 1, S128);
  rc |= make_tmap_3d_bf16(&m[2], k, ncol, S, units, ldk, kvus, 64, 128, 1, S128);
  rc |= make_tmap_3d_bf16(&m[4], v, ncol, S, units, ldv, kvus, 64, 128, 1, S128);
  const int rbox = std::max(rb, 16);
  rc |= make_tmap_3d_bf16(&m[6], q, ncol, S, units, ldq, qus, 64, rbox, 1, S128);
  rc |= make_tmap_3d_bf16(&m[8], k, ncol, S, units, ldk, kvus, 64, rbox, 1, S128);
  rc |= make_tmap_3d_bf16(&m[10], v, ncol, S, units, ldv, kvus, 64, rbox, 1, S128);
  if (tail) {
    rc |= make_tmap_3d_bf16(&m[1], q, ncol, S, units, ldq, qus, 16, 128, 1, S32);
    rc |= make_tmap_3d_bf16(&m[3], k, ncol, S, units, ldk, kvus, 16, 128, 1, S32);
    rc |= make_tmap_3d_bf16(&m[5], v, ncol, S, units, ldv, kvus, 16, 128, 1, S32);
    rc |= make_tmap_3d_bf16(&m[7], q, ncol, S, units, ldq, qus, 16, rbox, 1, S32);
    rc |= make_tmap_3d_bf16(&m[9], k, ncol, S, units, ldk, kvus, 16, rbox, 1, S32);
    rc |= make_tmap_3d_bf16(&m[11], v, ncol, S, units, ldv, kvus, 16, rbox, 1, S32);
  } else {
    for (int i = 1; i < 12; i += 2) m[i] = m[i - 1];
  }
  if (rc) return ZS_ERR_TMAP;
  int grid = num_sms();
  if (grid > p.items) grid = p.items;
  const bool reg = max_live <= 3;
  auto launch = [&](auto kern) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    { kern<<<grid, kThreads, smem, st>>>(m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7], m[8], m[9], m[10], m[11], p); count_launch(); }
  };
  if (dh == 64) {
    if (bqt) {
      if (reg) launch(zs_attn_win_kernel<64, true, true>);
      else launch(zs_attn_win_kernel<64, false, true>);
    } else {
      if (reg) launch(zs_attn_win_kernel<64, true, false>);
      else launch(zs_attn_win_kernel<64, false, false>);
    }
  } else {
    if (bqt) {
      if (reg) launch(zs_attn_win_kernel<80, true, true>);
      else launch(zs_attn_win_kernel<80, false, true>);
    } else {
      if (reg) launch(zs_attn_win_kernel<80, true, false>);
      else launch(zs_attn_win_kernel<80, false, false>);
    }
  }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

// debug: copy CTA 0's timeline (64 items x 32 slots of clock64) to host
extern "C" __attribute__((visibility("default"))) int zs_debug_win_trace(unsigned long long* host, int n) {
  if (n > 64 * 32) n = 64 * 32;
  return cudaMemcpyFromSymbol(host, g_win_trace, n * sizeof(unsigned long long)) == cudaSuccess ? 0 : -1;
}

// zs_attn_glob.cu — stripe-sort attention for the global blocks (S = 4096, 128-row query tiles,
// 128-key tiles: encoder.py:57-58 b_global = 128).
//
// Semantics as zs_attn.cu (attention.py:88-104, :167-221).  With b_row = b_col = 128 every
// work item (unit, head, query tile i) is one 128-row MMA tile and every key tile one 128-key
// chunk, so J_i = {0..p-1} ∪ {min(i, Tc-1)} is a list of whole chunks: no intra-chunk mask
// except keys / rows past S.
//
// B200 design (one persistent CTA per SM):
//  * Decomposed rel-pos bias on the tensor core: S' = q.k + Bq . OH^T, where Bq[r] =
//    [bh[σq(r)] | bw[σq(r)]] / tau (fp16, 128 columns, resident in TMEM for the item and used
//    as the A operand) and OH[k] = [e_{σk/64} | e_{σk%64}] (fp16 one-hot rows of the chunk's
//    keys, generated in shared memory).  logit = tau * S', so the softmax does no gathers.
//  * Chunk c's S' goes to TMEM S buffer c % 2, so S'(c + 1) is computed while chunk c is in
//    the softmax.  All 8 softmax warps work on every chunk: the two warps of a TMEM lane
//    quarter (warps 4 + q and 8 + q) split its 128 keys (64 each), and each key half runs its
//    own online softmax (reference max, O accumulator O_half with row sums, P -> its own PV
//    MMAs), with no per-chunk exchange: the two warps of an SMSP drift out of phase, so one's
//    row max overlaps the other's exponentials.  The halves merge once per item in the epilogue.
//  * P (bf16) overwrites the chunk's S columns in TMEM (half w's 64 keys at columns [64w, 64w+32),
//    inside its own S columns) and is the A operand of that half's PV MMAs into O_half;
//    the PV is ONE N = DH + 16 MMA per 16 keys: V is staged as MN-major SW32 atoms of 16 columns
//    followed by an atom of bf16 ones, so the 16 extra O columns hold the row sums (of the bf16 P
//    exactly as applied to V).  (N = 16 MMAs cost ~26 cycles each, as much as N = 64.)
//  * Lazy rescaling: O_half (and its row-sum columns) is rescaled in TMEM, warp-wide, only when
//    the half's row max grows by more than ln 256.
//  * The next item's Bq rows are prefetched from the fp16 table one item ahead and written into
//    TMEM (tcgen05.st) by the softmax threads as soon as the item's last S' MMA has completed,
//    Q tiles are loaded by their own producer lane (the K / V rings run ahead into the next
//    item), and the MMA stream runs across items (the next item's first S' before this item's
//    last PV): at an item boundary only the last PV and the epilogue remain serial.
//  * Epilogue on its own warps (12-15, one per TMEM lane quarter): when both halves published
//    their final reference maxima and the item's last PVs completed, they read O_0 / O_1 and the
//    row sums, free the accumulators for the next item's first PV, merge the halves and write the
//    tile through shared memory and one TMA tensor store per item, while the softmax warps are
//    already in the next item.  TMEM: S 256 + O_0 96 + O_1 96 + Bq 64 = 512 columns.
// Roles: warp 0 TMA (lane 0: Q per item + K per chunk, lane 1: V per chunk), warp 1 MMA (whole
// warp, elected lane), warps 2-3 one-hot key rows per chunk, warps 4-11 softmax, warps 12-15
// epilogue (registers 96 / 152 / 112 per warpgroup through setmaxnreg).
#include <cuda_fp16.h>

#include <algorithm>
#include <cstdlib>

#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {
namespace attng {

constexpr int BQ = 128;
constexpr int kThreads = 512;  // 4 producer / MMA / one-hot warps, 8 softmax warps, 4 epilogue warps
constexpr uint32_t kTmemCols = 512;
constexpr int KST = 3;  // K ring stages
constexpr int OST = 2;  // one-hot ring stages (generated on chip: no memory latency to hide)
constexpr int QST = 1;  // Q slots (the next item's Q loads once the last S' of the item completed)
constexpr int VST = 2;  // V ring stages
constexpr uint32_t TM_S = 0;     // S_w at [w*128, w*128+128)
constexpr uint32_t TM_O = 256;   // O_b at [256 + 96b, + DH), row sums (ones atom) at [+DH, +DH+16); b = item & 1
constexpr uint32_t TM_OS = 96;   // columns per O buffer
constexpr uint32_t TM_BQ = 448;  // Bq: 128 fp16 = 64 columns
constexpr int OH_BYTES = 2 * BQ * 128;  // two 64-column SW128 slabs (e_ky | e_kx)
constexpr int VATOM = BQ * 32;          // V: MN-major SW32 atoms of 16 columns x 128 keys

struct Params {
  int units, heads, S, bias_w, T, prefix, items;
  long long ldo, o_unit_stride;
  const int* o_rows;  // optional: output row of (unit, query row), -1 = not written
  const __half* btab;  // [heads, S, 128] fp16 rows: bh/tau in cols [0, w), bw/tau in [64, 64 + w)
  long long btab_us;   // halves between the tables of consecutive units (0: one table for all)
  const int* q_sp;
  const int* k_sp;
  float tau;
  __nv_bfloat16* out;
  int off_q, off_k, off_oh, off_v, off_ml, off_ost, off_bar, tile, vstage;
  int tma_out;  // 1: the O tile leaves through shared memory and one TMA tensor store (no o_rows)
  int trace;
  uint32_t w_magic;  // floor(2^32 / bias_w) + 1: s / bias_w == umulhi(s, w_magic) for s < 2^32 / bias_w
};

template <int DH>
struct Shape {
  static constexpr bool kTail = DH == 80;
  static constexpr int MAIN = BQ * 128;
  static constexpr int TILE = ((MAIN + (kTail ? BQ * 32 : 0) + 1023) / 1024) * 1024;
  // V stage: DH/16 column atoms + one atom of bf16 ones (row sums): the PV MMA is ONE N = DH + 16
  // instruction per 16 keys (an N = 16 MMA costs ~26 cycles, as much as N = 64: tools/glob_mma_bench.cu)
  static constexpr int VSTAGE = (DH / 16 + 1) * VATOM;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
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
// fp16 x fp16 -> fp32 instruction descriptor (A/B K-major)
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
  return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// chunks of item with query tile i: 0..p-1, then the diagonal min(i, T-1) when it is >= p
__device__ __forceinline__ int n_chunks(const Params& P, int i) {
  const int d = min(i, P.T - 1);
  return P.prefix + (d >= P.prefix ? 1 : 0);
}
__device__ __forceinline__ int chunk_of(const Params& P, int i, int j) { return j < P.prefix ? j : min(i, P.T - 1); }

// [rows, 128] fp16 bias operand rows: bh/tau in columns [0, w), bw/tau in [64, 64 + w), zeros elsewhere
__global__ void glob_bias_prep_kernel(const float* __restrict__ bh, const float* __restrict__ bw, int rows, int w,
                                      float inv_tau, __half* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (long long)rows * 128) return;
  const long long r = i >> 7;
  const int c = (int)(i & 127), j = c & 63;
  float v = 0.f;
  if (j < w) v = (c < 64 ? bh : bw)[r * w + j] * inv_tau;
  out[i] = __float2half_rn(v);
}

}  // namespace attng

// Debug timeline: build with -DZS_KERNEL_TRACE and run with ZS_GLOB_TRACE=1 to record clock64()
// stamps of CTA 0 (16 slots per item; 8 per chunk of item 5).  Compiled out by default: the
// stamps sit on the MMA issue path and would cost its uniform-datapath code.
__device__ unsigned long long g_glob_trace[64 * 16];
__device__ unsigned long long g_glob_trace2[128];
#ifdef ZS_KERNEL_TRACE
#define ZG_TR(k, slot)                                                                       \
  do {                                                                                       \
    if (P.trace && blockIdx.x == 0 && (k) < 64) g_glob_trace[(k) * 16 + (slot)] = clock64(); \
  } while (0)
#define ZG_T2(k, j, slot)                                                                                  \
  do {                                                                                                     \
    if (P.trace && blockIdx.x == 0 && (k) == 5 && (j) < 16) g_glob_trace2[(j) * 8 + (slot)] = clock64(); \
  } while (0)
#else
#define ZG_TR(k, slot) \
  do {             \
  } while (0)
#define ZG_T2(k, j, slot) \
  do {                \
  } while (0)
#endif

// Epilogue warps (12-15) of zs_attn_glob_kernel: warp 12 + q owns rows [32q, 32q + 32) of every
// item (TMEM lane quarter q).  See the role comment in the kernel.
template <int DH>
__device__ __forceinline__ void epilogue_warps(const attng::Params& P, uint8_t* smem, uint32_t tmem, uint64_t* m_full,
                                               uint64_t* o_last, uint64_t* o_free, const CUtensorMap& to,
                                               const CUtensorMap& to_t, int q, int lane, int nmb) {
  using namespace attng;
  using L = Shape<DH>;
  constexpr bool kTail = L::kTail;
  constexpr float L2E = 1.4426950408889634f;
  constexpr int NC = DH / 8;  // 16-byte pieces of an output row
  const int r = q * 32 + lane;
  const uint32_t lane_off = (uint32_t)(q * 32) << 16;
  const float* xch = reinterpret_cast<const float*>(smem + P.off_ml);  // [item parity][half][BQ]
  const bool issuer = q == 0 && lane == 0;
  uint8_t* st = smem + P.off_ost;
  int k = 0;
  for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
    const int i = it % nmb, uh = it / nmb, h = uh % P.heads, u = uh / P.heads;
    mbar_wait(&m_full[k & 1], (k >> 1) & 1);
    const float m0 = xch[(k & 1) * 2 * BQ + r], m1 = xch[(k & 1) * 2 * BQ + BQ + r];
    const float m = fmaxf(m0, m1);
    const float a0 = (m0 == -INFINITY) ? 0.f : ex2((m0 - m) * L2E);
    const float a1 = (m1 == -INFINITY) ? 0.f : ex2((m1 - m) * L2E);
    mbar_wait(o_last, k & 1);  // the item's last PVs of both halves
    tc_fence_after();
    const uint32_t o0 = tmem + TM_O + lane_off, o1 = o0 + TM_OS;
    uint32_t l01[2];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(l01[0]) : "r"(o0 + DH));
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(l01[1]) : "r"(o1 + DH));
    uint4 pk[NC];
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int cc = 0; cc < NC; cc += 2) {  // 16 columns of O_0 and O_1 per step
      uint32_t va[16], vb[16];
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(va[0]), "=r"(va[1]), "=r"(va[2]), "=r"(va[3]), "=r"(va[4]), "=r"(va[5]), "=r"(va[6]),
                     "=r"(va[7]), "=r"(va[8]), "=r"(va[9]), "=r"(va[10]), "=r"(va[11]), "=r"(va[12]), "=r"(va[13]),
                     "=r"(va[14]), "=r"(va[15])
                   : "r"(o0 + 8 * cc));
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                   : "=r"(vb[0]), "=r"(vb[1]), "=r"(vb[2]), "=r"(vb[3]), "=r"(vb[4]), "=r"(vb[5]), "=r"(vb[6]),
                     "=r"(vb[7]), "=r"(vb[8]), "=r"(vb[9]), "=r"(vb[10]), "=r"(vb[11]), "=r"(vb[12]), "=r"(vb[13]),
                     "=r"(vb[14]), "=r"(vb[15])
                   : "r"(o1 + 8 * cc));
      tmem_ld_wait();
      if (cc == 0) {  // the row sums arrived with the first columns
        const float l = a0 * __uint_as_float(l01[0]) + a1 * __uint_as_float(l01[1]);
        s0 = a0 / l;
        s1 = a1 / l;
      }
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        float f[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          f[e] = __uint_as_float(va[8 * t + e]) * s0 + __uint_as_float(vb[8 * t + e]) * s1;
        pk[cc + t] = make_uint4(pack_bf16(f[0], f[1]), pack_bf16(f[2], f[3]), pack_bf16(f[4], f[5]), pack_bf16(f[6], f[7]));
      }
    }
    tc_fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(o_free);  // O_0 / O_1 read: the next item's first PVs may start
    if (P.tma_out) {
      if (issuer) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // staging free
      named_bar_sync(7, 128);
#pragma unroll
      for (int gc = 0; gc < NC; ++gc) {
        const int off = gc < 8 ? r * 128 + ((gc ^ (r & 7)) << 4) : L::MAIN + r * 32 + (((gc - 8) ^ ((r >> 2) & 1)) << 4);
        *reinterpret_cast<uint4*>(st + off) = pk[gc];
      }
      fence_proxy_async_smem();
      named_bar_sync(7, 128);
      if (issuer) {
        asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                         reinterpret_cast<uint64_t>(&to)), "r"(h * DH), "r"(i * BQ), "r"(u), "r"(smem_u32(st))
                     : "memory");
        if constexpr (kTail)
          asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                           reinterpret_cast<uint64_t>(&to_t)), "r"(h * DH + 64), "r"(i * BQ), "r"(u),
                       "r"(smem_u32(st + L::MAIN))
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      }
    } else {
      const int row = i * BQ + r;
      bool valid = row < P.S;
      long long orow_off = (long long)u * P.o_unit_stride + (long long)row * P.ldo;
      if (valid && P.o_rows) {
        const int mrow = P.o_rows[(long long)u * P.S + row];
        valid = mrow >= 0;
        orow_off = (long long)mrow * P.ldo;
      }
      if (valid) {
        uint4* d4 = reinterpret_cast<uint4*>(P.out + orow_off + h * DH);  // 16-byte aligned
#pragma unroll
        for (int gc = 0; gc < NC; ++gc) d4[gc] = pk[gc];
      }
    }
  }
  if (P.tma_out && issuer) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int DH>
__global__ void __launch_bounds__(attng::kThreads, 1)
    zs_attn_glob_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tq_t,
                        const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tk_t,
                        const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tv_t,
                        const __grid_constant__ CUtensorMap to, const __grid_constant__ CUtensorMap to_t,
                        const attng::Params P) {
  using namespace attng;
  using L = Shape<DH>;
  constexpr bool kTail = L::kTail;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + P.off_bar);
  uint64_t* q_full = bar + 0;    // [QST]
  uint64_t* q_empty = bar + 2;   // [QST]
  uint64_t* k_full = bar + 4;    // [KST] K tile landed (TMA)
  uint64_t* k_empty = bar + 8;   // [KST] S' of the chunk done: K stage free
  uint64_t* oh_full = bar + 12;  // [OST] one-hot rows written (warps 2, 3)
  uint64_t* v_full = bar + 16;   // [VST]
  uint64_t* v_empty = bar + 20;  // [VST]
  uint64_t* s_full = bar + 24;   // [wg]
  uint64_t* p_full = bar + 44;   // [S buffer][half] 4 softmax warps: this half's P of the chunk in TMEM
  uint64_t* o_full = bar + 48;   // [half] PV_half of a chunk completed (one completion per chunk)
  uint64_t* o_last = bar + 29;   // the item's last PVs completed (one completion per item)
  uint64_t* o_free = bar + 30;   // 8 warps: O_0 / O_1 read by the item's epilogue
  uint64_t* bq_full = bar + 31;  // 8 warps: the item's Bq rows are in TMEM
  uint64_t* bq_free = bar + 32;  // the item's last S' completed (Bq may be replaced)
  uint64_t* oh_empty = bar + 36; // [OST] S' of the chunk done: one-hot stage free
  uint64_t* m_full = bar + 26;   // [item parity] 8 softmax warps: the item's final reference maxima in smem
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 34);
  static_assert(KST <= 4 && VST <= 4 && QST <= 2 && OST <= 4, "barrier slots");

  // warp index via shfl: provably warp-uniform, so role code can use uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv_t);
    for (int s = 0; s < QST; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1);
      mbar_init(&p_full[2 * s], 4);
      mbar_init(&p_full[2 * s + 1], 4);
      mbar_init(&o_full[s], 1);
    }
    mbar_init(o_last, 1);
    for (int s = 0; s < KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < OST; ++s) {
      mbar_init(&oh_full[s], 2);
      mbar_init(&oh_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(o_free, 4);
    mbar_init(&m_full[0], 8);
    mbar_init(&m_full[1], 8);
    mbar_init(bq_full, 8);
    mbar_init(bq_free, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int nmb = P.T;  // query tiles per (unit, head)

  if (warp < 4) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 96;");
    if (warp == 0) {
      // ---------------------------------------------------------- TMA producer
      if (lane == 2) {
        // Q tiles on their own lane: the K / V rings run ahead into the next item while the Q slot
        // waits for this item's last S'; the next item's Q tile is prefetched into L2 meanwhile
        int k = 0;
        for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
          const int i = it % nmb, uh = it / nmb, col = (uh % P.heads) * DH, u = uh / P.heads;
          const int qs = k % QST;
          mbar_wait_sleep(&q_empty[qs], ((k / QST) & 1) ^ 1);
          mbar_expect_tx(&q_full[qs], BQ * DH * 2);
          uint8_t* q = smem + P.off_q + qs * L::TILE;
          tma_load_3d(q, &tq, &q_full[qs], col, i * BQ, u);
          if constexpr (kTail) tma_load_3d(q + L::MAIN, &tq_t, &q_full[qs], col + 64, i * BQ, u);
          const int it2 = it + gridDim.x;
          if (it2 < P.items) {
            const int i2 = it2 % nmb, uh2 = it2 / nmb, col2 = (uh2 % P.heads) * DH, u2 = uh2 / P.heads;
            asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                             reinterpret_cast<uint64_t>(&tq)), "r"(col2), "r"(i2 * BQ), "r"(u2) : "memory");
            if constexpr (kTail)
              asm volatile("cp.async.bulk.prefetch.tensor.3d.L2.global.tile [%0, {%1, %2, %3}];" ::"l"(
                               reinterpret_cast<uint64_t>(&tq_t)), "r"(col2 + 64), "r"(i2 * BQ), "r"(u2) : "memory");
          }
        }
      } else if (lane < 2) {
        int k = 0, c = 0;
        for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
          const int i = it % nmb, uh = it / nmb, h = uh % P.heads, u = uh / P.heads, col = h * DH;
          const int nc = n_chunks(P, i);
          for (int j = 0; j < nc; ++j, ++c) {
            const int cj = chunk_of(P, i, j);
            if (lane == 0) {
              const int s = c % KST;
              mbar_wait_sleep(&k_empty[s], ((c / KST) & 1) ^ 1);
              mbar_expect_tx(&k_full[s], BQ * DH * 2);
              uint8_t* kk = smem + P.off_k + s * L::TILE;
              tma_load_3d(kk, &tk, &k_full[s], col, cj * BQ, u);
              if constexpr (kTail) tma_load_3d(kk + L::MAIN, &tk_t, &k_full[s], col + 64, cj * BQ, u);
            } else {
              const int s = c % VST;
              mbar_wait_sleep(&v_empty[s], ((c / VST) & 1) ^ 1);
              mbar_expect_tx(&v_full[s], BQ * DH * 2);
              uint8_t* vv = smem + P.off_v + s * L::VSTAGE;
#pragma unroll
              for (int a = 0; a < DH / 16; ++a) tma_load_3d(vv + a * VATOM, &tv_t, &v_full[s], col + 16 * a, cj * BQ, u);
            }
          }
        }
      }
    } else if (warp == 1) {
      // ---------------------------------------------------------- MMA issuer (whole warp)
      constexpr uint32_t id_s = idesc_bf16(BQ, BQ);
      constexpr uint32_t id_b = idesc_f16(BQ, BQ);
      constexpr uint32_t id_pv = idesc_bf16(BQ, DH + 16, false, true);
      constexpr uint32_t TILE16 = L::TILE >> 4;
      const uint64_t dq = sdesc_k_sw128(smem + P.off_q), dqt = sdesc_k_sw32(smem + P.off_q + L::MAIN);
      const uint64_t dk = sdesc_k_sw128(smem + P.off_k), dkt = sdesc_k_sw32(smem + P.off_k + L::MAIN);
      const uint64_t doh = sdesc_k_sw128(smem + P.off_oh);
      const uint64_t dv = sdesc(smem + P.off_v, VATOM, 256, 6);  // MN-major SW32 atoms, LBO = one atom
      // S'(c) of chunk ordinal c into S_w: q.k (bf16) then + Bq . OH^T (fp16, A from TMEM)
      int first_c = 0;  // chunk ordinal of the current item's first chunk (trace only)
      auto issue_s = [&](int c, int k, int w, bool last) {
        const int ks_ = c % KST, os_ = c % OST, qs = k % QST;
        mbar_wait(&k_full[ks_], (c / KST) & 1);
        if (lane == 0) ZG_T2(k, c - first_c, 4);
        mbar_wait(&oh_full[os_], (c / OST) & 1);
        if (lane == 0) ZG_T2(k, c - first_c, 5);
        tc_fence_after();
        const uint64_t q = dq + qs * TILE16, qt = dqt + qs * TILE16;
        const uint64_t kk = dk + ks_ * TILE16, kt = dkt + ks_ * TILE16;
        const uint64_t oh = doh + os_ * (OH_BYTES >> 4);
        const uint32_t d = tmem + TM_S + w * 128;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks) umma_ss(d, q + 2 * ks, kk + 2 * ks, id_s, ks > 0);
        if constexpr (kTail) umma_ss(d, qt, kt, id_s, 1);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks)  // slab e_ky (k-steps 0-3), slab e_kx (4-7)
          umma_ts(d, tmem + TM_BQ + 8 * ks, oh + (ks >> 2) * (BQ * 128 >> 4) + 2 * (ks & 3), id_b, 1);
        umma_commit_elect(&s_full[w]);
        umma_commit_elect(&k_empty[ks_]);
        umma_commit_elect(&oh_empty[os_]);
        if (last) {
          umma_commit_elect(&q_empty[qs]);
          umma_commit_elect(bq_free);
        }
      };
      // PV of one key half (keys [64x, 64x + 64) of chunk c) into that half's accumulator O_x:
      // [O_x | row sums] (+)= P_x . [V | 1], one N = DH + 16 MMA per 16 keys
      auto issue_pv_half = [&](int c, int w, bool first, int x) {
        const int vs = c % VST;
        const uint64_t v = dv + vs * (L::VSTAGE >> 4);
        const uint32_t a0 = tmem + TM_S + w * 128 + 64 * x;  // half x's P: its own S columns
        const uint32_t d = tmem + TM_O + x * TM_OS;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          umma_ts(d, a0 + 8 * ks, v + (4 * x + ks) * (16 * 32 / 16), id_pv, (!first || ks > 0) ? 1u : 0u);
        umma_commit_elect(&o_full[x]);
      };
      // PV(c-1) is issued right after S'(c): S'(c) goes to the other S buffer, and S'(c) into
      // buffer w always follows PV(c-2) in issue order, so P_w is read before it is overwritten
      // (tcgen05.mma executes in order).  The stream runs across items: the next item's first
      // S' is issued before this item's last PV (its Bq is installed as soon as this item's last
      // S' completed), so the tensor pipe does not drain at item boundaries.
      int npv[2] = {0, 0};
      int pend_c = -1, pend_w = 0, pend_k = 0;
      bool pend_first = false, pend_last = false;
      auto flush_pv = [&]() {
        const int vs = pend_c % VST;
        mbar_wait(&v_full[vs], (pend_c / VST) & 1);
        if (pend_first && pend_k > 0) mbar_wait(o_free, (pend_k - 1) & 1);  // previous epilogue read O_0 / O_1
        // each half's PV as soon as that half's P is in TMEM (the halves run their softmax independently)
#pragma unroll
        for (int x = 0; x < 2; ++x) {
          mbar_wait(&p_full[2 * pend_w + x], npv[pend_w] & 1);
          tc_fence_after();
          issue_pv_half(pend_c, pend_w, pend_first, x);
        }
        umma_commit_elect(&v_empty[vs]);
        if (lane == 0) ZG_T2(pend_k, pend_c - first_c, 3);
        npv[pend_w]++;
        if (pend_last) {
          umma_commit_elect(o_last);  // after the item's last PVs: the epilogue's own barrier
          if (lane == 0) ZG_TR(pend_k, 15);
        }
        pend_c = -1;
      };
      int k = 0, c = 0;
      for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
        const int i = it % nmb;
        const int nc = n_chunks(P, i);
        mbar_wait(&q_full[k % QST], (k / QST) & 1);
        mbar_wait(bq_full, k & 1);
        if (lane == 0) ZG_TR(k, 6);
        for (int j = 0; j < nc; ++j, ++c) {
          const int w = c & 1;
          if (j == 0) first_c = c;
          issue_s(c, k, w, j == nc - 1);
          if (lane == 0 && j < 6) ZG_TR(k, 7 + j);
          if (lane == 0) ZG_T2(k, j, 0);
          if (pend_c >= 0) flush_pv();
          pend_c = c;
          pend_w = w;
          pend_k = k;
          pend_first = j == 0;  // first chunk of the item: O starts fresh
          pend_last = j == nc - 1;
        }
      }
      if (pend_c >= 0) flush_pv();
    } else {
      // ---------------------------------------------------------- one-hot key rows (warps 2, 3)
      // chunk c, keys [64*(warp-2), +64): row kr of each SW128 slab = fp16 e_{σk/w} (slab 0) and
      // e_{σk%w} (slab 1); 16-byte chunk cc of row kr lives at kr*128 + ((cc ^ (kr & 7)) << 4).
      // The stage buffers are zeroed once; per chunk a lane clears the two hot chunks its row
      // had in that stage and writes the two new ones (4 stores instead of 16).  The next
      // chunk's key indices are loaded while the current chunk is written.
      const uint32_t one = 0x3C00u;  // fp16 1.0
      const int kbase = (warp - 2) * 64;
      const uint4 z4 = make_uint4(0u, 0u, 0u, 0u);
      {  // the ones atom of every V stage: bf16 ones [128 keys, 16] (every element 1.0, so the swizzle
         // is irrelevant); published to the tensor core by the fence before the first oh_full arrive
        const uint4 o4 = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
#pragma unroll
        for (int s = 0; s < VST; ++s)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            reinterpret_cast<uint4*>(smem + P.off_v + s * P.vstage + (DH / 16) * VATOM)[((warp - 2) * 32 + lane) * 4 + q] = o4;
      }
#pragma unroll
      for (int st = 0; st < OST; ++st)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int kr = kbase + lane + 32 * e;
#pragma unroll
          for (int cc = 0; cc < 16; ++cc)
            *reinterpret_cast<uint4*>(smem + P.off_oh + st * OH_BYTES + (cc >> 3) * (BQ * 128) + kr * 128 +
                                      (((cc & 7) ^ (kr & 7)) << 4)) = z4;
        }
      int prev[OST][2][2];  // byte offsets of the hot chunks last written per stage / row (-1: none)
#pragma unroll
      for (int st = 0; st < OST; ++st)
#pragma unroll
        for (int e = 0; e < 2; ++e) prev[st][e][0] = prev[st][e][1] = -1;
      auto load_sp = [&](int it_, int j_, int (&sp)[2]) {
        const int i_ = it_ % nmb, u_ = it_ / nmb / P.heads, cj = chunk_of(P, i_, j_);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int kg = cj * BQ + kbase + lane + 32 * e;
          sp[e] = kg < P.S ? __ldg(P.k_sp + (long long)u_ * P.S + kg) : -1;
        }
      };
      int it = blockIdx.x, j = 0, kk2 = 0;
      int spc[2] = {-1, -1};
      if (it < P.items) load_sp(it, 0, spc);
      for (int c = 0; it < P.items; ++c) {
        const int nc = n_chunks(P, it % nmb);
        int it2 = it, j2 = j + 1;
        if (j2 == nc) {
          it2 += gridDim.x;
          j2 = 0;
        }
        int spn[2] = {-1, -1};
        if (it2 < P.items) load_sp(it2, j2, spn);  // in flight while this chunk is written
        const int st = c % OST;
        mbar_wait_sleep(&oh_empty[st], ((c / OST) & 1) ^ 1);
        if (lane == 0 && warp == 2) ZG_T2(kk2, j, 7);
        uint8_t* oh = smem + P.off_oh + st * OH_BYTES;
        // stage index made compile-time (unrolled + matched) so prev[][][] stays in registers
#pragma unroll
        for (int sidx = 0; sidx < OST; ++sidx) {
          if (sidx != st) continue;
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int kr = kbase + lane + 32 * e;
            if (prev[sidx][e][0] >= 0) *reinterpret_cast<uint4*>(oh + prev[sidx][e][0]) = z4;
            if (prev[sidx][e][1] >= 0) *reinterpret_cast<uint4*>(oh + prev[sidx][e][1]) = z4;
            prev[sidx][e][0] = prev[sidx][e][1] = -1;
            const int sp = spc[e];
            if (sp >= 0) {
              const int ky = (int)__umulhi((uint32_t)sp, P.w_magic), kx = sp - ky * P.bias_w;
              const int oy = kr * 128 + (((ky >> 3) ^ (kr & 7)) << 4);
              const int ox = BQ * 128 + kr * 128 + (((kx >> 3) ^ (kr & 7)) << 4);
              const uint32_t vy = one << (16 * (ky & 1)), vx = one << (16 * (kx & 1));
              const int wy = (ky >> 1) & 3, wx = (kx >> 1) & 3;
              *reinterpret_cast<uint4*>(oh + oy) =
                  make_uint4(wy == 0 ? vy : 0u, wy == 1 ? vy : 0u, wy == 2 ? vy : 0u, wy == 3 ? vy : 0u);
              *reinterpret_cast<uint4*>(oh + ox) =
                  make_uint4(wx == 0 ? vx : 0u, wx == 1 ? vx : 0u, wx == 2 ? vx : 0u, wx == 3 ? vx : 0u);
              prev[sidx][e][0] = oy;
              prev[sidx][e][1] = ox;
            }
          }
        }
        fence_proxy_async_smem();  // generic-proxy smem writes -> tensor core
        __syncwarp();
        if (lane == 0) mbar_arrive(&oh_full[st]);
        if (lane == 0 && warp == 2) ZG_T2(kk2, j, 6);
        spc[0] = spn[0];
        spc[1] = spn[1];
        if (it2 != it) ++kk2;
        it = it2;
        j = j2;
      }
    }
  } else if (warp >= 12) {
    // ------------------------------------------------------------ epilogue warps (12-15)
    // Item k's output, off the softmax warps: once both halves published their final reference
    // maxima (m_full) and the item's last PVs completed (o_last), warp 12 + q reads rows
    // [32q, 32q + 32) of O_0 / O_1 and the row sums, frees the accumulators (o_free: the next
    // item's first PV may start), merges the halves out = (a_0 O_0 + a_1 O_1) / (a_0 l_0 +
    // a_1 l_1) and writes the row through shared memory and one TMA tensor store per item (or
    // direct stores through o_rows).
    asm volatile("setmaxnreg.dec.sync.aligned.u32 112;");
    epilogue_warps<DH>(P, smem, tmem, m_full, o_last, o_free, to, to_t, warp & 3, lane, nmb);
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 152;");
    // ------------------------------------------------------------ softmax warpgroups
    // Half w (warps 4 + 4w .. 7 + 4w) owns key columns [64w, 64w + 64) of every chunk with its own
    // online softmax: reference max m_w, accumulator O_w (+ row sums), P_w -> p_full[buf][w].  The
    // halves never synchronise per chunk (no partial-max exchange), so the two warps of an SMSP
    // drift out of phase and one's row max overlaps the other's exponentials; they merge once per
    // item: out = (a_0 O_0 + a_1 O_1) / (a_0 l_0 + a_1 l_1), a_w = 2^((m_w - max(m_0, m_1)) log2 e).
    // Thread = row wq*32 + lane (TMEM lane quarter of the warp).
    const int w = (warp - 4) >> 2;
    const int wq = warp & 3;
    const int r = wq * 32 + lane;  // row within the tile == TMEM lane
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    const uint32_t o_mine = tmem + TM_O + w * TM_OS + lane_off;  // O_w
    const uint32_t bq_addr = tmem + TM_BQ + w * 32 + lane_off;    // this half's 64 fp16 bias columns
    float* xch = reinterpret_cast<float*>(smem + P.off_ml);       // [item parity][half][BQ] reference max
    constexpr float L2E = 1.4426950408889634f;
    constexpr float kThr = 5.545177444479562f;  // ln 256
    const float tau = P.tau, cexp = P.tau * L2E;

    // Bq rows of item `it2` (this half: 64 fp16 = 128 bytes): loaded one item ahead (volatile
    // loads stay where they are issued), written into TMEM once the previous item's last S' has
    // completed (bq_free).  The item boundary then waits on no global-memory latency.
    // spatial position of this thread's query row in item it2 (volatile load: issued here,
    // consumed one item later)
    auto load_sp = [&](int it2) -> int {
      const int i2 = it2 % nmb, u2 = it2 / nmb / P.heads;
      const int row2 = i2 * BQ + r;
      int v = 0;
      if (it2 < P.items && row2 < P.S)
        asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(v) : "l"(P.q_sp + (long long)u2 * P.S + row2) : "memory");
      return v;
    };
    auto load_bq = [&](int it2, int sp, uint4 (&x)[8]) {
      const int i2 = it2 % nmb, uh2 = it2 / nmb, h2 = uh2 % P.heads, u2 = uh2 / P.heads;
      const bool ok = it2 < P.items && i2 * BQ + r < P.S;
      const uint4* src = reinterpret_cast<const uint4*>(P.btab + (long long)u2 * P.btab_us +
                                                    ((long long)h2 * P.S + sp) * 128 + w * 64);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        x[q] = make_uint4(0u, 0u, 0u, 0u);
        if (ok)
          asm volatile("ld.global.nc.v4.b32 {%0, %1, %2, %3}, [%4];"
                       : "=r"(x[q].x), "=r"(x[q].y), "=r"(x[q].z), "=r"(x[q].w)
                       : "l"(src + q)
                       : "memory");
      }
    };
    auto store_bq = [&](const uint4 (&x)[8], int k2) {
      uint32_t v[32];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        v[4 * q] = x[q].x;
        v[4 * q + 1] = x[q].y;
        v[4 * q + 2] = x[q].z;
        v[4 * q + 3] = x[q].w;
      }
      if (k2 > 0) mbar_wait(bq_free, (k2 - 1) & 1);
      tc_fence_after();
      tmem_st32(bq_addr, v);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(bq_full);
    };
    // O_w (DH + 16 columns incl. the row sums) *= alpha, 8 columns at a time (S values are live)
    auto o_scale = [&](float alpha) {
#pragma unroll
      for (int c0 = 0; c0 < DH + 16; c0 += 8) {
        uint32_t pr[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(pr[0]), "=r"(pr[1]), "=r"(pr[2]), "=r"(pr[3]), "=r"(pr[4]), "=r"(pr[5]), "=r"(pr[6]),
                       "=r"(pr[7])
                     : "r"(o_mine + c0));
        tmem_ld_wait();
#pragma unroll
        for (int q = 0; q < 8; ++q) pr[q] = __float_as_uint(__uint_as_float(pr[q]) * alpha);
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(o_mine + c0),
                     "r"(pr[0]), "r"(pr[1]), "r"(pr[2]), "r"(pr[3]), "r"(pr[4]), "r"(pr[5]), "r"(pr[6]), "r"(pr[7])
                     : "memory");
      }
    };
    // output columns [w*OH, w*OH + OH) of this row; OH = DH / 2 (40 or 32)

    const int G = gridDim.x;
    uint4 bqx[8];
    load_bq(blockIdx.x, load_sp(blockIdx.x), bqx);
    store_bq(bqx, 0);
    load_bq(blockIdx.x + G, load_sp(blockIdx.x + G), bqx);  // next item's rows, in flight during this item
    int sp_nn = load_sp(blockIdx.x + 2 * G);                  // and the row index of the one after
    int k = 0, c = 0;
    for (int it = blockIdx.x; it < P.items; it += gridDim.x, ++k) {
      const int i = it % nmb, uh = it / nmb, h = uh % P.heads, u = uh / P.heads;
      const int nc = n_chunks(P, i);
      if (lane == 0 && wq == 0) ZG_TR(k, 2 + w);
      float m_ref = -INFINITY;
      for (int j = 0; j < nc; ++j, ++c) {
        const int buf = c & 1;
        const int cj = chunk_of(P, i, j);
        const int kvalid = P.S - cj * BQ - 64 * w;  // keys of this half below S
        mbar_wait(&s_full[buf], (c >> 1) & 1);
        tc_fence_after();
        if (j == nc - 1 && it + G < P.items) {
          // the item's last S' completed, and with it every read of Bq: install the next item's
          // rows now, so its first S' does not wait for this chunk's softmax and the epilogue
          store_bq(bqx, k + 1);
          load_bq(it + 2 * G, sp_nn, bqx);
          sp_nn = load_sp(it + 3 * G);
        }
        if (lane == 0 && wq == 0 && j == 0 && w == 0) ZG_TR(k, 0);
        if (lane == 0 && wq == 0 && w == 0) ZG_T2(k, j, 1);
        const uint32_t s_addr = tmem + TM_S + buf * 128 + lane_off;
        uint32_t sr[64];
        tmem_ld32(s_addr + 64 * w, *reinterpret_cast<uint32_t(*)[32]>(sr));
        tmem_ld32(s_addr + 64 * w + 32, *reinterpret_cast<uint32_t(*)[32]>(sr + 32));
        tmem_ld_wait();
        if (kvalid < 64) {
#pragma unroll
          for (int jj = 0; jj < 64; ++jj)
            if (jj >= kvalid) sr[jj] = __float_as_uint(-INFINITY);
        }
        float m0 = -INFINITY, m1 = -INFINITY;
#pragma unroll
        for (int jj = 0; jj < 64; jj += 4) {
          m0 = max3f(m0, __uint_as_float(sr[jj]), __uint_as_float(sr[jj + 1]));
          m1 = max3f(m1, __uint_as_float(sr[jj + 2]), __uint_as_float(sr[jj + 3]));
        }
        const float mx = tau * fmaxf(m0, m1);  // this half's row max logit
        // lazy rescale of O_w: a warp-wide TMEM round trip when any row of the warp moves its
        // reference, alpha = 1 for the others
        float alpha = 1.f;
        const bool upd = mx > m_ref + kThr || (m_ref == -INFINITY && mx > -INFINITY);
        if (upd) alpha = (m_ref == -INFINITY) ? 0.f : ex2((m_ref - mx) * L2E);
        if (__any_sync(0xffffffffu, upd)) {
          if (j > 0) {
            mbar_wait(&o_full[w], (c - 1) & 1);  // PV_w(c - 1) complete before O_w is rescaled
            tc_fence_after();
            o_scale(alpha);
          }
          if (upd) m_ref = mx;
        }
        {  // P of this half's 64 keys -> TMEM columns [64w, 64w + 32) (its own S columns)
          const float mc = (m_ref == -INFINITY) ? 0.f : m_ref * L2E;
          const unsigned long long c2 = f32x2(cexp, cexp), m2 = f32x2(-mc, -mc);
#pragma unroll
          for (int g = 0; g < 2; ++g) {
            uint32_t pk[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
              pk[q] = exp2_pair_bf16_ns(__uint_as_float(sr[32 * g + 2 * q]), __uint_as_float(sr[32 * g + 2 * q + 1]),
                                        c2, m2);
            tmem_st16(s_addr + 64 * w + 16 * g, pk);
          }
        }
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[2 * buf + w]);
        if (lane == 0 && wq == 0 && j == 0 && w == 0) ZG_TR(k, 1);
        if (lane == 0 && wq == 0 && w == 0) ZG_T2(k, j, 2);
      }
      // publish this half's final reference max for the epilogue warps
      xch[(k & 1) * 2 * BQ + w * BQ + r] = m_ref;
      __syncwarp();
      if (lane == 0) mbar_arrive(&m_full[k & 1]);
      (void)h;
      (void)u;
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace zs

using namespace zs;

// Host launcher: returns 1 when outside this kernel's envelope (b_row = b_col = 128, bias
// width <= 64, dh 64 / 80), 0 on launch, negative on error.
int launch_attn_glob(const void* q, const void* k, const void* v, long long ldq, long long ldk, long long ldv,
                     long long qus, long long kvus, int units, int heads, int S, int dh, const float* bh,
                     const float* bw, int bias_w, const int* q_sp, const int* k_sp, int b_row, int b_col, int prefix,
                     float tau, void* out, long long ldo, long long ous, const int* o_rows, long long bias_us,
                     const __half* btab_ext, long long btab_us, void* ws, size_t ws_bytes, cudaStream_t st) {
  using namespace attng;
  if (b_row != BQ || b_col != BQ || (dh != 64 && dh != 80) || S < 1 || bias_w > 64 || !(tau > 0.f)) return 1;
  Params p{};
  p.units = units;
  p.heads = heads;
  p.S = S;
  p.bias_w = bias_w;
  p.T = (S + BQ - 1) / BQ;
  p.prefix = prefix;
  const long long items = (long long)units * heads * p.T;
  if (items > 0x7FFFFFFF) return ZS_ERR_SHAPE;
  p.items = (int)items;
  p.ldo = ldo;
  p.o_unit_stride = ous;
  p.o_rows = o_rows;
  p.q_sp = q_sp;
  p.k_sp = k_sp;
  p.tau = tau;
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  p.trace = getenv("ZS_GLOB_TRACE") ? 1 : 0;
  p.w_magic = (uint32_t)((1ull << 32) / (unsigned)bias_w + 1ull);
  const int tile = dh == 80 ? Shape<80>::TILE : Shape<64>::TILE;
  p.tile = tile;
  p.vstage = dh == 80 ? Shape<80>::VSTAGE : Shape<64>::VSTAGE;
  int off = 0;
  auto take = [&](int bytes, int align) {
    off = (off + align - 1) / align * align;
    const int o = off;
    off += bytes;
    return o;
  };
  p.off_q = take(QST * tile, 1024);
  p.off_k = take(KST * tile, 1024);
  p.off_oh = take(OST * OH_BYTES, 1024);
  p.off_v = take(VST * p.vstage, 1024);
  p.off_ml = take(2 * 4 * BQ * 4, 16);
  p.tma_out = o_rows == nullptr ? 1 : 0;
  p.off_ost = take(tile, 1024);  // O staging for the TMA store: [128, 64] SW128 + [128, 16] SW32
  p.off_bar = take(512, 8);
  const size_t smem = 1024 + (size_t)off;
  if (smem > 227 * 1024) return 1;
  // fp16 bias operand rows [heads, S, 128] (caller's workspace); per-unit fp32
  // tables (contiguous: bias_us == heads * S * w) -> [units, heads, S, 128]; or the caller's
  if (bias_us && !btab_ext && bias_us != (long long)heads * S * bias_w) return 1;
  if (btab_ext) {
    p.btab = btab_ext;
    p.btab_us = btab_us;
  } else {
    const size_t need = (size_t)heads * S * 128 * (bias_us ? units : 1);
    if (!ws || ws_bytes < need * sizeof(__half)) return ZS_ERR_WORKSPACE;  // zs_stripe_attn_ws_bytes
    if (reinterpret_cast<uintptr_t>(ws) & 255) return ZS_ERR_ALIGN;
    __half* buf = reinterpret_cast<__half*>(ws);
    const long long n = (long long)need;
    { glob_bias_prep_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(bh, bw, n / 128, bias_w, 1.0f / tau, buf); count_launch(); }
    p.btab = buf;
    p.btab_us = bias_us ? (long long)heads * S * 128 : 0;
  }
  CUtensorMap m[8];
  const uint64_t ncol = (uint64_t)heads * dh;
  int rc = 0;
  rc |= make_tmap_3d_bf16(&m[0], q, ncol, S, units, ldq, qus, 64, BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  rc |= make_tmap_3d_bf16(&m[2], k, ncol, S, units, ldk, kvus, 64, BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  rc |= make_tmap_3d_bf16(&m[4], v, ncol, S, units, ldv, kvus, 64, BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  // V: 16-column SW32 boxes only (the PV B operand is a row of MN-major SW32 atoms)
  rc |= make_tmap_3d_bf16(&m[5], v, ncol, S, units, ldv, kvus, 16, BQ, 1, CU_TENSOR_MAP_SWIZZLE_32B);
  if (dh == 80) {
    rc |= make_tmap_3d_bf16(&m[1], q, ncol, S, units, ldq, qus, 16, BQ, 1, CU_TENSOR_MAP_SWIZZLE_32B);
    rc |= make_tmap_3d_bf16(&m[3], k, ncol, S, units, ldk, kvus, 16, BQ, 1, CU_TENSOR_MAP_SWIZZLE_32B);
  } else {
    m[1] = m[0];
    m[3] = m[2];
  }
  // output [units, S, heads * dh] (row stride ldo, unit stride ous): the TMA store boxes
  rc |= make_tmap_3d_bf16(&m[6], out, ncol, S, units, ldo, ous, 64, BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  if (dh == 80) rc |= make_tmap_3d_bf16(&m[7], out, ncol, S, units, ldo, ous, 16, BQ, 1, CU_TENSOR_MAP_SWIZZLE_32B);
  else m[7] = m[6];
  if (rc) return ZS_ERR_TMAP;
  int grid = num_sms();
  if (grid > p.items) grid = p.items;
  if (dh == 64) {
    cudaFuncSetAttribute(zs_attn_glob_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    { zs_attn_glob_kernel<64><<<grid, kThreads, smem, st>>>(m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7], p); count_launch(); }
  } else {
    cudaFuncSetAttribute(zs_attn_glob_kernel<80>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    { zs_attn_glob_kernel<80><<<grid, kThreads, smem, st>>>(m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7], p); count_launch(); }
  }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

extern "C" __attribute__((visibility("default"))) int zs_debug_glob_trace(unsigned long long* host, int n) {
  if (n > 64 * 16 + 128) n = 64 * 16 + 128;
  if (cudaMemcpyFromSymbol(host, g_glob_trace, (n < 1024 ? n : 1024) * sizeof(unsigned long long)) != cudaSuccess)
    return -1;
  if (n > 1024 && cudaMemcpyFromSymbol(host + 1024, g_glob_trace2, (n - 1024) * sizeof(unsigned long long)) != cudaSuccess)
    return -1;
  return 0;
}

// zs_attn.cu — static block-sparse stripe-sort ("A-shape") attention on tcgen05.
//
// Semantics (attention.py:88-104, :167-221): inputs are already in scan (σ)
// order; query tile i (b_row rows) visits key tiles
//     J_i = {0 .. prefix-1} ∪ {min(i, Tc-1)}
// and computes softmax(tau * q k^T + bh[σq(q), σk(k)/w] + bw[σq(q), σk(k)%w]) v
// over exactly those columns (columns past Sk are excluded).
//
// B200 mapping.  A persistent CTA (one per SM) walks work items
// (unit, head, 128-row query block); for each item it streams the 128-key
// chunks holding at least one active (query tile, key tile) pair — the
// closed-form schedule above, never a dense mask — and applies the exact tile
// pattern as -inf (per 32-column group when tiles are multiples of 32).  All
// roles walk the same (item, chunk) sequence, so every ring runs across item
// boundaries and the next item's loads overlap the current item's math.
//   warp 0       TMA: Q ring (1-2 slots), K ring (3 stages), V ring (2 stages);
//                3-D maps [units, S, cols], rows past S zero-filled by TMA
//   warp 1       tcgen05.mma, issued as S(0), S(1), PV(0), S(2), PV(1), ... so a
//                PV never waits behind a later chunk's K load:
//                  S_c = Q K_c^T  (128x128xdh -> TMEM, 2 buffers)
//                  O  += P_c V_c  (128xdh x128 -> TMEM accumulator)
//   warp 2       TMEM allocation (512 columns)
//   warp 3       metadata loader: per chunk the byte offsets of bh[., σk/w] and
//                bw[., σk%w] for its 128 keys; per item the gathered bias rows
//                bh[σq], bw[σq] (cp.async), both double-buffered ahead
//   warps 4..11  softmax, two threads per query row (key halves 0-63 / 64-127):
//                tcgen05.ld of S, tau + bias from smem, row max exchanged
//                through smem, exp, P (bf16) into the UMMA 128B-swizzled K-major
//                layout, O rescaled in TMEM when the running max moves.
// dh = 80 (ViT-H) is a 64-column 128B-swizzle slab plus a 16-column 32B-swizzle
// slab: QK^T runs 4+1 K-steps, PV an N=64 and an N=16 MMA with V consumed
// MN-major straight from its TMA layout.
#include <algorithm>
#include <cstdlib>

#include <cuda_fp16.h>

#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {

namespace attn {
constexpr int BQ = 128;   // query rows per item (UMMA M)
constexpr int BKC = 128;  // keys per chunk (UMMA N of QK^T, K of PV)
constexpr int kSoftThreads = 256;
constexpr int kThreads = 128 + kSoftThreads;
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t TM_S = 0;    // S buffers at columns [0,128) and [128,256)
constexpr uint32_t TM_O = 256;  // O accumulator at [256, 256+dh)
constexpr int KST = 3;          // K ring stages
constexpr int VST = 2;          // V ring stages

struct Params {
  int units, heads, sq, sk, bias_w;
  long long ldo, o_unit_stride;
  const int* o_rows;  // optional: output row of (unit, query row), -1 = not written
  const float* bh;
  long long bias_us;  // floats between the bh / bw tables of consecutive units (0: shared)
  const float* bw;
  const int* q_sp;
  const int* k_sp;
  int b_row, b_col, prefix, tc, nmb, items;
  float tau;
  int q_slots;    // 1 or 2
  int bias_bufs;  // 1 or 2
  int off_bias;   // smem byte offset of the bias buffers
  __nv_bfloat16* out;
  // FAST path tables (b_row, b_col multiples of 32): key-tile range of every 128-key chunk and
  // key tile of every 32-key group, precomputed on the host so the hot loops never divide
  unsigned char ck_lo[64], ck_hi[64];
  unsigned char gkt[256];
  unsigned long long mbmask[64];  // needed-chunk bitmask of every 128-row query block
};

template <int DH>
struct Layout {
  static constexpr bool kTail = DH == 80;
  static constexpr int MAIN = BQ * 128;             // 64 bf16 x 128 rows, SW128
  static constexpr int TAIL = kTail ? BQ * 32 : 0;  // 16 bf16 x 128 rows, SW32
  static constexpr int TILE = ((MAIN + TAIL + 1023) / 1024) * 1024;
  static constexpr int OFF_K = 0;
  static constexpr int OFF_V = OFF_K + KST * TILE;
  static constexpr int OFF_P = OFF_V + VST * TILE;       // 2 atoms x 128 rows x 128 B
  static constexpr int OFF_KOFF = OFF_P + 2 * BQ * 128;  // [2][BKC] int2 byte offsets
  static constexpr int OFF_XMAX = OFF_KOFF + 2 * BKC * 8;  // [chunk parity][half][BQ]
  static constexpr int OFF_XSUM = OFF_XMAX + 4 * BQ * 4;
  static constexpr int OFF_BAR = OFF_XSUM + 4 * BQ * 4;   // xsum: [chunk parity][half][BQ]
  static constexpr int OFF_TAB = OFF_BAR + 512;           // ck_lo[64] ck_hi[64] gkt[256] | mbmask[64] at +512
  static constexpr int OFF_Q = OFF_BAR + 2048;            // q_slots x TILE (1024-aligned)
  static_assert(OFF_TAB + 1024 <= OFF_Q, "table region overflows");
  static constexpr int TX_Q = BQ * DH * 2;
  static constexpr int TX_KV = BKC * DH * 2;
  static int off_bias(int q_slots) { return OFF_Q + q_slots * TILE; }
  static size_t bias_bytes(int bias_w) { return (size_t)2 * BQ * (bias_w + 1) * 4; }
  static size_t smem_bytes(int q_slots, int bias_w, int bufs) {
    return 1024 + off_bias(q_slots) + bufs * bias_bytes(bias_w);
  }
};

template <bool FAST>
struct ChunkPlan {
  int nck, p, tc, bcol, dlo, dhi;
  const unsigned char* lo;  // shared-memory copies of Params::ck_lo / ck_hi / mbmask
  const unsigned char* hi;
  const unsigned long long* mbm;
  __device__ __forceinline__ void init(const Params& P, int row0) {
    if constexpr (FAST) mask = mbm[row0 / BQ];
    nck = (P.sk + BKC - 1) / BKC;
    p = P.prefix;
    tc = P.tc;
    bcol = P.b_col;
    const int qt_lo = row0 / P.b_row;
    const int qt_hi = min(row0 + BQ - 1, P.sq - 1) / P.b_row;
    dlo = min(qt_lo, tc - 1);
    dhi = min(qt_hi, tc - 1);
  }
  __device__ __forceinline__ bool needed(int cj) const {
    int kt_lo, kt_hi;
    if constexpr (FAST) {
      kt_lo = lo[cj];
      kt_hi = hi[cj];
    } else {
      kt_lo = (cj * BKC) / bcol;
      kt_hi = min((cj * BKC + BKC - 1) / bcol, tc - 1);
    }
    if (kt_lo < p) return true;
    return !(dhi < kt_lo || dlo > kt_hi);
  }
  unsigned long long mask;  // FAST: needed-chunk bitmask of this query block (from the smem table)
  __device__ __forceinline__ int next(int cj) const {  // next needed chunk after cj, or -1
    if constexpr (FAST) {
      const unsigned long long rest = (cj + 1 >= 64) ? 0ull : (mask >> (cj + 1)) << (cj + 1);
      return rest ? __ffsll((long long)rest) - 1 : -1;
    }
    for (int j = cj + 1; j < nck; ++j)
      if (needed(j)) return j;
    return -1;
  }
};

// Walks the (item, chunk) sequence of this CTA.  c = global chunk ordinal, k = item ordinal.
template <bool FAST>
struct Cursor {
  int it, k, c, cj, u, h, mb;
  bool valid, first, last;
  ChunkPlan<FAST> plan;
  __device__ __forceinline__ void init_tables(const unsigned char* tab) {
    plan.lo = tab;
    plan.hi = tab + 64;
    plan.mbm = reinterpret_cast<const unsigned long long*>(tab + 512);
  }
  __device__ __forceinline__ void load_item(const Params& P) {
    valid = it < P.items;
    if (!valid) return;
    mb = it % P.nmb;
    const int uh = it / P.nmb;
    h = uh % P.heads;
    u = uh / P.heads;
    plan.init(P, mb * BQ);
    cj = plan.next(-1);
    first = true;
    last = plan.next(cj) < 0;
  }
  __device__ __forceinline__ void start(const Params& P) {
    it = blockIdx.x;
    k = 0;
    c = 0;
    load_item(P);
  }
  __device__ __forceinline__ void advance(const Params& P) {
    ++c;
    const int n = plan.next(cj);
    if (n >= 0) {
      cj = n;
      first = false;
      last = plan.next(cj) < 0;
    } else {
      it += gridDim.x;
      ++k;
      load_item(P);
    }
  }
};

// wait with a short sleep between probes: for the single-lane producer / MMA / loader warps, so their
// spinning does not steal issue slots from the softmax warps sharing the SM sub-partitions
__device__ __forceinline__ void mbar_wait_backoff(uint64_t* bar, uint32_t parity) { mbar_wait_sleep(bar, parity); }

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void cp_async4(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

__device__ __forceinline__ uint4 scale_pack8(const uint32_t* v, float s) {
  uint4 w;
  w.x = pack_bf16(__uint_as_float(v[0]) * s, __uint_as_float(v[1]) * s);
  w.y = pack_bf16(__uint_as_float(v[2]) * s, __uint_as_float(v[3]) * s);
  w.z = pack_bf16(__uint_as_float(v[4]) * s, __uint_as_float(v[5]) * s);
  w.w = pack_bf16(__uint_as_float(v[6]) * s, __uint_as_float(v[7]) * s);
  return w;
}
}  // namespace attn

template <int DH, bool FAST>
__global__ void __launch_bounds__(attn::kThreads, 1)
    zs_attn_kernel(const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tq2,
                   const __grid_constant__ CUtensorMap tk, const __grid_constant__ CUtensorMap tk2,
                   const __grid_constant__ CUtensorMap tv, const __grid_constant__ CUtensorMap tv2,
                   attn::Params P) {
  using namespace attn;
  using L = Layout<DH>;
  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned base by pointer arithmetic on the __shared__ array (keeps the shared address space:
  // an integer round trip would turn every softmax smem access into a generic LD.E / ST.E)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::OFF_BAR);
  uint64_t* q_full = bar + 0;       // [2]
  uint64_t* q_empty = bar + 2;      // [2]
  uint64_t* k_full = bar + 4;       // [KST]
  uint64_t* k_empty = bar + 7;      // [KST]
  uint64_t* v_full = bar + 10;      // [VST]
  uint64_t* v_empty = bar + 12;     // [VST]
  uint64_t* s_full = bar + 14;      // [2]
  uint64_t* s_empty = bar + 16;     // [2]
  uint64_t* p_full = bar + 18;
  uint64_t* pv_full = bar + 19;
  uint64_t* ki_full = bar + 20;     // [2] key metadata
  uint64_t* ki_empty = bar + 22;    // [2]
  uint64_t* b_full = bar + 24;      // [2] bias rows
  uint64_t* b_empty = bar + 26;     // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 28);

  // warp index via shfl: provably warp-uniform, so role code can use uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tq);
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1);
      mbar_init(&q_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_empty[s], kSoftThreads);
      mbar_init(&ki_full[s], 32);
      mbar_init(&ki_empty[s], kSoftThreads);
      mbar_init(&b_full[s], kSoftThreads);
    }
    for (int s = 0; s < KST; ++s) {
      mbar_init(&k_full[s], 1);
      mbar_init(&k_empty[s], 1);
    }
    for (int s = 0; s < VST; ++s) {
      mbar_init(&v_full[s], 1);
      mbar_init(&v_empty[s], 1);
    }
    mbar_init(p_full, kSoftThreads);
    mbar_init(pv_full, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, kTmemCols);
  if constexpr (FAST) {
    unsigned char* tab = smem + L::OFF_TAB;
    for (int i = threadIdx.x; i < 384; i += blockDim.x)
      tab[i] = i < 64 ? P.ck_lo[i] : (i < 128 ? P.ck_hi[i - 64] : P.gkt[i - 128]);
    for (int i = threadIdx.x; i < 64; i += blockDim.x) reinterpret_cast<unsigned long long*>(tab + 512)[i] = P.mbmask[i];
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  uint8_t* sQ = smem + L::OFF_Q;
  uint8_t* sK = smem + L::OFF_K;
  uint8_t* sV = smem + L::OFF_V;
  uint8_t* sP = smem + L::OFF_P;
  int2* koff = reinterpret_cast<int2*>(smem + L::OFF_KOFF);
  const int W1 = P.bias_w + 1;
  float* bias_base = reinterpret_cast<float*>(smem + P.off_bias);
  const int bias_stride = 2 * BQ * W1;  // floats per bias buffer (bh rows then bw rows)

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (lane == 0) {
      Cursor<FAST> cu;
      cu.init_tables(smem + L::OFF_TAB);
      cu.start(P);
      while (cu.valid) {
        const int col = cu.h * DH;
        if (cu.first) {
          const int qs = cu.k % P.q_slots;
          const int qn = cu.k / P.q_slots;
          mbar_wait_backoff(&q_empty[qs], (qn & 1) ^ 1);
          mbar_expect_tx(&q_full[qs], L::TX_Q);
          uint8_t* q = sQ + qs * L::TILE;
          tma_load_3d(q, &tq, &q_full[qs], col, cu.mb * BQ, cu.u);
          if constexpr (L::kTail) tma_load_3d(q + L::MAIN, &tq2, &q_full[qs], col + 64, cu.mb * BQ, cu.u);
        }
        const int c = cu.c;
        {
          const int s = c % KST, n = c / KST;
          mbar_wait_backoff(&k_empty[s], (n & 1) ^ 1);
          mbar_expect_tx(&k_full[s], L::TX_KV);
          uint8_t* kk = sK + s * L::TILE;
          tma_load_3d(kk, &tk, &k_full[s], col, cu.cj * BKC, cu.u);
          if constexpr (L::kTail) tma_load_3d(kk + L::MAIN, &tk2, &k_full[s], col + 64, cu.cj * BKC, cu.u);
        }
        {
          const int s = c % VST, n = c / VST;
          mbar_wait_backoff(&v_empty[s], (n & 1) ^ 1);
          mbar_expect_tx(&v_full[s], L::TX_KV);
          uint8_t* vv = sV + s * L::TILE;
          tma_load_3d(vv, &tv, &v_full[s], col, cu.cj * BKC, cu.u);
          if constexpr (L::kTail) tma_load_3d(vv + L::MAIN, &tv2, &v_full[s], col + 64, cu.cj * BKC, cu.u);
        }
        cu.advance(P);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t id_s = idesc_bf16(BQ, BKC);
    constexpr uint32_t id_pv = idesc_bf16(BQ, 64, false, true);
    constexpr uint32_t id_pv2 = idesc_bf16(BQ, 16, false, true);
    // descriptors hoisted out of the issue loop (uniform registers); slots / k-steps are added
    // in 16-byte units and every MMA is issued by one elected lane of this warp
    constexpr uint32_t TILE16 = L::TILE >> 4;
    const uint64_t dq = sdesc_k_sw128(sQ), dqt = sdesc_k_sw32(sQ + L::MAIN);
    const uint64_t dk = sdesc_k_sw128(sK), dkt = sdesc_k_sw32(sK + L::MAIN);
    const uint64_t dp = sdesc_k_sw128(sP);
    const uint64_t dv = sdesc_mn_sw128(sV), dvt = sdesc_mn_sw32(sV + L::MAIN);
    auto issue_s = [&](const Cursor<FAST>& cu) {
      const int qs = cu.k % P.q_slots;
      if (cu.first) mbar_wait_backoff(&q_full[qs], (cu.k / P.q_slots) & 1);
      const int c = cu.c, ks_ = c % KST, st = c & 1;
      mbar_wait_backoff(&k_full[ks_], (c / KST) & 1);
      mbar_wait_backoff(&s_empty[st], ((c >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint64_t q = dq + qs * TILE16, qt = dqt + qs * TILE16;
      const uint64_t kk = dk + ks_ * TILE16, kt = dkt + ks_ * TILE16;
      const uint32_t d = tmem + TM_S + st * 128;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) umma_ss(d, q + 2 * ks, kk + 2 * ks, id_s, ks > 0);
      if constexpr (L::kTail) umma_ss(d, qt, kt, id_s, 1);
      umma_commit_elect(&s_full[st]);
      umma_commit_elect(&k_empty[ks_]);
      if (cu.last) umma_commit_elect(&q_empty[qs]);
    };
    auto issue_pv = [&](const Cursor<FAST>& cu) {
      const int c = cu.c, vs = c % VST;
      mbar_wait_backoff(p_full, c & 1);
      mbar_wait_backoff(&v_full[vs], (c / VST) & 1);
      tc_fence_after();
      const uint64_t v = dv + vs * TILE16, vt = dvt + vs * TILE16;
#pragma unroll
      for (int ks = 0; ks < BKC / 16; ++ks) {
        const uint64_t a = dp + (ks >> 2) * (BQ * 128 / 16) + 2 * (ks & 3);
        const uint32_t acc = (!cu.first || ks > 0) ? 1u : 0u;
        umma_ss(tmem + TM_O, a, v + ks * (16 * 128 / 16), id_pv, acc);
        if constexpr (L::kTail) umma_ss(tmem + TM_O + 64, a, vt + ks * (16 * 32 / 16), id_pv2, acc);
      }
      umma_commit_elect(pv_full);
      umma_commit_elect(&v_empty[vs]);
    };
    Cursor<FAST> cs, cp;
    cs.init_tables(smem + L::OFF_TAB);
    cp.init_tables(smem + L::OFF_TAB);
    cs.start(P);
    cp.start(P);
    for (int i = 0; i < 2 && cs.valid; ++i) {
      issue_s(cs);
      cs.advance(P);
    }
    while (cp.valid) {
      issue_pv(cp);
      cp.advance(P);
      if (cs.valid) {
        issue_s(cs);
        cs.advance(P);
      }
    }
  } else if (warp == 3) {
    // ------------------------------------------------------------ metadata loader
    Cursor<FAST> cu;
    cu.init_tables(smem + L::OFF_TAB);
    cu.start(P);
    while (cu.valid) {
      const int c = cu.c, st = c & 1;
      // the chunk's 128 key indices in flight at once (one memory latency per chunk)
      int ksp[BKC / 32];
#pragma unroll
      for (int i = 0; i < BKC / 32; ++i) {
        const int kg = cu.cj * BKC + lane + 32 * i;
        ksp[i] = kg < P.sk ? __ldg(P.k_sp + (long long)cu.u * P.sk + kg) : -1;
      }
      mbar_wait_backoff(&ki_empty[st], ((c >> 1) & 1) ^ 1);
#pragma unroll
      for (int i = 0; i < BKC / 32; ++i)
        koff[st * BKC + lane + 32 * i] =
            ksp[i] >= 0 ? make_int2((ksp[i] / P.bias_w) * 4, (ksp[i] % P.bias_w) * 4) : make_int2(0, 0);
      mbar_arrive(&ki_full[st]);
      cu.advance(P);
    }
  } else if (warp >= 4) {
    // ------------------------------------------------------------ softmax
    const int sw = warp - 4;
    const int q4 = warp & 3;
    const int half = sw >> 2;      // key half of every chunk this thread owns
    const int r = q4 * 32 + lane;  // row within the item == TMEM lane
    const uint32_t lane_off = (uint32_t)(q4 * 32) << 16;
    float* xmax = reinterpret_cast<float*>(smem + L::OFF_XMAX);  // [chunk parity][half][BQ]
    float* xsum = reinterpret_cast<float*>(smem + L::OFF_XSUM);  // [chunk parity][half][BQ]
    constexpr float L2E = 1.4426950408889634f;
    // lazy rescaling: P and ell stay relative to a reference max that only moves when a
    // row max exceeds it by more than ln(256); O is then rescaled once in TMEM
    constexpr float kRescaleThr = 5.545177444479562f;
    // O columns (32-aligned segments): half 0 -> [0,32) (+ [64,80) for dh 80), half 1 -> [32,64)
    const uint32_t o_addr = tmem + TM_O + lane_off + half * 32;
    const unsigned char* gkt = smem + L::OFF_TAB + 128;

    // stage this thread's bias row (half 0: bh[σq(row)], half 1: bw[σq(row)]) of an item
    auto stage_bias = [&](int u_, int h_, int mb_, int buf) {
      const int rw = mb_ * BQ + r;
      const int sp = P.q_sp[(long long)u_ * P.sq + (rw < P.sq ? rw : P.sq - 1)];
      const float* src = (half ? P.bw : P.bh) + (long long)u_ * P.bias_us + ((long long)h_ * P.sq + sp) * P.bias_w;
      float* dst = bias_base + buf * bias_stride + half * BQ * W1 + r * W1;
      for (int j = 0; j < P.bias_w; ++j) cp_async4(dst + j, src + j);
    };
    // O / ell -> bf16 -> global for a finished item (its last PV must be complete)
    auto epilogue = [&](int u_, int h_, int row_, float inv) {
      long long orow_off = (long long)u_ * P.o_unit_stride + (long long)row_ * P.ldo;
      bool valid = row_ < P.sq;
      if (valid && P.o_rows) {
        const int m = P.o_rows[(long long)u_ * P.sq + row_];
        valid = m >= 0;
        orow_off = (long long)m * P.ldo;
      }
      __nv_bfloat16* dst = P.out + orow_off + h_ * DH;
      {
        uint32_t pr[32];
        tmem_ld32(o_addr, pr);
        tmem_ld_wait();
        if (valid) {
          uint4* d4 = reinterpret_cast<uint4*>(dst + half * 32);
#pragma unroll
          for (int j = 0; j < 4; ++j) d4[j] = scale_pack8(pr + 8 * j, inv);
        }
      }
      if constexpr (DH == 80) {
        if (half == 0) {
          uint32_t p16[16];
          tmem_ld16(tmem + TM_O + lane_off + 64, p16);
          tmem_ld_wait();
          if (valid) {
            uint4* d4 = reinterpret_cast<uint4*>(dst + 64);
            d4[0] = scale_pack8(p16, inv);
            d4[1] = scale_pack8(p16 + 8, inv);
          }
        }
      }
      tc_fence_before();
    };

    Cursor<FAST> cu;
    cu.init_tables(smem + L::OFF_TAB);
    cu.start(P);
    int next_it = P.items;
    if (P.bias_bufs == 2 && cu.valid) {
      stage_bias(cu.u, cu.h, cu.mb, 0);
      cp_async_wait_all();
      mbar_arrive(&b_full[0]);
    }
    float m_ref = -INFINITY, ell = 0.f;
    int diag = 0, row = 0;
    const char* bh_row = nullptr;
    const char* bw_row = nullptr;
    // deferred epilogue of the previous item: runs after the next item's first pass 1,
    // hiding the latency of that item's last PV behind useful work
    bool pend = false;
    int pend_u = 0, pend_h = 0, pend_row = 0, pend_c = 0;
    float pend_ell = 0.f;
    while (cu.valid) {
      const int c = cu.c, st = c & 1;
      if (cu.first) {
        row = cu.mb * BQ + r;
        diag = min(row / P.b_row, P.tc - 1);
        const int bb = cu.k % P.bias_bufs;
        if (P.bias_bufs == 1) {  // stage now; the previous item's readers are past their last exchange barrier
          stage_bias(cu.u, cu.h, cu.mb, 0);
          cp_async_wait_all();
          mbar_arrive(&b_full[0]);
        }
        mbar_wait(&b_full[bb], (cu.k / P.bias_bufs) & 1);
        if (P.bias_bufs == 2) {  // prefetch the next item's rows; completed + published at the end of this item
          next_it = cu.it + gridDim.x;
          if (next_it < P.items) {
            const int nmb_ = next_it % P.nmb, nuh = next_it / P.nmb;
            stage_bias(nuh / P.heads, nuh % P.heads, nmb_, bb ^ 1);
          }
        }
        bh_row = reinterpret_cast<const char*>(bias_base + bb * bias_stride + r * W1);
        bw_row = bh_row + BQ * W1 * 4;
        m_ref = -INFINITY;
        ell = 0.f;
      }
      mbar_wait(&ki_full[st], (c >> 1) & 1);
      const int2* ko = koff + st * BKC + half * 64;
      const int cbase = cu.cj * BKC + half * 64;  // global key index of my first column

      mbar_wait(&s_full[st], (c >> 1) & 1);
      tc_fence_after();
      const uint32_t s_addr = tmem + TM_S + st * 128 + lane_off + half * 64;
      // pass 1: logits = tau*s + bh + bw (masked) written back over S; partial row max
      float mx = -INFINITY;
      unsigned live = 0;  // bit g: key group g has an unmasked column in this warp (warp-uniform)
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        const int c0 = cbase + g * 32;
        bool grp_ok = c0 < P.sk;
        if constexpr (FAST) {
          const int kt = gkt[c0 >> 5];
          grp_ok = grp_ok && ((kt < cu.plan.p) || (kt == diag));
        }
        if (__any_sync(0xffffffffu, grp_ok)) {
          live |= 1u << g;
          uint32_t sr[32];
          tmem_ld32(s_addr + g * 32, sr);
          tmem_ld_wait();
          if constexpr (FAST) {
#pragma unroll
            for (int j = 0; j < 32; j += 2) {
              const int4 oo = *reinterpret_cast<const int4*>(ko + g * 32 + j);
              float x0 = fmaf(P.tau, __uint_as_float(sr[j]), *reinterpret_cast<const float*>(bh_row + oo.x));
              float x1 = fmaf(P.tau, __uint_as_float(sr[j + 1]), *reinterpret_cast<const float*>(bh_row + oo.z));
              x0 += *reinterpret_cast<const float*>(bw_row + oo.y);
              x1 += *reinterpret_cast<const float*>(bw_row + oo.w);
              sr[j] = __float_as_uint(x0);
              sr[j + 1] = __float_as_uint(x1);
            }
            if (c0 + 32 > P.sk) {  // ragged last group (warp-uniform, rare)
#pragma unroll
              for (int j = 0; j < 32; ++j)
                if (c0 + j >= P.sk) sr[j] = __float_as_uint(-INFINITY);
            }
#pragma unroll
            for (int j = 0; j < 32; ++j) mx = fmaxf(mx, __uint_as_float(sr[j]));
          } else {
#pragma unroll 4
            for (int j = 0; j < 32; ++j) {
              const int kg = c0 + j;
              const int kt = kg / P.b_col;
              const bool ok = kg < P.sk && ((kt < cu.plan.p) || (kt == diag));
              const int2 oo = ko[g * 32 + j];
              float x = fmaf(P.tau, __uint_as_float(sr[j]), *reinterpret_cast<const float*>(bh_row + oo.x));
              x += *reinterpret_cast<const float*>(bw_row + oo.y);
              x = ok ? x : -INFINITY;
              mx = fmaxf(mx, x);
              sr[j] = __float_as_uint(x);
            }
          }
          tmem_st32(s_addr + g * 32, sr);
        }
      }
      tmem_st_wait();
      mbar_arrive(&ki_empty[st]);
      float* xm = xmax + st * 2 * BQ;
      float* xs = xsum + st * 2 * BQ;
      xm[half * BQ + r] = mx;
      if (pend) xs[half * BQ + r] = pend_ell;
      named_bar_sync(2, kSoftThreads);
      const float mrow = fmaxf(mx, xm[(half ^ 1) * BQ + r]);
      if (pend) {
        const float inv = 1.0f / (pend_ell + xs[(half ^ 1) * BQ + r]);
        mbar_wait(pv_full, pend_c & 1);
        tc_fence_after();
        epilogue(pend_u, pend_h, pend_row, inv);
        pend = false;
      } else if (!cu.first) {
        mbar_wait(pv_full, (c - 1) & 1);  // O current, P buffer free
        tc_fence_after();
      }
      // reference max: set on the first finite row max, moved only past the threshold
      float alpha = 1.f;
      bool resc = false;
      if (mrow > m_ref + kRescaleThr || (m_ref == -INFINITY && mrow > -INFINITY)) {
        alpha = (m_ref == -INFINITY) ? 0.f : ex2((m_ref - mrow) * L2E);
        resc = !cu.first;
        m_ref = mrow;
      }
      if (__any_sync(0xffffffffu, resc)) {
        uint32_t pr[32];
        tmem_ld32(o_addr, pr);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 32; ++j) pr[j] = __float_as_uint(__uint_as_float(pr[j]) * alpha);
        tmem_st32(o_addr, pr);
        if constexpr (DH == 80) {
          if (half == 0) {
            uint32_t p16[16];
            tmem_ld16(tmem + TM_O + lane_off + 64, p16);
            tmem_ld_wait();
#pragma unroll
            for (int j = 0; j < 16; ++j) p16[j] = __float_as_uint(__uint_as_float(p16[j]) * alpha);
            tmem_st16(tmem + TM_O + lane_off + 64, p16);
          }
        }
        tmem_st_wait();
      }
      const float mb2 = (m_ref == -INFINITY) ? 0.f : m_ref * L2E;
      // pass 2: p = exp(logit - m_ref) -> bf16 P in smem; partial row sum
      float rs = 0.f;
#pragma unroll
      for (int g = 0; g < 2; ++g) {
        uint4 w4[4];
        if (live & (1u << g)) {
          uint32_t sr[32];
          tmem_ld32(s_addr + g * 32, sr);
          tmem_ld_wait();
#pragma unroll
          for (int q8 = 0; q8 < 4; ++q8) {
            float pj[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              pj[j] = ex2(fmaf(__uint_as_float(sr[8 * q8 + j]), L2E, -mb2));
              rs += pj[j];
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
          const int g8 = half * 8 + g * 4 + q8;  // 16-byte chunk index along the 128 keys
          const int a = g8 >> 3, c16 = (g8 & 7) ^ (r & 7);
          *reinterpret_cast<uint4*>(sP + a * (BQ * 128) + r * 128 + c16 * 16) = w4[q8];
        }
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&s_empty[st]);
      mbar_arrive(p_full);
      ell = ell * alpha + rs;

      if (cu.last) {
        if (P.bias_bufs == 2 && next_it < P.items) {
          cp_async_wait_all();
          mbar_arrive(&b_full[(cu.k + 1) & 1]);
        }
        pend = true;
        pend_u = cu.u;
        pend_h = cu.h;
        pend_row = row;
        pend_c = c;
        pend_ell = ell;
      }
      cu.advance(P);
    }
    if (pend) {
      xsum[half * BQ + r] = pend_ell;
      named_bar_sync(3, kSoftThreads);
      const float inv = 1.0f / (pend_ell + xsum[(half ^ 1) * BQ + r]);
      mbar_wait(pv_full, pend_c & 1);
      tc_fence_after();
      epilogue(pend_u, pend_h, pend_row, inv);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc(tmem, kTmemCols);
}

}  // namespace zs

using namespace zs;

int launch_attn_win(const void* q, const void* k, const void* v, long long ldq, long long ldk, long long ldv,
                    long long qus, long long kvus, int units, int heads, int S, int dh, const float* bh,
                    const float* bw, int bias_w, const int* q_sp, const int* k_sp, int b_row, int b_col, int prefix,
                    float tau, void* out, long long ldo, long long ous, const int* o_rows, long long bias_us,
                    const __half* btab_ext, long long btab_us, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_attn_glob(const void* q, const void* k, const void* v, long long ldq, long long ldk, long long ldv,
                     long long qus, long long kvus, int units, int heads, int S, int dh, const float* bh,
                     const float* bw, int bias_w, const int* q_sp, const int* k_sp, int b_row, int b_col, int prefix,
                     float tau, void* out, long long ldo, long long ous, const int* o_rows, long long bias_us,
                     const __half* btab_ext, long long btab_us, void* ws, size_t ws_bytes, cudaStream_t st);
int launch_attn_local(const void* q, const void* k, const void* v, long long ldq, long long ldk, long long ldv,
                      long long qus, long long kvus, int units, int heads, int sq, int sk, int dh, const float* bh,
                      const float* bw, int bias_w, const int* q_sp, const int* k_sp, int b_row, int b_col,
                      int prefix, float tau, void* out, long long ldo, long long ous, const int* o_rows,
                      long long bias_us, cudaStream_t st);
namespace zs {
size_t relpos_r_bytes(int dh, int w);
int launch_relpos(const void* q, long long ldq, long long qus, int units, int heads, int S, int dh, int w,
                  const float* rel_h, const float* rel_w, const int* q_sp, float tau, int mode, __half* btab,
                  long long btab_us, int w16, float* bh, float* bw, void* ws, cudaStream_t st);
}  // namespace zs

template <int DH, bool FAST>
static int launch_attn(const CUtensorMap* m, attn::Params p, cudaStream_t st) {
  using L = attn::Layout<DH>;
  constexpr size_t kMaxSmem = 227 * 1024;
  // prefer: 2 Q slots + 2 bias buffers; then 1 Q slot; then 1 bias buffer
  int qs = 2, bb = 2;
  if (L::smem_bytes(qs, p.bias_w, bb) > kMaxSmem) qs = 1;
  if (L::smem_bytes(qs, p.bias_w, bb) > kMaxSmem) {
    qs = 2;
    bb = 1;
  }
  if (L::smem_bytes(qs, p.bias_w, bb) > kMaxSmem) qs = 1;
  const size_t smem = L::smem_bytes(qs, p.bias_w, bb);
  if (smem > kMaxSmem) return ZS_ERR_SHAPE;
  p.q_slots = qs;
  p.bias_bufs = bb;
  p.off_bias = L::off_bias(qs);
  cudaFuncSetAttribute(zs_attn_kernel<DH, FAST>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int grid = num_sms();
  if (grid > p.items) grid = p.items;
  { zs_attn_kernel<DH, FAST><<<grid, attn::kThreads, smem, st>>>(m[0], m[1], m[2], m[3], m[4], m[5], p); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

template <int DH>
static int launch_attn_dh(const void* q, const void* k, const void* v, long long ldq, long long ldk, long long ldv,
                          long long qus, long long kvus, attn::Params& p, cudaStream_t st) {
  CUtensorMap m[6];
  const uint64_t ncol = (uint64_t)p.heads * DH;
  int rc = 0;
  rc |= make_tmap_3d_bf16(&m[0], q, ncol, p.sq, p.units, ldq, qus, 64, attn::BQ, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  rc |= make_tmap_3d_bf16(&m[2], k, ncol, p.sk, p.units, ldk, kvus, 64, attn::BKC, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  rc |= make_tmap_3d_bf16(&m[4], v, ncol, p.sk, p.units, ldv, kvus, 64, attn::BKC, 1, CU_TENSOR_MAP_SWIZZLE_128B);
  if (DH == 80) {
    rc |= make_tmap_3d_bf16(&m[1], q, ncol, p.sq, p.units, ldq, qus, 16, attn::BQ, 1, CU_TENSOR_MAP_SWIZZLE_32B);
    rc |= make_tmap_3d_bf16(&m[3], k, ncol, p.sk, p.units, ldk, kvus, 16, attn::BKC, 1, CU_TENSOR_MAP_SWIZZLE_32B);
    rc |= make_tmap_3d_bf16(&m[5], v, ncol, p.sk, p.units, ldv, kvus, 16, attn::BKC, 1, CU_TENSOR_MAP_SWIZZLE_32B);
  } else {
    m[1] = m[0];
    m[3] = m[2];
    m[5] = m[4];
  }
  if (rc) return ZS_ERR_TMAP;
  const int nck = (p.sk + attn::BKC - 1) / attn::BKC;
  const int ngroups = (p.sk + 31) / 32;
  const bool fast = (p.b_row % 32) == 0 && (p.b_col % 32) == 0 && nck <= 64 && ngroups <= 256 && p.tc <= 255 &&
                    p.nmb <= 64;
  if (fast) {
    for (int cj = 0; cj < 64; ++cj) {
      const int lo = (cj * attn::BKC) / p.b_col;
      const int hi = std::min((cj * attn::BKC + attn::BKC - 1) / p.b_col, p.tc - 1);
      p.ck_lo[cj] = (unsigned char)std::min(lo, 255);
      p.ck_hi[cj] = (unsigned char)std::max(0, std::min(hi, 255));
    }
    for (int g = 0; g < 256; ++g) p.gkt[g] = (unsigned char)std::min((g * 32) / p.b_col, 255);
    for (int mb = 0; mb < 64; ++mb) {
      unsigned long long msk = 0;
      const int r0 = mb * attn::BQ;
      if (r0 < p.sq) {
        const int dlo = std::min(r0 / p.b_row, p.tc - 1);
        const int dhi = std::min(std::min(r0 + attn::BQ - 1, p.sq - 1) / p.b_row, p.tc - 1);
        for (int cj = 0; cj < nck; ++cj)
          if (p.ck_lo[cj] < p.prefix || !(dhi < p.ck_lo[cj] || dlo > p.ck_hi[cj])) msk |= 1ull << cj;
      }
      p.mbmask[mb] = msk;
    }
    return launch_attn<DH, true>(m, p, st);
  }
  return launch_attn<DH, false>(m, p, st);
}

// Validation + kernel choice shared by every public entry.  bias_us: floats between the bh / bw
// tables of consecutive units (0 = one [heads, S, w] table for all).  btab_ext: precomputed fp16
// operand rows (zs_relpos.cu mode 0) for the window / global kernels; with it only those two are
// tried and 1 is returned when neither accepts the shape.
static int attn_dispatch(const void* q, const void* k, const void* v, long long ldq, long long ldk, long long ldv,
                         long long q_unit_stride, long long kv_unit_stride, int units, int heads, int sq, int sk,
                         int dh, const float* bh, const float* bw, long long bias_us, int bias_w, const int32_t* q_sp,
                         const int32_t* k_sp, int b_row, int b_col, int prefix_tiles, float tau, void* out,
                         long long ldo, long long o_unit_stride, const int32_t* o_rows, const __half* btab_ext,
                         long long btab_us, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (units <= 0 || heads <= 0) return 0;
  if (!q || !k || !v || ((!bh || !bw) && !btab_ext) || !q_sp || !k_sp || !out) return ZS_ERR_ARG;
  if (sq <= 0 || sk <= 0 || b_row <= 0 || b_col <= 0 || bias_w <= 0 || bias_w > 255) return ZS_ERR_SHAPE;
  if (bias_w * bias_w != sk || bias_us < 0) return ZS_ERR_SHAPE;
  if (dh != 64 && dh != 80) return ZS_ERR_SHAPE;
  const int tc = (sk + b_col - 1) / b_col;
  if (prefix_tiles < 0 || prefix_tiles > tc) return ZS_ERR_SHAPE;
  if ((ldq | ldk | ldv | ldo | q_unit_stride | kv_unit_stride | o_unit_stride) & 7) return ZS_ERR_ALIGN;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(k) | reinterpret_cast<uintptr_t>(v) |
       reinterpret_cast<uintptr_t>(out)) & 15)
    return ZS_ERR_ALIGN;
  const long long nmb = (sq + attn::BQ - 1) / attn::BQ;
  const long long items = nmb * heads * (long long)units;
  if (items > 0x7FFFFFFF) return ZS_ERR_SHAPE;
  if (sq <= 256 && sk <= 256 && !getenv("ZS_ATTN_FORCE_GENERIC")) {
    // windows: one-pass TMEM-P kernel (zs_attn_win.cu) when the schedule fits its envelope,
    // else the ping-pong window kernel (zs_attn_local.cu)
    if (sq == sk && !getenv("ZS_ATTN_NO_WIN")) {
      const int rc = launch_attn_win(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, units, heads, sq, dh, bh,
                                     bw, bias_w, q_sp, k_sp, b_row, b_col, prefix_tiles, tau, out, ldo, o_unit_stride,
                                     o_rows, bias_us, btab_ext, btab_us, ws, ws_bytes, st);
      if (rc <= 0 || btab_ext) return rc;
    }
    if (btab_ext) return 1;
    return launch_attn_local(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, units, heads, sq, sk, dh, bh, bw,
                             bias_w, q_sp, k_sp, b_row, b_col, prefix_tiles, tau, out, ldo, o_unit_stride, o_rows,
                             bias_us, st);
  }
  if (sq == sk && !getenv("ZS_ATTN_NO_GLOB")) {  // 128x128 tiles: split-chunk TMEM-P kernel (zs_attn_glob.cu)
    const int rc = launch_attn_glob(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, units, heads, sq, dh, bh, bw,
                                    bias_w, q_sp, k_sp, b_row, b_col, prefix_tiles, tau, out, ldo, o_unit_stride, o_rows,
                                    bias_us, btab_ext, btab_us, ws, ws_bytes, st);
    if (rc <= 0 || btab_ext) return rc;
  }
  if (btab_ext) return 1;
  attn::Params p;
  p.units = units;
  p.heads = heads;
  p.sq = sq;
  p.sk = sk;
  p.bias_w = bias_w;
  p.ldo = ldo;
  p.o_unit_stride = o_unit_stride;
  p.o_rows = o_rows;
  p.bh = bh;
  p.bw = bw;
  p.bias_us = bias_us;
  p.q_sp = q_sp;
  p.k_sp = k_sp;
  p.b_row = b_row;
  p.b_col = b_col;
  p.prefix = prefix_tiles;
  p.tc = tc;
  p.nmb = (int)nmb;
  p.items = (int)items;
  p.tau = tau;
  p.q_slots = 1;
  p.bias_bufs = 1;
  p.off_bias = 0;
  p.out = reinterpret_cast<__nv_bfloat16*>(out);
  if (dh == 64) return launch_attn_dh<64>(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, p, st);
  return launch_attn_dh<80>(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, p, st);
}

// fp16 bias-operand rows the window / global kernels read (built per call from the fp32 tables
// into the caller's workspace): window [tables * heads * S + S, 32] halves (the trailing S rows are
// the one-hot key rows), global [tables * heads * S, 128] halves; tables = units for per-unit
// bias, else 1.  The generic kernels need none.
static size_t attn_ws_bytes(int units, int heads, int sq, int sk, int per_unit) {
  if (units <= 0 || heads <= 0 || sq <= 0 || sk <= 0) return 0;
  const size_t tables = per_unit ? (size_t)units : 1;
  const size_t halves = (sq <= 256 && sk <= 256) ? (tables * heads * sq + sq) * 32 : tables * heads * sq * 128;
  return (halves * sizeof(__half) + 255) & ~(size_t)255;
}

extern "C" size_t zs_stripe_attn_ws_bytes(int units, int heads, int sq, int sk, int dh, int per_unit_bias) {
  if (dh != 64 && dh != 80) return 0;
  return attn_ws_bytes(units, heads, sq, sk, per_unit_bias);
}

extern "C" int zs_stripe_attn_fwd(const void* q, const void* k, const void* v, long long ldq, long long ldk,
                                  long long ldv, long long q_unit_stride, long long kv_unit_stride, int units,
                                  int heads, int sq, int sk, int dh, const float* bh, const float* bw, int bias_w,
                                  const int32_t* q_sp, const int32_t* k_sp, int b_row, int b_col,
                                  int prefix_tiles, float tau, void* out, long long ldo, long long o_unit_stride,
                                  void* ws, size_t ws_bytes, zs_stream_t stream) {
  return attn_dispatch(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, units, heads, sq, sk, dh, bh, bw, 0,
                       bias_w, q_sp, k_sp, b_row, b_col, prefix_tiles, tau, out, ldo, o_unit_stride, nullptr, nullptr,
                       0, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int zs_stripe_attn_fwd_rows(const void* q, const void* k, const void* v, long long ldq, long long ldk,
                                       long long ldv, long long q_unit_stride, long long kv_unit_stride, int units,
                                       int heads, int sq, int sk, int dh, const float* bh, const float* bw,
                                       int bias_w, const int32_t* q_sp, const int32_t* k_sp, int b_row, int b_col,
                                       int prefix_tiles, float tau, void* out, long long ldo,
                                       long long o_unit_stride, const int32_t* o_rows, void* ws, size_t ws_bytes,
                                       zs_stream_t stream) {
  return attn_dispatch(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, units, heads, sq, sk, dh, bh, bw, 0,
                       bias_w, q_sp, k_sp, b_row, b_col, prefix_tiles, tau, out, ldo, o_unit_stride, o_rows, nullptr,
                       0, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

extern "C" int zs_stripe_attn_fwd_unit_bias(const void* q, const void* k, const void* v, long long ldq, long long ldk,
                                            long long ldv, long long q_unit_stride, long long kv_unit_stride,
                                            int units, int heads, int sq, int sk, int dh, const float* bh,
                                            const float* bw, long long bias_unit_stride, int bias_w,
                                            const int32_t* q_sp, const int32_t* k_sp, int b_row, int b_col,
                                            int prefix_tiles, float tau, void* out, long long ldo,
                                            long long o_unit_stride, const int32_t* o_rows, void* ws,
                                            size_t ws_bytes, zs_stream_t stream) {
  return attn_dispatch(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, units, heads, sq, sk, dh, bh, bw,
                       bias_unit_stride, bias_w, q_sp, k_sp, b_row, b_col, prefix_tiles, tau, out, ldo, o_unit_stride,
                       o_rows, nullptr, 0, ws, ws_bytes, reinterpret_cast<cudaStream_t>(stream));
}

// ---------------------------------------------------------------- SAM relative-position mode
static size_t relpos_tables_bytes(int units, int heads, int S, int bias_w) {
  const size_t w16 = S <= 256 ? 32 : 128;
  const size_t op = (size_t)units * heads * S * w16 * 2;           // fp16 operand rows
  const size_t f32 = 2 * (size_t)units * heads * S * bias_w * 4;   // fp32 bh, bw (fallback kernels)
  return ((op > f32 ? op : f32) + 255) & ~(size_t)255;
}

extern "C" size_t zs_relpos_ws_bytes(int units, int heads, int S, int dh, int bias_w) {
  if (units <= 0 || heads <= 0 || bias_w <= 0 || bias_w > 64 || (dh != 64 && dh != 80)) return 0;
  // [R scratch | fp16 operand rows or fp32 tables | the attention's operand workspace (fp32-table path)]
  return relpos_r_bytes(dh, bias_w) + relpos_tables_bytes(units, heads, S, bias_w) +
         attn_ws_bytes(units, heads, S, S, 1);
}

extern "C" int zs_relpos_bias(const void* q, long long ldq, long long q_unit_stride, int units, int heads, int S,
                              int dh, int bias_w, const float* rel_pos_h, const float* rel_pos_w,
                              const int32_t* q_sp, float* bh, float* bw, void* ws, size_t ws_bytes,
                              zs_stream_t stream) {
  if (units <= 0 || heads <= 0) return 0;
  if (!q || !rel_pos_h || !rel_pos_w || !q_sp || !bh || !bw || !ws) return ZS_ERR_ARG;
  if ((dh != 64 && dh != 80) || bias_w <= 0 || bias_w > 64 || bias_w * bias_w != S) return ZS_ERR_SHAPE;
  if (ws_bytes < relpos_r_bytes(dh, bias_w)) return ZS_ERR_SHAPE;
  if (((ldq | q_unit_stride) & 7) || (reinterpret_cast<uintptr_t>(q) & 15) || (reinterpret_cast<uintptr_t>(ws) & 255))
    return ZS_ERR_ALIGN;
  const int rc = launch_relpos(q, ldq, q_unit_stride, units, heads, S, dh, bias_w, rel_pos_h, rel_pos_w, q_sp, 1.0f, 1,
                               nullptr, 0, 0, bh, bw, ws, reinterpret_cast<cudaStream_t>(stream));
  return rc == 1 ? ZS_ERR_SHAPE : rc;
}

extern "C" int zs_stripe_attn_fwd_relpos(const void* q, const void* k, const void* v, long long ldq, long long ldk,
                                         long long ldv, long long q_unit_stride, long long kv_unit_stride, int units,
                                         int heads, int S, int dh, const float* rel_pos_h, const float* rel_pos_w,
                                         int bias_w, const int32_t* q_sp, const int32_t* k_sp, int b_row, int b_col,
                                         int prefix_tiles, float tau, void* out, long long ldo,
                                         long long o_unit_stride, const int32_t* o_rows, void* ws, size_t ws_bytes,
                                         zs_stream_t stream) {
  if (units <= 0 || heads <= 0) return 0;
  if (!rel_pos_h || !rel_pos_w || !ws) return ZS_ERR_ARG;
  if ((dh != 64 && dh != 80) || bias_w <= 0 || bias_w > 64 || bias_w * bias_w != S) return ZS_ERR_SHAPE;
  if (ws_bytes < zs_relpos_ws_bytes(units, heads, S, dh, bias_w)) return ZS_ERR_SHAPE;
  if (reinterpret_cast<uintptr_t>(ws) & 255) return ZS_ERR_ALIGN;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  uint8_t* tables = reinterpret_cast<uint8_t*>(ws) + relpos_r_bytes(dh, bias_w);
  // fast kernels: fp16 operand rows straight from the relpos GEMM epilogue, in the row width
  // the consuming kernel reads (window kernel: 16 + 16 halves, w <= 16; global: 64 + 64)
  const bool fast_shape = (S <= 256) ? (b_row % 32 == 0 && b_col % 32 == 0 && bias_w <= 16)
                                     : (b_row == 128 && b_col == 128);
  if (fast_shape) {
    const int w16 = S <= 256 ? 32 : 128;
    const long long us = (long long)heads * S * w16;
    __half* btab = reinterpret_cast<__half*>(tables);
    int rc = launch_relpos(q, ldq, q_unit_stride, units, heads, S, dh, bias_w, rel_pos_h, rel_pos_w, q_sp, tau, 0,
                           btab, us, w16, nullptr, nullptr, ws, st);
    if (rc < 0) return rc;
    if (rc == 0) {
      rc = attn_dispatch(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, units, heads, S, S, dh, nullptr,
                         nullptr, 0, bias_w, q_sp, k_sp, b_row, b_col, prefix_tiles, tau, out, ldo, o_unit_stride,
                         o_rows, btab, us, tables + relpos_tables_bytes(units, heads, S, bias_w),
                         attn_ws_bytes(units, heads, S, S, 1), st);
      if (rc <= 0) return rc;
    }
  }
  // any other schedule: fp32 per-unit tables, then the kernels that read them
  float* bh = reinterpret_cast<float*>(tables);
  float* bw = bh + (size_t)units * heads * S * bias_w;
  const int rc = zs_relpos_bias(q, ldq, q_unit_stride, units, heads, S, dh, bias_w, rel_pos_h, rel_pos_w, q_sp, bh, bw,
                                ws, relpos_r_bytes(dh, bias_w), stream);
  if (rc) return rc;
  return attn_dispatch(q, k, v, ldq, ldk, ldv, q_unit_stride, kv_unit_stride, units, heads, S, S, dh, bh, bw,
                       (long long)heads * S * bias_w, bias_w, q_sp, k_sp, b_row, b_col, prefix_tiles, tau, out, ldo,
                       o_unit_stride, o_rows, nullptr, 0,
                       tables + relpos_tables_bytes(units, heads, S, bias_w), attn_ws_bytes(units, heads, S, S, 1), st);
}

// zs_order.cu — token-importance scoring and top-K ordering (north-star (3)).
//
//  zs_sobel_saliency: Sobel gradient magnitude of the fp32 encoder input, for
//    the whole grid and for every zero-padded window in one pass over x.
//    Bit-exact with saliency.py:62-82: per pixel the fp32 accumulators are
//    updated channel by channel, taps row-major, each update a single
//    correctly-rounded add of an exact product (coefficients are 0/±1/±2, the
//    zero taps and the zero-padded taps add ±0 and are skipped), and the
//    magnitude is sqrt(gx*gx + gy*gy) with every operation rounded separately.
//  zs_rank_order: z-group energy (saliency.py:85-96, fixed t = 0..3 order),
//    stable descending sort by rank counting (saliency.py:99-118, ties by
//    ascending group index / Morton code, NaN last like numpy), and the stripe
//    interleave sigma[g*(N/G)+t] = pi[t*G+g] (stripesort.py:38-62).
#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {

namespace order {
constexpr int TY = 10, TX = 24;      // output pixels per CTA (70 x 70 padded grid: 3 % idle)
constexpr int kThreads = TY * TX;
constexpr int HY = TY + 2, HX = TX + 2;
constexpr int CC = 16;               // channels staged per pass
constexpr int CCP = CC + 1;          // padded channel stride (bank-conflict free)
}  // namespace order

__global__ void __launch_bounds__(order::kThreads) sobel_kernel(const float* __restrict__ x, int H, int W, int C, int win,
                                                    int Hp, int Wp, int nwx, float* __restrict__ sal_glob,
                                                    float* __restrict__ sal_win) {
  using namespace order;
  __shared__ float tile[HY * HX * CCP];
  const int b = blockIdx.z;
  const int y0 = blockIdx.y * TY, x0 = blockIdx.x * TX;
  const int ty = threadIdx.x / TX, tx = threadIdx.x % TX;
  const int py = y0 + ty, px = x0 + tx;
  const float* xb = x + (long long)b * H * W * C;

  float gxg = 0.f, gyg = 0.f, gxw = 0.f, gyw = 0.f;
  // Taps outside the grid read the zero-filled halo, so they add +-0 exactly like the
  // reference's zero padding (a zero addend changes only the sign of a zero accumulator, which
  // the magnitude squares away); the global map needs no masks.  The window map also drops the
  // taps outside the pixel's window: their values are ANDed with a per-tap bit mask (integer
  // pipe, no predicates per tap and channel), which turns them into +0.
  const bool rok0 = (py % win) != 0, rok2 = (py % win) != win - 1;
  const bool cok0 = (px % win) != 0, cok2 = (px % win) != win - 1;
  uint32_t mw[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const bool ra = a == 0 ? rok0 : (a == 2 ? rok2 : true), cc = c == 0 ? cok0 : (c == 2 ? cok2 : true);
      mw[a][c] = (ra && cc) ? 0xffffffffu : 0u;
    }

  // halo staging, software-pipelined: the 16-byte loads of pass c0 + CC are in flight (in
  // registers) while pass c0 is computed from shared memory
  constexpr int NLD = (HY * HX * (CC / 4) + kThreads - 1) / kThreads;
  const bool vec = (C & 3) == 0 && (C % CC) == 0;
  float4 pre[NLD];
  auto load_pass = [&](int c0) {
#pragma unroll
    for (int k = 0; k < NLD; ++k) {
      const int e = threadIdx.x + kThreads * k;
      pre[k] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (e < HY * HX * (CC / 4)) {
        const int q = e % (CC / 4), pp = e / (CC / 4);
        const int gy = y0 + pp / HX - 1, gx = x0 + pp % HX - 1;
        if (gy >= 0 && gx >= 0 && gy < H && gx < W)
          pre[k] = __ldg(reinterpret_cast<const float4*>(xb + ((long long)gy * W + gx) * C + c0) + q);
      }
    }
  };
  if (vec) load_pass(0);
  for (int c0 = 0; c0 < C; c0 += CC) {
    __syncthreads();
    if (vec) {
#pragma unroll
      for (int k = 0; k < NLD; ++k) {
        const int e = threadIdx.x + kThreads * k;
        if (e < HY * HX * (CC / 4)) {
          float* t = tile + (e / (CC / 4)) * CCP + 4 * (e % (CC / 4));
          t[0] = pre[k].x;
          t[1] = pre[k].y;
          t[2] = pre[k].z;
          t[3] = pre[k].w;
        }
      }
    } else {
      for (int e = threadIdx.x; e < HY * HX * CC; e += kThreads) {
        const int ch = e % CC;
        const int p = e / CC;
        const int hy = p / HX, hx = p % HX;
        const int gy = y0 + hy - 1, gx = x0 + hx - 1;
        float v = 0.f;
        if (gy >= 0 && gx >= 0 && gy < H && gx < W && c0 + ch < C) v = xb[((long long)gy * W + gx) * C + c0 + ch];
        tile[p * CCP + ch] = v;
      }
    }
    __syncthreads();
    if (vec && c0 + CC < C) load_pass(c0 + CC);
    const int cn = min(CC, C - c0);
    for (int ch = 0; ch < cn; ++ch) {
      float v[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) v[a][c] = tile[((ty + a) * HX + (tx + c)) * CCP + ch];
      float u[3][3];
#pragma unroll
      for (int a = 0; a < 3; ++a)
#pragma unroll
        for (int c = 0; c < 3; ++c) u[a][c] = __uint_as_float(__float_as_uint(v[a][c]) & mw[a][c]);
      // taps row-major; gx uses (0,0),(0,2),(1,0),(1,2),(2,0),(2,2); gy rows 0 and 2.  coef * v is
      // exact for coef in {+-1, +-2}, so the single-rounding fma equals the reference's separately
      // rounded multiply-then-add bit for bit
#define ZS_TAP(acc, vv, a, c, coef) acc = __fmaf_rn(coef, vv[a][c], acc);
      ZS_TAP(gxg, v, 0, 0, -1.f) ZS_TAP(gyg, v, 0, 0, -1.f)
      ZS_TAP(gyg, v, 0, 1, -2.f)
      ZS_TAP(gxg, v, 0, 2, 1.f) ZS_TAP(gyg, v, 0, 2, -1.f)
      ZS_TAP(gxg, v, 1, 0, -2.f)
      ZS_TAP(gxg, v, 1, 2, 2.f)
      ZS_TAP(gxg, v, 2, 0, -1.f) ZS_TAP(gyg, v, 2, 0, 1.f)
      ZS_TAP(gyg, v, 2, 1, 2.f)
      ZS_TAP(gxg, v, 2, 2, 1.f) ZS_TAP(gyg, v, 2, 2, 1.f)
      ZS_TAP(gxw, u, 0, 0, -1.f) ZS_TAP(gyw, u, 0, 0, -1.f)
      ZS_TAP(gyw, u, 0, 1, -2.f)
      ZS_TAP(gxw, u, 0, 2, 1.f) ZS_TAP(gyw, u, 0, 2, -1.f)
      ZS_TAP(gxw, u, 1, 0, -2.f)
      ZS_TAP(gxw, u, 1, 2, 2.f)
      ZS_TAP(gxw, u, 2, 0, -1.f) ZS_TAP(gyw, u, 2, 0, 1.f)
      ZS_TAP(gyw, u, 2, 1, 2.f)
      ZS_TAP(gxw, u, 2, 2, 1.f) ZS_TAP(gyw, u, 2, 2, 1.f)
#undef ZS_TAP
    }
  }
  if (py < H && px < W && sal_glob)
    sal_glob[(long long)b * H * W + py * W + px] =
        __fsqrt_rn(__fadd_rn(__fmul_rn(gxg, gxg), __fmul_rn(gyg, gyg)));
  if (py < Hp && px < Wp && sal_win) {
    const int wi = (py / win) * nwx + px / win;
    const int nwin = (Hp / win) * nwx;
    const int i = (py % win) * win + px % win;
    sal_win[((long long)b * nwin + wi) * win * win + i] =
        __fsqrt_rn(__fadd_rn(__fmul_rn(gxw, gxw), __fmul_rn(gyw, gyw)));
  }
}

// numpy lexsort order on (-key, tiebreak): j comes before i?
__device__ __forceinline__ bool ranks_before(float kj, int tj, float ki, int ti) {
  const bool nj = isnan(kj), ni = isnan(ki);
  if (nj || ni) {
    if (nj && ni) return tj < ti;
    return ni;  // non-NaN before NaN
  }
  return kj > ki || (kj == ki && tj < ti);
}

// One CTA per unit.  Dynamic smem: scores[N] | key[N] | tiebreak/rank[N] (ints) | pi[N] (ints)
__global__ void __launch_bounds__(1024) rank_kernel(const float* __restrict__ scores, int scores_are_energy, int N,
                                                    int gran, int gs, int G, int variant,
                                                    const int* __restrict__ morton_fwd, int* __restrict__ sigma,
                                                    float* __restrict__ energy_out) {
  extern __shared__ float sm[];
  float* sc = sm;                                  // [N]
  float* key = sm + N;                             // [N] (energies or token scores)
  int* tie = reinterpret_cast<int*>(sm + 2 * N);   // [N]
  int* pi = reinterpret_cast<int*>(sm + 3 * N);    // [N]
  const int u = blockIdx.x;
  const int tid = threadIdx.x, nt = blockDim.x;
  int* sig = sigma + (long long)u * N;

  if (variant == 2) {  // no_sort: interleave the plain Morton order
    const int per = N / G;
    for (int r = tid; r < N; r += nt) {
      const int gi = r / per, t = r % per;
      sig[r] = morton_fwd[t * G + gi];
    }
    return;
  }

  int nkeys;
  if (gran == 0) {  // zgroup
    nkeys = N / gs;
    if (scores_are_energy) {
      for (int q = tid; q < nkeys; q += nt) key[q] = scores[(long long)u * nkeys + q];
    } else {
      for (int i = tid; i < N; i += nt) sc[i] = scores[(long long)u * N + i];
      __syncthreads();
      for (int q = tid; q < nkeys; q += nt) {
        float e = 0.f;
        for (int t = 0; t < gs; ++t) e = __fadd_rn(e, sc[morton_fwd[q * gs + t]]);
        key[q] = e;
      }
    }
    for (int q = tid; q < nkeys; q += nt) tie[q] = q;
  } else {  // token: key = saliency, tie = Morton rank of the token
    nkeys = N;
    for (int i = tid; i < N; i += nt) key[i] = scores[(long long)u * N + i];
    for (int r = tid; r < N; r += nt) tie[morton_fwd[r]] = r;
  }
  __syncthreads();
  if (energy_out && gran == 0)
    for (int q = tid; q < nkeys; q += nt) energy_out[(long long)u * nkeys + q] = key[q];
  // rank by counting (stable)
  for (int q = tid; q < nkeys; q += nt) {
    const float kq = key[q];
    const int tq = tie[q];
    int rank = 0;
    for (int j = 0; j < nkeys; ++j) rank += ranks_before(key[j], tie[j], kq, tq) ? 1 : 0;
    if (gran == 0) {
      for (int t = 0; t < gs; ++t) pi[rank * gs + t] = morton_fwd[q * gs + t];
    } else {
      pi[rank] = q;
    }
  }
  __syncthreads();
  if (variant == 1) {  // no_interleave
    for (int r = tid; r < N; r += nt) sig[r] = pi[r];
  } else {
    const int per = N / G;
    for (int r = tid; r < N; r += nt) {
      const int gi = r / per, t = r % per;
      sig[r] = pi[t * G + gi];
    }
  }
}

}  // namespace zs

using namespace zs;

extern "C" int zs_sobel_saliency(const float* x, int B, int H, int W, int C, int window, float* sal_glob,
                                 float* sal_win, zs_stream_t stream) {
  if (B <= 0) return 0;
  if (!x || (!sal_glob && !sal_win)) return ZS_ERR_ARG;
  if (H <= 0 || W <= 0 || C <= 0 || window <= 0) return ZS_ERR_SHAPE;
  const int Hp = (H + window - 1) / window * window, Wp = (W + window - 1) / window * window;
  const int nwx = Wp / window;
  dim3 grid((Wp + order::TX - 1) / order::TX, (Hp + order::TY - 1) / order::TY, B);
  { sobel_kernel<<<grid, order::kThreads, 0, reinterpret_cast<cudaStream_t>(stream)>>>(x, H, W, C, window, Hp, Wp, nwx,
                                                                          sal_glob, sal_win); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

extern "C" int zs_rank_order(const float* scores, int scores_are_energy, int U, int N, int granularity,
                             int group_size, int g, int variant, const int32_t* morton_fwd, int32_t* sigma,
                             float* energy, zs_stream_t stream) {
  if (U <= 0) return 0;
  if (!scores || !morton_fwd || !sigma) return ZS_ERR_ARG;
  if (granularity < 0 || granularity > 1 || variant < 0 || variant > 2) return ZS_ERR_ARG;
  if (N <= 0 || g < 1 || N % g) return ZS_ERR_SHAPE;
  if (granularity == 0 && (group_size < 1 || N % group_size)) return ZS_ERR_SHAPE;
  if (scores_are_energy && granularity != 0) return ZS_ERR_ARG;
  const size_t smem = (size_t)4 * N * 4;
  if (smem > 200 * 1024) return ZS_ERR_SHAPE;
  cudaFuncSetAttribute(rank_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int threads = N >= 1024 ? 1024 : ((N + 31) / 32) * 32;
  { rank_kernel<<<U, threads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(
      scores, scores_are_energy, N, granularity, group_size, g, variant, morton_fwd, sigma, energy); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

// zs_rows.cu — HBM-bound row kernels of the hot path: layernorm (+gather),
// row permutation (window partition / σ / layout switches), layout maps,
// prefix keep-set compaction, and the SAM-frame im2col helpers.
//
// All of these are pure data movement or per-row reductions: one warp per
// row, 16-byte vector accesses, grids sized as a multiple of the SM count.
#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {

// ------------------------------------------------------------------ layernorm
// Two-pass per-row LN with population variance (tensor.py:214-236):
//   mean = sum(x)/C; c = x - mean; var = sum(c*c)/C; y = c * (1/sqrt(var+eps)) * g + b
// MAXV = float4 columns per lane (C <= 128*MAXV); exact-width instantiations keep the row in
// as few registers as possible (more rows in flight per SM)
template <bool OUT_F32, int MAXV>
__global__ void __launch_bounds__(256, MAXV <= 10 ? 3 : 2) ln_rows_kernel(const float* __restrict__ x, long long ldx,
                                                      const int* __restrict__ rows,
                                                      const int* __restrict__ out_rows, long long n,
                                                      const int* __restrict__ n_dev, int C,
                                                      const float* __restrict__ g, const float* __restrict__ b,
                                                      float eps, void* out, long long ldo) {
  long long nn = n;
  if (n_dev) nn = min((long long)*n_dev, n);
  const int lane = threadIdx.x & 31;
  const int C4 = C >> 2;
  const long long step = (long long)gridDim.x * 8;
  long long i = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);
  // source row index one row ahead, so a row's data loads never wait on its index load
  long long src_next = (rows && i < nn) ? (long long)__ldg(rows + i) : i;
  for (; i < nn; i += step) {
    const long long src = src_next;
    if (i + step < nn) src_next = rows ? (long long)__ldg(rows + i + step) : i + step;
    const long long dst = out_rows ? (long long)out_rows[i] : i;
    const float4* xr = reinterpret_cast<const float4*>(x + src * ldx);
    float4 v[MAXV];
    float s = 0.f;
#pragma unroll
    for (int j = 0; j < MAXV; ++j) {
      const int c = lane + 32 * j;
      if (c < C4) {
        v[j] = xr[c];
        s += (v[j].x + v[j].y) + (v[j].z + v[j].w);
      } else {
        v[j] = make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    const float mean = s / (float)C;
    float q = 0.f;
#pragma unroll
    for (int j = 0; j < MAXV; ++j) {
      const int c = lane + 32 * j;
      if (c < C4) {
        v[j].x -= mean;
        v[j].y -= mean;
        v[j].z -= mean;
        v[j].w -= mean;
        q += (v[j].x * v[j].x + v[j].y * v[j].y) + (v[j].z * v[j].z + v[j].w * v[j].w);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    const float inv = 1.0f / sqrtf(q / (float)C + eps);
#pragma unroll
    for (int j = 0; j < MAXV; ++j) {
      const int c = lane + 32 * j;
      if (c < C4) {
        const float4 gg = __ldg(reinterpret_cast<const float4*>(g) + c);
        const float4 bb = __ldg(reinterpret_cast<const float4*>(b) + c);
        float4 y;
        y.x = v[j].x * inv * gg.x + bb.x;
        y.y = v[j].y * inv * gg.y + bb.y;
        y.z = v[j].z * inv * gg.z + bb.z;
        y.w = v[j].w * inv * gg.w + bb.w;
        if constexpr (OUT_F32) {
          reinterpret_cast<float4*>(reinterpret_cast<float*>(out) + dst * ldo)[c] = y;
        } else {
          uint2 w;
          w.x = pack_bf16(y.x, y.y);
          w.y = pack_bf16(y.z, y.w);
          reinterpret_cast<uint2*>(reinterpret_cast<__nv_bfloat16*>(out) + dst * ldo)[c] = w;
        }
      }
    }
  }
}

static int grid_for_rows(long long rows, int rows_per_cta) {
  long long g = (rows + rows_per_cta - 1) / rows_per_cta;
  const long long cap = (long long)num_sms() * 16;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

int launch_layernorm(const float* x, long long ldx, const int* rows, const int* out_rows, long long n,
                     const int* n_dev, int C, const float* g, const float* b, float eps, void* out, long long ldo,
                     int out_f32, cudaStream_t st) {
  if (n <= 0) return 0;
  if (!x || !g || !b || !out) return ZS_ERR_ARG;
  if (C <= 0 || C % 4 || C > 2048 || ldx % 4 || (out_f32 ? ldo % 4 : ldo % 4)) return ZS_ERR_SHAPE;
  const int grid = grid_for_rows(n, 8);  // one warp per row, 8 rows per CTA
  const int nv = (C / 4 + 31) / 32;      // float4 per lane
#define ZS_LN(NV)                                                                                          \
  if (out_f32)                                                                                             \
    { ln_rows_kernel<true, NV><<<grid, 256, 0, st>>>(x, ldx, rows, out_rows, n, n_dev, C, g, b, eps, out, ldo); count_launch(); } \
  else                                                                                                     \
    { ln_rows_kernel<false, NV><<<grid, 256, 0, st>>>(x, ldx, rows, out_rows, n, n_dev, C, g, b, eps, out, ldo); count_launch(); }
  if (nv <= 2) {
    ZS_LN(2)
  } else if (nv <= 6) {
    ZS_LN(6)
  } else if (nv <= 8) {
    ZS_LN(8)
  } else if (nv <= 10) {
    ZS_LN(10)
  } else {
    ZS_LN(16)
  }
#undef ZS_LN
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

// ------------------------------------------------------------------ permute
template <typename V>
__global__ void __launch_bounds__(256) permute_rows_kernel(const V* __restrict__ src, V* __restrict__ dst,
                                                           const int* __restrict__ map, long long rows,
                                                           int nvec) {
  const int lane = threadIdx.x & 31;
  for (long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += (long long)gridDim.x * 8) {
    const int s = map[r];
    V* d = dst + r * nvec;
    if (s >= 0) {
      const V* a = src + (long long)s * nvec;
      for (int c = lane; c < nvec; c += 32) d[c] = a[c];
    } else {
      V z;
      memset(&z, 0, sizeof(V));
      for (int c = lane; c < nvec; c += 32) d[c] = z;
    }
  }
}

// ------------------------------------------------------------------ layout maps
__global__ void maps_local_kernel(const int* __restrict__ sig_loc, int B, int H, int W, int win, int nwx, int nwin,
                                  int* l_from_s, int* s_from_l, unsigned char* l_is_pad) {
  const long long S2 = (long long)win * win;
  const long long total = (long long)B * nwin * S2;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < total;
       r += (long long)gridDim.x * blockDim.x) {
    const int i = (int)(r % S2);
    const long long bw = r / S2;
    const int w = (int)(bw % nwin);
    const int b = (int)(bw / nwin);
    const int t = sig_loc[r];
    const int y = (w / nwx) * win + t / win;
    const int x = (w % nwx) * win + t % win;
    (void)i;
    if (y < H && x < W) {
      const int s = b * H * W + y * W + x;
      if (l_from_s) l_from_s[r] = s;
      if (s_from_l) s_from_l[s] = (int)r;
      if (l_is_pad) l_is_pad[r] = 0;
    } else {
      if (l_from_s) l_from_s[r] = -1;
      if (l_is_pad) l_is_pad[r] = 1;
    }
  }
}
__global__ void maps_global_kernel(const int* __restrict__ sig_glob, int B, int HW, int* s_from_g, int* g_from_s) {
  const long long total = (long long)B * HW;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < total;
       g += (long long)gridDim.x * blockDim.x) {
    const int b = (int)(g / HW);
    const int s = b * HW + sig_glob[g];
    if (s_from_g) s_from_g[s] = (int)g;
    if (g_from_s) g_from_s[g] = s;
  }
}

// fp32 rows -> bf16 rows through a row map (pads / negative map -> zeros)
__global__ void __launch_bounds__(256) permute_f32_bf16_kernel(const float4* __restrict__ src,
                                                               uint2* __restrict__ dst,
                                                               const int* __restrict__ map, long long rows,
                                                               int nvec) {
  const int lane = threadIdx.x & 31;
  for (long long r = (long long)blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += (long long)gridDim.x * 8) {
    const int s = map ? map[r] : (int)r;
    uint2* d = dst + r * nvec;
    for (int c = lane; c < nvec; c += 32) {
      uint2 w = make_uint2(0u, 0u);
      if (s >= 0) {
        const float4 v = src[(long long)s * nvec + c];
        w.x = pack_bf16(v.x, v.y);
        w.y = pack_bf16(v.z, v.w);
      }
      d[c] = w;
    }
  }
}
__global__ void maps_cross_kernel(const int* __restrict__ sig_glob, int B, int HW, long long nl,
                                  const int* __restrict__ s_from_l, const int* __restrict__ s_from_g,
                                  const int* __restrict__ l_from_s, int* g_from_l, int* l_from_g) {
  const long long ng = (long long)B * HW;
  const long long total = ng > nl ? ng : nl;
  for (long long r = blockIdx.x * (long long)blockDim.x + threadIdx.x; r < total;
       r += (long long)gridDim.x * blockDim.x) {
    if (r < ng && g_from_l) {
      const int b = (int)(r / HW);
      g_from_l[r] = s_from_l[(long long)b * HW + sig_glob[r]];
    }
    if (r < nl && l_from_g) {
      const int s = l_from_s[r];
      l_from_g[r] = s >= 0 ? s_from_g[s] : -1;
    }
  }
}

// ------------------------------------------------------------------ keep rows
// counts[u] = # non-pad rows among rows [k0, k1) of unit u
__global__ void keep_count_kernel(int U, int S, int k0, int k1, const unsigned char* __restrict__ is_pad,
                                  int* counts) {
  const int lane = threadIdx.x & 31;
  for (int u = blockIdx.x * 8 + (threadIdx.x >> 5); u < U; u += gridDim.x * 8) {
    int c = 0;
    for (int i = k0 + lane; i < k1; i += 32) c += is_pad ? (is_pad[(long long)u * S + i] == 0) : 1;
#pragma unroll
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if (lane == 0) counts[u] = c;
  }
}
// In-place exclusive scan of counts[0..U) by one CTA; counts[U] = total.
__global__ void __launch_bounds__(1024) keep_scan_kernel(int U, int* counts) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  for (int base = 0; base < U; base += 1024) {
    const int i = base + threadIdx.x;
    const int v = i < U ? counts[i] : 0;
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) warp_sums[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      int ws = warp_sums[lane];
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int t = __shfl_up_sync(0xffffffffu, ws, o);
        if (lane >= o) ws += t;
      }
      warp_sums[lane] = ws;
    }
    __syncthreads();
    const int excl = carry + (wid ? warp_sums[wid - 1] : 0) + incl - v;
    if (i < U) counts[i] = excl;
    __syncthreads();
    if (threadIdx.x == 0) carry += warp_sums[31];
    __syncthreads();
  }
  if (threadIdx.x == 0) counts[U] = carry;
}
__global__ void keep_write_kernel(int U, int S, int k0, int k1, const unsigned char* __restrict__ is_pad,
                                  const int* __restrict__ offsets, int* keep_rows) {
  const int lane = threadIdx.x & 31;
  for (int u = blockIdx.x * 8 + (threadIdx.x >> 5); u < U; u += gridDim.x * 8) {
    int pos = offsets[u];
    for (int i0 = k0; i0 < k1; i0 += 32) {
      const int i = i0 + lane;
      const long long r = (long long)u * S + i;
      const bool keep = i < k1 && (!is_pad || is_pad[r] == 0);
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (keep) keep_rows[pos + __popc(m & ((1u << lane) - 1u))] = (int)r;
      pos += __popc(m);
    }
  }
}

// ------------------------------------------------------------------ SAM frame
__global__ void patchify_kernel(const float* __restrict__ img, int B, int Cin, int H, int W, int P,
                                __nv_bfloat16* __restrict__ out) {
  const int gh = H / P, gw = W / P;
  const long long ncol = (long long)Cin * P * P;
  const long long total = (long long)B * gh * gw * ncol;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long row = e / ncol;
    const int col = (int)(e % ncol);
    const int c = col / (P * P), ky = (col / P) % P, kx = col % P;
    const int b = (int)(row / (gh * gw));
    const int t = (int)(row % (gh * gw));
    const int y = (t / gw) * P + ky, x = (t % gw) * P + kx;
    out[e] = __float2bfloat16_rn(img[(((long long)b * Cin + c) * H + y) * W + x]);
  }
}
// Vectorised patchify for P % 8 == 0 (SAM: P = 16): one thread moves one P-pixel image row
// segment of one patch (P floats in, P bf16 out, contiguous on both sides).  Consecutive
// threads take consecutive patches along x, so a warp reads 32 adjacent segments of one image
// row (coalesced) and writes whole 16-byte chunks of 32 patch rows.
template <int P>
__global__ void patchify_vec_kernel(const float* __restrict__ img, int B, int Cin, int H, int W,
                                    __nv_bfloat16* __restrict__ out) {
  const int gw = W / P, gh = H / P;
  const long long total = (long long)B * Cin * H * gw;
  const int ncol = Cin * P * P;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int tx = (int)(e % gw);
    const long long r1 = e / gw;  // (b * Cin + c) * H + y
    const int y = (int)(r1 % H);
    const long long bc = r1 / H;
    const int c = (int)(bc % Cin), b = (int)(bc / Cin);
    const float4* src = reinterpret_cast<const float4*>(img + r1 * W + (long long)tx * P);
    const long long row = ((long long)b * gh + y / P) * gw + tx;
    uint4* dst = reinterpret_cast<uint4*>(out + row * ncol + c * P * P + (y % P) * P);
#pragma unroll
    for (int q = 0; q < P / 8; ++q) {
      const float4 a = __ldg(src + 2 * q), d = __ldg(src + 2 * q + 1);
      dst[q] = make_uint4(pack_bf16(a.x, a.y), pack_bf16(a.z, a.w), pack_bf16(d.x, d.y), pack_bf16(d.z, d.w));
    }
  }
}

// 3x3 / stride 1 / pad 1 im2col of channels-last bf16 rows, TAP-MAJOR columns:
// out[row, (ky*3 + kx)*C + c] = x[b, y+ky-1, x+kx-1, c] (zeros outside).  One thread moves 8
// channels (16 bytes): reads and writes are contiguous runs of C channels.
__global__ void im2col3x3_kernel(const __nv_bfloat16* __restrict__ x, int B, int H, int W, int C,
                                 __nv_bfloat16* __restrict__ out) {
  const int cv = C >> 3;  // 16-byte vectors per pixel
  const long long total = (long long)B * H * W * 9 * cv;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const int v = (int)(e % cv);
    const long long rt = e / cv;
    const int tap = (int)(rt % 9);
    const long long row = rt / 9;
    const int b = (int)(row / (H * W)), t = (int)(row % (H * W));
    const int y = t / W + tap / 3 - 1, xx = t % W + tap % 3 - 1;
    uint4 val = make_uint4(0u, 0u, 0u, 0u);
    if (y >= 0 && y < H && xx >= 0 && xx < W)
      val = reinterpret_cast<const uint4*>(x + (((long long)b * H + y) * W + xx) * C)[v];
    reinterpret_cast<uint4*>(out + row * 9LL * C + (long long)tap * C)[v] = val;
  }
}

// map[rows[i]] = i for i < n (n = *n_dev when given); map must be pre-filled with -1
__global__ void invert_rows_kernel(const int* __restrict__ rows, long long n, const int* __restrict__ n_dev,
                                   int* __restrict__ map) {
  long long nn = n;
  if (n_dev) nn = min((long long)*n_dev, n);
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nn; i += (long long)gridDim.x * blockDim.x)
    map[rows[i]] = (int)i;
}
// dst[r, :] = src_row for every r with flag[r] != 0 (16-byte vectors): one warp per row, so
// unflagged rows cost one byte read
__global__ void fill_flagged_rows_kernel(uint4* __restrict__ dst, long long ld_vec, const uint4* __restrict__ src,
                                         const uint8_t* __restrict__ flag, long long rows, int nvec) {
  const int lane = threadIdx.x & 31;
  const long long w0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long r = w0; r < rows; r += nw) {
    if (!flag[r]) continue;
    for (int v = lane; v < nvec; v += 32) dst[r * ld_vec + v] = __ldg(src + v);
  }
}

}  // namespace zs

// ================================================================== C ABI
using namespace zs;

static inline cudaStream_t S(zs_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

extern "C" int zs_layernorm_rows(const float* x, long long ldx, const int32_t* rows, long long n, int C,
                                 const float* gamma, const float* beta, float eps, void* out, long long ldo,
                                 int out_f32, zs_stream_t stream) {
  return launch_layernorm(x, ldx, rows, nullptr, n, nullptr, C, gamma, beta, eps, out, ldo, out_f32, S(stream));
}

extern "C" int zs_layernorm_rows_ex(const float* x, long long ldx, const int32_t* rows, const int32_t* out_rows,
                                    long long n, const int32_t* n_dev, int C, const float* gamma, const float* beta,
                                    float eps, void* out, long long ldo, int out_f32, zs_stream_t stream) {
  return launch_layernorm(x, ldx, rows, out_rows, n, n_dev, C, gamma, beta, eps, out, ldo, out_f32, S(stream));
}

extern "C" int zs_permute_rows_f32(const float* src, float* dst, const int32_t* map, long long rows_out, int C,
                                   zs_stream_t stream) {
  if (rows_out <= 0) return 0;
  if (!src || !dst || !map) return ZS_ERR_ARG;
  if (C <= 0 || C % 4) return ZS_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) return ZS_ERR_ALIGN;
  { permute_rows_kernel<float4><<<grid_for_rows(rows_out, 8), 256, 0, S(stream)>>>(
      reinterpret_cast<const float4*>(src), reinterpret_cast<float4*>(dst), map, rows_out, C / 4); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

extern "C" int zs_permute_rows_bf16(const void* src, void* dst, const int32_t* map, long long rows_out, int C,
                                    zs_stream_t stream) {
  if (rows_out <= 0) return 0;
  if (!src || !dst || !map) return ZS_ERR_ARG;
  if (C <= 0 || C % 8) return ZS_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst)) & 15) return ZS_ERR_ALIGN;
  { permute_rows_kernel<uint4><<<grid_for_rows(rows_out, 8), 256, 0, S(stream)>>>(
      reinterpret_cast<const uint4*>(src), reinterpret_cast<uint4*>(dst), map, rows_out, C / 8); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

extern "C" int zs_permute_rows_f32_bf16(const float* src, void* dst, const int32_t* map, long long rows_out, int C,
                                        zs_stream_t stream) {
  if (rows_out <= 0) return 0;
  if (!src || !dst) return ZS_ERR_ARG;
  if (C <= 0 || C % 4) return ZS_ERR_SHAPE;
  if ((reinterpret_cast<uintptr_t>(src) & 15) || (reinterpret_cast<uintptr_t>(dst) & 7)) return ZS_ERR_ALIGN;
  { permute_f32_bf16_kernel<<<grid_for_rows(rows_out, 8), 256, 0, S(stream)>>>(
      reinterpret_cast<const float4*>(src), reinterpret_cast<uint2*>(dst), map, rows_out, C / 4); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

extern "C" int zs_layout_maps(const int32_t* sigma_glob, const int32_t* sigma_loc, int B, int H, int W, int window,
                              int32_t* l_from_s, int32_t* g_from_l, int32_t* l_from_g, int32_t* s_from_g,
                              int32_t* s_from_l, int32_t* g_from_s, uint8_t* l_is_pad, zs_stream_t stream) {
  if (B <= 0 || H <= 0 || W <= 0 || window <= 0) return ZS_ERR_SHAPE;
  const int nwy = (H + window - 1) / window, nwx = (W + window - 1) / window;
  const int nwin = nwy * nwx;
  const long long nl = (long long)B * nwin * window * window;
  const int HW = H * W;
  const int grid = num_sms() * 4;
  if ((g_from_l || l_from_g) && (!sigma_glob || !sigma_loc || !s_from_l || !s_from_g || !l_from_s))
    return ZS_ERR_ARG;
  if (sigma_loc) { maps_local_kernel<<<grid, 256, 0, S(stream)>>>(sigma_loc, B, H, W, window, nwx, nwin, l_from_s,
                                                                 s_from_l, l_is_pad); count_launch(); }
  if (sigma_glob && (s_from_g || g_from_s))
    { maps_global_kernel<<<grid, 256, 0, S(stream)>>>(sigma_glob, B, HW, s_from_g, g_from_s); count_launch(); }
  if (g_from_l || l_from_g)
    { maps_cross_kernel<<<grid, 256, 0, S(stream)>>>(sigma_glob, B, HW, nl, s_from_l, s_from_g, l_from_s, g_from_l,
                                                    l_from_g); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

// rows must hold U*(k1-k0) entries; unit_offsets must hold U+1 entries and
// receives the exclusive prefix of per-unit selected counts (total at [U]).
extern "C" int zs_unit_span_rows(int U, int S_, int k0, int k1, const uint8_t* is_pad, int32_t* rows,
                                 int32_t* unit_offsets, zs_stream_t stream) {
  if (U <= 0) return 0;
  if (k0 < 0 || k1 < k0 || k1 > S_ || !rows || !unit_offsets) return ZS_ERR_ARG;
  const int grid = grid_for_rows(U, 8);
  { keep_count_kernel<<<grid, 256, 0, S(stream)>>>(U, S_, k0, k1, is_pad, unit_offsets); count_launch(); }
  { keep_scan_kernel<<<1, 1024, 0, S(stream)>>>(U, unit_offsets); count_launch(); }
  { keep_write_kernel<<<grid, 256, 0, S(stream)>>>(U, S_, k0, k1, is_pad, unit_offsets, rows); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

extern "C" int zs_prefix_keep_rows(int U, int S_, int K, const uint8_t* is_pad, int32_t* keep_rows,
                                   int32_t* unit_offsets, zs_stream_t stream) {
  if (K <= 0) return ZS_ERR_ARG;
  return zs_unit_span_rows(U, S_, 0, K, is_pad, keep_rows, unit_offsets, stream);
}

extern "C" int zs_patchify(const float* img, int B, int Cin, int H, int W, int P, void* out, zs_stream_t stream) {
  if (B <= 0) return 0;
  if (!img || !out || P <= 0 || H % P || W % P) return ZS_ERR_SHAPE;
  if (P == 16 && (reinterpret_cast<uintptr_t>(img) & 15) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0)
    { patchify_vec_kernel<16><<<num_sms() * 8, 256, 0, S(stream)>>>(img, B, Cin, H, W,
                                                                 reinterpret_cast<__nv_bfloat16*>(out)); count_launch(); }
  else
    { patchify_kernel<<<num_sms() * 8, 256, 0, S(stream)>>>(img, B, Cin, H, W, P,
                                                           reinterpret_cast<__nv_bfloat16*>(out)); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

extern "C" int zs_im2col3x3(const void* x, int B, int H, int W, int C, void* out, zs_stream_t stream) {
  if (B <= 0) return 0;
  if (!x || !out) return ZS_ERR_ARG;
  if (C % 8 || (reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out)) & 15) return ZS_ERR_ALIGN;
  { im2col3x3_kernel<<<num_sms() * 8, 256, 0, S(stream)>>>(reinterpret_cast<const __nv_bfloat16*>(x), B, H, W, C,
                                                          reinterpret_cast<__nv_bfloat16*>(out)); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

extern "C" int zs_invert_rows(const int32_t* rows, long long n, const int32_t* n_dev, int32_t* map, long long map_len,
                              zs_stream_t stream) {
  if (map_len <= 0) return 0;
  if (!map || (n > 0 && !rows)) return ZS_ERR_ARG;
  if (cudaMemsetAsync(map, 0xFF, (size_t)map_len * sizeof(int32_t), S(stream)) != cudaSuccess) return ZS_ERR_LAUNCH;
  if (n > 0) { invert_rows_kernel<<<grid_for_rows(n, 256), 256, 0, S(stream)>>>(rows, n, n_dev, map); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

extern "C" int zs_fill_flagged_rows_bf16(void* dst, long long ld, const void* src_row, const uint8_t* flag,
                                         long long rows, int ncol, zs_stream_t stream) {
  if (rows <= 0) return 0;
  if (!dst || !src_row || !flag) return ZS_ERR_ARG;
  if (ncol % 8 || ld % 8 || (reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src_row)) & 15)
    return ZS_ERR_ALIGN;
  const int nvec = ncol / 8;
  { fill_flagged_rows_kernel<<<num_sms() * 8, 256, 0, S(stream)>>>(reinterpret_cast<uint4*>(dst), ld / 8,
                                                                 reinterpret_cast<const uint4*>(src_row), flag, rows,
                                                                 nvec); count_launch(); }
  return cudaGetLastError() == cudaSuccess ? 0 : ZS_ERR_LAUNCH;
}

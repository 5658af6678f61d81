/* zstripe_b200.h — C ABI of the B200-native SparseSAM encoder hot path.
 *
 * Drop-in boundary for the reference `zstripe` package (/root/reference/pkg/src/zstripe,
 * pure numpy).  Each entry point below replaces one reference function on the
 * hot path named by BASELINE.json `north_star`; the citation after every
 * declaration is the reference interface it stands in for.
 *
 * Conventions (all entry points):
 *   - returns ZS_OK (0) or a negative zs_status; never throws, never aborts;
 *   - asynchronous on `stream` (a cudaStream_t; NULL = legacy default stream);
 *   - every buffer is caller-allocated device memory, workspaces included (sized by the
 *     matching *_ws_bytes query, 256-byte aligned); the library never allocates;
 *   - reentrant: no mutable global state besides a lazily-resolved driver symbol and the
 *     cached SM count; a workspace must not be shared by calls that may run concurrently;
 *   - graph-capturable: no entry point synchronises or allocates, so calls may be recorded
 *     into a CUDA graph (the captured graph keeps the caller's pointers);
 *   - bf16 buffers are `void*` (IEEE bfloat16, little endian), indices are int32.
 * Only sm_100a (B200) is supported; there is no CPU fallback.
 */
#ifndef ZSTRIPE_B200_H_
#define ZSTRIPE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define ZS_API __attribute__((visibility("default")))
#else
#define ZS_API
#endif

typedef struct CUstream_st* zs_stream_t;

enum zs_status {
  ZS_OK = 0,
  ZS_ERR_ARG = -1,         /* bad enum / null pointer                        */
  ZS_ERR_SHAPE = -2,       /* extents violate a kernel constraint            */
  ZS_ERR_ALIGN = -3,       /* pointer / leading dimension misaligned         */
  ZS_ERR_LAUNCH = -4,      /* CUDA launch failure (see cudaGetLastError)     */
  ZS_ERR_TMAP = -5,        /* cuTensorMapEncodeTiled rejected the operand    */
  ZS_ERR_DEVICE = -6,      /* no sm_100 device / driver symbol unavailable   */
  ZS_ERR_WORKSPACE = -7    /* workspace NULL or below the *_ws_bytes query   */
};

/* Human-readable text for a zs_status value. */
ZS_API const char* zs_status_string(int status);
/* ABI version (major*100 + minor).  2.00: caller-owned attention workspaces (ws, ws_bytes). */
ZS_API int zs_abi_version(void);
/* Kernels this library has launched from the calling thread so far (a per-thread counter; the
 * host reads it around calls to count exactly what a composite entry point launched). */
ZS_API unsigned long long zs_launch_counter(void);

/* ------------------------------------------------------------------ ordering
 * Sobel gradient-magnitude saliency of an fp32 token grid x[B, H, W, C]
 * (zero padding), bit-exact with the reference accumulation order
 * (channels ascending, taps row-major, magnitude sqrt(gx*gx + gy*gy) with
 * separately rounded products).
 *   sal_glob  [B, H, W]          saliency over the whole grid     (or NULL)
 *   sal_win   [B, nwin, window^2] saliency of every zero-padded window, the
 *             window border zero-padded, windows row-major over the grid padded
 *             up to multiples of `window`                       (or NULL)
 * replaces: saliency.py:62-82 `sobel_magnitude`, as called by
 *           encoder.py:257-275 `_orderings` (global map and per padded window). */
ZS_API int zs_sobel_saliency(const float* x, int B, int H, int W, int C, int window, float* sal_glob, float* sal_win,
                      zs_stream_t stream);

/* Descending-importance order + stripe interleave for U independent units of N
 * tokens each.  `scores` [U, N] are per-token saliency (row-major spatial order
 * of the unit's grid) when `scores_are_energy` == 0, or per-group energies
 * [U, N/group_size] when 1 (the "fed the reference's scores" gate).
 *   granularity 0 = zgroup, 1 = token;   variant 0 = full, 1 = no_interleave, 2 = no_sort
 *   morton_fwd [N]  token index at each Morton rank of the unit grid (grid.py:98-104)
 *   sigma      [U, N] output: token index at each scan rank (Permutation.forward)
 *   energy     [U, N/group_size] optional output of the group energies
 * replaces: saliency.py:85-118 `group_energy` / `importance_order`,
 *           stripesort.py:38-62 `stripe_sort`. */
ZS_API int zs_rank_order(const float* scores, int scores_are_energy, int U, int N, int granularity, int group_size, int g,
                  int variant, const int32_t* morton_fwd, int32_t* sigma, float* energy, zs_stream_t stream);

/* --------------------------------------------------------- permute / partition
 * dst[r, :] = map[r] >= 0 ? src[map[r], :] : 0      (rows of C elements)
 * One kernel for window∘σ partition (pads -> map -1 -> zeros), σ⁻¹∘unpartition∘crop
 * and the local<->global layout switches.
 * replaces: grid.py:107-112 `apply_permutation`, encoder.py:232-254
 *           `_pad_grid` / `_split_windows` / `_merge_windows` and the crop at :366-368. */
ZS_API int zs_permute_rows_f32(const float* src, float* dst, const int32_t* map, long long rows_out, int C,
                        zs_stream_t stream);
ZS_API int zs_permute_rows_bf16(const void* src, void* dst, const int32_t* map, long long rows_out, int C,
                         zs_stream_t stream);
/* Same gather, fp32 rows in, bf16 rows out (map may be NULL = identity): the cast
 * that feeds a bf16 GEMM operand from the fp32 residual stream. */
ZS_API int zs_permute_rows_f32_bf16(const float* src, void* dst, const int32_t* map, long long rows_out, int C,
                             zs_stream_t stream);

/* Row maps between the three token layouts of a batch of B images on an
 * H x W grid with `window` windows (nwin = ceil(H/window)*ceil(W/window)):
 *   S  spatial      rows b*H*W + y*W + x
 *   L  local        rows (b*nwin + w)*window^2 + i, token sigma_loc[b,w,i] of window w
 *   G  global       rows b*H*W + i, token sigma_glob[b,i]
 * Outputs (each may be NULL):
 *   l_from_s [B*nwin*window^2]  S row feeding L row, -1 for pads
 *   g_from_l [B*H*W]            L row feeding G row
 *   l_from_g [B*nwin*window^2]  G row feeding L row, -1 for pads
 *   s_from_g [B*H*W]            G row feeding S row
 *   s_from_l [B*H*W]            L row feeding S row
 *   g_from_s [B*H*W]            S row feeding G row
 *   l_is_pad [B*nwin*window^2]  1 for pad rows of L
 * replaces: the per-block permute / inverse-permute in encoder.py:297-306, :343-368. */
ZS_API int zs_layout_maps(const int32_t* sigma_glob, const int32_t* sigma_loc, int B, int H, int W, int window,
                   int32_t* l_from_s, int32_t* g_from_l, int32_t* l_from_g, int32_t* s_from_g, int32_t* s_from_l,
                   int32_t* g_from_s, uint8_t* l_is_pad, zs_stream_t stream);

/* Prefix keep-set rows for RC-MLP routing in a σ-ordered layout: unit u owns
 * rows [u*S, (u+1)*S); its first K rows are kept unless is_pad (may be NULL) marks them.
 * Writes the kept row ids (ascending) to keep_rows [U*K]; unit_offsets [U+1]
 * receives the exclusive prefix of per-unit kept counts, the total at [U]
 * (usable directly as the device-side n_keep of zs_rc_mlp_fwd).
 * replaces: mlp.py:73-75,107 `keep_count` + `sigma.forward[:K]`. */
ZS_API int zs_prefix_keep_rows(int U, int S, int K, const uint8_t* is_pad, int32_t* keep_rows, int32_t* unit_offsets,
                        zs_stream_t stream);
/* Generalisation: rows [begin, end) of every unit, pads skipped (the bypass set is
 * the span [K, S)).  rows holds U*(end-begin) entries. */
/* Inverse of a row list: map[rows[i]] = i for i < n (n = min(*n_dev, n) when n_dev != NULL),
 * every other entry of map[0..map_len) = -1.  Used for the compacted output rows of the
 * window attention (zs_stripe_attn_fwd_rows) when window pad tokens are skipped. */
ZS_API int zs_invert_rows(const int32_t* rows, long long n, const int32_t* n_dev, int32_t* map, long long map_len,
                          zs_stream_t stream);
/* dst[r, 0..ncol) = src_row[0..ncol) for every row r < rows with flag[r] != 0 (bf16, ncol % 8 == 0).
 * Broadcasts the constant QKV row of the zero-padded window tokens (LN(0) = beta). */
ZS_API int zs_fill_flagged_rows_bf16(void* dst, long long ld, const void* src_row, const uint8_t* flag,
                                     long long rows, int ncol, zs_stream_t stream);
ZS_API int zs_unit_span_rows(int U, int S, int begin, int end, const uint8_t* is_pad, int32_t* rows,
                             int32_t* unit_offsets, zs_stream_t stream);

/* ------------------------------------------------------------------ layernorm
 * out[i, :] = LN(x[rows ? rows[i] : i, :]) * gamma + beta  (population variance),
 * out is bf16 (out_f32 == 0) or fp32 (out_f32 == 1; may alias x when rows maps i->i).
 * replaces: tensor.py:214-236 `layernorm` (as used at encoder.py:289, mlp.py:82,110). */
ZS_API int zs_layernorm_rows(const float* x, long long ldx, const int32_t* rows, long long n, int C, const float* gamma,
                      const float* beta, float eps, void* out, long long ldo, int out_f32, zs_stream_t stream);
/* Extended form: output row i goes to out_rows[i] (NULL = i) and only the first
 * min(n, *n_dev) rows are processed when n_dev is given (device-side count). */
ZS_API int zs_layernorm_rows_ex(const float* x, long long ldx, const int32_t* rows, const int32_t* out_rows, long long n,
                         const int32_t* n_dev, int C, const float* gamma, const float* beta, float eps, void* out,
                         long long ldo, int out_f32, zs_stream_t stream);

/* --------------------------------------------------------------------- GEMM
 * tcgen05 GEMM  D = A[M,K] · W[N,K]^T  (bf16, fp32 accumulate) with fused epilogue:
 *   epi 0: out_bf16 = D + bias            epi 1: out_bf16 = gelu(D + bias)
 *   epi 2: out_f32[row_map?row_map[m]:m] = res[res_mod? m%res_mod : row] + D + bias,
 *          zero_rows[m] -> row written as zeros.
 * m_dev (optional): device-side row count; rows >= *m_dev are skipped (M is the upper bound).
 * Constraints: K % 64 == 0, N % 32 == 0, 16-byte aligned operands.
 * replaces: tensor.py:189-211 `matmul` (+ the adds at encoder.py:290,307, mlp.py:82-85). */
ZS_API int zs_gemm_bf16(int epi, const void* A, long long lda, const void* W, long long ldw, int M, int N, int K,
                 const float* bias, void* out, long long ld_out, const float* res, long long ld_res,
                 const int32_t* row_map, const uint8_t* zero_rows, int res_mod, const int32_t* m_dev,
                 zs_stream_t stream);

/* ------------------------------------------------------- stripe-sort attention
 * Static block-sparse A-shape attention over `units` independent sequences and
 * `heads` heads, inputs already in scan (σ) order:
 *   q [units][Sq][ldq] bf16 (head h at columns h*dh), k/v [units][Sk][ldk/ldv]
 *   bh, bw  [heads][Sq][bias_w] fp32 decomposed rel-pos tables (shared by units)
 *   q_sp [units][Sq], k_sp [units][Sk]  spatial index of every scan row (σ.forward)
 *   tiles b_row x b_col, active key tiles J_i = {0..prefix-1} ∪ {min(i, Tc-1)}
 *   logits = tau*q·k + bh[q_sp, k_sp / w] + bw[q_sp, k_sp % w]
 *   out [units][Sq][ldo] bf16, head h at columns h*dh
 * dh must be 64 or 80.  Unit strides are in elements.  ws: caller-owned device workspace of at
 * least zs_stripe_attn_ws_bytes(units, heads, sq, sk, dh, 0) bytes, 256-byte aligned; the fp16
 * bias operand rows the tensor-core kernels read are built into it per call.
 * replaces: attention.py:167-221 `ashape_attention` (and :88-104 `build_active_set`). */
ZS_API size_t zs_stripe_attn_ws_bytes(int units, int heads, int sq, int sk, int dh, int per_unit_bias);
ZS_API int zs_stripe_attn_fwd(const void* q, const void* k, const void* v, long long ldq, long long ldk, long long ldv,
                       long long q_unit_stride, long long kv_unit_stride, int units, int heads, int sq, int sk,
                       int dh, const float* bh, const float* bw, int bias_w, const int32_t* q_sp,
                       const int32_t* k_sp, int b_row, int b_col, int prefix_tiles, float tau, void* out,
                       long long ldo, long long o_unit_stride, void* ws, size_t ws_bytes, zs_stream_t stream);
/* Same, with an output row map: row r of unit u goes to out row o_rows[u*sq + r] (head h at
 * columns h*dh), or is not written when o_rows[...] < 0 (o_rows == NULL: the layout above).
 * Lets a caller write only the query rows it keeps (e.g. skip SAM's window pad tokens,
 * whose outputs the reference crops, encoder.py:366-368) into a compacted buffer. */
ZS_API int zs_stripe_attn_fwd_rows(const void* q, const void* k, const void* v, long long ldq, long long ldk,
                            long long ldv, long long q_unit_stride, long long kv_unit_stride, int units, int heads,
                            int sq, int sk, int dh, const float* bh, const float* bw, int bias_w,
                            const int32_t* q_sp, const int32_t* k_sp, int b_row, int b_col, int prefix_tiles,
                            float tau, void* out, long long ldo, long long o_unit_stride, const int32_t* o_rows,
                            void* ws, size_t ws_bytes, zs_stream_t stream);

/* Same as zs_stripe_attn_fwd_rows with one bias table pair PER UNIT: bh / bw of unit u start at
 * u * bias_unit_stride floats (each [heads, S, w], spatial-position rows as above).  The
 * reference's BiasTables (attention.py:28-55) generalised to per-window / per-image tables.
 * ws >= zs_stripe_attn_ws_bytes(units, heads, sq, sk, dh, 1) bytes. */
ZS_API int zs_stripe_attn_fwd_unit_bias(const void* q, const void* k, const void* v, long long ldq, long long ldk,
                                        long long ldv, long long q_unit_stride, long long kv_unit_stride, int units,
                                        int heads, int sq, int sk, int dh, const float* bh, const float* bw,
                                        long long bias_unit_stride, int bias_w, const int32_t* q_sp,
                                        const int32_t* k_sp, int b_row, int b_col, int prefix_tiles, float tau,
                                        void* out, long long ldo, long long o_unit_stride, const int32_t* o_rows,
                                        void* ws, size_t ws_bytes, zs_stream_t stream);

/* ------------------------------------------------ SAM decomposed relative position (q-dependent)
 * SAM's add_decomposed_rel_pos (not in the reference, whose bias tables are static: SURVEY §8(f)
 * row 2).  For every unit u, head h and query row r (spatial s = q_sp[u, r] = (qy, qx) of a
 * w x w grid, S == w * w):
 *   bh[u, h, s, ky] = q[u, r, h*dh : (h+1)*dh] . rel_pos_h[qy - ky + w - 1, :]
 *   bw[u, h, s, kx] = q[u, r, h*dh : (h+1)*dh] . rel_pos_w[qx - kx + w - 1, :]
 * rel_pos_h / rel_pos_w: fp32 [2w - 1, dh] (shared by the heads); q bf16 rows as in
 * zs_stripe_attn_fwd (unscaled).  bf16 tensor-core products with fp32 accumulation.
 * ws: >= zs_relpos_ws_bytes(...) bytes, 256-byte aligned (zs_relpos_bias needs the first
 * 32 KB only).  w <= 64, dh 64 / 80. */
ZS_API size_t zs_relpos_ws_bytes(int units, int heads, int S, int dh, int bias_w);
ZS_API int zs_relpos_bias(const void* q, long long ldq, long long q_unit_stride, int units, int heads, int S, int dh,
                          int bias_w, const float* rel_pos_h, const float* rel_pos_w, const int32_t* q_sp, float* bh,
                          float* bw, void* ws, size_t ws_bytes, zs_stream_t stream);
/* Stripe-sort attention with SAM's q-dependent decomposed bias: the bias operand rows are
 * computed by a tcgen05 GEMM (q . [rel_pos_h; rel_pos_w]^T) straight into the attention kernels'
 * fp16 operand layout (no fp32 table round trip); other arguments as zs_stripe_attn_fwd_rows
 * with sq == sk == S. */
ZS_API int zs_stripe_attn_fwd_relpos(const void* q, const void* k, const void* v, long long ldq, long long ldk,
                                     long long ldv, long long q_unit_stride, long long kv_unit_stride, int units,
                                     int heads, int S, int dh, const float* rel_pos_h, const float* rel_pos_w,
                                     int bias_w, const int32_t* q_sp, const int32_t* k_sp, int b_row, int b_col,
                                     int prefix_tiles, float tau, void* out, long long ldo, long long o_unit_stride,
                                     const int32_t* o_rows, void* ws, size_t ws_bytes, zs_stream_t stream);

/* ------------------------------------------------------------------- RC-MLP
 * Residual-consistency MLP on an fp32 residual stream x[rows, C] in place:
 *   kept rows  (keep_rows[0..n_keep)):  x += fc2(gelu(fc1(LN(x)) + b1)) + b2
 *   bypass rows (bypass_mode 1 only, bypass_rows[0..n_bypass)): x = LN(x),
 *               n_bypass = n_bypass_dev ? min(*n_bypass_dev, max_bypass) : max_bypass
 * n_keep = n_keep_dev ? min(*n_keep_dev, max_keep) : max_keep (device-side count,
 * so a data-dependent keep-set needs no host synchronisation).
 * w1 [hidden, C], w2 [C, hidden] bf16; workspace ws >= max_keep*(C+hidden) bf16.
 * replaces: mlp.py:88-114 `route_mlp` (and :78-85 `mlp_forward`). */
ZS_API int zs_rc_mlp_fwd(float* x, long long ldx, const int32_t* keep_rows, int max_keep, const int32_t* n_keep_dev,
                  int C, int hidden, const float* ln_g, const float* ln_b, float eps, const void* w1,
                  const float* b1, const void* w2, const float* b2, int bypass_mode, const int32_t* bypass_rows,
                  int max_bypass, const int32_t* n_bypass_dev, void* ws, zs_stream_t stream);

/* ------------------------------------------------------- SAM frame helpers
 * im2col for non-overlapping PxP patches of an fp32 NCHW image batch:
 *   out [B*(H/P)*(W/P), 3*P*P] bf16, column order (c, ky, kx) = Conv2d weight flattening. */
ZS_API int zs_patchify(const float* img, int B, int Cin, int H, int W, int P, void* out, zs_stream_t stream);
/* 3x3 / pad 1 im2col of a channels-last bf16 map [B, H, W, C] -> [B*H*W, 9*C], tap-major column
 * order (ky, kx, c) (contiguous channel runs); the matching weight is Conv2d's [O, C, 3, 3]
 * permuted to [O, 3, 3, C].  C % 8 == 0, 16-byte aligned pointers. */
ZS_API int zs_im2col3x3(const void* x, int B, int H, int W, int C, void* out, zs_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* ZSTRIPE_B200_H_ */

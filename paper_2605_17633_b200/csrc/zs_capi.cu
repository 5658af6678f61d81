// zs_capi.cu — C ABI glue: status strings, device queries, TMA descriptor
// encoding, the GEMM entry point and the composite RC-MLP (gather-LN ->
// fc1+GELU -> fc2+scatter-add residual).
#include <cudaTypedefs.h>

#include <mutex>

#include "zs_common.cuh"
#include "zs_host.h"

namespace zs {

static thread_local unsigned long long t_launches = 0;
void count_launch() { ++t_launches; }

int num_sms() {
  static int cached[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return kNumSMs;
  if (!cached[dev]) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = kNumSMs;
    cached[dev] = n;
  }
  return cached[dev];
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int make_tmap_2d_bf16(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems,
                      uint32_t box_inner, uint32_t box_outer, CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) return ZS_ERR_DEVICE;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : ZS_ERR_TMAP;
}

int make_tmap_3d_bf16(CUtensorMap* m, const void* ptr, uint64_t d0, uint64_t d1, uint64_t d2, uint64_t ld1_elems,
                      uint64_t ld2_elems, uint32_t b0, uint32_t b1, uint32_t b2, CUtensorMapSwizzle swz) {
  auto fn = encode_fn();
  if (!fn) return ZS_ERR_DEVICE;
  if (d2 == 1 || ld2_elems < ld1_elems * d1) ld2_elems = ld1_elems * d1;  // single unit: stride is irrelevant
  cuuint64_t dims[3] = {d0, d1, d2};
  cuuint64_t strides[2] = {ld1_elems * 2, ld2_elems * 2};
  cuuint32_t box[3] = {b0, b1, b2};
  cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, swz, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? 0 : ZS_ERR_TMAP;
}

}  // namespace zs

using namespace zs;

extern "C" const char* zs_status_string(int status) {
  switch (status) {
    case ZS_OK: return "ok";
    case ZS_ERR_ARG: return "invalid argument (null pointer or bad enum)";
    case ZS_ERR_SHAPE: return "extents violate a kernel constraint";
    case ZS_ERR_ALIGN: return "pointer or leading dimension misaligned (16-byte rule)";
    case ZS_ERR_LAUNCH: return "CUDA kernel launch failed";
    case ZS_ERR_TMAP: return "cuTensorMapEncodeTiled rejected an operand";
    case ZS_ERR_DEVICE: return "no usable sm_100 device / driver entry point";
    case ZS_ERR_WORKSPACE: return "workspace missing or smaller than the *_ws_bytes query";
    default: return "unknown zs_status";
  }
}

extern "C" int zs_abi_version(void) { return 200; }

extern "C" unsigned long long zs_launch_counter(void) { return t_launches; }

extern "C" int zs_gemm_bf16(int epi, const void* A, long long lda, const void* W, long long ldw, int M, int N,
                            int K, const float* bias, void* out, long long ld_out, const float* res,
                            long long ld_res, const int32_t* row_map, const uint8_t* zero_rows, int res_mod,
                            const int32_t* m_dev, zs_stream_t stream) {
  if (!A || !W || !out) return ZS_ERR_ARG;
  GemmEpi ep{bias, out, ld_out, res, ld_res, row_map, m_dev, zero_rows, res_mod};
  return launch_gemm(epi, A, lda, W, ldw, M, N, K, ep, reinterpret_cast<cudaStream_t>(stream), 0);
}

extern "C" int zs_rc_mlp_fwd(float* x, long long ldx, const int32_t* keep_rows, int max_keep,
                             const int32_t* n_keep_dev, int C, int hidden, const float* ln_g, const float* ln_b,
                             float eps, const void* w1, const float* b1, const void* w2, const float* b2,
                             int bypass_mode, const int32_t* bypass_rows, int max_bypass,
                             const int32_t* n_bypass_dev, void* ws, zs_stream_t stream) {
  if (!x || !keep_rows || !ln_g || !ln_b || !w1 || !w2 || !ws) return ZS_ERR_ARG;
  if (bypass_mode != 0 && bypass_mode != 1) return ZS_ERR_ARG;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  __nv_bfloat16* hln = reinterpret_cast<__nv_bfloat16*>(ws);           // [max_keep, C]
  __nv_bfloat16* hid = hln + (size_t)max_keep * C;                       // [max_keep, hidden]
  int rc;
  if (max_keep > 0) {
    rc = launch_layernorm(x, ldx, keep_rows, nullptr, max_keep, n_keep_dev, C, ln_g, ln_b, eps, hln, C, 0, st);
    if (rc) return rc;
  }
  if (bypass_mode == 1 && max_bypass > 0) {
    if (!bypass_rows) return ZS_ERR_ARG;
    // x[bypass] = LN(x[bypass]) in place: per-row read-then-write, rows disjoint from keep_rows
    rc = launch_layernorm(x, ldx, bypass_rows, bypass_rows, max_bypass, n_bypass_dev, C, ln_g, ln_b, eps, x, ldx, 1,
                          st);
    if (rc) return rc;
  }
  if (max_keep <= 0) return 0;
  GemmEpi e1{b1, hid, hidden, nullptr, 0, nullptr, n_keep_dev, nullptr, 0};
  rc = launch_gemm(1, hln, C, w1, C, max_keep, hidden, C, e1, st, 0);
  if (rc) return rc;
  GemmEpi e2{b2, x, ldx, x, ldx, keep_rows, n_keep_dev, nullptr, 0};
  return launch_gemm(2, hid, hidden, w2, hidden, max_keep, C, hidden, e2, st, 0);
}

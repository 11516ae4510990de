#include <cstdlib>
#include <cstdio>
// Host side of the tcgen05 GEMM: TMA descriptor encoding + launch dispatch.
#include <cudaTypedefs.h>

#include <mutex>

#include "gemm_tcgen05.cuh"
#include "sf_internal.h"

namespace sf {

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// Row-major bf16 matrix [outer, inner] -> 2-D tiled map with a (box_inner x
// box_outer) box; box_inner * 2 bytes must equal the swizzle width (32/64/128).
int make_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
                      uint32_t box_inner, uint32_t box_outer, int swizzle_bytes) {
  auto fn = encode_fn();
  if (!fn) return SF_ERR_CUDA;
  CUtensorMapSwizzle sw = swizzle_bytes == 128  ? CU_TENSOR_MAP_SWIZZLE_128B
                          : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                          : swizzle_bytes == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                                : CU_TENSOR_MAP_SWIZZLE_NONE;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? SF_OK : SF_ERR_CUDA;
}

int gemm_bk(int bn) { return bn > 256 ? 32 : 64; }
int gemm_b_box_rows(int bn) { return bn > 256 ? bn / 2 : bn; }

// 2-SM pair tiles: each CTA loads BN/2 rows of W per stage.

int make_operand_maps(GemmMaps* m, const void* A, int64_t M, int64_t K, const void* W, int64_t N, int bn, int ctas) {
  const int bk = gemm_bk(bn);
  int rc = make_tmap_bf16_2d(&m->a, A, K, M, K, bk, 128, 2 * bk);
  rc |= make_tmap_bf16_2d(&m->b, W, K, N, K, bk, gemm_b_box_rows(bn) / ctas, 2 * bk);
  return rc == SF_OK ? SF_OK : SF_ERR_CUDA;
}

// Output map of a row-major bf16 [rows, cols] matrix for the 32-row x 64-column
// epilogue chunks (128B swizzle).
int make_out_map(CUtensorMap* m, const void* D, int64_t rows, int64_t cols) {
  return make_tmap_bf16_2d(m, D, cols, rows, cols, 64, 32, 128);
}

// Output map for the RES_LN epilogue: 32-row x 32-column chunks (64B swizzle).
int make_out_map32(CUtensorMap* m, const void* D, int64_t rows, int64_t cols) {
  return make_tmap_bf16_2d(m, D, cols, rows, cols, 32, 32, 64);
}

// QKV outputs: Q, K [rows*H*T, hd] and V^T [rows*H*hd, T].
//   hd 64: 32-token x 64-dim chunks (Q/K 128B swizzle, V^T 64B swizzle)
//   hd 72: whole heads, Q/K box 72 x 32 unswizzled (144-byte rows), V^T box 32 x 72 (64B swizzle)
int make_qkv_out_maps(GemmMaps* m, const void* q, const void* k, const void* vt, int64_t rows, int heads, int T,
                      int hd) {
  const int64_t bh = rows * heads;
  int rc;
  if (hd == 64) {
    rc = make_tmap_bf16_2d(&m->d[0], q, 64, bh * T, 64, 64, 32, 128);
    rc |= make_tmap_bf16_2d(&m->d[1], k, 64, bh * T, 64, 64, 32, 128);
    rc |= make_tmap_bf16_2d(&m->d[2], vt, T, bh * 64, T, 32, 64, 64);
  } else if (hd == 72) {
    rc = make_tmap_bf16_2d(&m->d[0], q, 72, bh * T, 72, 72, 32, 0);
    rc |= make_tmap_bf16_2d(&m->d[1], k, 72, bh * T, 72, 72, 32, 0);
    rc |= make_tmap_bf16_2d(&m->d[2], vt, T, bh * 72, T, 32, 72, 64);
  } else {
    return SF_ERR_PARAMETER;
  }
  return rc == SF_OK ? SF_OK : SF_ERR_CUDA;
}

// QKV tile width for head dim 64: 192 columns (3 heads per tile, 4 epilogue warps); with
// K = 384 the tiles run on CTA pairs (256 x 192, B resident: gemm_tcgen05.cuh GemmCfg::B_RES).
int qkv_bn64() { return 192; }
int qkv_ctas(int64_t K) { return K == 64 * GemmCfg<192, 8, EPI_QKV, 2>::KB_RES ? 2 : 1; }

template <int BN, int KIND, int CTAS = 1>
constexpr int epi_warps() {
  // QKV: 4 (pair tiles: 8 = two groups of 4 draining alternate tiles); RES_LN: 12;
  // RES with 192-wide tiles: 12 (64 columns per thread); bf16 / GELU with 256-wide tiles:
  // 16 (4 per TMEM lane quarter); else 8
  return KIND == EPI_QKV ? (BN == 192 ? (CTAS == 2 ? 8 : 4) : BN == 128 ? 8 : 4)
         : KIND == EPI_RES_LN ? 12
         : (KIND == EPI_RES && BN == 192) ? 12
         : ((KIND == EPI_BF16 || KIND == EPI_GELU) && BN == 256) ? 16 : 8;
}

// Whether the epilogue of (BN, KIND) stages 32-column chunks (output map: make_out_map32).
int gemm_narrow_out(int bn, int kind) {
  return (kind == EPI_RES_LN || kind == EPI_RES_LN2 || ((kind == EPI_BF16 || kind == EPI_GELU) && bn == 256)) ? 1 : 0;
}

template <int BN, int KIND, int CTAS = 1>
static int set_attr() {
  static bool done = false;
  if (!done) {
    constexpr int W = epi_warps<BN, KIND, CTAS>();
    using C = GemmCfg<BN, W, KIND, CTAS>;
    const cudaError_t err = cudaFuncSetAttribute(gemm_bf16_tcgen05<BN, KIND, W, CTAS>,
                                                 cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_BYTES);
    if (err != cudaSuccess) {
      fprintf(stderr, "streamflow: gemm<%d,%d,%d> smem attribute (%d B) failed: %s\n", BN, KIND, CTAS, C::SMEM_BYTES,
              cudaGetErrorString(err));
      return SF_ERR_CUDA;
    }
    done = true;
  }
  return SF_OK;
}


// Set every instantiation's smem attribute up front (never inside a graph capture).
int prepare_gemm_kernels() {
  int rc = SF_OK;
  rc |= set_attr<128, EPI_F32>();
  rc |= set_attr<128, EPI_BF16>();
  rc |= set_attr<128, EPI_GELU>();
  rc |= set_attr<256, EPI_F32>();
  rc |= set_attr<256, EPI_BF16>();
  rc |= set_attr<256, EPI_GELU>();
  rc |= set_attr<192, EPI_QKV>();
  rc |= set_attr<192, EPI_QKV, 2>();
  rc |= set_attr<144, EPI_QKV, 2>();
  rc |= set_attr<256, EPI_GELU, 2>();
  rc |= set_attr<192, EPI_RES, 2>();
  rc |= set_attr<128, EPI_QKV>();
  rc |= set_attr<384, EPI_RES_LN>();
  rc |= set_attr<144, EPI_QKV>();
  rc |= set_attr<128, EPI_RES>();
  rc |= set_attr<192, EPI_RES_LN2>();
  return rc;
}


static int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int BN, int KIND, int CTAS = 1>
static int launch_one(const GemmMaps& maps, int M, int N, int K, const EpiParams& ep, cudaStream_t st) {
  constexpr int W = epi_warps<BN, KIND, CTAS>();
  using C = GemmCfg<BN, W, KIND, CTAS>;
  if (K % C::BK) return SF_ERR_PARAMETER;
  if (C::B_RES && K != C::KB_RES * C::BK) return SF_ERR_PARAMETER;
  if (set_attr<BN, KIND, CTAS>() != SF_OK) return SF_ERR_CUDA;
  const int tiles = (N / BN) * ((M + C::BM - 1) / C::BM);
  const int grid = tiles < sm_count() ? tiles : sm_count();
  EpiParams e = ep;
  e.M = M;
  e.pdl = g_pdl ? 1 : 0;
  cudaError_t err;
  if constexpr (CTAS == 2) {
    const int num_n = N / BN, pair_tiles = num_n * ((M + 2 * C::BM - 1) / (2 * C::BM));
    int pairs = sm_count() / 2;
    if (pairs > pair_tiles) pairs = pair_tiles;
    if (C::B_RES) {  // a multiple of N / BN pairs, so every pair keeps one column slice
      pairs -= pairs % num_n;
      if (pairs < num_n) pairs = num_n;
    }
    err = launch_kernel_cl(gemm_bf16_tcgen05<BN, KIND, W, CTAS>, dim3((unsigned)(2 * pairs)), dim3(C::THREADS),
                           C::SMEM_BYTES, st, 2u, maps, N, K, e);
    if (err == cudaSuccess) err = cudaGetLastError();
  } else if constexpr (KIND == EPI_RES_LN2) {
    // one cluster of XCH_CL CTAs per row tile in flight: grid = whole clusters
    const int rows = (M + C::BM - 1) / C::BM, max_cl = sm_count() / XCH_CL;
    err = launch_kernel_cl(gemm_bf16_tcgen05<BN, KIND, W>, dim3((unsigned)(XCH_CL * (rows < max_cl ? rows : max_cl))),
                           dim3(C::THREADS), C::SMEM_BYTES, st, (unsigned)XCH_CL, maps, N, K, e);
    if (err == cudaSuccess) err = cudaGetLastError();
  } else {
    err = launch_kernel(gemm_bf16_tcgen05<BN, KIND, W>, dim3(grid), dim3(C::THREADS), C::SMEM_BYTES, st, maps, N,
                           K, e);
    if (err == cudaSuccess) err = cudaGetLastError();
  }
  if (err != cudaSuccess) {
    fprintf(stderr, "streamflow: gemm<%d,%d> launch failed: %s (smem %d, threads %d)\n", BN, KIND,
            cudaGetErrorString(err), C::SMEM_BYTES, C::THREADS);
    return SF_ERR_CUDA;
  }
  return SF_OK;
}



int launch_gemm(int kind, int bn, const GemmMaps& maps, int M, int N, int K, const EpiParams& ep,
                cudaStream_t st, int ctas) {
  if (K % 32 != 0 || N % bn != 0 || M <= 0) return SF_ERR_PARAMETER;
  if (ctas == 2) {
    if (bn == 192 && kind == EPI_QKV) return launch_one<192, EPI_QKV, 2>(maps, M, N, K, ep, st);
    if (bn == 144 && kind == EPI_QKV) return launch_one<144, EPI_QKV, 2>(maps, M, N, K, ep, st);
    if (bn == 256 && kind == EPI_GELU) return launch_one<256, EPI_GELU, 2>(maps, M, N, K, ep, st);
    if (bn == 192 && kind == EPI_RES) return launch_one<192, EPI_RES, 2>(maps, M, N, K, ep, st);
    return SF_ERR_PARAMETER;
  }
#define SF_CASE(BN_, KIND_) \
  if (bn == BN_ && kind == KIND_) return launch_one<BN_, KIND_>(maps, M, N, K, ep, st);
  SF_CASE(128, EPI_F32)
  SF_CASE(128, EPI_BF16)
  SF_CASE(128, EPI_GELU)
  SF_CASE(256, EPI_F32)
  SF_CASE(256, EPI_BF16)
  SF_CASE(256, EPI_GELU)
  SF_CASE(192, EPI_QKV)
  SF_CASE(128, EPI_QKV)
  SF_CASE(384, EPI_RES_LN)
  SF_CASE(144, EPI_QKV)
  SF_CASE(128, EPI_RES)
  SF_CASE(192, EPI_RES_LN2)
#undef SF_CASE
  return SF_ERR_PARAMETER;
}

}  // namespace sf

#if SF_GEMM_TRACE
extern "C" int sf_gemm_trace_read(long long* dst) {
  return cudaMemcpyFromSymbol(dst, sf::g_gemm_trace, sizeof(long long) * 8 * 64) == cudaSuccess ? 0 : -1;
}
extern "C" int sf_gemm_cta_end_read(unsigned long long* dst) {
  return cudaMemcpyFromSymbol(dst, sf::g_gemm_cta_end, sizeof(unsigned long long) * 1024) == cudaSuccess ? 0 : -1;
}
#endif

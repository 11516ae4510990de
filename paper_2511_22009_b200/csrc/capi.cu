// Misc C-ABI entry points: version, device query, standalone GEMM.
#include "gemm_tcgen05.cuh"
#include "sf_internal.h"

using namespace sf;

extern "C" {

const char* sf_version(void) { return "streamflow-b200 0.1 (sm_100a, tcgen05)"; }

int sf_device_sm_count(void) {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return SF_ERR_CUDA;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return SF_ERR_CUDA;
  return n;
}

int sf_gemm_bf16(const void* A, const void* W, const float* bias, void* C, int64_t M, int64_t N, int64_t K,
                 int32_t epi, void* stream) {
  if (M < 1 || N < 1 || K < 64 || K % 64 || N % 128) return SF_ERR_PARAMETER;
  if (epi < EPI_F32 || epi > EPI_GELU) return SF_ERR_PARAMETER;
  const int bn = (N % 256 == 0) ? 256 : 128;
  CUtensorMap ta, tb;
  if (make_tmap_bf16_2d(&ta, A, K, M, K, 64, 128) != SF_OK) return SF_ERR_CUDA;
  if (make_tmap_bf16_2d(&tb, W, K, N, K, 64, gemm_b_box_rows(bn)) != SF_OK) return SF_ERR_CUDA;
  EpiParams ep{};
  ep.bias = bias;
  ep.out = C;
  ep.ldo = N;
  ep.tokens_per_slot = 1 << 30;
  ep.M = (int)M;
  return launch_gemm(epi, bn, ta, tb, (int)M, (int)N, (int)K, ep, (cudaStream_t)stream);
}

int sf_gemm_qkv(const void* A, const void* W, const float* bias, void* q, void* k, void* vt, int64_t M, int32_t heads,
                int32_t T, float q_scale, void* stream) {
  const int64_t d = (int64_t)heads * 64, N = 3 * d, K = d;
  if (M < 1 || M % T || T % 128 || N % 192 || K % 64) return SF_ERR_PARAMETER;
  CUtensorMap ta, tb;
  if (make_tmap_bf16_2d(&ta, A, K, M, K, 64, 128) != SF_OK) return SF_ERR_CUDA;
  if (make_tmap_bf16_2d(&tb, W, K, N, K, 64, gemm_b_box_rows(192)) != SF_OK) return SF_ERR_CUDA;
  EpiParams ep{};
  ep.bias = bias;
  ep.q = (__nv_bfloat16*)q;
  ep.k = (__nv_bfloat16*)k;
  ep.vt = (__nv_bfloat16*)vt;
  ep.heads = heads;
  ep.q_scale = q_scale;
  ep.tokens_per_slot = T;
  ep.M = (int)M;
  return launch_gemm(EPI_QKV, 192, ta, tb, (int)M, (int)N, (int)K, ep, (cudaStream_t)stream);
}

int sf_gemm_res_ln(const void* A, const void* W, const float* bias, void* xres, void* xmod, const float* gate,
                   const float* shift, const float* scale, int64_t vec_stride, int64_t M, int64_t N, int64_t K,
                   int32_t tokens_per_slot, float ln_eps, void* stream) {
  if (N != 384 || K % 64 || M < 1 || M % tokens_per_slot || tokens_per_slot % 128) return SF_ERR_PARAMETER;
  CUtensorMap ta, tb;
  if (make_tmap_bf16_2d(&ta, A, K, M, K, 64, 128) != SF_OK) return SF_ERR_CUDA;
  if (make_tmap_bf16_2d(&tb, W, K, N, K, 64, gemm_b_box_rows(384)) != SF_OK) return SF_ERR_CUDA;
  EpiParams ep{};
  ep.bias = bias;
  ep.xres = (__nv_bfloat16*)xres;
  ep.xmod = (__nv_bfloat16*)xmod;
  ep.gate = gate;
  ep.shift = shift;
  ep.scale = scale;
  ep.vec_stride = vec_stride;
  ep.ln_eps = ln_eps;
  ep.tokens_per_slot = tokens_per_slot;
  ep.M = (int)M;
  return launch_gemm(EPI_RES_LN, 384, ta, tb, (int)M, (int)N, (int)K, ep, (cudaStream_t)stream);
}

}  // extern "C"

// Misc C-ABI entry points: version, device query, standalone GEMMs.
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
  const int ctas = (epi == EPI_GELU && bn == 256) ? 2 : 1;  // 256-row pair tiles, as the DiT-XL/2 fc1
  GemmMaps maps;
  if (make_operand_maps(&maps, A, M, K, W, N, bn, ctas) != SF_OK) return SF_ERR_CUDA;
  if (epi != EPI_F32 && (gemm_narrow_out(bn, epi) ? make_out_map32(&maps.d[0], C, M, N)
                                                  : make_out_map(&maps.d[0], C, M, N)) != SF_OK)
    return SF_ERR_CUDA;
  EpiParams ep{};
  ep.bias = bias;
  ep.out = C;
  ep.ldo = N;
  ep.tokens_per_slot = 1 << 30;
  ep.M = (int)M;
  return launch_gemm(epi, bn, maps, (int)M, (int)N, (int)K, ep, (cudaStream_t)stream, ctas);
}

int sf_gemm_qkv_hd(const void* A, const void* W, const float* bias, void* q, void* k, void* vt, int64_t M,
                   int32_t heads, int32_t T, int32_t hd, float q_scale, void* stream) {
  const int bn = hd == 64 ? qkv_bn64() : 144;
  const int64_t d = (int64_t)heads * hd, N = 3 * d, K = d;
  if ((hd != 64 && hd != 72) || M < 1 || T < 128 || M % T || T % 128 || N % bn || K % 64) return SF_ERR_PARAMETER;
  const int ctas = hd == 64 ? qkv_ctas(K) : 2;  // the runtime's configurations (dit_runtime.cu run_blocks)
  GemmMaps maps;
  if (make_operand_maps(&maps, A, M, K, W, N, bn, ctas) != SF_OK) return SF_ERR_CUDA;
  if (make_qkv_out_maps(&maps, q, k, vt, M / T, heads, T, hd) != SF_OK) return SF_ERR_CUDA;
  EpiParams ep{};
  ep.bias = bias;
  ep.heads = heads;
  ep.q_scale = q_scale;
  ep.tokens_per_slot = T;
  ep.M = (int)M;
  return launch_gemm(EPI_QKV, bn, maps, (int)M, (int)N, (int)K, ep, (cudaStream_t)stream, ctas);
}

int sf_gemm_qkv(const void* A, const void* W, const float* bias, void* q, void* k, void* vt, int64_t M, int32_t heads,
                int32_t T, float q_scale, void* stream) {
  return sf_gemm_qkv_hd(A, W, bias, q, k, vt, M, heads, T, 64, q_scale, stream);
}

int sf_gemm_res(const void* A, const void* W, const float* bias, void* xres, const float* gate, int64_t vec_stride,
                int64_t M, int64_t N, int64_t K, int32_t tokens_per_slot, void* stream) {
  if (N % 128 || K % 64 || M < 1 || tokens_per_slot < 128 || M % tokens_per_slot || tokens_per_slot % 128)
    return SF_ERR_PARAMETER;
  // N % 192 == 0: 256 x 192 pair tiles (the DiT-XL/2 proj / fc2 configuration), else 128 x 128
  const int bn = N % 192 == 0 ? 192 : 128, ctas = bn == 192 ? 2 : 1;
  GemmMaps maps;
  if (make_operand_maps(&maps, A, M, K, W, N, bn, ctas) != SF_OK) return SF_ERR_CUDA;
  if (make_out_map(&maps.d[0], xres, M, N) != SF_OK) return SF_ERR_CUDA;
  EpiParams ep{};
  ep.bias = bias;
  ep.gate = gate;
  ep.vec_stride = vec_stride;
  ep.tokens_per_slot = tokens_per_slot;
  ep.M = (int)M;
  return launch_gemm(EPI_RES, bn, maps, (int)M, (int)N, (int)K, ep, (cudaStream_t)stream, ctas);
}

int sf_ln_modulate(const void* xres, void* xmod, const float* shift, const float* scale, int64_t vec_stride,
                   int64_t M, int64_t N, int32_t tokens_per_slot, float ln_eps, void* stream) {
  if ((N != 384 && N != 1152) || M < 1 || tokens_per_slot < 1 || M % tokens_per_slot) return SF_ERR_PARAMETER;
  return launch_ln_modulate((const __nv_bfloat16*)xres, (__nv_bfloat16*)xmod, shift, scale, vec_stride, M, (int)N,
                            tokens_per_slot, ln_eps, (cudaStream_t)stream);
}

int sf_gemm_res_ln(const void* A, const void* W, const float* bias, void* xres, void* xmod, const float* gate,
                   const float* shift, const float* scale, int64_t vec_stride, int64_t M, int64_t N, int64_t K,
                   int32_t tokens_per_slot, float ln_eps, void* stream) {
  if (N != 384 || K % 64 || M < 1 || M % tokens_per_slot || tokens_per_slot % 128) return SF_ERR_PARAMETER;
  // long K: 2-CTA cluster kernel (192-column slices, statistics exchanged through DSMEM);
  // short K: one CTA per 384-wide row tile (its short main loop does not amortise the exchange)
  const bool cl = K >= 1024;
  GemmMaps maps;
  if (make_operand_maps(&maps, A, M, K, W, N, cl ? 192 : 384) != SF_OK) return SF_ERR_CUDA;
  if (make_out_map32(&maps.d[0], xres, M, N) != SF_OK || make_out_map32(&maps.d[1], xmod, M, N) != SF_OK)
    return SF_ERR_CUDA;
  EpiParams ep{};
  ep.bias = bias;
  ep.xres = (const __nv_bfloat16*)xres;
  ep.gate = gate;
  ep.shift = shift;
  ep.scale = scale;
  ep.vec_stride = vec_stride;
  ep.ln_eps = ln_eps;
  ep.tokens_per_slot = tokens_per_slot;
  ep.M = (int)M;
  return cl ? launch_gemm(EPI_RES_LN2, 192, maps, (int)M, (int)N, (int)K, ep, (cudaStream_t)stream)
            : launch_gemm(EPI_RES_LN, 384, maps, (int)M, (int)N, (int)K, ep, (cudaStream_t)stream);
}

}  // extern "C"

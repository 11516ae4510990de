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

}  // extern "C"

// Internal declarations shared by the .cu translation units.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <utility>

#include "../../include/streamflow.h"

namespace sf {
struct EpiParams;
struct GemmMaps;
int make_tmap_bf16_2d(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, uint64_t row_stride_elems,
                      uint32_t box_inner, uint32_t box_outer, int swizzle_bytes = 128);
int gemm_bk(int bn);
int gemm_b_box_rows(int bn);
int make_operand_maps(GemmMaps* m, const void* A, int64_t M, int64_t K, const void* W, int64_t N, int bn);
int make_out_map(CUtensorMap* m, const void* D, int64_t rows, int64_t cols);
int make_out_map32(CUtensorMap* m, const void* D, int64_t rows, int64_t cols);
int gemm_narrow_out(int bn, int kind);
int make_qkv_out_maps(GemmMaps* m, const void* q, const void* k, const void* vt, int64_t rows, int heads, int T,
                      int hd);
int launch_ln_modulate(const __nv_bfloat16* xres, __nv_bfloat16* xmod, const float* shift, const float* scale,
                       int64_t vec_stride, int64_t M, int N, int tokens_per_slot, float eps, cudaStream_t st);
int prepare_gemm_kernels();
int prepare_attn_kernel();
int launch_gemm(int kind, int bn, const GemmMaps& maps, int M, int N, int K, const EpiParams& ep,
                cudaStream_t st);
int make_operand_maps_2sm(GemmMaps* m, const void* A, int64_t M, int64_t K, const void* W, int64_t N, int bn);
int launch_gemm_2sm(int kind, int bn, const GemmMaps& maps, int M, int N, int K, const EpiParams& ep,
                    cudaStream_t st);

struct AttnMaps {
  CUtensorMap q, qh, k, kh, v;  // qh/kh: head-dim elements 64..79 (head dim 72 only)
  int hd;
};
int make_attn_maps(AttnMaps* m, const void* q, const void* k, const void* vt, int64_t rows, int heads, int T,
                   int hd);
int launch_attn(const AttnMaps& m, __nv_bfloat16* out, int64_t rows, int heads, int T, cudaStream_t st);

int launch_mlp_fused(const void* xmod_in, const void* w1, const void* w2, const float* b1, const float* b2,
                     __nv_bfloat16* xres, __nv_bfloat16* xmod_out, const float* gate, const float* shift,
                     const float* scale, int64_t vec_stride, float ln_eps, int64_t M, int T, cudaStream_t st);

int qkv_bn64();
int launch_block_tail(const void* attn, const void* wproj, const float* bproj, const void* w1, const void* w2,
                      const float* b1, const float* b2, __nv_bfloat16* xres, __nv_bfloat16* xmod_out,
                      const float* gate1, const float* shift1, const float* scale1, const float* gate2,
                      const float* shift2, const float* scale2, int64_t vec_stride, float ln_eps, int64_t M, int T,
                      cudaStream_t st, const void* wqkv = nullptr, const float* bqkv = nullptr, void* q = nullptr,
                      void* k = nullptr, void* vt = nullptr, int heads = 0, float q_scale = 0.f);

int launch_block_tail_pair(const void* attn, const void* wproj, const float* bproj, const void* w1, const void* w2,
                           const float* b1, const float* b2, __nv_bfloat16* xres, __nv_bfloat16* xmod_out,
                           const float* gate1, const float* shift1, const float* scale1, const float* gate2,
                           const float* shift2, const float* scale2, int64_t vec_stride, float ln_eps, int64_t M, int T,
                           cudaStream_t st);

inline int cuda_status() { return cudaGetLastError() == cudaSuccess ? SF_OK : SF_ERR_CUDA; }

// Programmatic dependent launch (PDL) for the per-layer chain QKV GEMM -> attention ->
// block tail: the next kernel's CTAs launch as the previous kernel's CTAs retire and run
// their prologue (barrier init, TMEM alloc, descriptor prefetch) under its tail; each
// PDL kernel executes griddepcontrol.wait before touching activations, so every kernel
// completes only after its predecessor did (transitive ordering). SF_PDL=1 enables: measured
// neutral (3067 vs 3080 frames/s power-capped; 2783 vs 2794 / 11180 vs 11186 at full clock on
// the 8-stream / 1-slot configs) -- graph replay already leaves no launch gap worth hiding.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_maybe_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
}  // namespace sf

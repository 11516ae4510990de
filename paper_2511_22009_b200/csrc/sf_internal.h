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
// ctas = 2: pair tiles (each CTA loads BN / 2 rows of W per box)
int make_operand_maps(GemmMaps* m, const void* A, int64_t M, int64_t K, const void* W, int64_t N, int bn,
                      int ctas = 1);
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
                cudaStream_t st, int ctas = 1);

struct AttnMaps {
  CUtensorMap q, qh, k, kh, v;  // qh/kh: head-dim elements 64..79 (head dim 72 only)
  int hd;
};
int make_attn_maps(AttnMaps* m, const void* q, const void* k, const void* vt, int64_t rows, int heads, int T,
                   int hd);
int launch_attn(const AttnMaps& m, __nv_bfloat16* out, int64_t rows, int heads, int T, cudaStream_t st);

int qkv_bn64();
int qkv_ctas(int64_t K);  // 2: the head-dim-64 QKV runs on CTA pairs with B resident (K = 384)
// csrc/block_tail.cu (M % 256 == 0, T % 128 == 0)
int launch_block_tail(const void* attn, const void* wproj, const float* bproj, const void* w1, const void* w2,
                           const float* b1, const float* b2, __nv_bfloat16* xres, __nv_bfloat16* xmod_out,
                           const float* gate1, const float* shift1, const float* scale1, const float* gate2,
                           const float* shift2, const float* scale2, int64_t vec_stride, float ln_eps, int64_t M, int T,
                           cudaStream_t st);

inline int cuda_status() { return cudaGetLastError() == cudaSuccess ? SF_OK : SF_ERR_CUDA; }

// Programmatic dependent launch for the kernels of one DiT step, switched on by the runtime for
// small batches only (PdlScope in dit_runtime.cu): with idle SMs the next kernel's prologue
// (TMEM alloc, barrier init, resident weights) runs under the previous kernel's tail, +4.5%
// frames/s at one stream; at 32 streams every SM is busy and it measured 0.5-1% slower.
inline thread_local bool g_pdl = false;

// Kernel launch through cudaLaunchKernelEx (one place to attach launch attributes): programmatic
// stream serialisation when g_pdl (the kernel may start once every CTA of the previous kernel has
// executed griddepcontrol.launch_dependents; every kernel launched here executes griddepcontrol.wait
// before touching the previous kernel's data, sf_ptx.cuh pdl_wait) and optionally a cluster shape.
template <typename... KArgs, typename... Args>
cudaError_t launch_kernel_cl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                             unsigned cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[2];
  unsigned na = 0;
  if (g_pdl) {
    at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}
template <typename... KArgs, typename... Args>
cudaError_t launch_kernel(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args&&... args) {
  return launch_kernel_cl(kern, grid, block, smem, st, 1u, std::forward<Args>(args)...);
}
}  // namespace sf

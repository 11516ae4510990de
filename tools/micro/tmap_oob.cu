// Does cuTensorMapEncodeTiled accept a box wider than the global inner dimension (OOB zero fill),
// or a global inner dimension wider than the row stride (overlapping rows)?  And does TMA fill the
// padding as expected?  (Layout probe for the final-layer tile rows, tools/micro.)
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  return (PFN_cuTensorMapEncodeTiled_v12000)p;
}

__global__ void probe(const __grid_constant__ CUtensorMap m, uint16_t* out, int bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((uint32_t)__cvta_generic_to_shared(&bar)), "r"(bytes));
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"((uint32_t)__cvta_generic_to_shared(sm)), "l"((uint64_t)&m), "r"(0), "r"(0),
                 "r"((uint32_t)__cvta_generic_to_shared(&bar)) : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p;}"
                   : "=r"(ok) : "r"((uint32_t)__cvta_generic_to_shared(&bar)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < bytes / 2; i += blockDim.x) out[i] = reinterpret_cast<uint16_t*>(sm)[i];
}

int main() {
  const int rows = 64, cols = 192;  // 32 tokens x 2 halves of 192
  std::vector<uint16_t> h(rows * cols);
  for (int i = 0; i < rows * cols; ++i) h[i] = (uint16_t)(i & 0x7fff);
  uint16_t *d, *o;
  cudaMalloc(&d, h.size() * 2);
  cudaMalloc(&o, 1 << 20);
  cudaMemcpy(d, h.data(), h.size() * 2, cudaMemcpyHostToDevice);
  auto fn = enc();
  for (int variant = 0; variant < 2; ++variant) {
    CUtensorMap m;
    cuuint64_t dims[2] = {(cuuint64_t)(variant == 0 ? cols : 208), (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
    cuuint32_t box[2] = {208, 32}, es[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("variant %d (%s): encode %d\n", variant, variant == 0 ? "box 208 > dim 192" : "dim 208 > stride 192", (int)r);
    if (r != CUDA_SUCCESS) continue;
    const int bytes = 208 * 32 * 2;
    cudaMemset(o, 0xff, 1 << 20);
    probe<<<1, 128, bytes + 1024>>>(m, o, bytes);
    cudaError_t e = cudaDeviceSynchronize();
    std::vector<uint16_t> g(bytes / 2);
    cudaMemcpy(g.data(), o, bytes, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int rr = 0; rr < 32; ++rr)
      for (int cc = 0; cc < 192; ++cc) bad += g[rr * 208 + cc] != h[rr * cols + cc];
    printf("  kernel %s, data mismatches %d, pad[0..3] of row 0: %u %u %u %u\n", cudaGetErrorString(e), bad,
           g[192], g[193], g[194], g[195]);
  }
  return 0;
}

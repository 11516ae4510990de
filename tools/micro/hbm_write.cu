// Pure-write HBM bandwidth on this B200 (the bound of the patch-embed kernel, which writes
// 201 MB and reads 8 MB): 16-byte st.global (default / .cs streaming), and bulk async stores
// (cp.async.bulk.global.shared::cta) of 16 KB chunks from shared memory.  Median of 20.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/hbm_write tools/micro/hbm_write.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void st_v4(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) p[i] = v;
}
__global__ void st_v4_cs(uint4* p, size_t n) {
  const uint4 v = make_uint4(threadIdx.x, 1, 2, 3);
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) __stcs(p + i, v);
}
__global__ void st_bulk(uint8_t* p, size_t bytes) {
  extern __shared__ __align__(128) uint8_t sm[];
  constexpr int CH = 16384;
  for (int i = threadIdx.x; i < CH / 16; i += blockDim.x) reinterpret_cast<uint4*>(sm)[i] = make_uint4(i, 1, 2, 3);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
    for (size_t off = (size_t)blockIdx.x * CH; off < bytes; off += (size_t)gridDim.x * CH) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off), "r"(s), "r"(CH) : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}

// the patch-embed kernel's store pattern without its compute: a warp owns 16 tokens of one
// latent row (T = 1024 tokens of HID = 384 bf16 per row), writes them to two [tokens, HID]
// outputs row by row with 8-byte lanes; CTA c: token group c % 64, rows (c / 64) * W + warp,
// stride (CTAs / 64) * W
__global__ void st_patch_pattern(uint2* a, uint2* b, int rows, int W) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tg = blockIdx.x % 64;
  const int rstride = (gridDim.x / 64) * W;
  const uint2 v = make_uint2(lane, 7);
  for (int ni = (blockIdx.x / 64) * W + warp; ni < rows; ni += rstride) {
    const size_t tok0 = (size_t)ni * 1024 + tg * 16;
#pragma unroll 2
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        a[(tok0 + r) * 96 + lane + 32 * j] = v;
        b[(tok0 + r) * 96 + lane + 32 * j] = v;
      }
  }
}

template <class F>
static float med(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) f();
  std::vector<float> t;
  for (int i = 0; i < 20; ++i) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    t.push_back(ms);
  }
  std::sort(t.begin(), t.end());
  return t[10];
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(st_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 16384);
  for (size_t mb : {201, 1024}) {
    const size_t bytes = mb << 20;
    uint8_t* p;
    cudaMalloc(&p, bytes);
    for (int occ : {4, 8, 16}) {
      const float t1 = med([&] { st_v4<<<sms * occ, 256>>>((uint4*)p, bytes / 16); });
      const float t2 = med([&] { st_v4_cs<<<sms * occ, 256>>>((uint4*)p, bytes / 16); });
      printf("%zu MB  st.v4 %d CTA/SM: %.0f GB/s   st.cs: %.0f GB/s\n", mb, occ, bytes / t1 / 1e6, bytes / t2 / 1e6);
    }
    for (int occ : {1, 4, 8}) {
      const float t3 = med([&] { st_bulk<<<sms * occ, 32, 16384>>>(p, bytes); });
      printf("%zu MB  bulk 16KB %d CTA/SM: %.0f GB/s\n", mb, occ, bytes / t3 / 1e6);
    }
    cudaFree(p);
  }
  {
    uint8_t *a, *b;
    const size_t half = (size_t)128 * 1024 * 384 * 2;  // 100.7 MB each: the bench's xres + xmod
    cudaMalloc(&a, half);
    cudaMalloc(&b, half);
    for (int W : {5, 8, 16}) {
      const int ctas = 64 * (W == 5 ? 4 : 2);
      const float t = med([&] { st_patch_pattern<<<ctas, 32 * W>>>((uint2*)a, (uint2*)b, 128, W); });
      printf("patch-embed store pattern, %d warps x %d CTAs: %.0f GB/s (%.1f us for 201 MB)\n", W, ctas, 2 * half / t / 1e6, t * 1e3);
    }
    cudaFree(a);
    cudaFree(b);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}

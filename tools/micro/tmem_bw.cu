// Microbenchmark: TMEM read (tcgen05.ld 32x32b.x32) and write (tcgen05.st) throughput per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2511_22009_b200/csrc tmem_bw.cu -o tmem_bw
#include <cstdio>
#include "../../paper_2511_22009_b200/csrc/sf_ptx.cuh"
using namespace sf;

template <int WARPS, bool STORE>
__global__ void __launch_bounds__(WARPS * 32) tmem_kernel(float* out, long long* cycles, int iters) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<512>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  const uint32_t base = tmem + (((warp & 3) * 32) << 16) + (warp >> 2) * 32;
  float acc = 0.f;
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = (float)i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if constexpr (STORE) {
      tmem_st32(base + (it & 7) * 64 % 256, v);
    } else {
      tmem_ld32(base + (it & 7) * 64 % 256, v);
      tmem_ld_wait();
      acc += v[0] + v[17] + v[31];
    }
  }
  if constexpr (STORE) tmem_st_wait();
  long long t1 = clock64();
  __syncthreads();
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<512>(tmem);
}

template <int WARPS, bool STORE>
void run(float* out, long long* cyc, int iters) {
  tmem_kernel<WARPS, STORE><<<148, WARPS * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
  const double bytes = (double)WARPS * iters * 32 * 32 * 4;  // per SM
  printf("%s warps=%2d: %.1f bytes/cycle per SM (%.1f cycles per warp-op)\n", STORE ? "tcgen05.st" : "tcgen05.ld",
         WARPS, bytes / mx, (double)mx * WARPS / ((double)WARPS * iters));
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  const int iters = 4096;
  run<4, false>(out, cyc, iters);
  run<8, false>(out, cyc, iters);
  run<16, false>(out, cyc, iters);
  run<4, true>(out, cyc, iters);
  run<8, true>(out, cyc, iters);
  run<16, true>(out, cyc, iters);
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}

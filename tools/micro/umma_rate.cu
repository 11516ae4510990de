// Microbenchmark: back-to-back tcgen05.mma (kind::f16, bf16 in / fp32 acc, both operands in smem)
// per SM, single CTA (M=128) vs CTA pair (cta_group::2, M=256), for several N; optionally with
// LSU shared-memory traffic running beside the MMAs (the epilogue / GELU warps of the fused kernels).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 umma_rate.cu -o umma_rate
#include <cstdio>
#include "../../paper_2511_22009_b200/csrc/sf_ptx.cuh"
using namespace sf;

constexpr int SMEM = 200 * 1024;

template <int PAIR, int N, int LSU_WARPS>
__global__ void __launch_bounds__(32 * (1 + LSU_WARPS), 1) umma_kernel(long long* cycles, int iters, float* sink) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t holder;
  __shared__ __align__(8) uint64_t done;
  __shared__ int stop;
  const int warp = threadIdx.x / 32;
  const uint32_t crank = PAIR ? cluster_ctarank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(&done, 1);
    stop = 0;
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < SMEM / 4; i += blockDim.x) reinterpret_cast<float*>(smem)[i] = 0.f;
  if (warp == 0) {
    if (PAIR) tmem_alloc_2sm<512>(&holder);
    else tmem_alloc<512>(&holder);
  }
  if (PAIR) cluster_sync_all();
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  if (warp == 0) {
    if (!PAIR || crank == 0) {
      const uint32_t idesc = idesc_bf16_f32(PAIR ? 256 : 128, N);
      const uint32_t a0 = smem_u32(smem), b0 = smem_u32(smem + 96 * 1024);
      long long t0 = clock64();
      if (elect_one()) {
        for (int it = 0; it < iters; ++it) {
          const uint64_t ad = sw128_kmajor_desc(a0 + (it % 6) * 16384) + 2 * (it & 3);
          const uint64_t bd = sw128_kmajor_desc(b0 + (it % 3) * 32768) + 2 * (it & 3);
          if (PAIR) mma_bf16_ss_2sm(tmem, ad, bd, idesc, it != 0);
          else mma_bf16_ss(tmem, ad, bd, idesc, it != 0);
        }
        if (PAIR) mma_commit_2sm_mc(&done, 0x3);
        else mma_commit(&done);
      }
      __syncwarp();
      mbar_wait(&done, 0);
      long long t1 = clock64();
      if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    } else {
      mbar_wait(&done, 0);
    }
    if (threadIdx.x == 0) *(volatile int*)&stop = 1;
  } else {
    // LSU traffic: 16-byte conflict-free smem reads + writes in the A region's tail
    float acc = 0.f;
    uint4* base = reinterpret_cast<uint4*>(smem + 136 * 1024) + (warp - 1) * 32 + (threadIdx.x & 31);
    for (int n = 0; !*(volatile int*)&stop && n < (1 << 22); ++n) {
      uint4 v = base[(n & 7) * 512];
      acc += __uint_as_float(v.x);
      base[((n + 3) & 7) * 512] = v;
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  }
  tc_fence_before();
  __syncthreads();
  if (PAIR) cluster_sync_all();
  if (warp == 0) {
    if (PAIR) tmem_dealloc_2sm<512>(tmem);
    else tmem_dealloc<512>(tmem);
  }
}

template <int PAIR, int N, int LSU_WARPS>
void run(long long* cyc, float* sink, int iters) {
  auto k = umma_kernel<PAIR, N, LSU_WARPS>;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(32 * (1 + LSU_WARPS));
  cfg.dynamicSmemBytes = SMEM;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaMemset(cyc, 0, 148 * sizeof(long long));
  cudaError_t e = cudaLaunchKernelEx(&cfg, k, cyc, iters, sink);
  cudaError_t e2 = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  long long mx = 0;
  int cnt = 0;
  for (int i = 0; i < 148; ++i)
    if (h[i]) {
      mx = h[i] > mx ? h[i] : mx;
      ++cnt;
    }
  const double per = (double)mx / iters;
  const double ideal = 128.0 * N / 256.0;  // per-SM cycles of an M128 x N x K16 slice at full rate
  printf("%s N=%3d lsu_warps=%d: %.1f cycles per MMA (ideal %.0f, %.0f%% of rate) [%s/%s, %d timers]\n",
         PAIR ? "pair  M=256" : "single M=128", N, LSU_WARPS, per, ideal, 100.0 * ideal / per, cudaGetErrorString(e),
         cudaGetErrorString(e2), cnt);
}

int main() {
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * sizeof(long long));
  cudaMalloc(&sink, 148 * 1024 * sizeof(float));
  const int iters = 4096;
  run<0, 64, 0>(cyc, sink, iters);
  run<1, 64, 0>(cyc, sink, iters);
  run<1, 64, 16>(cyc, sink, iters);
  run<1, 96, 0>(cyc, sink, iters);
  run<0, 32, 0>(cyc, sink, iters);
  run<0, 128, 0>(cyc, sink, iters);
  run<0, 192, 0>(cyc, sink, iters);
  run<0, 256, 0>(cyc, sink, iters);
  run<1, 128, 0>(cyc, sink, iters);
  run<1, 192, 0>(cyc, sink, iters);
  run<1, 256, 0>(cyc, sink, iters);
  run<0, 128, 8>(cyc, sink, iters);
  run<1, 128, 8>(cyc, sink, iters);
  run<1, 192, 8>(cyc, sink, iters);
  run<0, 128, 16>(cyc, sink, iters);
  run<1, 128, 16>(cyc, sink, iters);
  return 0;
}

// Microbenchmark: throughput of the attention softmax step (TMEM S load -> row max ->
// exp2 (poly + MUFU mix) -> fp16 pack -> TMEM P store) as a function of how many softmax
// warps share an SMSP (2 = the shipped kernel's two 128-row tiles, 3, 4).  No MMAs, no
// barriers: the pure instruction-stream bound of one 64-key softmax step per warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2511_22009_b200/csrc softmax_rate.cu -o softmax_rate
#include <cstdio>
#include "../../paper_2511_22009_b200/csrc/sf_ptx.cuh"
using namespace sf;

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_h2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  const float kMagic = 12582912.0f;
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const float2 t = __fadd2_rn(x, make_float2(kMagic, kMagic));
  const float2 jf = __fadd2_rn(t, make_float2(-kMagic, -kMagic));
  const float2 f = __ffma2_rn(jf, make_float2(-1.f, -1.f), x);
  float2 p = __ffma2_rn(f, make_float2(0.055088773f, 0.055088773f), make_float2(0.24260406f, 0.24260406f));
  p = __ffma2_rn(p, f, make_float2(0.69327623f, 0.69327623f));
  p = __ffma2_rn(p, f, make_float2(0.99992895f, 0.99992895f));
  const uint32_t b0 = __float_as_uint(p.x) + (__float_as_uint(t.x) << 23);
  const uint32_t b1 = __float_as_uint(p.y) + (__float_as_uint(t.y) << 23);
  return make_float2(__uint_as_float(b0), __uint_as_float(b1));
}

template <int WARPS, int EMU>
__global__ void __launch_bounds__(WARPS * 32, 1) softmax_kernel(long long* cycles, float* sink, int iters) {
  __shared__ uint32_t holder;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tmem_alloc<256>(&holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = holder;
  const uint32_t base = tmem + (((warp & 3) * 32) << 16) + (warp >> 2) * 64;
  // initialise this warp's S columns
  {
    float v[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = 0.01f * (i - 16) + 0.001f * threadIdx.x;
    tmem_st32(base, v);
    tmem_st32(base + 32, v);
    tmem_st_wait();
  }
  float m_ref = 0.f, acc = 0.f;
  const float L2E = 1.4426950408889634f;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    float s[64];
    tmem_ld32(base, *reinterpret_cast<float(*)[32]>(&s[0]));
    tmem_ld32(base + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
    tmem_ld_wait();
    float mx[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) mx[i] = fmaxf(s[i], s[i + 8]);
#pragma unroll
    for (int i = 16; i < 64; i += 16)
#pragma unroll
      for (int q = 0; q < 8; ++q) mx[q] = fmaxf(mx[q], fmaxf(s[i + q], s[i + 8 + q]));
    const float m_tile = L2E * fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])), fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
    m_ref = fmaxf(m_ref, m_tile);
    const float2 l2e2 = make_float2(L2E, L2E), negm = make_float2(-m_ref, -m_ref);
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float2 x = __ffma2_rn(make_float2(s[32 * c + 2 * i], s[32 * c + 2 * i + 1]), l2e2, negm);
        float2 p;
        if (i < EMU) {
          p = exp2_poly2(x);
        } else {
          p.x = ex2f(x.x);
          p.y = ex2f(x.y);
        }
        pk[i] = pack_h2(p.x, p.y);
      }
      tmem_st16u(base + 32 + 16 * c, pk);
    }
    tmem_st_wait();
    acc += m_ref;
  }
  const long long t1 = clock64();
  sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc<256>(tmem);
}

template <int WARPS, int EMU>
void run(long long* cyc, float* sink) {
  const int iters = 2000;
  softmax_kernel<WARPS, EMU><<<148, WARPS * 32>>>(cyc, sink, iters);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
  // one "tile-iteration" = 4 warps x 64 keys x 32 rows
  const double tile_iters = (double)iters * WARPS / 4;
  printf("warps/SMSP %d  emu %2d: %7.1f cycles per 128x64 softmax step per SM  (%.1f per warp-iteration)\n",
         WARPS / 4, EMU, mx / tile_iters, (double)mx / iters);
}

int main() {
  long long* cyc;
  float* sink;
  cudaMalloc(&cyc, 148 * 8);
  cudaMalloc(&sink, 148 * 1024 * 4);
  run<8, 6>(cyc, sink);
  run<12, 6>(cyc, sink);
  run<16, 6>(cyc, sink);
  run<8, 4>(cyc, sink);
  run<12, 4>(cyc, sink);
  run<16, 4>(cyc, sink);
  run<8, 8>(cyc, sink);
  run<16, 8>(cyc, sink);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return 0;
}

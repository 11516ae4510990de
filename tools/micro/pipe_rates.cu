// Microbenchmark: per-SM issue rates of the softmax instruction mix (MUFU.EX2, F2FP packs,
// FFMA2, FMNMX, HFMA2) alone and in pairs, to find which pipe bounds the attention softmax.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 pipe_rates.cu -o pipe_rates
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

#define CH 8  // independent chains per thread

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t cvt_f16x2(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ uint32_t cvt_bf16x2(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  uint64_t d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;"
               : "=l"(d)
               : "l"(*reinterpret_cast<uint64_t*>(&a)), "l"(*reinterpret_cast<uint64_t*>(&b)),
                 "l"(*reinterpret_cast<uint64_t*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float r;
  asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
  return r;
}
__device__ __forceinline__ uint32_t hfma2(uint32_t a, uint32_t b, uint32_t c) {
  uint32_t r;
  asm volatile("fma.rn.f16x2 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(c));
  return r;
}

__device__ __forceinline__ uint32_t ex2h2(uint32_t x) {
  uint32_t r;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) {
  uint32_t r;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ float tanh_a(float x) {
  float r;
  asm volatile("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}
// MODE bits (64 = ex2 f16x2, 128 = ex2 bf16x2, 256 = tanh f32): 1 = ex2, 2 = cvt f16x2, 4 = ffma2, 8 = fmax3, 16 = hfma2, 32 = cvt bf16x2
template <int MODE>
__global__ void rates(float* out, long long* cyc, int iters) {
  float x[CH];
  uint32_t h[CH];
  float2 y[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) {
    x[i] = -0.001f * (threadIdx.x + i);
    h[i] = 0x3c003c00u + i;
    y[i] = make_float2(x[i], 1.0f - x[i]);
  }
  const float2 m2 = make_float2(0.999f, 0.998f), a2 = make_float2(1e-3f, 2e-3f);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CH; ++i) {
      if (MODE & 1) x[i] = ex2(x[i]) - 1.0f;  // (FADD keeps the chain finite; counted separately)
      if (MODE & 2) h[i] ^= cvt_f16x2(x[i], y[i].x);
      if (MODE & 32) h[i] ^= cvt_bf16x2(x[i], y[i].y);
      if (MODE & 4) y[i] = ffma2(y[i], m2, a2);
      if (MODE & 8) x[i] = fmax3(x[i], y[i].x, y[i].y);
      if (MODE & 64) h[i] = ex2h2(h[i]) ^ 0xbc00bc00u;
      if (MODE & 128) h[i] = ex2bf2(h[i]) ^ 0xbf80bf80u;
      if (MODE & 256) x[i] = tanh_a(x[i]);
      if (MODE & 16) h[i] = hfma2(h[i], 0x3bff3bffu, 0x00010001u);
    }
  }
  long long t1 = clock64();
  float acc = 0.f;
#pragma unroll
  for (int i = 0; i < CH; ++i) acc += x[i] + y[i].x + y[i].y + (float)(h[i] & 0xff);
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, float* out, long long* cyc, int warps) {
  const int iters = 4096;
  rates<MODE><<<148, warps * 32>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long c[148];
  cudaMemcpy(c, cyc, sizeof(c), cudaMemcpyDeviceToHost);
  long long mx = 0;
  for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
  const double warp_instr = (double)iters * CH * warps;  // per SM, per op kind
  printf("%-28s warps=%2d  %7.3f cyc per warp-instr per SMSP (per op kind)\n", name, warps,
         mx / (warp_instr / 4.0));
}

int main() {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&cyc, 148 * 8);
  for (int w : {16}) {
    run<1>("ex2 (+fadd)", out, cyc, w);
    run<2>("cvt.rn.f16x2.f32", out, cyc, w);
    run<32>("cvt.rn.bf16x2.f32", out, cyc, w);
    run<4>("fma.rn.f32x2", out, cyc, w);
    run<8>("max.f32 x3", out, cyc, w);
    run<16>("fma.rn.f16x2", out, cyc, w);
    run<1 | 2>("ex2 + cvt f16x2", out, cyc, w);
    run<1 | 4>("ex2 + ffma2", out, cyc, w);
    run<2 | 4>("cvt f16x2 + ffma2", out, cyc, w);
    run<2 | 8>("cvt f16x2 + max3", out, cyc, w);
    run<4 | 8>("ffma2 + max3", out, cyc, w);
    run<4 | 16>("ffma2 + hfma2", out, cyc, w);
    run<64>("ex2 f16x2 (+lop)", out, cyc, w);
    run<128>("ex2 bf16x2 (+lop)", out, cyc, w);
    run<256>("tanh f32", out, cyc, w);
    run<64 | 4>("ex2 f16x2 + ffma2", out, cyc, w);
    run<1 | 64>("ex2 f32 + ex2 f16x2", out, cyc, w);
  }
  return 0;
}

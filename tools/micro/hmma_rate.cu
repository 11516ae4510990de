// Legacy warp-level MMA (mma.sync m16n8k16 bf16 -> f32, SASS HMMA.16816) throughput per SM on
// sm_100a, by warps per SM; the patch-embed and final-layer kernels run on it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hmma_rate hmma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CH 8
__global__ void hmma_loop(float* out, int iters) {
  float acc[CH][4] = {};
  const uint32_t a = 0x3f803f80u + threadIdx.x, b = 0x3f803f80u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(acc[c][0]), "+f"(acc[c][1]), "+f"(acc[c][2]), "+f"(acc[c][3])
          : "r"(a), "r"(a), "r"(a), "r"(a), "r"(b), "r"(b));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c][0] + acc[c][1] + acc[c][2] + acc[c][3];
  if (s == 12345.f) out[0] = s;
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* o;
  cudaMalloc(&o, 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096;
  for (int warps : {4, 8, 16, 32}) {
    hmma_loop<<<sms, 32 * warps>>>(o, 16);
    cudaEventRecord(e0);
    hmma_loop<<<sms, 32 * warps>>>(o, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double mmas = (double)sms * warps * iters * CH;
    const double tflops = mmas * 16 * 8 * 16 * 2 / (ms * 1e-3) / 1e12;
    printf("%2d warps/SM: %.1f TFLOP/s dense bf16, %.2f HMMA.16816 per SM per ns\n", warps, tflops,
           mmas / sms / (ms * 1e6));
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}

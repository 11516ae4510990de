// Persistent tcgen05 / TMEM / TMA GEMM for sm_100a with fused DiT epilogues.
//
//   D[M, N] = A[M, K] . B[N, K]^T      (A = activations, B = nn.Linear weight,
//                                       both bf16 K-major, fp32 accumulate)
//
// One CTA per SM loops over 128 x BN output tiles (N-fastest order, so CTAs
// running at the same time share the A tile in L2).  Warp roles:
//   warp 0       TMA producer (one lane): K-blocks of A/B into a STAGES-deep
//                smem ring that runs across tile boundaries
//   warp 1       TMEM allocator + MMA issuer (one lane issues tcgen05.mma)
//   warps 2..    EPI_WARPS epilogue warps; warp w reads TMEM lanes
//                32*(w%4)..+31 (one accumulator row per thread), two warps per
//                lane quarter split the columns when EPI_WARPS == 8
// The accumulator is double-buffered in TMEM when 2*BN <= 512 columns, so the
// epilogue of tile i overlaps the main loop of tile i+1.
#pragma once
#include "sf_ptx.cuh"

namespace sf {

enum EpiKind : int {
  EPI_F32 = 0,     // out f32 [M, ldo]  = acc + bias
  EPI_BF16 = 1,    // out bf16 [M, ldo] = acc + bias
  EPI_GELU = 2,    // out bf16 [M, ldo] = gelu_tanh(acc + bias)
  EPI_QKV = 3,     // scatter to Q,K [rows, H, T, 64] and V^T [rows, H, 64, T]; Q pre-scaled
  EPI_RES_LN = 4,  // x += gate*(acc+bias) (bf16 residual); xmod = LN(x)*(1+scale)+shift
};

struct EpiParams {
  const float* bias;  // [N]
  void* out;          // EPI_F32/BF16/GELU
  int64_t ldo;
  // EPI_QKV
  __nv_bfloat16* q;
  __nv_bfloat16* k;
  __nv_bfloat16* vt;
  int heads;
  float q_scale;
  // EPI_RES_LN
  __nv_bfloat16* xres;   // [M, N] residual stream, updated in place
  __nv_bfloat16* xmod;   // [M, N] modulated LayerNorm output
  const float* gate;     // per-slot vectors: ptr + slot * vec_stride
  const float* shift;
  const float* scale;
  int64_t vec_stride;
  float ln_eps;
  // common
  int tokens_per_slot;   // rows of one latent (1024); tiles never straddle a slot
  int M;                 // valid rows (tail rows of the last tile are masked)
};

template <int BN, int EPI_WARPS>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;  // 128 B of bf16 = one SW128 atom row
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 8 ? 8 : (200 * 1024) / STAGE_BYTES;
  static constexpr int MMA_N = BN > 256 ? BN / 2 : BN;  // UMMA N <= 256
  static constexpr int N_SPLIT = BN / MMA_N;
  static constexpr int B_BOX = BN > 256 ? BN / 2 : BN;  // TMA box rows <= 256
  static constexpr int ACC_STAGES = 2 * BN <= 512 ? 2 : 1;
  static constexpr int ACC_STRIDE = BN <= 128 ? 128 : 256;  // column offset between accumulator stages
  static constexpr int TMEM_COLS = ACC_STAGES == 2 ? (BN <= 128 ? 256 : 512) : (BN <= 256 ? 256 : 512);
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + 256;
  static_assert(MMA_N % 16 == 0 && MMA_N <= 256, "bad MMA N");
  static_assert(B_BOX <= 256, "bad box");
  static_assert(EPI_WARPS == 4 || EPI_WARPS == 8, "epilogue warps");
};

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * x * (1.0f + t);
}

__device__ __forceinline__ uint4 pack8_bf16(const float* v) {
  return make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
}

template <int BN, int KIND, int EPI_WARPS>
__global__ void __launch_bounds__(GemmCfg<BN, EPI_WARPS>::THREADS, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int N,
                      int K, EpiParams ep) {
  using C = GemmCfg<BN, EPI_WARPS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + C::ACC_STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + C::ACC_STAGES);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int num_n = N / BN;
  const int num_m = (ep.M + C::BM - 1) / C::BM;
  const int total = num_m * num_n;
  const int num_kb = K / C::BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::ACC_STAGES; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], EPI_WARPS * 32);
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (ring continues across tiles)
      uint32_t it = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x) {
        const int m0 = (tile / num_n) * C::BM, n0 = (tile % num_n) * BN;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          mbar_expect_tx(&full[s], C::STAGE_BYTES);
          tma_load_2d(sA + s * C::A_BYTES, &tmA, &full[s], kb * C::BK, m0);
#pragma unroll
          for (int h = 0; h < BN / C::B_BOX; ++h)
            tma_load_2d(sB + s * C::B_BYTES + h * C::B_BOX * 128, &tmB, &full[s], kb * C::BK, n0 + h * C::B_BOX);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(128, C::MMA_N);
      uint32_t it = 0, local = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++local) {
        const uint32_t acc = local % C::ACC_STAGES, aph = (local / C::ACC_STAGES) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);  // epilogue drained this accumulator
        tc_fence_after();
        const uint32_t d = tmem_base + acc * C::ACC_STRIDE;
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1;
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(sA + s * C::A_BYTES);
          const uint32_t b_addr = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < C::BK / 16; ++k) {
#pragma unroll
            for (int h = 0; h < C::N_SPLIT; ++h)
              mma_bf16_ss(d + h * C::MMA_N, sw128_kmajor_desc(a_addr + k * 32),
                          sw128_kmajor_desc(b_addr + h * C::MMA_N * 128 + k * 32), idesc, (kb | k) != 0);
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&tfull[acc]);
      }
    }
  } else {
    // ---------------- epilogue warps
    const uint32_t e = warp - 2;
    const uint32_t quarter = warp & 3;
    constexpr int COLS = EPI_WARPS == 8 ? BN / 2 : BN;
    const int c_lo = EPI_WARPS == 8 ? (int)(e / 4) * COLS : 0;
    uint32_t local = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++local) {
      const int m0 = (tile / num_n) * C::BM, n0 = (tile % num_n) * BN;
      const uint32_t acc = local % C::ACC_STAGES, aph = (local / C::ACC_STAGES) & 1;
      const int row = m0 + quarter * 32 + lane;
      const bool valid = row < ep.M;
      const uint32_t taddr = tmem_base + ((quarter * 32) << 16) + acc * C::ACC_STRIDE;
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();

      if constexpr (KIND == EPI_F32 || KIND == EPI_BF16 || KIND == EPI_GELU) {
#pragma unroll 1
        for (int c0 = c_lo; c0 < c_lo + COLS; c0 += 32) {
          float v[32];
          tmem_ld32(taddr + c0, v);
          tmem_ld_wait();
          const float4* bp = reinterpret_cast<const float4*>(ep.bias + n0 + c0);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 b = __ldg(bp + i);
            v[4 * i] += b.x;
            v[4 * i + 1] += b.y;
            v[4 * i + 2] += b.z;
            v[4 * i + 3] += b.w;
          }
          if constexpr (KIND == EPI_GELU) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = gelu_tanh(v[i]);
          }
          if (valid) {
            if constexpr (KIND == EPI_F32) {
              float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.out) + (int64_t)row * ep.ldo + n0 + c0);
#pragma unroll
              for (int i = 0; i < 8; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
            } else {
              uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(ep.out) + (int64_t)row * ep.ldo + n0 + c0);
#pragma unroll
              for (int i = 0; i < 4; ++i) dst[i] = pack8_bf16(v + 8 * i);
            }
          }
        }
      } else if constexpr (KIND == EPI_QKV) {
        // columns [0, d) -> Q, [d, 2d) -> K, [2d, 3d) -> V; 64 columns per head
        const int d = ep.heads * 64;
        const int T = ep.tokens_per_slot;
        const int slot = m0 / T;
        const int tok = row - slot * T;
#pragma unroll 1
        for (int c0 = c_lo; c0 < c_lo + COLS; c0 += 64) {
          const int gc = n0 + c0;
          const int which = gc / d;
          const int head = (gc - which * d) / 64;
          float v[64];
          tmem_ld32(taddr + c0, *reinterpret_cast<float(*)[32]>(&v[0]));
          tmem_ld32(taddr + c0 + 32, *reinterpret_cast<float(*)[32]>(&v[32]));
          tmem_ld_wait();
          const float sc = which == 0 ? ep.q_scale : 1.0f;
          const float4* bp = reinterpret_cast<const float4*>(ep.bias + gc);
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float4 b = __ldg(bp + i);
            v[4 * i] = (v[4 * i] + b.x) * sc;
            v[4 * i + 1] = (v[4 * i + 1] + b.y) * sc;
            v[4 * i + 2] = (v[4 * i + 2] + b.z) * sc;
            v[4 * i + 3] = (v[4 * i + 3] + b.w) * sc;
          }
          if (valid) {
            const int64_t hb = ((int64_t)slot * ep.heads + head);
            if (which < 2) {
              uint4* dst = reinterpret_cast<uint4*>((which == 0 ? ep.q : ep.k) + (hb * T + tok) * 64);
#pragma unroll
              for (int i = 0; i < 8; ++i) dst[i] = pack8_bf16(v + 8 * i);
            } else {
              __nv_bfloat16* base = ep.vt + hb * 64 * T + tok;
#pragma unroll
              for (int i = 0; i < 64; ++i) base[(int64_t)i * T] = __float2bfloat16_rn(v[i]);
            }
          }
        }
      } else if constexpr (KIND == EPI_RES_LN) {
        static_assert(KIND != EPI_RES_LN || EPI_WARPS == 4, "RES_LN needs whole rows per thread");
        const int slot = m0 / ep.tokens_per_slot;
        const float* gate = ep.gate + (int64_t)slot * ep.vec_stride + n0;
        const float* shift = ep.shift + (int64_t)slot * ep.vec_stride + n0;
        const float* scale = ep.scale + (int64_t)slot * ep.vec_stride + n0;
        // pass 1: residual update, write bf16 residual, keep fp32 copy in TMEM, row sum
        float sum = 0.f;
        __nv_bfloat16* xr = ep.xres + (int64_t)row * N + n0;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(taddr + c0, v);
          uint4 old[4];
          if (valid) {
#pragma unroll
            for (int i = 0; i < 4; ++i) old[i] = reinterpret_cast<const uint4*>(xr + c0)[i];
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) old[i] = make_uint4(0, 0, 0, 0);
          }
          tmem_ld_wait();
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 b = __ldg(reinterpret_cast<const float4*>(ep.bias + n0 + c0) + i);
            const float4 g = __ldg(reinterpret_cast<const float4*>(gate + c0) + i);
            const float2 o0 = unpack_bf16(reinterpret_cast<const uint32_t*>(old)[2 * i]);
            const float2 o1 = unpack_bf16(reinterpret_cast<const uint32_t*>(old)[2 * i + 1]);
            packed[2 * i] = pack_bf16(o0.x + g.x * (v[4 * i] + b.x), o0.y + g.y * (v[4 * i + 1] + b.y));
            packed[2 * i + 1] = pack_bf16(o1.x + g.z * (v[4 * i + 2] + b.z), o1.y + g.w * (v[4 * i + 3] + b.w));
            const float2 r0 = unpack_bf16(packed[2 * i]), r1 = unpack_bf16(packed[2 * i + 1]);
            v[4 * i] = r0.x;  // LayerNorm sees the stored (rounded) residual
            v[4 * i + 1] = r0.y;
            v[4 * i + 2] = r1.x;
            v[4 * i + 3] = r1.y;
            sum += (r0.x + r0.y) + (r1.x + r1.y);
          }
          if (valid) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<uint4*>(xr + c0)[i] =
                  make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
          }
          tmem_st32(taddr + c0, v);
        }
        tmem_st_wait();
        const float mean = sum * (1.0f / BN);
        float var = 0.f;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(taddr + c0, v);
          tmem_ld_wait();
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float dlt = v[i] - mean;
            var += dlt * dlt;
          }
        }
        const float rstd = rsqrtf(var * (1.0f / BN) + ep.ln_eps);
        __nv_bfloat16* xm = ep.xmod + (int64_t)row * N + n0;
#pragma unroll 1
        for (int c0 = 0; c0 < BN; c0 += 32) {
          float v[32];
          tmem_ld32(taddr + c0, v);
          tmem_ld_wait();
          if (c0 + 32 == BN) {  // last TMEM read of this tile: hand the accumulator back early
            tc_fence_before();
            mbar_arrive(&tempty[acc]);
          }
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const float4 sh = __ldg(reinterpret_cast<const float4*>(shift + c0) + i);
            const float4 sc = __ldg(reinterpret_cast<const float4*>(scale + c0) + i);
            packed[2 * i] = pack_bf16((v[4 * i] - mean) * rstd * (1.0f + sc.x) + sh.x,
                                      (v[4 * i + 1] - mean) * rstd * (1.0f + sc.y) + sh.y);
            packed[2 * i + 1] = pack_bf16((v[4 * i + 2] - mean) * rstd * (1.0f + sc.z) + sh.z,
                                          (v[4 * i + 3] - mean) * rstd * (1.0f + sc.w) + sh.w);
          }
          if (valid) {
#pragma unroll
            for (int i = 0; i < 4; ++i)
              reinterpret_cast<uint4*>(xm + c0)[i] =
                  make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
          }
        }
      }
      if constexpr (KIND != EPI_RES_LN) {
        tc_fence_before();
        mbar_arrive(&tempty[acc]);
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

}  // namespace sf

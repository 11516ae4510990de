// tcgen05 / TMEM / TMA GEMM for sm_100a with fused DiT epilogues.
//
//   D[M, N] = A[M, K] . B[N, K]^T      (A = activations, B = nn.Linear weight,
//                                       both bf16 K-major, fp32 accumulate)
//
// One CTA computes one 128 x BN tile.  Warp roles (192 threads):
//   warp 0      : TMA producer (one elected lane), kStages-deep smem ring
//   warp 1      : TMEM allocator + MMA issuer (one lane issues tcgen05.mma)
//   warps 2..5  : epilogue; warp w reads TMEM lanes 32*(w%4)..+31, one
//                 accumulator row per thread, via tcgen05.ld.32x32b.x32
// The epilogue stages its per-column vectors (bias / gate / shift / scale)
// into smem while the main loop runs, then applies one of the fused
// epilogues below and writes straight to global memory.
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

template <int BN>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = 64;  // 128 B of bf16 = one SW128 atom row
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = (200 * 1024) / STAGE_BYTES > 6 ? 6 : (200 * 1024) / STAGE_BYTES;
  static constexpr int MMA_N = BN > 256 ? BN / 2 : BN;  // UMMA N <= 256
  static constexpr int N_SPLIT = BN / MMA_N;
  static constexpr int B_BOX = BN > 256 ? BN / 2 : BN;  // TMA box rows <= 256
  static constexpr int TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : BN <= 256 ? 256 : 512;
  static constexpr int VEC_FLOATS = 4 * BN;  // bias, gate, shift, scale
  static constexpr int SMEM_BYTES = 1024 + STAGES * STAGE_BYTES + VEC_FLOATS * 4 + 256;
  static_assert(MMA_N % 16 == 0 && MMA_N <= 256, "bad MMA N");
  static_assert(B_BOX <= 256, "bad box");
};

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * x * (1.0f + t);
}

template <int BN, int KIND>
__global__ void __launch_bounds__(192, 1)
    gemm_bf16_tcgen05(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, int K,
                      EpiParams ep) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  float* svec = reinterpret_cast<float*>(smem + C::STAGES * C::STAGE_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(svec + C::VEC_FLOATS);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 2 * C::STAGES + 1);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * BN;
  const int m0 = blockIdx.y * C::BM;
  const int num_kb = K / C::BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<C::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % C::STAGES;
        const uint32_t ph = (kb / C::STAGES) & 1;
        mbar_wait(&empty[s], ph ^ 1);
        mbar_expect_tx(&full[s], C::STAGE_BYTES);
        tma_load_2d(sA + s * C::A_BYTES, &tmA, &full[s], kb * C::BK, m0);
#pragma unroll
        for (int h = 0; h < BN / C::B_BOX; ++h)
          tma_load_2d(sB + s * C::B_BYTES + h * C::B_BOX * 128, &tmB, &full[s], kb * C::BK, n0 + h * C::B_BOX);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(128, C::MMA_N);
      for (int kb = 0; kb < num_kb; ++kb) {
        const int s = kb % C::STAGES;
        const uint32_t ph = (kb / C::STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint32_t a_addr = smem_u32(sA + s * C::A_BYTES);
        const uint32_t b_addr = smem_u32(sB + s * C::B_BYTES);
#pragma unroll
        for (int k = 0; k < C::BK / 16; ++k) {
#pragma unroll
          for (int h = 0; h < C::N_SPLIT; ++h) {
            const uint64_t ad = sw128_kmajor_desc(a_addr + k * 32);
            const uint64_t bd = sw128_kmajor_desc(b_addr + h * C::MMA_N * 128 + k * 32);
            mma_bf16_ss(tmem_base + h * C::MMA_N, ad, bd, idesc, (kb | k) != 0);
          }
        }
        mma_commit(&empty[s]);
      }
      mma_commit(tfull);
    }
  } else {
    // ---------------- epilogue (warps 2..5)
    const int et = threadIdx.x - 64;  // 0..127
    const int slot = m0 / ep.tokens_per_slot;
    float* s_bias = svec;
    float* s_gate = svec + BN;
    float* s_shift = svec + 2 * BN;
    float* s_scale = svec + 3 * BN;
    for (int c = et; c < BN; c += 128) {
      s_bias[c] = ep.bias ? ep.bias[n0 + c] : 0.0f;
      if constexpr (KIND == EPI_RES_LN) {
        s_gate[c] = ep.gate[(int64_t)slot * ep.vec_stride + n0 + c];
        s_shift[c] = ep.shift[(int64_t)slot * ep.vec_stride + n0 + c];
        s_scale[c] = ep.scale[(int64_t)slot * ep.vec_stride + n0 + c];
      }
    }
    named_bar_sync(1, 128);

    const uint32_t quarter = warp & 3;
    const int row_in_tile = quarter * 32 + lane;
    const int row = m0 + row_in_tile;
    const bool valid = row < ep.M;
    const uint32_t taddr = tmem_base + ((quarter * 32) << 16);

    mbar_wait(tfull, 0);
    tc_fence_after();

    if constexpr (KIND == EPI_F32 || KIND == EPI_BF16 || KIND == EPI_GELU) {
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        float v[32];
        tmem_ld32(taddr + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          float x = v[i] + s_bias[c0 + i];
          if constexpr (KIND == EPI_GELU) x = gelu_tanh(x);
          v[i] = x;
        }
        if (valid) {
          if constexpr (KIND == EPI_F32) {
            float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.out) + (int64_t)row * ep.ldo + n0 + c0);
#pragma unroll
            for (int i = 0; i < 8; ++i) dst[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
          } else {
            uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(ep.out) + (int64_t)row * ep.ldo + n0 + c0);
#pragma unroll
            for (int i = 0; i < 4; ++i)
              dst[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                                  pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
          }
        }
      }
    } else if constexpr (KIND == EPI_QKV) {
      // columns [0, d) -> Q, [d, 2d) -> K, [2d, 3d) -> V; 64 columns per head
      const int d = ep.heads * 64;
      const int T = ep.tokens_per_slot;
      const int tok = row - slot * T;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 64) {
        const int gc = n0 + c0;
        const int which = gc / d;
        const int head = (gc - which * d) / 64;
        float v[64];
        tmem_ld32(taddr + c0, *reinterpret_cast<float(*)[32]>(&v[0]));
        tmem_ld32(taddr + c0 + 32, *reinterpret_cast<float(*)[32]>(&v[32]));
        tmem_ld_wait();
        const float sc = which == 0 ? ep.q_scale : 1.0f;
#pragma unroll
        for (int i = 0; i < 64; ++i) v[i] = (v[i] + s_bias[c0 + i]) * sc;
        if (valid) {
          const int64_t hb = ((int64_t)slot * ep.heads + head);
          if (which < 2) {
            __nv_bfloat16* base = (which == 0 ? ep.q : ep.k) + (hb * T + tok) * 64;
            uint4* dst = reinterpret_cast<uint4*>(base);
#pragma unroll
            for (int i = 0; i < 8; ++i)
              dst[i] = make_uint4(pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                                  pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
          } else {
            __nv_bfloat16* base = ep.vt + hb * 64 * T + tok;
#pragma unroll
            for (int i = 0; i < 64; ++i) base[(int64_t)i * T] = __float2bfloat16_rn(v[i]);
          }
        }
      }
    } else if constexpr (KIND == EPI_RES_LN) {
      // pass 1: residual update, write bf16 residual, keep fp32 copy in TMEM, row sum
      const int N = BN;
      float sum = 0.f;
      __nv_bfloat16* xr = ep.xres + (int64_t)row * N;
#pragma unroll 1
      for (int c0 = 0; c0 < N; c0 += 32) {
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
        for (int i = 0; i < 16; ++i) {
          const uint32_t ou = reinterpret_cast<const uint32_t*>(old)[i];
          float2 o = unpack_bf16(ou);
          float y0 = o.x + s_gate[c0 + 2 * i] * (v[2 * i] + s_bias[c0 + 2 * i]);
          float y1 = o.y + s_gate[c0 + 2 * i + 1] * (v[2 * i + 1] + s_bias[c0 + 2 * i + 1]);
          packed[i] = pack_bf16(y0, y1);
          float2 r = unpack_bf16(packed[i]);  // LayerNorm sees the stored (rounded) residual
          v[2 * i] = r.x;
          v[2 * i + 1] = r.y;
          sum += r.x + r.y;
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
      const float mean = sum * (1.0f / N);
      float var = 0.f;
#pragma unroll 1
      for (int c0 = 0; c0 < N; c0 += 32) {
        float v[32];
        tmem_ld32(taddr + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const float dlt = v[i] - mean;
          var += dlt * dlt;
        }
      }
      const float rstd = rsqrtf(var * (1.0f / N) + ep.ln_eps);
      __nv_bfloat16* xm = ep.xmod + (int64_t)row * N;
#pragma unroll 1
      for (int c0 = 0; c0 < N; c0 += 32) {
        float v[32];
        tmem_ld32(taddr + c0, v);
        tmem_ld_wait();
        uint32_t packed[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int c = c0 + 2 * i;
          float a = (v[2 * i] - mean) * rstd * (1.0f + s_scale[c]) + s_shift[c];
          float b = (v[2 * i + 1] - mean) * rstd * (1.0f + s_scale[c + 1]) + s_shift[c + 1];
          packed[i] = pack_bf16(a, b);
        }
        if (valid) {
#pragma unroll
          for (int i = 0; i < 4; ++i)
            reinterpret_cast<uint4*>(xm + c0)[i] =
                make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
        }
      }
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<C::TMEM_COLS>(tmem_base);
}

}  // namespace sf

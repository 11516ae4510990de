// Flash attention for the DiT velocity field on tcgen05 / TMEM / TMA (sm_100a).
//
// One CTA = one (latent row, head) pair x one 128-query tile; T = 1024
// tokens, head dim 64, no mask.  Q arrives pre-scaled by 1/sqrt(64) from the
// QKV GEMM epilogue, V arrives transposed ([hd, T]) so both MMAs read K-major
// operands.
//
//   warp 0      TMA producer: Q once, then K / V^T tiles into a 2-stage ring
//   warp 1      TMEM allocator + single-thread MMA issuer:
//                 S_j  = Q . K_j^T      (M=128, N=128, K=64)  -> TMEM S[j%2]
//                 O_j  = P_j . V_j      (M=128, N=64,  K=128) -> TMEM O
//   warps 2..5  softmax: thread r owns query row r.  Reads S_j from TMEM,
//               online max / exp2 / row sum in registers, writes P_j (bf16,
//               128B-swizzled) to smem for the PV MMA, and folds each O_j
//               into a register accumulator with the running rescale.
// S is double-buffered, so QK^T of tile j+1 runs on the tensor core while
// the softmax warps work on tile j.
#include "sf_internal.h"
#include "sf_ptx.cuh"

namespace sf {

namespace attn {
constexpr int BQ = 128;   // queries per CTA
constexpr int BKV = 128;  // keys per tile
constexpr int HD = 64;
constexpr int Q_BYTES = BQ * HD * 2;      // 16 KB
constexpr int K_BYTES = BKV * HD * 2;     // 16 KB
constexpr int V_BYTES = HD * BKV * 2;     // 16 KB (V^T tile: 64 rows x 128 kv, as 2 SW128 sub-tiles)
constexpr int P_BYTES = BQ * BKV * 2;     // 32 KB (2 SW128 sub-tiles of 128 rows x 64 kv)
constexpr int KV_STAGES = 2;
constexpr int SMEM = 1024 + Q_BYTES + KV_STAGES * (K_BYTES + V_BYTES) + P_BYTES + 256;
constexpr int TMEM_COLS = 512;  // S0 [0,128), S1 [128,256), O [256,320)
constexpr uint32_t O_COL = 256;
}  // namespace attn

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(192, 1)
    attn_fwd_tcgen05(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ out, int T, int heads) {
  using namespace attn;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;
  uint8_t* sK = sQ + Q_BYTES;
  uint8_t* sV = sK + KV_STAGES * K_BYTES;
  uint8_t* sP = sV + KV_STAGES * V_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + P_BYTES);
  uint64_t* bar_q = bars + 0;
  uint64_t* kv_full = bars + 1;   // [2]
  uint64_t* kv_empty = bars + 3;  // [2]
  uint64_t* s_full = bars + 5;    // [2]
  uint64_t* s_free = bars + 7;    // [2]
  uint64_t* p_full = bars + 9;
  uint64_t* o_full = bars + 10;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(bars + 11);

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * BQ;
  const int bh = blockIdx.y;  // row * heads + head
  const int nkv = T / BKV;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(bar_q, 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 1);
      mbar_init(&s_full[s], 1);
      mbar_init(&s_free[s], 128);
    }
    mbar_init(p_full, 128);
    mbar_init(o_full, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc<TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    if (lane == 0) {
      mbar_expect_tx(bar_q, Q_BYTES);
      tma_load_2d(sQ, &tmQ, bar_q, 0, bh * T + q0);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % KV_STAGES;
        mbar_wait(&kv_empty[s], ((j / KV_STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[s], K_BYTES + V_BYTES);
        tma_load_2d(sK + s * K_BYTES, &tmK, &kv_full[s], 0, bh * T + j * BKV);
        tma_load_2d(sV + s * V_BYTES, &tmV, &kv_full[s], j * BKV, bh * HD);
        tma_load_2d(sV + s * V_BYTES + V_BYTES / 2, &tmV, &kv_full[s], j * BKV + 64, bh * HD);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = idesc_bf16_f32(128, BKV);
      constexpr uint32_t idesc_o = idesc_bf16_f32(128, HD);
      const uint32_t q_addr = smem_u32(sQ);
      const uint32_t p_addr = smem_u32(sP);
      auto issue_s = [&](int j) {
        const int s = j % KV_STAGES;
        mbar_wait(&kv_full[s], (j / KV_STAGES) & 1);
        const int b = j & 1;
        if (j >= 2) mbar_wait(&s_free[b], ((j / 2) - 1) & 1);
        tc_fence_after();
        const uint32_t k_addr = smem_u32(sK + s * K_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          mma_bf16_ss(tmem + b * BKV, sw128_kmajor_desc(q_addr + k * 32), sw128_kmajor_desc(k_addr + k * 32),
                      idesc_s, k != 0);
        mma_commit(&s_full[b]);
      };
      mbar_wait(bar_q, 0);
      issue_s(0);
      for (int j = 0; j < nkv; ++j) {
        if (j + 1 < nkv) issue_s(j + 1);
        mbar_wait(p_full, j & 1);
        tc_fence_after();
        const int s = j % KV_STAGES;
        const uint32_t v_addr = smem_u32(sV + s * V_BYTES);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k) {
          const uint32_t sub = (k / 4) * (BQ * 128), off = (k % 4) * 32;
          const uint32_t vsub = (k / 4) * (HD * 128);
          mma_bf16_ss(tmem + O_COL, sw128_kmajor_desc(p_addr + sub + off), sw128_kmajor_desc(v_addr + vsub + off),
                      idesc_o, k != 0);
        }
        mma_commit(o_full);
        mma_commit(&kv_empty[s]);
      }
    }
  } else {
    // ---------------- softmax warps: thread r <-> query row r
    const uint32_t quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t trow = tmem + ((quarter * 32) << 16);
    const float L2E = 1.4426950408889634f;
    float o_acc[HD];
#pragma unroll
    for (int i = 0; i < HD; ++i) o_acc[i] = 0.f;
    float m_run = -INFINITY;  // log2-domain max used by the latest P
    float m_prev = -INFINITY; // max used by P_{j-1}
    float l_run = 0.f;
    uint8_t* prow0 = sP + r * 128;
    const uint32_t sw = (uint32_t)(r & 7);

    for (int j = 0; j < nkv; ++j) {
      const int b = j & 1;
      mbar_wait(&s_full[b], (j / 2) & 1);
      tc_fence_after();
      const uint32_t sbase = trow + b * BKV;
      // pass 1: row max of this tile
      float mx = -INFINITY;
#pragma unroll
      for (int c0 = 0; c0 < BKV; c0 += 32) {
        float v[32];
        tmem_ld32(sbase + c0, v);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) mx = fmaxf(mx, v[i]);
      }
      const float m_new = fmaxf(m_run, mx * L2E);
      // fold O_{j-1} (computed with max m_run) before P_j overwrites P_{j-1}
      if (j > 0) {
        mbar_wait(o_full, (j - 1) & 1);
        tc_fence_after();
        const float a = ex2(m_prev - m_run);  // rescale accumulated units m_prev -> m_run
        float ov[32];
        tmem_ld32(trow + O_COL, ov);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) o_acc[i] = o_acc[i] * a + ov[i];
        tmem_ld32(trow + O_COL + 32, ov);
        tmem_ld_wait();
#pragma unroll
        for (int i = 0; i < 32; ++i) o_acc[32 + i] = o_acc[32 + i] * a + ov[i];
        m_prev = m_run;
      }
      // pass 2: P = exp2(s*log2e - m_new) -> bf16 -> swizzled smem; row sum
      float psum = 0.f;
#pragma unroll
      for (int c0 = 0; c0 < BKV; c0 += 32) {
        float v[32];
        tmem_ld32(sbase + c0, v);
        tmem_ld_wait();
        uint32_t pk[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const float p0 = ex2(fmaf(v[2 * i], L2E, -m_new));
          const float p1 = ex2(fmaf(v[2 * i + 1], L2E, -m_new));
          pk[i] = pack_bf16(p0, p1);
          const float2 pr = unpack_bf16(pk[i]);  // sum what the MMA will see
          psum += pr.x + pr.y;
        }
        // 32 columns = 4 16-byte chunks; column c0 lies in sub-tile c0/64
        uint8_t* sub = prow0 + (c0 / 64) * (BQ * 128);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const uint32_t chunk = ((c0 % 64) / 8 + q) ^ sw;
          *reinterpret_cast<uint4*>(sub + chunk * 16) = make_uint4(pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
        }
      }
      tc_fence_before();
      mbar_arrive(&s_free[b]);
      fence_proxy_async_smem();
      mbar_arrive(p_full);
      l_run = l_run * ex2(m_run - m_new) + psum;
      if (j == 0) m_prev = m_new;
      m_run = m_new;
    }
    // fold the last O
    mbar_wait(o_full, (nkv - 1) & 1);
    tc_fence_after();
    {
      const float a = ex2(m_prev - m_run);
      float ov[32];
      tmem_ld32(trow + O_COL, ov);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) o_acc[i] = o_acc[i] * a + ov[i];
      tmem_ld32(trow + O_COL + 32, ov);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 32; ++i) o_acc[32 + i] = o_acc[32 + i] * a + ov[i];
    }
    const float inv = 1.0f / l_run;
    const int row = bh / heads, head = bh % heads;
    __nv_bfloat16* dst = out + ((int64_t)row * T + q0 + r) * (heads * HD) + head * HD;
#pragma unroll
    for (int i = 0; i < HD / 8; ++i)
      reinterpret_cast<uint4*>(dst)[i] =
          make_uint4(pack_bf16(o_acc[8 * i] * inv, o_acc[8 * i + 1] * inv),
                     pack_bf16(o_acc[8 * i + 2] * inv, o_acc[8 * i + 3] * inv),
                     pack_bf16(o_acc[8 * i + 4] * inv, o_acc[8 * i + 5] * inv),
                     pack_bf16(o_acc[8 * i + 6] * inv, o_acc[8 * i + 7] * inv));
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<attn::TMEM_COLS>(tmem);
}

int make_attn_maps(AttnMaps* m, const void* q, const void* k, const void* vt, int64_t rows, int heads, int T) {
  const uint64_t bhT = (uint64_t)rows * heads * T;
  if (make_tmap_bf16_2d(&m->q, q, 64, bhT, 64, 64, attn::BQ) != SF_OK) return SF_ERR_CUDA;
  if (make_tmap_bf16_2d(&m->k, k, 64, bhT, 64, 64, attn::BKV) != SF_OK) return SF_ERR_CUDA;
  if (make_tmap_bf16_2d(&m->v, vt, T, (uint64_t)rows * heads * 64, T, 64, 64) != SF_OK) return SF_ERR_CUDA;
  return SF_OK;
}

int prepare_attn_kernel() {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_fwd_tcgen05, cudaFuncAttributeMaxDynamicSharedMemorySize, attn::SMEM) !=
        cudaSuccess)
      return SF_ERR_CUDA;
    attr = true;
  }
  return SF_OK;
}

int launch_attn(const AttnMaps& m, __nv_bfloat16* out, int64_t rows, int heads, int T, cudaStream_t st) {
  if (prepare_attn_kernel() != SF_OK) return SF_ERR_CUDA;
  dim3 grid(T / attn::BQ, (unsigned)(rows * heads));
  attn_fwd_tcgen05<<<grid, 192, attn::SMEM, st>>>(m.q, m.k, m.v, out, T, heads);
  return cuda_status();
}

}  // namespace sf

extern "C" int sf_attention(const void* q, const void* k, const void* vt, void* out, int64_t rows, int32_t heads,
                            int32_t T, void* stream) {
  if (rows < 1 || heads < 1 || T < 128 || T % 128) return SF_ERR_PARAMETER;
  sf::AttnMaps m;
  if (sf::make_attn_maps(&m, q, k, vt, rows, heads, T) != SF_OK) return SF_ERR_CUDA;
  return sf::launch_attn(m, reinterpret_cast<__nv_bfloat16*>(out), rows, heads, T, (cudaStream_t)stream);
}

// Flash attention for the DiT velocity field on tcgen05 / TMEM / TMA (sm_100a).
//
// One CTA = one (latent row, head) pair x TWO 128-query tiles (A, B) that
// ping-pong on the tensor core; T tokens (1024), head dim 64, no mask.  Q
// arrives pre-scaled by 1/sqrt(64) from the QKV GEMM epilogue and V arrives
// transposed ([hd, T]) so every MMA reads K-major operands.  KV tiles are 64
// keys wide.
//
//   warps 0-3   softmax of tile A (thread r = query row r)
//   warps 4-7   softmax of tile B
//   warp 8      TMA producer: Q_A, Q_B once; K_j / V_j^T into a 6-stage ring
//   warps 9,10  MMA issuers, one per query tile (warp 9 also owns TMEM), so the
//               two tiles progress independently
//                 S_t[j%2] = Q_t . K_j^T   (M=128, N=64, K=64)
//                 O_t     += P_t . V_j     (M=128, N=64, K=64)
// TMEM columns: S_A0 [0,64) S_A1 [64,128) S_B0 [128,192) S_B1 [192,256)
//               O_A [256,320) O_B [320,384).
//
// S and P are double-buffered per tile and S is issued two KV tiles ahead, so
// a softmax warp finds its scores ready and never waits for the PV of the
// previous tile; each S buffer is released (s_free) as soon as the softmax has
// the 64-wide score row in registers, so S two tiles ahead overlaps the exp.
// Softmax per KV tile: tree max, P = exp2(s*log2e - m) -> fp16 -> 128B-swizzled
// smem (A operand of the fp16 PV MMA); the row sum l comes out of the PV MMA as
// column 64 of O (V^T carries a ones-row).  The O accumulator stays in TMEM and
// the exponent reference m is updated lazily: only when a row max exceeds it by
// more than 8 (log2 units, i.e. P <= 256) does the warp wait for the in-flight
// PV and rescale its O rows in place (tcgen05.ld/st) -- exact, since l uses
// the same reference.
#include "sf_internal.h"
#include "sf_ptx.cuh"

#ifndef SF_ATTN_SFREE
#define SF_ATTN_SFREE 1  // release S buffers right after the score load
#endif
#ifndef SF_ATTN_F16PV
#define SF_ATTN_F16PV 1  // fp16 P/V^T with the ones-row row sum
#endif

namespace sf {

namespace attn {
constexpr int BQ = 128;  // queries per tile (2 tiles per CTA)
constexpr int BKV = 64;  // keys per KV tile
constexpr int HD = 64;
constexpr int Q_BYTES = BQ * HD * 2;   // 16 KB per tile
constexpr int K_BYTES = BKV * HD * 2;  // 8 KB  (64 kv rows x 128 B)
constexpr int V_ROWS = HD + 16;        // V^T rows 0..63 from TMA; row 64 = ones (-> row sum l), 65..79 = 0
constexpr int V_TMA_BYTES = HD * BKV * 2;   // 8 KB loaded per stage
constexpr int V_BYTES = V_ROWS * BKV * 2;   // 10 KB per stage
constexpr int P_BYTES = BQ * BKV * 2;  // 16 KB per tile and buffer (128 rows x 128 B)
constexpr int KV_STAGES = 6;  // refill of tile j+6 starts after tile j: 3 iterations of slack
constexpr int SMEM = 1024 + 2 * Q_BYTES + KV_STAGES * (K_BYTES + V_BYTES) + 4 * P_BYTES + 256;
constexpr float RESCALE_LOG2 = 8.0f;  // lazy-rescale threshold
constexpr int TMEM_COLS = 512;
__host__ __device__ constexpr uint32_t S_COL(int t, int b) { return 64u * (2 * t + b); }
__host__ __device__ constexpr uint32_t O_COL(int t) { return 256u + 96u * t; }  // 80 used (64 O + l), 96 apart
constexpr int THREADS = 352;  // 8 softmax warps + TMA warp + one MMA warp per tile
}  // namespace attn

// exp2 of two fp32 arguments via one f16x2 MUFU op; returns the packed f16 pair
// (lo = first argument), i.e. the P words for the fp16 PV MMA.
__device__ __forceinline__ uint32_t ex2_f16x2(float lo, float hi) {
  uint32_t x, y;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(x) : "f"(hi), "f"(lo));
  asm("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(attn::THREADS, 1)
    attn_fwd_tcgen05(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                     const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ out, int T, int heads) {
  using namespace attn;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                      // [2][Q_BYTES]
  uint8_t* sK = sQ + 2 * Q_BYTES;          // [KV_STAGES][K_BYTES]
  uint8_t* sV = sK + KV_STAGES * K_BYTES;  // [KV_STAGES][V_BYTES]
  uint8_t* sP = sV + KV_STAGES * V_BYTES;  // [tile][buffer][P_BYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 4 * P_BYTES);
  uint64_t* q_full = bars + 0;
  uint64_t* kv_full = bars + 1;                 // [KV_STAGES]
  uint64_t* kv_empty = bars + 1 + KV_STAGES;    // [KV_STAGES]
  uint64_t* s_full = bars + 1 + 2 * KV_STAGES;  // [tile][buffer] = 4
  // [tile][P buffer]: P written, S buffer consumed, O rescaled.  One barrier per
  // buffer: a softmax warpgroup may run a full tile ahead of the MMA thread, and
  // per-buffer phases can never be lapped (tile j+2 needs S issued after tile j).
  uint64_t* p_full = s_full + 4;
  uint64_t* o_full = p_full + 4;                // [tile][P buffer]: PV that read that buffer is done
  uint64_t* s_free = o_full + 4;                // [tile][S buffer]: scores copied to registers
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(s_free + 4);
  static_assert(8 * (1 + 2 * KV_STAGES + 4 + 4 + 4 + 4) + 4 <= 256, "barrier area");

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int q0 = blockIdx.x * (2 * BQ);
  const int bh = blockIdx.y;  // row * heads + head
  const int nkv = T / BKV;

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    mbar_init(q_full, 1);
    for (int s = 0; s < KV_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 2);  // released by both MMA issuers
    }
    for (int i = 0; i < 4; ++i) mbar_init(&s_full[i], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&p_full[i], 128);
    for (int i = 0; i < 4; ++i) mbar_init(&o_full[i], 1);
    for (int i = 0; i < 4; ++i) mbar_init(&s_free[i], 128);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<TMEM_COLS>(tmem_holder);
  // V^T rows 64..79 of every stage: row 64 = fp16 ones (its PV output column is
  // the softmax row sum), rows 65..79 = 0.  Constant rows are swizzle-invariant.
  for (int i = threadIdx.x; i < KV_STAGES * 16 * 8; i += blockDim.x) {
    const int stg = i / 128, rr = i % 128 / 8, ch = i % 8;
    const uint32_t w = rr == 0 ? 0x3C003C00u : 0u;
    *reinterpret_cast<uint4*>(sV + stg * V_BYTES + (HD + rr) * 128 + ch * 16) = make_uint4(w, w, w, w);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 8) {
    if (lane == 0) {
      // ---------------- TMA producer
      mbar_expect_tx(q_full, 2 * Q_BYTES);
      tma_load_2d(sQ, &tmQ, q_full, 0, bh * T + q0);
      tma_load_2d(sQ + Q_BYTES, &tmQ, q_full, 0, bh * T + q0 + BQ);
      for (int j = 0; j < nkv; ++j) {
        const int s = j % KV_STAGES;
        mbar_wait(&kv_empty[s], ((j / KV_STAGES) & 1) ^ 1);
        mbar_expect_tx(&kv_full[s], K_BYTES + V_TMA_BYTES);
        tma_load_2d(sK + s * K_BYTES, &tmK, &kv_full[s], 0, bh * T + j * BKV);
        tma_load_2d(sV + s * V_BYTES, &tmV, &kv_full[s], j * BKV, bh * HD);
      }
    }
  } else if (warp == 9 || warp == 10) {
    if (lane == 0) {
      const int t = warp - 9;  // the query tile this thread issues for
      // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16_f32(128, 64);  // S = Q K^T: bf16, 128 x 64
      // O = P V: fp16 P and V^T, 128 x 80 (the extra ones-row of V^T yields the row sum)
#if SF_ATTN_F16PV
      constexpr uint32_t idesc_pv = (1u << 4) | ((uint32_t)V_ROWS >> 3 << 17) | ((128u >> 4) << 24);
#else
      constexpr uint32_t idesc_pv = idesc_bf16_f32(128, 64);
#endif
      auto issue_s = [&](int t, int j) {
        const uint32_t q_addr = smem_u32(sQ + t * Q_BYTES);
        const uint32_t k_addr = smem_u32(sK + (j % KV_STAGES) * K_BYTES);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          mma_bf16_ss(tmem + S_COL(t, j & 1), sw128_kmajor_desc(q_addr + k * 32),
                      sw128_kmajor_desc(k_addr + k * 32), idesc, k != 0);
        mma_commit(&s_full[2 * t + (j & 1)]);
      };
      auto issue_pv = [&](int t, int j) {
        const uint32_t p_addr = smem_u32(sP + (2 * t + (j & 1)) * P_BYTES);
        const uint32_t v_addr = smem_u32(sV + (j % KV_STAGES) * V_BYTES);
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)
          mma_bf16_ss(tmem + O_COL(t), sw128_kmajor_desc(p_addr + k * 32), sw128_kmajor_desc(v_addr + k * 32),
                      idesc_pv, (j | k) != 0);
        mma_commit(&o_full[2 * t + (j & 1)]);
      };
      mbar_wait(q_full, 0);
      for (int j = 0; j < 2 && j < nkv; ++j) {
        mbar_wait(&kv_full[j % KV_STAGES], (j / KV_STAGES) & 1);
        tc_fence_after();
        issue_s(t, j);
      }
#pragma unroll 1
      for (int j = 0; j < nkv; ++j) {
#if SF_ATTN_SFREE
        if (j + 2 < nkv) {
          // S buffer j%2 is free as soon as the softmax has the scores in registers
          mbar_wait(&kv_full[(j + 2) % KV_STAGES], ((j + 2) / KV_STAGES) & 1);
          mbar_wait(&s_free[2 * t + (j & 1)], (j >> 1) & 1);
          tc_fence_after();
          issue_s(t, j + 2);
        }
        mbar_wait(&p_full[2 * t + (j & 1)], (j >> 1) & 1);  // P_t(j) written, O_t rescaled
        tc_fence_after();
        issue_pv(t, j);
#else
        if (j + 2 < nkv) mbar_wait(&kv_full[(j + 2) % KV_STAGES], ((j + 2) / KV_STAGES) & 1);
        mbar_wait(&p_full[2 * t + (j & 1)], (j >> 1) & 1);
        tc_fence_after();
        issue_pv(t, j);
        if (j + 2 < nkv) issue_s(t, j + 2);
#endif
        mma_commit(&kv_empty[j % KV_STAGES]);  // this tile is done with K_j / V_j
      }
    }
  } else if (warp < 8) {
    // ---------------- softmax warpgroups: warps 0-3 -> tile A, 4-7 -> tile B
    const int t = warp >> 2;
    const uint32_t quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((quarter * 32) << 16);
    const uint32_t o_addr = lane_base + O_COL(t);
    const float L2E = 1.4426950408889634f;
    float m_ref = -INFINITY;  // log2-domain exponent reference (the O accumulator's units)
    float lsum = 0.f;         // (bf16 P variant only)
    uint8_t* prow = sP + (2 * t) * P_BYTES + r * 128;
    const uint32_t sw = (uint32_t)(r & 7);

#pragma unroll 1
    for (int j = 0; j < nkv; ++j) {
      mbar_wait(&s_full[2 * t + (j & 1)], (j >> 1) & 1);
      tc_fence_after();
      float s[BKV];
      tmem_ld32(lane_base + S_COL(t, j & 1), *reinterpret_cast<float(*)[32]>(&s[0]));
      tmem_ld32(lane_base + S_COL(t, j & 1) + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
      tmem_ld_wait();
#if SF_ATTN_SFREE
      tc_fence_before();
      mbar_arrive(&s_free[2 * t + (j & 1)]);  // the MMA may overwrite this S buffer now
#endif
      float mx[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) mx[i] = s[i];
#pragma unroll
      for (int i = 8; i < BKV; ++i) mx[i & 7] = fmaxf(mx[i & 7], s[i]);
      const float m_tile = L2E * fmaxf(fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3])),
                                       fmaxf(fmaxf(mx[4], mx[5]), fmaxf(mx[6], mx[7])));
      if (j == 0) {
        m_ref = m_tile;
      } else {
        const bool grow = m_tile > m_ref + RESCALE_LOG2;
        if (__any_sync(0xffffffffu, grow)) {
          // the PV of tile j-1 must land in O before O is rescaled
          mbar_wait(&o_full[2 * t + ((j - 1) & 1)], ((j - 1) >> 1) & 1);
          tc_fence_after();
          const float a = grow ? ex2(m_ref - m_tile) : 1.0f;
          if (grow) m_ref = m_tile;
#pragma unroll
          for (int h = 0; h < 3; ++h) {  // O and its l column (+16 padding columns)
            float ov[32];
            tmem_ld32(o_addr + 32 * h, ov);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 32; ++i) ov[i] *= a;
            tmem_st32(o_addr + 32 * h, ov);
          }
          tmem_st_wait();
        }
      }
      // P buffer j%2 was last read by the PV of tile j-2
      if (j >= 2) mbar_wait(&o_full[2 * t + (j & 1)], ((j - 2) >> 1) & 1);
      uint8_t* pbuf = prow + (j & 1) * P_BYTES;
#pragma unroll
      for (int c = 0; c < BKV / 8; ++c) {  // 8 chunks of 8 columns = one 16-byte P chunk each
        uint32_t pk[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          // two exponentials per MUFU op: x in f16 (|x| <= 8 + range of s), P in f16
#if SF_ATTN_F16PV
          pk[i] = ex2_f16x2(fmaf(s[8 * c + 2 * i], L2E, -m_ref), fmaf(s[8 * c + 2 * i + 1], L2E, -m_ref));
#else
          const float p0 = ex2(fmaf(s[8 * c + 2 * i], L2E, -m_ref)), p1 = ex2(fmaf(s[8 * c + 2 * i + 1], L2E, -m_ref));
          lsum += p0 + p1;
          pk[i] = pack_bf16(p0, p1);
#endif
        }
        *reinterpret_cast<uint4*>(pbuf + (((uint32_t)c ^ sw) * 16)) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
      }
      fence_proxy_async_smem();
      tc_fence_before();
      mbar_arrive(&p_full[2 * t + (j & 1)]);
    }
    // epilogue: O / l -> bf16 -> out[row*T + q, head*64 ...]  (PVs complete in issue order)
    mbar_wait(&o_full[2 * t + ((nkv - 1) & 1)], ((nkv - 1) >> 1) & 1);
    tc_fence_after();
    float lv[32];
    tmem_ld32(o_addr + 64, lv);  // column 64 = sum_k P[r, k] (ones-row of V^T), exactly the P the MMA saw
    tmem_ld_wait();
#if SF_ATTN_F16PV
    const float inv = 1.0f / lv[0];
#else
    const float inv = 1.0f / (lv[0] * 0.0f + lsum);
#endif
    const int row = bh / heads, head = bh % heads;
    __nv_bfloat16* dst = out + ((int64_t)row * T + q0 + t * BQ + r) * (heads * HD) + head * HD;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      float ov[32];
      tmem_ld32(o_addr + 32 * h, ov);
      tmem_ld_wait();
#pragma unroll
      for (int i = 0; i < 4; ++i)
        reinterpret_cast<uint4*>(dst + 32 * h)[i] =
            make_uint4(pack_bf16(ov[8 * i] * inv, ov[8 * i + 1] * inv), pack_bf16(ov[8 * i + 2] * inv, ov[8 * i + 3] * inv),
                       pack_bf16(ov[8 * i + 4] * inv, ov[8 * i + 5] * inv), pack_bf16(ov[8 * i + 6] * inv, ov[8 * i + 7] * inv));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<attn::TMEM_COLS>(tmem);
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
  dim3 grid(T / (2 * attn::BQ), (unsigned)(rows * heads));
  attn_fwd_tcgen05<<<grid, attn::THREADS, attn::SMEM, st>>>(m.q, m.k, m.v, out, T, heads);
  return cuda_status();
}

}  // namespace sf

extern "C" int sf_attention(const void* q, const void* k, const void* vt, void* out, int64_t rows, int32_t heads,
                            int32_t T, void* stream) {
  if (rows < 1 || heads < 1 || T < 256 || T % 256) return SF_ERR_PARAMETER;
  sf::AttnMaps m;
  if (sf::make_attn_maps(&m, q, k, vt, rows, heads, T) != SF_OK) return SF_ERR_CUDA;
  return sf::launch_attn(m, reinterpret_cast<__nv_bfloat16*>(out), rows, heads, T, (cudaStream_t)stream);
}

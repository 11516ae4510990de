// Flash attention for the DiT velocity field on tcgen05 / TMEM / TMA (sm_100a).
//
// Persistent kernel: one CTA per SM walks work items (latent row, head, pair of
// 128-query tiles A/B); T tokens (1024), head dim 64, no mask.  Q arrives
// pre-scaled by 1/sqrt(64) from the QKV GEMM epilogue, V arrives transposed
// ([hd, T], fp16) so every MMA reads K-major operands.  KV tiles are 64 keys.
//
//   warps 0-3   softmax of tile A (thread r = query row r = TMEM lane r)
//   warps 4-7   softmax of tile B
//   warp 8      TMA producer: Q (double-buffered across items), K_j / V_j^T ring
//   warps 9,10  MMA issuers, one per query tile (warp 9 owns TMEM)
//
// TMEM (512 columns): S_A0 [0,64) S_A1 [64,128) S_B0 [128,192) S_B1 [192,256)
//                     O_A [256,336) O_B [384,464)
// S is double-buffered per tile; P_t(j) (fp16 pairs) is written by the softmax
// into the upper 32 columns of S_t(j)'s buffer and consumed from TMEM by the PV
// MMA (A operand in TMEM, "TS" form), so P never touches shared memory.  Per
// tile t the tensor-core program is
//     S_t(j) = Q_t K_j^T        (M=128, N=64, K=64, bf16 -> f32)
//     O_t   += P_t(j) V_j       (M=128, N=80, K=64, fp16 -> f32; A from TMEM)
// with S_t(j+2) issued right after PV_t(j) into the same buffer (tcgen05 MMAs of
// one thread execute in issue order, so S_t(j+2) cannot overwrite P_t(j) before
// PV_t(j) has read it); S is therefore computed a full softmax iteration ahead.
// V^T carries a ones-row (row 64) so column 64 of O is the softmax row sum l of
// exactly the fp16 P the MMA consumed.  The exponent reference m is updated
// lazily (only when a row max grows by > 8 in log2 units; then the softmax
// rescales O in TMEM).  Exponentials: a fixed share of each row goes through a
// degree-3 polynomial 2^x on the FMA pipe (packed f32x2 ops), the rest through
// MUFU.EX2.  Across items the MMA warps start S(0), S(1) of the next item right
// after the last PVs of the current one and the producer prefetches the next Q,
// so CTA prologues are hidden.
#include "sf_internal.h"
#include "sf_ptx.cuh"

#ifndef SF_ATTN_TRACE
#define SF_ATTN_TRACE 0  // diagnostics: clock64 timeline of CTA 0 (sf_attn_trace_read)
#endif

namespace sf {

#if SF_ATTN_TRACE
__device__ long long g_attn_trace[16 * 64];
#define ATR(role, idx)                                                               \
  do {                                                                               \
    if (blockIdx.x == 0 && (idx) < 64) g_attn_trace[(role) * 64 + (idx)] = clock64(); \
  } while (0)
#else
#define ATR(role, idx) \
  do {                 \
  } while (0)
#endif

namespace attn {
constexpr int BQ = 128;  // queries per tile (2 tiles per item)
constexpr int BKV = 64;  // keys per KV tile
constexpr int KV_STAGES = 6;  // K/V^T ring depth (64-key stages of 18 KB at head dim 64)
constexpr int EMU_PAIRS = 6;  // exp2 pairs per 32-key chunk evaluated by the FMA-pipe polynomial (of 16)
constexpr int QBUF = 2;
constexpr float RESCALE_LOG2 = 8.0f;
constexpr int TMEM_COLS = 512;
// S_t,b: tile t, buffer b (64 fp32 columns); P_t,b (fp16 pairs) aliases its upper 32 columns
__host__ __device__ constexpr uint32_t S_COL(int t, int b) { return 64u * (2 * t + b); }
__host__ __device__ constexpr uint32_t P_COL(int t, int b) { return 64u * (2 * t + b) + 32u; }
__host__ __device__ constexpr uint32_t O_COL(int t) { return 256u + 128u * t; }
// head dim 64: Q_t is copied into TMEM (tcgen05.cp) and the S MMA reads it from there,
// so K is the only shared-memory operand of QK^T (halves its smem traffic)
__host__ __device__ constexpr uint32_t Q_COL(int t) { return 352u + 128u * t; }
constexpr int THREADS = 352;
}  // namespace attn

// Head-dim dependent layout.  Q / K rows are split into a 64-element part
// (128-byte rows, SW128) and, for HD > 64, a 16-element part (32-byte rows,
// SW32) holding head-dim elements 64..79 (72..79 zero-filled by TMA out of
// bounds), so the QK^T MMA runs over K = 80.  V^T tiles hold HD data rows, a
// ones-row at HD (-> softmax row sum in O column HD) and zero rows up to 80.
template <int HD>
struct AttnCfg {
  static_assert(HD == 64 || HD == 72, "head dim");
  static constexpr int HI = HD > 64 ? 16 : 0;
  static constexpr int KSTEPS = (64 + HI) / 16;
  static constexpr int Q_LO = attn::BQ * 128;
  static constexpr int Q_TILE = Q_LO + attn::BQ * HI * 2;   // 16 / 20 KB
  static constexpr int Q_BYTES = 2 * Q_TILE;                // both tiles of an item
  static constexpr int K_LO = attn::BKV * 128;
  static constexpr int K_BYTES = K_LO + attn::BKV * HI * 2;  // 8 / 10 KB
  static constexpr int V_ROWS = 80;
  static constexpr int V_BYTES = V_ROWS * 128;
  static constexpr int V_TMA = HD * 128;  // bytes loaded per stage
  static constexpr int STAGE = K_BYTES + V_BYTES;
  static constexpr int SMEM = 1024 + attn::QBUF * Q_BYTES + attn::KV_STAGES * STAGE + 256;
  static constexpr int O_LD = HD == 64 ? 64 : 80;  // O columns read by the epilogue (O, then l at column HD)
};

// K-major SW32 descriptor (32-byte rows, 8-row atoms of 256 B).
__device__ __forceinline__ uint64_t sw32_kmajor_desc(uint32_t smem_addr) {
  return (uint64_t)((smem_addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_f16(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// 2^x for a pair, on the FMA pipe: x = j + f (j = rint(x), |f| <= 1/2),
// 2^f by a degree-3 minimax polynomial (rel. err 7.7e-5 < half an fp16 ulp),
// 2^j added into the exponent field.  x is clamped to >= -127 (P underflows to 0 in fp16 anyway).
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  const float kMagic = 12582912.0f;  // 1.5 * 2^23: x + magic rounds x to an integer in the low mantissa bits
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

// D[tmem] (+)= A[tmem] * B[smem]^T (A operand read from TMEM, "TS" form).
// smem -> TMEM copy of a 128-row x 32-byte block described by an smem matrix descriptor.
__device__ __forceinline__ void tmem_cp_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

__device__ __forceinline__ void mma_f16_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(accumulate)
      : "memory");
}

// PDL = launched with programmatic serialisation (small batches, sf_internal.h g_pdl): a separate
// instantiation, because any PDL code in the kernel measured 2-5% slower at full occupancy through
// the softmax's register allocation
template <int HD, bool PDL>
__global__ void __launch_bounds__(attn::THREADS, 1)
    attn_fwd_tcgen05(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmQh,
                     const __grid_constant__ CUtensorMap tmK, const __grid_constant__ CUtensorMap tmKh,
                     const __grid_constant__ CUtensorMap tmV, __nv_bfloat16* __restrict__ out, int T, int heads,
                     int nitems) {
  using namespace attn;
  using AC = AttnCfg<HD>;
  constexpr bool Q_IN_TMEM = HD == 64;  // Q staged in TMEM (tcgen05.cp), S MMA in TS form
  constexpr int Q_TILE = AC::Q_TILE, Q_BYTES = AC::Q_BYTES, K_BYTES = AC::K_BYTES, STAGE = AC::STAGE;
  constexpr int V_ROWS = AC::V_ROWS, V_TMA = AC::V_TMA;
  extern __shared__ uint8_t smem_raw[];
  // 1024-align by offsetting into the shared array (keeps the pointer in the shared window: LDS/STS, not generic)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sQ = smem;                  // [QBUF][2 tiles][Q_TILE]
  uint8_t* sKV = sQ + QBUF * Q_BYTES;  // [KV_STAGES][K (64 x 128 B) | V^T (80 x 128 B)]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sKV + KV_STAGES * STAGE);
  uint64_t* q_full = bars;                   // [QBUF]
  uint64_t* q_empty = bars + 2;              // [QBUF]   both tiles issued their last S on this Q
  uint64_t* kv_full = bars + 4;              // [KV_STAGES]
  uint64_t* kv_empty = kv_full + KV_STAGES;  // [KV_STAGES]  both tiles' PV on this K/V done
  uint64_t* s_full = kv_empty + KV_STAGES;   // [tile][buffer]  S_t(j) landed in TMEM
  uint64_t* p_full = s_full + 4;             // [tile][buffer]  P_t(j) written to TMEM (O rescaled if needed)
  // [tile][buffer]  PV_t(j) complete.  Per buffer so that a wait is never two
  // phases behind: when softmax(j) runs, PV_t(j-2) is known complete (S_t(j)
  // was issued after it) but PV_t(j-1) need not be.
  uint64_t* o_full = p_full + 4;
  uint64_t* o_free = o_full + 4;             // [tile]  epilogue has read O_t
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(o_free + 2);
  static_assert(8 * (4 + 2 * KV_STAGES + 14) + 4 <= 256, "barrier area");

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int nkv = T / BKV;  // even (T % 256 == 0): buffer of global KV iteration G is G & 1
  const int qpairs = T / (2 * BQ);

  if (warp == 8 && lane == 0) {
    tma_prefetch(&tmQ);
    tma_prefetch(&tmK);
    tma_prefetch(&tmV);
    if constexpr (AC::HI > 0) {
      tma_prefetch(&tmQh);
      tma_prefetch(&tmKh);
    }
    for (int i = 0; i < QBUF; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 2);
    }
    for (int s = 0; s < KV_STAGES; ++s) {
      mbar_init(&kv_full[s], 1);
      mbar_init(&kv_empty[s], 2);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 128);
      mbar_init(&o_full[i], 1);
    }
    for (int t = 0; t < 2; ++t) mbar_init(&o_free[t], 128);
    fence_barrier_init();
  }
  if (warp == 9) tmem_alloc<TMEM_COLS>(tmem_holder);
  // V^T rows HD..79 of every stage: row HD = fp16 ones (its PV output column is
  // the softmax row sum), the rest 0 (constant rows are swizzle-invariant).
  constexpr int CROWS = V_ROWS - HD;
  for (int i = threadIdx.x; i < KV_STAGES * CROWS * 8; i += blockDim.x) {
    const int stg = i / (CROWS * 8), rr = i % (CROWS * 8) / 8, ch = i % 8;
    const uint32_t w = rr == 0 ? 0x3C003C00u : 0u;
    *reinterpret_cast<uint4*>(sKV + stg * STAGE + K_BYTES + (HD + rr) * 128 + ch * 16) = make_uint4(w, w, w, w);
  }
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if constexpr (PDL) {
    if (threadIdx.x == 0) pdl_trigger(true);  // the next kernel's CTAs may start their prologue
    pdl_wait(true);                           // Q / K / V^T of the previous kernel are complete
  }

  if (warp == 8) {
    if (lane == 0) {
      // ---------------- TMA producer
      int kv = 0, local = 0;
      for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++local) {
        const int bh = item / qpairs, q0 = (item % qpairs) * 2 * BQ;
        const int qb = local & 1;
        mbar_wait(&q_empty[qb], ((local >> 1) & 1) ^ 1);
        mbar_expect_tx(&q_full[qb], Q_BYTES);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
          tma_load_2d(sQ + qb * Q_BYTES + t * Q_TILE, &tmQ, &q_full[qb], 0, bh * T + q0 + t * BQ);
          if constexpr (AC::HI > 0)
            tma_load_2d(sQ + qb * Q_BYTES + t * Q_TILE + AC::Q_LO, &tmQh, &q_full[qb], 64, bh * T + q0 + t * BQ);
        }
        for (int j = 0; j < nkv; ++j, ++kv) {
          const int s = kv % KV_STAGES;
          mbar_wait(&kv_empty[s], ((kv / KV_STAGES) & 1) ^ 1);
          uint8_t* st = sKV + s * STAGE;
          mbar_expect_tx(&kv_full[s], K_BYTES + V_TMA);
          tma_load_2d(st, &tmK, &kv_full[s], 0, bh * T + j * BKV);
          if constexpr (AC::HI > 0) tma_load_2d(st + AC::K_LO, &tmKh, &kv_full[s], 64, bh * T + j * BKV);
          tma_load_2d(st + K_BYTES, &tmV, &kv_full[s], j * BKV, bh * HD);
        }
      }
    }
  } else if (warp == 9 || warp == 10) {
    // ---------------- MMA issuer, one warp per query tile (the two progress independently).
    // The whole warp runs the loop so every operand is warp-uniform (uniform
    // registers, no per-MMA R2UR waterfall); one elected lane issues.
    const int t = warp - 9;
    constexpr uint32_t idesc_s = idesc_bf16_f32(128, BKV);
    constexpr uint32_t idesc_pv = (1u << 4) | ((uint32_t)V_ROWS >> 3 << 17) | ((128u >> 4) << 24);  // f16 A/B
    const uint64_t q_desc0 = sw128_kmajor_desc(smem_u32(sQ + t * Q_TILE));
    const uint64_t kv_desc0 = sw128_kmajor_desc(smem_u32(sKV));
    // descriptor address field is addr >> 4: +32 B per K step = +2, +STAGE per stage
    auto issue_s = [&](int qb, int s, int b) {
      const uint64_t qd = q_desc0 + (uint64_t)((qb * Q_BYTES) >> 4);
      const uint64_t kd = kv_desc0 + (uint64_t)((s * STAGE) >> 4);
      if (elect_one()) {
        if constexpr (Q_IN_TMEM) {
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_f16_ts(tmem + S_COL(t, b), tmem + Q_COL(t) + 8 * k, kd + 2 * k, idesc_s, k != 0);
        } else {
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem + S_COL(t, b), qd + 2 * k, kd + 2 * k, idesc_s, k != 0);
        }
        if constexpr (AC::HI > 0)  // head-dim elements 64..79 from the SW32 parts
          mma_bf16_ss(tmem + S_COL(t, b), sw32_kmajor_desc(smem_u32(sQ + qb * Q_BYTES + t * Q_TILE + AC::Q_LO)),
                      sw32_kmajor_desc(smem_u32(sKV + s * STAGE + AC::K_LO)), idesc_s, 1);
        mma_commit(&s_full[2 * t + b]);
      }
      __syncwarp();
    };
    auto issue_pv = [&](int s, int b, bool acc) {
      const uint64_t vd = kv_desc0 + (uint64_t)((s * STAGE + K_BYTES) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < BKV / 16; ++k)
            mma_f16_ts(tmem + O_COL(t), tmem + P_COL(t, b) + 8 * k, vd + 2 * k, idesc_pv, acc || k != 0);
        mma_commit(&o_full[2 * t + b]);
        mma_commit(&kv_empty[s]);
      }
      __syncwarp();
    };
    int kv = 0, local = 0;
    for (int item = blockIdx.x; item < nitems; item += gridDim.x, ++local) {
      const int qb = local & 1;
      mbar_wait(&q_full[qb], (local >> 1) & 1);
      if constexpr (Q_IN_TMEM) {
        // the previous item's last S on this tile (buffer 1) has finished reading Q_t in TMEM
        if (kv > 0) mbar_wait(&s_full[2 * t + 1], ((kv - 1) >> 1) & 1);
        tc_fence_after();
        const uint64_t qd = q_desc0 + (uint64_t)((qb * Q_BYTES) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < 4; ++k) tmem_cp_128x256b(tmem + Q_COL(t) + 8 * k, qd + 2 * k);
          mma_commit(&q_empty[qb]);  // Q smem buffer free once the copy has read it
        }
        __syncwarp();
      }
      for (int j = 0; j < 2; ++j) {
        const int G = kv + j;
        mbar_wait(&kv_full[G % KV_STAGES], (G / KV_STAGES) & 1);
        tc_fence_after();
        issue_s(qb, G % KV_STAGES, j);
      }
#pragma unroll 1
      for (int j = 0; j < nkv; ++j) {
        const int G = kv + j, b = j & 1;
        mbar_wait(&p_full[2 * t + b], (G >> 1) & 1);          // P_t(j) in TMEM, O_t rescaled
        if (lane == 0) ATR(4 + 2 * t, G);
        if (j == 0) mbar_wait(&o_free[t], (local & 1) ^ 1);  // previous item's O read out
        tc_fence_after();
        issue_pv(G % KV_STAGES, b, j != 0);
        if (j + 2 < nkv) {
          // S_t(j+2) reuses buffer b: issued after PV_t(j), which reads P_t(j) from it
          mbar_wait(&kv_full[(G + 2) % KV_STAGES], ((G + 2) / KV_STAGES) & 1);
          tc_fence_after();
          if (lane == 0) ATR(5 + 2 * t, G + 2);
          issue_s(qb, (G + 2) % KV_STAGES, b);
          if (!Q_IN_TMEM && j + 3 == nkv) {
            if (elect_one()) mma_commit(&q_empty[qb]);  // last S of this tile on this Q
            __syncwarp();
          }
        }
      }
      kv += nkv;
    }
  } else {
    // ---------------- softmax warpgroups: warps 0-3 -> tile A, 4-7 -> tile B
    const int t = warp >> 2;
    const uint32_t quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const uint32_t lane_base = tmem + ((quarter * 32) << 16);
    const uint32_t o_addr = lane_base + O_COL(t);
    const float L2E = 1.4426950408889634f;
    int G = 0;
#pragma unroll 1
    for (int item = blockIdx.x; item < nitems; item += gridDim.x) {
      float m_ref = -INFINITY;  // log2-domain exponent reference (the O accumulator's units)
#pragma unroll 1
      for (int j = 0; j < nkv; ++j, ++G) {
        const int b = j & 1;
        mbar_wait(&s_full[2 * t + b], (G >> 1) & 1);
        if (lane == 0 && quarter == 0) ATR(2 * t, G);
        tc_fence_after();
        float s[BKV];
        tmem_ld32(lane_base + S_COL(t, b), *reinterpret_cast<float(*)[32]>(&s[0]));
        tmem_ld32(lane_base + S_COL(t, b) + 32, *reinterpret_cast<float(*)[32]>(&s[32]));
        tmem_ld_wait();
        if (lane == 0 && quarter == 0) ATR(8 + 4 * t, G);  // S in registers
        // four chains of 3-input maxima over 16 scores each (7 + 1 FMNMX3 per chain), then 4 -> 1
        float mx[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) mx[q] = fmaxf(fmaxf(s[q], s[q + 4]), s[q + 8]);
#pragma unroll
        for (int i = 12; i < BKV - 4; i += 8)
#pragma unroll
          for (int q = 0; q < 4; ++q) mx[q] = fmaxf(fmaxf(mx[q], s[i + q]), s[i + 4 + q]);
#pragma unroll
        for (int q = 0; q < 4; ++q) mx[q] = fmaxf(mx[q], s[BKV - 4 + q]);
        const float m_tile = L2E * fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        if (j == 0) {
          m_ref = m_tile;
        } else {
          const bool grow = m_tile > m_ref + RESCALE_LOG2;
          if (__any_sync(0xffffffffu, grow)) {
            // PV_t(j-1) must have landed in O before O is rescaled
            mbar_wait(&o_full[2 * t + (b ^ 1)], ((G - 1) >> 1) & 1);
            tc_fence_after();
            const float a = grow ? ex2(m_ref - m_tile) : 1.0f;
            if (grow) m_ref = m_tile;
#pragma unroll
            for (int h = 0; h < 5; ++h) {  // O (64) and its l column (+15 zero columns)
              float ov[16];
              tmem_ld16(o_addr + 16 * h, ov);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 16; ++i) ov[i] *= a;
              tmem_st16(o_addr + 16 * h, ov);
            }
            tmem_st_wait();
          }
        }
        if (lane == 0 && quarter == 0) ATR(9 + 4 * t, G);  // max + rescale check done
        const float2 l2e2 = make_float2(L2E, L2E), negm = make_float2(-m_ref, -m_ref);
#pragma unroll
        for (int c = 0; c < BKV / 32; ++c) {
          uint32_t pk[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 x = __ffma2_rn(make_float2(s[32 * c + 2 * i], s[32 * c + 2 * i + 1]), l2e2, negm);
            float2 p;
            if (i < attn::EMU_PAIRS) {
              p = exp2_poly2(x);
            } else {
              p.x = ex2(x.x);
              p.y = ex2(x.y);
            }
            pk[i] = pack_f16(p.x, p.y);
          }
          tmem_st16u(lane_base + P_COL(t, b) + 16 * c, pk);
        }
        if (lane == 0 && quarter == 0) ATR(10 + 4 * t, G);  // P computed, stores issued
        tmem_st_wait();
        if (lane == 0 && quarter == 0) ATR(11 + 4 * t, G);  // stores complete
        tc_fence_before();
        mbar_arrive(&p_full[2 * t + b]);
        if (lane == 0 && quarter == 0) ATR(2 * t + 1, G);
      }
      // epilogue: O / l -> bf16 -> out[row*T + q, head*HD ...]
      mbar_wait(&o_full[2 * t + 1], ((G - 1) >> 1) & 1);  // last PV (odd buffer); earlier PVs completed before it
      tc_fence_after();
      float ov[80];
      tmem_ld32(o_addr, *reinterpret_cast<float(*)[32]>(&ov[0]));
      tmem_ld32(o_addr + 32, *reinterpret_cast<float(*)[32]>(&ov[32]));
      tmem_ld16(o_addr + 64, *reinterpret_cast<float(*)[16]>(&ov[64]));
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&o_free[t]);
      const float inv = 1.0f / ov[HD];  // column HD = sum_k P[r, k], exactly the P the MMA saw
      const int bh = item / qpairs, q0 = (item % qpairs) * 2 * BQ;
      const int row = bh / heads, head = bh % heads;
      __nv_bfloat16* dst = out + ((int64_t)row * T + q0 + t * BQ + r) * (heads * HD) + head * HD;
#pragma unroll
      for (int i = 0; i < HD / 8; ++i)
        reinterpret_cast<uint4*>(dst)[i] =
            make_uint4(pack_bf16(ov[8 * i] * inv, ov[8 * i + 1] * inv), pack_bf16(ov[8 * i + 2] * inv, ov[8 * i + 3] * inv),
                       pack_bf16(ov[8 * i + 4] * inv, ov[8 * i + 5] * inv), pack_bf16(ov[8 * i + 6] * inv, ov[8 * i + 7] * inv));
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 9) tmem_dealloc<attn::TMEM_COLS>(tmem);
}

int make_attn_maps(AttnMaps* m, const void* q, const void* k, const void* vt, int64_t rows, int heads, int T,
                   int hd) {
  const uint64_t bhT = (uint64_t)rows * heads * T;
  m->hd = hd;
  if (make_tmap_bf16_2d(&m->q, q, hd, bhT, hd, 64, attn::BQ) != SF_OK) return SF_ERR_CUDA;
  if (make_tmap_bf16_2d(&m->k, k, hd, bhT, hd, 64, attn::BKV) != SF_OK) return SF_ERR_CUDA;
  if (make_tmap_bf16_2d(&m->v, vt, T, (uint64_t)rows * heads * hd, T, 64, hd) != SF_OK) return SF_ERR_CUDA;
  if (hd > 64) {  // elements 64..79 (72..79 out of bounds -> zero fill), 32-byte rows
    if (make_tmap_bf16_2d(&m->qh, q, hd, bhT, hd, 16, attn::BQ, 32) != SF_OK) return SF_ERR_CUDA;
    if (make_tmap_bf16_2d(&m->kh, k, hd, bhT, hd, 16, attn::BKV, 32) != SF_OK) return SF_ERR_CUDA;
  } else {
    m->qh = m->q;
    m->kh = m->k;
  }
  return SF_OK;
}

static int attn_sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <int HD, bool PDL>
static int prepare_attn_hd() {
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(attn_fwd_tcgen05<HD, PDL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             AttnCfg<HD>::SMEM) != cudaSuccess)
      return SF_ERR_CUDA;
    attr = true;
  }
  return SF_OK;
}

int prepare_attn_kernel() {
  return prepare_attn_hd<64, false>() == SF_OK && prepare_attn_hd<72, false>() == SF_OK &&
                 prepare_attn_hd<64, true>() == SF_OK && prepare_attn_hd<72, true>() == SF_OK
             ? SF_OK
             : SF_ERR_CUDA;
}

template <int HD>
static cudaError_t launch_attn_hd(const AttnMaps& m, __nv_bfloat16* out, int T, int heads, int items, int grid,
                                  cudaStream_t st) {
  if (g_pdl)
    return launch_kernel(attn_fwd_tcgen05<HD, true>, dim3(grid), dim3(attn::THREADS), AttnCfg<HD>::SMEM, st, m.q, m.qh,
                         m.k, m.kh, m.v, out, T, heads, items);
  return launch_kernel(attn_fwd_tcgen05<HD, false>, dim3(grid), dim3(attn::THREADS), AttnCfg<HD>::SMEM, st, m.q, m.qh,
                       m.k, m.kh, m.v, out, T, heads, items);
}

int launch_attn(const AttnMaps& m, __nv_bfloat16* out, int64_t rows, int heads, int T, cudaStream_t st) {
  if (prepare_attn_kernel() != SF_OK) return SF_ERR_CUDA;
  const int64_t items = rows * heads * (T / (2 * attn::BQ));
  const int grid = (int)(items < attn_sm_count() ? items : attn_sm_count());
  cudaError_t err;
  if (m.hd == 64)
    err = launch_attn_hd<64>(m, out, T, heads, (int)items, grid, st);
  else if (m.hd == 72)
    err = launch_attn_hd<72>(m, out, T, heads, (int)items, grid, st);
  else
    return SF_ERR_PARAMETER;
  return err == cudaSuccess ? cuda_status() : SF_ERR_CUDA;
}

}  // namespace sf

#if SF_ATTN_TRACE
extern "C" int sf_attn_trace_read(long long* dst) {
  return cudaMemcpyFromSymbol(dst, sf::g_attn_trace, sizeof(long long) * 16 * 64) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" int sf_attention_hd(const void* q, const void* k, const void* vt, void* out, int64_t rows, int32_t heads,
                               int32_t T, int32_t hd, void* stream) {
  if (rows < 1 || heads < 1 || T < 256 || T % 256 || (hd != 64 && hd != 72)) return SF_ERR_PARAMETER;
  sf::AttnMaps m;
  if (sf::make_attn_maps(&m, q, k, vt, rows, heads, T, hd) != SF_OK) return SF_ERR_CUDA;
  return sf::launch_attn(m, reinterpret_cast<__nv_bfloat16*>(out), rows, heads, T, (cudaStream_t)stream);
}

extern "C" int sf_attention(const void* q, const void* k, const void* vt, void* out, int64_t rows, int32_t heads,
                            int32_t T, void* stream) {
  return sf_attention_hd(q, k, vt, out, rows, heads, T, 64, stream);
}

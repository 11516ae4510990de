// Fused DiT-S/2 MLP block: fc1 + GELU + fc2 + gated residual + LayerNorm + modulate
// in one persistent tcgen05 kernel (hidden 384, MLP 1536).  Replaces the fc1 GEMM
// (which wrote the 128 x 1536 GELU'd hidden of every row tile to HBM: 403 MB per
// layer at the bench shape) and the fc2 GEMM (which read it back): the hidden lives
// only in TMEM and shared memory, 64 columns at a time.
//
// Per 128-row tile (one CTA, 14 warps):
//   warp 0      TMA producer: the X tile (xmod rows, 6 x 16 KB SW128 atoms, resident
//               for the tile) and a 3-stage ring of 24 KB weight blocks in MMA order
//   warp 1      MMA issuer: fc1(c) = X . W1[64c:64c+64]^T  (M128 N64 K384) into one of
//               two 64-column TMEM buffers; fc2(c) += GELU(H_c) . W2[:, 64c:64c+64]^T
//               (M128 N384 as two N192 MMAs, K64) into a 384-column TMEM accumulator;
//               issue order fc1(0) fc1(1) fc2(0) fc1(2) fc2(1) ... so the GELU of chunk c
//               overlaps fc1(c+1) and fc2(c-1)
//   warps 2-5   GELU: TMEM -> +b1 -> tanh-GELU -> bf16 -> the SW128 smem H buffer the
//               fc2 MMA reads (double-buffered)
//   warps 6-13  epilogue (2 per TMEM lane quarter, 192 columns each):
//               x = bf16(xres + gate * (acc + b2)) -> xres; row mean / mean-square across
//               the two warps of a quarter; xmod = bf16(LN(x) * (1 + scale) + shift)
// TMEM: fc2 accumulator columns 0-383, fc1 buffers 384-447 and 448-511.
#include <cstdint>
#include <cstdio>

#include "gemm_tcgen05.cuh"
#include "sf_internal.h"
#include "sf_ptx.cuh"

namespace sf {
namespace mlp {
#ifndef SF_MLP_TRACE
#define SF_MLP_TRACE 0
#endif
#if SF_MLP_TRACE
__device__ long long g_mlp_trace[16 * 64];
#define MTR(role, idx)                                                              \
  do {                                                                              \
    if (blockIdx.x == 0 && (idx) < 64) g_mlp_trace[(role) * 64 + (idx)] = clock64(); \
  } while (0)
#else
#define MTR(role, idx) \
  do {                 \
  } while (0)
#endif

#ifndef SF_MLP_PAIR
#define SF_MLP_PAIR 0  // 2-CTA pairs (measured slower: 384 vs 315 us; cross-CTA GELU handoffs): cta_group::2 MMAs (M=256), the weight operand split between the SMs
#endif
#ifndef SF_MLP_HC
#define SF_MLP_HC 128  // hidden columns per chunk: 128 (one TMEM / smem buffer; 275 us) or 64 (two; 317 us)
#endif
constexpr int D = 384, FF = 1536, BM = 128, HC = SF_MLP_HC, NCH = FF / HC;
constexpr int NB = HC == 64 ? 2 : 1;  // fc1 accumulator and H buffers
constexpr int X_ATOM = BM * 64 * 2;                                   // 16 KB: 128 rows x 64 K
constexpr int X_BYTES = 6 * X_ATOM;                                   // 96 KB
constexpr int WBLOCK = 24576;                                         // 24 KB weight block (both CTAs)
constexpr int STAGE = HC == 128 ? 16384 : WBLOCK / (SF_MLP_PAIR ? 2 : 1);  // this CTA's share
constexpr int NSTAGE = HC == 128 ? 4 : (SF_MLP_PAIR ? 6 : 3);
constexpr int H_BYTES = BM * HC * 2;  // 16 / 32 KB
#ifndef SF_MLP_GELU_WARPS
#define SF_MLP_GELU_WARPS 8
#endif
#ifndef SF_MLP_PF
#define SF_MLP_PF -1  // hidden chunk at which the boundary's residual / next X are prefetched to L2 (-1: off)
#endif
#ifndef SF_MLP_PFX
#define SF_MLP_PFX -1  // hidden chunk at which the next tile's X is prefetched to L2 (-1: off)
#endif
#ifndef SF_MLP_CL
#define SF_MLP_CL 1  // CTAs per cluster sharing (TMA-multicasting) the weight stream
#endif
constexpr bool PAIR = SF_MLP_PAIR;
constexpr int CL = PAIR ? 2 : SF_MLP_CL;
static_assert(!PAIR || SF_MLP_CL == 1, "pair mode and weight multicast are exclusive");
constexpr uint16_t CL_MASK = (1u << CL) - 1;
constexpr int WSPLIT = PAIR ? 2 : 1;  // each CTA holds 1/WSPLIT of every weight block
#ifndef SF_MLP_EPI_WARPS
#define SF_MLP_EPI_WARPS 8  // dedicated epilogue warps (the GELU warps join them per tile)
#endif
constexpr int GELU_WARPS = SF_MLP_GELU_WARPS, EPI_WARPS = SF_MLP_EPI_WARPS;
constexpr int WORKERS = GELU_WARPS + EPI_WARPS;  // warps sharing the epilogue
constexpr int PARTS = WORKERS / 4;                // per TMEM lane quarter
constexpr int ECOLS = D / PARTS;                  // output columns per epilogue thread
constexpr int GCOLS = HC / (GELU_WARPS / 4);  // hidden columns per GELU thread
constexpr int THREADS = 32 * (2 + GELU_WARPS + EPI_WARPS);
constexpr int ACC2 = 0, ACC1 = 384;
constexpr int SMEM = 1024 + X_BYTES + NSTAGE * STAGE + NB * H_BYTES + 4 * D * 4 + 2 * 4 * BM * 4 + FF * 4 + 256;
static_assert(HC == 64 || (HC == 128 && !SF_MLP_PAIR && SF_MLP_CL == 1), "128-column chunks: single CTA");

// 2-D TMA load multicast to the CTAs of `mask` (same smem offset and barrier in each).
__device__ __forceinline__ void tma_load_2d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int32_t c0, int32_t c1,
                                               uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
      " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "h"(mask)
      : "memory");
}
// L2 prefetch of one TMA box (no smem, no barrier).
__device__ __forceinline__ void tma_prefetch_2d(const CUtensorMap* m, int32_t c0, int32_t c1) {
  asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global [%0, {%1, %2}];" ::"l"(reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1)
               : "memory");
}
// Arrive on the same-offset mbarrier of every CTA in `mask` once this thread's prior MMAs complete.
__device__ __forceinline__ void mma_commit_mc(uint64_t* bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(mask)
      : "memory");
}

struct Params {
  const float* b1;  // [1536]
  const float* b2;  // [384]
  __nv_bfloat16* xres;
  __nv_bfloat16* xmod;
  const float* gate;   // per-slot vectors: ptr + slot * vec_stride
  const float* shift;
  const float* scale;
  int64_t vec_stride;
  float ln_eps;
  int T;   // tokens per slot
  int M;   // rows
};

__global__ void __maxnreg__(16384 / ((THREADS / 32 + 3) / 4) / 32 / 8 * 8)  // per-SMSP register file
    mlp_fused_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW1,
                     const __grid_constant__ CUtensorMap tmW2, const __grid_constant__ CUtensorMap tmR,
                     const __grid_constant__ CUtensorMap tmRs, const __grid_constant__ CUtensorMap tmMs, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;
  uint8_t* sW = sX + X_BYTES;
  uint8_t* sH = sW + NSTAGE * STAGE;
  float* sVec = reinterpret_cast<float*>(sH + NB * H_BYTES);  // b2 | gate | shift | scale  [4][384]
  float* sRed = sVec + 4 * D;                                 // [2 stats][<= 4 parts][128 rows]
  float* sB1 = sRed + 2 * 4 * BM;                             // fc1 bias [1536]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB1 + FF);
  uint64_t* wfull = bars;               // [NSTAGE]
  uint64_t* wempty = wfull + NSTAGE;    // [NSTAGE]
  uint64_t* xfull = wempty + NSTAGE;
  uint64_t* xempty = xfull + 1;
  uint64_t* a1full = xempty + 1;        // [2] fc1 accumulator ready
  uint64_t* a1empty = a1full + 2;       // [2] GELU warps have read it
  uint64_t* hfull = a1empty + 2;        // [2] H buffer written
  uint64_t* hempty = hfull + 2;         // [2] fc2 has read it
  uint64_t* a2full = hempty + 2;
  uint64_t* a2empty = a2full + 1;
  uint64_t* rfull = a2empty + 1;  // this tile's residual rows landed in the X buffer
  uint64_t* xfree = rfull + 1;    // the epilogue is done with the X buffer (next X may load)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(xfree + 1);

  const uint32_t warp = warp_id(), lane = threadIdx.x & 31;
  const int tiles = p.M / BM;
  const int crank = CL > 1 ? (int)cluster_ctarank() : 0;
  const bool leader = crank == 0;
  // barriers that collect arrivals from both CTAs of a pair live in the leader
  auto lead = [&](uint64_t* bar) -> uint32_t { return mapa_shared(smem_u32(bar), 0); };
  // CTA `crank` of cluster k takes tiles (k + i * nclusters) * CL + crank: every CTA of a
  // cluster runs the same number of tiles (tiles % CL == 0), so their weight streams match
  const int tile0 = (blockIdx.x / CL) * CL + crank, tstride = gridDim.x;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmX);
    tma_prefetch(&tmW1);
    tma_prefetch(&tmW2);
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], PAIR ? 1 : CL);  // multicast: every CTA's MMAs must have consumed the slot
    }
    mbar_init(xfull, 1);
    mbar_init(xempty, 1);
    for (int b = 0; b < 2; ++b) {
      mbar_init(&a1full[b], 1);
      mbar_init(&a1empty[b], WSPLIT * GELU_WARPS * 32);
      mbar_init(&hfull[b], WSPLIT * GELU_WARPS * 32);
      mbar_init(&hempty[b], 1);
    }
    mbar_init(a2full, 1);
    mbar_init(a2empty, WSPLIT * WORKERS * 32);
    mbar_init(rfull, 1);
    mbar_init(xfree, WORKERS * 32);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < FF; i += THREADS) sB1[i] = p.b1[i];
  if (warp == 1) {
    if constexpr (PAIR)
      tmem_alloc_2sm<512>(tmem_holder);
    else
      tmem_alloc<512>(tmem_holder);
  }
  if constexpr (CL > 1) cluster_sync_all();  // the peer's barriers exist before any remote arrive
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      int ws = 0;  // weight blocks issued
      // a 24 KB weight block = nload TMA boxes; with CL > 1 each CTA loads rows
      // [crank * rows/CL, ...) of every box and multicasts them to the whole cluster
      auto wblock = [&](const CUtensorMap* m, int c0, int c1, int nload, int step_c0, int rows) {
        const int s = ws % NSTAGE;
        mbar_wait(&wempty[s], ((ws / NSTAGE) & 1) ^ 1);
        if constexpr (PAIR) {
          // this CTA's half of the block's rows (the pair MMA reads B from both CTAs);
          // both halves complete on the leader's full barrier
          const int part = rows / 2;
          if (leader) mbar_expect_tx(&wfull[s], WBLOCK);
          for (int i = 0; i < nload; ++i)
            tma_load_2d_2sm(sW + s * STAGE + i * (STAGE / nload), m, lead(&wfull[s]), c0 + i * step_c0,
                            c1 + crank * part);
        } else {
          mbar_expect_tx(&wfull[s], STAGE);
          const int part = rows / CL;
          for (int i = 0; i < nload; ++i) {
            uint8_t* dst = sW + s * STAGE + i * (STAGE / nload) + crank * part * 128;
            if constexpr (CL > 1)
              tma_load_2d_mc(dst, m, &wfull[s], c0 + i * step_c0, c1 + crank * part, CL_MASK);
            else
              tma_load_2d(dst, m, &wfull[s], c0 + i * step_c0, c1);
          }
        }
        ++ws;
      };
      int local = 0;
      auto w1 = [&](int c) {
        if constexpr (HC == 128) {  // W1 rows [128c, +128): one 16 KB K-atom per stage
          for (int kb = 0; kb < 6; ++kb) wblock(&tmW1, kb * 64, c * HC, 1, 0, HC);
        } else {  // W1 rows [64c, 64c+64), K halves of 192 (3 atoms of 8 KB each)
          wblock(&tmW1, 0, c * HC, 3, 64, HC);
          wblock(&tmW1, 192, c * HC, 3, 64, HC);
        }
      };
      auto w2 = [&](int c) {
        if constexpr (HC == 128) {  // W2 rows [128n, +128) x K atom a of the chunk
          for (int n = 0; n < 3; ++n)
            for (int a = 0; a < 2; ++a) wblock(&tmW2, c * HC + 64 * a, 128 * n, 1, 0, 128);
        } else {  // W2 rows [0,192) and [192,384), K columns [64c, 64c+64)
          wblock(&tmW2, c * HC, 0, 1, 0, 192);
          wblock(&tmW2, c * HC, 192, 1, 0, 192);
        }
      };
      for (int tile = tile0; tile < tiles; tile += tstride, ++local) {
        // the X buffer: X(tile) for fc1, then the tile's residual rows for the epilogue.
        // W1(0) is requested first (it fits the ring) so it lands during the previous epilogue.
        if constexpr (HC == 64) w1(0);
        mbar_wait(xfree, (local & 1) ^ 1);  // previous tile's epilogue left the buffer
        MTR(8, local);
        if constexpr (PAIR) {
          if (leader) mbar_expect_tx(xfull, 2 * X_BYTES);
          for (int kb = 0; kb < 6; ++kb) tma_load_2d_2sm(sX + kb * X_ATOM, &tmX, lead(xfull), kb * 64, tile * BM);
        } else {
          mbar_expect_tx(xfull, X_BYTES);
          for (int kb = 0; kb < 6; ++kb) tma_load_2d(sX + kb * X_ATOM, &tmX, xfull, kb * 64, tile * BM);
        }
        if constexpr (HC == 128) w1(0);  // six 16 KB blocks: more than the ring holds
        w1(1);
        for (int c = 0; c < NCH; ++c) {
          // L2 prefetch of what the tile boundary waits on: this tile's residual rows and
          // the next tile's X (the X buffer is reloaded twice per tile, serially)
          if (SF_MLP_PF >= 0 && c == SF_MLP_PF)
            for (int kb = 0; kb < 6; ++kb) tma_prefetch_2d(&tmR, kb * 64, tile * BM);
          if (SF_MLP_PFX >= 0 && c == SF_MLP_PFX && tile + tstride < tiles)
            for (int kb = 0; kb < 6; ++kb) tma_prefetch_2d(&tmX, kb * 64, (tile + tstride) * BM);
          w2(c);
          if (c + 2 < NCH) w1(c + 2);
          if (c == NCH - 2) {  // all fc1 of this tile issued: residual rows replace X when it is consumed
            mbar_wait(xempty, local & 1);
            MTR(9, local);
            mbar_expect_tx(rfull, X_BYTES);
            for (int kb = 0; kb < 6; ++kb) tma_load_2d(sX + kb * X_ATOM, &tmR, rfull, kb * 64, tile * BM);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (the pair's leader)
    constexpr uint32_t idesc1 = idesc_bf16_f32(PAIR ? 256 : 128, HC);
    constexpr uint32_t idesc2 = idesc_bf16_f32(PAIR ? 256 : 128, HC == 128 ? 128 : 192);
    const uint32_t sX0 = smem_u32(sX), sW0 = smem_u32(sW), sH0 = smem_u32(sH);
    int ws = 0, g1 = 0, g2 = 0, local = 0;  // weight blocks consumed, fc1 chunks issued, fc2 chunks issued
    auto take = [&]() {
      const int s = ws % NSTAGE;
      if (lane == 0) MTR(6, ws);
      mbar_wait(&wfull[s], (ws / NSTAGE) & 1);
      if (lane == 0) MTR(7, ws);
      tc_fence_after();
      return s;
    };
    auto commit = [&](uint64_t* bar) {  // arrive on this barrier in every CTA of the cluster
      if constexpr (PAIR)
        mma_commit_2sm_mc(bar, CL_MASK);
      else if constexpr (CL > 1)
        mma_commit_mc(bar, CL_MASK);
      else
        mma_commit(bar);
    };
    auto mma = [&](uint32_t d, uint64_t ad, uint64_t bd, uint32_t idesc, bool acc) {
      if constexpr (PAIR)
        mma_bf16_ss_2sm(d, ad, bd, idesc, acc);
      else
        mma_bf16_ss(d, ad, bd, idesc, acc);
    };
    // leader-owned barriers with arrivals from both CTAs: cluster-scope acquire
    auto wait_pair = [&](uint64_t* bar, uint32_t parity) {
      if constexpr (PAIR)
        mbar_wait_cluster(bar, parity);
      else
        mbar_wait(bar, parity);
    };
    auto give = [&](int s) {
      if (elect_one()) {
        if constexpr (PAIR || CL > 1)
          commit(&wempty[s]);  // the slot is refilled in every CTA
        else
          mma_commit(&wempty[s]);
      }
      __syncwarp();
      ++ws;
    };
    for (int tile = tile0; tile < (PAIR && !leader ? tile0 : tiles); tile += tstride, ++local) {
      mbar_wait(xfull, local & 1);
      auto fc1 = [&](int c) {
        const int b = g1 % NB;
        if (lane == 0) MTR(0, g1);
        wait_pair(&a1empty[b], ((g1 / NB) & 1) ^ 1);  // GELU warps drained this buffer
        if (lane == 0) MTR(1, g1);
        if constexpr (HC == 128) {
          for (int kb = 0; kb < 6; ++kb) {
            const int s = take();
            if (elect_one()) {
              const uint64_t ad = sw128_kmajor_desc(sX0 + kb * X_ATOM);
              const uint64_t bd = sw128_kmajor_desc(sW0 + s * STAGE);
#pragma unroll
              for (int k = 0; k < 4; ++k) mma(tmem + ACC1, ad + 2 * k, bd + 2 * k, idesc1, (kb | k) != 0);
            }
            __syncwarp();
            give(s);
          }
        } else {
          for (int half = 0; half < 2; ++half) {
            const int s = take();
            if (elect_one()) {
#pragma unroll
              for (int a = 0; a < 3; ++a) {
                const int kb = 3 * half + a;
                const uint64_t ad = sw128_kmajor_desc(sX0 + kb * X_ATOM);
                const uint64_t bd = sw128_kmajor_desc(sW0 + s * STAGE + a * (HC / WSPLIT * 128));
#pragma unroll
                for (int k = 0; k < 4; ++k) mma(tmem + ACC1 + 64 * b, ad + 2 * k, bd + 2 * k, idesc1, (kb | k) != 0);
              }
            }
            __syncwarp();
            give(s);
          }
        }
        if (c == NCH - 1) {
          if (elect_one()) commit(xempty);  // X tile fully consumed
          __syncwarp();
        }
        if (elect_one()) commit(&a1full[b]);
        __syncwarp();
        ++g1;
      };
      auto fc2 = [&](int c) {
        const int b = g2 % NB;
        if (c == 0) wait_pair(a2empty, (local & 1) ^ 1);  // epilogue drained the previous tile
        if (lane == 0) MTR(2, g2);
        wait_pair(&hfull[b], (g2 / NB) & 1);
        if (lane == 0) MTR(3, g2);
        tc_fence_after();
        if constexpr (HC == 128) {
          for (int n = 0; n < 3; ++n)
            for (int a = 0; a < 2; ++a) {
              const int s = take();
              if (elect_one()) {
                const uint64_t ad = sw128_kmajor_desc(sH0 + a * X_ATOM);
                const uint64_t bd = sw128_kmajor_desc(sW0 + s * STAGE);
#pragma unroll
                for (int k = 0; k < 4; ++k) mma(tmem + ACC2 + 128 * n, ad + 2 * k, bd + 2 * k, idesc2, (c | a | k) != 0);
              }
              __syncwarp();
              give(s);
            }
        } else {
          for (int half = 0; half < 2; ++half) {
            const int s = take();
            if (elect_one()) {
              const uint64_t ad = sw128_kmajor_desc(sH0 + b * H_BYTES);
              const uint64_t bd = sw128_kmajor_desc(sW0 + s * STAGE);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma(tmem + ACC2 + 192 * half, ad + 2 * k, bd + 2 * k, idesc2, (c | k) != 0);
            }
            __syncwarp();
            give(s);
          }
        }
        if (elect_one()) {
          commit(&hempty[b]);
          if (c == NCH - 1) commit(a2full);
        }
        __syncwarp();
        ++g2;
      };
      fc1(0);
      fc1(1);
      for (int c = 0; c < NCH; ++c) {
        fc2(c);
        if (c + 2 < NCH) fc1(c + 2);
      }
    }
  } else {
    // ------------------------------------------------------------ worker warps 2..17
    // Warps 2..(1+GELU_WARPS) run the GELU of every hidden chunk; after a tile's last
    // chunk they join the dedicated epilogue warps, so all WORKERS warps share the
    // residual + LayerNorm epilogue (the MMA pipe waits on it at the tile boundary).
    const bool is_gelu = warp < 2 + GELU_WARPS;
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;
    const uint32_t gpart = (warp - 2) >> 2;  // GELU: which GCOLS columns of a chunk
    const uint32_t gaddr = tmem + ((quarter * 32) << 16) + ACC1 + gpart * GCOLS;
    const uint32_t e = warp - 2;              // epilogue: 0..WORKERS-1
    const uint32_t part = e >> 2;             // ECOLS-column slice of the row
    const int col0 = ECOLS * part;
    const uint32_t eaddr = tmem + ((quarter * 32) << 16) + ACC2 + col0;
    constexpr int NQ = ECOLS / 32;
    // 16-byte chunk j (8 columns) of this thread's row within 64-column atom a
    auto xp = [&](int col) -> uint4* {
      const int a = col >> 6, j = (col & 63) >> 3;
      return reinterpret_cast<uint4*>(sX + a * X_ATOM + row * 128 + ((j ^ (row & 7)) * 16));
    };
    // TMA-store the quarter's 32 rows of the X buffer (6 atoms; warp k of the quarter
    // issues atoms k, k + 4) once every warp of the quarter has written its columns
    auto store_quarter = [&](const CUtensorMap* m, int r0) {
      fence_proxy_async_smem();
      named_bar_sync(2 + quarter, 32 * PARTS);
      if (lane == 0) {
        for (int a = (int)part; a < 6; a += PARTS)
          tma_store_2d(m, sX + a * X_ATOM + quarter * 32 * 128, 64 * a, r0 + quarter * 32);
        bulk_commit();
        bulk_wait_read<0>();
      }
      __syncwarp();
      named_bar_sync(2 + quarter, 32 * PARTS);  // the stores have read the quarter's rows
    };
    int g = 0, local = 0;
    for (int tile = tile0; tile < tiles; tile += tstride, ++local) {
      if (is_gelu) {
        for (int c = 0; c < NCH; ++c, ++g) {
          const int b = g % NB;
          mbar_wait(&a1full[b], (g / NB) & 1);
          if (warp == 2 && lane == 0) MTR(4, g);
          tc_fence_after();
          // 32 columns at a time (register budget); the TMEM buffer is released after the last read
          const float* bb = sB1 + c * HC + gpart * GCOLS;
          uint32_t pk[GCOLS / 2];
#pragma unroll
          for (int h = 0; h < GCOLS / 32; ++h) {
            float v[32];
            tmem_ld32(gaddr + HC * b + 32 * h, v);
            tmem_ld_wait();
            if (h + 1 == GCOLS / 32) {
              tc_fence_before();
              if constexpr (PAIR)
                mbar_arrive_cluster(lead(&a1empty[b]));
              else
                mbar_arrive(&a1empty[b]);
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 bv = reinterpret_cast<const float2*>(bb + 32 * h)[i];
              float2 y = __fadd2_rn(make_float2(v[2 * i], v[2 * i + 1]), bv);
              y = gelu_tanh2(y);
              pk[16 * h + i] = pack_bf16(y.x, y.y);
            }
          }
          mbar_wait(&hempty[b], ((g / NB) & 1) ^ 1);  // fc2 has read this buffer
          // this thread's GCOLS columns: 16-byte chunks of its row in the 64-column H atom(s)
          uint8_t* hrow = sH + b * H_BYTES + row * 128;
#pragma unroll
          for (int j = 0; j < GCOLS / 8; ++j) {
            const int col = gpart * GCOLS + 8 * j;
            const int at = col >> 6, cj = (col & 63) >> 3;
            *reinterpret_cast<uint4*>(hrow + at * X_ATOM + ((cj ^ (row & 7)) * 16)) =
                make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          }
          fence_proxy_async_smem();
          if constexpr (PAIR)
            mbar_arrive_cluster(lead(&hfull[b]));  // the leader's pair MMA reads this CTA's H
          else
            mbar_arrive(&hfull[b]);
          if (warp == 2 && lane == 0) MTR(5, g);
        }
      }
      // ---------------- residual + LayerNorm epilogue of this tile (all workers)
      // The tile's residual rows arrive by TMA in the X buffer (free once fc1 is done);
      // the updated residual and then the modulated LayerNorm output are written back in
      // place and leave by TMA stores, so global traffic is bulk, not per thread.
      const int r0 = tile * BM;
      const int64_t slot = r0 / p.T;
      named_bar_sync(1, WORKERS * 32);  // previous tile's readers are done with sVec
      for (int i = e * 32 + lane; i < D; i += WORKERS * 32) {
        const int64_t o = slot * p.vec_stride + i;
        sVec[i] = p.b2[i];
        sVec[D + i] = p.gate[o];
        sVec[2 * D + i] = p.shift[o];
        sVec[3 * D + i] = p.scale[o];
      }
      named_bar_sync(1, WORKERS * 32);
      mbar_wait(a2full, local & 1);
      if (e == 0 && lane == 0) MTR(10, local);
      mbar_wait(rfull, local & 1);
      if (e == 0 && lane == 0) MTR(11, local);
      tc_fence_after();
      float sum = 0.f, sq = 0.f;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        float v[32];
        tmem_ld32(eaddr + 32 * q, v);
        tmem_ld_wait();
        if (q + 1 == NQ) {
          tc_fence_before();
          if constexpr (PAIR)
            mbar_arrive_cluster(lead(a2empty));  // accumulator drained: the next tile's fc2 may start
          else
            mbar_arrive(a2empty);
        }
        const float* vb = sVec + col0 + 32 * q;
        const float* vg = sVec + D + col0 + 32 * q;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4* ptr = xp(col0 + 32 * q + 8 * j);
          const uint4 ov = *ptr;
          const uint32_t ow[4] = {ov.x, ov.y, ov.z, ov.w};
          uint32_t nw[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = 8 * j + 2 * i;
            const float2 o = unpack_bf16(ow[i]);
            nw[i] = pack_bf16(o.x + vg[c] * (v[c] + vb[c]), o.y + vg[c + 1] * (v[c + 1] + vb[c + 1]));
            const float2 n = unpack_bf16(nw[i]);
            sum += n.x + n.y;
            sq += n.x * n.x + n.y * n.y;
          }
          *ptr = make_uint4(nw[0], nw[1], nw[2], nw[3]);
        }
      }
      // row statistics over the column parts of this lane quarter
      sRed[(0 * PARTS + part) * BM + row] = sum;
      sRed[(1 * PARTS + part) * BM + row] = sq;
      store_quarter(&tmRs, r0);  // updated residual out (its barriers also publish sRed)
      float tsum = 0.f, tsq = 0.f;
#pragma unroll
      for (int k = 0; k < PARTS; ++k) {
        tsum += sRed[k * BM + row];
        tsq += sRed[(PARTS + k) * BM + row];
      }
      const float mean = tsum * (1.0f / D);
      const float var = fmaxf(tsq * (1.0f / D) - mean * mean, 0.f);
      const float rstd = rsqrtf(var + p.ln_eps);
      if (e == 0 && lane == 0) MTR(12, local);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float* vsh = sVec + 2 * D + col0 + 32 * q;
        const float* vsc = sVec + 3 * D + col0 + 32 * q;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4* ptr = xp(col0 + 32 * q + 8 * j);
          const uint4 xv = *ptr;
          const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
          uint32_t o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = 8 * j + 2 * i;
            const float2 x = unpack_bf16(xw[i]);
            o[i] = pack_bf16((x.x - mean) * rstd * (1.0f + vsc[c]) + vsh[c],
                             (x.y - mean) * rstd * (1.0f + vsc[c + 1]) + vsh[c + 1]);
          }
          *ptr = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      store_quarter(&tmMs, r0);  // modulated LayerNorm out; the X buffer is then free
      if (e == 0 && lane == 0) MTR(13, local);
      mbar_arrive(xfree);
    }
  }
  tc_fence_before();
  __syncthreads();
  if constexpr (CL > 1) cluster_sync_all();  // peers still multicast into / arrive on this CTA until done
  if (warp == 1) {
    if constexpr (PAIR)
      tmem_dealloc_2sm<512>(tmem);
    else
      tmem_dealloc<512>(tmem);
  }
}

}  // namespace mlp

// X = xmod [M, 384], W1 [1536, 384], W2 [384, 1536] (all bf16, K-major).
int launch_mlp_fused(const void* xmod_in, const void* w1, const void* w2, const float* b1, const float* b2,
                     __nv_bfloat16* xres, __nv_bfloat16* xmod_out, const float* gate, const float* shift,
                     const float* scale, int64_t vec_stride, float ln_eps, int64_t M, int T, cudaStream_t st) {
  using namespace mlp;
  if (M % BM || T % BM) return SF_ERR_PARAMETER;
  static bool attr = false;
  if (!attr) {
    const cudaError_t err = cudaFuncSetAttribute(mlp_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (err != cudaSuccess) {
      fprintf(stderr, "streamflow: mlp_fused smem attribute: %s\n", cudaGetErrorString(err));
      return SF_ERR_CUDA;
    }
    attr = true;
  }
  CUtensorMap tx, t1, t2, tr, trs, tms;
  int rc = make_tmap_bf16_2d(&tx, xmod_in, D, (uint64_t)M, D, 64, BM, 128);
  rc |= make_tmap_bf16_2d(&tr, xres, D, (uint64_t)M, D, 64, BM, 128);
  rc |= make_tmap_bf16_2d(&trs, xres, D, (uint64_t)M, D, 64, 32, 128);
  rc |= make_tmap_bf16_2d(&tms, xmod_out, D, (uint64_t)M, D, 64, 32, 128);
  rc |= make_tmap_bf16_2d(&t1, w1, D, FF, D, 64, HC / CL, 128);  // CL = 2: each CTA loads half the rows
  rc |= make_tmap_bf16_2d(&t2, w2, FF, D, FF, 64, (HC == 128 ? 128 : 192) / CL, 128);
  if (rc != SF_OK) return SF_ERR_CUDA;
  Params p{b1, b2, xres, xmod_out, gate, shift, scale, vec_stride, ln_eps, T, (int)M};
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = (int)(M / BM);
  if (tiles % CL) return SF_ERR_PARAMETER;
  const int grid = (tiles < sms ? tiles : sms) / CL * CL;
  if (CL == 1) {
    mlp_fused_kernel<<<grid, THREADS, SMEM, st>>>(tx, t1, t2, tr, trs, tms, p);
    return cuda_status();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)grid);
  cfg.blockDim = dim3(THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = CL;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  const cudaError_t err = cudaLaunchKernelEx(&cfg, mlp_fused_kernel, tx, t1, t2, tr, trs, tms, p);
  if (err != cudaSuccess) {
    fprintf(stderr, "streamflow: mlp_fused launch failed: %s\n", cudaGetErrorString(err));
    return SF_ERR_CUDA;
  }
  return SF_OK;
}

}  // namespace sf

#if SF_MLP_TRACE
extern "C" int sf_mlp_trace_read(long long* dst) {
  return cudaMemcpyFromSymbol(dst, sf::mlp::g_mlp_trace, sizeof(long long) * 16 * 64) == cudaSuccess ? 0 : -1;
}
#endif

extern "C" int sf_mlp_fused(const void* xmod_in, const void* w1, const void* w2, const float* b1, const float* b2,
                            void* xres, void* xmod_out, const float* gate, const float* shift, const float* scale,
                            int64_t vec_stride, float ln_eps, int64_t M, int32_t T, void* stream) {
  if (!xmod_in || !w1 || !w2 || !b1 || !b2 || !xres || !xmod_out || !gate || !shift || !scale || M < 1 || T < 1)
    return SF_ERR_PARAMETER;
  return sf::launch_mlp_fused(xmod_in, w1, w2, b1, b2, (__nv_bfloat16*)xres, (__nv_bfloat16*)xmod_out, gate, shift,
                              scale, vec_stride, ln_eps, M, T, (cudaStream_t)stream);
}

// Post-attention half of a DiT-S/2 block in one persistent kernel on CTA PAIRS (cta_group::2):
//   x   = xres + gate_msa * (attn . Wproj^T + b_proj)                   (-> xres)
//   h   = LN(x) * (1 + scale_mlp) + shift_mlp                            (stays in smem)
//   x'  = x + gate_mlp * (GELU(h . W1^T + b1) . W2^T + b2)               (-> xres)
//   out = LN(x') * (1 + scale_next) + shift_next                         (-> xmod)
//
// The MLP's input h never goes to HBM (the projection epilogue leaves it in smem as the fc1 A
// operand) and the 128 x 1536 GELU'd hidden of a row tile lives only in TMEM / smem, chunk by
// chunk.  Two CTAs of a cluster run one M=256 MMA over their two 128-row tiles: each CTA stages
// only HALF of every weight block (the B operand is split between the pair), so per 128 rows
// the layer's 2.6 MB of weights cost 1.3 MB of L2->smem traffic; proj and fc2 run as two N=192
// halves.  (Round 1 ran one CTA per 128-row tile: 5.48 vs 4.34 ms per step, profiles/r02.)
// Cross-CTA handshakes use one arrival per warp with cta-scope mbarrier semantics (release /
// acquire at cluster scope cost ~1.5k cycles per handoff: 388 vs 300 us standalone).
//
// Roles (each CTA: 18 warps): warp 0 TMA producer (own rows + own half of every weight block;
// pair-operand loads complete on the LEADER's barriers), warp 1 MMA issuer (leader CTA only;
// its commits multicast to both CTAs), warps 2..17 workers exactly as in block_tail.cu
// (all 16 run both LayerNorm epilogues and the GELU of every hidden chunk).  Barriers that gate a
// pair MMA on both CTAs' workers (xready, a1empty, hfull, a2empty) live in the leader and
// take one release.cluster arrival per worker warp.  TMEM per CTA: ACC2 = 384 columns (two
// N=192 halves, output column c at column c), ACC1 = 128 (one hidden chunk).
#include <cstdint>
#include <cstdio>

#include "gemm_tcgen05.cuh"
#include "sf_internal.h"
#include "sf_ptx.cuh"

#ifndef SF_TAIL2_TRACE
#define SF_TAIL2_TRACE 0  // diagnostics: clock64 timeline of cluster 0 (tools/tail_trace.py)
#endif

namespace sf {
namespace tail2 {

constexpr int D = 384, FF = 1536, BM = 128, HC = 128, NCH = FF / HC;  // 12 hidden chunks
constexpr int X_ATOM = BM * 64 * 2;  // 16 KB: 128 rows x 64 K (SW128)
constexpr int X_BYTES = 6 * X_ATOM;  // 96 KB
constexpr int NH = 192;              // pair-MMA N of proj / fc2 (two halves of the 384 outputs)
constexpr int BROWS = NH / 2;        // 96 B rows per CTA for proj / fc2 blocks
constexpr int W1ROWS = HC / 2;       // 64 B rows per CTA for fc1 blocks
constexpr int STAGE = BROWS * 128;   // 12 KB (fc1 blocks use 8 KB of it)
constexpr int NSTAGE = 6;
constexpr int H_BYTES = BM * HC * 2;  // 32 KB (two 64-column atoms)
constexpr int WORKERS = 16;                   // epilogue + GELU warps
constexpr int PARTS = WORKERS / 4;            // worker warps per TMEM lane quarter
constexpr int ECOLS = D / PARTS;              // 96 output columns per worker thread
constexpr int GCOLS = HC / PARTS;             // 32 hidden columns per worker thread
constexpr int THREADS = 32 * (2 + WORKERS);
constexpr int ACC2 = 0, ACC1 = 384;
constexpr uint16_t PAIR_MASK = 0x3;
constexpr int SMEM = 1024 + X_BYTES + NSTAGE * STAGE + H_BYTES + 2 * 4 * D * 4 + 2 * 4 * BM * 4 + FF * 4 + 512;
static_assert(SMEM <= 232448, "shared memory");

struct Params {
  __nv_bfloat16* xres;  // residual stream [M, 384] (read by TMA, written by the epilogues)
  __nv_bfloat16* xmod;  // LN_next output [M, 384]
  const float* bp;  // b_proj [384]
  const float* b1;  // [1536]
  const float* b2;  // [384]
  const float* g1;  // gate_msa  (per-slot vectors: ptr + slot * vec_stride)
  const float* sh1;  // shift_mlp
  const float* sc1;  // scale_mlp
  const float* g2;  // gate_mlp
  const float* sh2;  // shift of the next LayerNorm
  const float* sc2;  // scale of the next LayerNorm
  int64_t vec_stride;
  float ln_eps;
  int T;
  int M;
  int pdl;  // launched with programmatic serialisation (sf_internal.h g_pdl)
};

#if SF_TAIL2_TRACE
__device__ long long g_trace[16 * 128];
#define TTR(role, idx) \
  if (blockIdx.x < 2 && (idx) < 128) g_trace[((role) + 8 * (blockIdx.x & 1)) * 128 + (idx)] = clock64()
#else
#define TTR(role, idx)
#endif

// acquire.cluster wait on a barrier of this CTA that receives remote arrivals (bounded: a
// protocol bug traps instead of hanging the GPU)
__device__ __forceinline__ void wait_cl(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  for (uint32_t n = 0;; ++n) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n\t}\n"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    if (n > (1u << 26)) {
      printf("streamflow: pair mbarrier wait timeout (block %d thread %d, smem 0x%x)\n", (int)blockIdx.x,
             (int)threadIdx.x, addr);
      asm volatile("trap;");
    }
  }
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    block_tail_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmWp,
                           const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmW2,
                           const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmRs,
                           const __grid_constant__ CUtensorMap tmMs, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;
  uint8_t* sW = sX + X_BYTES;
  uint8_t* sH = sW + NSTAGE * STAGE;
  // per-column vectors of the two epilogues, [4][384] each (bias | gate | shift | scale): the
  // projection epilogue's (sVecP) and the final epilogue's (sVecF), filled during the MLP phase of
  // the tile before / the same tile so neither epilogue starts with global loads
  float* sVecP = reinterpret_cast<float*>(sH + H_BYTES);
  float* sVecF = sVecP + 4 * D;
  float* sRed = sVecF + 4 * D;                           // [2 stats][PARTS][128 rows]
  float* sB1 = sRed + 2 * 4 * BM;                        // fc1 bias [1536]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sB1 + FF);
  uint64_t* wfull = bars;               // [NSTAGE] (leader) both halves of a weight block landed
  uint64_t* wempty = wfull + NSTAGE;    // [NSTAGE] pair MMAs done with the slot (multicast)
  uint64_t* hafull = wempty + NSTAGE;   // [2] (leader) attention K-atom landed in an H slot, both CTAs
  uint64_t* haempty = hafull + 2;       // [2] projection MMAs done with the slot (multicast)
  uint64_t* pfull = haempty + 2;        // projection accumulator ready (multicast)
  uint64_t* r1full = pfull + 1;         // residual rows landed in X (local)
  uint64_t* xready = r1full + 1;        // (leader) both CTAs: X holds h, ACC2 drained
  uint64_t* xempty = xready + 1;        // fc1 done reading X (multicast)
  uint64_t* a1full = xempty + 1;        // fc1 chunk accumulator ready (multicast)
  uint64_t* a1empty = a1full + 1;       // (leader) both CTAs' GELU warps have read it
  uint64_t* hfull = a1empty + 1;        // (leader) both CTAs' H written
  uint64_t* hempty = hfull + 1;         // fc2 has read H (multicast)
  uint64_t* a2full = hempty + 1;        // fc2 accumulator ready (multicast)
  uint64_t* a2empty = a2full + 1;       // (leader) both CTAs' final epilogue drained ACC2
  uint64_t* r2full = a2empty + 1;       // x rows landed in X (local)
  uint64_t* xfree = r2full + 1;         // final epilogue done with X (local)
  uint64_t* stored = xfree + 1;         // projection epilogue's x stores landed (local)
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(stored + 1);

  const uint32_t warp = warp_id(), lane = threadIdx.x & 31;
  const uint32_t crank = cluster_ctarank();
  const bool leader = crank == 0;
  const int pairs = p.M / (2 * BM);
  const int pair0 = blockIdx.x >> 1, pstride = gridDim.x >> 1;
  auto lead = [&](uint64_t* bar) -> uint32_t { return mapa_shared(smem_u32(bar), 0); };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmWp);
    tma_prefetch(&tmW1);
    tma_prefetch(&tmW2);
    tma_prefetch(&tmR);
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&hafull[i], 1);
      mbar_init(&haempty[i], 1);
    }
    for (uint64_t* b : {pfull, r1full, xempty, a1full, hempty, a2full, r2full}) mbar_init(b, 1);
    mbar_init(xready, 2 * WORKERS);      // one arrival per worker warp of both CTAs
    mbar_init(a2empty, 2 * WORKERS);
    mbar_init(a1empty, 2 * WORKERS);
    mbar_init(hfull, 2 * WORKERS);
    mbar_init(xfree, WORKERS);           // local, one arrival per worker warp
    mbar_init(stored, WORKERS);
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < FF; i += THREADS) sB1[i] = p.b1[i];
  if (warp == 1) tmem_alloc_2sm<512>(tmem_holder);
  cluster_sync_all();  // the peer's barriers exist before any remote arrive / complete_tx
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;
  if (threadIdx.x == 0) pdl_trigger(p.pdl);  // the next kernel's CTAs may start their prologue
  pdl_wait(p.pdl);                           // the attention output / residual stream are complete

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer (both CTAs)
    if (elect_one()) {
      int ws = 0;
      // this CTA's half (rows [c1, c1 + rows)) of one weight block; both halves complete on
      // the leader's full barrier, which expects the whole block
      auto wblock = [&](const CUtensorMap* m, int c0, int c1, int bytes) {
        const int s = ws % NSTAGE;
        mbar_wait(&wempty[s], ((ws / NSTAGE) & 1) ^ 1);
        if (leader) mbar_expect_tx(&wfull[s], 2 * bytes);
        tma_load_2d_2sm(sW + s * STAGE, m, lead(&wfull[s]), c0, c1);
        ++ws;
      };
      auto xload = [&](uint64_t* bar, int r0) {  // local: own rows into X for own workers
        mbar_expect_tx(bar, X_BYTES);
        for (int kb = 0; kb < 6; ++kb) tma_load_2d(sX + kb * X_ATOM, &tmR, bar, kb * 64, r0);
      };
      auto w1 = [&](int c) {
        for (int kb = 0; kb < 6; ++kb) wblock(&tmW1, kb * 64, c * HC + W1ROWS * crank, W1ROWS * 128);
      };
      auto w2 = [&](int c) {
        for (int a = 0; a < 2; ++a)
          for (int nh = 0; nh < 2; ++nh) wblock(&tmW2, c * HC + 64 * a, NH * nh + BROWS * crank, STAGE);
      };
      int local = 0;
      for (int pr = pair0; pr < pairs; pr += pstride, ++local) {
        const int r0 = (2 * pr + (int)crank) * BM;
        // projection operands: attention K-atoms through the two H slots (idle between the previous
        // tile's last fc2 and this tile's first GELU), so the projection overlaps the previous
        // tile's final epilogue, which still owns X
        // (a2full = after the previous tile's last fc2; a per-tile barrier, so the parity wait
        // cannot alias the way a per-chunk hempty phase could with a 6-deep weight ring)
        if (local > 0) mbar_wait(a2full, (local - 1) & 1);
        for (int kb = 0; kb < 6; ++kb) {
          const int u = local * 6 + kb, slot = kb & 1;
          mbar_wait(&haempty[slot], ((u >> 1) & 1) ^ 1);
          if (leader) mbar_expect_tx(&hafull[slot], 2 * X_ATOM);
          tma_load_2d_2sm(sH + slot * X_ATOM, &tmA, lead(&hafull[slot]), kb * 64, r0);
          for (int nh = 0; nh < 2; ++nh) wblock(&tmWp, kb * 64, NH * nh + BROWS * crank, STAGE);
        }
        mbar_wait(xfree, (local & 1) ^ 1);  // previous tile's final epilogue left X
        xload(r1full, r0);
        w1(0);
        w1(1);
        for (int c = 0; c < NCH; ++c) {
          w2(c);
          if (c + 2 < NCH) w1(c + 2);
          if (c == NCH - 2) {  // all fc1 issued: the updated rows replace h once fc1 is done
            mbar_wait(xempty, local & 1);
            mbar_wait(stored, local & 1);  // ... and once the projection epilogue's stores landed
            xload(r2full, r0);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer (leader CTA)
    if (leader) {
      constexpr uint32_t idesc_n192 = idesc_bf16_f32(256, NH);
      constexpr uint32_t idesc_n128 = idesc_bf16_f32(256, HC);
      const uint32_t sX0 = smem_u32(sX), sW0 = smem_u32(sW), sH0 = smem_u32(sH);
      int ws = 0, g = 0, local = 0;
#if SF_TAIL2_TRACE
      long long tw_full = 0, tw_a1e = 0, tw_hfull = 0;
#define TACC(var, stmt)            \
  {                                \
    const long long _t = clock64(); \
    stmt;                          \
    var += clock64() - _t;         \
  }
#else
#define TACC(var, stmt) stmt;
#endif
      auto take = [&]() {
        const int s = ws % NSTAGE;
        TACC(tw_full, wait_cl(&wfull[s], (ws / NSTAGE) & 1));
        tc_fence_after();
        return s;
      };
      auto commit = [&](uint64_t* bar) {  // arrive on this barrier in both CTAs when the MMAs complete
        if (elect_one()) mma_commit_2sm_mc(bar, PAIR_MASK);
        __syncwarp();
      };
      auto give = [&](int s) {
        commit(&wempty[s]);
        ++ws;
      };
      auto mma4 = [&](uint32_t d, uint32_t a_addr, uint32_t b_addr, uint32_t idesc, bool first) {
        if (elect_one()) {
          const uint64_t ad = sw128_kmajor_desc(a_addr), bd = sw128_kmajor_desc(b_addr);
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_bf16_ss_2sm(d, ad + 2 * k, bd + 2 * k, idesc, !(first && k == 0));
        }
        __syncwarp();
      };
      for (int pr = pair0; pr < pairs; pr += pstride, ++local) {
        // projection: acc2[:, 192 nh : +192] = attn . Wproj[192 nh : +192]^T (M = 256 over the pair)
        TTR(0, 4 * local);
        wait_cl(a2empty, (local & 1) ^ 1);  // both CTAs' final epilogues drained the accumulator
        TTR(0, 4 * local + 1);
        for (int kb = 0; kb < 6; ++kb) {
          const int u = local * 6 + kb, slot = kb & 1;
          wait_cl(&hafull[slot], (u >> 1) & 1);
          tc_fence_after();
          for (int nh = 0; nh < 2; ++nh) {
            const int s = take();
            mma4(tmem + ACC2 + NH * nh, sH0 + slot * X_ATOM, sW0 + s * STAGE, idesc_n192, kb == 0);
            give(s);
          }
          commit(&haempty[slot]);
        }
        commit(pfull);
        wait_cl(xready, local & 1);  // both CTAs: X holds h, the projection accumulator is drained
        TTR(0, 4 * local + 2);
        tc_fence_after();
        // g + c: global index of hidden chunk c (fc1, GELU and fc2 of a chunk share it)
        auto fc1 = [&](int c) {
          TTR(3, (g + c) & 127);
          TACC(tw_a1e, wait_cl(a1empty, ((g + c) & 1) ^ 1));  // both CTAs' GELU warps read the previous chunk
          TTR(4, (g + c) & 127);
          tc_fence_after();
          for (int kb = 0; kb < 6; ++kb) {
            const int s = take();
            mma4(tmem + ACC1, sX0 + kb * X_ATOM, sW0 + s * STAGE, idesc_n128, kb == 0);
            give(s);
          }
          if (c == NCH - 1) commit(xempty);
          commit(a1full);
        };
        auto fc2 = [&](int c) {
          TTR(5, (g + c) & 127);
          TACC(tw_hfull, wait_cl(hfull, (g + c) & 1));
          TTR(6, (g + c) & 127);
          tc_fence_after();
          for (int a = 0; a < 2; ++a)
            for (int nh = 0; nh < 2; ++nh) {
              const int s = take();
              mma4(tmem + ACC2 + NH * nh, sH0 + a * X_ATOM, sW0 + s * STAGE, idesc_n192, c == 0 && a == 0);
              give(s);
            }
          commit(hempty);
          if (c == NCH - 1) commit(a2full);
        };
        fc1(0);
        fc1(1);
        for (int c = 0; c < NCH; ++c) {
          fc2(c);
          if (c + 2 < NCH) fc1(c + 2);
        }
        TTR(0, 4 * local + 3);
#if SF_TAIL2_TRACE
        if (blockIdx.x == 0 && local < 16) {  // cumulative wait cycles of the MMA warp
          g_trace[0 * 128 + 64 + 4 * local] = tw_full;
          g_trace[0 * 128 + 64 + 4 * local + 1] = tw_a1e;
          g_trace[0 * 128 + 64 + 4 * local + 2] = tw_hfull;
        }
#endif
        g += NCH;
      }
    }
  } else {
    // ------------------------------------------------------------ worker warps 2..17 (both CTAs)
    // Every worker warp runs both LayerNorm epilogues (96 output columns per thread) and the
    // GELU of every hidden chunk (32 hidden columns per thread): the GELU of chunk c is on the
    // MMA pipe's critical path (fc2(c) waits for it, fc1(c+1) for its TMEM read).
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;
    const uint32_t e = warp - 2, part = e >> 2;
    const uint32_t lane_base = tmem + ((quarter * 32) << 16);
    const uint32_t gaddr = lane_base + ACC1 + part * GCOLS;
    const int col0 = ECOLS * part;
    const uint32_t eaddr = lane_base + ACC2 + col0;
    constexpr int NQ = ECOLS / 32;
    // one release.cluster arrival per warp on the leader's barrier (covers the whole warp's
    // prior writes / TMEM reads via __syncwarp)
    auto arrive_lead = [&](uint64_t* bar) {
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(lead(bar)) : "memory");
      __syncwarp();
    };
    auto arrive_local = [&](uint64_t* bar) {
      __syncwarp();
      if (lane == 0) mbar_arrive(bar);
      __syncwarp();
    };
    auto xp = [&](int col) -> uint4* {
      const int a = col >> 6, j = (col & 63) >> 3;
      return reinterpret_cast<uint4*>(sX + a * X_ATOM + row * 128 + ((j ^ (row & 7)) * 16));
    };
    // TMA store of the quarter's 32 rows of X (one 32 x 64 box per atom, issued by the quarter's
    // warps in turn); returns once the stores have read X, so X may be overwritten
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
    // per-column vectors of one epilogue, pre-combined: [gate * bias | gate | shift | 1 + scale]
    // (called where every worker is past the previous readers of sVec: between two GELU chunks)
    auto load_vecs = [&](float* sVec, const float* bias, const float* gate, const float* shift, const float* scale,
                         int64_t slot) {
      named_bar_sync(1, WORKERS * 32);  // the previous readers are done with sVec
      for (int i = e * 32 + lane; i < D; i += WORKERS * 32) {
        const int64_t o = slot * p.vec_stride + i;
        const float gt = gate[o];
        sVec[i] = gt * bias[i];
        sVec[D + i] = gt;
        sVec[2 * D + i] = shift[o];
        sVec[3 * D + i] = 1.0f + scale[o];
      }
      named_bar_sync(1, WORKERS * 32);
    };
    auto f2 = [](float a, float b) { return make_float2(a, b); };
    // x = xres + gate * acc + gate * bias in place in X (packed f32x2 math) + TMA store of x +
    // row statistics of the stored bf16 values; then LN(x) * (1 + scale) + shift in place.
    // `done_acc` runs after the last TMEM read.
    int ep_mark = 0;  // trace slot base of this epilogue (diagnostics build only)
    auto mark = [&](int k) {
#if SF_TAIL2_TRACE
      if (e == 0 && lane == 0 && ep_mark + k < 64) g_trace[(8 * (blockIdx.x & 1) + 1) * 128 + 32 + ep_mark + k] = clock64();
#endif
    };
    auto res_ln = [&](const float* sVec, int r0, uint64_t* acc_full, uint32_t acc_ph, uint64_t* rows_full,
                      uint32_t rows_ph, auto done_acc) {
      mbar_wait(acc_full, acc_ph);
      mark(0);
      mbar_wait(rows_full, rows_ph);
      mark(1);
      tc_fence_after();
      float2 sum2 = f2(0.f, 0.f), sq2 = f2(0.f, 0.f);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        float v[32];
        tmem_ld32(eaddr + 32 * q, v);
        tmem_ld_wait();
        if (q + 1 == NQ) {
          tc_fence_before();
          done_acc();
        }
        const float4* va = reinterpret_cast<const float4*>(sVec + col0 + 32 * q);
        const float4* vg = reinterpret_cast<const float4*>(sVec + D + col0 + 32 * q);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4* ptr = xp(col0 + 32 * q + 8 * j);
          const uint4 ov = *ptr;
          const uint32_t ow[4] = {ov.x, ov.y, ov.z, ov.w};
          const float4 a0 = va[2 * j], a1 = va[2 * j + 1], g0 = vg[2 * j], g1 = vg[2 * j + 1];
          const float2 A[4] = {f2(a0.x, a0.y), f2(a0.z, a0.w), f2(a1.x, a1.y), f2(a1.z, a1.w)};
          const float2 G[4] = {f2(g0.x, g0.y), f2(g0.z, g0.w), f2(g1.x, g1.y), f2(g1.z, g1.w)};
          uint32_t nw[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const int c = 8 * j + 2 * i;
            const float2 n = __ffma2_rn(G[i], f2(v[c], v[c + 1]), __fadd2_rn(unpack_bf16(ow[i]), A[i]));
            nw[i] = pack_bf16(n.x, n.y);
            const float2 nr = unpack_bf16(nw[i]);
            sum2 = __fadd2_rn(sum2, nr);
            sq2 = __ffma2_rn(nr, nr, sq2);
          }
          *ptr = make_uint4(nw[0], nw[1], nw[2], nw[3]);
        }
      }
      sRed[(0 * PARTS + part) * BM + row] = sum2.x + sum2.y;
      sRed[(1 * PARTS + part) * BM + row] = sq2.x + sq2.y;
      mark(2);
      store_quarter(&tmRs, r0);  // x out (its barriers also publish sRed)
      mark(3);
      float tsum = 0.f, tsq = 0.f;
#pragma unroll
      for (int k = 0; k < PARTS; ++k) {
        tsum += sRed[k * BM + row];
        tsq += sRed[(PARTS + k) * BM + row];
      }
      const float mean = tsum * (1.0f / D);
      const float var = fmaxf(tsq * (1.0f / D) - mean * mean, 0.f);
      const float rstd = rsqrtf(var + p.ln_eps);
      const float2 r2 = f2(rstd, rstd), c2 = f2(-mean * rstd, -mean * rstd);
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float4* vsh = reinterpret_cast<const float4*>(sVec + 2 * D + col0 + 32 * q);
        const float4* vsc = reinterpret_cast<const float4*>(sVec + 3 * D + col0 + 32 * q);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint4* ptr = xp(col0 + 32 * q + 8 * j);
          const uint4 xv = *ptr;
          const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w};
          const float4 h0 = vsh[2 * j], h1 = vsh[2 * j + 1], s0 = vsc[2 * j], s1 = vsc[2 * j + 1];
          const float2 SH[4] = {f2(h0.x, h0.y), f2(h0.z, h0.w), f2(h1.x, h1.y), f2(h1.z, h1.w)};
          const float2 SC[4] = {f2(s0.x, s0.y), f2(s0.z, s0.w), f2(s1.x, s1.y), f2(s1.z, s1.w)};
          uint32_t o[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 y = __ffma2_rn(__ffma2_rn(unpack_bf16(xw[i]), r2, c2), SC[i], SH[i]);
            o[i] = pack_bf16(y.x, y.y);
          }
          *ptr = make_uint4(o[0], o[1], o[2], o[3]);
        }
      }
      mark(4);
    };
    int g = 0, local = 0;
    if (pair0 < pairs) load_vecs(sVecP, p.bp, p.g1, p.sh1, p.sc1, (2 * pair0 + (int)crank) * BM / p.T);
    for (int pr = pair0; pr < pairs; pr += pstride, ++local) {
      const int r0 = (2 * pr + (int)crank) * BM;
      const int64_t slot = r0 / p.T;
      // ---- projection epilogue: x = xres + gate_msa * (acc + b_proj) -> xres; X <- LN_mlp(x)
      if (e == 0 && lane == 0) TTR(1, 4 * local);
      ep_mark = 16 * local;
      res_ln(sVecP, r0, pfull, local & 1, r1full, local & 1, [] {});
      fence_proxy_async_smem();  // h is read by the fc1 MMAs (async proxy)
      arrive_lead(xready);       // (all TMEM reads of the projection accumulator precede this)
      if (e == 0 && lane == 0) TTR(1, 4 * local + 1);
      if (lane == 0) bulk_wait<0>();  // this warp's x stores have landed (the final epilogue reloads x)
      arrive_local(stored);
      // ---- MLP: GELU of every hidden chunk (ACC1 fp32 -> bf16 H in smem, the fc2 A operand)
      for (int c = 0; c < NCH; ++c, ++g) {
        mbar_wait(a1full, g & 1);
        tc_fence_after();
        if (e == 0 && lane == 0) TTR(2, g & 127);
        float v[32];
        tmem_ld32(gaddr, v);
        tmem_ld_wait();
#if SF_TAIL2_TRACE
        if (e == 0 && lane == 0 && g < 32) g_trace[(8 * (blockIdx.x & 1) + 1) * 128 + 64 + g] = clock64();
#endif
        tc_fence_before();
        arrive_lead(a1empty);
#if SF_TAIL2_TRACE
        if (e == 0 && lane == 0 && g < 32) g_trace[(8 * (blockIdx.x & 1) + 1) * 128 + 96 + g] = clock64();
#endif
        const float4* bb = reinterpret_cast<const float4*>(sB1 + c * HC + part * GCOLS);
        uint32_t pk[GCOLS / 2];
#pragma unroll
        for (int i = 0; i < GCOLS / 4; ++i) {
          const float4 bv = bb[i];
          const float2 y0 = gelu_tanh2(__fadd2_rn(f2(v[4 * i], v[4 * i + 1]), f2(bv.x, bv.y)));
          const float2 y1 = gelu_tanh2(__fadd2_rn(f2(v[4 * i + 2], v[4 * i + 3]), f2(bv.z, bv.w)));
          pk[2 * i] = pack_bf16(y0.x, y0.y);
          pk[2 * i + 1] = pack_bf16(y1.x, y1.y);
        }
        if (e == 0 && lane == 0) TTR(7, g & 127);
        mbar_wait(hempty, (g & 1) ^ 1);  // fc2 has read H
        uint8_t* hrow = sH + row * 128 + (part >> 1) * X_ATOM;
#pragma unroll
        for (int j = 0; j < GCOLS / 8; ++j) {
          const int cj = (int)(part & 1) * 4 + j;
          *reinterpret_cast<uint4*>(hrow + ((cj ^ (row & 7)) * 16)) =
              make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
        }
        fence_proxy_async_smem();
        arrive_lead(hfull);
        // the two epilogues' vectors, between GELU chunks (off the epilogues' critical path)
        if (c == 1) load_vecs(sVecF, p.b2, p.g2, p.sh2, p.sc2, slot);
        if (c == 6 && pr + pstride < pairs)
          load_vecs(sVecP, p.bp, p.g1, p.sh1, p.sc1, (2 * (pr + pstride) + (int)crank) * BM / p.T);
      }
      // ---- final epilogue: x' = x + gate_mlp * (acc + b2) -> xres; LN_next(x') -> xmod
      if (e == 0 && lane == 0) TTR(1, 4 * local + 2);
      ep_mark = 16 * local + 8;
      res_ln(sVecF, r0, a2full, local & 1, r2full, local & 1, [&] { arrive_lead(a2empty); });
      store_quarter(&tmMs, r0);  // LN_next(x') out
      mark(5);
      arrive_local(xfree);
      if (e == 0 && lane == 0) TTR(1, 4 * local + 3);
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the leader's MMAs / the peer's remote arrivals are done with both CTAs' smem
  if (warp == 1) tmem_dealloc_2sm<512>(tmem);
}

}  // namespace tail2

// M a multiple of 256 (pairs of 128-row tiles; the DiT has 8 tiles per slot), T a multiple of 128.
int launch_block_tail(const void* attn, const void* wproj, const float* bproj, const void* w1, const void* w2,
                           const float* b1, const float* b2, __nv_bfloat16* xres, __nv_bfloat16* xmod_out,
                           const float* gate1, const float* shift1, const float* scale1, const float* gate2,
                           const float* shift2, const float* scale2, int64_t vec_stride, float ln_eps, int64_t M, int T,
                           cudaStream_t st) {
  using namespace tail2;
  if (M % (2 * BM) || T % BM) return SF_ERR_PARAMETER;
  static bool attr = false;
  if (!attr) {
    const cudaError_t err =
        cudaFuncSetAttribute(block_tail_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (err != cudaSuccess) {
      fprintf(stderr, "streamflow: block_tail smem attribute: %s\n", cudaGetErrorString(err));
      return SF_ERR_CUDA;
    }
    attr = true;
  }
  CUtensorMap ta, tp, t1, t2, tr, trs, tms;
  int rc = make_tmap_bf16_2d(&ta, attn, D, (uint64_t)M, D, 64, BM, 128);
  rc |= make_tmap_bf16_2d(&tp, wproj, D, D, D, 64, BROWS, 128);
  rc |= make_tmap_bf16_2d(&t1, w1, D, FF, D, 64, W1ROWS, 128);
  rc |= make_tmap_bf16_2d(&t2, w2, FF, D, FF, 64, BROWS, 128);
  rc |= make_tmap_bf16_2d(&tr, xres, D, (uint64_t)M, D, 64, BM, 128);
  rc |= make_tmap_bf16_2d(&trs, xres, D, (uint64_t)M, D, 64, 32, 128);
  rc |= make_tmap_bf16_2d(&tms, xmod_out, D, (uint64_t)M, D, 64, 32, 128);
  if (rc != SF_OK) return SF_ERR_CUDA;
  Params p{xres, xmod_out, bproj, b1, b2, gate1, shift1, scale1, gate2, shift2, scale2, vec_stride, ln_eps, T, (int)M,
           g_pdl ? 1 : 0};
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int pairs = (int)(M / (2 * BM));
  const int clusters = pairs < sms / 2 ? pairs : sms / 2;
  const cudaError_t err = launch_kernel(block_tail_pair_kernel, dim3(2 * clusters), dim3(THREADS), SMEM, st, ta, tp,
                                           t1, t2, tr, trs, tms, p);
  return err == cudaSuccess ? cuda_status() : SF_ERR_CUDA;
}

}  // namespace sf

extern "C" int sf_block_tail(const void* attn, const void* wproj, const float* bproj, const void* w1, const void* w2,
                             const float* b1, const float* b2, void* xres, void* xmod_out, const float* gate1,
                             const float* shift1, const float* scale1, const float* gate2, const float* shift2,
                             const float* scale2, int64_t vec_stride, float ln_eps, int64_t M, int32_t T,
                             void* stream) {
  if (!attn || !wproj || !bproj || !w1 || !w2 || !b1 || !b2 || !xres || !xmod_out || !gate1 || !shift1 || !scale1 ||
      !gate2 || !shift2 || !scale2 || M < 1 || T < 1)
    return SF_ERR_PARAMETER;
  return sf::launch_block_tail(attn, wproj, bproj, w1, w2, b1, b2, (__nv_bfloat16*)xres, (__nv_bfloat16*)xmod_out,
                               gate1, shift1, scale1, gate2, shift2, scale2, vec_stride, ln_eps, M, T,
                               (cudaStream_t)stream);
}

#if SF_TAIL2_TRACE
extern "C" int sf_tail2_trace_read(long long* dst) {
  return cudaMemcpyFromSymbol(dst, sf::tail2::g_trace, sizeof(long long) * 16 * 128) == cudaSuccess ? 0 : -1;
}
#endif

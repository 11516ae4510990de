// Post-attention half of a DiT-S/2 block in one persistent tcgen05 kernel:
//   x   = xres + gate_msa * (attn . Wproj^T + b_proj)                   (-> xres)
//   h   = LN(x) * (1 + scale_mlp) + shift_mlp                            (stays in smem)
//   x'  = x + gate_mlp * (GELU(h . W1^T + b1) . W2^T + b2)               (-> xres)
//   out = LN(x') * (1 + scale_next) + shift_next                         (-> xmod)
// It joins the attention-projection GEMM (csrc/gemm_tcgen05.cuh RES_LN) and the fused MLP
// (csrc/mlp_fused.cu, whose structure it follows with 128-column hidden chunks): the
// MLP's input h never goes to HBM (the projection epilogue leaves it in the X buffer),
// saving a 100 MB write + read per layer at the bench shape and one kernel boundary.
//
// Per 128-row tile: [X <- attn rows (TMA)] -> 18 projection MMA blocks (M128 N128, K=384)
// into the 384-column TMEM accumulator -> [X <- xres rows] -> 16 worker warps: residual
// update in place + TMA store, row statistics, LN_mlp in place (X now holds h) -> the
// fused MLP chunks (fc1 / GELU / fc2) -> [X <- x rows] -> residual + LN_next epilogue.
#include <cstdint>
#include <cstdio>

#include "gemm_tcgen05.cuh"
#include "sf_internal.h"
#include "sf_ptx.cuh"

#ifndef SF_TAIL_FINAL_DIRECT
#define SF_TAIL_FINAL_DIRECT 0  // 1: final epilogue from registers, direct stores (measured 462 vs 378 us)
#endif

namespace sf {
namespace tail {

constexpr int D = 384, FF = 1536, BM = 128, HC = 128, NCH = FF / HC;  // 12 hidden chunks
constexpr int X_ATOM = BM * 64 * 2;  // 16 KB: 128 rows x 64 K (SW128)
constexpr int X_BYTES = 6 * X_ATOM;  // 96 KB
constexpr int STAGE = 16384;         // weight block: 128 rows x 64 K
constexpr int NSTAGE = 4;
constexpr int H_BYTES = BM * HC * 2;  // 32 KB (two 64-column atoms)
constexpr int GELU_WARPS = 8, EPI_WARPS = 8;
constexpr int WORKERS = GELU_WARPS + EPI_WARPS;
constexpr int PARTS = WORKERS / 4;    // worker warps per TMEM lane quarter
constexpr int ECOLS = D / PARTS;      // 96 output columns per worker thread
constexpr int GCOLS = HC / (GELU_WARPS / 4);  // 64 hidden columns per GELU thread
constexpr int THREADS = 32 * (2 + WORKERS);
constexpr int ACC2 = 0, ACC1 = 384;
constexpr int SMEM = 1024 + X_BYTES + NSTAGE * STAGE + H_BYTES + 4 * D * 4 + 2 * 4 * BM * 4 + FF * 4 + 3 * D * 4 + 512;

struct Params {
  const float* bp;  // b_proj [384]
  const float* b1;  // [1536]
  const float* b2;  // [384]
  __nv_bfloat16* xres;
  __nv_bfloat16* xmod_out;
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
  // next layer's QKV projection fused at the end of the tile (qkv != 0): xmod stays in smem
  int qkv;
  const float* bq;  // [1152]
  float q_scale;
  int heads;
};
constexpr int QN = 3 * D;        // 1152 QKV columns
constexpr int QCH = QN / 128;    // 9 chunks of 128 columns (two heads each)

__global__ void __maxnreg__(16384 / ((THREADS / 32 + 3) / 4) / 32 / 8 * 8)  // per-SMSP register file
    block_tail_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmWp,
                      const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmW2,
                      const __grid_constant__ CUtensorMap tmR, const __grid_constant__ CUtensorMap tmRs,
                      const __grid_constant__ CUtensorMap tmMs, const __grid_constant__ CUtensorMap tmWq,
                      const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
                      const __grid_constant__ CUtensorMap tmV, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sX = smem;
  uint8_t* sW = sX + X_BYTES;
  uint8_t* sH = sW + NSTAGE * STAGE;
  float* sVec = reinterpret_cast<float*>(sH + H_BYTES);  // bias | gate | shift | scale  [4][384]
  float* sRed = sVec + 4 * D;                            // [2 stats][PARTS][128 rows]
  float* sB1 = sRed + 2 * 4 * BM;                        // fc1 bias [1536]
  float* sBq = sB1 + FF;                                 // QKV bias [1152]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sBq + QN);
  uint64_t* wfull = bars;             // [NSTAGE]
  uint64_t* wempty = wfull + NSTAGE;  // [NSTAGE]
  uint64_t* afull = wempty + NSTAGE;  // attention rows landed in X
  uint64_t* aempty = afull + 1;       // projection MMAs done reading X
  uint64_t* pfull = aempty + 1;       // projection accumulator ready
  uint64_t* r1full = pfull + 1;       // residual rows landed in X (projection epilogue)
  uint64_t* xready = r1full + 1;      // X holds h; the accumulator is drained
  uint64_t* xempty = xready + 1;      // fc1 done reading X
  uint64_t* a1full = xempty + 1;      // fc1 chunk accumulator ready
  uint64_t* a1empty = a1full + 1;     // GELU warps have read it
  uint64_t* hfull = a1empty + 1;      // H written
  uint64_t* hempty = hfull + 1;       // fc2 has read H
  uint64_t* a2full = hempty + 1;      // fc2 accumulator ready
  uint64_t* a2empty = a2full + 1;     // final epilogue drained it
  uint64_t* r2full = a2empty + 1;     // x rows landed in X (final epilogue)
  uint64_t* xfree = r2full + 1;       // final epilogue done with X (next tile's attention may load)
  uint64_t* stored = xfree + 1;       // the projection epilogue's x stores have landed (r2 may load)
  uint64_t* mready = stored + 1;      // (qkv) X holds the next layer's xmod
  uint64_t* qfull = mready + 1;       // (qkv) [3] QKV chunk accumulator ready
  uint64_t* qempty = qfull + 3;       // (qkv) [3] drained
  uint64_t* qxfree = qempty + 3;      // (qkv) QKV MMAs done reading X
  uint64_t* hafull = qxfree + 1;      // (!qkv) [2] attention K-atom landed in an H slot
  uint64_t* haempty = hafull + 2;     // (!qkv) [2] projection MMAs done with it
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(haempty + 2);

  const uint32_t warp = warp_id(), lane = threadIdx.x & 31;
  const int tiles = p.M / BM;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmWp);
    tma_prefetch(&tmW1);
    tma_prefetch(&tmW2);
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&wfull[s], 1);
      mbar_init(&wempty[s], 1);
    }
    for (uint64_t* b : {afull, aempty, pfull, r1full, xempty, a1full, hempty, a2full, r2full}) mbar_init(b, 1);
    mbar_init(xready, WORKERS * 32);
    mbar_init(a1empty, GELU_WARPS * 32);
    mbar_init(hfull, GELU_WARPS * 32);
    mbar_init(a2empty, WORKERS * 32);
    mbar_init(xfree, WORKERS * 32);
    mbar_init(stored, WORKERS);  // one arrival per worker warp (its store-issuing lane)
    mbar_init(mready, WORKERS * 32);
    for (int i = 0; i < 3; ++i) {
      mbar_init(&qfull[i], 1);
      mbar_init(&qempty[i], WORKERS * 32);
    }
    mbar_init(qxfree, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&hafull[i], 1);
      mbar_init(&haempty[i], 1);
    }
    fence_barrier_init();
  }
  for (int i = threadIdx.x; i < FF; i += THREADS) sB1[i] = p.b1[i];
  if (p.qkv)
    for (int i = threadIdx.x; i < QN; i += THREADS) sBq[i] = p.bq[i];
  if (warp == 1) tmem_alloc<512>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  grid_dep_sync();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ------------------------------------------------------------ TMA producer
    if (elect_one()) {
      int ws = 0;
      auto wblock = [&](const CUtensorMap* m, int c0, int c1) {  // one 128-row x 64-K block
        const int s = ws % NSTAGE;
        mbar_wait(&wempty[s], ((ws / NSTAGE) & 1) ^ 1);
        mbar_expect_tx(&wfull[s], STAGE);
        tma_load_2d(sW + s * STAGE, m, &wfull[s], c0, c1);
        ++ws;
      };
      auto xload = [&](const CUtensorMap* m, uint64_t* bar, int r0) {
        mbar_expect_tx(bar, X_BYTES);
        for (int kb = 0; kb < 6; ++kb) tma_load_2d(sX + kb * X_ATOM, m, bar, kb * 64, r0);
      };
      auto w1 = [&](int c) {
        for (int kb = 0; kb < 6; ++kb) wblock(&tmW1, kb * 64, c * HC);
      };
      auto w2 = [&](int c) {
        for (int n = 0; n < 3; ++n)
          for (int a = 0; a < 2; ++a) wblock(&tmW2, c * HC + 64 * a, 128 * n);
      };
      int local = 0;
      for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
        const int r0 = tile * BM;
        if (!p.qkv) {
          // projection operands without the X buffer: attention K-atoms through the two H
          // slots (idle between the previous tile's last fc2 and this tile's first GELU),
          // Wproj blocks through the ring -- so this projection overlaps the previous
          // tile's final epilogue, which still owns X
          if (local > 0) mbar_wait(hempty, (NCH * local - 1) & 1);  // previous tile's last fc2 read H
          for (int kb = 0; kb < 6; ++kb) {
            const int u = local * 6 + kb, slot = kb & 1;
            mbar_wait(&haempty[slot], ((u >> 1) & 1) ^ 1);
            mbar_expect_tx(&hafull[slot], X_ATOM);
            tma_load_2d(sH + slot * X_ATOM, &tmA, &hafull[slot], kb * 64, r0);
            for (int n = 0; n < 3; ++n) wblock(&tmWp, kb * 64, 128 * n);
          }
          mbar_wait(xfree, (local & 1) ^ 1);  // previous tile's final epilogue left X
          xload(&tmR, r1full, r0);
        } else {
          mbar_wait(qxfree, (local & 1) ^ 1);  // previous tile's QKV MMAs left X
          xload(&tmA, afull, r0);
          for (int n = 0; n < 3; ++n)
            for (int kb = 0; kb < 6; ++kb) wblock(&tmWp, kb * 64, 128 * n);
          mbar_wait(aempty, local & 1);  // projection MMAs have read the attention rows
          xload(&tmR, r1full, r0);
        }
        w1(0);
        w1(1);
        for (int c = 0; c < NCH; ++c) {
          w2(c);
          if (c + 2 < NCH) w1(c + 2);
          if (c == NCH - 2) {  // all fc1 issued: the updated rows replace h once fc1 is done
            mbar_wait(xempty, local & 1);
            mbar_wait(stored, local & 1);  // ... and once the projection epilogue's stores landed
            xload(&tmR, r2full, r0);
          }
        }
        if (p.qkv)  // next layer's Wqkv: rows [128k, +128) x K atom kb
          for (int k = 0; k < QCH; ++k)
            for (int kb = 0; kb < 6; ++kb) wblock(&tmWq, kb * 64, 128 * k);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t idesc = idesc_bf16_f32(128, 128);
    const uint32_t sX0 = smem_u32(sX), sW0 = smem_u32(sW), sH0 = smem_u32(sH);
    int ws = 0, g = 0, local = 0;
    auto take = [&]() {
      const int s = ws % NSTAGE;
      mbar_wait(&wfull[s], (ws / NSTAGE) & 1);
      tc_fence_after();
      return s;
    };
    auto give = [&](int s) {
      if (elect_one()) mma_commit(&wempty[s]);
      __syncwarp();
      ++ws;
    };
    auto commit = [&](uint64_t* bar) {
      if (elect_one()) mma_commit(bar);
      __syncwarp();
    };
    int gq = 0;  // QKV chunks issued
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      // projection: acc2[:, 128n:+128] = attn . Wproj[128n:+128]^T
      mbar_wait(a2empty, (local & 1) ^ 1);  // previous tile's final epilogue drained the accumulator
      if (p.qkv && gq > 0)
        for (int i = 1; i <= 3; ++i) {  // ... and its QKV epilogue drained the last three chunks
          const int q = gq - i;
          mbar_wait(&qempty[q % 3], (q / 3) & 1);
        }
      if (!p.qkv) {
        for (int kb = 0; kb < 6; ++kb) {  // A = attention K-atom kb in H slot kb & 1
          const int u = local * 6 + kb, slot = kb & 1;
          mbar_wait(&hafull[slot], (u >> 1) & 1);
          tc_fence_after();
          for (int n = 0; n < 3; ++n) {
            const int s = take();
            if (elect_one()) {
              const uint64_t ad = sw128_kmajor_desc(sH0 + slot * X_ATOM);
              const uint64_t bd = sw128_kmajor_desc(sW0 + s * STAGE);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_ss(tmem + ACC2 + 128 * n, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
            }
            __syncwarp();
            give(s);
          }
          commit(&haempty[slot]);
        }
      } else {
        mbar_wait(afull, local & 1);
        tc_fence_after();
        for (int n = 0; n < 3; ++n)
          for (int kb = 0; kb < 6; ++kb) {
            const int s = take();
            if (elect_one()) {
              const uint64_t ad = sw128_kmajor_desc(sX0 + kb * X_ATOM);
              const uint64_t bd = sw128_kmajor_desc(sW0 + s * STAGE);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_ss(tmem + ACC2 + 128 * n, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
            }
            __syncwarp();
            give(s);
          }
        commit(aempty);
      }
      commit(pfull);
      mbar_wait(xready, local & 1);  // X holds h, the projection accumulator is drained
      tc_fence_after();
      // g + c: the global index of hidden chunk c (fc1, GELU and fc2 of a chunk share it)
      auto fc1 = [&](int c) {
        mbar_wait(a1empty, ((g + c) & 1) ^ 1);  // GELU warps read the previous chunk
        for (int kb = 0; kb < 6; ++kb) {
          const int s = take();
          if (elect_one()) {
            const uint64_t ad = sw128_kmajor_desc(sX0 + kb * X_ATOM);
            const uint64_t bd = sw128_kmajor_desc(sW0 + s * STAGE);
#pragma unroll
            for (int k = 0; k < 4; ++k) mma_bf16_ss(tmem + ACC1, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          }
          __syncwarp();
          give(s);
        }
        if (c == NCH - 1) commit(xempty);
        commit(a1full);
      };
      auto fc2 = [&](int c) {
        mbar_wait(hfull, (g + c) & 1);
        tc_fence_after();
        for (int n = 0; n < 3; ++n)
          for (int a = 0; a < 2; ++a) {
            const int s = take();
            if (elect_one()) {
              const uint64_t ad = sw128_kmajor_desc(sH0 + a * X_ATOM);
              const uint64_t bd = sw128_kmajor_desc(sW0 + s * STAGE);
#pragma unroll
              for (int k = 0; k < 4; ++k)
                mma_bf16_ss(tmem + ACC2 + 128 * n, ad + 2 * k, bd + 2 * k, idesc, (c | a | k) != 0);
            }
            __syncwarp();
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
      g += NCH;
      if (p.qkv) {
        // next layer's QKV: 9 chunks of 128 columns through three 128-column TMEM buffers
        mbar_wait(mready, local & 1);  // X holds xmod; the fc2 accumulator is drained
        tc_fence_after();
        for (int k = 0; k < QCH; ++k, ++gq) {
          const int b = gq % 3;
          mbar_wait(&qempty[b], ((gq / 3) & 1) ^ 1);
          tc_fence_after();
          for (int kb = 0; kb < 6; ++kb) {
            const int s = take();
            if (elect_one()) {
              const uint64_t ad = sw128_kmajor_desc(sX0 + kb * X_ATOM);
              const uint64_t bd = sw128_kmajor_desc(sW0 + s * STAGE);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk)
                mma_bf16_ss(tmem + ACC2 + 128 * b, ad + 2 * kk, bd + 2 * kk, idesc, (kb | kk) != 0);
            }
            __syncwarp();
            give(s);
          }
          if (k == QCH - 1) commit(qxfree);
          commit(&qfull[b]);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ worker warps 2..17
    const bool is_gelu = warp < 2 + GELU_WARPS;
    const uint32_t quarter = warp & 3;
    const uint32_t row = quarter * 32 + lane;
    const uint32_t e = warp - 2, part = e >> 2;
    const uint32_t gaddr = tmem + ((quarter * 32) << 16) + ACC1 + part * GCOLS;
    const int col0 = ECOLS * part;
    const uint32_t eaddr = tmem + ((quarter * 32) << 16) + ACC2 + col0;
    constexpr int NQ = ECOLS / 32;
    auto xp = [&](int col) -> uint4* {
      const int a = col >> 6, j = (col & 63) >> 3;
      return reinterpret_cast<uint4*>(sX + a * X_ATOM + row * 128 + ((j ^ (row & 7)) * 16));
    };
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
    auto load_vecs = [&](const float* bias, const float* gate, const float* shift, const float* scale, int64_t slot) {
      named_bar_sync(1, WORKERS * 32);  // the previous readers are done with sVec
      for (int i = e * 32 + lane; i < D; i += WORKERS * 32) {
        const int64_t o = slot * p.vec_stride + i;
        sVec[i] = bias[i];
        sVec[D + i] = gate[o];
        sVec[2 * D + i] = shift[o];
        sVec[3 * D + i] = scale[o];
      }
      named_bar_sync(1, WORKERS * 32);
    };
    // residual update (in place in X) + TMA store of x + row statistics -> (mean, rstd);
    // then LN * (1 + scale) + shift in place.  `done_acc` is called after the last TMEM read.
    auto res_ln = [&](int r0, uint64_t* acc_full, uint32_t acc_ph, uint64_t* rows_full, uint32_t rows_ph,
                      auto done_acc) {
      mbar_wait(acc_full, acc_ph);
      mbar_wait(rows_full, rows_ph);
      tc_fence_after();
      float sum = 0.f, sq = 0.f;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        float v[32];
        tmem_ld32(eaddr + 32 * q, v);
        tmem_ld_wait();
        if (q + 1 == NQ) {
          tc_fence_before();
          done_acc();
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
      sRed[(0 * PARTS + part) * BM + row] = sum;
      sRed[(1 * PARTS + part) * BM + row] = sq;
      store_quarter(&tmRs, r0);  // x out (its barriers also publish sRed)
      float tsum = 0.f, tsq = 0.f;
#pragma unroll
      for (int k = 0; k < PARTS; ++k) {
        tsum += sRed[k * BM + row];
        tsq += sRed[(PARTS + k) * BM + row];
      }
      const float mean = tsum * (1.0f / D);
      const float var = fmaxf(tsq * (1.0f / D) - mean * mean, 0.f);
      const float rstd = rsqrtf(var + p.ln_eps);
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
    };
    int g = 0, gq = 0, local = 0;
    for (int tile = blockIdx.x; tile < tiles; tile += gridDim.x, ++local) {
      const int r0 = tile * BM;
      const int64_t slot = r0 / p.T;
      // ---- projection epilogue: x = xres + gate_msa * (acc + b_proj) -> xres; X <- LN_mlp(x)
      load_vecs(p.bp, p.g1, p.sh1, p.sc1, slot);
      res_ln(r0, pfull, local & 1, r1full, local & 1, [] {});
      fence_proxy_async_smem();  // h is read by the fc1 MMAs (async proxy)
      mbar_arrive(xready);       // (all TMEM reads of the projection accumulator precede this)
      if (lane == 0) {
        bulk_wait<0>();          // this warp's x stores have landed (the final epilogue reloads x)
        mbar_arrive(stored);
      }
      __syncwarp();
      // ---- MLP: GELU of every hidden chunk
      if (is_gelu) {
        for (int c = 0; c < NCH; ++c, ++g) {
          mbar_wait(a1full, g & 1);
          tc_fence_after();
          const float* bb = sB1 + c * HC + part * GCOLS;
          uint32_t pk[GCOLS / 2];
#pragma unroll
          for (int h = 0; h < GCOLS / 32; ++h) {
            float v[32];
            tmem_ld32(gaddr + 32 * h, v);
            tmem_ld_wait();
            if (h + 1 == GCOLS / 32) {
              tc_fence_before();
              mbar_arrive(a1empty);
            }
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const float2 bv = reinterpret_cast<const float2*>(bb + 32 * h)[i];
              float2 y = __fadd2_rn(make_float2(v[2 * i], v[2 * i + 1]), bv);
              y = gelu_tanh2(y);
              pk[16 * h + i] = pack_bf16(y.x, y.y);
            }
          }
          mbar_wait(hempty, (g & 1) ^ 1);  // fc2 has read H
          uint8_t* hrow = sH + row * 128;
#pragma unroll
          for (int j = 0; j < GCOLS / 8; ++j) {
            const int col = part * GCOLS + 8 * j;
            const int at = col >> 6, cj = (col & 63) >> 3;
            *reinterpret_cast<uint4*>(hrow + at * X_ATOM + ((cj ^ (row & 7)) * 16)) =
                make_uint4(pk[4 * j], pk[4 * j + 1], pk[4 * j + 2], pk[4 * j + 3]);
          }
          fence_proxy_async_smem();
          mbar_arrive(hfull);
        }
      }
      // ---- final epilogue: x' = x + gate_mlp * (acc + b2) -> xres; LN_next(x') -> xmod
      load_vecs(p.b2, p.g2, p.sh2, p.sc2, slot);
#if SF_TAIL_FINAL_DIRECT
      if (!p.qkv) {
        // x' stays in registers (bf16 pairs), so X is released as soon as the old rows are read;
        // both outputs leave by direct 16-byte stores, overlapping the next tile's projection
        // epilogue, which may then load its residual rows into X at once
        mbar_wait(a2full, local & 1);
        mbar_wait(r2full, local & 1);
        tc_fence_after();
        uint32_t xq[NQ][16];
        float sum = 0.f, sq = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            float v[16];
            tmem_ld16(eaddr + 32 * q + 16 * hh, v);
            tmem_ld_wait();
            const float* vb = sVec + col0 + 32 * q + 16 * hh;
            const float* vg = sVec + D + col0 + 32 * q + 16 * hh;
#pragma unroll
            for (int j = 0; j < 2; ++j) {
              const uint4 ov = *xp(col0 + 32 * q + 16 * hh + 8 * j);
              const uint32_t ow[4] = {ov.x, ov.y, ov.z, ov.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const int c = 8 * j + 2 * i;
                const float2 o = unpack_bf16(ow[i]);
                const uint32_t nw = pack_bf16(o.x + vg[c] * (v[c] + vb[c]), o.y + vg[c + 1] * (v[c + 1] + vb[c + 1]));
                xq[q][8 * hh + 4 * j + i] = nw;
                const float2 n = unpack_bf16(nw);
                sum += n.x + n.y;
                sq += n.x * n.x + n.y * n.y;
              }
            }
          }
        tc_fence_before();
        mbar_arrive(a2empty);
        mbar_arrive(xfree);
        __nv_bfloat16* xr = p.xres + (int64_t)(r0 + row) * D + col0;
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            reinterpret_cast<uint4*>(xr + 32 * q)[i] =
                make_uint4(xq[q][4 * i], xq[q][4 * i + 1], xq[q][4 * i + 2], xq[q][4 * i + 3]);
        sRed[(0 * PARTS + part) * BM + row] = sum;
        sRed[(1 * PARTS + part) * BM + row] = sq;
        named_bar_sync(2 + quarter, 32 * PARTS);
        float tsum = 0.f, tsq = 0.f;
#pragma unroll
        for (int k = 0; k < PARTS; ++k) {
          tsum += sRed[k * BM + row];
          tsq += sRed[(PARTS + k) * BM + row];
        }
        named_bar_sync(2 + quarter, 32 * PARTS);  // all read before sRed is reused
        const float mean = tsum * (1.0f / D);
        const float var = fmaxf(tsq * (1.0f / D) - mean * mean, 0.f);
        const float rstd = rsqrtf(var + p.ln_eps);
        __nv_bfloat16* xm = p.xmod_out + (int64_t)(r0 + row) * D + col0;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float* vsh = sVec + 2 * D + col0 + 32 * q;
          const float* vsc = sVec + 3 * D + col0 + 32 * q;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            uint32_t o[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const int c = 8 * j + 2 * i;
              const float2 x = unpack_bf16(xq[q][4 * j + i]);
              o[i] = pack_bf16((x.x - mean) * rstd * (1.0f + vsc[c]) + vsh[c],
                               (x.y - mean) * rstd * (1.0f + vsc[c + 1]) + vsh[c + 1]);
            }
            reinterpret_cast<uint4*>(xm + 32 * q)[j] = make_uint4(o[0], o[1], o[2], o[3]);
          }
        }
        continue;
      }
#endif
      res_ln(r0, a2full, local & 1, r2full, local & 1, [&] { mbar_arrive(a2empty); });
      if (!p.qkv) {
        store_quarter(&tmMs, r0);
        mbar_arrive(xfree);
        continue;
      }
      // ---- next layer's QKV from the xmod rows in X: scatter head-major Q (scaled), K, V^T
      fence_proxy_async_smem();  // xmod is read by the QKV MMAs (async proxy)
      mbar_arrive(mready);
      const int tok0 = r0 - (int)slot * p.T + quarter * 32;  // this warp's 32 tokens within the slot
      uint8_t* stg = sH + e * 2048;                            // 32 rows x 64 B (SW64) staging
      for (int k = 0; k < QCH; ++k, ++gq) {
        const int b = gq % 3;
        mbar_wait(&qfull[b], (gq / 3) & 1);
        tc_fence_after();
        float v[32];
        tmem_ld32(tmem + ((quarter * 32) << 16) + ACC2 + 128 * b + 32 * part, v);
        tmem_ld_wait();
        tc_fence_before();
        mbar_arrive(&qempty[b]);
        const int gc = 128 * k + 32 * part;  // QKV column of v[0]
        const int which = gc / D, head = (gc - which * D) / 64, dim0 = gc & 63;
        const float sc = which == 0 ? p.q_scale : 1.0f;
        if (lane == 0) bulk_wait_read<0>();  // the previous chunk's store has read the staging
        __syncwarp();
        if (which < 2) {  // Q / K rows: 32 tokens x 32 dims (64 B, SW64)
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t pk[4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
              pk[i] = pack_bf16((v[8 * c + 2 * i] + sBq[gc + 8 * c + 2 * i]) * sc,
                                (v[8 * c + 2 * i + 1] + sBq[gc + 8 * c + 2 * i + 1]) * sc);
            *reinterpret_cast<uint4*>(stg + lane * 64 + ((c ^ ((lane >> 1) & 3)) * 16)) =
                make_uint4(pk[0], pk[1], pk[2], pk[3]);
          }
        } else {  // V^T rows: 32 dims x 32 tokens (fp16, 64 B, SW64)
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const uint32_t dd = i;
            *reinterpret_cast<__half*>(stg + dd * 64 + (((lane >> 3) ^ ((dd >> 1) & 3)) * 16) + (lane & 7) * 2) =
                __float2half_rn(v[i] + sBq[gc + i]);
          }
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int64_t bh = slot * p.heads + head;
          if (which == 0)
            tma_store_2d(&tmQ, stg, dim0, (int)(bh * p.T + tok0));
          else if (which == 1)
            tma_store_2d(&tmK, stg, dim0, (int)(bh * p.T + tok0));
          else
            tma_store_2d(&tmV, stg, tok0, (int)(bh * 64 + dim0));
          bulk_commit();
        }
        __syncwarp();
      }
      if (lane == 0) bulk_wait_read<0>();  // H is the next tile's hidden buffer
      __syncwarp();
    }
    if (lane == 0) bulk_wait<0>();
    __syncwarp();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<512>(tmem);
}

}  // namespace tail

int launch_block_tail(const void* attn, const void* wproj, const float* bproj, const void* w1, const void* w2,
                      const float* b1, const float* b2, __nv_bfloat16* xres, __nv_bfloat16* xmod_out,
                      const float* gate1, const float* shift1, const float* scale1, const float* gate2,
                      const float* shift2, const float* scale2, int64_t vec_stride, float ln_eps, int64_t M, int T,
                      cudaStream_t st, const void* wqkv, const float* bqkv, void* q, void* k, void* vt, int heads,
                      float q_scale) {
  using namespace tail;
  if (M % BM || T % BM) return SF_ERR_PARAMETER;
  static int pair = -1;  // TEMP A/B switch (SF_TAIL_PAIR=0: single-CTA kernel)
  if (pair < 0) {
    const char* e = getenv("SF_TAIL_PAIR");
    pair = (e && e[0] == '0') ? 0 : 1;
  }
  if (pair && !wqkv && M % (2 * BM) == 0)
    return launch_block_tail_pair(attn, wproj, bproj, w1, w2, b1, b2, xres, xmod_out, gate1, shift1, scale1, gate2,
                                  shift2, scale2, vec_stride, ln_eps, M, T, st);
  static bool attr = false;
  if (!attr) {
    const cudaError_t err = cudaFuncSetAttribute(block_tail_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
    if (err != cudaSuccess) {
      fprintf(stderr, "streamflow: block_tail smem attribute: %s\n", cudaGetErrorString(err));
      return SF_ERR_CUDA;
    }
    attr = true;
  }
  CUtensorMap ta, tp, t1, t2, tr, trs, tms;
  int rc = make_tmap_bf16_2d(&ta, attn, D, (uint64_t)M, D, 64, BM, 128);
  rc |= make_tmap_bf16_2d(&tp, wproj, D, D, D, 64, 128, 128);
  rc |= make_tmap_bf16_2d(&t1, w1, D, FF, D, 64, HC, 128);
  rc |= make_tmap_bf16_2d(&t2, w2, FF, D, FF, 64, 128, 128);
  rc |= make_tmap_bf16_2d(&tr, xres, D, (uint64_t)M, D, 64, BM, 128);
  rc |= make_tmap_bf16_2d(&trs, xres, D, (uint64_t)M, D, 64, 32, 128);
  rc |= make_tmap_bf16_2d(&tms, xmod_out, D, (uint64_t)M, D, 64, 32, 128);
  CUtensorMap twq = tp, tq = tms, tk = tms, tv = tms;  // placeholders when the QKV phase is off
  const bool qkv = wqkv != nullptr;
  if (qkv) {
    if (heads * 64 != D) return SF_ERR_PARAMETER;
    const uint64_t bh = (uint64_t)(M / T) * heads;
    rc |= make_tmap_bf16_2d(&twq, wqkv, D, QN, D, 64, 128, 128);
    rc |= make_tmap_bf16_2d(&tq, q, 64, bh * T, 64, 32, 32, 64);
    rc |= make_tmap_bf16_2d(&tk, k, 64, bh * T, 64, 32, 32, 64);
    rc |= make_tmap_bf16_2d(&tv, vt, T, bh * 64, T, 32, 32, 64);
  }
  if (rc != SF_OK) return SF_ERR_CUDA;
  Params p{bproj, b1, b2, xres, xmod_out, gate1, shift1, scale1, gate2, shift2, scale2, vec_stride, ln_eps, T, (int)M,
           qkv ? 1 : 0, bqkv, q_scale, heads};
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int tiles = (int)(M / BM);
  const cudaError_t err = launch_maybe_pdl(block_tail_kernel, dim3(tiles < sms ? tiles : sms), dim3(THREADS), SMEM, st,
                                           ta, tp, t1, t2, tr, trs, tms, twq, tq, tk, tv, p);
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
                               (cudaStream_t)stream, nullptr, nullptr, nullptr, nullptr, nullptr, 0, 0.f);
}

extern "C" int sf_block_tail_qkv(const void* attn, const void* wproj, const float* bproj, const void* w1,
                                 const void* w2, const float* b1, const float* b2, void* xres, const float* gate1,
                                 const float* shift1, const float* scale1, const float* gate2, const float* shift2,
                                 const float* scale2, int64_t vec_stride, float ln_eps, int64_t M, int32_t T,
                                 const void* wqkv, const float* bqkv, void* q, void* k, void* vt, int32_t heads,
                                 float q_scale, void* stream) {
  if (!attn || !wproj || !bproj || !w1 || !w2 || !b1 || !b2 || !xres || !gate1 || !shift1 || !scale1 || !gate2 ||
      !shift2 || !scale2 || !wqkv || !bqkv || !q || !k || !vt || M < 1 || T < 1)
    return SF_ERR_PARAMETER;
  return sf::launch_block_tail(attn, wproj, bproj, w1, w2, b1, b2, (__nv_bfloat16*)xres, (__nv_bfloat16*)xres,
                               gate1, shift1, scale1, gate2, shift2, scale2, vec_stride, ln_eps, M, T,
                               (cudaStream_t)stream, wqkv, bqkv, q, k, vt, heads, q_scale);
}

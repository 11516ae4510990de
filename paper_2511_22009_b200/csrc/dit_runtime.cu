// DiT velocity-field runtime: the per-step launch sequence of the stream batch.
//
//   prepare (K11 ring bookkeeping) -> cond (K1: t-embed MLP + y-embed + SiLU)
//   -> adaLN GEMM (K3, all blocks at once) -> patch-embed + pos + LN1 (K2/K4)
//   -> 12 x [QKV GEMM (K5) -> flash attention (K6) -> proj GEMM + gated
//            residual + LN2 (K7+K4) -> fc1 GEMM + GELU (K8) -> fc2 GEMM +
//            gated residual + next LN (K9+K4)]
//   -> final layer fused with CFG combine + Euler + emit + refill (K10+K11)
//
// The handle owns host-side state only (config, TMA descriptors, graph
// cache).  All device memory (weights, workspace, ring state) is owned by the
// caller and passed as raw pointers.
#include <algorithm>
#include <map>
#include <tuple>
#include <vector>

#include "gemm_tcgen05.cuh"
#include "sf_internal.h"


namespace sf {

// ============================================================ shared helpers
__device__ __forceinline__ float silu(float x) { return x / (1.0f + __expf(-x)); }

__device__ __forceinline__ uint4 philox4x32(uint4 c, uint2 k) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
    const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
    c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    k.x += 0x9E3779B9u;
    k.y += 0xBB67AE85u;
  }
  return c;
}
// N(0,1) sample #idx of generation `gen` of a stream seeded `seed` (Philox + Box-Muller).
__device__ __forceinline__ float philox_normal(uint64_t seed, int64_t gen, int64_t idx) {
  const uint4 r = philox4x32(make_uint4((uint32_t)(idx >> 2), (uint32_t)gen, (uint32_t)(gen >> 32), 0x5f1u),
                             make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
  const int lane = idx & 3;
  const uint32_t a = (lane < 2) ? r.x : r.z, b = (lane < 2) ? r.y : r.w;
  const float u1 = ((float)a + 1.0f) * 2.3283064365386963e-10f;  // (0, 1]
  const float u2 = (float)b * 2.3283064365386963e-10f;
  const float rad = sqrtf(-2.0f * __logf(u1));
  float s, c;
  __sincosf(6.283185307179586f * u2, &s, &c);
  return (lane & 1) ? rad * s : rad * c;
}

// philox_normal for the final layer's 8 elements per lane (idx[nt][i], see final_layer_mma_kernel):
// the four lanes 8k + (c & 1) + {0, 2, 4, 6} own the four samples of one Philox counter
// (idx >> 2) for every element slot u = 4 nt + i, so lane r = 2 (g & 1) + (c >> 1) of the group
// runs the generator for slots 2r, 2r + 1 (all four samples each) and the samples are
// exchanged with shuffles: 2 Philox calls per lane instead of 8, the same values.
__device__ __forceinline__ void philox_normal_group8(uint64_t seed, int64_t gen, const int64_t (&idx)[2][4], int lane,
                                                     float (&out)[2][4]) {
  const int g = lane >> 2, c = lane & 3;
  const int r = 2 * (g & 1) + (c >> 1);  // this lane's sample within a counter = idx % 4
  const int base = lane & ~0x6;  // lane of r = 0 in this group: 8k + (c & 1)
  float v[2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    // slot u = 2r + h: every lane computes its own slot's counter from its own idx (the four lanes
    // of the group hold the same counter for a given slot)
    int64_t myidx = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (u == 2 * r + h) myidx = idx[u >> 2][u & 3];
    const uint4 q = philox4x32(make_uint4((uint32_t)(myidx >> 2), (uint32_t)gen, (uint32_t)(gen >> 32), 0x5f1u),
                               make_uint2((uint32_t)seed, (uint32_t)(seed >> 32)));
#pragma unroll
    for (int pr = 0; pr < 2; ++pr) {
      const uint32_t a = pr ? q.z : q.x, b = pr ? q.w : q.y;
      const float u1 = ((float)a + 1.0f) * 2.3283064365386963e-10f;  // (0, 1]
      const float u2 = (float)b * 2.3283064365386963e-10f;
      const float rad = sqrtf(-2.0f * __logf(u1));
      float sn, cs;
      __sincosf(6.283185307179586f * u2, &sn, &cs);
      v[h][2 * pr] = rad * cs;
      v[h][2 * pr + 1] = rad * sn;
    }
  }
  // slot u lives in lane base + 2 (u >> 1) (its r = u >> 1), register v[u & 1][.]; lane r needs sample r
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int src = base + 2 * (u >> 1);
    float got = 0.f;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const float t = __shfl_sync(0xffffffffu, v[u & 1][k], src);
      if (k == r) got = t;
    }
    out[u >> 2][u & 3] = got;
  }
}

// Where a network row takes its inputs from (stream mode vs direct forward).
struct RowSrc {
  const int64_t* row_info;  // stream mode: ring bookkeeping; nullptr in direct mode
  const double* ts;         // stream: row_t per ring row; direct: t per net row
  int64_t R;                // ring rows (stream) / net rows (direct)
  int cfg;                  // stream mode: net rows [0,R) uncond, [R,2R) cond
  const double* emb;        // stream: [S, E]; direct: [rows, E]
  const double* neg;        // stream + cfg: [S, E] or nullptr (zeros)
  int E;
  int pdl;                  // launched with programmatic serialisation (sf_internal.h g_pdl)
};

// ============================================================ K1: conditioning
// c = MLP(sinusoid(1000 t)) + Linear(emb); out = bf16(SiLU(c)) (adaLN input).
// Two launches, grid (net rows, hidden / 128), one output feature per thread,
// weights in the transposed [in][out] layout so a warp's loads are coalesced:
//   cond_h1_kernel:  h1 = SiLU(W1 . sinusoid(1000 t) + b1)            (fp32 scratch)
//   cond_out_kernel: out = bf16(SiLU(W2 . h1 + b2 + Wy . emb + by))
__device__ __forceinline__ const double* cond_emb_row(const RowSrc& src, int64_t i, bool* zero_emb) {
  const int64_t lr = i % src.R;
  *zero_emb = false;
  if (src.row_info) {
    const int64_t s = src.row_info[lr * 4 + 3];
    if (src.cfg && i < src.R) {
      *zero_emb = src.neg == nullptr;
      return src.neg ? src.neg + s * src.E : nullptr;
    }
    return src.emb + s * src.E;
  }
  return src.emb + i * src.E;
}

// Block = 8 warps x 32 output features: lane = feature (coalesced 64-byte weight
// rows), warp w reduces k in [w K/8, (w+1) K/8) with 8 loads in flight, then the
// 8 partial sums meet in shared memory.
__device__ __forceinline__ float dot_col_split(const float* __restrict__ v, const __nv_bfloat16* __restrict__ wt,
                                               int K, int ld, int n, float* red) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int k0 = (int)((int64_t)K * w / 8), k1 = (int)((int64_t)K * (w + 1) / 8);
  float a[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  int k = k0;
  if (n < ld) {
    for (; k + 8 <= k1; k += 8)
#pragma unroll
      for (int u = 0; u < 8; ++u) a[u] += v[k + u] * __bfloat162float(wt[(int64_t)(k + u) * ld + n]);
    for (; k < k1; ++k) a[0] += v[k] * __bfloat162float(wt[(int64_t)k * ld + n]);
  }
  red[w * 32 + lane] = ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
  __syncthreads();
  float r = 0.f;
  if (w == 0)
#pragma unroll
    for (int q = 0; q < 8; ++q) r += red[q * 32 + lane];
  __syncthreads();
  return r;  // valid in warp 0
}

__global__ void __launch_bounds__(256) cond_h1_kernel(RowSrc src, int hidden, int freq_dim,
                                                      const __nv_bfloat16* __restrict__ w1t,
                                                      const float* __restrict__ b1, float* __restrict__ h1) {
  extern __shared__ float sh[];
  float* f = sh;               // [freq_dim]
  float* red = sh + freq_dim;  // [8][32]
  pdl_wait(src.pdl);
  if (threadIdx.x == 0) pdl_trigger(src.pdl);
  const int64_t i = blockIdx.x;
  const double t = src.ts[i % src.R];
  const int half = freq_dim / 2;
  const float tm = (float)(1000.0 * t);
  for (int k = threadIdx.x; k < half; k += blockDim.x) {
    const float fr = expf(-9.210340371976184f * (float)k / (float)half);  // ln(10000)
    const float a = tm * fr;
    f[k] = cosf(a);
    f[half + k] = sinf(a);
  }
  __syncthreads();
  const int n = blockIdx.y * 32 + (threadIdx.x & 31);
  const float acc = dot_col_split(f, w1t, freq_dim, hidden, n, red);
  if (threadIdx.x < 32 && n < hidden) h1[i * hidden + n] = silu(b1[n] + acc);
}

__global__ void __launch_bounds__(256) cond_out_kernel(RowSrc src, int hidden, const float* __restrict__ h1g,
                                                       const __nv_bfloat16* __restrict__ w2t,
                                                       const float* __restrict__ b2,
                                                       const __nv_bfloat16* __restrict__ ywt,
                                                       const float* __restrict__ yb, __nv_bfloat16* __restrict__ out) {
  extern __shared__ float sh[];
  float* h1 = sh;             // [hidden]
  float* e = sh + hidden;     // [64]
  float* red = e + 64;        // [8][32]
  pdl_wait(src.pdl);
  if (threadIdx.x == 0) pdl_trigger(src.pdl);
  const int64_t i = blockIdx.x;
  bool zero_emb;
  const double* er = cond_emb_row(src, i, &zero_emb);
  for (int k = threadIdx.x; k < hidden; k += blockDim.x) h1[k] = h1g[i * hidden + k];
  for (int k = threadIdx.x; k < src.E; k += blockDim.x) e[k] = zero_emb ? 0.0f : (float)er[k];
  __syncthreads();
  const int n = blockIdx.y * 32 + (threadIdx.x & 31);
  const float acc = dot_col_split(h1, w2t, hidden, hidden, n, red);
  if (threadIdx.x < 32 && n < hidden) {
    float y = yb[n];
    for (int k = 0; k < src.E; ++k) y += e[k] * __bfloat162float(ywt[(int64_t)k * hidden + n]);
    out[i * hidden + n] = __float2bfloat16_rn(silu(b2[n] + acc + y));
  }
}

// 16-byte streaming load (read once: no L1 allocation)
__device__ __forceinline__ uint4 ldg_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}

// d += A(16x16 bf16) * B(16x8 bf16), fp32 accumulate (warp-level tensor path)
__device__ __forceinline__ void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                               uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, {%8, %9}, "
      "{%0, %1, %2, %3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}


// Patch embed + LN1 modulate on the warp-level tensor path (mma.sync m16n8k16): one warp per
// 16 consecutive tokens, K = 16 = the patch vector (C=4, P=2), HID/8 n8 tiles.  x is fp32, so
// it enters as a bf16 hi/lo pair (x = hi + lo to 2^-17 relative; two MMAs per tile) against the
// bf16 weights, fp32 accumulate.  Lane (g = lane/4, c = lane%4) holds A pairs k = 2c, 2c+1
// (channel c/2, patch row c%2: one float2 of x) and k = 2c+8, 2c+9 (channel c/2 + 2), and
// after each MMA tokens g, g+8 x fragment columns 2c, 2c+1 of each tile.  Output columns are
// permuted over blocks of four tiles: fragment column 2c+e of tile q of block blk is hidden
// column 32 blk + 8c + 2q + e, so a lane owns 8 consecutive columns per block (one 16-byte
// bf16 run).  The B fragments (weight rows in that order) are pre-arranged in smem as one
// uint2 per lane per tile (conflict-free LDS.64).
//
// Work split: CTA c owns the 16-token group tg = c % (T/16) of every latent row it visits
// (rows c / (T/16), + CTAs / (T/16), ...; the host makes the grid a multiple of T/16), so the
// group's slice of the positional table (16 x HID fp32, with the patch bias pre-added in the
// reference's order) is loaded into shared memory ONCE per CTA instead of per group from L2
// (the long-scoreboard stall that bounded the previous version).  The next group's x is
// prefetched into registers.  The 16 residual rows are staged in shared memory as NSEG = HID/192
// segments of 208 elements (416 B: consecutive rows alternate 64-byte bank halves, conflict-
// free 16-byte writes); the copy-out loop reads them back in a row-contiguous layout (8 bytes
// per lane) and writes both the residual and LN + modulate with coalesced stores.  (The residual
// used to leave by a TMA store of the staged rows; waiting for that store to have read the
// buffer before the next row cost 5%.)
template <int HID>
struct PatchMma {
  static constexpr int NT = HID / 8;
  static constexpr int NSEG = HID / 192;
  static constexpr int TROW = NSEG * 416;                     // staged row (bytes)
  static constexpr int WARPS = HID <= 384 ? 5 : 2;            // per CTA
  static constexpr int CPS = HID <= 384 ? 2 : 1;              // resident CTAs per SM (shared-memory bound)
  static constexpr int WBUF = 16 * TROW + 16 * 2 * 4;         // per warp: 16 rows + (mean, rstd) x 16
  static constexpr int PROW = HID + 4;                        // pos row (floats), padded: the LDS.128 of rows
                                                              // g and g+1 land on disjoint banks (was 2-way)
  static constexpr int POS = 16 * PROW * 4;                   // the CTA's pos (+ bias) slice, fp32
  static constexpr int SMEM = NT * 32 * 8 + POS + WARPS * WBUF;
  static_assert((TROW % 128) == 64, "staged rows must alternate 64-byte bank halves");
};

template <int HID>
__device__ __forceinline__ int patch_seg_off(int col) {  // byte offset of hidden column col in a staged row
  return (col / 192) * 416 + (col % 192) * 2;
}

template <int HID>
__global__ void __launch_bounds__(32 * PatchMma<HID>::WARPS) patch_embed_ln_mma_kernel(
    const float* __restrict__ x, int64_t lat_rows, int HW, int P, int C, const __nv_bfloat16* __restrict__ pw,
    const float* __restrict__ pb, const float* __restrict__ pos, const float* __restrict__ mod, int64_t mod_stride,
    float ln_eps, __nv_bfloat16* __restrict__ xres, __nv_bfloat16* __restrict__ xmod, int64_t total_tokens,
    int pdl) {
  using PM = PatchMma<HID>;
  constexpr int NT = PM::NT, TROW = PM::TROW;
  extern __shared__ __align__(128) uint8_t psm[];
  uint2* sB = reinterpret_cast<uint2*>(psm);  // [NT][32 lanes]
  float* sPos = reinterpret_cast<float*>(psm + NT * 32 * 8);  // [16][PROW]: bias + pos of this CTA's tokens
  const uint32_t* pw32 = reinterpret_cast<const uint32_t*>(pw);  // [HID][8] bf16 pairs
  const int gw = HW / P, T = gw * gw, TG = T / 16;
  const int tg = blockIdx.x % TG, tau0 = tg * 16;
  // (compile-time trip counts, fully unrolled: every load of the prologue is in flight at once
  // instead of ~10 dependent L2 round trips per thread)
  constexpr int NTHR = 32 * PM::WARPS;
#pragma unroll
  for (int idx = threadIdx.x; idx < NT * 32; idx += NTHR) {
    const int tile = idx / 32, gg = (idx % 32) / 4, cc = idx % 4;
    const int n = 32 * (tile / 4) + 8 * (gg >> 1) + 2 * (tile % 4) + (gg & 1);  // permuted weight row
    sB[idx] = make_uint2(pw32[n * 8 + cc], pw32[n * 8 + 4 + cc]);
  }
#pragma unroll
  for (int idx = threadIdx.x; idx < 16 * HID / 4; idx += NTHR) {
    const int r = idx / (HID / 4), c4 = idx % (HID / 4);
    const float4 pv = __ldg(reinterpret_cast<const float4*>(pos + (int64_t)(tau0 + r) * HID) + c4);
    const float4 bv = __ldg(reinterpret_cast<const float4*>(pb) + c4);
    reinterpret_cast<float4*>(sPos + r * PM::PROW)[c4] = make_float4(bv.x + pv.x, bv.y + pv.y, bv.z + pv.z, bv.w + pv.w);
  }
  __syncthreads();
  // weights and the positional slice are no kernel's output: staged above under the previous
  // kernel's tail; the latents and the adaLN vectors are read after the dependency wait
  pdl_wait(pdl);
  if (threadIdx.x == 0) pdl_trigger(pdl);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  uint8_t* sY = psm + NT * 32 * 8 + PM::POS + warp * PM::WBUF;  // [16][TROW] staged bf16 residual rows
  float* sStat = reinterpret_cast<float*>(sY + 16 * TROW);      // [16][rstd, -mean * rstd]
  const int64_t rows = total_tokens / T;
  const int64_t rstride = (int64_t)(gridDim.x / TG) * PM::WARPS;
  const float* pos0 = sPos + g * PM::PROW + 8 * c;
  const float* pos1 = pos0 + 8 * PM::PROW;
  uint8_t* y0 = sY + g * TROW + 16 * c;
  uint8_t* y1 = y0 + 8 * TROW;
  // x of this lane for latent row ni: (row g, k 2c) (row g+8, k 2c) (row g, k 2c+8) (row g+8, k 2c+8)
  auto load_x = [&](int64_t ni, float2 (&v)[4]) {
    const float* xl = x + (ni % lat_rows) * (int64_t)C * HW * HW;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int tau = tau0 + g + 8 * (i & 1);
      const int pi = tau / gw, pj = tau % gw;
      const int ch = (c >> 1) + 2 * (i >> 1), p = c & 1;
      v[i] = __ldg(reinterpret_cast<const float2*>(xl + (int64_t)ch * HW * HW + (pi * 2 + p) * HW + pj * 2));
    }
  };
  int64_t ni = (int64_t)(blockIdx.x / TG) * PM::WARPS + warp;
  float2 xv[4];
  if (ni < rows) load_x(ni, xv);
  constexpr int J = HID / 128;
  for (; ni < rows; ni += rstride) {
    // (the bulk wait comes before the next row's x loads: it compiles to a scoreboard wait that
    // would otherwise also wait for those loads)
    __syncwarp();
    uint32_t ahi[4], alo[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      ahi[i] = pack_bf16(xv[i].x, xv[i].y);
      const float2 h = unpack_bf16(ahi[i]);
      alo[i] = pack_bf16(xv[i].x - h.x, xv[i].y - h.y);
    }
    if (ni + rstride < rows) load_x(ni + rstride, xv);  // next row's x in flight during this one
    // this row's shift / scale for the copy-out (lane columns 4k, k = lane + 32j), also in flight
    const float* shift = mod + ni * mod_stride;  // block 0: shift_msa at 0, scale_msa at HID
    const float* scale = shift + HID;
    float4 sh[J], sc[J];
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {
      sh[jj] = __ldg(reinterpret_cast<const float4*>(shift + 4 * (lane + 32 * jj)));
      sc[jj] = __ldg(reinterpret_cast<const float4*>(scale + 4 * (lane + 32 * jj)));
    }
#pragma unroll
    for (int jj = 0; jj < J; ++jj) {  // 1 + scale, once per row
      sc[jj].x += 1.0f;
      sc[jj].y += 1.0f;
      sc[jj].z += 1.0f;
      sc[jj].w += 1.0f;
    }
    const int64_t tok0 = ni * T + tau0;
    // row statistics of the stored bf16 values in packed f32x2 (even / odd columns), as the block tail
    float2 sum0 = make_float2(0.f, 0.f), sum1 = sum0, sq0 = sum0, sq1 = sum0;
#pragma unroll 2
    for (int blk = 0; blk < HID / 32; ++blk) {
      float acc[4][4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint2 b = sB[(4 * blk + q) * 32 + lane];
#pragma unroll
        for (int i = 0; i < 4; ++i) acc[q][i] = 0.f;
        mma_bf16_16816(acc[q], ahi[0], ahi[1], ahi[2], ahi[3], b.x, b.y);
        mma_bf16_16816(acc[q], alo[0], alo[1], alo[2], alo[3], b.x, b.y);
      }
      // lane columns 32 blk + 8c + {0..7}: column 2q + e <- acc[q][e] (row g), acc[q][2 + e] (row g+8)
      float pb0[8], pb1[8];
      *reinterpret_cast<float4*>(&pb0[0]) = *reinterpret_cast<const float4*>(pos0 + 32 * blk);
      *reinterpret_cast<float4*>(&pb0[4]) = *reinterpret_cast<const float4*>(pos0 + 32 * blk + 4);
      *reinterpret_cast<float4*>(&pb1[0]) = *reinterpret_cast<const float4*>(pos1 + 32 * blk);
      *reinterpret_cast<float4*>(&pb1[4]) = *reinterpret_cast<const float4*>(pos1 + 32 * blk + 4);
      uint32_t r0[4], r1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {  // residual, stored bf16 (bias + pos first)
        const float2 v0 = __fadd2_rn(make_float2(acc[q][0], acc[q][1]), make_float2(pb0[2 * q], pb0[2 * q + 1]));
        const float2 v1 = __fadd2_rn(make_float2(acc[q][2], acc[q][3]), make_float2(pb1[2 * q], pb1[2 * q + 1]));
        r0[q] = pack_bf16(v0.x, v0.y);
        r1[q] = pack_bf16(v1.x, v1.y);
        const float2 f0 = unpack_bf16(r0[q]), f1 = unpack_bf16(r1[q]);
        sum0 = __fadd2_rn(sum0, f0);
        sum1 = __fadd2_rn(sum1, f1);
        sq0 = __ffma2_rn(f0, f0, sq0);
        sq1 = __ffma2_rn(f1, f1, sq1);
      }
      const int off = (blk / 6) * 416 + (blk % 6) * 64;
      *reinterpret_cast<uint4*>(y0 + off) = make_uint4(r0[0], r0[1], r0[2], r0[3]);
      *reinterpret_cast<uint4*>(y1 + off) = make_uint4(r1[0], r1[1], r1[2], r1[3]);
    }
    float s0 = sum0.x + sum0.y, s1 = sum1.x + sum1.y, q0 = sq0.x + sq0.y, q1 = sq1.x + sq1.y;
#pragma unroll
    for (int o = 1; o <= 2; o <<= 1) {
      s0 += __shfl_xor_sync(0xffffffffu, s0, o);
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      q0 += __shfl_xor_sync(0xffffffffu, q0, o);
      q1 += __shfl_xor_sync(0xffffffffu, q1, o);
    }
    if (c == 0) {  // per row: rstd and -mean * rstd (LN(x) = x * rstd - mean * rstd)
      const float mean0 = s0 / HID, mean1 = s1 / HID;
      const float rs0 = rsqrtf(fmaxf(q0 / HID - mean0 * mean0, 0.f) + ln_eps);
      const float rs1 = rsqrtf(fmaxf(q1 / HID - mean1 * mean1, 0.f) + ln_eps);
      sStat[2 * g] = rs0;
      sStat[2 * g + 1] = -mean0 * rs0;
      sStat[2 * (g + 8)] = rs1;
      sStat[2 * (g + 8) + 1] = -mean1 * rs1;
    }
    __syncwarp();  // staged rows and statistics visible to the whole warp
    // copy-out of the residual and of LN + modulate: 8 B (4 columns) per lane and row, each lane on fixed columns 4k
#pragma unroll 2
    for (int row = 0; row < 16; ++row) {
      const float2 r2 = make_float2(sStat[2 * row], sStat[2 * row]);
      const float2 c2 = make_float2(sStat[2 * row + 1], sStat[2 * row + 1]);
#pragma unroll
      for (int jj = 0; jj < J; ++jj) {
        const int k = lane + 32 * jj;
        const uint2 v = *reinterpret_cast<const uint2*>(sY + row * TROW + patch_seg_off<HID>(4 * k));
        // LN(x) * (1 + scale) + shift in packed f32x2, the block tail's epilogue form
        const float2 ya = __ffma2_rn(__ffma2_rn(unpack_bf16(v.x), r2, c2), make_float2(sc[jj].x, sc[jj].y),
                                     make_float2(sh[jj].x, sh[jj].y));
        const float2 yb = __ffma2_rn(__ffma2_rn(unpack_bf16(v.y), r2, c2), make_float2(sc[jj].z, sc[jj].w),
                                     make_float2(sh[jj].z, sh[jj].w));
        *reinterpret_cast<uint2*>(xmod + (tok0 + row) * HID + 4 * k) =
            make_uint2(pack_bf16(ya.x, ya.y), pack_bf16(yb.x, yb.y));
        *reinterpret_cast<uint2*>(xres + (tok0 + row) * HID + 4 * k) = v;  // the residual itself
      }
    }
    __syncwarp();  // staged rows / stats consumed before the next row overwrites them
  }
}

// ============================================================ K4: LayerNorm + adaLN modulate (wide rows)
// xmod = LN(xres) * (1 + scale[slot]) + shift[slot]; one warp per token, lane owns columns
// 128u + 4 lane + {0..3}.  Used where the row is wider than one TMEM accumulator tile (DiT-XL
// hidden 1152), after the gated-residual GEMM.  A warp walks LN_TPW consecutive tokens with the
// next token's row in flight (rows kept as packed bf16); when a
// CTA's 8 * LN_TPW tokens share a slot (STAGE: tokens_per_slot % (8 * LN_TPW) == 0, every DiT
// shape) the slot's shift and 1 + scale are staged in shared memory once per CTA, under the row
// loads.  (The first version loaded them per token after the row reductions and ran one token
// per warp: 12.1-13.2 us for the 8192 tokens of the XL batch under ncu, long-scoreboard bound;
// this one 10.9-12.0, bit-identical.)
constexpr int LN_TPW = 2;   // tokens per warp per group
constexpr int LN_CTAS = 2;  // resident CTAs per SM (the prefetched row doubles the live registers)
template <int HID, bool STAGE>
__global__ void __launch_bounds__(256, LN_CTAS) ln_modulate_kernel(const __nv_bfloat16* __restrict__ xres,
                                                             __nv_bfloat16* __restrict__ xmod,
                                                             const float* __restrict__ shift,
                                                             const float* __restrict__ scale, int64_t vec_stride,
                                                             int64_t M, int T, float ln_eps, int pdl) {
  constexpr int U = HID / 128;
  __shared__ float4 sv[STAGE ? 2 * HID / 4 : 1];  // [shift | 1 + scale] of the CTA's slot
  pdl_wait(pdl);
  if (threadIdx.x == 0) pdl_trigger(pdl);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t groups = (M + 8 * LN_TPW - 1) / (8 * LN_TPW);
  int64_t staged = -1;
  auto load_row = [&](int64_t tok, uint2 (&r)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = *reinterpret_cast<const uint2*>(xres + tok * HID + 128 * u + 4 * lane);
  };
  for (int64_t gi = blockIdx.x; gi < groups; gi += gridDim.x) {
    const int64_t tok0 = gi * 8 * LN_TPW + warp * LN_TPW;
    uint2 raw[U];
    if (tok0 < M) load_row(tok0, raw);
    if constexpr (STAGE) {
      const int64_t slot = gi * 8 * LN_TPW / T;  // block-uniform
      if (slot != staged) {
        __syncthreads();  // the previous slot's readers are done
        const float4* sh4 = reinterpret_cast<const float4*>(shift + slot * vec_stride);
        const float4* sc4 = reinterpret_cast<const float4*>(scale + slot * vec_stride);
        for (int i = threadIdx.x; i < HID / 4; i += blockDim.x) {
          const float4 c = sc4[i];
          sv[i] = sh4[i];
          sv[HID / 4 + i] = make_float4(1.0f + c.x, 1.0f + c.y, 1.0f + c.z, 1.0f + c.w);
        }
        __syncthreads();
        staged = slot;
      }
    }
#pragma unroll 1
    for (int k = 0; k < LN_TPW; ++k) {
      const int64_t tok = tok0 + k;
      if (tok >= M) break;
      uint2 nxt[U];
      if (k + 1 < LN_TPW && tok + 1 < M) load_row(tok + 1, nxt);
      float sum = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float2 a = unpack_bf16(raw[u].x), b = unpack_bf16(raw[u].y);
        sum += (a.x + a.y) + (b.x + b.y);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
      const float mean = sum / HID;
      float var = 0.f;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const float2 a = unpack_bf16(raw[u].x), b = unpack_bf16(raw[u].y);
        var += (a.x - mean) * (a.x - mean);
        var += (a.y - mean) * (a.y - mean);
        var += (b.x - mean) * (b.x - mean);
        var += (b.y - mean) * (b.y - mean);
      }
#pragma unroll
      for (int o = 16; o; o >>= 1) var += __shfl_xor_sync(0xffffffffu, var, o);
      const float rstd = rsqrtf(var / HID + ln_eps);
      const int64_t slot = tok / T;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int n0 = 128 * u + 4 * lane;
        float4 s4, c4;
        if constexpr (STAGE) {
          s4 = sv[n0 / 4];
          c4 = sv[HID / 4 + n0 / 4];
        } else {
          s4 = *reinterpret_cast<const float4*>(shift + slot * vec_stride + n0);
          const float4 c = *reinterpret_cast<const float4*>(scale + slot * vec_stride + n0);
          c4 = make_float4(1.0f + c.x, 1.0f + c.y, 1.0f + c.z, 1.0f + c.w);
        }
        const float2 a = unpack_bf16(raw[u].x), b = unpack_bf16(raw[u].y);
        const float o0 = (a.x - mean) * rstd * c4.x + s4.x;
        const float o1 = (a.y - mean) * rstd * c4.y + s4.y;
        const float o2 = (b.x - mean) * rstd * c4.z + s4.z;
        const float o3 = (b.y - mean) * rstd * c4.w + s4.w;
        *reinterpret_cast<uint2*>(xmod + tok * HID + n0) = make_uint2(pack_bf16(o0, o1), pack_bf16(o2, o3));
      }
      if (k + 1 < LN_TPW) {
#pragma unroll
        for (int u = 0; u < U; ++u) raw[u] = nxt[u];
      }
    }
  }
}

template <int HID>
static cudaError_t launch_ln_hid(const __nv_bfloat16* xres, __nv_bfloat16* xmod, const float* shift,
                                 const float* scale, int64_t vec_stride, int64_t M, int T, float eps,
                                 cudaStream_t st) {
  const int64_t groups = (M + 8 * LN_TPW - 1) / (8 * LN_TPW);
  const unsigned blocks = (unsigned)std::min<int64_t>(groups, 148 * LN_CTAS);
  if (T % (8 * LN_TPW) == 0)
    return launch_kernel(ln_modulate_kernel<HID, true>, dim3(blocks), dim3(256), 0, st, xres, xmod, shift, scale,
                         vec_stride, M, T, eps, g_pdl ? 1 : 0);
  return launch_kernel(ln_modulate_kernel<HID, false>, dim3(blocks), dim3(256), 0, st, xres, xmod, shift, scale,
                       vec_stride, M, T, eps, g_pdl ? 1 : 0);
}

int launch_ln_modulate(const __nv_bfloat16* xres, __nv_bfloat16* xmod, const float* shift, const float* scale,
                       int64_t vec_stride, int64_t M, int N, int tokens_per_slot, float eps, cudaStream_t st) {
  cudaError_t err;
  if (N == 384)
    err = launch_ln_hid<384>(xres, xmod, shift, scale, vec_stride, M, tokens_per_slot, eps, st);
  else if (N == 1152)
    err = launch_ln_hid<1152>(xres, xmod, shift, scale, vec_stride, M, tokens_per_slot, eps, st);
  else
    return SF_ERR_PARAMETER;
  return err == cudaSuccess ? cuda_status() : SF_ERR_CUDA;
}

// ============================================================ K10: final layer (+ CFG + Euler + emit + refill)
// Same layer on the warp-level tensor path (mma.sync m16n8k16, bf16 in, fp32
// accumulate): one warp per 16 consecutive tokens (T % 16 == 0), N = 16 output
// features as two n8 tiles, K = HID in 16-wide steps.  The projection is ~0.4% of the
// network's FLOPs, so the legacy HMMA rate is ample; what matters is that xmod (the
// kernel's only large input, T*HID bf16 per row) streams at HBM rate.  Each warp (up to 12 per
// CTA, one CTA per SM) owns a 16-token tile buffer in shared memory filled by TMA (one box per
// tile) and completing on an mbarrier: the buffer is refilled with the warp's next group as soon
// as the projection has read it, so that load is in flight during the Euler/emit/refill
// epilogue, and the epilogue's own loads (ring row, noise, stage parameters) are issued before
// the tile wait.  The tensor map views a token row as NSEG = HID/192 segments of 192 elements and
// the box is 208 elements wide: TMA zero-fills the 16 out-of-bounds elements, so every
// staged segment is 416 B and consecutive token rows start 64 B apart modulo 128 B -- the
// fragment loads of a quarter-warp (two token rows) are conflict-free without a per-row
// copy.  The weights use the same layout.  K is permuted so that a lane's 16-byte run feeds
// its own fragments (logical k {2c, 2c+1, 2c+8, 2c+9} of a 16-step <-> physical 8c + {0..3},
// the same map for A and B, so the dot products are unchanged).  Fragment ownership after
// the MMA: lane (g = lane/4, c = lane%4) holds tokens g and g+8, features {2c, 2c+1} and
// {8+2c, 9+2c}.
template <int HID>
struct FinalCfg {
  // one tile buffer per warp (refilled right after its fragments are loaded, so the next group's
  // load overlaps this group's epilogue) and up to 12 warps: more warps in flight beat a deeper
  // per-warp ring (ncu: 26.5 vs 29.3 us with two buffers x 8 warps, profiles/r02s3/experiments.md)
  static constexpr int ST = 1;
  static constexpr int MAXW = 12;
  static constexpr int PK = 16;
  static constexpr int SEG = 192, SEG_BOX = 208;       // elements per segment / per staged segment
  static constexpr int NSEG = HID / SEG;
  static constexpr int SROW = SEG_BOX * 2;             // staged segment (bytes)
  static constexpr int TROW = NSEG * SROW;             // staged token / weight row (bytes)
  static constexpr int TILE = 16 * TROW;
  static constexpr int HEAD = ((PK * TROW + PK * 4 + (ST * MAXW + 1) * 8) + 127) / 128 * 128;  // weights, bias, barriers
  static_assert(HID % SEG == 0 && (TROW % 128) == 64, "token rows must alternate 64-byte bank halves");
  // warps per CTA: ST ring buffers per warp of 1 (2 with CFG: cond + uncond rows) tiles
  static int warps(int tiles) {
    const int w = (227 * 1024 - HEAD) / (ST * tiles * TILE);
    return w > MAXW ? MAXW : (w < 1 ? 1 : w);
  }
  static size_t smem(int tiles) { return HEAD + (size_t)warps(tiles) * ST * tiles * TILE; }
};

// [rows, HID] bf16 -> [rows * NSEG, 192] with 208-wide boxes of 16 * NSEG segment rows
template <int HID>
int make_final_map(CUtensorMap* m, const void* p, int64_t rows) {
  using FC = FinalCfg<HID>;
  return make_tmap_bf16_2d(m, p, FC::SEG, (uint64_t)rows * FC::NSEG, FC::SEG, FC::SEG_BOX, 16 * FC::NSEG, 0);
}

template <int HID, bool STREAM>
__global__ void __launch_bounds__(32 * FinalCfg<HID>::MAXW) final_layer_mma_kernel(
    const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmW, const float* __restrict__ fb, int HW,
    int P, int C, int64_t lat_rows, float* __restrict__ eps_out, const int64_t* __restrict__ ctl, int n, int64_t m,
    const double* __restrict__ stage_params, const int64_t* __restrict__ row_info, int cfg, float w,
    const double* __restrict__ w_streams, float* __restrict__ x_ring, const float* __restrict__ noise_in, uint64_t noise_seed, float* __restrict__ frames_out,
    int64_t* __restrict__ frame_ids, int64_t total_tokens, int pdl) {
  using FC = FinalCfg<HID>;
  constexpr int PK = FC::PK, TROW = FC::TROW, SROW = FC::SROW;
  extern __shared__ __align__(128) uint8_t fsm[];  // [PK][TROW] bf16 weights, bias[PK], barriers, tile rings
  float* sbias = reinterpret_cast<float*>(fsm + PK * TROW);
  uint64_t* bars = reinterpret_cast<uint64_t*>(fsm + PK * TROW + PK * 4);  // [warp][2], then the weight barrier
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, c = lane & 3;
  const int WARPS = blockDim.x >> 5;
  const int NT = (STREAM && cfg) ? 2 : 1;  // tiles per group: cond (+ uncond) rows
  uint8_t* ring = fsm + FC::HEAD + (size_t)warp * FC::ST * NT * FC::TILE;
  uint64_t* bar = bars + FC::ST * warp;
  uint64_t* wbar = bars + FC::ST * WARPS;
  if (threadIdx.x == 0) {
    tma_prefetch(&tmX);
    mbar_init(wbar, 1);
    fence_barrier_init();
    mbar_expect_tx(wbar, (uint32_t)(PK * TROW));
    tma_load_2d(fsm, &tmW, wbar, 0, 0);
  }
  if (lane == 0) {
    for (int i = 0; i < FC::ST; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  if (threadIdx.x < PK) sbias[threadIdx.x] = fb[threadIdx.x];
  __syncthreads();
  pdl_wait(pdl);  // (the weight TMA above reads no kernel's output)
  if (threadIdx.x == 0) pdl_trigger(pdl);
  const int gw = HW / P, T = gw * gw;
  int64_t j = 0;
  if constexpr (STREAM) j = ctl[1];
  const uint8_t* wrow0 = fsm + g * TROW + 16 * c;        // feature g      (n-tile 0)
  const uint8_t* wrow1 = fsm + (g + 8) * TROW + 16 * c;  // feature g + 8  (n-tile 1)
  const int64_t groups = total_tokens / 16;
  const int64_t gstride = (int64_t)gridDim.x * WARPS;

  // the 16 token rows of group grp (net rows: cond = lr (+ lat_rows with CFG), uncond = lr) -> buffer b
  auto issue = [&](int64_t grp, int b) {
    if (lane == 0) {
      const int64_t tok0 = grp * 16, lr = tok0 / T;
      const int tau0 = (int)(tok0 % T);
      mbar_expect_tx(&bar[b], (uint32_t)(NT * FC::TILE));
      for (int t = 0; t < NT; ++t) {
        const int64_t net_row = (t == 0 && NT == 2) ? lr + lat_rows : lr;
        tma_load_2d(ring + (b * NT + t) * FC::TILE, &tmX, &bar[b], 0, (int)((net_row * T + tau0) * FC::NSEG));
      }
    }
    __syncwarp();
  };
  // acc[nt][0..1]: token g, features 8nt + 2c + {0,1}; acc[nt][2..3]: token g + 8
  auto project = [&](const uint8_t* tile, float (&acc)[2][4]) {
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[nt][i] = 0.f;
    const uint8_t* a0 = tile + g * TROW + 16 * c;
    const uint8_t* a1 = a0 + 8 * TROW;
    constexpr int NCH = HID / 32;  // 32 K elements (two k-steps) per 16-byte lane run; 6 per segment
#pragma unroll 2
    for (int ch = 0; ch < NCH; ++ch) {
      const int off = (ch / 6) * SROW + (ch % 6) * 64;
      const uint4 xa = *reinterpret_cast<const uint4*>(a0 + off);
      const uint4 xb = *reinterpret_cast<const uint4*>(a1 + off);
      const uint4 b0 = *reinterpret_cast<const uint4*>(wrow0 + off);
      const uint4 b1 = *reinterpret_cast<const uint4*>(wrow1 + off);
      mma_bf16_16816(acc[0], xa.x, xb.x, xa.y, xb.y, b0.x, b0.y);
      mma_bf16_16816(acc[1], xa.x, xb.x, xa.y, xb.y, b1.x, b1.y);
      mma_bf16_16816(acc[0], xa.z, xb.z, xa.w, xb.w, b0.z, b0.w);
      mma_bf16_16816(acc[1], xa.z, xb.z, xa.w, xb.w, b1.z, b1.w);
    }
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const float bl = sbias[8 * nt + 2 * c], bh = sbias[8 * nt + 2 * c + 1];
      acc[nt][0] += bl;
      acc[nt][1] += bh;
      acc[nt][2] += bl;
      acc[nt][3] += bh;
    }
  };

  const int64_t D = (int64_t)C * HW * HW;
  const int64_t gw0 = (int64_t)blockIdx.x * WARPS + warp;
  for (int k = 0; k < FC::ST; ++k)
    if (gw0 + k * gstride < groups) issue(gw0 + k * gstride, k);
  int it = 0;
  for (int64_t grp = gw0; grp < groups; grp += gstride, ++it) {
    const int b = it % FC::ST;
    const int64_t tok0 = grp * 16, lr = tok0 / T;
    const int tau0 = (int)(tok0 % T);
    // this lane's 8 latent elements u = 4 nt + i: token tau0 + g + 8 (i >> 1), feature
    // f = 8 nt + 2c + (i & 1) = (p P + q) C + ch with P = 2, C = 4 (sf_dit_create) -> pixel
    // (2 pi + nt, 2 pj + (c >> 1)) of channel 2 (c & 1) + (i & 1).  The 16 tokens of a group share
    // pi (gw % 16 == 0), so only the group's first token is divided.
    const int pi0 = tau0 / gw, pj0 = tau0 - pi0 * gw;
    const int64_t HW2 = (int64_t)HW * HW;
    int64_t idx[2][4];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        idx[nt][i] = (2 * (c & 1) + (i & 1)) * HW2 + (int64_t)(2 * pi0 + nt) * HW + 2 * (pj0 + g + 8 * (i >> 1)) +
                     (c >> 1);
    // stream epilogue inputs, loaded before the tile wait (velocity.py:125-130 Euler,
    // pipeline.py:172-207 emit / admit)
    bool active = false, admit = false, retiring = false, at_end = false;
    float lam = 0.f, eta = 0.f, span = 1.f, dt = 0.f, wl = w;
    int64_t s = 0;
    float xo[2][4], nz[2][4];
    if constexpr (STREAM) {
      const int64_t stage = row_info[lr * 4 + 0], gen = row_info[lr * 4 + 1];
      active = row_info[lr * 4 + 2] != 0;
      s = row_info[lr * 4 + 3];
      const bool refill_slot = (lr % n) == (j + 1) % n;
      admit = refill_slot && (j + 1 < m);
      retiring = active && (stage + 1 == n);
      if (refill_slot && tau0 == 0 && lane == 0) frame_ids[s] = retiring ? gen : -1;
      if (active) {
        const double* pp = stage_params + stage * SF_PARAM_STRIDE;
        lam = __double2float_rn(pp[SF_P_LAMBDA_T]);
        eta = __double2float_rn(pp[SF_P_ETA_T]);
        span = __double2float_rn(pp[SF_P_SPAN]);
        dt = __double2float_rn(pp[SF_P_DT]);
        at_end = pp[SF_P_AT_END] != 0.0;
      }
      // per-stream guidance: a stream with w == 1 takes the conditional eps as is (apply_cfg is
      // the identity for it, models.py:254-255; row independence makes its cond row exact)
      if (w_streams) wl = (float)w_streams[s];
      const float* xr = x_ring + lr * D;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          xo[nt][i] = active ? xr[idx[nt][i]] : 0.f;
          nz[nt][i] = (admit && noise_in) ? noise_in[s * D + idx[nt][i]] : 0.f;
        }
      if (admit && !noise_in) philox_normal_group8(noise_seed + (uint64_t)s, j + 1, idx, lane, nz);
    }
    if (it == 0) mbar_wait(wbar, 0);  // weights staged
    mbar_wait(&bar[b], (it / FC::ST) & 1);
    float e[2][4];
    project(ring + b * NT * FC::TILE, e);
    if constexpr (STREAM) {
      if (NT == 2 && wl != 1.0f) {
        float eu[2][4];
        project(ring + (b * NT + 1) * FC::TILE, eu);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
#pragma unroll
          for (int i = 0; i < 4; ++i)  // handle_cfg (models.py:288-293)
            e[nt][i] = __fadd_rn(eu[nt][i], __fmul_rn(wl, __fsub_rn(e[nt][i], eu[nt][i])));
      }
    }
    __syncwarp();  // every lane's fragment loads of buffer b are done: refill it
    if (grp + FC::ST * gstride < groups) issue(grp + FC::ST * gstride, b);
#pragma unroll
    for (int nt = 0; nt < 2; ++nt)
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        if constexpr (!STREAM) {
          eps_out[lr * D + idx[nt][i]] = e[nt][i];
        } else {
          float* xr = x_ring + lr * D + idx[nt][i];
          if (active) {
            // velocity.py:125-130 in fp32
            const float x_pred = __fadd_rn(__fmul_rn(lam, xo[nt][i]), __fmul_rn(eta, e[nt][i]));
            const float v = at_end ? 0.0f : __fdiv_rn(__fsub_rn(x_pred, xo[nt][i]), span);
            const float xn = __fadd_rn(xo[nt][i], __fmul_rn(dt, v));
            if (retiring) frames_out[s * D + idx[nt][i]] = xn;
            *xr = admit ? nz[nt][i] : xn;
          } else if (admit) {
            *xr = nz[nt][i];
          }
        }
      }
  }
}

__global__ void stream_reset_f32_kernel(int64_t* ctl, int64_t S, int n, int64_t D, float* x_ring,
                                        const float* noise0, uint64_t noise_seed) {
  const int64_t s = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x)
    x_ring[(s * n) * D + i] = noise0 ? noise0[s * D + i] : philox_normal(noise_seed + (uint64_t)s, 0, i);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    ctl[0] = 0;
    ctl[1] = -1;
  }
}

__global__ void philox_fill_kernel(float* out, int64_t S, int64_t D, uint64_t seed, int64_t gen) {
  const int64_t s = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x)
    out[s * D + i] = philox_normal(seed + (uint64_t)s, gen, i);
}

}  // namespace sf

// ============================================================ handle
using namespace sf;

struct sf_dit {
  sf_dit_config cfg;
  sf_dit_weights w;
  int64_t max_rows;
  int tokens;
  int64_t mod_stride;
  // workspace carve-out
  __nv_bfloat16 *cond, *xres, *xmod, *q, *k, *vt, *attn, *hmid;
  float* mod;
  float* h1;  // conditioning MLP hidden
  // TMA descriptors
  GemmMaps g_ada;                                  // TMA descriptors per GEMM call site
  std::vector<GemmMaps> g_qkv, g_proj, g_fc1, g_fc2;  // [depth]
  AttnMaps attn_maps;
  CUtensorMap fin_x, fin_w;  // final layer: xmod / final weight rows as 208-wide segment boxes
  // One instantiated graph per distinct argument set of sf_dit_stream_step: every pointer and
  // value the capture bakes into a launch is part of the key, so a replay is always the launch
  // sequence an eager call with the same arguments would enqueue.  Owners release their graphs
  // (sf_dit_graph_release) when their buffers are freed; the cache is also capped.
  using GraphKey = std::tuple<const void*, int64_t, int, int64_t, const void*, const void*, const void*, const void*,
                              const void*, const void*, double, const void*, const void*, uint64_t, const void*,
                              const void*>;
  std::map<GraphKey, cudaGraphExec_t> graphs;
  cudaStream_t cap_stream = nullptr;
  // profiling / accounting
  int64_t launch_count = 0;
  bool profiling = false;
  std::vector<cudaEvent_t> prof_events;
  std::vector<int> prof_cls;
};

static constexpr size_t kMaxGraphs = 16;

static int64_t align_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

static int64_t ws_layout(const sf_dit_config& c, int64_t rows, int64_t* off /*[10]*/) {
  const int64_t T = (int64_t)(c.latent_hw / c.patch) * (c.latent_hw / c.patch);
  const int64_t M = rows * T, H = c.hidden;
  const int64_t mod_stride = (int64_t)c.depth * 6 * H + 2 * H;
  const int64_t rows_pad = align_up(rows, 128);
  int64_t o = 0;
  auto take = [&](int i, int64_t bytes) {
    off[i] = o;
    o = align_up(o + bytes, 1024);
  };
  take(0, rows_pad * H * 2);          // cond (bf16 SiLU(c))
  take(1, rows * mod_stride * 4);     // mod (fp32)
  take(2, M * H * 2);                 // xres
  take(3, M * H * 2);                 // xmod
  take(4, M * H * 2);                 // q
  take(5, M * H * 2);                 // k
  take(6, M * H * 2);                 // vt
  take(7, M * H * 2);                 // attn out
  take(8, c.hidden == 384 ? 0 : M * (int64_t)c.mlp_hidden * 2);  // MLP hidden (the DiT-S/2 block tail keeps it on chip)
  take(9, rows * H * 4);                   // conditioning MLP hidden (fp32)
  return o;
}

// Kernel classes for per-launch profiling (sf_dit_profile_step).
enum ProfClass { P_PREPARE = 0, P_COND, P_ADALN, P_PATCH, P_QKV, P_ATTN, P_PROJ, P_FC1, P_FC2, P_FINAL, P_TAIL, P_NCLS };

// Called after every launch: counts launches and, in a profiled step, records
// a CUDA event so each launch's duration can be attributed to its class.
// Programmatic dependent launch for the step's kernels when the batch leaves SMs idle (<= 16
// latent rows: the block tail then fills fewer than half of the 74 CTA pairs); see g_pdl.
struct PdlScope {
  bool prev;
  explicit PdlScope(int64_t rows) : prev(g_pdl) { g_pdl = rows <= 16; }
  ~PdlScope() { g_pdl = prev; }
};

static void mark(sf_dit* h, int cls, cudaStream_t st) {
  h->launch_count++;
  if (!h->profiling) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, st);
  h->prof_events.push_back(e);
  h->prof_cls.push_back(cls);
}

static int run_forward_core(sf_dit* h, int64_t rows, cudaStream_t st) {
  const sf_dit_config& c = h->cfg;
  const int H = c.hidden, T = h->tokens;
  const int64_t M = rows * T;
  int rc;
  // adaLN for every block + final layer at once: mod[rows, mod_stride]
  {
    EpiParams ep{};
    ep.bias = h->w.ada_b;
    ep.out = h->mod;
    ep.ldo = h->mod_stride;
    ep.tokens_per_slot = 1 << 30;
    ep.M = (int)rows;
    if ((rc = launch_gemm(EPI_F32, 256, h->g_ada, (int)rows, (int)h->mod_stride, H, ep, st))) return rc;
    mark(h, P_ADALN, st);
  }
  return SF_OK;
}

static int run_blocks(sf_dit* h, int64_t rows, cudaStream_t st) {
  const sf_dit_config& c = h->cfg;
  const int H = c.hidden, T = h->tokens, hd = H / c.heads;
  const int64_t M = rows * T;
  const int64_t B6 = 6 * (int64_t)H;
  int rc;
  for (int l = 0; l < c.depth; ++l) {
    {
      EpiParams ep{};
      ep.bias = h->w.qkv_b + (int64_t)l * 3 * H;
      ep.heads = c.heads;
      ep.q_scale = 1.0f / sqrtf((float)hd);
      ep.tokens_per_slot = T;
      ep.M = (int)M;
      if ((rc = launch_gemm(EPI_QKV, hd == 64 ? qkv_bn64() : 144, h->g_qkv[l], (int)M, 3 * H, H, ep, st,
                            hd == 64 ? qkv_ctas(H) : 2)))
        return rc;
      mark(h, P_QKV, st);
    }
    if ((rc = launch_attn(h->attn_maps, h->attn, rows, c.heads, T, st))) return rc;
    mark(h, P_ATTN, st);
    // LayerNorm modulate for what follows the block: the next block (shift_msa, scale_msa) or
    // the final layer (shift, scale)
    const float* nxt = l + 1 < c.depth ? h->mod + (l + 1) * B6 : h->mod + c.depth * B6;
    const float* mb = h->mod + l * B6;
    if (H == 384) {
      // DiT-S/2: projection + gated residual + LN + MLP + gated residual + next LN in one
      // kernel on CTA pairs (csrc/block_tail.cu)
      if ((rc = launch_block_tail(h->attn, (const __nv_bfloat16*)h->w.proj_w + (int64_t)l * H * H,
                                  h->w.proj_b + (int64_t)l * H,
                                  (const __nv_bfloat16*)h->w.fc1_w + (int64_t)l * c.mlp_hidden * H,
                                  (const __nv_bfloat16*)h->w.fc2_w + (int64_t)l * H * c.mlp_hidden,
                                  h->w.fc1_b + (int64_t)l * c.mlp_hidden, h->w.fc2_b + (int64_t)l * H, h->xres,
                                  h->xmod, mb + 2 * H, mb + 3 * H, mb + 4 * H, mb + 5 * H, nxt, nxt + H,
                                  h->mod_stride, c.ln_eps, M, T, st)))
        return rc;
      mark(h, P_TAIL, st);
      continue;
    }
    // DiT-XL/2 (1152-wide rows): gated-residual GEMM epilogues + a LayerNorm / modulate pass, with
    // fc1 + GELU in between; every GEMM on 256-row CTA-pair tiles (B split across the pair)
    for (int half = 0; half < 2; ++half) {  // 0: attention proj (gate_msa), 1: MLP (fc1 + GELU, fc2, gate_mlp)
      if (half == 1) {
        EpiParams ep{};
        ep.bias = h->w.fc1_b + (int64_t)l * c.mlp_hidden;
        ep.ldo = c.mlp_hidden;
        ep.tokens_per_slot = T;
        ep.M = (int)M;
        if ((rc = launch_gemm(EPI_GELU, 256, h->g_fc1[l], (int)M, c.mlp_hidden, H, ep, st, 2))) return rc;
        mark(h, P_FC1, st);
      }
      const GemmMaps& gm = half == 0 ? h->g_proj[l] : h->g_fc2[l];
      const int K = half == 0 ? H : c.mlp_hidden;
      const int cls = half == 0 ? P_PROJ : P_FC2;
      EpiParams ep{};
      ep.bias = (half == 0 ? h->w.proj_b : h->w.fc2_b) + (int64_t)l * H;
      ep.xres = h->xres;
      ep.gate = mb + (half == 0 ? 2 : 5) * H;  // gate_msa / gate_mlp
      ep.vec_stride = h->mod_stride;
      ep.tokens_per_slot = T;
      ep.M = (int)M;
      if ((rc = launch_gemm(EPI_RES, 192, gm, (int)M, H, K, ep, st, 2))) return rc;
      mark(h, cls, st);
      const float* ln = half == 0 ? mb + 3 * H : nxt;  // the MLP's (shift_mlp, scale_mlp) / what follows
      if ((rc = launch_ln_modulate(h->xres, h->xmod, ln, ln + H, h->mod_stride, M, H, T, c.ln_eps, st))) return rc;
      mark(h, cls, st);
    }
  }
  return SF_OK;
}

static int launch_cond(sf_dit* h, const RowSrc& src, int64_t rows, cudaStream_t st) {
  const sf_dit_config& c = h->cfg;
  const dim3 grid((unsigned)rows, (unsigned)((c.hidden + 31) / 32));
  if (launch_kernel(cond_h1_kernel, grid, dim3(256), (c.freq_dim + 256) * sizeof(float), st, src, c.hidden, c.freq_dim,
                    (const __nv_bfloat16*)h->w.t_w1t, (const float*)h->w.t_b1, h->h1) != cudaSuccess)
    return SF_ERR_CUDA;
  mark(h, P_COND, st);
  if (launch_kernel(cond_out_kernel, grid, dim3(256), (c.hidden + 64 + 256) * sizeof(float), st, src, c.hidden,
                    (const float*)h->h1, (const __nv_bfloat16*)h->w.t_w2t, (const float*)h->w.t_b2,
                    (const __nv_bfloat16*)h->w.y_wt, (const float*)h->w.y_b, h->cond) != cudaSuccess)
    return SF_ERR_CUDA;
  mark(h, P_COND, st);
  return cuda_status();
}

static int launch_patch(sf_dit* h, const float* x, int64_t lat_rows, int64_t rows, cudaStream_t st) {
  const sf_dit_config& c = h->cfg;
  const int64_t tokens = rows * h->tokens;
  const size_t sm = c.hidden == 384 ? PatchMma<384>::SMEM : PatchMma<1152>::SMEM;
  const int wpb = c.hidden == 384 ? PatchMma<384>::WARPS : PatchMma<1152>::WARPS;
  // CTA c: token group c % TG of latent rows c / TG + k * (CTAs / TG); as many row blocks per
  // group as fill the resident CTA slots (smem-limited: 2 per SM at hidden 384, 1 at 1152)
  const int TG = h->tokens / 16;
  const int64_t slots = c.hidden == 384 ? PatchMma<384>::CPS * 148 : 148;
  int64_t per = std::max<int64_t>(1, slots / TG);
  per = std::min<int64_t>(per, (rows + wpb - 1) / wpb);
  auto kern = c.hidden == 384 ? patch_embed_ln_mma_kernel<384> : patch_embed_ln_mma_kernel<1152>;
  if (launch_kernel(kern, dim3((unsigned)(TG * per)), dim3(32 * wpb), sm, st, x, lat_rows, c.latent_hw, c.patch, c.in_ch,
                    (const __nv_bfloat16*)h->w.patch_w, (const float*)h->w.patch_b, (const float*)h->w.pos_embed,
                    (const float*)h->mod, h->mod_stride, c.ln_eps, h->xres, h->xmod, tokens, g_pdl ? 1 : 0) != cudaSuccess)
    return SF_ERR_CUDA;
  mark(h, P_PATCH, st);
  return cuda_status();
}

// Final layer + Euler/emit/refill (mma.sync kernel).
template <bool STREAM>
static void launch_final(sf_dit* h, int64_t lat_rows, float* eps_out, const int64_t* ctl, int n, int64_t m,
                         const double* stage_params, const int64_t* row_info, int cfg, float w,
                         const double* w_streams, float* x_ring,
                         const float* noise_in, uint64_t noise_seed, float* frames_out, int64_t* frame_ids,
                         int64_t tokens, cudaStream_t st) {
  const sf_dit_config& c = h->cfg;
  const int tiles = (STREAM && cfg) ? 2 : 1;
  const size_t sm = c.hidden == 384 ? FinalCfg<384>::smem(tiles) : FinalCfg<1152>::smem(tiles);
  const int wpb = c.hidden == 384 ? FinalCfg<384>::warps(tiles) : FinalCfg<1152>::warps(tiles);
  // persistent: one CTA per SM (the tile rings fill its shared memory), each warp walks groups
  const unsigned blocks = (unsigned)std::min<int64_t>((tokens / 16 + wpb - 1) / wpb, 148);
  auto fk = c.hidden == 384 ? final_layer_mma_kernel<384, STREAM> : final_layer_mma_kernel<1152, STREAM>;
  launch_kernel(fk, dim3(blocks), dim3(32 * wpb), sm, st, h->fin_x, h->fin_w, (const float*)h->w.final_b, c.latent_hw,
                c.patch, c.in_ch, lat_rows, eps_out, ctl, n, m, stage_params, row_info, cfg, w, w_streams, x_ring,
                noise_in, noise_seed, frames_out, frame_ids, tokens, g_pdl ? 1 : 0);
}

extern "C" {

int64_t sf_dit_workspace_bytes(const sf_dit_config* cfg, int64_t max_rows) {
  int64_t off[10];
  return ws_layout(*cfg, max_rows, off);
}

int sf_dit_create(const sf_dit_config* cfg, const sf_dit_weights* w, int64_t max_rows, void* workspace,
                  int64_t ws_bytes, sf_dit** out) {
  if (!cfg || !w || !out || max_rows < 1) return SF_ERR_PARAMETER;
  const sf_dit_config& c = *cfg;
  // kernels exist for DiT-S/2 (hidden 384, head dim 64) and DiT-XL/2 (hidden 1152, head dim 72), patch 2
  const bool s2 = c.hidden == 384 && c.heads == 6, xl2 = c.hidden == 1152 && c.heads == 16;
  if (!(s2 || xl2) || c.patch != 2 || c.in_ch != 4 || c.latent_hw % 32 || c.mlp_hidden != 4 * c.hidden ||
      c.freq_dim % 2 || c.freq_dim > 1024 || c.embed_dim < 1 || c.embed_dim > 64 || c.depth < 1)
    return SF_ERR_PARAMETER;
  int64_t off[10];
  if (ws_layout(c, max_rows, off) > ws_bytes) return SF_ERR_PARAMETER;
  auto* h = new sf_dit();
  h->cfg = c;
  h->w = *w;
  h->max_rows = max_rows;
  const int gw = c.latent_hw / c.patch;
  h->tokens = gw * gw;
  const int H = c.hidden;
  h->mod_stride = (int64_t)c.depth * 6 * H + 2 * H;
  uint8_t* base = (uint8_t*)workspace;
  h->cond = (__nv_bfloat16*)(base + off[0]);
  h->mod = (float*)(base + off[1]);
  h->xres = (__nv_bfloat16*)(base + off[2]);
  h->xmod = (__nv_bfloat16*)(base + off[3]);
  h->q = (__nv_bfloat16*)(base + off[4]);
  h->k = (__nv_bfloat16*)(base + off[5]);
  h->vt = (__nv_bfloat16*)(base + off[6]);
  h->attn = (__nv_bfloat16*)(base + off[7]);
  h->hmid = (__nv_bfloat16*)(base + off[8]);
  h->h1 = (float*)(base + off[9]);
  const int64_t M = max_rows * h->tokens;
  const int64_t rows_pad = align_up(max_rows, 128);
  int rc = SF_OK;
  rc |= make_operand_maps(&h->g_ada, h->cond, rows_pad, H, w->ada_w, h->mod_stride, 256);
  h->g_qkv.resize(c.depth);
  h->g_proj.resize(c.depth);
  h->g_fc1.resize(c.depth);
  h->g_fc2.resize(c.depth);
  for (int l = 0; l < c.depth; ++l) {
    const __nv_bfloat16* qkv = (const __nv_bfloat16*)w->qkv_w + (int64_t)l * 3 * H * H;
    const __nv_bfloat16* proj = (const __nv_bfloat16*)w->proj_w + (int64_t)l * H * H;
    const __nv_bfloat16* fc1 = (const __nv_bfloat16*)w->fc1_w + (int64_t)l * c.mlp_hidden * H;
    const __nv_bfloat16* fc2 = (const __nv_bfloat16*)w->fc2_w + (int64_t)l * H * c.mlp_hidden;
    const int hd = H / c.heads;
    rc |= make_operand_maps(&h->g_qkv[l], h->xmod, M, H, qkv, 3 * H, hd == 64 ? qkv_bn64() : 144,
                            hd == 64 ? qkv_ctas(H) : 2);
    rc |= make_qkv_out_maps(&h->g_qkv[l], h->q, h->k, h->vt, max_rows, c.heads, h->tokens, hd);
    if (H != 384) {  // DiT-XL/2 MLP + projection as GEMMs: RES epilogue (128-wide tiles) + LayerNorm pass
      rc |= make_operand_maps(&h->g_fc1[l], h->xmod, M, H, fc1, c.mlp_hidden, 256, 2);
      rc |= make_out_map32(&h->g_fc1[l].d[0], h->hmid, M, c.mlp_hidden);  // 256-wide GELU tiles: 32-column chunks
      rc |= make_operand_maps(&h->g_proj[l], h->attn, M, H, proj, H, 192, 2);
      rc |= make_out_map(&h->g_proj[l].d[0], h->xres, M, H);
      rc |= make_operand_maps(&h->g_fc2[l], h->hmid, M, c.mlp_hidden, fc2, H, 192, 2);
      rc |= make_out_map(&h->g_fc2[l].d[0], h->xres, M, H);
    }
  }
  rc |= make_attn_maps(&h->attn_maps, h->q, h->k, h->vt, max_rows, c.heads, h->tokens, c.hidden / c.heads);
  if (c.hidden == 384) {
    rc |= make_final_map<384>(&h->fin_x, h->xmod, max_rows * h->tokens);
    rc |= make_final_map<384>(&h->fin_w, w->final_w, 16);
  } else {
    rc |= make_final_map<1152>(&h->fin_x, h->xmod, max_rows * h->tokens);
    rc |= make_final_map<1152>(&h->fin_w, w->final_w, 16);
  }
  if (rc != SF_OK) {
    delete h;
    return SF_ERR_CUDA;
  }
  // kernel attributes (dynamic smem > 48 KB) set once, outside any graph capture
  if (prepare_gemm_kernels() != SF_OK || prepare_attn_kernel() != SF_OK) {
    delete h;
    return SF_ERR_CUDA;
  }
  cudaFuncSetAttribute(patch_embed_ln_mma_kernel<384>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       PatchMma<384>::SMEM);
  cudaFuncSetAttribute(patch_embed_ln_mma_kernel<1152>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       PatchMma<1152>::SMEM);
  cudaFuncSetAttribute(final_layer_mma_kernel<384, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)std::max(FinalCfg<384>::smem(1), FinalCfg<384>::smem(2)));
  cudaFuncSetAttribute(final_layer_mma_kernel<384, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)FinalCfg<384>::smem(1));
  cudaFuncSetAttribute(final_layer_mma_kernel<1152, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)std::max(FinalCfg<1152>::smem(1), FinalCfg<1152>::smem(2)));
  cudaFuncSetAttribute(final_layer_mma_kernel<1152, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       (int)FinalCfg<1152>::smem(1));
  *out = h;
  return cuda_status();
}

int sf_dit_destroy(sf_dit* h) {
  if (!h) return SF_OK;
  for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
  if (h->cap_stream) cudaStreamDestroy(h->cap_stream);
  delete h;
  return SF_OK;
}

int sf_dit_forward(sf_dit* h, int64_t rows, const float* x, const double* ts, const double* row_embs, float* eps_out,
                   void* stream) {
  if (!h || rows < 1 || rows > h->max_rows) return SF_ERR_PARAMETER;
  cudaStream_t st = (cudaStream_t)stream;
  const sf_dit_config& c = h->cfg;
  const PdlScope pdl(rows);
  RowSrc src{nullptr, ts, rows, 0, row_embs, nullptr, c.embed_dim, g_pdl ? 1 : 0};
  int rc;
  if ((rc = launch_cond(h, src, rows, st))) return rc;
  if ((rc = run_forward_core(h, rows, st))) return rc;
  if ((rc = launch_patch(h, x, rows, rows, st))) return rc;
  if ((rc = run_blocks(h, rows, st))) return rc;
  const int64_t tokens = rows * h->tokens;
  launch_final<false>(h, rows, eps_out, nullptr, 1, 1, nullptr, nullptr, 0, 1.0f, nullptr, nullptr, nullptr, 0, nullptr,
                      nullptr, tokens, st);
  return cuda_status();
}

static int stream_step_launches(sf_dit* h, int64_t* ctl, int64_t S, int32_t n, int64_t m, const double* stage_params,
                                int64_t* row_info, double* row_t, float* x_ring, const double* emb, const double* neg,
                                double w, const double* w_streams, const float* noise_in, uint64_t noise_seed,
                                float* frames_out, int64_t* frame_ids, cudaStream_t st) {
  const sf_dit_config& c = h->cfg;
  const int64_t R = S * n;
  const int cfg = (w != 1.0) ? 1 : 0;
  const int64_t rows = cfg ? 2 * R : R;
  const PdlScope pdl(rows);
  int rc;
  if ((rc = sf_stream_prepare(ctl, S, n, m, stage_params, row_info, row_t, st))) return rc;
  mark(h, P_PREPARE, st);
  RowSrc src{row_info, row_t, R, cfg, emb, neg, c.embed_dim, g_pdl ? 1 : 0};
  if ((rc = launch_cond(h, src, rows, st))) return rc;
  if ((rc = run_forward_core(h, rows, st))) return rc;
  if ((rc = launch_patch(h, x_ring, R, rows, st))) return rc;
  if ((rc = run_blocks(h, rows, st))) return rc;
  const int64_t tokens = R * h->tokens;
  launch_final<true>(h, R, nullptr, ctl, n, m, stage_params, row_info, cfg, (float)w, w_streams, x_ring, noise_in,
                     noise_seed, frames_out, frame_ids, tokens, st);
  mark(h, P_FINAL, st);
  return cuda_status();
}

int sf_dit_profile_step(sf_dit* h, int64_t* ctl, int64_t S, int32_t n, int64_t m, const double* stage_params,
                        int64_t* row_info, double* row_t, float* x_ring, const double* emb, const double* neg,
                        double w, const double* w_streams, const float* noise_in, uint64_t noise_seed,
                        float* frames_out, int64_t* frame_ids,
                        float* ms_per_class, int32_t* launches_per_class, void* stream) {
  if (!h || S < 1 || n < 1 || m < 1 || !ms_per_class || !launches_per_class) return SF_ERR_PARAMETER;
  const int64_t rows = (w != 1.0 ? 2 : 1) * S * n;
  if (rows > h->max_rows) return SF_ERR_PARAMETER;
  cudaStream_t st = (cudaStream_t)stream;
  h->profiling = true;
  h->prof_events.clear();
  h->prof_cls.clear();
  cudaEvent_t start;
  cudaEventCreate(&start);
  cudaEventRecord(start, st);
  int rc = stream_step_launches(h, ctl, S, n, m, stage_params, row_info, row_t, x_ring, emb, neg, w, w_streams, noise_in,
                                noise_seed, frames_out, frame_ids, st);
  h->profiling = false;
  if (cudaStreamSynchronize(st) != cudaSuccess) rc = SF_ERR_CUDA;
  for (int c = 0; c < P_NCLS; ++c) {
    ms_per_class[c] = 0.f;
    launches_per_class[c] = 0;
  }
  cudaEvent_t prev = start;
  for (size_t i = 0; i < h->prof_events.size(); ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, prev, h->prof_events[i]);
    ms_per_class[h->prof_cls[i]] += ms;
    launches_per_class[h->prof_cls[i]] += 1;
    prev = h->prof_events[i];
  }
  for (auto e : h->prof_events) cudaEventDestroy(e);
  cudaEventDestroy(start);
  h->prof_events.clear();
  h->prof_cls.clear();
  return rc;
}

int64_t sf_dit_launch_count(const sf_dit* h) { return h ? h->launch_count : -1; }

int sf_dit_stream_step(sf_dit* h, int64_t* ctl, int64_t S, int32_t n, int64_t m, const double* stage_params,
                       int64_t* row_info, double* row_t, float* x_ring, const double* emb, const double* neg, double w,
                       const double* w_streams, const float* noise_in, uint64_t noise_seed, float* frames_out, int64_t* frame_ids,
                       int32_t use_graph, void* stream) {
  if (!h || S < 1 || n < 1 || m < 1) return SF_ERR_PARAMETER;
  const int64_t rows = (w != 1.0 ? 2 : 1) * S * n;
  if (rows > h->max_rows) return SF_ERR_PARAMETER;
  cudaStream_t st = (cudaStream_t)stream;
  if (!use_graph)
    return stream_step_launches(h, ctl, S, n, m, stage_params, row_info, row_t, x_ring, emb, neg, w, w_streams, noise_in,
                                noise_seed, frames_out, frame_ids, st);
  const sf_dit::GraphKey key{(const void*)ctl, S,          n, m, (const void*)stage_params, (const void*)row_info,
                             (const void*)row_t, (const void*)x_ring, (const void*)emb, (const void*)neg, w,
                             (const void*)w_streams, (const void*)noise_in, noise_seed, (const void*)frames_out,
                             (const void*)frame_ids};
  auto it = h->graphs.find(key);
  if (it == h->graphs.end()) {
    if (h->graphs.size() >= kMaxGraphs) {  // cap: drop every cached graph (re-captured on next use)
      cudaStreamSynchronize(st);
      for (auto& kv : h->graphs) cudaGraphExecDestroy(kv.second);
      h->graphs.clear();
    }
    // Capture on a private stream (the caller's may be the legacy default
    // stream, which cannot be captured); the graph is launched on the caller's.
    if (!h->cap_stream && cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
      return SF_ERR_CUDA;
    cudaGraph_t g;
    if (cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal) != cudaSuccess) return SF_ERR_CUDA;
    int rc = stream_step_launches(h, ctl, S, n, m, stage_params, row_info, row_t, x_ring, emb, neg, w, w_streams, noise_in,
                                  noise_seed, frames_out, frame_ids, h->cap_stream);
    cudaError_t e = cudaStreamEndCapture(h->cap_stream, &g);
    if (rc != SF_OK || e != cudaSuccess) return rc != SF_OK ? rc : SF_ERR_CUDA;
    cudaGraphExec_t ge;
    e = cudaGraphInstantiate(&ge, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return SF_ERR_CUDA;
    it = h->graphs.emplace(key, ge).first;
  }
  return cudaGraphLaunch(it->second, st) == cudaSuccess ? SF_OK : SF_ERR_CUDA;
}

int sf_dit_graph_release(sf_dit* h, const int64_t* ctl) {
  if (!h) return SF_ERR_PARAMETER;
  bool any = false;
  for (auto it = h->graphs.begin(); it != h->graphs.end();) {
    if (std::get<0>(it->first) == (const void*)ctl) {
      if (!any) cudaDeviceSynchronize();  // a replay of this graph may still be in flight
      any = true;
      cudaGraphExecDestroy(it->second);
      it = h->graphs.erase(it);
    } else {
      ++it;
    }
  }
  return SF_OK;
}

int64_t sf_dit_graph_count(const sf_dit* h) { return h ? (int64_t)h->graphs.size() : -1; }

int sf_dit_stream_reset(int64_t* ctl, int64_t S, int32_t n, int64_t D, float* x_ring, const float* noise0,
                        uint64_t noise_seed, void* stream) {
  if (S < 1 || n < 1 || D < 1 || S > 65535) return SF_ERR_PARAMETER;
  dim3 grid(16, (unsigned)S);
  stream_reset_f32_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(ctl, S, n, D, x_ring, noise0, noise_seed);
  return cuda_status();
}

int sf_philox_normal(float* out, int64_t S, int64_t D, uint64_t seed, int64_t gen, void* stream) {
  if (S < 1 || D < 1 || S > 65535) return SF_ERR_PARAMETER;
  dim3 grid(16, (unsigned)S);
  philox_fill_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(out, S, D, seed, gen);
  return cuda_status();
}


int sf_dit_mod_stride(const sf_dit_config* c) { return c->depth * 6 * c->hidden + 2 * c->hidden; }

}  // extern "C"

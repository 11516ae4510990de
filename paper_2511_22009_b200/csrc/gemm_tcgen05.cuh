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
// epilogue of tile i overlaps the main loop of tile i+1.  Epilogue outputs are
// staged per warp in 128B-swizzled smem (32 rows x 64 columns, double-buffered)
// and written with TMA bulk stores, so HBM sees full-line writes.
#pragma once
#include "sf_ptx.cuh"

namespace sf {

#ifndef SF_GEMM_TRACE
#define SF_GEMM_TRACE 0  // diagnostics: clock64 timeline of CTA 0 (sf_gemm_trace_read)
#endif
#if SF_GEMM_TRACE
__device__ long long g_gemm_trace[8 * 64];
__device__ unsigned long long g_gemm_cta_end[1024];  // %globaltimer at each CTA's end (ns, GPU-wide clock)
#define GTR(role, idx)                                                               \
  do {                                                                               \
    if (blockIdx.x == 0 && (idx) < 64) g_gemm_trace[(role) * 64 + (idx)] = clock64(); \
  } while (0)
#else
#define GTR(role, idx) \
  do {                 \
  } while (0)
#endif

enum EpiKind : int {
  EPI_F32 = 0,     // out f32 [M, ldo]  = acc + bias
  EPI_BF16 = 1,    // out bf16 [M, ldo] = acc + bias
  EPI_GELU = 2,    // out bf16 [M, ldo] = gelu_tanh(acc + bias)
  EPI_QKV = 3,     // scatter to Q,K [rows, H, T, 64] bf16 and V^T [rows, H, 64, T] fp16; Q pre-scaled
  EPI_RES_LN = 4,  // x += gate*(acc+bias) (bf16 residual); xmod = LN(x)*(1+scale)+shift
  EPI_RES = 5,     // x += gate*(acc+bias) only (wide rows; LayerNorm runs as its own pass)
  EPI_RES_LN2 = 6, // RES_LN over a cluster of N/BN CTAs (BN = 192): each CTA owns a column slice of
                   // the same 128 rows, LayerNorm row statistics meet in distributed shared memory
};
constexpr int XCH_CL = 2;  // RES_LN2 cluster size (384-wide rows / 192-column tiles)

struct EpiParams {
  const float* bias;  // [N]
  void* out;          // EPI_F32 direct stores
  int64_t ldo;
  // EPI_QKV
  int heads;
  float q_scale;
  // EPI_RES_LN
  const __nv_bfloat16* xres;  // [M, N] residual stream (read; the update goes out through d[0])
  const float* gate;          // per-slot vectors: ptr + slot * vec_stride
  const float* shift;
  const float* scale;
  int64_t vec_stride;
  float ln_eps;
  // common
  int tokens_per_slot;  // rows of one latent (1024); tiles never straddle a slot
  int M;                // valid rows (tail rows of the last tile are masked)
  int pdl;              // launched with programmatic serialisation (sf_internal.h g_pdl)
};

// TMA descriptors: A, B operands and up to three outputs
//   BF16/GELU: d[0] = out [M, N]          (box 64 x 32, SW128)
//   QKV:       d[0] = Q [R*H*T, 64], d[1] = K (box 64 x 32, SW128),
//              d[2] = V^T [R*H*64, T]     (box 32 x 64, SW64)
//   RES_LN:    d[0] = xres, d[1] = xmod [M, N] (box 64 x 32, SW128)
struct GemmMaps {
  CUtensorMap a, b, d[3];
};

template <int BN, int EPI_WARPS, int KIND, int CTAS = 1>
struct GemmCfg {
  static constexpr int BM = 128;
  static constexpr int BK = BN > 256 ? 32 : 64;  // K elements per stage (64 B / 128 B rows)
  static constexpr int SWZ = BK * 2;             // swizzle width of the operand tiles (bytes)
  static constexpr int A_BYTES = BM * BK * 2;
  // CTAS = 2: a cluster pair computes 256 x BN tiles with cta_group::2 MMAs; each CTA
  // holds its 128 A rows and BN/2 B rows (the pair MMA reads B from both), so per 128-row
  // tile a CTA pulls half the B bytes from L2 (the DiT-XL/2 GEMMs, K = 1152 / 4608: their
  // single-CTA tiles are fed at ~64-85 FLOP per L2 byte).  For the DiT-S/2 QKV (K = 384,
  // BN = 192) the pair keeps one column slice n for its whole life and its half of that B
  // slice stays RESIDENT in smem (K = KB_RES * BK), so only A streams through the ring: per
  // 128 x BN tile a CTA pulls 96 KB of A from L2 instead of 96 KB of A + 144 KB of B (the
  // single-CTA QKV GEMM waits on its operand ring, not on the tensor pipe: profiles/r02).
  static constexpr bool B_RES = CTAS == 2 && KIND == EPI_QKV && BN == 192;
  static constexpr int KB_RES = 6;  // resident K blocks (K = 384, the DiT-S/2 hidden size)
  static constexpr int B_ROWS = BN / CTAS;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int BRES_BYTES = B_RES ? KB_RES * B_BYTES : 0;
  static constexpr int STAGE_BYTES = B_RES ? A_BYTES : A_BYTES + B_BYTES;
  static constexpr int MMA_N = BN > 256 ? BN / 2 : BN;  // UMMA N <= 256
  static constexpr int N_SPLIT = BN / MMA_N;
  static constexpr int B_BOX = B_ROWS > 256 ? B_ROWS / 2 : B_ROWS;  // TMA box rows <= 256
  static constexpr int ACC_STAGES = 2 * BN <= 512 ? 2 : 1;
  static constexpr int ACC_STRIDE = BN <= 128 ? 128 : 256;  // column offset between accumulator stages
  static constexpr int TMEM_COLS = ACC_STAGES == 2 ? (BN <= 128 ? 256 : 512) : (BN <= 256 ? 256 : 512);
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  // QKV with 8 epilogue warps: two 4-warp groups take alternate tiles (group g drains
  // accumulator stage g) instead of splitting a tile's columns
  static constexpr int TILE_GROUPS = (KIND == EPI_QKV && BN == 192 && EPI_WARPS == 8) ? 2 : 1;
  static constexpr int RED_BYTES = 2 * EPI_WARPS * 32 * 4;  // LN partial sums of the warps sharing a row
  static constexpr int VEC_BYTES = 2 * 4 * BN * 4;          // per-tile column vectors, double-buffered
  // per-warp output staging, double-buffered: 32 rows x 128 B (SW128), or 32 x 64 B (SW64) with 12 warps
  // (RES_LN: a 3-deep ring per warp; residual chunks are TMA-loaded into it and
  // overwritten in place by the updated residual before its TMA store)
  // (head dim 72 QKV, BN = 144: 32 x 144 B Q/K rows or 72 x 64 B V^T rows per buffer)
  static constexpr bool LN_RING = KIND == EPI_RES_LN || KIND == EPI_RES_LN2;  // 32-column SW64 chunks
  static constexpr bool NARROW = LN_RING || ((KIND == EPI_BF16 || KIND == EPI_GELU) && EPI_WARPS == 16);
  static constexpr int OUT_BUF = BN == 144 ? 5120 : NARROW ? 2048 : 4096;
  // RES_LN(2): one buffer per chunk; QKV (head dim 64): 3 store buffers per warp
  // RES: one 64-column residual chunk per buffer, as many buffers as the warp has chunks (a
  // second buffer for one-chunk warps would only cost operand-ring stages: 4 -> 6 at BN = 192);
  // GELU at BN = 256: one buffer per warp (its two 32-column chunks take turns), 4 -> 5 stages
  static constexpr int OUT_NBUF = KIND == EPI_F32                                  ? 0  // writes fp32 directly
                                  : LN_RING                                        ? BN / (EPI_WARPS / 4) / 32
                                  : KIND == EPI_RES                                ? BN / (EPI_WARPS / 4) / 64
                                  : (KIND == EPI_QKV && BN == 192 && TILE_GROUPS == 1) ? 3
                                  : (KIND == EPI_GELU && BN == 256)                 ? 1  // 5 stages, not 4
                                                                                   : 2;
  static constexpr int OUT_BYTES = EPI_WARPS * OUT_NBUF * OUT_BUF;
  static constexpr int RBAR_BYTES = EPI_WARPS * 4 * 8;  // residual-chunk barriers (one per staging buffer)
  // RES_LN2 exchange: [tile parity][pass][source CTA][column group][128 rows] floats
  static constexpr int XCH_BYTES = KIND == EPI_RES_LN2 ? 2 * 2 * XCH_CL * 2 * 128 * 4 : 0;
  static constexpr int FIXED = 1024 + 256 + RED_BYTES + VEC_BYTES + OUT_BYTES + RBAR_BYTES + XCH_BYTES;
  static constexpr int STAGES_FIT = (227 * 1024 - FIXED - BRES_BYTES) / STAGE_BYTES;
  static constexpr int STAGES = STAGES_FIT > 8 ? 8 : STAGES_FIT;
  static constexpr int SMEM_BYTES = FIXED + STAGES * STAGE_BYTES + BRES_BYTES;
  static_assert(STAGES >= 3, "pipeline too shallow");
  static_assert(MMA_N % 16 == 0 && MMA_N <= 256, "bad MMA N");
  static_assert(B_BOX <= 256, "bad box");
  static_assert(EPI_WARPS == 4 || EPI_WARPS == 8 || EPI_WARPS == 12 || EPI_WARPS == 16, "epilogue warps");
  static_assert(TILE_GROUPS == 1 || ACC_STAGES == 2, "tile groups drain one accumulator stage each");
};

__device__ __forceinline__ float gelu_tanh(float x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  float u = k0 * (x + k1 * x * x * x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * x * (1.0f + t);
}

// tanh-GELU of a pair: packed f32x2 arithmetic (FFMA2/FMUL2) around two MUFU.TANH.
__device__ __forceinline__ float2 gelu_tanh2(float2 x) {
  const float k0 = 0.7978845608028654f, k1 = 0.044715f;
  const float2 x2 = __fmul2_rn(x, x);
  const float2 t = __ffma2_rn(x2, make_float2(k0 * k1, k0 * k1), make_float2(k0, k0));  // k0 (1 + k1 x^2)
  const float2 u = __fmul2_rn(x, t);
  float2 th;
  asm("tanh.approx.f32 %0, %1;" : "=f"(th.x) : "f"(u.x));
  asm("tanh.approx.f32 %0, %1;" : "=f"(th.y) : "f"(u.y));
  const float2 h = __fmul2_rn(x, make_float2(0.5f, 0.5f));
  return __ffma2_rn(h, th, h);  // 0.5 x (1 + tanh u)
}

__device__ __forceinline__ uint4 pack8_bf16(const float* v) {
  return make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
}

// K-major operand descriptor for a 64 B (SW64) or 128 B (SW128) swizzled tile.
template <int SWZ>
__device__ __forceinline__ uint64_t kmajor_desc(uint32_t smem_addr) {
  if constexpr (SWZ == 128) return sw128_kmajor_desc(smem_addr);
  return (uint64_t)((smem_addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(512 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)4 << 61);
}

// Per-warp output staging: a 32-row tile in the TMA swizzle layout, 128-byte
// rows (SW128: 16-byte chunk c of row r at c ^ (r & 7)) or 64-byte rows (SW64:
// chunk c at c ^ ((r >> 1) & 3)).  Lane = row.
template <int BUF, int NB = 2>
struct OutStageT {
  uint8_t* base;     // this warp's NB x BUF bytes
  uint32_t count;    // chunks issued so far by this warp (buffer = count % NB)
  __device__ __forceinline__ uint8_t* acquire(uint32_t lane) {
    if (count >= NB && lane == 0) bulk_wait_read<NB - 1>();  // the store issued NB chunks ago left this buffer
    __syncwarp();
    return base + (count % NB) * BUF;
  }
  __device__ __forceinline__ static void put16(uint8_t* buf, uint32_t row, uint32_t chunk, uint4 v) {
    if constexpr (BUF == 4096)
      *reinterpret_cast<uint4*>(buf + row * 128 + ((chunk ^ (row & 7)) * 16)) = v;
    else
      *reinterpret_cast<uint4*>(buf + row * 64 + ((chunk ^ ((row >> 1) & 3)) * 16)) = v;
  }
  __device__ __forceinline__ void release(uint32_t lane, const CUtensorMap* map, uint8_t* buf, int c0, int c1,
                                          bool store) {
    fence_proxy_async_smem();
    __syncwarp();
    if (lane == 0) {
      if (store) {
        tma_store_2d(map, buf, c0, c1);
      }
      bulk_commit();
    }
    ++count;
  }
};

template <int BN, int KIND, int EPI_WARPS, int CTAS = 1>
__global__ void __launch_bounds__(GemmCfg<BN, EPI_WARPS, KIND, CTAS>::THREADS, 1)
    gemm_bf16_tcgen05(const __grid_constant__ GemmMaps maps, int N, int K, EpiParams ep) {
  using C = GemmCfg<BN, EPI_WARPS, KIND, CTAS>;
  constexpr bool TWO_SM = CTAS == 2;
  static_assert(!TWO_SM || (BN <= 256 && KIND != EPI_RES_LN2), "2-SM tiles: BN <= 256");
  extern __shared__ uint8_t smem_raw[];
  // 1024-align by offsetting into the shared array (keeps the pointer in the shared window: LDS/STS, not generic)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sOut = smem;                             // [EPI_WARPS][OUT_NBUF][OUT_BUF]   (1024-aligned)
  uint8_t* sA = sOut + C::OUT_BYTES;                // [STAGES][A_BYTES]
  uint8_t* sB = sA + C::STAGES * C::A_BYTES;        // [STAGES][B_BYTES] (B_RES: [KB_RES][B_BYTES])
  float* red = reinterpret_cast<float*>(sB + (C::B_RES ? C::BRES_BYTES : C::STAGES * C::B_BYTES));  // [2][8 warps][32]
  float* vecs = red + C::RED_BYTES / 4;                                // [2][4][BN]
  uint64_t* bars = reinterpret_cast<uint64_t*>(vecs + C::VEC_BYTES / 4);
  uint64_t* full = bars;
  uint64_t* empty = bars + C::STAGES;
  uint64_t* tfull = bars + 2 * C::STAGES;
  uint64_t* tempty = tfull + C::ACC_STAGES;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tempty + C::ACC_STAGES);
  uint64_t* rbar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(bars) + 256);  // [EPI_WARPS][3]
  float* xch = reinterpret_cast<float*>(rbar + EPI_WARPS * 4);  // RES_LN2 exchange
  uint64_t* xbar = tempty + C::ACC_STAGES + 1;                   // RES_LN2: [parity][pass], one arrive per CTA
  uint64_t* bfull = xbar;                                        // B_RES: both halves of the resident B landed (leader)
  constexpr bool CLUSTER = KIND == EPI_RES_LN2;

  const uint32_t warp = warp_id();
  const uint32_t lane = threadIdx.x & 31;
  const int num_n = N / BN;
  const int num_m = (ep.M + C::BM - 1) / C::BM;
  const int total = num_m * num_n;
  const int num_kb = K / C::BK;
  // Tile sequence: default = all (m, n) tiles N-fastest over the grid; cluster mode =
  // the cluster walks row tiles m, CTA rank r of the cluster owns column slice n = r.
  // 2-SM mode: the pair walks (row-pair, n) tiles, CTA rank r owns rows 2*pair + r.
  const uint32_t crank = (CLUSTER || TWO_SM) ? cluster_ctarank() : 0u;
  const bool leader = crank == 0;
  const int num_mp = (num_m + 1) / 2;
  const int t_first = CLUSTER ? (int)(blockIdx.x / XCH_CL) : TWO_SM ? (int)(blockIdx.x / 2) : (int)blockIdx.x;
  const int t_stride = CLUSTER ? (int)(gridDim.x / XCH_CL) : TWO_SM ? (int)(gridDim.x / 2) : (int)gridDim.x;
  const int t_limit = CLUSTER ? num_m : TWO_SM ? num_mp * num_n : total;
  auto tile_m0 = [&](int tile) {
    return CLUSTER ? tile * C::BM : TWO_SM ? (2 * (tile / num_n) + (int)crank) * C::BM : (tile / num_n) * C::BM;
  };
  auto tile_n0 = [&](int tile) { return CLUSTER ? (int)crank * BN : (tile % num_n) * BN; };
  // epilogue -> MMA accumulator release (2-SM: one arrival per epilogue warp of both CTAs on the
  // leader's barrier, cta-scope semantics as in the block tail: the TMEM reads are complete
  // (tcgen05.wait::ld) before the arrive)
  auto acc_release = [&](uint32_t a) {
    tc_fence_before();
    if constexpr (TWO_SM) {
      __syncwarp();
      if ((threadIdx.x & 31) == 0)
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(mapa_shared(smem_u32(&tempty[a]), 0))
                     : "memory");
      __syncwarp();
    } else {
      mbar_arrive(&tempty[a]);
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch(&maps.a);
    tma_prefetch(&maps.b);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < C::ACC_STAGES; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], TWO_SM ? CTAS * EPI_WARPS / C::TILE_GROUPS : EPI_WARPS * 32 / C::TILE_GROUPS);
    }
    if constexpr (C::B_RES) mbar_init(bfull, 1);
    if constexpr (KIND == EPI_RES_LN || KIND == EPI_RES || KIND == EPI_RES_LN2)
      for (int i = 0; i < EPI_WARPS * 4; ++i) mbar_init(&rbar[i], 1);
    if constexpr (CLUSTER)
      for (int i = 0; i < 4; ++i) mbar_init(&xbar[i], XCH_CL * EPI_WARPS * 32);
    fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (TWO_SM)
      tmem_alloc_2sm<C::TMEM_COLS>(tmem_holder);
    else
      tmem_alloc<C::TMEM_COLS>(tmem_holder);
  }
  if constexpr (CLUSTER || TWO_SM) cluster_sync_all();  // peers' barriers initialised before any remote arrive
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;
  if (threadIdx.x == 0) pdl_trigger(ep.pdl);  // the next kernel's CTAs may start their prologue

  if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (ring continues across tiles)
      uint32_t it = 0;
      if constexpr (C::B_RES) {
        // the pair's column slice is fixed (the host sizes the grid to a multiple of N / BN
        // pairs): this CTA's half of B, all K blocks, once; both halves complete on the leader.
        // The weights are no kernel's output, so they load before the dependency wait, under the
        // previous kernel's tail.
        if (t_first < t_limit) {
          if (leader) mbar_expect_tx(bfull, 2 * C::BRES_BYTES);
          for (int kb = 0; kb < C::KB_RES; ++kb)
            tma_load_2d_2sm(sB + kb * C::B_BYTES, &maps.b, mapa_shared(smem_u32(bfull), 0), kb * C::BK,
                            tile_n0(t_first) + (int)crank * C::B_ROWS);
        }
      }
      pdl_wait(ep.pdl);
      for (int tile = t_first; tile < t_limit; tile += t_stride) {
        const int m0 = tile_m0(tile), n0 = tile_n0(tile);
        for (int kb = 0; kb < num_kb; ++kb, ++it) {
          const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1;
          mbar_wait(&empty[s], ph ^ 1);
          if constexpr (TWO_SM) {
            // both CTAs' operand bytes land on the leader's full barrier
            const uint32_t fb = mapa_shared(smem_u32(&full[s]), 0);
            if (leader) mbar_expect_tx(&full[s], 2 * C::STAGE_BYTES);
            tma_load_2d_2sm(sA + s * C::A_BYTES, &maps.a, fb, kb * C::BK, m0);
            if constexpr (!C::B_RES)
              tma_load_2d_2sm(sB + s * C::B_BYTES, &maps.b, fb, kb * C::BK, n0 + (int)crank * C::B_ROWS);
            continue;
          }
          mbar_expect_tx(&full[s], C::STAGE_BYTES);
          tma_load_2d(sA + s * C::A_BYTES, &maps.a, &full[s], kb * C::BK, m0);
#pragma unroll
          for (int h = 0; h < BN / C::B_BOX; ++h) {
            tma_load_2d(sB + s * C::B_BYTES + h * C::B_BOX * C::SWZ, &maps.b, &full[s], kb * C::BK,
                        n0 + h * C::B_BOX);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp runs the loop so descriptors
    // stay warp-uniform (uniform registers, no per-MMA R2UR waterfall); one
    // elected lane issues.  Descriptor address field = addr >> 4.
    pdl_wait(ep.pdl);
    constexpr uint32_t idesc = idesc_bf16_f32(TWO_SM ? 256 : 128, C::MMA_N);
    const uint64_t a_desc0 = kmajor_desc<C::SWZ>(smem_u32(sA));
    const uint64_t b_desc0 = kmajor_desc<C::SWZ>(smem_u32(sB));
    uint32_t it = 0, local = 0;
    if constexpr (C::B_RES) {
      if (leader && t_first < t_limit) {
        mbar_wait(bfull, 0);
        tc_fence_after();
      }
    }
    for (int tile = t_first; tile < ((TWO_SM && !leader) ? t_first : t_limit); tile += t_stride, ++local) {
      const uint32_t acc = local % C::ACC_STAGES, aph = (local / C::ACC_STAGES) & 1;
      mbar_wait(&tempty[acc], aph ^ 1);  // epilogue drained this accumulator
      tc_fence_after();
      if (lane == 0) GTR(0, local);
      const uint32_t d = tmem_base + acc * C::ACC_STRIDE;
      for (int kb = 0; kb < num_kb; ++kb, ++it) {
        const uint32_t s = it % C::STAGES, ph = (it / C::STAGES) & 1;
        mbar_wait(&full[s], ph);
        tc_fence_after();
        const uint64_t ad = a_desc0 + (uint64_t)((s * C::A_BYTES) >> 4);
        const uint64_t bd = b_desc0 + (uint64_t)(((C::B_RES ? kb : (int)s) * C::B_BYTES) >> 4);
        if (elect_one()) {
          if constexpr (TWO_SM) {
#pragma unroll
            for (int k = 0; k < C::BK / 16; ++k) mma_bf16_ss_2sm(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
            mma_commit_2sm_mc(&empty[s], 0x3);                     // both CTAs may refill stage s
            if (kb + 1 == num_kb) mma_commit_2sm_mc(&tfull[acc], 0x3);  // both epilogues may start
          } else {
#pragma unroll
            for (int k = 0; k < C::BK / 16; ++k) {
#pragma unroll
              for (int h = 0; h < C::N_SPLIT; ++h)
                mma_bf16_ss(d + h * C::MMA_N, ad + 2 * k, bd + (uint64_t)((h * C::MMA_N * C::SWZ) >> 4) + 2 * k,
                            idesc, (kb | k) != 0);
            }
            mma_commit(&empty[s]);
            if (kb + 1 == num_kb) mma_commit(&tfull[acc]);
          }
        }
        __syncwarp();
      }
      if (lane == 0) GTR(1, local);
    }
  } else {
    // ---------------- epilogue warps
    pdl_wait(ep.pdl);
    const uint32_t e = warp - 2;
    const uint32_t quarter = warp & 3;
    constexpr int EPI_THREADS = EPI_WARPS * 32;
    constexpr int COLS = BN / (EPI_WARPS / 4 / C::TILE_GROUPS);  // columns per thread (warps sharing a lane quarter split them)
    const int c_lo = C::TILE_GROUPS > 1 ? 0 : (int)(e / 4) * COLS;
    const uint32_t tgroup = C::TILE_GROUPS > 1 ? e / 4 : 0;
    const int et = threadIdx.x - 64;
    using OutStage = OutStageT<C::OUT_BUF, C::LN_RING ? 2 : C::OUT_NBUF>;
    OutStage out{sOut + e * C::OUT_NBUF * C::OUT_BUF, 0};
    uint32_t ring = 0;  // RES: per-buffer load parity bits
    uint32_t local = 0;
    // QKV: the whole bias row (3*hidden floats) fits the vector area, so it is staged
    // once instead of per tile (the per-tile global-load latency sat on the epilogue's
    // critical path, which bounds this GEMM: ~4400 vs ~2900 MMA cycles per tile)
    const bool bias_all = KIND == EPI_QKV && N * 4 <= C::VEC_BYTES;
    if (bias_all) {
      for (int c = et; c < N; c += EPI_THREADS) vecs[c] = ep.bias[c];
      named_bar_sync(5, EPI_THREADS);
    }
    for (int tile = t_first; tile < t_limit; tile += t_stride, ++local) {
      if (C::TILE_GROUPS > 1 && (local & 1) != tgroup) continue;  // the other group's tile
      const int m0 = tile_m0(tile), n0 = tile_n0(tile);
      const uint32_t acc = local % C::ACC_STAGES, aph = (local / C::ACC_STAGES) & 1;
      const int r0 = m0 + quarter * 32;  // first row of this warp
      const int row = r0 + lane;
      const bool valid = row < ep.M;
      const uint32_t taddr = tmem_base + ((quarter * 32) << 16) + acc * C::ACC_STRIDE;
      const int slot = m0 / ep.tokens_per_slot;
      // Stage this tile's per-column vectors in smem (double-buffered by tile
      // parity) and start the residual loads *before* waiting for the
      // accumulator: their latency hides under the main loop.
      float* vb = vecs + (local & 1) * (4 * BN);
      for (int c = et; c < (bias_all ? 0 : BN); c += EPI_THREADS) {
        vb[c] = ep.bias[n0 + c];
        if constexpr (KIND == EPI_RES) vb[BN + c] = ep.gate[(int64_t)slot * ep.vec_stride + n0 + c];
        if constexpr (KIND == EPI_RES_LN || KIND == EPI_RES_LN2) {
          const int64_t o = (int64_t)slot * ep.vec_stride + n0 + c;
          vb[BN + c] = ep.gate[o];
          vb[2 * BN + c] = ep.shift[o];
          vb[3 * BN + c] = ep.scale[o];
        }
      }
      // RES_LN / RES_LN2: all residual chunks (32 rows x 32 columns) of this thread's
      // columns are TMA-loaded into the warp's staging buffers (chunk q -> buffer q)
      // before the accumulator wait, so their latency hides under the main loop;
      // pass 1 overwrites them in place with the updated residual (then stored),
      // pass 3 with the modulated LayerNorm output.
      uint8_t* const rbuf0 = sOut + e * C::OUT_NBUF * C::OUT_BUF;
      if constexpr (KIND == EPI_RES_LN || KIND == EPI_RES_LN2) {
        if (lane == 0) {
          bulk_wait_read<0>();  // the previous tile's stores have read every buffer
#pragma unroll
          for (int q = 0; q < COLS / 32; ++q) {
            mbar_expect_tx(&rbar[e * 4 + q], C::OUT_BUF);
            tma_load_2d(rbuf0 + q * C::OUT_BUF, &maps.d[0], &rbar[e * 4 + q], n0 + c_lo + 32 * q, r0);
          }
        }
        __syncwarp();
      }
      // RES (wide rows): the residual chunks of this thread's columns (64 at a
      // time, SW128 staging) are TMA-loaded into the warp's two staging buffers.
      if constexpr (KIND == EPI_RES) {
        static_assert(KIND != EPI_RES || COLS <= 128, "RES: at most two 64-column chunks per warp");
        if (lane == 0) {
          bulk_wait_read<0>();  // previous tile's stores have read both buffers
#pragma unroll
          for (int c = 0; c < COLS / 64; ++c) {
            mbar_expect_tx(&rbar[e * 4 + c], 4096);
            tma_load_2d(rbuf0 + c * 4096, &maps.d[0], &rbar[e * 4 + c], n0 + c_lo + 64 * c, r0);
          }
        }
        __syncwarp();
      }
      if (!bias_all)  // vectors staged (tile groups: per group)
        named_bar_sync(C::TILE_GROUPS > 1 ? 6 + tgroup : 5, EPI_THREADS / C::TILE_GROUPS);
      if (warp == 2 && lane == 0) GTR(2, local);
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      if (warp == 2 && lane == 0) GTR(3, local);
      const float* vbias = bias_all ? vecs + n0 + c_lo : vb + c_lo;

      if constexpr (KIND == EPI_F32) {
#pragma unroll 1
        for (int c0 = 0; c0 < COLS; c0 += 32) {
          float v[32];
          tmem_ld32(taddr + c_lo + c0, v);
          tmem_ld_wait();
          if (valid) {
            float4* dst =
                reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.out) + (int64_t)row * ep.ldo + n0 + c_lo + c0);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 b = reinterpret_cast<const float4*>(vbias + c0)[i];
              dst[i] = make_float4(v[4 * i] + b.x, v[4 * i + 1] + b.y, v[4 * i + 2] + b.z, v[4 * i + 3] + b.w);
            }
          }
        }
        acc_release(acc);
      } else if constexpr ((KIND == EPI_BF16 || KIND == EPI_GELU) && C::NARROW) {
        // 16 epilogue warps (4 per TMEM lane quarter): 32-column chunks, 64B-swizzled
        // staging (box 32 x 32), bias + GELU in packed f32x2 arithmetic
#pragma unroll 1
        for (int c0 = 0; c0 < COLS; c0 += 32) {
          uint8_t* buf = out.acquire(lane);
          float v[32];
          tmem_ld32(taddr + c_lo + c0, v);
          tmem_ld_wait();
          if (c0 + 32 >= COLS) {  // last TMEM read of this tile by this warp
            acc_release(acc);
          }
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 bb = reinterpret_cast<const float2*>(vbias + c0)[i];
            float2 y = __fadd2_rn(make_float2(v[2 * i], v[2 * i + 1]), bb);
            if constexpr (KIND == EPI_GELU) y = gelu_tanh2(y);
            v[2 * i] = y.x;
            v[2 * i + 1] = y.y;
          }
#pragma unroll
          for (int i = 0; i < 4; ++i) OutStage::put16(buf, lane, i, pack8_bf16(v + 8 * i));
          out.release(lane, &maps.d[0], buf, n0 + c_lo + c0, r0, r0 < ep.M);
        }
      } else if constexpr (KIND == EPI_BF16 || KIND == EPI_GELU) {
#pragma unroll 1
        for (int c0 = 0; c0 < COLS; c0 += 64) {
          uint8_t* buf = out.acquire(lane);
          if (warp == 2 && lane == 0) GTR(4, 3 * local + c0 / 64);
          // both 32-column halves of the head in flight before one wait; the
          // accumulator is released as soon as the tile's last columns are in registers
          float v64[64];
          tmem_ld32(taddr + c_lo + c0, *reinterpret_cast<float(*)[32]>(&v64[0]));
          tmem_ld32(taddr + c_lo + c0 + 32, *reinterpret_cast<float(*)[32]>(&v64[32]));
          tmem_ld_wait();
          if (warp == 2 && lane == 0) GTR(5, 3 * local + c0 / 64);
          if (c0 + 64 >= COLS) acc_release(acc);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float* v = v64 + 32 * h;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 b = reinterpret_cast<const float4*>(vbias + c0 + 32 * h)[i];
              v[4 * i] += b.x;
              v[4 * i + 1] += b.y;
              v[4 * i + 2] += b.z;
              v[4 * i + 3] += b.w;
            }
            if constexpr (KIND == EPI_GELU) {
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = gelu_tanh(v[i]);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) OutStage::put16(buf, lane, 4 * h + i, pack8_bf16(v + 8 * i));
          }
          if (c0 + 64 >= COLS) {  // last TMEM read of this tile by this warp
            acc_release(acc);
          }
          out.release(lane, &maps.d[0], buf, n0 + c_lo + c0, r0, r0 < ep.M);
        }
      } else if constexpr (KIND == EPI_QKV && BN == 144) {
        // head dim 72: a 144-column tile = two whole heads of one of Q / K / V.
        // Q, K rows (72 bf16 = 144 B) staged unswizzled, box 72 x 32; V^T staged as
        // 72 head-dim rows x 32 tokens (fp16, 64-byte rows, 64B swizzle).
        const int d = ep.heads * 72;
        const int T = ep.tokens_per_slot;
        const int tok0 = r0 - slot * T;
#pragma unroll 1
        for (int hh = 0; hh < 2; ++hh) {
          const int gc = n0 + 72 * hh;
          const int which = gc / d;
          const int head = (gc - which * d) / 72;
          const int64_t hb = ((int64_t)slot * ep.heads + head);
          const float sc = which == 0 ? ep.q_scale : 1.0f;
          uint8_t* buf = out.acquire(lane);
          float v[80];
          tmem_ld32(taddr + 72 * hh, *reinterpret_cast<float(*)[32]>(&v[0]));
          tmem_ld32(taddr + 72 * hh + 32, *reinterpret_cast<float(*)[32]>(&v[32]));
          tmem_ld16(taddr + 72 * hh + 64, *reinterpret_cast<float(*)[16]>(&v[64]));
          tmem_ld_wait();
          if (hh == 1) {
            acc_release(acc);
          }
#pragma unroll
          for (int i = 0; i < 18; ++i) {
            const float4 b = reinterpret_cast<const float4*>(vbias + 72 * hh)[i];
            v[4 * i] = (v[4 * i] + b.x) * sc;
            v[4 * i + 1] = (v[4 * i + 1] + b.y) * sc;
            v[4 * i + 2] = (v[4 * i + 2] + b.z) * sc;
            v[4 * i + 3] = (v[4 * i + 3] + b.w) * sc;
          }
          if (which < 2) {
#pragma unroll
            for (int i = 0; i < 9; ++i) *reinterpret_cast<uint4*>(buf + lane * 144 + 16 * i) = pack8_bf16(v + 8 * i);
          } else {
#pragma unroll
            for (int i = 0; i < 72; ++i)
              *reinterpret_cast<__half*>(buf + i * 64 + ((((lane >> 3) ^ ((i >> 1) & 3))) * 16) + (lane & 7) * 2) =
                  __float2half_rn(v[i]);
          }
          if (which < 2)
            out.release(lane, &maps.d[which < 2 ? which : 1], buf, 0, (int)(hb * T + tok0), r0 < ep.M);
          else
            out.release(lane, &maps.d[2], buf, tok0, (int)(hb * 72), r0 < ep.M);
        }
      } else if constexpr (KIND == EPI_RES) {
        const float* vgate = vb + BN + c_lo;
        const bool st_ok = r0 < ep.M;
#pragma unroll 1
        for (int c = 0; c < COLS / 64; ++c) {
          uint8_t* buf = rbuf0 + c * 4096;
          mbar_wait(&rbar[e * 4 + c], (ring >> c) & 1);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float v[32];
            tmem_ld32(taddr + c_lo + 64 * c + 32 * h, v);
            tmem_ld_wait();
            if (c + 1 == COLS / 64 && h == 1) {
              acc_release(acc);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              uint4* slotp = reinterpret_cast<uint4*>(buf + lane * 128 + (((4 * h + i) ^ (lane & 7)) * 16));
              const uint4 o = *slotp;
              const uint32_t ow[4] = {o.x, o.y, o.z, o.w};
              uint32_t nw[4];
#pragma unroll
              for (int k = 0; k < 4; ++k) {
                const int col = 64 * c + 32 * h + 8 * i + 2 * k;
                const float2 x0 = unpack_bf16(ow[k]);
                nw[k] = pack_bf16(x0.x + vgate[col] * (v[8 * i + 2 * k] + vbias[col]),
                                  x0.y + vgate[col + 1] * (v[8 * i + 2 * k + 1] + vbias[col + 1]));
              }
              *slotp = make_uint4(nw[0], nw[1], nw[2], nw[3]);
            }
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (st_ok) {
              tma_store_2d(&maps.d[0], buf, n0 + c_lo + 64 * c, r0);
            }
            bulk_commit();
          }
          __syncwarp();
        }
        ring ^= (1u << (COLS / 64)) - 1;  // per-buffer load parity
      } else if constexpr (KIND == EPI_QKV) {
        // columns [0, d) -> Q, [d, 2d) -> K, [2d, 3d) -> V; 64 columns per head
        const int d = ep.heads * 64;
        const int T = ep.tokens_per_slot;
        const int tok0 = r0 - slot * T;
#pragma unroll 1
        for (int c0 = 0; c0 < COLS; c0 += 64) {
          const int gc = n0 + c_lo + c0;
          const int which = gc / d;
          const int head = (gc - which * d) / 64;
          const int64_t hb = ((int64_t)slot * ep.heads + head);
          const float sc = which == 0 ? ep.q_scale : 1.0f;
          uint8_t* buf = out.acquire(lane);
          if (warp == 2 && lane == 0) GTR(4, 3 * local + c0 / 64);
          // both 32-column halves of the head in flight before one wait; the
          // accumulator is released as soon as the tile's last columns are in registers
          float v64[64];
          tmem_ld32(taddr + c_lo + c0, *reinterpret_cast<float(*)[32]>(&v64[0]));
          tmem_ld32(taddr + c_lo + c0 + 32, *reinterpret_cast<float(*)[32]>(&v64[32]));
          tmem_ld_wait();
          if (warp == 2 && lane == 0) GTR(5, 3 * local + c0 / 64);
          if (c0 + 64 >= COLS) acc_release(acc);
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            float* v = v64 + 32 * h;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 b = reinterpret_cast<const float4*>(vbias + c0 + 32 * h)[i];
              v[4 * i] = (v[4 * i] + b.x) * sc;
              v[4 * i + 1] = (v[4 * i + 1] + b.y) * sc;
              v[4 * i + 2] = (v[4 * i + 2] + b.z) * sc;
              v[4 * i + 3] = (v[4 * i + 3] + b.w) * sc;
            }
            if (which < 2) {
#pragma unroll
              for (int i = 0; i < 4; ++i) OutStage::put16(buf, lane, 4 * h + i, pack8_bf16(v + 8 * i));
            } else {
              // V^T staging: 64 rows (head dim) x 64 B (32 tokens), 64B swizzle:
              // 16-byte chunk c of row dd lives at chunk c ^ ((dd >> 1) & 3)
              // dims (2p, 2p+1) x tokens (2j, 2j+1) are swapped across lane pairs with one
              // shuffle, so each lane stores a 4-byte token pair: 16 STS.32 (1 wavefront
              // each: the two rows are adjacent 64-byte halves) instead of 32 STS.16
              const uint32_t odd = lane & 1;
#pragma unroll
              for (int pi = 0; pi < 16; ++pi) {
                uint32_t own;
                asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(own) : "f"(v[2 * pi + 1]), "f"(v[2 * pi]));
                const uint32_t other = __shfl_xor_sync(0xffffffffu, own, 1);
                const uint32_t w = __byte_perm(own, other, odd ? 0x3276 : 0x5410);
                const uint32_t dd = 32 * h + 2 * pi + odd;
                *reinterpret_cast<uint32_t*>(buf + dd * 64 + ((((lane >> 3) ^ ((dd >> 1) & 3))) * 16) +
                                             (lane & 6) * 2) = w;  // V^T is fp16 (PV runs in fp16)
              }
            }
          }
          if (warp == 2 && lane == 0) GTR(6, 3 * local + c0 / 64);
          if (which < 2)
            out.release(lane, &maps.d[which < 2 ? which : 1], buf, 0, (int)(hb * T + tok0), r0 < ep.M);
          else
            out.release(lane, &maps.d[2], buf, tok0, (int)(hb * 64), r0 < ep.M);
          if (warp == 2 && lane == 0) GTR(7, 3 * local + c0 / 64);
        }
      } else if constexpr (KIND == EPI_RES_LN || KIND == EPI_RES_LN2) {
        // RES_LN: 12 epilogue warps; the 3 warps of a lane quarter split each
        // 384-column row into 128-column thirds.  RES_LN2: this CTA owns a
        // 192-column slice; 8 warps, 2 per lane quarter (96 columns each), and the
        // row statistics of the XCH_CL slices meet in distributed shared memory.
        // Either way 32-column chunks are staged in 64B-swizzled smem and stored by
        // TMA (box 32 x 32).
        static_assert(KIND != EPI_RES_LN || (EPI_WARPS == 12 && COLS % 32 == 0), "RES_LN layout");
        static_assert(KIND != EPI_RES_LN2 || (EPI_WARPS == 8 && COLS == 96), "RES_LN2 layout");
        // row statistic over the whole (384-wide) row from this thread's partial
        auto row_total = [&](float part, int pass) -> float {
          if constexpr (KIND == EPI_RES_LN) {
            const uint32_t eq = e & 3;
            float* rr = red + pass * EPI_WARPS * 32;
            rr[e * 32 + lane] = part;
            named_bar_sync(1 + quarter, 96);
            return rr[eq * 32 + lane] + rr[(eq + 4) * 32 + lane] + rr[(eq + 8) * 32 + lane];
          } else {
            const uint32_t par = local & 1, g = e >> 2, row = quarter * 32 + lane;
            // xch[par][pass][src][g][row]: push this partial into every cluster peer
            const uint32_t off = (uint32_t)((((par * 2 + pass) * XCH_CL + crank) * 2 + g) * 128 + row) * 4u;
#pragma unroll
            for (uint32_t q = 0; q < (uint32_t)XCH_CL; ++q) st_cluster_f32(mapa_shared(smem_u32(xch) + off, q), part);
            // each thread releases its own DSMEM stores to every peer (count XCH_CL * EPI_THREADS)
#pragma unroll
            for (uint32_t q = 0; q < (uint32_t)XCH_CL; ++q)
              mbar_arrive_cluster(mapa_shared(smem_u32(&xbar[par * 2 + pass]), q));
            mbar_wait_cluster(&xbar[par * 2 + pass], (local >> 1) & 1);
            if (pass == 0 && warp == 2 && lane == 0) GTR(6, local);
            float tot = 0.f;
#pragma unroll
            for (int q = 0; q < XCH_CL; ++q)
#pragma unroll
              for (int gg = 0; gg < 2; ++gg) tot += xch[(((par * 2 + pass) * XCH_CL + q) * 2 + gg) * 128 + row];
            return tot;
          }
        };
        const float* vgate = vb + BN + c_lo;
        const float* vshift = vb + 2 * BN + c_lo;
        const float* vscale = vb + 3 * BN + c_lo;
        const uint32_t tcol = taddr + c_lo;
        const bool st_ok = r0 < ep.M;
        // pass 1: x_new = x + gate*(acc + bias) -> bf16 residual (TMA store), kept in
        // registers as bf16 pairs (LayerNorm sees the stored, rounded residual);
        // partial row sum.  The accumulator is released right after its last TMEM
        // read, so the next tile's main loop overlaps the LayerNorm passes.
        constexpr int NQ = COLS / 32;
        uint32_t xr[NQ][16];
        float sum = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          uint8_t* buf = rbuf0 + q * C::OUT_BUF;
          mbar_wait(&rbar[e * 4 + q], local & 1);  // one residual load per buffer per tile
          uint4 oldv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i)
            oldv[i] = *reinterpret_cast<const uint4*>(buf + lane * 64 + ((i ^ ((lane >> 1) & 3)) * 16));
          const uint32_t* ow = reinterpret_cast<const uint32_t*>(oldv);
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int u = 2 * q + hh;  // 16-column sub-chunk
            float v[16];
            tmem_ld16(tcol + 16 * u, v);
            tmem_ld_wait();
            if (u + 1 == 2 * NQ) {  // last TMEM read: the next tile's main loop may start
              acc_release(acc);
            }
#pragma unroll
            for (int i = 0; i < 4; ++i) {
              const float4 bb = reinterpret_cast<const float4*>(vbias + 16 * u)[i];
              const float4 g = reinterpret_cast<const float4*>(vgate + 16 * u)[i];
              const int w = 8 * hh + 2 * i;
              const float2 o0 = unpack_bf16(ow[w]), o1 = unpack_bf16(ow[w + 1]);
              xr[q][w] = pack_bf16(o0.x + g.x * (v[4 * i] + bb.x), o0.y + g.y * (v[4 * i + 1] + bb.y));
              xr[q][w + 1] = pack_bf16(o1.x + g.z * (v[4 * i + 2] + bb.z), o1.y + g.w * (v[4 * i + 3] + bb.w));
              const float2 r0v = unpack_bf16(xr[q][w]), r1v = unpack_bf16(xr[q][w + 1]);
              sum += (r0v.x + r0v.y) + (r1v.x + r1v.y);
            }
          }
#pragma unroll
          for (int i = 0; i < 4; ++i)
            OutStage::put16(buf, lane, i, make_uint4(xr[q][4 * i], xr[q][4 * i + 1], xr[q][4 * i + 2], xr[q][4 * i + 3]));
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (st_ok) tma_store_2d(&maps.d[0], buf, n0 + c_lo + 32 * q, r0);
            bulk_commit();
          }
          __syncwarp();
        }
        const float mean = row_total(sum, 0) * (1.0f / N);
        float var = 0.f;
#pragma unroll
        for (int q = 0; q < NQ; ++q)
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const float2 xv = unpack_bf16(xr[q][i]);
            const float d0 = xv.x - mean, d1 = xv.y - mean;
            var += d0 * d0 + d1 * d1;
          }
        const float var_all = row_total(var, 1);
        const float rstd = rsqrtf(var_all * (1.0f / N) + ep.ln_eps);
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          uint8_t* buf = rbuf0 + q * C::OUT_BUF;
          if (lane == 0) bulk_wait_read<NQ - 1>();  // the residual store out of buffer q has read it
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float o[8];
#pragma unroll
            for (int k = 0; k < 2; ++k) {
              const float4 sh = reinterpret_cast<const float4*>(vshift + 32 * q)[2 * i + k];
              const float4 sc = reinterpret_cast<const float4*>(vscale + 32 * q)[2 * i + k];
              const float2 xa = unpack_bf16(xr[q][4 * i + 2 * k]), xb = unpack_bf16(xr[q][4 * i + 2 * k + 1]);
              o[4 * k] = (xa.x - mean) * rstd * (1.0f + sc.x) + sh.x;
              o[4 * k + 1] = (xa.y - mean) * rstd * (1.0f + sc.y) + sh.y;
              o[4 * k + 2] = (xb.x - mean) * rstd * (1.0f + sc.z) + sh.z;
              o[4 * k + 3] = (xb.y - mean) * rstd * (1.0f + sc.w) + sh.w;
            }
            OutStage::put16(buf, lane, i, pack8_bf16(o));
          }
          fence_proxy_async_smem();
          __syncwarp();
          if (lane == 0) {
            if (st_ok) tma_store_2d(&maps.d[1], buf, n0 + c_lo + 32 * q, r0);
            bulk_commit();
          }
          __syncwarp();
        }
      }
    }
    if (lane == 0) bulk_wait<0>();  // all output stores of this warp have landed
    __syncwarp();
  }

  tc_fence_before();
  __syncthreads();
#if SF_GEMM_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 1024) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_gemm_cta_end[blockIdx.x] = t;
  }
#endif
  if constexpr (TWO_SM) cluster_sync_all();  // the pair's MMAs / barrier traffic are over
  if (warp == 1) {
    if constexpr (TWO_SM)
      tmem_dealloc_2sm<C::TMEM_COLS>(tmem_base);
    else
      tmem_dealloc<C::TMEM_COLS>(tmem_base);
  }
  if constexpr (CLUSTER) cluster_sync_all();  // no CTA leaves while a peer may still write its smem
}

}  // namespace sf

// Tiny-VAE (TAESD) decoder of retired frames (the reference's
// decode_stub, src/pipeline.py:86-89, replaced by the paper's taesd decoder).
//
// Network (madebyollin/taesd Decoder, state-dict layout of taesd_decoder.pth):
//   Clamp(tanh(x/3)*3) -> conv(4,64) -> ReLU -> 3 x Block -> Up2 -> conv(64,64,no bias)
//   -> 3 x Block -> Up2 -> conv -> 3 x Block -> Up2 -> conv -> Block -> conv(64,3)
//   Block(x) = ReLU(conv(ReLU(conv(ReLU(conv(x))))) + x)
// 64x64x4 latent -> 512x512x3 image.
//
// B200 layout: activations are bf16 NHWC with a one-pixel zero border, stored as
// one flat pixel array per frame (row pitch Wp = W + 2, (H + 2) rows; 128 bytes per
// pixel = one 128B-swizzle row).  In that layout a 3x3 conv is a 1-D convolution
// over the flat array with tap offsets (dy-1)*Wp + (dx-1): a tile of 128
// consecutive output pixels needs three 130-pixel input runs (one per dy), each
// a single TMA box, and the three dx taps are the same smem run shifted by one
// 128-byte row (descriptor start + dx*128).  K = 9 taps x 64 channels = 36
// tcgen05 MMAs (M=128, N=64, K=16) per tile; the weights (72 KB) stay resident in
// smem; fp32 accumulators in TMEM (4 buffers); epilogue warps add bias /
// residual, apply ReLU, and write only interior pixels, so borders stay zero.
// The 2x nearest upsample is fused into the last conv of each stage (the
// epilogue writes every output pixel to its 2x2 block of the next stage).
#include <cstdint>

#include "sf_internal.h"
#include "sf_ptx.cuh"

namespace sf {
namespace vae {

constexpr int CH = 64;
constexpr int BM = 128;                       // output pixels per tile
constexpr int HALO = 136;                     // input pixels per dy run (BM + 2, rounded to 8 rows)
constexpr int HALO_BYTES = HALO * 128;        // 17408 = 17 KB, 1024-aligned
constexpr int STAGE_BYTES = 3 * HALO_BYTES;   // three dy runs
constexpr int STAGES = 2;
constexpr int ACC = 4;                        // TMEM accumulator buffers
constexpr int EPI_WARPS = 4;

enum Epi : int { EPI_NONE = 0, EPI_RELU = 1, EPI_RES_RELU = 2, EPI_RES_RELU_UP2 = 3, EPI_FINAL = 4 };

template <int NW>
struct Cfg {
  static constexpr int W_BYTES = 9 * NW * 128;
  static constexpr int TMEM_COLS = ACC * NW < 32 ? 32 : ACC * NW;
  static constexpr int STG_BYTES = EPI_WARPS * 32 * 144;  // per-warp 32-pixel staging, 144 B pitch
  static constexpr int SMEM = 1024 + W_BYTES + STAGES * STAGE_BYTES + 1024 + STG_BYTES;
};

struct ConvArgs {
  const float* bias;             // [NW] or null
  const __nv_bfloat16* res;      // residual (input geometry) or null
  void* out;                     // bf16 padded NHWC (same or 2x geometry) / fp32 NCHW image (FINAL)
  int F, H, W;
  int tiles_per_frame;
};

__device__ __forceinline__ uint4 relu_add_pack(const float* v, const float* b, const uint4 (&r)[8], int j,
                                               bool has_res, bool relu) {
  float x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = v[8 * j + i] + b[8 * j + i];
  if (has_res) {
    const uint4 rv = r[j];
    const uint32_t rr[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = unpack_bf16(rr[i]);
      x[2 * i] += f.x;
      x[2 * i + 1] += f.y;
    }
  }
  if (relu) {
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = fmaxf(x[i], 0.f);
  }
  return make_uint4(pack_bf16(x[0], x[1]), pack_bf16(x[2], x[3]), pack_bf16(x[4], x[5]), pack_bf16(x[6], x[7]));
}

template <int NW, int EPI>
__global__ void __launch_bounds__(192, 1)
    conv3x3_tcgen05(const __grid_constant__ CUtensorMap tm_in, const __grid_constant__ CUtensorMap tm_w, ConvArgs a) {
  using Cf = Cfg<NW>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  uint8_t* sW = smem;
  uint8_t* sA = sW + Cf::W_BYTES;
  uint64_t* bars = reinterpret_cast<uint64_t*>(sA + STAGES * STAGE_BYTES);
  uint64_t* full = bars;                 // [STAGES]
  uint64_t* empty = full + STAGES;       // [STAGES]
  uint64_t* tfull = empty + STAGES;      // [ACC]
  uint64_t* tempty = tfull + ACC;        // [ACC]
  uint64_t* wbar = tempty + ACC;
  uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(wbar + 1);
  float* sBias = reinterpret_cast<float*>(bars + 64);
  uint8_t* sStage = reinterpret_cast<uint8_t*>(bars + 128);

  const uint32_t warp = warp_id(), lane = threadIdx.x & 31;
  const int Wp = a.W + 2;
  const int64_t P = (int64_t)(a.H + 2) * Wp;
  const int total = a.F * a.tiles_per_frame;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tm_in);
    tma_prefetch(&tm_w);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int i = 0; i < ACC; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], EPI_WARPS * 32);
    }
    mbar_init(wbar, 1);
    fence_barrier_init();
  }
  if (threadIdx.x < NW) sBias[threadIdx.x] = a.bias ? a.bias[threadIdx.x] : 0.f;
  if (warp == 1) tmem_alloc<Cf::TMEM_COLS>(tmem_holder);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_holder;

  if (warp == 0) {
    // ---------------- TMA producer: resident weights, then three dy runs per tile
    if (elect_one()) {
      mbar_expect_tx(wbar, Cf::W_BYTES);
      for (int tap = 0; tap < 9; ++tap) tma_load_2d(sW + tap * NW * 128, &tm_w, wbar, 0, tap * NW);
      int it = 0;
      for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
        const int f = tile / a.tiles_per_frame, tt = tile % a.tiles_per_frame;
        const int64_t g0 = (int64_t)f * P + Wp + (int64_t)tt * BM;
        const int s = it % STAGES;
        mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
        mbar_expect_tx(&full[s], STAGE_BYTES);
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
          tma_load_2d(sA + s * STAGE_BYTES + dy * HALO_BYTES, &tm_in, &full[s], 0,
                      (int32_t)(g0 + (int64_t)(dy - 1) * Wp - 1));
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: 9 taps x 4 K-steps per tile
    constexpr uint32_t idesc = idesc_bf16_f32(128, NW);
    mbar_wait(wbar, 0);
    tc_fence_after();
    const uint32_t sA0 = smem_u32(sA), sW0 = smem_u32(sW);
    int it = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      const int s = it % STAGES, acc = it % ACC;
      mbar_wait(&tempty[acc], ((it / ACC) & 1) ^ 1);
      mbar_wait(&full[s], (it / STAGES) & 1);
      tc_fence_after();
      if (elect_one()) {
#pragma unroll
        for (int tap = 0; tap < 9; ++tap) {
          const int dy = tap / 3, dx = tap % 3;
          const uint64_t ad = sw128_kmajor_desc(sA0 + s * STAGE_BYTES + dy * HALO_BYTES + dx * 128);
          const uint64_t bd = sw128_kmajor_desc(sW0 + tap * NW * 128);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_bf16_ss(tmem + acc * NW, ad + 2 * k, bd + 2 * k, idesc, (tap | k) != 0);
        }
        mma_commit(&empty[s]);
        mma_commit(&tfull[acc]);
      }
      __syncwarp();
    }
  } else {
    // ---------------- epilogue: TMEM lane quarter (warp & 3) = 32 output pixels
    const uint32_t quarter = warp & 3;
    const uint32_t taddr0 = tmem + ((quarter * 32) << 16);
    int it = 0;
    for (int tile = blockIdx.x; tile < total; tile += gridDim.x, ++it) {
      const int acc = it % ACC;
      const int f = tile / a.tiles_per_frame, tt = tile % a.tiles_per_frame;
      mbar_wait(&tfull[acc], (it / ACC) & 1);
      tc_fence_after();
      float v[NW];
      if constexpr (NW == 64) {
        tmem_ld32(taddr0 + acc * NW, *reinterpret_cast<float(*)[32]>(&v[0]));
        tmem_ld32(taddr0 + acc * NW + 32, *reinterpret_cast<float(*)[32]>(&v[32]));
      } else {
        tmem_ld16(taddr0 + acc * NW, *reinterpret_cast<float(*)[16]>(&v[0]));
      }
      tmem_ld_wait();
      tc_fence_before();
      mbar_arrive(&tempty[acc]);

      const int qf0 = Wp + tt * BM + quarter * 32;  // flat padded pixel of lane 0 within the frame
      const int qf = qf0 + lane;
      const int y = qf / Wp, x = qf - y * Wp;
      const bool valid = y <= a.H && x >= 1 && x <= a.W;  // borders / beyond the last row: never written
      if constexpr (EPI == EPI_FINAL) {
        if (valid) {
          float* img = reinterpret_cast<float*>(a.out) + (int64_t)f * 3 * a.H * a.W + (int64_t)(y - 1) * a.W + (x - 1);
#pragma unroll
          for (int c = 0; c < 3; ++c) img[(int64_t)c * a.H * a.W] = v[c] + sBias[c];
        }
      } else {
        // The warp moves its 32 pixels (128 B each) through smem so that global loads /
        // stores are whole 128-byte lines (8 lanes per pixel) instead of 32 lines per
        // instruction.
        constexpr bool RES = EPI == EPI_RES_RELU || EPI == EPI_RES_RELU_UP2;
        constexpr bool RELU = EPI != EPI_NONE;
        uint8_t* stg = sStage + quarter * (32 * 144);
        const uint32_t vmask = __ballot_sync(0xffffffffu, valid);
        const int64_t gp0 = (int64_t)f * P + qf0;
        uint4 rr[8];
        if constexpr (RES) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int p = 4 * i + (lane >> 3), c = lane & 7;
            uint4 val = make_uint4(0u, 0u, 0u, 0u);
            if ((vmask >> p) & 1) val = reinterpret_cast<const uint4*>(a.res + (gp0 + p) * CH)[c];
            *reinterpret_cast<uint4*>(stg + p * 144 + c * 16) = val;
          }
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 8; ++j) rr[j] = *reinterpret_cast<const uint4*>(stg + lane * 144 + j * 16);
          __syncwarp();
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
          *reinterpret_cast<uint4*>(stg + lane * 144 + j * 16) = relu_add_pack(v, sBias, rr, j, RES, RELU);
        __syncwarp();
        __nv_bfloat16* outp = reinterpret_cast<__nv_bfloat16*>(a.out);
        if constexpr (EPI == EPI_RES_RELU_UP2) {
          // pixel (y, x) -> (2y-1, 2x-1), (2y-1, 2x), (2y, 2x-1), (2y, 2x) of the next stage:
          // 256 contiguous bytes in each of two rows; 2 pixels per instruction per row
          const int Wp2 = 2 * a.W + 2;
          const int64_t P2 = (int64_t)(2 * a.H + 2) * Wp2;
#pragma unroll 4
          for (int i = 0; i < 16; ++i) {
            const int p = 2 * i + (lane >> 4), c = lane & 15;
            const int yp = __shfl_sync(0xffffffffu, y, p), xp = __shfl_sync(0xffffffffu, x, p);
            if ((vmask >> p) & 1) {
              const uint4 val = *reinterpret_cast<const uint4*>(stg + p * 144 + (c & 7) * 16);
#pragma unroll
              for (int ry = 0; ry < 2; ++ry)
                reinterpret_cast<uint4*>(outp + ((int64_t)f * P2 + (int64_t)(2 * yp - 1 + ry) * Wp2 + 2 * xp - 1) * CH)[c] =
                    val;
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int p = 4 * i + (lane >> 3), c = lane & 7;
            if ((vmask >> p) & 1)
              reinterpret_cast<uint4*>(outp + (gp0 + p) * CH)[c] =
                  *reinterpret_cast<const uint4*>(stg + p * 144 + c * 16);
          }
        }
        __syncwarp();  // staging is rewritten by the next tile
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc<Cf::TMEM_COLS>(tmem);
}

// Clamp + conv(4 -> 64) + ReLU at 64x64: reads the fp32 NCHW latent, writes the
// padded NHWC bf16 stage-0 activation.  2.4 kMAC per pixel: CUDA cores.
__global__ void __launch_bounds__(256) taesd_first_kernel(const float* __restrict__ lat, const float* __restrict__ w,
                                                          const float* __restrict__ b, __nv_bfloat16* __restrict__ out) {
  constexpr int H = 64, W = 64, Wp = 66;
  __shared__ float sx[4][3][Wp];
  __shared__ float sw[36][64];  // [ic*9 + ky*3 + kx][oc]
  const int f = blockIdx.y, y = blockIdx.x, t = threadIdx.x;
  for (int i = t; i < 64 * 36; i += 256) sw[i % 36][i / 36] = w[i];  // w: [oc][ic][ky][kx]
  for (int i = t; i < 4 * 3 * Wp; i += 256) {
    const int c = i / (3 * Wp), r = (i / Wp) % 3, xx = i % Wp;
    const int yy = y + r - 1, xs = xx - 1;
    float v = 0.f;
    if (yy >= 0 && yy < H && xs >= 0 && xs < W) v = tanhf(lat[(((int64_t)f * 4 + c) * H + yy) * W + xs] / 3.f) * 3.f;
    sx[c][r][xx] = v;
  }
  __syncthreads();
  const int px = t & 63, cg = t >> 6;  // 16 output channels per thread
  float acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = b[cg * 16 + i];
  for (int c = 0; c < 4; ++c)
#pragma unroll
    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
      for (int kx = 0; kx < 3; ++kx) {
        const float xv = sx[c][ky][px + kx];
        const float* wr = &sw[c * 9 + ky * 3 + kx][cg * 16];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = fmaf(xv, wr[i], acc[i]);
      }
  uint4* d = reinterpret_cast<uint4*>(out + (((int64_t)f * (H + 2) + y + 1) * Wp + px + 1) * CH + cg * 16);
  uint32_t p[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) p[i] = pack_bf16(fmaxf(acc[2 * i], 0.f), fmaxf(acc[2 * i + 1], 0.f));
  d[0] = make_uint4(p[0], p[1], p[2], p[3]);
  d[1] = make_uint4(p[4], p[5], p[6], p[7]);
}

template <int NW, int EPI>
int launch_conv(const void* in, const void* w, const float* bias, const void* res, void* out, int F, int H, int W,
                cudaStream_t st) {
  using Cf = Cfg<NW>;
  static bool attr = false;
  if (!attr) {
    if (cudaFuncSetAttribute(conv3x3_tcgen05<NW, EPI>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cf::SMEM) !=
        cudaSuccess)
      return SF_ERR_CUDA;
    attr = true;
  }
  const int Wp = W + 2;
  const int64_t P = (int64_t)(H + 2) * Wp;
  CUtensorMap tm_in, tm_w;
  if (make_tmap_bf16_2d(&tm_in, in, CH, (uint64_t)F * P, CH, CH, HALO, 128) != SF_OK) return SF_ERR_CUDA;
  if (make_tmap_bf16_2d(&tm_w, w, CH, 9 * NW, CH, CH, NW, 128) != SF_OK) return SF_ERR_CUDA;
  ConvArgs a{bias, reinterpret_cast<const __nv_bfloat16*>(res), out, F, H, W, (int)((H * Wp + BM - 1) / BM)};
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const int total = F * a.tiles_per_frame;
  const int grid = total < sms ? total : sms;
  conv3x3_tcgen05<NW, EPI><<<grid, 192, Cf::SMEM, st>>>(tm_in, tm_w, a);
  return cuda_status();
}

}  // namespace vae
}  // namespace sf

using namespace sf::vae;

extern "C" {

int64_t sf_taesd_act_elems(int64_t F, int32_t H, int32_t W) { return F * (int64_t)(H + 2) * (W + 2) * CH; }

int sf_conv3x3(const void* in, const void* w, const float* bias, const void* res, void* out, int64_t F, int32_t H,
               int32_t W, int32_t epi, void* stream) {
  if (F < 1 || H < 1 || W < 1 || !in || !w || !out || (int64_t)F * (H + 2) * (W + 2) > 2147483647LL)
    return SF_ERR_PARAMETER;
  if ((epi == EPI_RES_RELU || epi == EPI_RES_RELU_UP2) && !res) return SF_ERR_PARAMETER;
  cudaStream_t st = (cudaStream_t)stream;
  switch (epi) {
    case EPI_NONE: return launch_conv<64, EPI_NONE>(in, w, bias, res, out, (int)F, H, W, st);
    case EPI_RELU: return launch_conv<64, EPI_RELU>(in, w, bias, res, out, (int)F, H, W, st);
    case EPI_RES_RELU: return launch_conv<64, EPI_RES_RELU>(in, w, bias, res, out, (int)F, H, W, st);
    case EPI_RES_RELU_UP2: return launch_conv<64, EPI_RES_RELU_UP2>(in, w, bias, res, out, (int)F, H, W, st);
    case EPI_FINAL: return launch_conv<16, EPI_FINAL>(in, w, bias, res, out, (int)F, H, W, st);
  }
  return SF_ERR_PARAMETER;
}

int sf_taesd_first(const float* lat, const float* w, const float* b, void* out, int64_t F, void* stream) {
  if (F < 1 || F > 65535 || !lat || !w || !b || !out) return SF_ERR_PARAMETER;
  taesd_first_kernel<<<dim3(64, (unsigned)F), 256, 0, (cudaStream_t)stream>>>(lat, w, b,
                                                                              (__nv_bfloat16*)out);
  return sf::cuda_status();
}

int64_t sf_taesd_workspace_bytes(int64_t F) {
  int64_t total = 0;
  for (int s = 0; s < 4; ++s) total += 3 * sf_taesd_act_elems(F, 64 << s, 64 << s) * 2;
  return total;
}

int sf_taesd_decode(const sf_taesd_weights* w, const float* lat, int64_t F, int64_t F_cap, void* ws, int64_t ws_bytes,
                    float* img, void* stream) {
  if (!w || !lat || !ws || !img || F < 1 || F > F_cap || F_cap > 65535) return SF_ERR_PARAMETER;
  if (ws_bytes < sf_taesd_workspace_bytes(F_cap)) return SF_ERR_PARAMETER;
  __nv_bfloat16* buf[4][3];  // layout fixed by F_cap, so zero borders stay valid for any F <= F_cap
  __nv_bfloat16* p = (__nv_bfloat16*)ws;
  for (int s = 0; s < 4; ++s)
    for (int i = 0; i < 3; ++i) {
      buf[s][i] = p;
      p += sf_taesd_act_elems(F_cap, 64 << s, 64 << s);
    }
  int rc = sf_taesd_first(lat, w->first_w, w->first_b, buf[0][0], F, stream);
  int li = 0;  // conv_w / conv_b index
  for (int s = 0; s < 4 && rc == SF_OK; ++s) {
    const int H = 64 << s;
    int in = 0, t1 = 1, t2 = 2;  // block input / temporaries (buffer indices of this stage)
    if (s > 0) {                 // conv(64, 64, bias=False) after the upsample
      rc |= sf_conv3x3(buf[s][0], w->conv_w[li], w->conv_b[li], nullptr, buf[s][1], F, H, H, EPI_NONE, stream);
      ++li;
      in = 1, t1 = 2, t2 = 0;
    }
    const int blocks = s < 3 ? 3 : 1;
    for (int bl = 0; bl < blocks && rc == SF_OK; ++bl) {
      const bool up = s < 3 && bl == blocks - 1;
      rc |= sf_conv3x3(buf[s][in], w->conv_w[li], w->conv_b[li], nullptr, buf[s][t1], F, H, H, EPI_RELU, stream);
      rc |= sf_conv3x3(buf[s][t1], w->conv_w[li + 1], w->conv_b[li + 1], nullptr, buf[s][t2], F, H, H, EPI_RELU,
                       stream);
      rc |= sf_conv3x3(buf[s][t2], w->conv_w[li + 2], w->conv_b[li + 2], buf[s][in], up ? buf[s + 1][0] : buf[s][t1],
                       F, H, H, up ? EPI_RES_RELU_UP2 : EPI_RES_RELU, stream);
      li += 3;
      const int nin = t1;
      t1 = in;
      in = nin;
    }
    if (s == 3) rc |= sf_conv3x3(buf[3][in], w->final_w, w->final_b, nullptr, img, F, H, H, EPI_FINAL, stream);
  }
  return rc == SF_OK ? SF_OK : (rc < 0 ? rc : SF_ERR_CUDA);
}

}  // extern "C"

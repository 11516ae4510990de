// Scheduler (K1), Euler step (K10-lite), CFG combine, mock velocity model
// (K12) and the device-resident ring buffer (K11) of the stream batch.
//
// Bit-exactness: every floating-point operation is written with the
// explicit round-to-nearest intrinsics (__dadd_rn, __dmul_rn, ...), which
// ptxas never contracts into FMAs, in the same literal order as the numpy
// reference, so results are identical bit for bit.
#include <cstdint>

#include "sf_internal.h"

namespace sf {

// ============================================================ K1: window coefficients
__device__ __forceinline__ int abar_index(double tau, int t_max) {
  // schedule.py:201-205  idx = clip(floor((1 - tau) * (t_max - 1) + 0.5))
  const double raw = __dmul_rn(__dsub_rn(1.0, tau), (double)(t_max - 1));
  double f = floor(__dadd_rn(raw, 0.5));
  int idx = (int)f;
  return idx < 0 ? 0 : (idx > t_max - 1 ? t_max - 1 : idx);
}

// grid_indices (schedule.py:266-284): nearest of grid[pos-1], grid[pos] (ties to the upper)
__device__ __forceinline__ int grid_index(const sf_schedule& s, double t) {
  const int G = s.num_steps;
  int pos = 0;
  while (pos < G && s.grid[pos] < t) ++pos;  // searchsorted(side='left')
  const int lo = pos - 1 < 0 ? 0 : (pos - 1 > G - 1 ? G - 1 : pos - 1);
  const int hi = pos > G - 1 ? G - 1 : pos;
  return fabs(__dsub_rn(s.grid[hi], t)) <= fabs(__dsub_rn(s.grid[lo], t)) ? hi : lo;
}

__device__ void window_coeffs_row(const sf_schedule& s, double t, double* p, uint32_t& status) {
  if (!(t >= 0.0 && t <= 1.0)) status |= SF_STATUS_TIME_RANGE;
  // window_lookup (schedule.py:208-221): count interior boundaries strictly below t (+eps)
  int k = 0;
  for (int j = 1; j < s.num_windows; ++j) k += (t > __dadd_rn(s.boundaries[j], s.eps)) ? 1 : 0;
  const double t_s = s.boundaries[k];
  const double t_e = s.boundaries[k + 1];
  // window_params (schedule.py:238-262)
  const double a_s = s.abar[abar_index(t_s, s.t_max)];
  const double a_e = s.abar[abar_index(t_e, s.t_max)];
  const double gamma = __dsqrt_rn(__ddiv_rn(a_s, a_e));
  const double lambda_s = __ddiv_rn(1.0, gamma);
  const double eta_s = __ddiv_rn(-__dsqrt_rn(__dsub_rn(1.0, __dmul_rn(gamma, gamma))), gamma);
  const double denom = __dadd_rn(__dmul_rn(lambda_s, __dsub_rn(t, t_s)), __dsub_rn(t_e, t));
  if (!(denom > 0.0)) status |= SF_STATUS_DENOM;
  const double lambda_t = __ddiv_rn(__dmul_rn(lambda_s, __dsub_rn(t_e, t_s)), denom);
  const double eta_t = __ddiv_rn(__dmul_rn(eta_s, __dsub_rn(t_e, t)), denom);
  // grid_indices / next_timestep (schedule.py:266-295)
  const int G = s.num_steps;
  const int idx = grid_index(s, t);
  double t_next;
  if (fabs(__dsub_rn(s.grid[idx], t)) > s.eps) {
    status |= SF_STATUS_OFF_GRID;
    t_next = __longlong_as_double(0x7ff8000000000000LL);
  } else {
    t_next = idx + 1 < G ? s.grid[idx + 1] : 1.0;
  }
  const double span = __dsub_rn(t_e, t);  // velocity.py:123
  p[SF_P_T] = t;
  p[SF_P_TNEXT] = t_next;
  p[SF_P_TS] = t_s;
  p[SF_P_TE] = t_e;
  p[SF_P_GAMMA] = gamma;
  p[SF_P_LAMBDA_S] = lambda_s;
  p[SF_P_ETA_S] = eta_s;
  p[SF_P_LAMBDA_T] = lambda_t;
  p[SF_P_ETA_T] = eta_t;
  p[SF_P_SPAN] = span;
  p[SF_P_DT] = __dsub_rn(t_next, t);  // velocity.py:129
  p[SF_P_AT_END] = span <= s.eps ? 1.0 : 0.0;
}

__global__ void window_params_kernel(sf_schedule s, const double* __restrict__ ts, int64_t B, double* out,
                                     uint32_t* status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= B) return;
  uint32_t st = 0;
  window_coeffs_row(s, ts[i], out + i * SF_PARAM_STRIDE, st);
  if (st) atomicOr(status, st);
}

__global__ void schedule_indices_kernel(sf_schedule s, const double* __restrict__ ts, int64_t B, int64_t* abar_idx,
                                        int64_t* grid_idx, uint32_t* status) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= B) return;
  const double t = ts[i];
  if (abar_idx) abar_idx[i] = abar_index(t, s.t_max);
  if (grid_idx) {
    uint32_t st = (t >= 0.0 && t <= 1.0) ? 0u : (uint32_t)SF_STATUS_TIME_RANGE;
    const int g = grid_index(s, t);
    if (fabs(__dsub_rn(s.grid[g], t)) > s.eps) st |= SF_STATUS_OFF_GRID;
    grid_idx[i] = g;
    if (st) atomicOr(status, st);
  }
}

// ============================================================ K10-lite: Euler step
struct StepCoef64 {
  double lam, eta, span, dt;
  bool at_end;
};
__device__ __forceinline__ StepCoef64 load_coef(const double* p) {
  return {p[SF_P_LAMBDA_T], p[SF_P_ETA_T], p[SF_P_SPAN], p[SF_P_DT], p[SF_P_AT_END] != 0.0};
}

// velocity.py:125-130 in the latent dtype (coefficients rounded to it first, :120-122)
__device__ __forceinline__ double euler(double x, double e, const StepCoef64& c) {
  const double x_pred = __dadd_rn(__dmul_rn(c.lam, x), __dmul_rn(c.eta, e));
  const double v = c.at_end ? 0.0 : __ddiv_rn(__dsub_rn(x_pred, x), c.span);
  return __dadd_rn(x, __dmul_rn(c.dt, v));
}
__device__ __forceinline__ float euler(float x, float e, const StepCoef64& c) {
  const float lam = __double2float_rn(c.lam), eta = __double2float_rn(c.eta);
  const float span = __double2float_rn(c.span), dt = __double2float_rn(c.dt);
  const float x_pred = __fadd_rn(__fmul_rn(lam, x), __fmul_rn(eta, e));
  const float v = c.at_end ? 0.0f : __fdiv_rn(__fsub_rn(x_pred, x), span);
  return __fadd_rn(x, __fmul_rn(dt, v));
}
template <typename T>
__device__ __forceinline__ T cast_to(double v);
template <>
__device__ __forceinline__ double cast_to<double>(double v) { return v; }
template <>
__device__ __forceinline__ float cast_to<float>(double v) { return __double2float_rn(v); }
template <typename T>
__device__ __forceinline__ T cast_from_f32(float v);
template <>
__device__ __forceinline__ double cast_from_f32<double>(float v) { return (double)v; }
template <>
__device__ __forceinline__ float cast_from_f32<float>(float v) { return v; }

template <typename TX, typename TE>
__global__ void velocity_step_kernel(const TE* __restrict__ eps, const TX* x, TX* x_out,
                                     const double* __restrict__ params, int64_t B, int64_t D) {
  const int64_t row = blockIdx.y;
  const StepCoef64 c = load_coef(params + row * SF_PARAM_STRIDE);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t o = row * D + i;
    TX e;
    if constexpr (sizeof(TE) == 8) e = cast_to<TX>((double)eps[o]);
    else e = cast_from_f32<TX>((float)eps[o]);
    x_out[o] = euler(x[o], e, c);
  }
}

template <typename T>
__global__ void cfg_combine_kernel(const T* __restrict__ e2, int64_t B, int64_t D, double w, T* out) {
  const int64_t n = B * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const T u = e2[i], c = e2[i + n];
    if constexpr (sizeof(T) == 8) out[i] = __dadd_rn(u, __dmul_rn(w, __dsub_rn(c, u)));
    else out[i] = __fadd_rn(u, __fmul_rn((float)w, __fsub_rn(c, u)));
  }
}

// ============================================================ K12: mock velocity model
__constant__ uint64_t kB2IV[8] = {0x6a09e667f3bcc908ULL, 0xbb67ae8584caa73bULL, 0x3c6ef372fe94f82bULL,
                                  0xa54ff53a5f1d36f1ULL, 0x510e527fade682d1ULL, 0x9b05688c2b3e6c1fULL,
                                  0x1f83d9abfb41bd6bULL, 0x5be0cd19137e2179ULL};
__constant__ uint8_t kB2Sigma[12][16] = {
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3},
    {11, 8, 12, 0, 5, 2, 15, 13, 10, 14, 3, 6, 7, 1, 9, 4}, {7, 9, 3, 1, 13, 12, 11, 14, 2, 6, 5, 10, 4, 0, 15, 8},
    {9, 0, 5, 7, 2, 4, 10, 15, 14, 1, 11, 12, 6, 8, 3, 13}, {2, 12, 6, 10, 0, 11, 8, 3, 4, 13, 7, 5, 15, 14, 1, 9},
    {12, 5, 1, 15, 14, 13, 4, 10, 0, 7, 6, 3, 9, 2, 8, 11}, {13, 11, 7, 14, 12, 1, 3, 9, 5, 0, 15, 4, 8, 6, 2, 10},
    {6, 15, 14, 9, 11, 3, 0, 8, 12, 2, 13, 7, 1, 4, 10, 5}, {10, 2, 8, 4, 7, 6, 1, 5, 15, 11, 9, 14, 3, 12, 13, 0},
    {0, 1, 2, 3, 4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14, 15}, {14, 10, 4, 8, 9, 15, 13, 6, 1, 12, 0, 2, 11, 7, 5, 3}};

__device__ __forceinline__ uint64_t rotr64(uint64_t x, int n) { return (x >> n) | (x << (64 - n)); }

__device__ void blake2b_compress(uint64_t h[8], const uint64_t m[16], uint64_t t, bool last) {
  uint64_t v[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = h[i];
    v[i + 8] = kB2IV[i];
  }
  v[12] ^= t;
  if (last) v[14] = ~v[14];
#define B2G(a, b, c, d, x, y)       \
  a = a + b + x;                    \
  d = rotr64(d ^ a, 32);            \
  c = c + d;                        \
  b = rotr64(b ^ c, 24);            \
  a = a + b + y;                    \
  d = rotr64(d ^ a, 16);            \
  c = c + d;                        \
  b = rotr64(b ^ c, 63);
  for (int r = 0; r < 12; ++r) {
    const uint8_t* s = kB2Sigma[r];
    B2G(v[0], v[4], v[8], v[12], m[s[0]], m[s[1]]);
    B2G(v[1], v[5], v[9], v[13], m[s[2]], m[s[3]]);
    B2G(v[2], v[6], v[10], v[14], m[s[4]], m[s[5]]);
    B2G(v[3], v[7], v[11], v[15], m[s[6]], m[s[7]]);
    B2G(v[0], v[5], v[10], v[15], m[s[8]], m[s[9]]);
    B2G(v[1], v[6], v[11], v[12], m[s[10]], m[s[11]]);
    B2G(v[2], v[7], v[8], v[13], m[s[12]], m[s[13]]);
    B2G(v[3], v[4], v[9], v[14], m[s[14]], m[s[15]]);
  }
#undef B2G
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] ^= v[i] ^ v[i + 8];
}

// blake2b(digest_size=8) of <qqq(seed, id, round(t*1e9)) || emb[:E] (fp64 LE) (models.py:223-228)
__device__ uint64_t mock_row_key(int64_t seed, int64_t id, double t, const double* emb, int E) {
  const int64_t tq = __double2ll_rn(__dmul_rn(t, 1e9));  // Python round(): nearest, ties to even
  const int nwords = 3 + E;
  const int nbytes = nwords * 8;
  uint64_t h[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) h[i] = kB2IV[i];
  h[0] ^= 0x01010000ULL ^ 8ULL;
  uint64_t m[16];
  int w = 0;  // next message word
  uint64_t counted = 0;
  while (true) {
    const int remaining = nwords - w;
    const bool last = remaining <= 16;
    for (int i = 0; i < 16; ++i) {
      const int gw = w + i;
      uint64_t word = 0;
      if (gw < nwords) {
        if (gw == 0) word = (uint64_t)seed;
        else if (gw == 1) word = (uint64_t)id;
        else if (gw == 2) word = (uint64_t)tq;
        else word = (uint64_t)__double_as_longlong(emb[gw - 3]);
      }
      m[i] = word;
    }
    counted += last ? (uint64_t)(nbytes - w * 8) : 128ULL;
    blake2b_compress(h, m, counted, last);
    if (last) break;
    w += 16;
  }
  return h[0];
}

// splitmix64 finaliser of coordinate j, mapped to [-1, 1) (models.py:188-196)
__device__ __forceinline__ double splitmix_unit(uint64_t key, uint64_t j) {
  uint64_t z = key ^ (j * 0x9E3779B97F4A7C15ULL);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
  z = z ^ (z >> 31);
  const double unit = __dmul_rn((double)(z >> 11), 0x1.0p-53);
  return __dsub_rn(__dmul_rn(2.0, unit), 1.0);
}

__global__ void mock_keys_kernel(int64_t seed, const int64_t* ids, const double* ts, const double* embs, int64_t B,
                                 int E, uint64_t* keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < B) keys[i] = mock_row_key(seed, ids[i], ts[i], embs + i * E, E);
}

__global__ void mock_eps_kernel(const uint64_t* __restrict__ keys, int64_t B, int64_t D, double* out) {
  const int64_t row = blockIdx.y;
  const uint64_t key = keys[row];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < D; j += (int64_t)gridDim.x * blockDim.x)
    out[row * D + j] = splitmix_unit(key, (uint64_t)j);
}

// ============================================================ K11: device ring buffer
__global__ void stream_prepare_kernel(int64_t* ctl, int64_t S, int n, int64_t m, const double* stage_params,
                                      int64_t* row_info, double* row_t) {
  const int64_t j = ctl[0];
  for (int64_t r = threadIdx.x; r < S * n; r += blockDim.x) {
    const int64_t s = r / n, k = r % n;
    const int64_t stage = (((j - k) % n) + n) % n;
    const int64_t g = j - stage;
    row_info[r * 4 + 0] = stage;
    row_info[r * 4 + 1] = g;
    row_info[r * 4 + 2] = (g >= 0 && g < m) ? 1 : 0;
    row_info[r * 4 + 3] = s;
    row_t[r] = stage_params[stage * SF_PARAM_STRIDE + SF_P_T];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ctl[1] = j;
    ctl[0] = j + 1;
  }
}

// The mock's blake2b row keys of every ring row, one thread per (row, cond / uncond key): computed
// once per step in parallel instead of by one thread of each of the step kernel's blocks (the
// serial blake2b on that thread bounded the step: 360 -> see profiles/r02s3/experiments.md).
// keys[2 r + 1] = cond key, keys[2 r] = uncond key (guided rows only).
__global__ void stream_mock_keys_kernel(int64_t R, const int64_t* __restrict__ row_info,
                                        const double* __restrict__ row_t, int64_t seed, const double* emb,
                                        const double* neg, int E, double w, const double* __restrict__ w_streams,
                                        uint64_t* __restrict__ keys) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= 2 * R) return;
  const int64_t r = i >> 1;
  const bool cond = i & 1;
  if (row_info[r * 4 + 2] == 0) return;  // inactive row: no eps
  const int64_t g = row_info[r * 4 + 1], s = row_info[r * 4 + 3];
  const double ws = w_streams ? w_streams[s] : w;
  if (!cond && ws == 1.0) return;  // unguided (pipeline.py:113): no uncond half
  // apply_cfg (models.py:257-268): the uncond half uses the negative embedding (zeros when absent)
  double zeros[64];
  const double* e = emb + s * E;
  if (!cond) {
    if (neg) {
      e = neg + s * E;
    } else {
      for (int k = 0; k < E; ++k) zeros[k] = 0.0;
      e = zeros;
    }
  }
  keys[i] = mock_row_key(seed, g, row_t[r], e, E);
}

// One block = (chunk of D, ring row).  Guided mock eps -> Euler -> emit -> refill.
template <typename TX>
__global__ void stream_mock_step_kernel(const int64_t* ctl, int64_t S, int n, int64_t m, int64_t D, TX* x_ring,
                                        const double* __restrict__ stage_params, const int64_t* __restrict__ row_info,
                                        const uint64_t* __restrict__ keys, double w,
                                        const double* __restrict__ w_streams, const double* __restrict__ noise_in,
                                        TX* frames_out, int64_t* frame_ids) {
  const int64_t r = blockIdx.y;
  const int64_t j = ctl[1];
  const int64_t stage = row_info[r * 4 + 0];
  const int64_t g = row_info[r * 4 + 1];
  const bool active = row_info[r * 4 + 2] != 0;
  const int64_t s = row_info[r * 4 + 3];
  const int64_t k = r % n;
  const bool refill_slot = (k == (j + 1) % n);
  const bool admit = refill_slot && (j + 1 < m);
  const bool retiring = active && (stage + 1 == n);
  const double ws = w_streams ? w_streams[s] : w;  // this stream's guidance scale
  const bool guided = (ws != 1.0);                 // pipeline.py:113
  const uint64_t key_c = active ? keys[2 * r + 1] : 0, key_u = (active && guided) ? keys[2 * r] : 0;
  if (blockIdx.x == 0 && threadIdx.x == 0 && refill_slot) frame_ids[s] = retiring ? g : -1;
  const StepCoef64 c = load_coef(stage_params + stage * SF_PARAM_STRIDE);
  TX* xr = x_ring + r * D;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x) {
    if (active) {
      double e = splitmix_unit(key_c, (uint64_t)i);
      if (guided) {  // handle_cfg (models.py:288-293), fp64 like the mock's output
        const double eu = splitmix_unit(key_u, (uint64_t)i);
        e = __dadd_rn(eu, __dmul_rn(ws, __dsub_rn(e, eu)));
      }
      const TX xn = euler(xr[i], cast_to<TX>(e), c);
      if (retiring) frames_out[s * D + i] = xn;
      xr[i] = admit ? cast_to<TX>(noise_in[s * D + i]) : xn;
    } else if (admit) {
      xr[i] = cast_to<TX>(noise_in[s * D + i]);
    }
  }
}

template <typename TX>
__global__ void stream_reset_kernel(int64_t* ctl, int64_t S, int n, int64_t D, TX* x_ring, const double* noise0) {
  const int64_t s = blockIdx.y;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < D; i += (int64_t)gridDim.x * blockDim.x)
    x_ring[(s * n) * D + i] = cast_to<TX>(noise0[s * D + i]);
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0) {
    ctl[0] = 0;
    ctl[1] = -1;
  }
}

static inline int grid_for(int64_t n, int threads) {
  int64_t b = (n + threads - 1) / threads;
  return (int)(b > 65535 ? 65535 : (b < 1 ? 1 : b));
}

}  // namespace sf

using namespace sf;

namespace sf {
// ---------------------------------------------------------------- K13: analytic linear model
// eps_i = A x_i + t_i b (models.py:176-185), fp64, row by row: output (i, j) is a
// sequential fp64 dot product over k, so a row's result never depends on the
// batch it was submitted in (dispatcher bit-identity, models.py:142-146).
template <typename XT>
__global__ void analytic_eps_kernel(const double* __restrict__ A, const double* __restrict__ bvec,
                                    const XT* __restrict__ x, const double* __restrict__ ts, int64_t D,
                                    double* __restrict__ out) {
  const int64_t i = blockIdx.y;
  const XT* xi = x + i * D;
  const double ti = ts[i];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < D; j += (int64_t)gridDim.x * blockDim.x) {
    const double* aj = A + j * D;
    double acc = 0.0;
    for (int64_t k = 0; k < D; ++k) acc = __dadd_rn(acc, __dmul_rn(aj[k], (double)xi[k]));
    out[i * D + j] = __dadd_rn(acc, __dmul_rn(ti, bvec[j]));
  }
}

}  // namespace sf

extern "C" {

int sf_schedule_indices(const sf_schedule* sched, const double* ts, int64_t B, int64_t* abar_idx, int64_t* grid_idx,
                        uint32_t* status, void* stream) {
  if (!sched || !ts || B < 1 || sched->t_max < 1 || (grid_idx && (!status || sched->num_steps < 1 || !sched->grid)))
    return SF_ERR_PARAMETER;
  schedule_indices_kernel<<<(unsigned)((B + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*sched, ts, B, abar_idx,
                                                                                         grid_idx, status);
  return cuda_status();
}

int sf_window_params(const sf_schedule* sched, const double* ts, int64_t B, double* out, uint32_t* status,
                     void* stream) {
  if (!sched || B < 0 || sched->num_windows < 1 || sched->num_steps < 1 || sched->t_max < 2) return SF_ERR_PARAMETER;
  if (B == 0) return SF_OK;
  window_params_kernel<<<grid_for(B, 128), 128, 0, (cudaStream_t)stream>>>(*sched, ts, B, out, status);
  return cuda_status();
}

int sf_velocity_step(const void* eps, int eps_dtype, const void* x, void* x_out, int x_dtype, const double* params,
                     int64_t B, int64_t D, void* stream) {
  if (B < 0 || D < 0) return SF_ERR_PARAMETER;
  if (B == 0 || D == 0) return SF_OK;
  if (B > 65535) return SF_ERR_PARAMETER;
  dim3 grid(grid_for(D, 256) > 64 ? 64 : grid_for(D, 256), (unsigned)B);
  cudaStream_t st = (cudaStream_t)stream;
  if (x_dtype == SF_F64 && eps_dtype == SF_F64)
    velocity_step_kernel<double, double><<<grid, 256, 0, st>>>((const double*)eps, (const double*)x, (double*)x_out,
                                                                params, B, D);
  else if (x_dtype == SF_F64 && eps_dtype == SF_F32)
    velocity_step_kernel<double, float><<<grid, 256, 0, st>>>((const float*)eps, (const double*)x, (double*)x_out,
                                                               params, B, D);
  else if (x_dtype == SF_F32 && eps_dtype == SF_F64)
    velocity_step_kernel<float, double><<<grid, 256, 0, st>>>((const double*)eps, (const float*)x, (float*)x_out,
                                                               params, B, D);
  else if (x_dtype == SF_F32 && eps_dtype == SF_F32)
    velocity_step_kernel<float, float><<<grid, 256, 0, st>>>((const float*)eps, (const float*)x, (float*)x_out,
                                                              params, B, D);
  else
    return SF_ERR_PARAMETER;
  return cuda_status();
}

int sf_cfg_combine(const void* eps2, int dtype, int64_t B, int64_t D, double w, void* out, void* stream) {
  if (B < 0 || D < 0) return SF_ERR_PARAMETER;
  if (B * D == 0) return SF_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == SF_F64)
    cfg_combine_kernel<double><<<grid_for(B * D, 256), 256, 0, st>>>((const double*)eps2, B, D, w, (double*)out);
  else if (dtype == SF_F32)
    cfg_combine_kernel<float><<<grid_for(B * D, 256), 256, 0, st>>>((const float*)eps2, B, D, w, (float*)out);
  else
    return SF_ERR_PARAMETER;
  return cuda_status();
}

int sf_mock_keys(int64_t model_seed, const int64_t* ids, const double* ts, const double* row_embs, int64_t B,
                 int32_t E, uint64_t* keys, void* stream) {
  if (B < 0 || E < 1 || E > 64) return SF_ERR_PARAMETER;
  if (B == 0) return SF_OK;
  mock_keys_kernel<<<grid_for(B, 64), 64, 0, (cudaStream_t)stream>>>(model_seed, ids, ts, row_embs, B, E, keys);
  return cuda_status();
}

int sf_analytic_eps(const double* A, const double* b, const void* x, int x_dtype, const double* ts, int64_t B,
                    int64_t D, double* out, void* stream) {
  if (B < 0 || D < 1 || B > 65535 || (x_dtype != SF_F64 && x_dtype != SF_F32)) return SF_ERR_PARAMETER;
  if (B == 0) return SF_OK;
  dim3 grid(grid_for(D, 128) > 64 ? 64 : grid_for(D, 128), (unsigned)B);
  cudaStream_t st = (cudaStream_t)stream;
  if (x_dtype == SF_F64)
    sf::analytic_eps_kernel<double><<<grid, 128, 0, st>>>(A, b, (const double*)x, ts, D, out);
  else
    sf::analytic_eps_kernel<float><<<grid, 128, 0, st>>>(A, b, (const float*)x, ts, D, out);
  return cuda_status();
}

int sf_mock_eps(const uint64_t* keys, int64_t B, int64_t D, double* out, void* stream) {
  if (B < 0 || D < 0 || B > 65535) return SF_ERR_PARAMETER;
  if (B * D == 0) return SF_OK;
  dim3 grid(grid_for(D, 256) > 64 ? 64 : grid_for(D, 256), (unsigned)B);
  mock_eps_kernel<<<grid, 256, 0, (cudaStream_t)stream>>>(keys, B, D, out);
  return cuda_status();
}

int sf_stream_prepare(int64_t* ctl, int64_t S, int32_t n, int64_t m, const double* stage_params, int64_t* row_info,
                      double* row_t, void* stream) {
  if (S < 1 || n < 1 || m < 1) return SF_ERR_PARAMETER;
  stream_prepare_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(ctl, S, n, m, stage_params, row_info, row_t);
  return cuda_status();
}

int sf_stream_mock_step(const int64_t* ctl, int64_t S, int32_t n, int64_t m, int64_t D, int x_dtype, void* x_ring,
                        const double* stage_params, const int64_t* row_info, const double* row_t, int64_t model_seed,
                        const double* emb, const double* neg, int32_t E, double w, const double* w_streams,
                        const double* noise_in, void* frames_out, int64_t* frame_ids, uint64_t* keys,
                        void* stream) {
  if (S < 1 || n < 1 || m < 1 || D < 1 || E < 1 || E > 64 || S * n > 65535 || !keys) return SF_ERR_PARAMETER;
  if (x_dtype != SF_F64 && x_dtype != SF_F32) return SF_ERR_PARAMETER;
  const int64_t R = S * n;
  cudaStream_t st = (cudaStream_t)stream;
  stream_mock_keys_kernel<<<(unsigned)((2 * R + 127) / 128), 128, 0, st>>>(R, row_info, row_t, model_seed, emb, neg, E,
                                                                          w, w_streams, keys);
  dim3 grid(grid_for(D, 256) > 16 ? 16 : grid_for(D, 256), (unsigned)R);
  if (x_dtype == SF_F64)
    stream_mock_step_kernel<double><<<grid, 256, 0, st>>>(ctl, S, n, m, D, (double*)x_ring, stage_params, row_info,
                                                          keys, w, w_streams, noise_in, (double*)frames_out,
                                                          frame_ids);
  else
    stream_mock_step_kernel<float><<<grid, 256, 0, st>>>(ctl, S, n, m, D, (float*)x_ring, stage_params, row_info,
                                                         keys, w, w_streams, noise_in, (float*)frames_out,
                                                         frame_ids);
  return cuda_status();
}

int sf_stream_reset(int64_t* ctl, int64_t S, int32_t n, int64_t D, int x_dtype, void* x_ring, const double* noise0,
                    void* stream) {
  if (S < 1 || n < 1 || D < 1 || S > 65535) return SF_ERR_PARAMETER;
  dim3 grid(grid_for(D, 256) > 16 ? 16 : grid_for(D, 256), (unsigned)S);
  cudaStream_t st = (cudaStream_t)stream;
  if (x_dtype == SF_F64)
    stream_reset_kernel<double><<<grid, 256, 0, st>>>(ctl, S, n, D, (double*)x_ring, noise0);
  else if (x_dtype == SF_F32)
    stream_reset_kernel<float><<<grid, 256, 0, st>>>(ctl, S, n, D, (float*)x_ring, noise0);
  else
    return SF_ERR_PARAMETER;
  return cuda_status();
}

}  // extern "C"

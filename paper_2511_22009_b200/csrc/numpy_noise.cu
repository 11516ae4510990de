// Generation noise identical to numpy, on the device.
//
// The reference draws a generation's initial latent with
//   np.random.default_rng([seed, gen_id]).standard_normal(dim)      (src/pipeline.py:92-98)
// i.e. SeedSequence -> PCG64 (XSL-RR 128/64) -> 256-level ziggurat.  This kernel
// reproduces those bits (fp64, or their fp32 cast as pipeline.py:176 does), so the
// parity-mode stream batch no longer computes noise on the host and uploads it.
//
// Layout: one CTA per generation row, 256 threads.  Thread t owns PCG64 draw
// t of every 256-draw round (its own LCG state, advanced by the 256-step jump
// (A^256, c_256) each round).  ~99% of draws take the ziggurat fast path and map
// to one output each; the rare rejection draws (wedge / tail, which consume
// further uniforms from the same stream) are evaluated speculatively by their own
// threads (stepping the LCG from their own state), and one thread walks them in
// sequence order to decide which are live (a draw consumed by an earlier rejection
// draw is not).  A block scan over "this draw produces an output" gives every
// output its index.
//
// Floating point: every operation that decides or forms an output is written with
// explicit _rn intrinsics in numpy's literal order (no FMA contraction), except the
// tail's log1p, which restates this platform's glibc 2.39 x86-64 FMA log1p
// (libm ifunc variant; checked bit-for-bit against math.log1p in
// tests/test_noise_oracle.py), and the wedge test's exp(), which is only compared
// against (a mismatch needs a uniform within one ulp of exp's value).
#include <cstdint>

#include "sf_internal.h"

#define SF_ZIG_QUAL static __device__ const
#include "ziggurat_tables.h"

namespace sf {
namespace npn {

typedef unsigned __int128 u128;
constexpr int T = 256;
constexpr uint64_t MULT_HI = 2549297995355413924ULL, MULT_LO = 4865540595714422341ULL;
constexpr double ZIG_R = 3.6541528853610088, ZIG_INV_R = 0.27366123732975828;

__device__ __forceinline__ u128 mult() { return ((u128)MULT_HI << 64) | MULT_LO; }
__device__ __forceinline__ u128 step(u128 s, u128 inc) { return s * mult() + inc; }

// pcg_output_xsl_rr_128_64
__device__ __forceinline__ uint64_t xsl_rr(u128 s) {
  const uint64_t v = (uint64_t)(s >> 64) ^ (uint64_t)s;
  const unsigned rot = (unsigned)(s >> 122);
  return (v >> rot) | (v << ((64u - rot) & 63u));
}
__device__ __forceinline__ double next_double(uint64_t r) {
  return __dmul_rn((double)(r >> 11), 1.0 / 9007199254740992.0);
}

// S_{i+delta} = am * S_i + ap (pcg advance)
__device__ void lcg_jump(u128 inc, uint64_t delta, u128& am, u128& ap) {
  u128 cm = mult(), cp = inc;
  am = 1;
  ap = 0;
  while (delta) {
    if (delta & 1) {
      am *= cm;
      ap = ap * cm + cp;
    }
    cp = (cm + 1) * cp;
    cm *= cm;
    delta >>= 1;
  }
}

// SeedSequence([seed, gen]).generate_state(4, uint64) -> PCG64 srandom (bit_generator.pyx,
// pcg64.h pcg_setseq_128_srandom_r).
__device__ void seed_pcg64(uint64_t seed, uint64_t gen, u128& state, u128& inc) {
  uint32_t ent[4];
  int n = 0;
  for (uint64_t v : {seed, gen}) {
    if (v == 0) ent[n++] = 0;
    while (v) {
      ent[n++] = (uint32_t)v;
      v >>= 32;
    }
  }
  uint32_t hc = 0x43b0d7e5u;
  auto hashmix = [&](uint32_t v) {
    v ^= hc;
    hc *= 0x931e8875u;
    v *= hc;
    return v ^ (v >> 16);
  };
  auto mix = [](uint32_t x, uint32_t y) {
    uint32_t r = 0xca01f9ddu * x - 0x4973f715u * y;
    return r ^ (r >> 16);
  };
  uint32_t pool[4];
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < n ? ent[i] : 0u);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s]));
  uint32_t hb = 0x8b51f9ddu, w[8];
  for (int i = 0; i < 8; ++i) {
    uint32_t v = pool[i & 3] ^ hb;
    hb *= 0x58f38dedu;
    v *= hb;
    w[i] = v ^ (v >> 16);
  }
  const uint64_t s0 = w[0] | ((uint64_t)w[1] << 32), s1 = w[2] | ((uint64_t)w[3] << 32);
  const uint64_t s2 = w[4] | ((uint64_t)w[5] << 32), s3 = w[6] | ((uint64_t)w[7] << 32);
  const u128 initstate = ((u128)s0 << 64) | s1, initseq = ((u128)s2 << 64) | s3;
  inc = (initseq << 1) | 1;
  u128 st = step(0, inc);
  st += initstate;
  state = step(st, inc);
}

// glibc 2.39 x86-64 log1p (FMA ifunc variant, fdlibm-derived), restated operation for
// operation; only the branches reachable from log1p(-u), u in [0, 1), plus x >= 0 below 2^53.
__device__ double glibc_log1p(double x) {
  const double LN2_HI = 6.93147180369123816490e-01, LN2_LO = 1.90821492927058770002e-10;
  const double LP1 = 6.666666666666735130e-01, LP2 = 3.999999999940941908e-01, LP3 = 2.857142874366239149e-01,
               LP4 = 2.222219843214978396e-01, LP5 = 1.818357216161805012e-01, LP6 = 1.531383769920937332e-01,
               LP7 = 1.479819860511658591e-01;
  const int32_t hx = (int32_t)(__double_as_longlong(x) >> 32);
  double f, c = 0.0, u;
  int k;
  uint32_t hu;
  if (hx <= 0x3fda8279) {
    const int32_t ax = hx & 0x7fffffff;
    if (ax > 0x3fefffff) return x == -1.0 ? -INFINITY : __longlong_as_double(0x7ff8000000000000LL);
    if (ax <= 0x3e1fffff) return ax <= 0x3c8fffff ? x : __fma_rn(-__dmul_rn(x, x), 0.5, x);
    if ((uint32_t)(hx + 0x402d413c) > 0x402d413cu) {  // -0.2929 < x < 0.41422: k = 0, f = x
      k = 0;
      f = x;
      hu = 1;
      goto poly;
    }
  } else if (hx > 0x7fefffff) {
    return __dadd_rn(x, x);
  }
  u = __dadd_rn(x, 1.0);
  {
    uint32_t h = (uint32_t)(__double_as_longlong(u) >> 32);
    k = (int)(h >> 20) - 1023;
    c = k > 0 ? __ddiv_rn(__dsub_rn(1.0, __dsub_rn(u, x)), u) : __ddiv_rn(__dsub_rn(x, __dsub_rn(u, 1.0)), u);
    hu = h & 0xfffffu;
    const uint64_t lo = (uint64_t)__double_as_longlong(u) & 0xffffffffull;
    if (hu <= 0x6a09du) {
      u = __longlong_as_double((long long)(((uint64_t)(hu | 0x3ff00000u) << 32) | lo));
    } else {
      k += 1;
      u = __longlong_as_double((long long)(((uint64_t)(hu | 0x3fe00000u) << 32) | lo));
      hu = (0x100000u - hu) >> 2;
    }
    f = __dsub_rn(u, 1.0);
  }
  if (hu == 0) {
    const double hfsq = __dmul_rn(__dmul_rn(f, 0.5), f);
    if (f == 0.0) {
      if (k == 0) return 0.0;
      const double kd = (double)k;
      return __fma_rn(kd, LN2_HI, __fma_rn(kd, LN2_LO, c));
    }
    const double R = __dmul_rn(__fma_rn(-f, 0.6666666666666666, 1.0), hfsq);
    if (k == 0) return __dsub_rn(f, R);
    const double kd = (double)k;
    return __fma_rn(kd, LN2_HI, -__dsub_rn(__dsub_rn(R, __fma_rn(kd, LN2_LO, c)), f));
  }
poly : {
  const double hfsq = __dmul_rn(__dmul_rn(f, 0.5), f);
  const double s = __ddiv_rn(f, __dadd_rn(f, 2.0));
  const double z = __dmul_rn(s, s);
  const double R2 = __fma_rn(z, LP3, LP2), R3 = __fma_rn(z, LP5, LP4), R4 = __fma_rn(z, LP7, LP6);
  const double z2 = __dmul_rn(z, z), z4 = __dmul_rn(z2, z2), z6 = __dmul_rn(z2, z4);
  double t = __fma_rn(z, LP1, __dmul_rn(z2, R2));
  t = __fma_rn(z4, R3, t);
  const double R = __fma_rn(z6, R4, t);
  const double w = __dmul_rn(__dadd_rn(R, hfsq), s);
  if (k == 0) return __dsub_rn(f, __dsub_rn(hfsq, w));
  const double kd = (double)k;
  return __fma_rn(kd, LN2_HI, -__dsub_rn(__dsub_rn(hfsq, __dadd_rn(__fma_rn(kd, LN2_LO, c), w)), f));
}
}

struct Draw {
  int idx;
  uint64_t rabs;
  double x;
};
__device__ __forceinline__ Draw ziggurat_draw(uint64_t r, const double* wi) {
  Draw d;
  d.idx = (int)(r & 0xff);
  r >>= 8;
  d.rabs = (r >> 1) & 0x000fffffffffffffull;
  d.x = __dmul_rn((double)d.rabs, wi[d.idx]);
  if (r & 1) d.x = -d.x;
  return d;
}

template <typename OUT>
__device__ __forceinline__ OUT cvt_out(double v);
template <>
__device__ __forceinline__ double cvt_out<double>(double v) {
  return v;
}
template <>
__device__ __forceinline__ float cvt_out<float>(double v) {
  return __double2float_rn(v);
}

template <typename OUT>
__global__ void __launch_bounds__(T) numpy_normal_kernel(const int64_t* __restrict__ seeds, int64_t gen, int64_t D,
                                                         OUT* __restrict__ out_all) {
  __shared__ uint64_t s_ki[256];
  __shared__ double s_wi[256], s_fi[256];
  __shared__ double s_val[T];
  __shared__ uint32_t s_special[T / 32], s_spec_acc[T / 32], s_consumed[T / 32], s_accept[T / 32];
  __shared__ long long s_pos[T];  // a rejection draw's first draw after the ones it consumes
  __shared__ int s_cnt[T / 32];
  __shared__ u128 s_seed[2];
  __shared__ long long s_skip;

  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  s_ki[t] = SF_ZIG_KI[t];
  s_wi[t] = SF_ZIG_WI[t];
  s_fi[t] = SF_ZIG_FI[t];
  if (t == 0) {
    u128 st, inc;
    seed_pcg64((uint64_t)seeds[blockIdx.x], (uint64_t)gen, st, inc);
    s_seed[0] = st;
    s_seed[1] = inc;
    s_skip = 0;
  }
  __syncthreads();
  const u128 inc = s_seed[1];
  u128 st;
  {
    u128 am, ap;
    lcg_jump(inc, (uint64_t)t + 1, am, ap);  // draw t comes from S_{t+1}
    st = am * s_seed[0] + ap;
  }
  u128 jm, jp;
  lcg_jump(inc, T, jm, jp);
  OUT* out = out_all + (int64_t)blockIdx.x * D;

  long long out_base = 0, round_base = 0;
  while (out_base < D) {
    const Draw d = ziggurat_draw(xsl_rr(st), s_wi);
    const bool fast = d.rabs < s_ki[d.idx];
    // A rejection draw (wedge / tail, distributions.c random_standard_normal) is evaluated by its
    // own thread, speculatively (as if no earlier rejection draw consumed it): its outcome and the
    // extra draws it consumes depend only on the raw stream, so one thread then only has to walk
    // the round's rejection draws in sequence order to decide which are live.
    bool acc = false;
    if (!fast) {
      u128 cs = st;
      long long pos = round_base + t + 1;
      double val = d.x;
      if (d.idx == 0) {
        for (;;) {
          cs = step(cs, inc);
          const double u1 = next_double(xsl_rr(cs));
          cs = step(cs, inc);
          const double u2 = next_double(xsl_rr(cs));
          pos += 2;
          const double xx = __dmul_rn(-ZIG_INV_R, glibc_log1p(-u1));
          const double yy = -glibc_log1p(-u2);
          if (__dadd_rn(yy, yy) > __dmul_rn(xx, xx)) {
            val = ((d.rabs >> 8) & 1) ? -__dadd_rn(ZIG_R, xx) : __dadd_rn(ZIG_R, xx);
            break;
          }
        }
        acc = true;
      } else {
        cs = step(cs, inc);
        const double u = next_double(xsl_rr(cs));
        pos += 1;
        const double lhs = __dadd_rn(__dmul_rn(__dsub_rn(s_fi[d.idx - 1], s_fi[d.idx]), u), s_fi[d.idx]);
        acc = lhs < exp(__dmul_rn(__dmul_rn(-0.5, d.x), d.x));
      }
      s_pos[t] = pos;
      s_val[t] = val;
    }
    const uint32_t spec = __ballot_sync(0xffffffffu, !fast);
    const uint32_t spec_acc = __ballot_sync(0xffffffffu, !fast && acc);
    if (lane == 0) {
      s_special[w] = spec;
      s_spec_acc[w] = spec_acc;
    }
    __syncthreads();
    if (t == 0) {
      // the live rejection draws of this round, in sequence order; draws a live one consumes are
      // not outputs of their own
      long long skip = s_skip;
      const long long round_end = round_base + T;
      for (int k = 0; k < T / 32; ++k) s_consumed[k] = s_accept[k] = 0;
      auto mark = [&](long long a, long long b) {  // consumed global draws [a, b) within this round
        a = a < round_base ? round_base : a;
        b = b > round_end ? round_end : b;
        for (long long g = a; g < b; ++g) s_consumed[(g - round_base) >> 5] |= 1u << ((g - round_base) & 31);
      };
      mark(round_base, skip);
      for (int k = 0; k < T / 32; ++k) {
        uint32_t m = s_special[k];
        while (m) {
          const int p = k * 32 + __ffs(m) - 1;
          m &= m - 1;
          const long long g = round_base + p;
          if (g < skip) continue;
          const long long pos = s_pos[p];
          mark(g + 1, pos);
          skip = pos;
          s_accept[k] |= s_spec_acc[k] & (1u << (p & 31));
        }
      }
      s_skip = skip > round_end ? skip : round_end;
    }
    __syncthreads();
    const bool produces = !((s_consumed[w] >> lane) & 1) && (fast || ((s_accept[w] >> lane) & 1));
    const uint32_t b = __ballot_sync(0xffffffffu, produces);
    if (lane == 0) s_cnt[w] = __popc(b);
    __syncthreads();
    int prefix = __popc(b & ((1u << lane) - 1)), total = 0;
#pragma unroll
    for (int k = 0; k < T / 32; ++k) {
      prefix += k < w ? s_cnt[k] : 0;
      total += s_cnt[k];
    }
    if (produces && out_base + prefix < D) out[out_base + prefix] = cvt_out<OUT>(fast ? d.x : s_val[t]);
    out_base += total;
    round_base += T;
    st = jm * st + jp;
    __syncthreads();
  }
}

}  // namespace npn
}  // namespace sf

extern "C" {

int sf_numpy_normal(const int64_t* seeds, int64_t gen, int64_t S, int64_t D, void* out, int out_dtype,
                    void* stream) {
  if (S < 1 || S > 2147483647 || D < 1 || gen < 0 || !seeds || !out) return SF_ERR_PARAMETER;
  cudaStream_t st = (cudaStream_t)stream;
  if (out_dtype == SF_F64)
    sf::npn::numpy_normal_kernel<double><<<(unsigned)S, sf::npn::T, 0, st>>>(seeds, gen, D, (double*)out);
  else if (out_dtype == SF_F32)
    sf::npn::numpy_normal_kernel<float><<<(unsigned)S, sf::npn::T, 0, st>>>(seeds, gen, D, (float*)out);
  else
    return SF_ERR_PARAMETER;
  return sf::cuda_status();
}

}  // extern "C"

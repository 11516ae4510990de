/*
 * streamflow.h -- C ABI of the B200-native StreamFlow stream-batch hot path.
 *
 * The reference (`flowpipe`, /root/reference/pkg/src/flowpipe) is a pure
 * Python/numpy package with no FFI; its boundary is a Python API.  This header
 * is the native boundary our Python drop-in (package `paper_2511_22009_b200`)
 * binds with ctypes; every entry point names the reference function it
 * replaces (file:line, relative to pkg/src/flowpipe/).
 *
 * Conventions
 *  - Plain pointers and sizes only.  All array pointers are DEVICE pointers
 *    owned by the caller; the library never allocates device memory on the
 *    hot path (the DiT runtime handle holds host-side state only).
 *  - `stream` is a cudaStream_t passed as void*; every call is stream-ordered,
 *    asynchronous and reentrant.
 *  - Return value: SF_OK (0) or a negative SF_ERR_* code.  Error kinds map to
 *    the reference's exception classes (errors.py:4-39).  Data-dependent
 *    checks (off-grid t, non-positive window denominator) are reported through
 *    a device-side `status` word with the SF_STATUS_* bits; the caller reads it
 *    when it needs to raise.
 */
#ifndef STREAMFLOW_H_
#define STREAMFLOW_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status / error codes (errors.py:4-39) ---- */
#define SF_OK 0
#define SF_ERR_PARAMETER (-1)   /* ParameterError   (errors.py:8)  */
#define SF_ERR_TIME_DOMAIN (-2) /* TimeDomainError  (errors.py:12) */
#define SF_ERR_INVARIANT (-3)   /* InvariantError   (errors.py:24) */
#define SF_ERR_STATE (-4)       /* StateError       (errors.py:16) */
#define SF_ERR_CUDA (-5)        /* CUDA launch / driver failure    */

#define SF_STATUS_TIME_RANGE 1u /* t outside [0,1]        schedule.py:195-198 */
#define SF_STATUS_OFF_GRID 2u   /* t not on the grid      schedule.py:279-283 */
#define SF_STATUS_DENOM 4u      /* denominator <= 0       schedule.py:248-252 */

/* ---- dtypes ---- */
#define SF_F32 0
#define SF_F64 1
#define SF_BF16 2

/* Per-row step coefficients written by sf_window_params: SF_PARAM_STRIDE
 * doubles per row, in this order. */
#define SF_P_T 0
#define SF_P_TNEXT 1
#define SF_P_TS 2
#define SF_P_TE 3
#define SF_P_GAMMA 4
#define SF_P_LAMBDA_S 5
#define SF_P_ETA_S 6
#define SF_P_LAMBDA_T 7
#define SF_P_ETA_T 8
#define SF_P_SPAN 9
#define SF_P_DT 10
#define SF_P_AT_END 11 /* 1.0 / 0.0 */
#define SF_PARAM_STRIDE 12

/* Device-resident scheduler arguments (schedule.py:87-133): boundaries
 * [num_windows+1], abar [t_max], grid [num_steps], all fp64 device arrays. */
typedef struct sf_schedule {
  const double* boundaries;
  const double* abar;
  const double* grid;
  int32_t num_windows;
  int32_t t_max;
  int32_t num_steps;
  int32_t _pad;
  double eps;
} sf_schedule;

const char* sf_version(void);
int sf_device_sm_count(void);

/* Table indices of flow times (schedule.py:201-205 alpha_bar_index and :266-284
 * grid_indices): abar_idx[i] = clip(floor((1 - t) (t_max - 1) + 0.5)), grid_idx[i] =
 * nearest inference-grid point (either output may be NULL; grid_idx needs the grid and
 * status, where SF_STATUS_OFF_GRID / SF_STATUS_TIME_RANGE are OR-ed). */
int sf_schedule_indices(const sf_schedule* sched, const double* ts, int64_t B, int64_t* abar_idx, int64_t* grid_idx,
                        uint32_t* status, void* stream);

/* K1 -- window coefficients + grid successor for B flow times.
 * Replaces window_params (schedule.py:224-263), window_lookup (:208-221),
 * alpha_bar_index (:201-205), next_timestep / grid_indices (:266-295).
 * out: [B, SF_PARAM_STRIDE] fp64.  status: device uint32, OR-ed SF_STATUS_*.
 * Off-grid rows get t_next = NaN (the caller raises TimeDomainError). */
int sf_window_params(const sf_schedule* sched, const double* ts, int64_t B, double* out, uint32_t* status,
                     void* stream);

/* K10-lite -- heterogeneous-t Euler step, bit-exact with numpy.
 * Replaces batched_velocity_step (velocity.py:93-135).
 * eps: [B, D] of eps_dtype (F32/F64); x, x_out: [B, D] of x_dtype (F32/F64);
 * params: [B, SF_PARAM_STRIDE] from sf_window_params.  x_out may alias x. */
int sf_velocity_step(const void* eps, int eps_dtype, const void* x, void* x_out, int x_dtype, const double* params,
                     int64_t B, int64_t D, void* stream);

/* CFG combine: out[i] = e[i] + w * (e[i+B] - e[i]) over a [2B, D] block.
 * Replaces handle_cfg (models.py:278-296); fp64 or fp32. */
int sf_cfg_combine(const void* eps2, int dtype, int64_t B, int64_t D, double w, void* out, void* stream);

/* K12 -- seeded mock velocity model (models.py:199-241).
 * sf_mock_keys: blake2b-64 row keys of (model_seed, ids[i], round(ts[i]*1e9),
 *   row_embs[i, :E]) (models.py:223-228).  row_embs: [B, E] fp64.
 * sf_mock_eps: splitmix64 expansion of each key into D fp64 values in
 *   [-1, 1) (models.py:188-196), out [B, D]. */
int sf_mock_keys(int64_t model_seed, const int64_t* ids, const double* ts, const double* row_embs, int64_t B,
                 int32_t E, uint64_t* keys, void* stream);
int sf_mock_eps(const uint64_t* keys, int64_t B, int64_t D, double* out, void* stream);

/* K13 -- AnalyticLinearModel._compute (models.py:176-185): eps_i = A x_i + t_i b in fp64,
 * row by row (batch-decomposition invariant).  A [D, D] and b [D] fp64, x [B, D] in
 * x_dtype (SF_F64 / SF_F32), ts [B] fp64 -> out [B, D] fp64. */
int sf_analytic_eps(const double* A, const double* b, const void* x, int x_dtype, const double* ts, int64_t B,
                    int64_t D, double* out, void* stream);

/* ---- device-resident stream batch (pipeline.py:139-220) ----
 * S independent streams x n in-flight slots.  Ring row r = s*n + k holds the
 * generation g of stream s with g = k (mod n); at iteration j its stage is
 * (j - k) mod n and it is active iff 0 <= g < m.  The
 * queue shift is the implicit advance of j; nothing moves in memory.
 *
 * ctl: device int64[4]: [0] = next iteration j, [1] = iteration being run.
 * stage_params: [n, SF_PARAM_STRIDE] (sf_window_params of grid[:n]).
 * row_info: device int64[S*n*4] written by sf_stream_prepare:
 *   [r*4+0] stage, [r*4+1] gen id, [r*4+2] active, [r*4+3] stream.
 * row_t: device fp64[S*n] flow time of each ring row. */
int sf_stream_prepare(int64_t* ctl, int64_t S, int32_t n, int64_t m, const double* stage_params, int64_t* row_info,
                      double* row_t, void* stream);

/* Mock-model stream step: guided mock eps (CFG fused when w != 1) + Euler on
 * every active ring row + emission of retiring rows + refill of the slot that
 * admits generation j+1.
 *   x_ring [S*n, D] (x_dtype), frames_out [S, D] (x_dtype), frame_ids [S]
 *   (-1 when nothing retired this iteration), noise_in [S, D] fp64: initial
 *   noise of generation j+1 per stream (pipeline.py:92-98), ignored when
 *   j+1 >= m.  emb / neg: [S, E] fp64 (neg may be NULL = zeros,
 *   models.py:258-260).  model_seed: SeededMockModel seed.  w_streams: NULL (every
 *   stream uses w) or device fp64 [S] per-stream guidance scales (a stream with
 *   w_s == 1 runs unguided, exactly as its own run_stream would).  keys: device scratch of
 *   2 * S * n uint64 (the step's blake2b row keys, computed by a first launch). */
int sf_stream_mock_step(const int64_t* ctl, int64_t S, int32_t n, int64_t m, int64_t D, int x_dtype, void* x_ring,
                        const double* stage_params, const int64_t* row_info, const double* row_t, int64_t model_seed,
                        const double* emb, const double* neg, int32_t E, double w, const double* w_streams,
                        const double* noise_in, void* frames_out, int64_t* frame_ids, uint64_t* keys,
                        void* stream);

/* Write generation-0 noise into slot 0 of every stream and reset ctl (j = 0). */
int sf_stream_reset(int64_t* ctl, int64_t S, int32_t n, int64_t D, int x_dtype, void* x_ring,
                    const double* noise0, void* stream);

/* ---- tcgen05 GEMM (DiT dense contractions) ----
 * C[M, N] = A[M, K] . W[N, K]^T + bias, bf16 in, fp32 accumulate.
 * epi: 0 = f32 out, 1 = bf16 out, 2 = bf16 GELU(tanh) out.
 * K % 64 == 0, N % 128 == 0 (N % 256 == 0 uses 256-wide tiles). */
int sf_gemm_bf16(const void* A, const void* W, const float* bias, void* C, int64_t M, int64_t N, int64_t K,
                 int32_t epi, void* stream);

/* QKV projection with head-major scatter: Q, K -> [M/T, heads, T, 64] bf16 (Q
 * multiplied by q_scale), V -> V^T [M/T, heads, 64, T] fp16.  K = heads*64. */
int sf_gemm_qkv(const void* A, const void* W, const float* bias, void* q, void* k, void* vt, int64_t M, int32_t heads,
                int32_t T, float q_scale, void* stream);
/* Same with head dim hd in {64, 72}: Q, K [M/T, heads, T, hd] bf16, V^T [M/T, heads, hd, T] fp16. */
int sf_gemm_qkv_hd(const void* A, const void* W, const float* bias, void* q, void* k, void* vt, int64_t M,
                   int32_t heads, int32_t T, int32_t hd, float q_scale, void* stream);

/* Gated residual only (rows wider than one TMEM tile, e.g. DiT-XL hidden 1152):
 *   xres += gate[slot] * (A . W^T + bias)     (bf16, in place); N % 128 == 0. */
int sf_gemm_res(const void* A, const void* W, const float* bias, void* xres, const float* gate, int64_t vec_stride,
                int64_t M, int64_t N, int64_t K, int32_t tokens_per_slot, void* stream);

/* xmod = LayerNorm(xres) * (1 + scale[slot]) + shift[slot]  (no affine LN params), N in {384, 1152}. */
int sf_ln_modulate(const void* xres, void* xmod, const float* shift, const float* scale, int64_t vec_stride,
                   int64_t M, int64_t N, int32_t tokens_per_slot, float ln_eps, void* stream);

/* Gated residual + LayerNorm + adaLN modulate fused into the GEMM epilogue:
 *   xres += gate[slot] * (A . W^T + bias)            (bf16 residual, in place)
 *   xmod  = LN(xres) * (1 + scale[slot]) + shift[slot]
 * slot = row / tokens_per_slot; per-slot vectors at ptr + slot*vec_stride.
 * N must be 384 (one 128 x 384 tile holds whole rows). */
int sf_gemm_res_ln(const void* A, const void* W, const float* bias, void* xres, void* xmod, const float* gate,
                   const float* shift, const float* scale, int64_t vec_stride, int64_t M, int64_t N, int64_t K,
                   int32_t tokens_per_slot, float ln_eps, void* stream);
/* Post-attention half of a DiT-S/2 block in one kernel on CTA pairs: attention projection +
 * gated residual + LayerNorm/modulate (kept on chip) + MLP (fc1 + GELU + fc2, the hidden kept on
 * chip) + gated residual + next LayerNorm/modulate.  attn [M, 384] bf16; wproj [384, 384];
 * w1 [1536, 384]; w2 [384, 1536]; xres updated in place; xmod_out = next LN output.
 * M % 256 == 0 and tokens_per_slot % 128 == 0 (else SF_ERR_PARAMETER). */
int sf_block_tail(const void* attn, const void* wproj, const float* bproj, const void* w1, const void* w2,
                  const float* b1, const float* b2, void* xres, void* xmod_out, const float* gate_msa,
                  const float* shift_mlp, const float* scale_mlp, const float* gate_mlp, const float* shift_next,
                  const float* scale_next, int64_t vec_stride, float ln_eps, int64_t M, int32_t tokens_per_slot,
                  void* stream);

/* K6 -- flash attention, T tokens per row (multiple of 256), head dim 64, no mask.
 * q, k: [rows, heads, T, 64] bf16 (q pre-scaled), vt: [rows, heads, 64, T] fp16;
 * out: [rows * T, heads * 64] bf16 (token-major, heads concatenated). */
int sf_attention(const void* q, const void* k, const void* vt, void* out, int64_t rows, int32_t heads, int32_t T,
                 void* stream);
/* Same with head dim hd in {64, 72} (DiT-S/2, DiT-XL/2): q, k [rows, heads, T, hd]
 * bf16, vt [rows, heads, hd, T] fp16, out [rows * T, heads * hd] bf16.  For hd 72
 * the QK^T contraction is zero-padded to 80 on chip (no padding in memory). */
int sf_attention_hd(const void* q, const void* k, const void* vt, void* out, int64_t rows, int32_t heads, int32_t T,
                    int32_t hd, void* stream);

/* ---- DiT velocity-field runtime (the network behind VelocityModel.forward,
 * models.py:89-136; it has no reference implementation -- SURVEY 8(c)) ----
 * DiT-S/2 geometry: hidden 384, 6 heads of 64, depth 12, patch 2, 4 latent
 * channels, 64x64 latent (1024 tokens), MLP 1536, 256 sinusoid features,
 * conditioning vector of embed_dim (8).  Weights are bf16 [out, in]
 * row-major unless marked (t), which are transposed [in, out]; biases fp32. */
typedef struct sf_dit_config {
  int32_t depth, hidden, heads, patch, in_ch, latent_hw, embed_dim, freq_dim, mlp_hidden;
  float ln_eps;
} sf_dit_config;

typedef struct sf_dit_weights {
  const void* patch_w;    /* bf16 [hidden, in_ch*p*p]  (Conv2d weight, (c,p,q) order) */
  const float* patch_b;   /* [hidden] */
  const float* pos_embed; /* [tokens, hidden] fixed 2-D sin-cos */
  const void* t_w1t;      /* bf16 (t) [freq_dim, hidden] */
  const float* t_b1;
  const void* t_w2t;      /* bf16 (t) [hidden, hidden] */
  const float* t_b2;
  const void* y_wt;       /* bf16 (t) [embed_dim, hidden] */
  const float* y_b;
  const void* ada_w;      /* bf16 [depth*6*hidden + 2*hidden, hidden]: every block's adaLN then the final's */
  const float* ada_b;
  const void* qkv_w;      /* bf16 [depth, 3*hidden, hidden] */
  const float* qkv_b;     /* [depth, 3*hidden] */
  const void* proj_w;     /* bf16 [depth, hidden, hidden] */
  const float* proj_b;
  const void* fc1_w;      /* bf16 [depth, mlp_hidden, hidden] */
  const float* fc1_b;
  const void* fc2_w;      /* bf16 [depth, hidden, mlp_hidden] */
  const float* fc2_b;
  const void* final_w;    /* bf16 [p*p*in_ch, hidden]; output feature f = (p*P+q)*C + c */
  const float* final_b;
} sf_dit_weights;

typedef struct sf_dit sf_dit; /* opaque runtime handle (host state + TMA descriptors + graph cache) */

int64_t sf_dit_workspace_bytes(const sf_dit_config* cfg, int64_t max_rows);
int sf_dit_mod_stride(const sf_dit_config* cfg);
int sf_dit_create(const sf_dit_config* cfg, const sf_dit_weights* w, int64_t max_rows, void* workspace,
                  int64_t ws_bytes, sf_dit** out);
int sf_dit_destroy(sf_dit* h);

/* One velocity-field evaluation (VelocityModel.forward, models.py:111-114):
 * x [rows, in_ch, hw, hw] fp32, ts [rows] fp64 flow times (model time 1000 t),
 * row_embs [rows, embed_dim] fp64 -> eps_out [rows, in_ch*hw*hw] fp32. */
int sf_dit_forward(sf_dit* h, int64_t rows, const float* x, const double* ts, const double* row_embs, float* eps_out,
                   void* stream);

/* One stream-batch iteration with the DiT (pipeline.py:171-219) fully on device:
 * ring bookkeeping, one guided velocity evaluation over all S*n slots (2x rows
 * when w != 1, models.py:244-296; w_streams = NULL or device fp64 [S] per-stream
 * scales, w != 1 then only says "some stream is guided"), fused CFG + Euler + emit + refill on the
 * fp32 ring x_ring [S*n, D].  noise_in [S, D] fp32 = initial noise of
 * generation j+1 per stream, or NULL for on-device Philox(noise_seed + s).
 * use_graph != 0 captures the launch sequence into a CUDA graph on first use
 * and replays it afterwards; the cache key is every argument the capture bakes
 * in (all pointers, S, n, m, w, noise_seed), so a replay always equals the
 * eager launch sequence for the same arguments. */
int sf_dit_stream_step(sf_dit* h, int64_t* ctl, int64_t S, int32_t n, int64_t m, const double* stage_params,
                       int64_t* row_info, double* row_t, float* x_ring, const double* emb, const double* neg, double w,
                       const double* w_streams, const float* noise_in, uint64_t noise_seed, float* frames_out,
                       int64_t* frame_ids, int32_t use_graph, void* stream);

/* One eager (non-graph) stream step with a CUDA event after every launch;
 * synchronises and returns, per kernel class, the summed duration (ms) and the
 * launch count.  Classes: 0 prepare, 1 cond, 2 adaLN GEMM, 3 patch-embed+LN,
 * 4 QKV GEMM, 5 attention, 6 proj GEMM+res+LN, 7 fc1 GEMM+GELU,
 * 8 fc2 GEMM+res+LN, 9 final+CFG+Euler+refill (arrays of >= 10 entries). */
int sf_dit_profile_step(sf_dit* h, int64_t* ctl, int64_t S, int32_t n, int64_t m, const double* stage_params,
                        int64_t* row_info, double* row_t, float* x_ring, const double* emb, const double* neg,
                        double w, const double* w_streams, const float* noise_in, uint64_t noise_seed,
                        float* frames_out, int64_t* frame_ids, float* ms_per_class, int32_t* launches_per_class,
                        void* stream);

/* Number of kernel launches this handle has issued or captured so far. */
int64_t sf_dit_launch_count(const sf_dit* h);

/* Destroy every cached stream-step graph whose ring control word is ctl (the
 * owner of those buffers calls this before freeing them); synchronises the device
 * if any graph is released.  sf_dit_graph_count: graphs currently cached. */
int sf_dit_graph_release(sf_dit* h, const int64_t* ctl);
int64_t sf_dit_graph_count(const sf_dit* h);

/* Reset a fp32 ring: generation-0 noise into slot 0 of each stream (noise0 [S, D]
 * or Philox when NULL), ctl <- j = 0. */
int sf_dit_stream_reset(int64_t* ctl, int64_t S, int32_t n, int64_t D, float* x_ring, const float* noise0,
                        uint64_t noise_seed, void* stream);

/* On-device N(0,1) noise: out[s, i] = Philox(seed + s, gen, i) (Box-Muller). */
int sf_philox_normal(float* out, int64_t S, int64_t D, uint64_t seed, int64_t gen, void* stream);

/* numpy-identical generation noise (replaces the host call of
 * generation_noise, src/pipeline.py:92-98 -> np.random.default_rng([seed, gen])
 * .standard_normal(D)): out[s, :] = those D draws for seeds[s] (device int64 [S],
 * each >= 0), bit-identical in fp64 (out_dtype SF_F64) or their round-to-nearest
 * fp32 cast (SF_F32, pipeline.py:176).  gen >= 0. */
int sf_numpy_normal(const int64_t* seeds, int64_t gen, int64_t S, int64_t D, void* out, int out_dtype, void* stream);

/* ---- Tiny-VAE (TAESD) decoder of retired frames (replaces decode_stub,
 * src/pipeline.py:86-89).  Activations: bf16 NHWC, 64 channels, one-pixel zero
 * border, [F][H+2][W+2][64]; buffers must be zero-initialised once (borders are
 * never written). */
typedef struct sf_taesd_weights {
  const float* first_w; /* conv(4, 64): fp32 [64][4][3][3] (torch layout) */
  const float* first_b; /* [64] */
  const void* conv_w[33]; /* the 33 conv(64, 64) in network order: bf16 [9 taps][64 oc][64 ic] */
  const float* conv_b[33]; /* [64] fp32, NULL for the three bias-free post-upsample convs */
  const void* final_w;  /* conv(64, 3): bf16 [9][16][64], output channels 3..15 zero */
  const float* final_b; /* [16] fp32 (3 used) */
} sf_taesd_weights;

/* Elements of one padded activation tensor. */
int64_t sf_taesd_act_elems(int64_t F, int32_t H, int32_t W);
/* 3x3 conv, 64 input channels, on padded NHWC bf16 (tcgen05 implicit GEMM).
 * epi: 0 bias, 1 bias+ReLU, 2 bias+residual+ReLU (res: input geometry),
 *      3 = 2 then 2x nearest upsample into out ([F][2H+2][2W+2][64]),
 *      4 final: w [9][16][64], out fp32 NCHW image [F][3][H][W]. */
int sf_conv3x3(const void* in, const void* w, const float* bias, const void* res, void* out, int64_t F, int32_t H,
               int32_t W, int32_t epi, void* stream);
/* Clamp(tanh(x/3)*3) + conv(4, 64) + ReLU: latent fp32 [F][4][64][64] -> padded stage-0 activation. */
int sf_taesd_first(const float* lat, const float* w, const float* b, void* out, int64_t F, void* stream);
/* Workspace of sf_taesd_decode for up to F_cap frames (4 stages x 3 padded
 * activations), zero-initialised once by the caller and reused across calls. */
int64_t sf_taesd_workspace_bytes(int64_t F_cap);
/* Whole decoder: latents fp32 [F][4][64][64] -> images fp32 [F][3][512][512], F <= F_cap. */
int sf_taesd_decode(const sf_taesd_weights* w, const float* lat, int64_t F, int64_t F_cap, void* ws, int64_t ws_bytes,
                    float* img, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* STREAMFLOW_H_ */

/*
 * leorzf_b200 -- C ABI of the B200-native (sm_100a) RZF precoder update.
 *
 * Drop-in boundary for the numerical core of the reference package
 * leorzf 0.1.0 (pkg/src/leorzf/__init__.py:17-31).  The reference is pure
 * Python; its public functions are re-exposed by the Python package
 * paper_2512_16543_b200 (same names/signatures/exceptions) which calls the
 * entry points below through ctypes.  Foreign callers can bind them the
 * same way.
 *
 * Conventions
 *  - All pointers are DEVICE pointers (caller-allocated, e.g. torch tensors)
 *    unless stated; `stream` is a cudaStream_t (NULL = legacy default).
 *  - Complex data is interleaved (re, im); dtype LRZ_C64 = float2,
 *    LRZ_C128 = double2.  Matrices are row-major like numpy unless stated;
 *    low-rank factors U, V are stored column-major per item ([D][K]: column
 *    j contiguous) with D = d_max columns reserved.
 *  - Batched calls take an item count and an element stride per item.
 *  - Return value: LRZ_OK, or < 0 (bad argument / launch error; message in
 *    lrz_last_error()).  Per-item numerical outcomes go to `info[item]`
 *    (LRZ_INFO_*), which the Python layer maps to the reference exceptions
 *    (pkg/src/leorzf/errors.py:28-50).
 *  - No host synchronisation inside calls, no allocation, deterministic
 *    (fixed reduction orders, no atomics on values).
 */
#ifndef LEORZF_B200_H
#define LEORZF_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LRZ_C64 0
#define LRZ_C128 1

#define LRZ_OK 0
#define LRZ_EINVAL (-1)
#define LRZ_ELAUNCH (-2)
#define LRZ_EDEVICE (-3)

#define LRZ_INFO_OK 0
#define LRZ_INFO_SINGULAR 1          /* SingularMatrixError      lowrank.py:136-137 */
#define LRZ_INFO_SINGULAR_AUX 2      /* SingularAuxiliaryError   lowrank.py:213-216 */
#define LRZ_INFO_ZERO_PRECODER 3     /* ZeroPrecoderError        precoding.py:49-50 */
#define LRZ_INFO_INDEFINITE 4        /* not PD: pivoted path used (lowrank.py:142-144) */

/* method codes, same as harness._DECISION_CODES (harness.py:29) */
#define LRZ_METHOD_FULL 0
#define LRZ_METHOD_WOODBURY 1
#define LRZ_METHOD_NONE 2

int lrz_version(void);
const char *lrz_last_error(void);
/* 0 if `device` is a compute-capability 10.0 part this library was built for. */
int lrz_device_check(int device);

/* Per-kernel device timing: lrz_prof_enable(1) brackets every instrumented
 * launch with CUDA events on its stream (0 turns it off); lrz_prof_collect()
 * waits for them and returns "kernel=ms_total:launches;..." for the launches
 * since the last enable/collect (bench.py's per-kernel roofline timing). */
int lrz_prof_enable(int on);
const char *lrz_prof_collect(void);

/* K1  Gram + regularisation: A[i] = 0.5 (H H^H + (H H^H)^H) + alpha I.
 *     Replaces lowrank.py:160-162 (and :365-366).  H: [B][K][N] dtype,
 *     A: [B][K][K] complex128 (always: the reference promotes via alpha I).
 *     Runs on the FP64 tensor pipe (DMMA) for both dtypes, complex64 H widened
 *     to fp64 on load; exactly Hermitian output with a real diagonal. */
int lrz_gram(int dtype, int64_t B, int K, int N, const void *H, int64_t h_stride,
             double alpha, void *A, int64_t a_stride, void *stream);

/* K1' Gram correction (lowrank.py:167-179):
 *     dA = H dH^H + dH H^H + dH dH^H  computed as X dH^H + dH X^H,
 *     X = H + dH/2.  mode 0: P = H, Q = dH.  mode 1: P = H_prev, Q = H_cur
 *     (dH = Q - P formed on the fly, exactly harness.py:235).
 *     dA: [B][K][K] complex128, exactly Hermitian. */
int lrz_gram_delta(int dtype, int64_t B, int K, int N, const void *P, int64_t p_stride,
                   const void *Q, int64_t q_stride, int mode, void *dA, int64_t a_stride,
                   void *stream);

/* K5  Hermitian inverse with the reference's condition guard
 *     (lowrank.py:127-144): Gauss-Jordan without pivoting while PD, pivoted
 *     otherwise; info = SINGULAR when cond_2 > cond_limit or non-finite.
 *     A, A_inv: complex128 [B][K][K].  item_mask (nullable): skip items with 0.
 *     workspace: lrz_workspace_bytes(LRZ_WS_INVERSE, ...) bytes. */
int lrz_herm_inverse(int64_t B, int K, const void *A, int64_t a_stride, void *A_inv,
                     int64_t ai_stride, int32_t *info, double cond_limit,
                     const uint8_t *item_mask, void *workspace, void *stream);

/* K2+K3 adaptive randomised SVD (lowrank.py:243-316, Alg. 1).
 *   item i reads dA[i] (complex128 K x K), sketch normals
 *   omega + omega_row[i] * omega_stride starting at cursor[i] (the real block
 *   of width d then the imaginary block, lowrank.py:284-286).
 *   Writes U, V ([D][K] column-major, complex128), S (D, descending),
 *   k_est, iters (sketch iterations run), fallback (1 = iteration-cap
 *   tail), consumed (normals used).  omega_row / item_mask nullable.
 *   want_factor 1: U/S/V always written; 0: only when 2*k_est <= K (the
 *   dispatcher's Woodbury candidates) -- the batched runner's mode, which
 *   lets iterations that cannot reach the energy target skip the SVD.
 *   hermitian 1 promises dA == dA^H exactly (Gram corrections are): with
 *   want_factor 0 and K <= 32 a warp-per-item front end runs first.
 *   want_factor 2 (hermitian, d_max <= 40): cursor-resolution mode -- only
 *   the screening front end runs and writes iters / consumed from the
 *   screened energies (estimates inside the CholeskyQR error band; no
 *   factors, k_est untouched).  The batched runner alternates it with
 *   lrz_spec_verify to settle the sketch cursors before the exact pass. */
typedef struct {
  double eta;
  int k_init, p, i_max;
  int d_max;               /* >= min(k_init * 2^(i_max-1) + p, K) */
  const double *eta_row;   /* nullable device array: eta per omega row (several
                              methods batched as rows of one call); overrides eta */
  int64_t omega_len;       /* > 0: normals per omega row; a call that would read
                              past it stops with iters = -1 (0 = unchecked) */
} lrz_arsvd_cfg;

int lrz_arsvd(int64_t B, int K, const void *dA, int64_t a_stride, const double *omega,
              int64_t omega_stride, const int32_t *omega_row, const int64_t *cursor,
              const lrz_arsvd_cfg *cfg, void *U, void *V, double *S, int32_t *k_est,
              int32_t *iters, int32_t *fallback, int64_t *consumed,
              const uint8_t *item_mask, int want_factor, int hermitian, void *workspace,
              void *stream);

/* K4  Woodbury update (lowrank.py:182-227):
 *     A_inv_out = A_inv - (A_inv U aux^-1)(V^H A_inv), aux = S^-1 + V^H A_inv U,
 *     A_out = A + U S V^H (skipped when A/A_out are NULL).
 *     info = SINGULAR_AUX (outputs untouched) when cond_2(aux) > 1e12.
 *     r[i] <= d_max <= 256. */
int lrz_woodbury(int64_t B, int K, int d_max, const void *A, const void *A_inv,
                 int64_t a_stride, const void *U, const void *V, const double *S,
                 const int32_t *r, void *A_out, void *A_inv_out, int32_t *info,
                 void *workspace, void *stream);

/* Chain step of the batched runner (harness.py:228-241 per trial): walks the
 * T steps of each trial in order.  plan[b][t]: 0 = full (A_inv_seq[b][t]
 * already holds inv(G[b][t])), 1 = Woodbury candidate (factor in U/V/S/r),
 * 2 = none.  A_inv_seq[b][t] <- state after step t; A_state updated in
 * place when non-NULL.  On SingularAuxiliary the step falls back to
 * inv(G[b][t]) (lowrank.py:353-367).  method/info per (b,t). */
int lrz_chain(int64_t B, int T, int K, int d_max, const uint8_t *plan, const void *G,
              const void *A_inv_prev, void *A_inv_seq, void *A_state, const void *U,
              const void *V, const double *S, const int32_t *r, uint8_t *method,
              int32_t *info, void *workspace, void *stream);

/* Same chain, step-parallel: the B trials advance one time step per launch
 * group and every product of the Woodbury step is batched over the trials
 * (2 batched GEMMs, the r x r core per trial, tiled A^-1 / A update, fallback
 * inversions).  Same arguments, results and workspace as lrz_chain; faster
 * when K is large and B small (one CTA per trial leaves SMs idle there). */
int lrz_chain_steps(int64_t B, int T, int K, int d_max, const uint8_t *plan, const void *G,
                    const void *A_inv_prev, void *A_inv_seq, void *A_state, const void *U,
                    const void *V, const double *S, const int32_t *r, uint8_t *method,
                    int32_t *info, void *workspace, void *stream);

/* Dispatcher decision (lowrank.py:345-359) for n steps: plan = 2 (none,
 * k_est == 0), 1 (Woodbury, k_est/K <= 0.5), 0 (full); is_sketch == 0 -> 0. */
int lrz_plan(int64_t n, int K, const uint8_t *is_sketch, const int32_t *k_est, uint8_t *plan,
             void *stream);

/* K6  fully-digital precoder + rate (precoding.py:37-80 with F_RF = I):
 *     W = H^H A_inv (N x K, dtype of H, UNSCALED), scale = sqrt(P_t)/||W||_F,
 *     G = scale * H W, SINR_n = |G_nn|^2 / (sum_{i != n}|G_ni|^2 + noise_n),
 *     rates = log2(1 + SINR), sum.  noise row = item / noise_div.
 *     W may be NULL (then kept in workspace).  info = ZERO_PRECODER if ||W||=0.
 *     G_true (nullable, complex128 [B][K][K]) = H H^H + alpha I of the same H:
 *     then H W is formed as G_true A^-1 - alpha A^-1 in K^3
 *     instead of K^2 N work; for K <= 32 W, ||W||, the coupling and the
 *     SINR / rate reduction are one fused DMMA kernel. */
int lrz_precode_rate(int dtype, int64_t B, int K, int N, const void *H, int64_t h_stride,
                     const void *A_inv, int64_t ai_stride, double P_t, const double *noise,
                     int64_t noise_div, void *W, int64_t w_stride, const void *G_true,
                     double alpha, double *scale, double *rates, double *sinr,
                     double *sum_rate, int32_t *info, void *workspace, void *stream);

/* Batched complex GEMM C[i] = op(A[i]) op(B[i]) (op: 0 = N, 1 = T, 2 = C^H),
 * all operands of `dtype`, row-major with leading dims.  Used by the
 * single-call precoder/rate with an explicit F_RF (precoding.py:47-48,74). */
int lrz_cgemm(int dtype, int64_t batch, int M, int N, int Kd, int opA, const void *A,
              int64_t lda, int64_t sA, int opB, const void *Bm, int64_t ldb, int64_t sB,
              void *C, int64_t ldc, int64_t sC, void *stream);

/* Z = a X + b Y elementwise over n complex elements (Y nullable); used for
 * F_BB = scale * F_raw (precoding.py:51) and H_new = H + dH (lowrank.py:364). */
int lrz_axpby(int dtype, int64_t n, double a, const void *X, double b, const void *Y, void *Z,
              void *stream);

/* ||X[i]||_F^2 in fp64 for `n` complex elements per item. */
int lrz_fro2(int dtype, int64_t batch, int64_t n, const void *X, int64_t sX, double *out,
             void *stream);

/* SINR / rate from a K x K coupling matrix G (dtype), scaled by scale[i]
 * (nullable = 1): precoding.py:74-80. */
int lrz_sinr_rate(int dtype, int64_t batch, int K, const void *G, int64_t sG,
                  const double *scale, const double *noise, int64_t noise_div, double *rates,
                  double *sinr, double *sum_rate, void *stream);

/* Device sketch streams, bit-exact with numpy's Generator(PCG64).standard_normal
 * (the reference's Omega source, lowrank.py:284-286).  For each of B streams
 * with PCG64 state/inc (uint64 lo, hi pairs, as numpy's bit_generator.state
 * reports them) positioned `raw0[b]` raw draws in, writes the next L
 * normals to out[b][0..L).  startpos must be NULL (positions are recovered
 * on demand by lrz_rng_locate).  status[b] != 0 if the window could not be
 * produced.  Workspace: lrz_workspace_bytes(LRZ_WS_RNG, 0, B, 0, L, 0); it
 * keeps the window's segment tables for lrz_rng_locate. */
int lrz_rng_normals(int64_t B, int64_t L, const uint64_t *state, const uint64_t *inc,
                    const int64_t *raw0, double *out, int32_t *startpos, int32_t *status,
                    void *workspace, void *stream);

/* After lrz_rng_normals(B, L, state, inc, raw0, ..., workspace): raw draws
 * taken by the first consumed[b] normals of the window (consumed[b] <= L),
 * i.e. the amount to add to raw0[b] to skip exactly those normals.  Same
 * B, L, state, inc, raw0 and workspace as the window call. */
int lrz_rng_locate(int64_t B, int64_t L, const uint64_t *state, const uint64_t *inc,
                   const int64_t *raw0, const int64_t *consumed, int64_t *raw_advance,
                   void *workspace, void *stream);

/* On-device synthetic channels (scenario.py, SURVEY 8(f) "next" #1): H for
 * steps [t0, t0 + T) of B trials, [B][T][K][N] of `dtype`.  params: [B][6][K]
 * doubles (theta0, psi, phi, beta, kappa, drift per user); scatter: [B] rows
 * of 2 K N standard normals (real block then imaginary block, the trial's
 * channel stream), row stride scatter_stride.  N = n_side^2. */
int lrz_channels(int dtype, int64_t B, int t0, int T, int K, int N, int n_side,
                 const double *params, const double *scatter, int64_t scatter_stride, void *H,
                 void *stream);

/* ---- hybrid (analog beams + digital RZF) LEO pass, SURVEY 8(f) "next" #3/#4 ---- */

/* Scenario constants of one LEO pass (reference config.py:27-60, channel.py:24-29). */
typedef struct {
  int K, n_x, n_y, N_RF;
  int beam_hold;        /* snapshots the analog beams are held for (config.py:62) */
  int nlos_block;       /* snapshots an NLOS draw is held for (config.py:61) */
  double wavelength;    /* c / carrier_Hz */
  double spacing_m;     /* spacing_wavelengths * wavelength */
  double orbit_radius;  /* R_earth + altitude_m */
  double orbit_rate;    /* sqrt(GM / R^3) */
  double pass_s, dt;    /* pass length, 1 / update_rate_Hz */
  double min_elev_rad;  /* elevation mask */
  double atm_loss_dB;
} lrz_leo_cfg;

/* One snapshot per (trial, step) for steps [t0, t0 + T) of B trials
 * (channel.py:352-384 + harness.py:221-226): pass geometry at t*dt, the
 * conjugated unit-gain manifold rows H~, Rician H = w_los g H~ + w_nlos
 * (g/sqrt(N)) S, the DFT beam powers |fft2(H~)|^2 (ortho), the greedy beam
 * choice (channel.py:202-233; beams re-selected every beam_hold steps), and
 *   H_eff = H~ F_RF  (K x N_RF),   H_rf = H F_RF  (K x N_RF),   cols (N_RF),
 * F_RF = codebook columns `cols` of kron(DFT(n_x), DFT(n_y)).
 * ut: [B][K][5] doubles (ECEF x, y, z, gain dBi, Rician K linear).
 * dft: the two unitary DFT factors, n_x^2 then n_y^2 complex128.
 * nlos: [B] rows (stride nlos_stride) of standard normals starting at NLOS
 * block floor(t0 / nlos_block) (each block: K*N real then K*N imaginary).
 * H_full / H_tilde (nullable): [B][T][K][N] complex128 for parity tests.
 * info[b][t] = LRZ_INFO_BELOW_MASK if a UT is under the elevation mask. */
#define LRZ_INFO_BELOW_MASK 5        /* BelowMinElevationError  channel.py:280-284 */
int lrz_leo_snapshot(const lrz_leo_cfg *cfg, int64_t B, int t0, int T, const double *ut,
                     const void *dft, const double *nlos, int64_t nlos_stride, void *H_eff,
                     void *H_rf, int32_t *cols, int32_t *info, void *H_full, void *H_tilde,
                     void *stream);

/* Hybrid precoder + rate per item (precoding.py:37-80 with F_RF = DFT codebook
 * columns `cols`): F_raw = H_eff^H A^-1, scale = sqrt(P_t)/||F_RF F_raw||_F,
 * G = H_rf (scale F_raw), SINR / log2(1 + SINR).  All complex128; items are
 * contiguous [B][K][N_RF] / [B][K][K] / [B][N_RF]; F_BB nullable [B][N_RF][K];
 * noise row = item / noise_div. */
int lrz_hybrid_precode_rate(int64_t B, int K, int N_RF, int n_x, int n_y, const void *H_eff,
                            const void *A_inv, const void *H_rf, const int32_t *cols,
                            const void *dft, double P_t, const double *noise, int64_t noise_div,
                            void *F_BB, double *scale, double *rates, double *sum_rate,
                            int32_t *info, void *stream);

/* Per-trial campaign aggregates over steps [t_base, t_base + T) of B trials,
 * ACCUMULATED into stats[b][6] = (total cost units, k_sum, k_count, n_full,
 * n_woodbury, n_none) with the harness's accounting (harness.py:227-251):
 * reset steps (t == 0, t % n_reset == 0, or conventional) cost K^3;
 * otherwise the dispatcher's cost (lowrank.py:101-118, 345-373). */
int lrz_campaign_reduce(int64_t B, int T, int t_base, int K, int n_reset, int conventional,
                        const uint8_t *method, const int32_t *k_est, double *stats,
                        void *stream);

/* ---- fused entry points: what a non-Python caller binds ---- */

/* Alg. 2 dispatcher over B items (lowrank.py:319-373): dA = gram_delta(H, dH),
 * arSVD of dA from item b's sketch stream (omega row b, starting at
 * cursor[b]), then 'none' (k_est = 0: the state is copied), Woodbury
 * (k_est <= K/2 and cond(aux) <= 1e12) or full (the true Gram of H + dH,
 * inverted with the 1e14 guard) -- the reference's decisions.  H, dH:
 * [B][K][N] dtype; A, A_inv (in) and A_out, A_inv_out (out): complex128
 * [B][K][K] (A / A_out nullable: GramState.A not maintained).  method
 * (LRZ_METHOD_*), k_est, consumed (normals drawn), cost (cost units,
 * lowrank.py:101-118; nullable), info (LRZ_INFO_* of the full inversion).
 * Workspace: lrz_update_inverse_ws(dtype, B, K, N, cfg->d_max) bytes. */
size_t lrz_update_inverse_ws(int dtype, int64_t B, int K, int N, int d_max);
int lrz_update_inverse(int dtype, int64_t B, int K, int N, const void *H, const void *dH,
                       double alpha, const void *A, const void *A_inv, const double *omega,
                       int64_t omega_stride, const int64_t *cursor, const lrz_arsvd_cfg *cfg,
                       void *A_out, void *A_inv_out, uint8_t *method, int32_t *k_est,
                       int64_t *consumed, double *cost, int32_t *info, void *workspace,
                       void *stream);

/* One time chunk of the per-trial sweep (harness._sweep_trial,
 * harness.py:221-255), fully digital: for B trials x T steps, the Grams, the
 * Gram corrections, the arSVD of every dispatcher step in order per trial at
 * the exact sketch cursors, the dispatcher, the batched full inversions, the
 * Woodbury chain, the precoder and the rates -- in stream order, no host
 * synchronisation.  H [B][T][K][N] dtype, noise [B][K]; t0 = global index of
 * the chunk's first step (resets at t % n_reset == 0); cfg NULL = the
 * conventional method.  omega: [B] rows (stride omega_stride) starting at each
 * trial's first unconsumed normal; consumed[b] = normals the chunk used.
 * State in/out: A_inv_state, A_state (nullable) [B][K][K] complex128; G_prev
 * = the previous chunk's last Gram (NULL at the start of a pass), G_last
 * (nullable) receives this chunk's.  Outputs per (b, t): rates (sum-rate),
 * per_ut [B][T][K], method, k_est, info; A_inv_seq nullable [B][T][K][K].
 * Workspace: lrz_trajectory_ws(dtype, B, T, K, N, d_max) bytes (d_max = 1
 * for the conventional method). */
size_t lrz_trajectory_ws(int dtype, int64_t B, int T, int K, int N, int d_max);
int lrz_trajectory(int dtype, int64_t B, int T, int K, int N, const void *H, double alpha,
                   double P_t, const double *noise, int64_t t0, int n_reset,
                   const lrz_arsvd_cfg *cfg, const double *omega, int64_t omega_stride,
                   void *A_inv_state, void *A_state, const void *G_prev, void *G_last,
                   double *rates, double *per_ut, uint8_t *method, int32_t *k_est,
                   int32_t *info, int64_t *consumed, void *A_inv_seq, void *workspace,
                   void *stream);

/* Campaign summary on the device (harness.py:336-367) for M methods (method 0
 * = the conventional baseline): rates [M][B][T] (per-step sum-rates), stats
 * [M][B][6] (lrz_campaign_reduce) -> trial_mean [M][B], summary [M][6] =
 * (pooled mean rate, mean cost units per trial, mean rank, n_full,
 * n_woodbury, n_none), table [M][2] = (savings %, degradation %). */
int lrz_campaign_summary(int M, int64_t B, int T, const double *rates, const double *stats,
                         double *trial_mean, double *summary, double *table, void *stream);

/* Workspace sizing for the calls that take one. */
#define LRZ_WS_INVERSE 0
#define LRZ_WS_ARSVD 1
#define LRZ_WS_WOODBURY 2
#define LRZ_WS_CHAIN 3
#define LRZ_WS_PRECODE 4
#define LRZ_WS_RNG 5
size_t lrz_workspace_bytes(int op, int dtype, int64_t B, int K, int N, int d_max);

/* In-order arSVD of the unverified suffix of each trial (the sequential
 * fallback of the speculative runner): items are [B][T] row-major (dA
 * contiguous K x K per item, factor outputs as lrz_arsvd with B*T items),
 * one CTA per trial b walks the sketch steps t >= first_unverified[b]
 * (is_sketch[b][t] != 0) starting at cursor[b][first_unverified[b]] and
 * advancing by each call's consumption; writes cursor[b][t] and
 * iters_pred[b][t] = iters[b][t] of every step it visits.  Omega row of
 * trial b = omega + b * omega_stride.  Workspace as lrz_arsvd for B*T items. */
int lrz_arsvd_seq(int64_t B, int T, int K, const void *dA, const double *omega,
                  int64_t omega_stride, const lrz_arsvd_cfg *cfg, const uint8_t *is_sketch,
                  const int32_t *first_unverified, int64_t *cursor, int32_t *iters_pred,
                  void *U, void *V, double *S, int32_t *k_est, int32_t *iters,
                  int32_t *fallback, int64_t *consumed, int want_factor, void *workspace,
                  void *stream);

/* Cursor walk (K <= 32, sketch widths <= 24): one warp per trial walks the
 * steps t >= first_unverified[b] in order and fixes each sketch step's cursor
 * and iteration count from the CholeskyQR energy total alone (a step's normal
 * consumption depends only on its hit iteration, lowrank.py:284-300), without
 * QR / SVD.  Writes cursor[b][t] and iters_pred[b][t]; stops at a step whose
 * total is within the rounding bound of the target.  The factors are then
 * computed by one speculative lrz_arsvd pass at these cursors. */
int lrz_arsvd_walk(int64_t B, int T, int K, const void *dA, const double *omega,
                   int64_t omega_stride, const lrz_arsvd_cfg *cfg, const uint8_t *is_sketch,
                   const int32_t *first_unverified, int64_t *cursor, int32_t *iters_pred,
                   void *stream);

/* Speculative sketch-cursor resolution for the batched runner: one thread
 * per trial walks its T steps, accepts every step whose observed iteration
 * count matches the prediction, and re-predicts the suffix after the first
 * mismatch.  Adds, to
 * *pending (device int32), the number of trials with unverified steps.
 * iters_act == NULL: initialise cursors/active from iters_pred only. */
int lrz_spec_verify(int64_t B, int T, int K, const lrz_arsvd_cfg *cfg,
                    const uint8_t *is_sketch, int32_t *iters_pred,
                    const int32_t *iters_act, int64_t *cursor, const int64_t *cursor0,
                    int32_t *first_unverified, uint8_t *active, int32_t *pending,
                    void *stream);

/* The same with a per-step tally of the iteration counts observed so far
 * (votes: uint8 [B][T][LRZ_SPEC_VOTE_W], nullable = lrz_spec_verify): the
 * suffix behind the first mismatch is re-predicted by majority instead of by
 * the last observation.  Counts that hinge on the sketch drawn (not on the
 * step's spectrum) are then not carried over from a pass at shifted cursors.
 * iters_act == NULL also clears the tally (the prediction counts as one vote).
 * Used by the runner's screen-only rounds (lrz_arsvd want_factor 2). */
#define LRZ_SPEC_VOTE_W 16
int lrz_spec_verify_vote(int64_t B, int T, int K, const lrz_arsvd_cfg *cfg,
                         const uint8_t *is_sketch, int32_t *iters_pred,
                         const int32_t *iters_act, int64_t *cursor, const int64_t *cursor0,
                         int32_t *first_unverified, uint8_t *active, int32_t *pending,
                         uint8_t *votes, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* LEORZF_B200_H */

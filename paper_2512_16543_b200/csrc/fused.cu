// Fused C entry points of SURVEY 8(b): the dispatcher (update_inverse,
// lowrank.py:319-373) and one chunk of the per-trial sweep (trajectory,
// harness.py:221-255), composed from the library's kernels in stream order
// with no host synchronisation -- the boundary a non-Python caller binds
// (INTEGRATION.md).  The Python runner (trajectory.py) is the speculative,
// faster form of lrz_trajectory; both give the reference's results.

#include <algorithm>

#include "common.cuh"

extern "C" int lrz_gram_delta(int dtype, int64_t B, int K, int N, const void *P,
                              int64_t p_stride, const void *Q, int64_t q_stride, int mode,
                              void *dA, int64_t a_stride, void *stream);
extern "C" int lrz_gram(int dtype, int64_t B, int K, int N, const void *H, int64_t h_stride,
                        double alpha, void *A, int64_t a_stride, void *stream);
extern "C" int lrz_axpby(int dtype, int64_t n, double a, const void *X, double b, const void *Y,
                         void *Z, void *stream);
extern "C" size_t lrz_workspace_bytes(int op, int dtype, int64_t B, int K, int N, int d_max);

namespace lrz {

static size_t al256(size_t x) { return (x + 255) & ~size_t(255); }

static int d_need(const lrz_arsvd_cfg *c, int K) {
  int d = 0;
  long long k0 = c->k_init;
  for (int i = 0; i < c->i_max; ++i) {
    d = int(std::min<long long>(k0 + c->p, K));
    k0 *= 2;
  }
  return d;
}

// dispatcher epilogue per item (lowrank.py:345-373): none copies the state,
// Woodbury keeps lrz_woodbury's output, full (rank > K/2 or SingularAuxiliary)
// takes inv(G(H + dH)) and A = G; cost units as the reference's cost model.
__global__ void ui_select_kernel(int64_t B, int K, const int32_t *__restrict__ k,
                                 const int32_t *__restrict__ wb_info, uint8_t *__restrict__ full,
                                 uint8_t *__restrict__ method, double *__restrict__ cost) {
  const int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (b >= B) return;
  const int r = k[b];
  const double Kf = K, rf = r;
  int m;
  if (r == 0)
    m = LRZ_METHOD_NONE;
  else if (2 * r <= K && wb_info[b] == LRZ_INFO_OK)
    m = LRZ_METHOD_WOODBURY;
  else
    m = LRZ_METHOD_FULL;
  full[b] = m == LRZ_METHOD_FULL;
  method[b] = uint8_t(m);
  if (cost)
    cost[b] = m == LRZ_METHOD_NONE ? Kf * Kf
              : m == LRZ_METHOD_WOODBURY ? Kf * Kf + Kf * Kf * rf + rf * rf * rf + rf * rf * Kf
                                         : Kf * Kf * Kf + Kf * Kf * rf + rf * rf * Kf;
}

__global__ void ui_assemble_kernel(int64_t B, int64_t KK, const uint8_t *__restrict__ method,
                                   const c128 *__restrict__ A, const c128 *__restrict__ Ai,
                                   const c128 *__restrict__ G, c128 *__restrict__ A_out,
                                   c128 *__restrict__ Ai_out) {
  const int64_t n = B * KK;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = e / KK;
    const int m = method[b];
    if (m == LRZ_METHOD_NONE) {  // the state aliases (lowrank.py:345-351)
      A_out[e] = A[e];
      Ai_out[e] = Ai[e];
    } else if (m == LRZ_METHOD_FULL && A_out) {
      A_out[e] = G[e];
    }
  }
}

// per-step flags of a chunk: reset steps (t_global == 0, every n_reset, no
// previous channel, conventional method) run the full inversion only
__global__ void traj_sketch_kernel(int64_t B, int T, int64_t t0, int n_reset, int has_prev,
                                   int conventional, uint8_t *__restrict__ is_sketch) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e >= B * T) return;
  const int t = int(e % T);
  const int64_t tg = t0 + t;
  const bool reset = conventional || tg == 0 || (n_reset > 0 && tg % n_reset == 0) ||
                     (t == 0 && !has_prev);
  is_sketch[e] = reset ? 0 : 1;
}

// dA[b][t] = G[b][t] - G[b][t-1] (G_prev for t = 0): the fp64 Grams differenced
// exactly as the Python runner does (trajectory.py, delta "diff")
__global__ void traj_delta_kernel(int64_t B, int T, int64_t KK, const c128 *__restrict__ G,
                                  const c128 *__restrict__ G_prev, c128 *__restrict__ dA) {
  const int64_t n = B * T * KK;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t bt = e / KK, i = e - bt * KK;
    const int t = int(bt % T);
    const int64_t b = bt / T;
    c128 z = czero<double>();
    if (t > 0)
      z = csub(G[e], G[e - KK]);
    else if (G_prev)
      z = csub(G[e], G_prev[b * KK + i]);
    dA[e] = z;
  }
}

__global__ void traj_tail_kernel(int64_t B, int T, int64_t KK, const c128 *__restrict__ Ai_seq,
                                 const c128 *__restrict__ G, c128 *__restrict__ Ai_state,
                                 c128 *__restrict__ G_last) {
  const int64_t n = B * KK;
  for (int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; e < n;
       e += int64_t(gridDim.x) * blockDim.x) {
    const int64_t b = e / KK, i = e - b * KK;
    const int64_t src = (b * T + (T - 1)) * KK + i;
    Ai_state[e] = Ai_seq[src];
    if (G_last) G_last[e] = G[src];
  }
}

__global__ void traj_fullmask_kernel(int64_t n, const uint8_t *__restrict__ plan,
                                     uint8_t *__restrict__ mask) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e < n) mask[e] = plan[e] == 0;
}

__global__ void traj_info_kernel(int64_t n, const int32_t *__restrict__ pinfo,
                                 int32_t *__restrict__ info) {
  const int64_t e = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (e < n && info[e] == LRZ_INFO_OK) info[e] = pinfo[e];
}

__global__ void traj_consumed_kernel(int64_t B, int T, const int64_t *__restrict__ cursor,
                                     const int64_t *__restrict__ used,
                                     const uint8_t *__restrict__ is_sketch,
                                     int64_t *__restrict__ consumed) {
  const int64_t b = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
  if (b >= B) return;
  const int64_t bt = b * T + (T - 1);
  consumed[b] = cursor[bt] + (is_sketch[bt] ? used[bt] : 0);
}

static unsigned grid_for(int64_t n) {
  return unsigned(std::min<int64_t>((n + 255) / 256, 148 * 32));
}

}  // namespace lrz

using namespace lrz;

// ------------------------------------------------------------------ update_inverse

extern "C" size_t lrz_update_inverse_ws(int dtype, int64_t B, int K, int N, int d_max) {
  const size_t es = dtype == LRZ_C64 ? 8 : 16, KK = size_t(K) * K;
  size_t b = 0;
  b += al256(B * KK * 16);                                  // dA
  b += al256(B * KK * 16);                                  // G of H + dH
  b += 2 * al256(size_t(B) * d_max * K * 16);               // U, V
  b += al256(size_t(B) * d_max * 8);                        // S
  b += 4 * al256(size_t(B) * 8);                            // iters, fallback, wb_info, full
  b += al256(size_t(B) * K * N * es);                       // H + dH
  b += al256(lrz_workspace_bytes(LRZ_WS_ARSVD, dtype, B, K, N, d_max));
  b += al256(lrz_workspace_bytes(LRZ_WS_WOODBURY, dtype, B, K, N, d_max));
  b += al256(lrz_workspace_bytes(LRZ_WS_INVERSE, dtype, B, K, N, d_max));
  return b;
}

// Alg. 2 dispatcher over B items (lowrank.py:319-373): dA = gram_delta(H, dH),
// arSVD of dA from each item's sketch stream (omega row b at cursor[b]),
// then none / Woodbury / full exactly as the reference decides (rank ratio,
// SingularAuxiliary fallback, the full branch re-forming the Gram of H + dH).
// A / A_inv in (complex128 [B][K][K], the GramState), A_out / A_inv_out out;
// method, k_est, consumed (normals), cost (cost units, nullable), info.
extern "C" int lrz_update_inverse(int dtype, int64_t B, int K, int N, const void *H,
                                  const void *dH, double alpha, const void *A, const void *A_inv,
                                  const double *omega, int64_t omega_stride,
                                  const int64_t *cursor, const lrz_arsvd_cfg *cfg, void *A_out,
                                  void *A_inv_out, uint8_t *method, int32_t *k_est,
                                  int64_t *consumed, double *cost, int32_t *info,
                                  void *workspace, void *stream) {
  if (B < 0 || K < 1 || N < 1 || !H || !dH || !A_inv || !omega || !cursor || !cfg ||
      !A_inv_out || !method || !k_est || !consumed || !info || !workspace) {
    lrz_set_error("lrz_update_inverse: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  const int D = cfg->d_max;
  if (D < d_need(cfg, K)) {
    lrz_set_error("lrz_update_inverse: d_max too small");
    return LRZ_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const size_t es = dtype == LRZ_C64 ? 8 : 16, KK = size_t(K) * K;
  char *w = (char *)workspace;
  auto take = [&](size_t n) {
    char *p = w;
    w += al256(n);
    return p;
  };
  c128 *dA = (c128 *)take(B * KK * 16);
  c128 *G = (c128 *)take(B * KK * 16);
  c128 *U = (c128 *)take(size_t(B) * D * K * 16);
  c128 *V = (c128 *)take(size_t(B) * D * K * 16);
  double *S = (double *)take(size_t(B) * D * 8);
  int32_t *iters = (int32_t *)take(size_t(B) * 8);
  int32_t *fallback = (int32_t *)take(size_t(B) * 8);
  int32_t *wb_info = (int32_t *)take(size_t(B) * 8);
  uint8_t *full = (uint8_t *)take(size_t(B) * 8);
  void *Hn = take(size_t(B) * K * N * es);
  void *ws_ar = take(lrz_workspace_bytes(LRZ_WS_ARSVD, dtype, B, K, N, D));
  void *ws_wb = take(lrz_workspace_bytes(LRZ_WS_WOODBURY, dtype, B, K, N, D));
  void *ws_inv = take(lrz_workspace_bytes(LRZ_WS_INVERSE, dtype, B, K, N, D));
  const int64_t hs = int64_t(K) * N;
  int rc;
  // 1. Gram correction of the previous channel and its change (lowrank.py:343)
  if ((rc = lrz_gram_delta(dtype, B, K, N, H, hs, dH, hs, 0, dA, KK, stream))) return rc;
  // 2. arSVD (lowrank.py:344), factor always produced
  if ((rc = lrz_arsvd(B, K, dA, KK, omega, omega_stride, nullptr, cursor, cfg, U, V, S, k_est,
                      iters, fallback, consumed, nullptr, 1, 1, ws_ar, stream)))
    return rc;
  // 3. Woodbury on every item with a factor (lowrank.py:353-359)
  cudaMemsetAsync(wb_info, 0, size_t(B) * 4, s);
  if ((rc = lrz_woodbury(B, K, D, A, A_inv, KK, U, V, S, k_est, A_out, A_inv_out, wb_info,
                         ws_wb, stream)))
    return rc;
  ui_select_kernel<<<unsigned((B + 127) / 128), 128, 0, s>>>(B, K, k_est, wb_info, full, method,
                                                               cost);
  if ((rc = lrz_launch_status("ui_select_kernel"))) return rc;
  // 4. full branch: the true Gram of H + dH and its inverse (lowrank.py:361-373)
  if ((rc = lrz_axpby(dtype, int64_t(B) * hs, 1.0, H, 1.0, dH, Hn, stream))) return rc;
  if ((rc = lrz_gram(dtype, B, K, N, Hn, hs, alpha, G, KK, stream))) return rc;
  cudaMemsetAsync(info, 0, size_t(B) * 4, s);
  if ((rc = lrz_herm_inverse(B, K, G, KK, A_inv_out, KK, info, 1e14, full, ws_inv, stream)))
    return rc;
  ui_assemble_kernel<<<grid_for(B * int64_t(KK)), 256, 0, s>>>(
      B, KK, method, (const c128 *)A, (const c128 *)A_inv, G, (c128 *)A_out, (c128 *)A_inv_out);
  (void)es;
  return lrz_launch_status("lrz_update_inverse");
}

// ------------------------------------------------------------------ trajectory

extern "C" size_t lrz_trajectory_ws(int dtype, int64_t B, int T, int K, int N, int d_max) {
  const int64_t BT = B * T;
  const size_t KK = size_t(K) * K;
  size_t b = 0;
  b += 3 * al256(BT * KK * 16);                                   // G, dA, A^-1 sequence
  b += 2 * al256(size_t(BT));                                     // is_sketch, plan
  b += 2 * al256(size_t(BT) * 8);                                 // cursor, used
  b += 3 * al256(size_t(BT) * 4);                                 // iters_pred, iters, fallback
  b += al256(size_t(B) * 4);                                      // first_unverified
  b += 2 * al256(size_t(BT) * d_max * K * 16);                    // U, V
  b += al256(size_t(BT) * d_max * 8);                             // S
  b += al256(size_t(BT) * 8);                                     // scale
  b += al256(lrz_workspace_bytes(LRZ_WS_ARSVD, dtype, BT, K, N, d_max));
  b += al256(lrz_workspace_bytes(LRZ_WS_INVERSE, dtype, BT, K, N, d_max));
  b += al256(lrz_workspace_bytes(LRZ_WS_CHAIN, dtype, B, K, N, d_max));
  b += al256(lrz_workspace_bytes(LRZ_WS_PRECODE, dtype, BT, K, N, d_max));
  return b;
}

// One time chunk of B trials x T steps of the per-trial sweep
// (harness._sweep_trial, harness.py:221-255), fully digital (F_RF = I):
// Grams, Gram corrections, the arSVD of every dispatcher step IN ORDER per
// trial with the exact sketch cursors (lrz_arsvd_seq), the dispatcher, the
// batched full inversions, the Woodbury chain, the precoder and the rates.
//   H: [B][T][K][N] dtype; noise [B][K]; t0 = global index of the chunk's
//   first step (reset every n_reset steps, config.py:59); cfg NULL = the
//   conventional method.  omega [B] rows (stride omega_stride) start at each
//   trial's first unconsumed normal; consumed[b] (out) = normals this chunk used.
//   State in/out: A_inv_state, A_state ([B][K][K] complex128; A_state nullable),
//   G_prev ([B][K][K], the previous chunk's last Gram; NULL when t0 == 0 or no
//   previous chunk) and G_last (out, nullable) for the next call.
//   Outputs per (b, t): rates, per_ut ([B][T][K]), method, k_est, info;
//   A_inv_seq nullable ([B][T][K][K]).
extern "C" int lrz_trajectory(int dtype, int64_t B, int T, int K, int N, const void *H,
                              double alpha, double P_t, const double *noise, int64_t t0,
                              int n_reset, const lrz_arsvd_cfg *cfg, const double *omega,
                              int64_t omega_stride, void *A_inv_state, void *A_state,
                              const void *G_prev, void *G_last, double *rates, double *per_ut,
                              uint8_t *method, int32_t *k_est, int32_t *info, int64_t *consumed,
                              void *A_inv_seq_out, void *workspace, void *stream) {
  if (B < 0 || T < 1 || K < 1 || N < 1 || !H || !noise || !A_inv_state || !rates || !per_ut ||
      !method || !k_est || !info || !consumed || !workspace || (cfg && !omega)) {
    lrz_set_error("lrz_trajectory: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  const int D = cfg ? cfg->d_max : 1;
  if (cfg && D < d_need(cfg, K)) {
    lrz_set_error("lrz_trajectory: d_max too small");
    return LRZ_EINVAL;
  }
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t BT = B * T;
  const size_t KK = size_t(K) * K;
  char *w = (char *)workspace;
  auto take = [&](size_t n) {
    char *p = w;
    w += al256(n);
    return p;
  };
  c128 *G = (c128 *)take(BT * KK * 16);
  c128 *dA = (c128 *)take(BT * KK * 16);
  c128 *Aseq = (c128 *)take(BT * KK * 16);
  if (A_inv_seq_out) Aseq = (c128 *)A_inv_seq_out;
  uint8_t *is_sketch = (uint8_t *)take(size_t(BT));
  uint8_t *plan = (uint8_t *)take(size_t(BT));
  int64_t *cursor = (int64_t *)take(size_t(BT) * 8);
  int64_t *used = (int64_t *)take(size_t(BT) * 8);
  int32_t *iters_pred = (int32_t *)take(size_t(BT) * 4);
  int32_t *iters = (int32_t *)take(size_t(BT) * 4);
  int32_t *fallback = (int32_t *)take(size_t(BT) * 4);
  int32_t *first = (int32_t *)take(size_t(B) * 4);
  c128 *U = (c128 *)take(size_t(BT) * D * K * 16);
  c128 *V = (c128 *)take(size_t(BT) * D * K * 16);
  double *S = (double *)take(size_t(BT) * D * 8);
  double *scale = (double *)take(size_t(BT) * 8);
  void *ws_ar = take(lrz_workspace_bytes(LRZ_WS_ARSVD, dtype, BT, K, N, D));
  void *ws_inv = take(lrz_workspace_bytes(LRZ_WS_INVERSE, dtype, BT, K, N, D));
  void *ws_ch = take(lrz_workspace_bytes(LRZ_WS_CHAIN, dtype, B, K, N, D));
  void *ws_pr = take(lrz_workspace_bytes(LRZ_WS_PRECODE, dtype, BT, K, N, D));
  int rc;
  // 1. true Grams of every step (harness.py:232 / lowrank.py:160-162)
  if ((rc = lrz_gram(dtype, BT, K, N, H, int64_t(K) * N, alpha, G, KK, stream))) return rc;
  traj_sketch_kernel<<<unsigned((BT + 255) / 256), 256, 0, s>>>(B, T, t0, n_reset,
                                                                G_prev ? 1 : 0, cfg ? 0 : 1,
                                                                is_sketch);
  cudaMemsetAsync(k_est, 0, size_t(BT) * 4, s);
  cudaMemsetAsync(iters, 0, size_t(BT) * 4, s);
  cudaMemsetAsync(used, 0, size_t(BT) * 8, s);
  cudaMemsetAsync(cursor, 0, size_t(BT) * 8, s);
  cudaMemsetAsync(first, 0, size_t(B) * 4, s);
  cudaMemsetAsync(info, 0, size_t(BT) * 4, s);
  if (cfg) {
    // 2. Gram corrections, 3. arSVD of every dispatcher step in order per trial
    traj_delta_kernel<<<grid_for(BT * int64_t(KK)), 256, 0, s>>>(
        B, T, KK, G, (const c128 *)G_prev, dA);
    if ((rc = lrz_arsvd_seq(B, T, K, dA, omega, omega_stride, cfg, is_sketch, first, cursor,
                            iters_pred, U, V, S, k_est, iters, fallback, used, 0, ws_ar,
                            stream)))
      return rc;
  }
  // 4. dispatcher (lowrank.py:345-359)
  if ((rc = lrz_plan(BT, K, is_sketch, k_est, plan, stream))) return rc;
  traj_consumed_kernel<<<unsigned((B + 127) / 128), 128, 0, s>>>(B, T, cursor, used, is_sketch,
                                                                   consumed);
  // 5. full inversions batched (mask = plan == 0, in is_sketch's buffer)
  traj_fullmask_kernel<<<unsigned((BT + 255) / 256), 256, 0, s>>>(BT, plan, is_sketch);
  if ((rc = lrz_herm_inverse(BT, K, G, KK, Aseq, KK, info, 1e14, is_sketch, ws_inv, stream)))
    return rc;
  // 6. the Woodbury chain per trial (lowrank.py:182-227; step-parallel for K > 64,
  //    resident per-trial CTAs up to K = 64)
  if (cfg) {
    rc = K > 64 ? lrz_chain_steps(B, T, K, D, plan, G, A_inv_state, Aseq, A_state, U, V, S,
                                  k_est, method, info, ws_ch, stream)
                : lrz_chain(B, T, K, D, plan, G, A_inv_state, Aseq, A_state, U, V, S, k_est,
                            method, info, ws_ch, stream);
    if (rc) return rc;
  } else {
    cudaMemsetAsync(method, LRZ_METHOD_FULL, size_t(BT), s);
  }
  // 7. precoder + rate, H W from the Gram
  if ((rc = lrz_precode_rate(dtype, BT, K, N, H, int64_t(K) * N, Aseq, KK, P_t, noise, T,
                             nullptr, 0, G, alpha, scale, per_ut, nullptr, rates, iters,
                             ws_pr, stream)))
    return rc;
  // per-step status: the inverse's code (singular / indefinite) first, then the
  // precoder's (zero norm) -- a singular step is never hidden by a later code
  traj_info_kernel<<<unsigned((BT + 255) / 256), 256, 0, s>>>(BT, iters, info);
  // state for the next chunk
  traj_tail_kernel<<<grid_for(B * int64_t(KK)), 256, 0, s>>>(B, T, KK, Aseq, G,
                                                            (c128 *)A_inv_state, (c128 *)G_last);
  return lrz_launch_status("lrz_trajectory");
}

// On-device synthesis of the synthetic LEO Rician-drift channels
// (paper_2512_16543_b200/scenario.py, SURVEY.md 8(d)/(f) "next" #1).
//
// H_t[k][m] = sqrt(beta_k) ( a_k e^{j phi_k} e^{-j 2 pi sin th_k(t)
//             (cos psi_k x_m + sin psi_k y_m)} + b_k S[k][m] ),
// th_k(t) = th0_k + drift_k t, a_k = sqrt(kappa/(1+kappa)), b_k = sqrt(1/(1+kappa)),
// element m = ix * n + iy at ((ix - (n-1)/2)/2, (iy - (n-1)/2)/2) wavelengths
// (reference channel.py:46-59, conjugated rows channel.py:128-137).
// The scatter S comes from the trial's channel stream (device RNG, same
// normals as numpy); per-trial angles/gains are drawn on the host.  The
// arithmetic follows scenario.trial_channels operation by operation, so the
// result equals the host generator to the last bits of sin/cos/exp.

#include "common.cuh"

namespace lrz {

template <typename E>
__global__ void channel_kernel(int64_t B, int t0, int T, int K, int N, int n_side,
                               const double *__restrict__ par,   // [B][6][K]
                               const double *__restrict__ scat,  // [B][2 K N] (re block, im block)
                               int64_t scat_stride, cplx<E> *__restrict__ H) {
  // one warp per channel row (b, t, k): the per-row terms (sin / cos of the
  // angles, the LoS phase offset, the Rician weights, the gain) are computed
  // once per lane and reused for the row's N / 32 antennas per lane, instead
  // of once per entry; the arithmetic per entry is unchanged (same operations,
  // same order), so the result is still the host generator's to the last bit
  const int64_t rows = B * int64_t(T) * K;
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int64_t nw = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const double c = (n_side - 1) / 2.0;
  const double twopi = 2.0 * 3.141592653589793;
  for (int64_t row = w0; row < rows; row += nw) {
    const int k = int(row % K);
    int64_t r = row / K;
    const int t = int(r % T);
    const int64_t b = r / T;
    const double *p = par + b * 6 * K;
    const double th0 = p[k], psi = p[K + k], phi = p[2 * K + k], beta = p[3 * K + k],
                 kap = p[4 * K + k], drift = p[5 * K + k];
    // every product and sum rounded separately, in numpy's order (no FMA contraction)
    const double theta = __dadd_rn(th0, __dmul_rn(drift, double(t0 + t)));
    const double st = sin(theta);
    const double kx = __dmul_rn(st, cos(psi)), ky = __dmul_rn(st, sin(psi));
    double sp, cp;
    sincos(phi, &sp, &cp);
    const double al = sqrt(__ddiv_rn(kap, __dadd_rn(1.0, kap)));
    const double an = sqrt(__ddiv_rn(1.0, __dadd_rn(1.0, kap)));
    const double g = sqrt(beta);
    const double *sc = scat + b * scat_stride;
    cplx<E> *h = H + row * N;
    for (int m = lane; m < N; m += 32) {
      const double x = __dmul_rn(double(m / n_side) - c, 0.5);
      const double y = __dmul_rn(double(m % n_side) - c, 0.5);
      const double phase = __dmul_rn(twopi, __dadd_rn(__dmul_rn(kx, x), __dmul_rn(ky, y)));
      double sph, cph;
      sincos(phase, &sph, &cph);
      // exp(-j phase) * exp(j phi) as numpy's complex product (a c - b d, a d + b c)
      const double lr = __dsub_rn(__dmul_rn(cph, cp), __dmul_rn(-sph, sp));
      const double li = __dadd_rn(__dmul_rn(cph, sp), __dmul_rn(-sph, cp));
      const double sr = __dmul_rn(sc[int64_t(k) * N + m], 0.7071067811865476);
      const double si = __dmul_rn(sc[int64_t(K) * N + int64_t(k) * N + m], 0.7071067811865476);
      const double hr = __dmul_rn(g, __dadd_rn(__dmul_rn(al, lr), __dmul_rn(an, sr)));
      const double hi = __dmul_rn(g, __dadd_rn(__dmul_rn(al, li), __dmul_rn(an, si)));
      h[m] = mk<E>(E(hr), E(hi));
    }
  }
}

}  // namespace lrz

using namespace lrz;

extern "C" int lrz_channels(int dtype, int64_t B, int t0, int T, int K, int N, int n_side,
                            const double *params, const double *scatter, int64_t scatter_stride,
                            void *H, void *stream) {
  if (B < 0 || T < 1 || K < 1 || N < 1 || n_side * n_side != N || !params || !scatter || !H) {
    lrz_set_error("lrz_channels: bad arguments");
    return LRZ_EINVAL;
  }
  if (B == 0) return LRZ_OK;
  const int64_t rows = B * int64_t(T) * K;  // one warp per row
  const unsigned nb = unsigned(std::min<int64_t>((rows + 7) / 8, 148 * 64));
  cudaStream_t s = (cudaStream_t)stream;
  LrzProf prof("channel_kernel", s);
  if (dtype == LRZ_C64)
    channel_kernel<float><<<nb, 256, 0, s>>>(B, t0, T, K, N, n_side, params, scatter,
                                             scatter_stride, (c64 *)H);
  else
    channel_kernel<double><<<nb, 256, 0, s>>>(B, t0, T, K, N, n_side, params, scatter,
                                              scatter_stride, (c128 *)H);
  return lrz_launch_status("lrz_channels");
}

// kspace.cu -- Fourier-space scaling and Green's-table kernels.
//
// k-space scaling (reference: ewald_fourier.py:393-483 fused kernels and the
// NumPy wall-channel block :578-611) is done in ONE pass over the R2C half
// spectrum: every k-point reads all source-channel spectra and the two real
// tables once, and writes the six output spectra T1 = t1 + e3 phi and
// T2 = i k phi in place (HBM-bound, 16 B per complex channel per k-point).
// The scipy inverse normalisation 1/N_pad is folded in.
//
// R2C/C2R vs the reference's full complex FFT + `.real`: Re(ifftn(Y)) equals
// ifftn of the Hermitian part (Y(k) + conj(Y(-k)))/2.  Off the Nyquist planes
// the multipliers already satisfy Y(-k) = conj(Y(k)); on a Nyquist plane the
// fftfreq value -pi/h maps to itself under k -> -k, so we symmetrise
// explicitly: out = (m(k) C + conj(m(k~) conj(C)))/2 with k~ = k on Nyquist
// components and -k elsewhere.  This keeps terms even in the Nyquist component
// and cancels odd ones, exactly like the reference's `.real`.
//
// Channel layouts (spectra, channel-major, each (px, py, pz/2+1) complex):
//   stokeslet: F0 F1 F2 | S V0 V1 V2            (7, half) / 3 (free)
//   stresslet: C00 C01 C02 C11 C12 C22 | V2 M00 M01 M02 M11 M12 M22   (13 / 6)
//              (symmetric parts only: the kernel multiplier depends on sym(C) alone)
//   rotlet:    W0 W1 W2 | V0 V1                  (5 / 3)
//   outputs:   T1x T1y T1z [T2x T2y T2z]  written to channels 0..5
#define HS_TU_ID 6  // checked build: source of a failing HS_CHECK
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace hs {

struct cplx {
  double re, im;
};
__device__ __forceinline__ cplx cmul_i(cplx a) { return {-a.im, a.re}; }      // i a
__device__ __forceinline__ cplx cscale(double s, cplx a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cplx cconj(cplx a) { return {a.re, -a.im}; }

// numpy fftfreq * 2 pi: index i of n (even n): i < n/2 -> i, else i - n
__device__ __forceinline__ double kval(int i, int n, double kscale) {
  const int j = (i < n / 2) ? i : i - n;
  return (2.0 * kPi) * ((double)j * kscale);
}

// m(k) applied to channels C -> out (6 complex).  G, F, Fc already include normalisation.
template <int KIND, bool HALF>
__device__ __forceinline__ void apply_multiplier(double kx, double ky, double kz, double G, double Fc,
                                                 const cplx* C, cplx* out) {
  const double k2 = kx * kx + ky * ky + kz * kz;
  if (KIND == HS_STOKESLET) {
    // t1_j = -G (k^2 C_j - k_j (k.C))   (ewald_fourier.py:394-414)
    const cplx kd = cadd(cadd(cscale(kx, C[0]), cscale(ky, C[1])), cscale(kz, C[2]));
    out[0] = cscale(-G, csub(cscale(k2, C[0]), cscale(kx, kd)));
    out[1] = cscale(-G, csub(cscale(k2, C[1]), cscale(ky, kd)));
    out[2] = cscale(-G, csub(cscale(k2, C[2]), cscale(kz, kd)));
  } else if (KIND == HS_STRESSLET) {
    // sym C: 0:00 1:01 2:02 3:11 4:12 5:22.  u + w = 2 S k, tr = S00+S11+S22, s = k.S.k
    // t1_j = -iG [k^2 (2 (Sk)_j + k_j tr) - 2 k_j s]   (ewald_fourier.py:417-459)
    const cplx Sk0 = cadd(cadd(cscale(kx, C[0]), cscale(ky, C[1])), cscale(kz, C[2]));
    const cplx Sk1 = cadd(cadd(cscale(kx, C[1]), cscale(ky, C[3])), cscale(kz, C[4]));
    const cplx Sk2 = cadd(cadd(cscale(kx, C[2]), cscale(ky, C[4])), cscale(kz, C[5]));
    const cplx tr = cadd(cadd(C[0], C[3]), C[5]);
    const cplx s = cadd(cadd(cscale(kx, Sk0), cscale(ky, Sk1)), cscale(kz, Sk2));
    const cplx v0 = csub(cscale(k2, cadd(cscale(2.0, Sk0), cscale(kx, tr))), cscale(2.0 * kx, s));
    const cplx v1 = csub(cscale(k2, cadd(cscale(2.0, Sk1), cscale(ky, tr))), cscale(2.0 * ky, s));
    const cplx v2 = csub(cscale(k2, cadd(cscale(2.0, Sk2), cscale(kz, tr))), cscale(2.0 * kz, s));
    out[0] = cscale(-G, cmul_i(v0));
    out[1] = cscale(-G, cmul_i(v1));
    out[2] = cscale(-G, cmul_i(v2));
  } else {
    // t1 = -2i F (C x k)   (ewald_fourier.py:462-483); G carries F here
    const cplx x0 = csub(cscale(kz, C[1]), cscale(ky, C[2]));
    const cplx x1 = csub(cscale(kx, C[2]), cscale(kz, C[0]));
    const cplx x2 = csub(cscale(ky, C[0]), cscale(kx, C[1]));
    out[0] = cscale(-2.0 * G, cmul_i(x0));
    out[1] = cscale(-2.0 * G, cmul_i(x1));
    out[2] = cscale(-2.0 * G, cmul_i(x2));
  }
  if (HALF) {
    // phi = Fc (S + i k.V - k_l k_m M_lm)   (ewald_fourier.py:578-611)
    cplx phi;
    if (KIND == HS_STOKESLET) {
      const cplx kv = cadd(cadd(cscale(kx, C[4]), cscale(ky, C[5])), cscale(kz, C[6]));
      phi = cscale(Fc, cadd(C[3], cmul_i(kv)));
    } else if (KIND == HS_STRESSLET) {
      const cplx kMk = cadd(cadd(cadd(cscale(kx * kx, C[7]), cscale(2.0 * kx * ky, C[8])),
                                 cadd(cscale(2.0 * kx * kz, C[9]), cscale(ky * ky, C[10]))),
                            cadd(cscale(2.0 * ky * kz, C[11]), cscale(kz * kz, C[12])));
      phi = cscale(Fc, csub(cmul_i(cscale(kz, C[6])), kMk));
    } else {
      const cplx kv = cadd(cscale(kx, C[3]), cscale(ky, C[4]));
      phi = cscale(Fc, cmul_i(kv));
    }
    out[2] = cadd(out[2], phi);
    out[3] = cmul_i(cscale(kx, phi));
    out[4] = cmul_i(cscale(ky, phi));
    out[5] = cmul_i(cscale(kz, phi));
  }
}

template <int KIND, bool HALF>
__global__ void __launch_bounds__(256) k_scale(KGeom g, const double* __restrict__ tabB, const double* __restrict__ tabH,
                                               double2* __restrict__ spec, int64_t ch_stride) {
  constexpr int NIN = KIND == HS_STOKESLET ? (HALF ? 7 : 3) : KIND == HS_STRESSLET ? (HALF ? 13 : 6) : (HALF ? 5 : 3);
  constexpr int NOUT = HALF ? 6 : 3;
  const int64_t npt = (int64_t)g.p[0] * g.p[1] * g.nzh;
  const double s8 = 1.0 / (8.0 * kPi), s4 = 1.0 / (4.0 * kPi);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npt; i += (int64_t)gridDim.x * blockDim.x) {
    const int iz = (int)(i % g.nzh);
    const int iy = (int)((i / g.nzh) % g.p[1]);
    const int ix = (int)(i / ((int64_t)g.nzh * g.p[1]));
    const double kx = kval(ix, g.p[0], g.kscale[0]);
    const double ky = kval(iy, g.p[1], g.kscale[1]);
    const double kz = kval(iz, g.p[2], g.kscale[2]);
    const double k2 = kx * kx + ky * ky + kz * kz;
    const double E = exp(-g.a * k2);
    double G;
    if (KIND == HS_ROTLET)
      G = tabH[i] * E * s4 * g.inv_n;
    else
      G = tabB[i] * E * (1.0 + g.b * k2) * s8 * g.inv_n;
    const double Fc = HALF ? tabH[i] * E * s4 * g.inv_n : 0.0;
    cplx C[NIN];
#pragma unroll
    for (int c = 0; c < NIN; ++c) {
      const double2 v = spec[c * ch_stride + i];
      C[c] = {v.x, v.y};
    }
    cplx out[6];
    apply_multiplier<KIND, HALF>(kx, ky, kz, G, Fc, C, out);
    const bool nyq = (2 * ix == g.p[0]) || (2 * iy == g.p[1]) || (2 * iz == g.p[2]);
    if (nyq) {
      const double tx = (2 * ix == g.p[0]) ? kx : -kx;
      const double ty = (2 * iy == g.p[1]) ? ky : -ky;
      const double tz = (2 * iz == g.p[2]) ? kz : -kz;
      cplx Cc[NIN], o2[6];
#pragma unroll
      for (int c = 0; c < NIN; ++c) Cc[c] = cconj(C[c]);
      apply_multiplier<KIND, HALF>(tx, ty, tz, G, Fc, Cc, o2);
#pragma unroll
      for (int c = 0; c < NOUT; ++c) out[c] = cscale(0.5, cadd(out[c], cconj(o2[c])));
    }
#pragma unroll
    for (int c = 0; c < NOUT; ++c) spec[c * ch_stride + i] = make_double2(out[c].re, out[c].im);
  }
}

hs_status launch_kscale(hs_ctx* ctx, int kind, int half, const KGeom& k, const double* tabB, const double* tabH,
                        double2* spec, int64_t ch_stride) {
  const int64_t npt = (int64_t)k.p[0] * k.p[1] * k.nzh;
  const int gs = (int)std::min<int64_t>(ceil_div(npt, 256), (int64_t)ctx->sm_count * 16);
#define HS_KS(K, H) k_scale<K, H><<<gs, 256, 0, ctx->stream>>>(k, tabB, tabH, spec, ch_stride)
  if (half) {
    if (kind == HS_STOKESLET) HS_KS(HS_STOKESLET, true);
    else if (kind == HS_STRESSLET) HS_KS(HS_STRESSLET, true);
    else HS_KS(HS_ROTLET, true);
  } else {
    if (kind == HS_STOKESLET) HS_KS(HS_STOKESLET, false);
    else if (kind == HS_STRESSLET) HS_KS(HS_STRESSLET, false);
    else HS_KS(HS_ROTLET, false);
  }
#undef HS_KS
  HS_LAUNCHED(ctx);
  return HS_OK;
}

// ---------------------------------------------------------------------------
// Green's tables (ewald_fourier.py:154-174 truncated_greens_hat, :207-244 precompute_greens)
// truncated Green's function at |k| (ewald_fourier.py:154-174)
__device__ __forceinline__ double greens_hat_value(int kind, double R, double kmag) {
  const double x = R * kmag;
  if (kind == HS_HARMONIC) {
    // 2 pi R^2 sinc(x / 2 pi)^2, np.sinc(t) = sin(pi t)/(pi t)
    const double t = x / (2.0 * kPi);
    double sc = 1.0;
    if (t != 0.0) {
      const double pt = kPi * t;
      sc = sin(pt) / pt;
    }
    return 2.0 * kPi * R * R * sc * sc;
  }
  const double R4 = R * R * R * R;
  const double x2 = x * x;
  if (x < 0.3) return kPi * R4 * (1.0 - x2 / 9.0 + x2 * x2 / 240.0 - x2 * x2 * x2 / 12600.0);
  return 4.0 * kPi * R4 * ((2.0 - x2) * cos(x) + 2.0 * x * sin(x) - 2.0) / (x2 * x2);
}

__global__ void k_greens_hat(int kind, double R, double ks0, double ks1, double ks2, int64_t n0, int64_t n1,
                             int64_t n2, int64_t nzh, double2* __restrict__ out) {
  const int64_t npt = n0 * n1 * nzh;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npt; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t iz = i % nzh, iy = (i / nzh) % n1, ix = i / (nzh * n1);
    // fftfreq for n0 (even or odd): i <= (n-1)/2 -> i, else i - n
    const int64_t fx = ix <= (n0 - 1) / 2 ? ix : ix - n0;
    const int64_t fy = iy <= (n1 - 1) / 2 ? iy : iy - n1;
    const double kx = (2.0 * kPi) * ((double)fx * ks0);
    const double ky = (2.0 * kPi) * ((double)fy * ks1);
    const double kz = (2.0 * kPi) * ((double)iz * ks2);  // rfftfreq: 0..n/2
    out[i] = make_double2(greens_hat_value(kind, R, sqrt(kx * kx + ky * ky + kz * kz)), 0.0);
  }
}

// ---- separable, pruned table precompute (no big-grid array) --------------------------------
// The truncated Green's function is real and even in every frequency index, so the
// irfftn on the oversampled grid is a product of three cosine transforms, each a 1-D C2R
// of a real "half spectrum".  Evaluated dimension by dimension (z, then y, then x), keeping
// after each stage only the real-space nodes the crop needs (0..k_i, with the crop's
// wrapped half following from evenness), the largest intermediate is
// h0 x (k2+1) x h1 complex instead of the big grid.
// stage-1 input: lines l = (kx, ky) in [0,h0) x [0,h1), values at kz in [0, h2)
__global__ void k_hat_lines(int kind, double R, double ks0, double ks1, double ks2, int64_t l0, int64_t nl, int64_t h1,
                            int64_t h2, int64_t ltot, double2* __restrict__ out) {
  const int64_t npt = nl * h2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npt; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t line = l0 + i / h2, kz = i % h2;
    double v = 0.0;
    if (line < ltot) {
      const int64_t kx = line / h1, ky = line % h1;
      const double a = (2.0 * kPi) * ((double)kx * ks0), b = (2.0 * kPi) * ((double)ky * ks1),
                   c = (2.0 * kPi) * ((double)kz * ks2);
      v = greens_hat_value(kind, R, sqrt(a * a + b * b + c * c));
    }
    out[i] = make_double2(v, 0.0);
  }
}

// real C2R outputs of lines [l0, l0+nl) (length n each) -> next stage, keeping nodes 0..kp-1:
// line l = (a, b), b in [0, nb), a in [0, na): dst[((node * na) + a) * nb + b] = (scale v, 0)
// (complex rows of the next transform, b contiguous), or, when dst_real != null,
// dst_real[l * kp + node] = scale v
__global__ void k_sep_scatter(const double* __restrict__ src, int64_t l0, int64_t nl, int64_t ltot, int64_t n,
                              int64_t kp, int64_t na, int64_t nb, double scale, double2* __restrict__ dst,
                              double* __restrict__ dst_real) {
  const int64_t npt = nl * kp;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npt; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t li = i / kp, node = i % kp, line = l0 + li;
    if (line >= ltot) continue;
    const double v = scale * src[li * n + node];
    if (dst_real) {
      dst_real[line * kp + node] = v;
    } else {
      const int64_t a = line / nb, b = line % nb;
      dst[(node * na + a) * nb + b] = make_double2(v, 0.0);
    }
  }
}

// crop[cx][cy][cz] (shape 2k) = F[|y|][|z|][|x|] with |c| = c < k ? c : 2k - c; F: (k1+1, k2+1, k0+1)
__global__ void k_sep_crop(const double* __restrict__ F, int64_t k0, int64_t k1, int64_t k2,
                           double* __restrict__ crop) {
  const int64_t c0 = 2 * k0, c1 = 2 * k1, c2 = 2 * k2;
  const int64_t npt = c0 * c1 * c2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npt; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % c2, y = (i / c2) % c1, x = i / (c2 * c1);
    const int64_t ax = x < k0 ? x : c0 - x, ay = y < k1 ? y : c1 - y, az = z < k2 ? z : c2 - z;
    crop[i] = F[(ay * (k2 + 1) + az) * (k0 + 1) + ax];
  }
}

hs_status launch_hat_lines(hs_ctx* ctx, int kind, double R, double h, const int64_t big[3], int64_t l0, int64_t nl,
                           int64_t h1, int64_t h2, int64_t ltot, double2* out) {
  const int gs = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nl * h2, 256), (int64_t)ctx->sm_count * 16));
  k_hat_lines<<<gs, 256, 0, ctx->stream>>>(kind, R, 1.0 / ((double)big[0] * h), 1.0 / ((double)big[1] * h),
                                           1.0 / ((double)big[2] * h), l0, nl, h1, h2, ltot, out);
  HS_LAUNCHED(ctx);
  return HS_OK;
}
hs_status launch_sep_scatter(hs_ctx* ctx, const double* src, int64_t l0, int64_t nl, int64_t ltot, int64_t n,
                             int64_t kp, int64_t na, int64_t nb, double scale, double2* dst, double* dst_real) {
  const int gs = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nl * kp, 256), (int64_t)ctx->sm_count * 16));
  k_sep_scatter<<<gs, 256, 0, ctx->stream>>>(src, l0, nl, ltot, n, kp, na, nb, scale, dst, dst_real);
  HS_LAUNCHED(ctx);
  return HS_OK;
}
hs_status launch_sep_crop(hs_ctx* ctx, const double* F, const int64_t k[3], double* crop) {
  const int64_t npt = 8 * k[0] * k[1] * k[2];
  const int gs = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(npt, 256), (int64_t)ctx->sm_count * 16));
  k_sep_crop<<<gs, 256, 0, ctx->stream>>>(F, k[0], k[1], k[2], crop);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

hs_status launch_greens_hat(hs_ctx* ctx, int kind, double R, double h, const int64_t big[3], double2* out) {
  const int64_t nzh = big[2] / 2 + 1;
  const int64_t npt = big[0] * big[1] * nzh;
  const int gs = (int)std::min<int64_t>(ceil_div(npt, 256), (int64_t)ctx->sm_count * 16);
  // numpy fftfreq spacing: 1/(n*d)
  k_greens_hat<<<gs, 256, 0, ctx->stream>>>(kind, R, 1.0 / ((double)big[0] * h), 1.0 / ((double)big[1] * h),
                                            1.0 / ((double)big[2] * h), big[0], big[1], big[2], nzh, out);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

// crop = field[ix_(keep_x, keep_y, keep_z)], keep_i = [0:k_i] U [b_i - k_i : b_i] (k_i = d_i + g_i)
__global__ void k_crop(const double* __restrict__ field, int64_t b0, int64_t b1, int64_t b2, int64_t k0, int64_t k1,
                       int64_t k2, double scale, double* __restrict__ crop) {
  const int64_t c0 = 2 * k0, c1 = 2 * k1, c2 = 2 * k2;
  const int64_t npt = c0 * c1 * c2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npt; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t z = i % c2, y = (i / c2) % c1, x = i / (c2 * c1);
    const int64_t sx = x < k0 ? x : b0 - 2 * k0 + x;
    const int64_t sy = y < k1 ? y : b1 - 2 * k1 + y;
    const int64_t sz = z < k2 ? z : b2 - 2 * k2 + z;
    crop[i] = field[(sx * b1 + sy) * b2 + sz] * scale;
  }
}

hs_status launch_crop(hs_ctx* ctx, const double* field, const int64_t big[3], const int64_t keep[3], double scale,
                      double* crop) {
  const int64_t npt = 8 * keep[0] * keep[1] * keep[2];
  const int gs = (int)std::min<int64_t>(ceil_div(npt, 256), (int64_t)ctx->sm_count * 16);
  k_crop<<<gs, 256, 0, ctx->stream>>>(field, big[0], big[1], big[2], keep[0], keep[1], keep[2], scale, crop);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

__global__ void k_real_part(const double2* __restrict__ spec, int64_t n, double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = spec[i].x;
}

hs_status launch_real_part(hs_ctx* ctx, const double2* spec, int64_t n, double* out) {
  const int gs = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->sm_count * 16);
  k_real_part<<<gs, 256, 0, ctx->stream>>>(spec, n, out);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

// full[ix,iy,iz] (real, shape p) from the real part of an R2C half spectrum: for iz > p2/2 use the
// Hermitian partner (-ix, -iy, p2 - iz).
__global__ void k_expand_half(const double2* __restrict__ half_spec, int64_t p0, int64_t p1, int64_t p2,
                              double* __restrict__ full) {
  const int64_t nzh = p2 / 2 + 1;
  const int64_t npt = p0 * p1 * p2;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npt; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t iz = i % p2, iy = (i / p2) % p1, ix = i / (p2 * p1);
    double v;
    if (iz < nzh) {
      v = half_spec[(ix * p1 + iy) * nzh + iz].x;
    } else {
      const int64_t jx = (p0 - ix) % p0, jy = (p1 - iy) % p1, jz = p2 - iz;
      v = half_spec[(jx * p1 + jy) * nzh + jz].x;
    }
    full[i] = v;
  }
}

hs_status launch_expand_half(hs_ctx* ctx, const double2* half_spec, const int64_t p[3], double* full) {
  const int64_t npt = p[0] * p[1] * p[2];
  const int gs = (int)std::min<int64_t>(ceil_div(npt, 256), (int64_t)ctx->sm_count * 16);
  k_expand_half<<<gs, 256, 0, ctx->stream>>>(half_spec, p[0], p[1], p[2], full);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

__global__ void k_take_half(const double* __restrict__ full, int64_t p0, int64_t p1, int64_t p2,
                            double* __restrict__ half) {
  const int64_t nzh = p2 / 2 + 1;
  const int64_t npt = p0 * p1 * nzh;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < npt; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t iz = i % nzh, r = i / nzh;
    half[i] = full[r * p2 + iz];
  }
}

hs_status launch_take_half(hs_ctx* ctx, const double* full, const int64_t p[3], double* half) {
  const int64_t npt = p[0] * p[1] * (p[2] / 2 + 1);
  const int gs = (int)std::min<int64_t>(ceil_div(npt, 256), (int64_t)ctx->sm_count * 16);
  k_take_half<<<gs, 256, 0, ctx->stream>>>(full, p[0], p[1], p[2], half);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

HS_DEFINE_CHECK_COLLECT(kspace)

}  // namespace hs

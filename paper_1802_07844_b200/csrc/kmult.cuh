// kmult.cuh -- k-space multipliers of the half-space Spectral-Ewald kernels
// (reference: ewald_fourier.py:393-483 fused kernels, :578-611 wall channels).
//
// Channel layouts (spectra, one per source channel):
//   stokeslet: F0 F1 F2 | S V0 V1 V2                          (7 half / 3 free)
//   stresslet: C00 C01 C02 C11 C12 C22 | V2 M00 M01 M02 M11 M12 M22   (13 / 6)
//              (symmetric parts only: the multiplier depends on sym(C) alone)
//   rotlet:    W0 W1 W2 | V0 V1                               (5 / 3)
//   mixed plan (19 / 9 spectra): F0 F1 F2 S V0 V1 V2 M00 M01 M02 M11 M12 M22 | C00 C01 C02 C11 C12 C22
//              (wall channels shared by both kinds: s, v = v_stokeslet + v_stresslet, M =
//              M_stresslet).  Two x-stage passes: the first 13 as HS_MIXED (stokeslet kernel +
//              the shared wall channels; 13 / 3 inputs half / free), then the C channels as
//              HS_STRESSLET without wall channels, added to T1.  (A three-pass split with <= 7
//              inputs per pass measured slower at px = 864: 400 vs 325 ms for cfg5 -- six more
//              inverse line FFTs, and the register x stage keeps one CTA per SM there either way.)
//   outputs:   T1x T1y T1z [T2x T2y T2z]
#pragma once
#include "common.cuh"

namespace hs {

struct cplx {
  double re, im;
};
__device__ __forceinline__ cplx cmul_i(cplx a) { return {-a.im, a.re}; }  // i a
__device__ __forceinline__ cplx cscale(double s, cplx a) { return {s * a.re, s * a.im}; }
__device__ __forceinline__ cplx cadd(cplx a, cplx b) { return {a.re + b.re, a.im + b.im}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cplx cconj(cplx a) { return {a.re, -a.im}; }

template <int KIND, bool HALF>
struct KChan {
  static constexpr int NIN = KIND == HS_STOKESLET ? (HALF ? 7 : 3)
                           : KIND == HS_STRESSLET ? (HALF ? 13 : 6)
                           : KIND == HS_MIXED     ? (HALF ? 13 : 3)
                                                  : (HALF ? 5 : 3);
  static constexpr int NOUT = HALF ? 6 : 3;
};

// numpy fftfreq * 2 pi: index i of n (even n): i < n/2 -> i, else i - n
__device__ __forceinline__ double kval(int i, int n, double kscale) {
  const int j = (i < n / 2) ? i : i - n;
  return (2.0 * kPi) * ((double)j * kscale);
}

// m(k) applied to channels C -> out.  G (or F for the rotlet) and Fc include the normalisation.
template <int KIND, bool HALF>
__device__ __forceinline__ void apply_multiplier(double kx, double ky, double kz, double G, double Fc, const cplx* C,
                                                 cplx* out) {
  const double k2 = kx * kx + ky * ky + kz * kz;
  if (KIND == HS_STOKESLET || KIND == HS_MIXED) {
    // t1_j = -G (k^2 C_j - k_j (k.C))   (ewald_fourier.py:394-414)
    const cplx kd = cadd(cadd(cscale(kx, C[0]), cscale(ky, C[1])), cscale(kz, C[2]));
    out[0] = cscale(-G, csub(cscale(k2, C[0]), cscale(kx, kd)));
    out[1] = cscale(-G, csub(cscale(k2, C[1]), cscale(ky, kd)));
    out[2] = cscale(-G, csub(cscale(k2, C[2]), cscale(kz, kd)));
  } else if (KIND == HS_STRESSLET) {
    // u + w = 2 S k, tr = S00+S11+S22, s = k.S.k ; t1_j = -iG [k^2 (2 (Sk)_j + k_j tr) - 2 k_j s]
    // (ewald_fourier.py:417-459)
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
    // t1 = -2i F (C x k)   (ewald_fourier.py:462-483)
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
    } else if (KIND == HS_MIXED) {
      // both kinds' wall channels: Fc (S + i k.V - k_l k_m M_lm)
      const cplx kv = cadd(cadd(cscale(kx, C[4]), cscale(ky, C[5])), cscale(kz, C[6]));
      const cplx kMk = cadd(cadd(cadd(cscale(kx * kx, C[7]), cscale(2.0 * kx * ky, C[8])),
                                 cadd(cscale(2.0 * kx * kz, C[9]), cscale(ky * ky, C[10]))),
                            cadd(cscale(2.0 * ky * kz, C[11]), cscale(kz * kz, C[12])));
      phi = cscale(Fc, csub(cadd(C[3], cmul_i(kv)), kMk));
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

// Full scaling at one k-point including the Nyquist symmetrisation that reproduces the
// reference's Re(ifftn(.)) (see kspace.cu header).  ix/iy/iz are FFT indices.
template <int KIND, bool HALF>
__device__ __forceinline__ void scale_point(int ix, int iy, int iz, const int* p, const double* kscale, double a,
                                            double b, double inv_n, double tB, double tH, const cplx* C, cplx* out) {
  constexpr int NIN = KChan<KIND, HALF>::NIN, NOUT = KChan<KIND, HALF>::NOUT;
  const double s8 = 1.0 / (8.0 * kPi), s4 = 1.0 / (4.0 * kPi);
  const double kx = kval(ix, p[0], kscale[0]);
  const double ky = kval(iy, p[1], kscale[1]);
  const double kz = kval(iz, p[2], kscale[2]);
  const double k2 = kx * kx + ky * ky + kz * kz;
  const double E = exp(-a * k2);
  const double G = (KIND == HS_ROTLET) ? tH * E * s4 * inv_n : tB * E * (1.0 + b * k2) * s8 * inv_n;
  const double Fc = HALF ? tH * E * s4 * inv_n : 0.0;
  apply_multiplier<KIND, HALF>(kx, ky, kz, G, Fc, C, out);
  const bool nx_ = 2 * ix == p[0], ny_ = 2 * iy == p[1], nz_ = 2 * iz == p[2];
  if (nx_ || ny_ || nz_) {
    cplx Cc[NIN], o2[6];
#pragma unroll
    for (int c = 0; c < NIN; ++c) Cc[c] = cconj(C[c]);
    apply_multiplier<KIND, HALF>(nx_ ? kx : -kx, ny_ ? ky : -ky, nz_ ? kz : -kz, G, Fc, Cc, o2);
#pragma unroll
    for (int c = 0; c < NOUT; ++c) out[c] = cscale(0.5, cadd(out[c], cconj(o2[c])));
  }
}

}  // namespace hs

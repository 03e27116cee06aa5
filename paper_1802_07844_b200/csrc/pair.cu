// pair.cu -- FP64 screened pair kernel for the real-space Ewald sum
// (reference: ewald_real.py:258-374 `_real_pair_sums`, assembled at :381-455)
// and the unscreened O(N Nt) direct sum (kernels_direct.py:211-294).
//
// Work decomposition (B200): one CTA per non-empty target cell (cell edge
// r_c/2, reach 2 => the 5x5x5 neighbourhood of the cell = 25 contiguous
// z-runs of the cell-sorted source array).  Candidates are staged through
// shared memory in chunks of PT_K rows; each warp owns PT_G targets.  Lanes
// test 32 candidates at a time against all PT_G targets with the reference's
// exact comparison r2 = (d0*d0 + d1*d1) + d2*d2 <= rc*rc (explicitly rounded,
// no FMA contraction, so accepted neighbour sets are bit-identical), and the
// accepted (target, candidate) pairs are compacted per target into a warp
// queue (ballot + popc).  Every full queue of 32 pairs is evaluated with all
// 32 lanes busy and accumulated lane-privately; per-target sums are reduced
// with warp shuffles at the end.  Divergence is therefore confined to the
// cheap test, not the erfc/exp-heavy kernel evaluation.
//
// The screened harmonic coefficients use closed forms free of the
// reference's 1/r - erf(xi r)/r cancellation (kernels_direct.py:130-151):
//   c0 = C/r, c1 = (C/r + e)/r^2, c2 = (3 c1 + 2 xi^2 e)/r^2,
//   c3 = -(5 c2 + 4 xi^4 e)/r^2,  e = (2 xi/sqrt(pi)) exp(-xi^2 r^2), C = erfc(xi r)
// which reduce to (1/r, 1/r^3, 3/r^5, -15/r^7) for the direct sum (C=1, e=0).
#define HS_TU_ID 1  // checked build: source of a failing HS_CHECK
#include "common.cuh"
#include "kernels.cuh"

namespace hs {

namespace {
#include "erfcx_table.inc"
}
__device__ double2 g_erfcx_coef[HS_ERFCX_NPAIR * HS_ERFCX_NINT];
static bool g_erfcx_ready = false;

// erfc(x) = exp(-x^2) erfcx(x); E = exp(-x^2) is already computed by the caller.
// Piecewise degree-10 polynomials on [0, 8) (tools/gen_erfcx.py, max rel. error ~1.3e-15),
// coefficient pairs read with one 16-byte shared-memory load each.
// Branch-free: x >= 8 (only reachable when xi r_c >= 8) evaluates the last interval's
// polynomial outside its interval; there erfc(x) < 1.2e-29, so the pair's contribution is
// below the double resolution of any sum it enters, and E * p stays finite.
// xw = x / W (interval units): k = trunc(xw), t = 2 (xw - k) - 1
__device__ __forceinline__ double erfc_from_E(double xw, double E, const double2* __restrict__ tab) {
  const int k = min((int)xw, HS_ERFCX_NINT - 1);
  const double t = fma(2.0, xw, -(double)(2 * k + 1));
  const double2 top = tab[(HS_ERFCX_NPAIR - 1) * HS_ERFCX_NINT + k];
  double p = (HS_ERFCX_DEG & 1) ? fma(top.y, t, top.x) : top.x;
#pragma unroll
  for (int j = HS_ERFCX_NPAIR - 2; j >= 0; --j) {
    const double2 c = tab[j * HS_ERFCX_NINT + k];
    p = fma(p, t, c.y);
    p = fma(p, t, c.x);
  }
  return E * p;
}

// erfc(x) = exp(-x^2) erfcx(x) without tables (default; HS_ERFC_TABLE=1 at build time selects
// the piecewise table above): erfcx as one degree-18 polynomial in s = S0 + S1/(x + 3) on
// [0, 8] (tools/gen_erfcx_poly.py, max rel. error 6.9e-15; the reference's own Hermite table
// is ~2e-13, ewald_real.py:33-58), coefficients as constant-bank DFMA operands.  Trades the
// table's six lane-divergent 16-byte shared-memory loads per pair (the pair kernel's
// shared-memory pipe is its co-bottleneck) for ~12 more DFMAs.
#include "erfcx_poly.inc"
// Newton steps after the hardware rsqrt / rcp approximations (~2^-23): 1 step leaves ~2^-46
// relative error (erfc ~1e-14, far below the 2e-13 of the reference's own erfc table), 2 steps
// round-off level
#ifndef PC_NEWTON
#define PC_NEWTON 3
#endif
// PC_NEWTON = 3 (default): ONE third-order step, y (1 + e + e^2) for 1/v and y (1 + e/2 + 3e^2/8)
// for 1/sqrt(v) (e the residual of the ~2^-22 hardware value): error ~e^3, i.e. round-off
// level like two Newton steps, in 3 / 5 instead of 4 / 8 FP64 operations
#if PC_NEWTON == 3
__device__ __forceinline__ double rcp_pos(double v) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
  const double e = fma(-v, y, 1.0);
  return fma(y, fma(e, e, e), y);
}
#else
__device__ __forceinline__ double rcp_pos(double v) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(v));
#pragma unroll
  for (int it = 0; it < PC_NEWTON; ++it) y = fma(y, fma(-v, y, 1.0), y);
  return y;
}
#endif
#ifndef PC_DRAIN2
#define PC_DRAIN2 1   // queue drains by two-pair rounds where lanes have >= 2 entries
#endif
// (Estrin's scheme for the erfcx / exp polynomials -- dependency depth ~log2(deg) instead of
// deg -- measured 83 vs 38 ms for the HL pair kernel: Horner with constant-bank operands stays.)
// x > HS_EP_XMAX (xi r_c > 8 only) is not clamped: s stays in (1, HS_EP_S0], where the polynomial
// is bounded by 0.07, so E p < 1e-29 -- below the resolution of any sum it enters.
// EP6: the degree-15 polynomial on [0, 6] (3 DFMAs fewer; max rel. error 5.8e-15), used when
// xi r_c <= 6, i.e. every accepted pair has x <= 6
template <bool EP6 = false>
__device__ __forceinline__ double erfc_poly_from_E(double x, double E) {
  if (EP6) {
    const double s = fma(HS_EP6_S1, rcp_pos(x + HS_EP6_K), HS_EP6_S0);
    double p = c_erfcx_poly6[0];
#pragma unroll
    for (int j = 1; j <= HS_EP6_DEG; ++j) p = fma(p, s, c_erfcx_poly6[j]);
    return E * p;
  }
  const double s = fma(HS_EP_S1, rcp_pos(x + HS_EP_K), HS_EP_S0);
  double p = c_erfcx_poly[0];
#pragma unroll
  for (int j = 1; j <= HS_EP_DEG; ++j) p = fma(p, s, c_erfcx_poly[j]);
  return E * p;
}
#ifndef HS_ERFC_TABLE
#define HS_ERFC_TABLE 0
#endif

// exp(x) for x <= 0, branch-free (no special-case slow path, so two pair evaluations
// interleave freely): x = n ln2 + r, |r| <= ln2/2, degree-11 near-minimax polynomial
// (Chebyshev interpolation on [-ln2/2, ln2/2], max rel. error 3.8e-16 incl. Horner rounding;
// two DFMAs fewer than the degree-13 Taylor series), 2^n assembled in the exponent field;
// below -708 (2^n subnormal) the result flushes to 0.  Coefficients live in constant memory
// so the DFMAs take them as c[] operands.
__constant__ double c_exp_poly[12] = {
    2.710963222255011e-08,  2.752918835347435e-07,  2.755038996576078e-06, 2.480178099872014e-05,
    0.00019841278462872085, 0.001388888866033683,   0.008333333328692896,  0.04166666666766274,
    0.1666666666667613,     0.4999999999999831,     0.9999999999999999,    1.0000000000000002};
__device__ __forceinline__ double exp_nonpos(double x) {
  const double kShift = 6755399441055744.0;  // 1.5 * 2^52
  const double t = fma(x, 1.4426950408889634, kShift);
  const double n = t - kShift;
  const int ni = __double2loint(t);
  // one ln 2 constant: error <= |n| 5.5e-17, below 3e-15 wherever exp(x) > 1e-16 (one DFMA fewer
  // than a hi / lo split)
  const double r = fma(n, -0.6931471805599453094, x);
  double p = c_exp_poly[0];
#pragma unroll
  for (int j = 1; j < 12; ++j) p = fma(p, r, c_exp_poly[j]);
  return p * __hiloint2double(max(ni + 1023, 0) << 20, 0);
}

// 1/sqrt(r2) for normal r2 > 0, branch-free: hardware approximation + refinement
__device__ __forceinline__ double rsqrt_pos(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
#if PC_NEWTON == 3
  const double h = r2 * y;
  const double e = fma(-h, y, 1.0);
  return fma(y * e, fma(e, 0.375, 0.5), y);
#else
#pragma unroll
  for (int it = 0; it < PC_NEWTON; ++it) {  // ~2^-23 -> 2^-46 -> rounding level
    const double h = r2 * y;
    const double e = fma(-h, y, 1.0);
    y = fma(0.5 * y, e, y);
  }
  return y;
#endif
}

constexpr int PT_MAXRUN = 25;  // 5 x 5 (x, y) cell columns

struct PairConst {
  double xi, xi2, c2xs;  // xi, xi^2, 2 xi / sqrt(pi)
  double xiw;            // xi / HS_ERFCX_W (erfc argument in table-interval units)
};

// Radial coefficients of one pair (the transcendental part; branch-free when SCREENED).
struct PairCoef {
  double ri, ri2, c0, c1, e;
};
template <bool SCREENED, bool EP6 = false>
__device__ __forceinline__ PairCoef pair_coef(const PairConst& pc, double r2, const double2* __restrict__ etab) {
  PairCoef q;
  double C = 1.0;
  q.e = 0.0;
  if (SCREENED) {
    q.ri = rsqrt_pos(r2);
    const double rn = r2 * q.ri;
    const double E = exp_nonpos(-pc.xi2 * r2);
    C = HS_ERFC_TABLE ? erfc_from_E(pc.xiw * rn, E, etab) : erfc_poly_from_E<EP6>(pc.xi * rn, E);
    q.e = pc.c2xs * E;
  } else {
    q.ri = rsqrt(r2);
  }
  q.ri2 = q.ri * q.ri;
  q.c0 = C * q.ri;
  q.c1 = (q.c0 + q.e) * q.ri2;
  return q;
}

// Accumulate one pair.  d = x - y (target minus source), r2 = |d|^2 (> 0).
// k[0..2]: kernel part (raw), c[0..2]: wall correction (raw, 4 pi G convention).
template <int KIND>
__device__ __forceinline__ void apply_pair(const PairConst& pc, const PairCoef& q, double d0, double d1, double d2,
                                           double r2, double x2, const double4& S, const double4& A,
                                           const double4& B, bool image, double* k, double* c) {
  const double ri = q.ri, ri2 = q.ri2, c0 = q.c0, c1 = q.c1, e = q.e;
  if (KIND == HS_STOKESLET) {
    // a = 2(xi E/sqrt(pi) + C/(2r)) = C/r + e ; a - b = C/r - e   (ewald_real.py:303-309)
    const double a = c0 + e, amb = c0 - e;
    const double fd = (d0 * A.x + d1 * A.y + d2 * A.z) * ri2;
    k[0] += amb * A.x + a * fd * d0;
    k[1] += amb * A.y + a * fd * d1;
    k[2] += amb * A.z + a * fd * d2;
    if (image) {
      // image row holds -f^I: s = -f3 = -A.z ; v = -y3 f^I = -zI * A   (kernels_direct.py:112-116)
      const double s = -A.z;
      const double v0 = -S.z * A.x, v1 = -S.z * A.y, v2 = -S.z * A.z;
      const double c2 = (3.0 * c1 + 2.0 * pc.xi2 * e) * ri2;
      const double dv = d0 * v0 + d1 * v1 + d2 * v2;
      const double phi = s * c0 - c1 * dv;
      const double wd = c2 * dv - c1 * s;
      c[0] += -x2 * (wd * d0 - c1 * v0);
      c[1] += -x2 * (wd * d1 - c1 * v1);
      c[2] += -x2 * (wd * d2 - c1 * v2) + phi;
    }
  } else if (KIND == HS_STRESSLET) {
    const double sign = image ? -1.0 : 1.0;
    const double dg = d0 * A.x + d1 * A.y + d2 * A.z;
    const double dq = d0 * B.x + d1 * B.y + d2 * B.z;
    const double gq = A.x * B.x + A.y * B.y + A.z * B.z;
    // c1 = -(2/r)(3C/r + (2xi/sqrt(pi))(3 + 2 xi^2 r^2) E), c2 = 4 xi^3 E/sqrt(pi)  (ewald_real.py:315-321)
    const double k1 = -2.0 * ri * (3.0 * c0 + (3.0 + 2.0 * pc.xi2 * r2) * e);
    const double k2 = 2.0 * pc.xi2 * e;
    const double w1 = sign * k1 * dg * dq * ri2 * ri;
    const double w2 = sign * k2;
    k[0] += w1 * d0 + w2 * (gq * d0 + dq * A.x + dg * B.x);
    k[1] += w1 * d1 + w2 * (gq * d1 + dq * A.y + dg * B.y);
    k[2] += w1 * d2 + w2 * (gq * d2 + dq * A.z + dg * B.z);
    if (image) {
      // v = (0,0,2 gI.qI), M = -y3 (gI qI^T + qI gI^T) = zI (...)   (kernels_direct.py:117-122)
      const double zI = S.z;
      const double v2 = 2.0 * gq;
      const double trM = 2.0 * zI * gq;
      const double Md0 = zI * (A.x * dq + B.x * dg);
      const double Md1 = zI * (A.y * dq + B.y * dg);
      const double Md2 = zI * (A.z * dq + B.z * dg);
      const double qq = 2.0 * zI * dg * dq;
      const double c2 = (3.0 * c1 + 2.0 * pc.xi2 * e) * ri2;
      const double c3 = -(5.0 * c2 + 4.0 * pc.xi2 * pc.xi2 * e) * ri2;
      const double dv = d2 * v2;
      const double phi = -c1 * (dv + trM) + c2 * qq;
      const double wd = c2 * dv + c2 * trM + c3 * qq;
      c[0] += -x2 * (wd * d0 + 2.0 * c2 * Md0);
      c[1] += -x2 * (wd * d1 + 2.0 * c2 * Md1);
      c[2] += -x2 * (wd * d2 + 2.0 * c2 * Md2 - c1 * v2) + phi;
    }
  } else {
    // rotlet: A = sign * (g x q); u += 2 (C/r^3 + e/r^2) (omega x d)   (ewald_real.py:324-331)
    const double w = 2.0 * c1;
    k[0] += w * (A.y * d2 - A.z * d1);
    k[1] += w * (A.z * d0 - A.x * d2);
    k[2] += w * (A.x * d1 - A.y * d0);
    if (image) {
      // v = 4 (q3 gI - g3 qI) precomputed into B.x, B.y (v3 = 0)   (kernels_direct.py:123-127)
      const double c2 = (3.0 * c1 + 2.0 * pc.xi2 * e) * ri2;
      const double dv = d0 * B.x + d1 * B.y;
      const double phi = -c1 * dv;
      const double wd = c2 * dv;
      c[0] += -x2 * (wd * d0 - c1 * B.x);
      c[1] += -x2 * (wd * d1 - c1 * B.y);
      c[2] += -x2 * (wd * d2) + phi;
    }
  }
}

template <int KIND, bool SCREENED>
__device__ __forceinline__ void eval_pair(const PairConst& pc, double d0, double d1, double d2, double r2,
                                          double x2, const double4& S, const double4& A, const double4& B,
                                          bool image, double* k, double* c, const double2* __restrict__ etab) {
  apply_pair<KIND>(pc, pair_coef<SCREENED>(pc, r2, etab), d0, d1, d2, r2, x2, S, A, B, image, k, c);
}

// FP32 prefilter distance^2 with a fixed operation order
__device__ __forceinline__ float dist2f(float tx, float ty, float tz, const float4& F) {
  const float dx = tx - F.x, dy = ty - F.y, dz = tz - F.z;
  return __fmaf_rn(dz, dz, __fmaf_rn(dy, dy, __fmul_rn(dx, dx)));
}

__device__ __forceinline__ float4 lds_f4(unsigned addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
  return v;
}

__device__ __forceinline__ void sts_u16(unsigned addr, int v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"((unsigned short)v) : "memory");
}

// index of the highest set bit (x != 0)
__device__ __forceinline__ int bfind_u32(unsigned x) {
  int r;
  asm("bfind.u32 %0, %1;" : "=r"(r) : "r"(x));
  return r;
}

__device__ __forceinline__ double exact_r2(double d0, double d1, double d2) {
  // numba: r2 = d0 * d0 + d1 * d1 + d2 * d2, each op rounded, left to right
  return __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
}

// ---------------------------------------------------------------------------
// Queue design (used by launch_pair): one thread per target.  A CTA owns up to
// PC_TG consecutive cell-sorted targets of ONE (ix,iy) cell column, so all its
// targets share a compact candidate region: 25 z-runs over
// [cz_first-2, cz_last+2].  Candidates are staged in shared memory and scanned
// in lock-step with broadcast reads (one smem wavefront per candidate per
// warp); each lane pushes the candidates IT accepts (exact reference test)
// into a lane-private queue, and the warp evaluates queued pairs in rounds
// whenever >= 3/4 of its lanes have work, so the erfc/exp-heavy evaluation
// runs with nearly full SIMT utilisation while every thread accumulates only
// its own target (no cross-lane reductions, no atomics, deterministic order).
#ifndef PC_WARPS_DEF
#define PC_WARPS_DEF 4
#endif
constexpr int PC_WARPS = PC_WARPS_DEF;
constexpr int PC_TG = PC_WARPS * 32;  // targets per work item
// plan.cu sizes the work-item buffer (nt / 128 + columns + 2) for at least 128 targets per item
static_assert(PC_TG >= 128, "pair work items must hold >= 128 targets (PC_WARPS_DEF >= 4)");
// candidates per chunk (a multiple of PC_TG, a power of two): the stokeslet stages 256 per
// barrier pair (2 per thread) in a 2-chunk ring; the larger stresslet / rotlet records keep
// 128-candidate chunks in a 3-chunk ring (4 CTAs per SM either way)
#ifndef PC_H_STOKESLET
#define PC_H_STOKESLET 256
#endif
template <int KIND>
constexpr int pc_h() { return KIND == HS_STOKESLET ? PC_H_STOKESLET : (PC_TG > 128 ? PC_TG : 128); }
#ifndef PC_NH_STOKESLET
#define PC_NH_STOKESLET 2
#endif
#ifndef PC_NH_OTHER
#define PC_NH_OTHER 3
#endif
// chunks held in the staging ring (stokeslet: 3, so a lane's FIFO entries of the chunk being
// restaged -- which force partial-round drains -- are rarer; the stresslet / rotlet records
// leave room for 2 within 48 KB of static shared memory)
template <int KIND>
constexpr int pc_nh() { return KIND == HS_STOKESLET ? PC_NH_STOKESLET : (KIND == HS_MIXED ? 2 : PC_NH_OTHER); }
// candidate record bytes in shared memory (dynamic): xy, z a.x, a.y a.z, FP32 view, (+ b)
// (mixed: a = f, then g.x g.y | g.z q.x | q.y q.z)
template <int KIND, bool HALF>
constexpr int pc_rec_bytes() {
  return KIND == HS_MIXED ? 112
                          : 64 + ((KIND == HS_STRESSLET) || (KIND == HS_ROTLET && HALF) ? 16 : 0) +
                                (KIND == HS_STRESSLET ? 8 : 0);
}

#ifndef PC_Q_DEF
#define PC_Q_DEF 64
#endif
#ifndef PC_ROUND_SLACK
#define PC_ROUND_SLACK 0
#endif
#ifndef PC_ODD_SINGLE
#define PC_ODD_SINGLE 0
#endif
constexpr int PC_Q = PC_Q_DEF;        // per-lane queue capacity (power of two)
static_assert(PC_Q >= 64 && (PC_Q & (PC_Q - 1)) == 0,
              "a group of 32 candidates must fit behind a backlog: the overflow guard drains to PC_Q - 32");
#ifndef PC_MINB
#define PC_MINB 4                     // resident CTAs per SM (register budget 128)
#endif
// resident CTAs per SM: the mixed evaluation (stokeslet + stresslet per pair, sharing the
// transcendentals) needs more registers than 128
template <int KIND>
constexpr int pc_minb() { return KIND == HS_MIXED ? 3 : PC_MINB; }

// splitmix64 finaliser (neighbour-set hash of the audit launch; oracle/hs_oracle.c)
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  unsigned long long z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// AUDIT: the same kernel also records every target's accepted neighbour set (count, image
// count, id hash) -- a separate instantiation so the production launch carries no extra work.
template <int KIND, bool HALF, bool AUDIT, bool EP6>
__global__ void __launch_bounds__(PC_TG, pc_minb<KIND>()) k_pair_q(const PairArgs a) {
  // Candidate rows as 16-byte columns: the evaluation reads them at lane-random rows, and a
  // 16-byte array spreads those reads over 8 bank groups (a 32-byte row only over 4).
  constexpr int PC_H = pc_h<KIND>(), PC_PER = PC_H / PC_TG;
  constexpr int PC_HSHIFT = PC_H == 128 ? 7 : (PC_H == 256 ? 8 : 9);
  constexpr int PC_K = pc_nh<KIND>() * PC_H;  // staged candidates (dynamic shared memory)
  constexpr bool kNeedB = (KIND == HS_STRESSLET) || (KIND == HS_ROTLET && HALF);
  extern __shared__ __align__(16) unsigned char pc_dyn[];
  double2* sXY = reinterpret_cast<double2*>(pc_dyn);  // x, y
  double2* sZA = sXY + PC_K;                          // z (sign bit = image in the half space), a.x
  double2* sAA = sZA + PC_K;                          // a.y, a.z
  float4* sF = reinterpret_cast<float4*>(sAA + PC_K);  // position relative to the item's first target (FP32)
  double2* sB0 = reinterpret_cast<double2*>(sF + PC_K);  // b.x, b.y (kNeedB)
  double* sB1 = reinterpret_cast<double*>(sB0 + (kNeedB ? PC_K : 0));  // b.z (stresslet)
  constexpr bool kMixed = KIND == HS_MIXED;
  double2* sG0 = reinterpret_cast<double2*>(sF + PC_K);  // mixed: g.x g.y
  double2* sG1 = sG0 + PC_K;                             // mixed: g.z q.x
  double2* sG2 = sG1 + PC_K;                             // mixed: q.y q.z
  __shared__ unsigned short sq[PC_WARPS][PC_Q][32];
  __shared__ int run_beg[PT_MAXRUN];
  __shared__ int run_pre[PT_MAXRUN + 1];
  __shared__ int s_nrun;
  __shared__ double2 s_erfcx[HS_ERFC_TABLE ? HS_ERFCX_NPAIR * HS_ERFCX_NINT : 1];
  if (HS_ERFC_TABLE)
    for (int i = threadIdx.x; i < HS_ERFCX_NPAIR * HS_ERFCX_NINT; i += blockDim.x) s_erfcx[i] = g_erfcx_coef[i];

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nx = a.dims[0], ny = a.dims[1], nz = a.dims[2];
  PairConst pc;
  pc.xi = a.xi;
  pc.xi2 = a.xi * a.xi;
  pc.c2xs = 2.0 * a.xi / kSqrtPi;
  pc.xiw = a.xi * (1.0 / HS_ERFCX_W);
  const double norm_k = (KIND == HS_ROTLET) ? 1.0 / (4.0 * kPi) : 1.0 / (8.0 * kPi);
  const double norm_c = 1.0 / (4.0 * kPi);
  unsigned short(*q)[32] = sq[warp];

  const int n_items = *a.n_items_d;
  // work items are taken from a global counter (a.work), so a CTA that drew cheap items (cells
  // near the wall or the box faces) simply takes more: no tail of idle SMs behind the slowest
  // static share.  Which CTA evaluates an item does not affect any result.
  __shared__ int s_item;
  for (int it0 = blockIdx.x;; it0 += gridDim.x) {
    int it = it0;
    if (a.work) {
      __syncthreads();
      if (threadIdx.x == 0) s_item = atomicAdd(a.work, 1);
      __syncthreads();
      it = s_item;
    }
    if (it >= n_items) break;
    const int2 item = a.items[it];
    const int col = item.x, t0 = item.y;
    const int t1 = min(t0 + PC_TG, a.t_start[(col + 1) * nz * a.t_sub]);
    const int ix = col / ny, iy = col % ny;
    __syncthreads();
    if (threadIdx.x == 0) {
      const int cz0 = a.cell_z(a.TP[t0].z), cz1 = a.cell_z(a.TP[t1 - 1].z);
      int nr = 0, tot = 0;
      const int zlo = max(cz0 - 2, 0), zhi = min(cz1 + 2, nz - 1);
      for (int jx = max(ix - 2, 0); jx <= min(ix + 2, nx - 1); ++jx)
        for (int jy = max(iy - 2, 0); jy <= min(iy + 2, ny - 1); ++jy) {
          const int f = (jx * ny + jy) * nz;
          const int b = a.start[f + zlo], e = a.start[f + zhi + 1];
          if (e > b) {
            run_beg[nr] = b;
            run_pre[nr] = tot;
            tot += e - b;
            ++nr;
          }
        }
      run_pre[nr] = tot;
      s_nrun = nr;
    }
    __syncthreads();
    const int nrun = s_nrun;
    const int ncand = run_pre[nrun];
    const int t = t0 + threadIdx.x;
    const bool tvalid = t < t1;
    const double4 T = a.TP[tvalid ? t : t0];
    const long long tcol = tvalid ? (long long)T.w : -2;  // -2 never matches a source id
    const int tcol_i = (int)tcol;
    // the target's own z cell: the reference scans cz - 2 .. cz + 2 (ewald_real.py:285-287);
    // the item's candidate range covers all its targets' ranges, so shell candidates are
    // also checked against this target's reach (sure-accepts lie well inside it)
    const int tcz = a.cell_z(T.z);
    unsigned long long a_hash = 0;
    // FP32 view relative to the item's first target, and this warp's target bounding box
    const double4 R0 = a.TP[t0];
    // (a lane without a target tests a point 1e30 away: it never accepts nor meets the shell)
    const float tfx = tvalid ? (float)(T.x - R0.x) : 1.0e30f, tfy = tvalid ? (float)(T.y - R0.y) : 1.0e30f,
                tfz = tvalid ? (float)(T.z - R0.z) : 1.0e30f;
    float bmin[3] = {tfx, tfy, tfz}, bmax[3] = {tfx, tfy, tfz};
    if (!tvalid) {
      bmin[0] = bmin[1] = bmin[2] = 3.0e38f;
      bmax[0] = bmax[1] = bmax[2] = -3.0e38f;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        bmin[k] = fminf(bmin[k], __shfl_xor_sync(0xffffffffu, bmin[k], o));
        bmax[k] = fmaxf(bmax[k], __shfl_xor_sync(0xffffffffu, bmax[k], o));
      }
    }
    double acc[6] = {0, 0, 0, 0, 0, 0};
    bool singular = false;
    unsigned long long n_acc = 0, n_img = 0;

    // candidate row j as (S, A, B); S.w unused; image <=> sign bit of z (k_pair_records).
    // Mixed: A = f, B = g, and the q of the row is read by load_q
    auto load_cand = [&](int jj, double4& S, double4& A, double4& B, bool& img) {
      const double2 xy = sXY[jj], za = sZA[jj], aa = sAA[jj];
      S = make_double4(xy.x, xy.y, za.x, 0.0);
      A = make_double4(za.y, aa.x, aa.y, 0.0);
      img = HALF && __double2hiint(za.x) < 0;
      B = make_double4(0, 0, 0, 0);
      if (kMixed) {
        const double2 g0 = sG0[jj], g1 = sG1[jj];
        B = make_double4(g0.x, g0.y, g1.x, g1.y);  // .w carries q.x
      } else if (KIND == HS_STRESSLET) {
        const double2 b = sB0[jj];
        B = make_double4(b.x, b.y, sB1[jj], 0.0);
      } else if (kNeedB && img) {  // rotlet: the wall channel exists for images only
        const double2 b = sB0[jj];
        B = make_double4(b.x, b.y, 0.0, 0.0);
      }
    };
    // one pair's contribution(s) for the kernel kind (mixed: stokeslet + stresslet sharing the
    // radial coefficients, i.e. one rsqrt / exp / erfc for both)
    auto apply_kind = [&](const PairCoef& qc, int jj, double d0, double d1, double d2, double rr, const double4& S,
                          const double4& A, const double4& B, bool img) {
      if constexpr (kMixed) {
        const double2 q12 = sG2[jj];
        const double4 Q = make_double4(B.w, q12.x, q12.y, 0.0);
        apply_pair<HS_STOKESLET>(pc, qc, d0, d1, d2, rr, T.z, S, A, B, img, &acc[0], &acc[3]);
        apply_pair<HS_STRESSLET>(pc, qc, d0, d1, d2, rr, T.z, S, B, Q, img, &acc[0], &acc[3]);
      } else {
        apply_pair<KIND>(pc, qc, d0, d1, d2, rr, T.z, S, A, B, img, &acc[0], &acc[3]);
      }
    };
    auto eval_one = [&](int jj) {
      double4 S, A, B;
      bool img;
      load_cand(jj, S, A, B, img);
      const double e0 = T.x - S.x, e1 = T.y - S.y, e2 = T.z - S.z;
      const double rr = fma(e0, e0, fma(e1, e1, e2 * e2));  // (neighbour test done exactly in the scan)
      if (img) ++n_img;
      if (AUDIT) a_hash += splitmix64((unsigned long long)__float_as_int(sF[jj].w));
      apply_kind(pair_coef<true, EP6>(pc, rr, s_erfcx), jj, e0, e1, e2, rr, S, A, B, img);
    };

    // Two-half ring of staged candidates + per-lane FIFO queues: entries of chunk c may be
    // evaluated while chunk c+1 is scanned, so queues never have to be drained at every
    // chunk boundary (only the leftovers of chunk c-2 before its half is restaged).
    int head = 0, tail = 0;
    // stride coprime with ncand (a few primes larger than any realistic candidate count)
    int pstride = 1;
    {
      const int primes[4] = {1000003, 999983, 1000033, 1000037};
      for (int k = 0; k < 4; ++k)
        if (ncand % primes[k] != 0) {
          pstride = primes[k] % max(ncand, 1);
          if (pstride == 0) pstride = 1;
          break;
        }
    }
    // stride permutation, incrementally: thread tid stages v = ((c0 + tid) * pstride) mod ncand,
    // and c0 advances by PC_H per chunk (PC_PER candidates per thread per chunk)
    static_assert(PC_H % PC_TG == 0 && (1 << PC_HSHIFT) == PC_H, "chunk = whole CTA rounds, power of two");
    const int vstep = (int)(((long long)PC_H * pstride) % max(ncand, 1));
    int vcur[PC_PER];
#pragma unroll
    for (int k = 0; k < PC_PER; ++k)
      vcur[k] = (int)(((long long)(threadIdx.x + k * PC_TG) * pstride) % max(ncand, 1));
    auto pop_eval = [&]() {
      const int jj = q[head & (PC_Q - 1)][lane];
      HS_CHECK(jj < PC_K && head < tail);
      ++head;
      ++n_acc;
      eval_one(jj);
    };
    // two queued pairs in straight-line code: their exp / erfc / rsqrt chains are
    // independent and interleave (the evaluation is latency-, not issue-bound)
    auto eval2 = [&](int j1, int j2) {
      HS_CHECK(j1 < PC_K && j2 < PC_K && head + 2 <= tail);
      head += 2;
      n_acc += 2;
      double4 S1, A1, B1, S2, A2, B2;
      bool i1, i2;
      load_cand(j1, S1, A1, B1, i1);
      load_cand(j2, S2, A2, B2, i2);
      const double f0 = T.x - S1.x, f1 = T.y - S1.y, f2 = T.z - S1.z;
      const double g0 = T.x - S2.x, g1 = T.y - S2.y, g2 = T.z - S2.z;
      const double r1 = fma(f0, f0, fma(f1, f1, f2 * f2)), r2 = fma(g0, g0, fma(g1, g1, g2 * g2));
      const PairCoef q1 = pair_coef<true, EP6>(pc, r1, s_erfcx);
      const PairCoef q2 = pair_coef<true, EP6>(pc, r2, s_erfcx);
      n_img += (unsigned)i1 + (unsigned)i2;
      if (AUDIT)
        a_hash += splitmix64((unsigned long long)__float_as_int(sF[j1].w)) +
                  splitmix64((unsigned long long)__float_as_int(sF[j2].w));
      apply_kind(q1, j1, f0, f1, f2, r1, S1, A1, B1, i1);
      apply_kind(q2, j2, g0, g1, g2, r2, S2, A2, B2, i2);
    };
    auto pop_eval2 = [&]() {
      const int j1 = q[head & (PC_Q - 1)][lane];
      const int j2 = q[(head + 1) & (PC_Q - 1)][lane];
      eval2(j1, j2);
    };
    for (int c = 0, c0 = 0; c0 < ncand; ++c, c0 += PC_H) {
      const int h = c % pc_nh<KIND>(), hb = h * PC_H;
      // drain the (oldest) entries that still reference half h
      while (__any_sync(0xffffffffu, tail > head && (q[head & (PC_Q - 1)][lane] >> PC_HSHIFT) == h)) {
        if (tail > head && (q[head & (PC_Q - 1)][lane] >> PC_HSHIFT) == h) pop_eval();
      }
      __syncthreads();
#pragma unroll
      for (int kk = 0; kk < PC_PER; ++kk) {
        const int j = threadIdx.x + kk * PC_TG;
        const int v0 = c0 + j;
        const int v = vcur[kk];
        vcur[kk] += vstep;
        if (vcur[kk] >= ncand) vcur[kk] -= ncand;
        if (v0 < ncand) {
          // stride permutation of the candidate list: every chunk samples the whole
          // neighbourhood, so each lane's acceptance rate per chunk is about its average
          // and the full-round evaluation below keeps all lanes busy.  Run of v: binary search
          // for the last run_pre[r] <= v (run_pre[0] = 0)
          int r = 0, rhi = nrun - 1;
          while (r < rhi) {
            const int mid = (r + rhi + 1) >> 1;
            if (run_pre[mid] <= v) r = mid;
            else rhi = mid - 1;
          }
          const int row = run_beg[r] + (v - run_pre[r]);
          HS_CHECK(r >= 0 && r < nrun && v >= run_pre[r] && v < run_pre[r + 1] && hb + j < PC_K &&
                   row < a.start[nx * ny * nz]);
          const double4 S = a.P[row];
          const double4 A = a.A[row];
          sXY[hb + j] = make_double2(S.x, S.y);
          sZA[hb + j] = make_double2(S.z, A.x);
          sAA[hb + j] = make_double2(A.y, A.z);
          // .w carries the combined source index as int bits (no per-pair FP64->int conversions)
          sF[hb + j] = make_float4((float)(S.x - R0.x), (float)(S.y - R0.y), (float)(S.z - R0.z),
                                   __int_as_float((int)S.w));
          if (kMixed) {
            const double4 G = a.B[row], Q = a.C[row];
            sG0[hb + j] = make_double2(G.x, G.y);
            sG1[hb + j] = make_double2(G.z, Q.x);
            sG2[hb + j] = make_double2(Q.y, Q.z);
          } else if (kNeedB) {
            const double4 B = a.B[row];
            sB0[hb + j] = make_double2(B.x, B.y);
            if (KIND == HS_STRESSLET) sB1[hb + j] = B.z;
          }
        }
      }
      __syncthreads();
      const int nc = min(PC_H, ncand - c0);
      for (int j0 = 0; j0 < nc; j0 += 32) {
        // warp-level culling: candidates farther than rc (+margin) from the warp's target box
        unsigned near;
        {
          const int j = j0 + lane;
          bool keep = false;
          if (j < nc) {
            const float4 F = sF[hb + j];
            const float dx = fmaxf(fmaxf(bmin[0] - F.x, F.x - bmax[0]), 0.0f);
            const float dy = fmaxf(fmaxf(bmin[1] - F.y, F.y - bmax[1]), 0.0f);
            const float dz = fmaxf(fmaxf(bmin[2] - F.z, F.z - bmax[2]), 0.0f);
            keep = dx * dx + dy * dy + dz * dz <= a.rc2_hi;
          }
          near = __ballot_sync(0xffffffffu, keep);
        }
        // FP32 distance inside r_c by a margin far above its rounding error (sure accept: the
        // exact reference test accepts too) -> pushed at once; the shell around r_c and FP32
        // distance 0 (the target itself, coincident sources) are collected as bits and decided
        // by the exact test after the group -- bit-identical neighbour sets.  The slot at `tail`
        // is free (tail - head < PC_Q), so every tested candidate is written there and `tail`
        // advances only on accept.  Two near candidates per iteration, highest bits first
        // (bfind gives the index; the bit doubles as the shell-mask bit).
        const unsigned sFg_s = (unsigned)__cvta_generic_to_shared(sF + hb + j0);
        const unsigned q_s = (unsigned)__cvta_generic_to_shared(&q[0][lane]);  // this lane's slot 0
        const int qb = hb + j0;
        unsigned msh = 0;
        while (near) {  // warp-uniform (lanes without a target test far-away coordinates)
          const int ia = bfind_u32(near);
          const unsigned ba = 1u << ia;
          const unsigned rest = near ^ ba;
          const bool two = rest != 0;
          const int ib = two ? bfind_u32(rest) : ia;
          const unsigned bb = two ? 1u << ib : 0u;
          near = rest ^ bb;
          const float4 Fa = lds_f4(sFg_s + (ia << 4)), Fb = lds_f4(sFg_s + (ib << 4));  // broadcast
          const float ra = dist2f(tfx, tfy, tfz, Fa), rb = dist2f(tfx, tfy, tfz, Fb);
          const bool oka = ra > 0.0f && ra <= a.rc2_lo;
          const bool okb = two && rb > 0.0f && rb <= a.rc2_lo;
          msh |= (!oka && ra <= a.rc2_hi ? ba : 0u) | (!okb && rb <= a.rc2_hi ? bb : 0u);
          sts_u16(q_s + (((unsigned)tail & (PC_Q - 1)) << 6), qb + ia);
          tail += oka ? 1 : 0;
          sts_u16(q_s + (((unsigned)tail & (PC_Q - 1)) << 6), qb + ib);
          tail += okb ? 1 : 0;
        }
        if (__any_sync(0xffffffffu, msh != 0)) {
          while (msh) {
            const int ib = bfind_u32(msh);
            msh ^= 1u << ib;
            const int j = qb + ib;
            const double2 xy = sXY[j];
            const double sz = sZA[j].x;
            const double d0 = __dsub_rn(T.x, xy.x), d1 = __dsub_rn(T.y, xy.y), d2 = __dsub_rn(T.z, sz);
            const double r2 = exact_r2(d0, d1, d2);
            const bool other = __float_as_int(sF[j].w) != tcol_i;
            singular |= other && r2 == 0.0;
            const bool ok = other && r2 <= a.rc2 && r2 != 0.0 && abs(a.cell_z(sz) - tcz) <= 2;
            q[tail & (PC_Q - 1)][lane] = (unsigned short)j;
            tail += ok ? 1 : 0;
            // (a lane's backlog after a group stays < PC_Q: <= PC_Q - 32 before it, <= 32 pushes)
          }
        }
        // full rounds while every valid lane has work; partial rounds only against overflow
        unsigned mn = __reduce_min_sync(0xffffffffu, (unsigned)(tvalid ? tail - head : 0x7fffffff));
        if (mn == 0x7fffffffu) mn = 0;
        if (tvalid) {
          unsigned r = 0;
          for (; r + 1 < mn; r += 2) pop_eval2();
          // an odd leftover stays queued for the next two-pair round (PC_ODD_SINGLE=1: evaluate it now)
          if (PC_ODD_SINGLE && r < mn) pop_eval();
        }
        if (PC_ROUND_SLACK > 0) {
          // more two-pair rounds while all but PC_ROUND_SLACK of the valid lanes have work (the idle
          // lanes' slots are cheaper than the partial single rounds a growing backlog forces later)
          const int nv = __popc(__ballot_sync(0xffffffffu, tvalid));
          while (__popc(__ballot_sync(0xffffffffu, tvalid && tail - head >= 2)) >= nv - PC_ROUND_SLACK &&
                 nv > PC_ROUND_SLACK) {
            if (tvalid && tail - head >= 2) pop_eval2();
          }
        }
        HS_CHECK(tail - head <= PC_Q);
        // overflow guard: two-pair rounds for the lanes with a backlog (the fullest lane has
        // > PC_Q - 32 >= 2 entries, so every round makes progress; single entries wait)
        while ((int)__reduce_max_sync(0xffffffffu, (unsigned)(tail - head)) > PC_Q - 32) {
          if (PC_DRAIN2) {
            if (tail - head >= 2) pop_eval2();
          } else if (tail > head) {
            pop_eval();
          }
        }
      }
    }
    if (PC_DRAIN2) {
      while (__any_sync(0xffffffffu, tail - head >= 2)) {
        if (tail - head >= 2) pop_eval2();
      }
    }
    while (__any_sync(0xffffffffu, tail > head)) {
      if (!PC_DRAIN2 && tail - head >= 2)
        pop_eval2();
      else if (tail > head)
        pop_eval();
    }
    if (singular) atomicOr(a.flags, FLAG_SINGULAR);
    if (a.counts) {
      const unsigned long long w_acc = __reduce_add_sync(0xffffffffu, (unsigned)n_acc);
      const unsigned long long w_img = __reduce_add_sync(0xffffffffu, (unsigned)n_img);
      if (lane == 0) {
        atomicAdd(&a.counts[0], w_acc);
        atomicAdd(&a.counts[1], w_img);
      }
    }
    if (tvalid) {
      const int o = a.torig[t];
      if (AUDIT) {
        a.audit[3 * (size_t)o] = n_acc;
        a.audit[3 * (size_t)o + 1] = n_img;
        a.audit[3 * (size_t)o + 2] = a_hash;
      }
      double u[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) u[k] = acc[k] * norm_k + acc[3 + k] * norm_c;
      if ((KIND == HS_STOKESLET || kMixed) && a.self_f != nullptr && tcol >= 0 && tcol < a.n_real) {
        const double sc = -(4.0 * a.xi / kSqrtPi);
#pragma unroll
        for (int k = 0; k < 3; ++k) u[k] += sc * a.self_f[3 * tcol + k] / (8.0 * kPi);
      }
#pragma unroll
      for (int k = 0; k < 3; ++k) a.u[3 * o + k] = u[k];
      if (a.uk) {
#pragma unroll
        for (int k = 0; k < 3; ++k) a.uk[3 * o + k] = acc[k] * norm_k;
      }
      if (a.uc) {
#pragma unroll
        for (int k = 0; k < 3; ++k) a.uc[3 * o + k] = acc[3 + k] * norm_c;
      }
    }
  }
}

// work items: (column, first target) for every group of PC_TG targets of a cell column
__global__ void k_count_groups(const int* __restrict__ t_start, int ncol, int nz, int* __restrict__ cnt) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncol; c += gridDim.x * blockDim.x) {
    const int n = t_start[(c + 1) * nz] - t_start[c * nz];  // nz here = cells per column * sub-slabs
    cnt[c] = (n + PC_TG - 1) / PC_TG;
  }
}

__global__ void k_fill_items(const int* __restrict__ t_start, const int* __restrict__ gstart, int ncol, int nz,
                             int2* __restrict__ items) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < ncol; c += gridDim.x * blockDim.x) {
    const int b = t_start[c * nz];
    for (int g = gstart[c]; g < gstart[c + 1]; ++g) items[g] = make_int2(c, b + (g - gstart[c]) * PC_TG);
  }
}

hs_status build_pair_items(hs_ctx* ctx, const int* t_start, int ncol, int nz, int* work, int2* items,
                           const int** n_items_d) {
  int* cnt = work;             // ncol
  int* gstart = work + ncol;   // ncol + 1
  int* scratch = work + 2 * ncol + 1;
  const int gs = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(ncol, 256), ctx->sm_count * 4));
  k_count_groups<<<gs, 256, 0, ctx->stream>>>(t_start, ncol, nz, cnt);
  HS_LAUNCHED(ctx);
  HS_TRY(exclusive_scan(ctx, cnt, ncol, gstart, scratch));
  k_fill_items<<<gs, 256, 0, ctx->stream>>>(t_start, gstart, ncol, nz, items);
  HS_LAUNCHED(ctx);
  *n_items_d = gstart + ncol;
  return HS_OK;
}

hs_status launch_pair(hs_ctx* ctx, const PairArgs& a) {
  if (a.max_items == 0) return HS_OK;
  if (!g_erfcx_ready) {
    HS_CUDA(cudaMemcpyToSymbol(g_erfcx_coef, hs_erfcx_coef, sizeof(hs_erfcx_coef)));
    g_erfcx_ready = true;
  }
  const int kind = a.kind & 15;
  const bool is_half = (a.kind & 16) != 0;
  // persistent-style grid: enough CTAs to fill the machine, looping over the device-side item count
  // (capping it at 2 / 3 / 4 CTAs per SM, to leave register file for the concurrently issued
  // Fourier kernels, measured 103 / 94.5 / 90.4 ms per HL step vs 89.3 ms: not useful)
  const int grid = std::max(1, std::min(a.max_items, ctx->sm_count * 16));
  // every accepted pair has x = xi r <= xi r_c: the short erfcx polynomial covers it when <= 6
  const bool ep6 = !HS_ERFC_TABLE && a.xi * std::sqrt(a.rc2) <= HS_EP6_XMAX * (1.0 - 1e-12);
#define HS_PAIR_CASE1(K, H, AU, E6)                                                                         \
  do {                                                                                                      \
    const int dyn = pc_nh<K>() * pc_h<K>() * pc_rec_bytes<K, H>();                                          \
    HS_CUDA(cudaFuncSetAttribute(k_pair_q<K, H, AU, E6>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn)); \
    k_pair_q<K, H, AU, E6><<<grid, PC_TG, dyn, ctx->stream>>>(a);                                            \
  } while (0)
#define HS_PAIR_CASE(K, H)                    \
  do {                                        \
    if (a.audit)                              \
      HS_PAIR_CASE1(K, H, true, false);       \
    else if (ep6)                             \
      HS_PAIR_CASE1(K, H, false, true);       \
    else                                      \
      HS_PAIR_CASE1(K, H, false, false);      \
  } while (0)
  if (is_half) {
    if (kind == HS_STOKESLET) HS_PAIR_CASE(HS_STOKESLET, true);
    else if (kind == HS_STRESSLET) HS_PAIR_CASE(HS_STRESSLET, true);
    else if (kind == HS_MIXED) HS_PAIR_CASE(HS_MIXED, true);
    else HS_PAIR_CASE(HS_ROTLET, true);
  } else {
    if (kind == HS_STOKESLET) HS_PAIR_CASE(HS_STOKESLET, false);
    else if (kind == HS_STRESSLET) HS_PAIR_CASE(HS_STRESSLET, false);
    else if (kind == HS_MIXED) HS_PAIR_CASE(HS_MIXED, false);
    else HS_PAIR_CASE(HS_ROTLET, false);
  }
#undef HS_PAIR_CASE
#undef HS_PAIR_CASE1
  HS_LAUNCHED(ctx);
  return HS_OK;
}

// ---------------------------------------------------------------------------
// Direct sum: thread per target, sources staged through shared memory.
template <int KIND>
__global__ void __launch_bounds__(256) k_direct(int half, int n_real, int n_src, const double4* __restrict__ P,
                                                const double4* __restrict__ A, const double4* __restrict__ B,
                                                int nt, const double4* __restrict__ TP, double* __restrict__ u,
                                                unsigned* flags) {
  __shared__ double4 sP[256], sA[256], sB[256];
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const bool tv = t < nt;
  const double4 T = TP[tv ? t : 0];
  const long long tcol = (long long)T.w;
  PairConst pc{0.0, 0.0, 0.0};
  double k[3] = {0, 0, 0}, c[3] = {0, 0, 0};
  bool bad = false;
  for (int base = 0; base < n_src; base += 256) {
    __syncthreads();
    const int j = base + threadIdx.x;
    if (j < n_src) {
      sP[threadIdx.x] = P[j];
      sA[threadIdx.x] = A[j];
      sB[threadIdx.x] = B[j];
    }
    __syncthreads();
    const int m = min(256, n_src - base);
    for (int i = 0; i < m; ++i) {
      const double4 S = sP[i];
      if ((long long)S.w == tcol) continue;
      const double d0 = T.x - S.x, d1 = T.y - S.y, d2 = T.z - S.z;
      const double r2 = exact_r2(d0, d1, d2);
      if (r2 == 0.0) {
        bad = true;
        continue;
      }
      const bool img = half && ((long long)S.w >= n_real);
      eval_pair<KIND, false>(pc, d0, d1, d2, r2, T.z, S, sA[i], sB[i], img, k, c, nullptr);
    }
  }
  if (bad && tv) atomicOr(flags, FLAG_SINGULAR);
  if (tv) {
    const double nk = (KIND == HS_ROTLET) ? 1.0 / (4.0 * kPi) : 1.0 / (8.0 * kPi);
    const double nc = 1.0 / (4.0 * kPi);
    for (int q = 0; q < 3; ++q) u[3 * t + q] = k[q] * nk + c[q] * nc;
  }
}

hs_status launch_direct(hs_ctx* ctx, int kind, int half, int n_real, int n_src, const double4* P,
                        const double4* A, const double4* B, int nt, const double4* TP, double* u) {
  if (nt == 0) return HS_OK;
  const int gs = (int)ceil_div(nt, 256);
  if (kind == HS_STOKESLET)
    k_direct<HS_STOKESLET><<<gs, 256, 0, ctx->stream>>>(half, n_real, n_src, P, A, B, nt, TP, u, ctx->d_flags);
  else if (kind == HS_STRESSLET)
    k_direct<HS_STRESSLET><<<gs, 256, 0, ctx->stream>>>(half, n_real, n_src, P, A, B, nt, TP, u, ctx->d_flags);
  else
    k_direct<HS_ROTLET><<<gs, 256, 0, ctx->stream>>>(half, n_real, n_src, P, A, B, nt, TP, u, ctx->d_flags);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

HS_DEFINE_CHECK_COLLECT(pair)

}  // namespace hs

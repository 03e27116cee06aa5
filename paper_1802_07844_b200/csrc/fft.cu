// fft.cu -- the x-direction stage of the pruned 3-D FFT, fused with the k-space scaling.
//
// Pipeline per evaluation (plan.cu), with data (nx,ny,nz) zero-padded to (px,py,pz):
//   Z  : cuFFT D2Z along z on the ny*nx nonzero lines          -> A[y][x][kz]
//   Y  : cuFFT Z2Z along y (input rows y >= ny are zero)         -> B_c[ky][x][kz]
//   X  : THIS KERNEL, one CTA per (ky, kz..kz+KB-1) column group:
//          load the nx nonzero x-values of every source channel (zero-extend to px),
//          forward FFT along x (warp-per-line Stockham in shared memory),
//          k-space multipliers + wall channels + Nyquist symmetrisation (kmult.cuh),
//          inverse FFT along x of the 6 (or 3) output channels,
//          store only the x < nx outputs (output pruning)          -> B_o[ky][x][kz]
//   Y^-1, Z^-1: cuFFT Z2Z inverse along y, Z2D along z (only the y < ny lines)
// The full (px,py,pz/2+1) spectrum of a channel therefore never exists in HBM;
// the x-stage replaces 13 full-spectrum passes + the scale pass of a 3-D cuFFT
// pipeline with one read of the sources and one write of the outputs.
#define HS_TU_ID 3  // checked build: source of a failing HS_CHECK
#include <cmath>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "kmult.cuh"

namespace hs {

// ---- warp-cooperative in-place Stockham FFT of one line in shared memory -------------
// Lines are stored padded (one spare element per 8) so that the strided butterfly
// writes of the early passes hit 8 distinct 16-byte bank groups per quarter-warp.
__device__ __forceinline__ int pd8(int i) { return i + (i >> 3); }
__host__ __device__ __forceinline__ int padded_line(int n) { return n + (n >> 3) + 1; }
__device__ __forceinline__ double2 cm(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 ad(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 sb(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 mi(double2 a) { return make_double2(a.y, -a.x); }  // -i a

template <int R>
__device__ __forceinline__ void dft(double2* a) {
  if (R == 2) {
    const double2 t = a[0];
    a[0] = ad(t, a[1]);
    a[1] = sb(t, a[1]);
  } else if (R == 3) {
    const double c = 0.86602540378443864676;  // sin(2 pi/3)
    const double2 s = ad(a[1], a[2]), d = sb(a[1], a[2]);
    const double2 m = make_double2(a[0].x - 0.5 * s.x, a[0].y - 0.5 * s.y);
    a[0] = ad(a[0], s);
    const double2 t = make_double2(c * d.y, -c * d.x);  // -i c d
    a[1] = ad(m, t);
    a[2] = sb(m, t);
  } else if (R == 4) {
    const double2 t0 = ad(a[0], a[2]), t1 = sb(a[0], a[2]), t2 = ad(a[1], a[3]), t3 = mi(sb(a[1], a[3]));
    a[0] = ad(t0, t2);
    a[2] = sb(t0, t2);
    a[1] = ad(t1, t3);
    a[3] = sb(t1, t3);
  } else if (R == 5) {
    const double c1 = 0.30901699437494742410, c2 = -0.80901699437494742410;
    const double s1 = 0.95105651629515357212, s2 = 0.58778525229247312917;
    const double2 p1 = ad(a[1], a[4]), d1 = sb(a[1], a[4]), p2 = ad(a[2], a[3]), d2 = sb(a[2], a[3]);
    const double2 a0 = a[0];
    a[0] = ad(a0, ad(p1, p2));
    const double2 t1 = make_double2(a0.x + c1 * p1.x + c2 * p2.x, a0.y + c1 * p1.y + c2 * p2.y);
    const double2 t2 = make_double2(a0.x + c2 * p1.x + c1 * p2.x, a0.y + c2 * p1.y + c1 * p2.y);
    const double2 u1 = make_double2(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y);
    const double2 u2 = make_double2(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y);
    a[1] = ad(t1, mi(u1));
    a[4] = sb(t1, mi(u1));
    a[2] = ad(t2, mi(u2));
    a[3] = sb(t2, mi(u2));
  } else if (R == 8) {
    double2 e[4] = {a[0], a[2], a[4], a[6]}, o[4] = {a[1], a[3], a[5], a[7]};
    dft<4>(e);
    dft<4>(o);
    const double h = 0.70710678118654752440;
    const double2 w1 = make_double2(h, -h), w3 = make_double2(-h, -h);
    o[1] = cm(o[1], w1);
    o[2] = mi(o[2]);
    o[3] = cm(o[3], w3);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      a[k] = ad(e[k], o[k]);
      a[k + 4] = sb(e[k], o[k]);
    }
  } else {
    // generic small prime (7, 11): direct DFT with exact-angle twiddles
    double2 y[R];
#pragma unroll
    for (int k = 0; k < R; ++k) {
      double2 s = make_double2(0.0, 0.0);
#pragma unroll
      for (int m = 0; m < R; ++m) {
        double sn, cs;
        sincospi(-2.0 * ((m * k) % R) / R, &sn, &cs);
        s = ad(s, cm(a[m], make_double2(cs, sn)));
      }
      y[k] = s;
    }
#pragma unroll
    for (int k = 0; k < R; ++k) a[k] = y[k];
  }
}

// One radix-R pass of a length-N line (current sub-transform length L) by one warp:
// each lane loads its butterflies' inputs into registers, __syncwarp, writes them back
// (in-place Stockham autosort).
template <int R, int MAXB>
__device__ __forceinline__ void warp_pass(double2* line, int N, int L, const double2* tw, int lane) {
  const int nb = N / R;
  const int tstep = N / (L * R);
  double2 v[MAXB][R];
#pragma unroll
  for (int q = 0; q < MAXB; ++q) {
    const int b = lane + 32 * q;
    if (b < nb) {
      const int k = b % L;
#pragma unroll
      for (int m = 0; m < R; ++m) {
        double2 x = line[pd8(b + m * nb)];
        if (m > 0 && k > 0) x = cm(x, tw[m * k * tstep]);
        v[q][m] = x;
      }
      dft<R>(v[q]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int q = 0; q < MAXB; ++q) {
    const int b = lane + 32 * q;
    if (b < nb) {
      const int k = b % L;
      const int base = (b / L) * L * R + k;
#pragma unroll
      for (int m = 0; m < R; ++m) line[pd8(base + m * L)] = v[q][m];
    }
  }
  __syncwarp();
}

// Compile-time radix plan: FFT length N = product of Rs (natural-order output).
template <int N, int L, int R, int... Rest>
__device__ __forceinline__ void fft_passes(double2* line, const double2* tw, int lane) {
  warp_pass<R, (N / R + 31) / 32>(line, N, L, tw, lane);
  if constexpr (sizeof...(Rest) > 0) fft_passes<N, L * R, Rest...>(line, tw, lane);
}

template <int... Rs>
struct FixedFFT {
  static constexpr int N = (Rs * ...);
  __device__ __forceinline__ static void run(double2* line, const FftPlan&, const double2* tw, int lane) {
    fft_passes<N, 1, Rs...>(line, tw, lane);
  }
};

// Runtime radix plan (any 11-smooth N <= 1024): one non-inlined function per
// (radix, butterflies-per-lane) variant.
template <int R, int MAXB>
__device__ __noinline__ void warp_pass_v(double2* line, int N, int L, const double2* tw, int lane) {
  warp_pass<R, MAXB>(line, N, L, tw, lane);
}

template <int R, int M0, int... Ms>
__device__ __forceinline__ void warp_pass_pick(int need, double2* line, int N, int L, const double2* tw, int lane) {
  if constexpr (sizeof...(Ms) == 0) {
    warp_pass_v<R, M0>(line, N, L, tw, lane);
  } else {
    if (need <= M0) warp_pass_v<R, M0>(line, N, L, tw, lane);
    else warp_pass_pick<R, Ms...>(need, line, N, L, tw, lane);
  }
}

struct AnyFFT {
  static constexpr int N = 0;
  __device__ __forceinline__ static void run(double2* line, const FftPlan& pl, const double2* tw, int lane) {
    int L = 1;
    const int n = pl.n;
    for (int s = 0; s < pl.npass; ++s) {
      const int R = pl.radix[s];
      const int need = (n / R + 31) / 32;
      switch (R) {
        case 2: warp_pass_pick<2, 1, 2, 4, 8, 16>(need, line, n, L, tw, lane); break;
        case 3: warp_pass_pick<3, 1, 2, 3, 4, 6, 11>(need, line, n, L, tw, lane); break;
        case 4: warp_pass_pick<4, 1, 2, 4, 8>(need, line, n, L, tw, lane); break;
        case 5: warp_pass_pick<5, 1, 2, 4, 7>(need, line, n, L, tw, lane); break;
        case 7: warp_pass_pick<7, 1, 2, 5>(need, line, n, L, tw, lane); break;
        case 8: warp_pass_pick<8, 1, 2, 4>(need, line, n, L, tw, lane); break;
        default: warp_pass_pick<11, 1, 3>(need, line, n, L, tw, lane); break;
      }
      L *= R;
    }
  }
};

hs_status make_fft_plan(int n, FftPlan* pl) {
  pl->n = n;
  pl->npass = 0;
  int m = n;
  const int order[] = {8, 4, 2, 3, 5, 7, 11};
  while (m > 1) {
    bool found = false;
    for (int r : order) {
      if (m % r == 0) {
        if (pl->npass >= FftPlan::kMaxPass) return fail(HS_ERR_PARAMETER, "FFT length has too many factors");
        pl->radix[pl->npass++] = r;
        m /= r;
        found = true;
        break;
      }
    }
    if (!found) return fail(HS_ERR_PARAMETER, "padded FFT length must be 11-smooth");
  }
  if (n > 1024) return fail(HS_ERR_PARAMETER, "padded FFT length > 1024 is not supported by the x-stage");
  return HS_OK;
}

// ---- fused x-stage ----------------------------------------------------------------------
// Nyquist planes (rare): full scale_point with the Hermitian symmetrisation, kept out of line so
// its register footprint does not limit the main kernel.
template <int KIND, bool HALF>
__device__ __noinline__ void scale_nyquist(double2* col, int cstride, int kx, int ky, int kz, const int* p,
                                           const double* kscale, double ka, double kb, double inv_n, double tB,
                                           double tH) {
  constexpr int NIN = KChan<KIND, HALF>::NIN, NOUT = KChan<KIND, HALF>::NOUT;
  cplx C[NIN], out[6];
#pragma unroll
  for (int c = 0; c < NIN; ++c) {
    const double2 v = col[c * cstride];
    C[c] = {v.x, v.y};
  }
  scale_point<KIND, HALF>(kx, ky, kz, p, kscale, ka, kb, inv_n, tB, tH, C, out);
#pragma unroll
  for (int o = 0; o < NOUT; ++o) col[o * cstride] = make_double2(out[o].re, -out[o].im);
}

constexpr int XF_THREADS = 256;  // 2 CTAs per SM: one CTA's loads overlap the other's FFTs
#ifndef XR_THREADS_DEF
#define XR_THREADS_DEF 256
#endif
constexpr int XR_THREADS = XR_THREADS_DEF;  // register x-stage CTA size

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// output store of the x stage: into Bout (the pass's inputs by default), or added to what is
// there (a.accum: a second channel group's contribution, e.g. the mixed plan's stresslet pass)
__device__ __forceinline__ void xstore(const XArgs& a, double2* dst, double2 v) {
  if (a.accum) {
    const double2 o = *dst;
    v.x += o.x;
    v.y += o.y;
  }
  *dst = v;
}

template <int KIND, bool HALF, int KB, class FFT>
__global__ void __launch_bounds__(XF_THREADS, 2) k_xfused(const XArgs a) {
  constexpr int NIN = KChan<KIND, HALF>::NIN, NOUT = KChan<KIND, HALF>::NOUT;
  constexpr int NL = NIN > NOUT ? NIN : NOUT;
  extern __shared__ double2 smem[];
  const int px = a.plan.n;
  const int LS = padded_line(px);
  double2* lines = smem;                    // [max(NIN,NOUT)][KB][LS]
  double2* tw = smem + NL * KB * LS;        // [px]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < px; i += blockDim.x) tw[i] = a.tw[i];
  const int nkb = (a.nzh + KB - 1) / KB;
  const int n_items = a.py * nkb;
  const int p[3] = {a.px, a.py, a.pz};
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int ky = item / nkb;
    const int kz0 = (item % nkb) * KB;
    const int kbn = min(KB, a.nzh - kz0);
    __syncthreads();
    // load the nx nonzero x-values of every channel (cp.async, all in flight at once),
    // zero-extend to px
#pragma unroll 1
    for (int c = 0; c < NIN; ++c) {
      const double2* src = a.B + c * a.ch_stride + (int64_t)ky * a.nx * a.nzh + kz0;
      for (int x = tid; x < px; x += blockDim.x) {
#pragma unroll
        for (int kb = 0; kb < KB; ++kb) {
          double2* dst = &lines[(c * KB + kb) * LS + pd8(x)];
          if (x < a.nx && kb < kbn)
            cp_async16(dst, src + (int64_t)x * a.nzh + kb);
          else
            *dst = make_double2(0.0, 0.0);
        }
      }
    }
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    for (int l = warp; l < NIN * KB; l += blockDim.x / 32) FFT::run(lines + l * LS, a.plan, tw, lane);
    __syncthreads();
    // k-space scaling at every (kx, ky, kz) of the group
    for (int i = tid; i < KB * px; i += blockDim.x) {
      const int kb = i / px, kx = i - kb * px;
      if (kb >= kbn) continue;
      const int kzl = kz0 + kb, kz = a.kz0 + kzl;  // local column, global wavenumber index
      const int64_t ti = ((int64_t)ky * a.nzh + kzl) * px + kx;
      const double tB = (KIND == HS_ROTLET) ? 0.0 : a.tabB[ti];
      const double tH = (KIND == HS_ROTLET || HALF) ? a.tabH[ti] : 0.0;
      double2* col = lines + kb * LS + pd8(kx);  // channel c at col[c * KB * LS]
      if (2 * kx == px || 2 * ky == a.py || 2 * kz == a.pz) {
        scale_nyquist<KIND, HALF>(col, KB * LS, kx, ky, kz, p, a.kscale, a.ka, a.kb, a.inv_n, tB, tH);
        continue;
      }
      cplx C[NIN], out[6];
#pragma unroll
      for (int c = 0; c < NIN; ++c) {
        const double2 v = col[c * KB * LS];
        C[c] = {v.x, v.y};
      }
      const double s8 = 1.0 / (8.0 * kPi), s4 = 1.0 / (4.0 * kPi);
      const double kxv = kval(kx, px, a.kscale[0]), kyv = kval(ky, a.py, a.kscale[1]),
                   kzv = kval(kz, a.pz, a.kscale[2]);
      const double k2 = kxv * kxv + kyv * kyv + kzv * kzv;
      const double E = exp(-a.ka * k2);
      const double G = (KIND == HS_ROTLET) ? tH * E * s4 * a.inv_n : tB * E * (1.0 + a.kb * k2) * s8 * a.inv_n;
      const double Fc = HALF ? tH * E * s4 * a.inv_n : 0.0;
      apply_multiplier<KIND, HALF>(kxv, kyv, kzv, G, Fc, C, out);
      // inverse transform by conjugation: IFFT(y) = conj(FFT(conj(y))) (normalisation already in inv_n)
#pragma unroll
      for (int o = 0; o < NOUT; ++o) col[o * KB * LS] = make_double2(out[o].re, -out[o].im);
    }
    __syncthreads();
    for (int l = warp; l < NOUT * KB; l += blockDim.x / 32) FFT::run(lines + l * LS, a.plan, tw, lane);
    __syncthreads();
    // store the x < nx outputs (conjugated back)
    for (int i = tid; i < NOUT * a.nx; i += blockDim.x) {
      const int o = i / a.nx, x = i - o * a.nx;
      double2* dst = a.Bout + o * a.ch_stride + ((int64_t)ky * a.nx + x) * a.nzh + kz0;
#pragma unroll
      for (int kb = 0; kb < KB; ++kb) {
        if (kb < kbn) {
          const double2 v = lines[(o * KB + kb) * LS + pd8(x)];
          xstore(a, &dst[kb], make_double2(v.x, -v.y));
        }
      }
    }
  }
}

// ---- register-resident x-stage (N = 32 M) -------------------------------------------------
// One warp transforms one line: lane l holds x[l + 32 j] (j < M) and computes the M-point DFTs
// over j in registers; twiddles W_N^{l k1}; one transpose through shared memory
// (S[k1][l], rows padded to 33); the 32-point DFTs over l are split over lane pairs
// (r = lane/2 < M, h = lane%2: a 16-point DFT of the even/odd half each, then one radix-2
// combine across the pair by shuffles).  Lane (r,h) ends with X[r + M (k' + 16 h)], k' < 16.
// Shared-memory traffic per line: one write + one read of the line (the Stockham version
// makes a round trip per radix pass).
__constant__ double2 c_w15[15];  // exp(-2 pi i m / 15)
__constant__ double2 c_w11[11];  // exp(-2 pi i m / 11)
__constant__ double2 c_w27[27];  // exp(-2 pi i m / 27)
__constant__ double2 c_w16[16];  // exp(-2 pi i m / 16)
__constant__ double2 c_w32[16];  // exp(-2 pi i m / 32)
__constant__ double2 c_w25[25];  // exp(-2 pi i m / 25)
__constant__ double2 c_w30[15];  // exp(-2 pi i m / 30)
static bool g_xreg_consts = false;

static hs_status xreg_constants() {
  if (g_xreg_consts) return HS_OK;
  double2 w15[15], w16[16], w32[16], w11[11], w27[27];
  const long double tp = 6.283185307179586476925286766559005768L;
  for (int m = 0; m < 15; ++m) w15[m] = make_double2((double)std::cos(tp * m / 15), (double)-std::sin(tp * m / 15));
  for (int m = 0; m < 27; ++m) w27[m] = make_double2((double)std::cos(tp * m / 27), (double)-std::sin(tp * m / 27));
  for (int m = 0; m < 11; ++m) w11[m] = make_double2((double)std::cos(tp * m / 11), (double)-std::sin(tp * m / 11));
  for (int m = 0; m < 16; ++m) w16[m] = make_double2((double)std::cos(tp * m / 16), (double)-std::sin(tp * m / 16));
  for (int m = 0; m < 16; ++m) w32[m] = make_double2((double)std::cos(tp * m / 32), (double)-std::sin(tp * m / 32));
  HS_CUDA(cudaMemcpyToSymbol(c_w15, w15, sizeof(w15)));
  HS_CUDA(cudaMemcpyToSymbol(c_w11, w11, sizeof(w11)));
  HS_CUDA(cudaMemcpyToSymbol(c_w27, w27, sizeof(w27)));
  HS_CUDA(cudaMemcpyToSymbol(c_w16, w16, sizeof(w16)));
  HS_CUDA(cudaMemcpyToSymbol(c_w32, w32, sizeof(w32)));
  double2 w25[25], w30[15];
  for (int m = 0; m < 25; ++m) w25[m] = make_double2((double)std::cos(tp * m / 25), (double)-std::sin(tp * m / 25));
  for (int m = 0; m < 15; ++m) w30[m] = make_double2((double)std::cos(tp * m / 30), (double)-std::sin(tp * m / 30));
  HS_CUDA(cudaMemcpyToSymbol(c_w25, w25, sizeof(w25)));
  HS_CUDA(cudaMemcpyToSymbol(c_w30, w30, sizeof(w30)));
  g_xreg_consts = true;
  return HS_OK;
}

// DFT-15 in place: j = j1 + 3 j2, k = 5 k1 + k2 (DFT5 over j2, twiddle W15^{j1 k2}, DFT3 over j1)
__device__ __forceinline__ void dft15(double2* v) {
  double2 Y[3][5];
#pragma unroll
  for (int j1 = 0; j1 < 3; ++j1) {
    double2 t[5];
#pragma unroll
    for (int j2 = 0; j2 < 5; ++j2) t[j2] = v[j1 + 3 * j2];
    dft<5>(t);
#pragma unroll
    for (int k2 = 0; k2 < 5; ++k2) Y[j1][k2] = (j1 * k2 == 0) ? t[k2] : cm(t[k2], c_w15[j1 * k2]);
  }
#pragma unroll
  for (int k2 = 0; k2 < 5; ++k2) {
    double2 t[3] = {Y[0][k2], Y[1][k2], Y[2][k2]};
    dft<3>(t);
#pragma unroll
    for (int k1 = 0; k1 < 3; ++k1) v[5 * k1 + k2] = t[k1];
  }
}

// DFT-16 in place: m = m1 + 4 m2, k = k2 + 4 k1 (DFT4 over m2, twiddle W16^{m1 k2}, DFT4 over m1)
__device__ __forceinline__ void dft16(double2* a) {
  double2 B[4][4];
#pragma unroll
  for (int m1 = 0; m1 < 4; ++m1) {
    double2 t[4] = {a[m1], a[m1 + 4], a[m1 + 8], a[m1 + 12]};
    dft<4>(t);
#pragma unroll
    for (int k2 = 0; k2 < 4; ++k2) B[m1][k2] = (m1 * k2 == 0) ? t[k2] : cm(t[k2], c_w16[m1 * k2]);
  }
#pragma unroll
  for (int k2 = 0; k2 < 4; ++k2) {
    double2 t[4] = {B[0][k2], B[1][k2], B[2][k2], B[3][k2]};
    dft<4>(t);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) a[k2 + 4 * k1] = t[k1];
  }
}

// DFT-11 in place (direct, symmetric pairs: 5 cos/sin pairs per output)
__device__ __forceinline__ void dft11(double2* v) {
  double2 sp[5], sm[5];
#pragma unroll
  for (int m = 1; m <= 5; ++m) {
    sp[m - 1] = ad(v[m], v[11 - m]);
    sm[m - 1] = sb(v[m], v[11 - m]);
  }
  double2 y[11];
  double2 s0 = v[0];
#pragma unroll
  for (int m = 0; m < 5; ++m) s0 = ad(s0, sp[m]);
  y[0] = s0;
#pragma unroll
  for (int k = 1; k <= 5; ++k) {
    double2 re = v[0], im = make_double2(0.0, 0.0);
#pragma unroll
    for (int m = 1; m <= 5; ++m) {
      const double2 w = c_w11[(m * k) % 11];  // (cos, -sin)
      re = make_double2(fma(w.x, sp[m - 1].x, re.x), fma(w.x, sp[m - 1].y, re.y));
      im = make_double2(fma(w.y, sm[m - 1].x, im.x), fma(w.y, sm[m - 1].y, im.y));
    }
    // X_k = re + i im, X_{11-k} = re - i im  (im holds -sin * (a_m - a_{11-m}))
    y[k] = make_double2(re.x - im.y, re.y + im.x);
    y[11 - k] = make_double2(re.x + im.y, re.y - im.x);
  }
#pragma unroll
  for (int k = 0; k < 11; ++k) v[k] = y[k];
}

// DFT-9 in place: j = j1 + 3 j2, k = 3 k1 + k2 (W9^m = W27^{3m})
__device__ __forceinline__ void dft9(double2* v) {
  double2 Y[3][3];
#pragma unroll
  for (int j1 = 0; j1 < 3; ++j1) {
    double2 t[3] = {v[j1], v[j1 + 3], v[j1 + 6]};
    dft<3>(t);
#pragma unroll
    for (int k2 = 0; k2 < 3; ++k2) Y[j1][k2] = (j1 * k2 == 0) ? t[k2] : cm(t[k2], c_w27[3 * j1 * k2]);
  }
#pragma unroll
  for (int k2 = 0; k2 < 3; ++k2) {
    double2 t[3] = {Y[0][k2], Y[1][k2], Y[2][k2]};
    dft<3>(t);
#pragma unroll
    for (int k1 = 0; k1 < 3; ++k1) v[3 * k1 + k2] = t[k1];
  }
}

// DFT-27 in place: j = j1 + 3 j2 (j2 < 9), k = 9 k1 + k2 (DFT9 over j2, twiddle W27^{j1 k2}, DFT3)
__device__ __forceinline__ void dft27(double2* v) {
  double2 Y[3][9];
#pragma unroll
  for (int j1 = 0; j1 < 3; ++j1) {
    double2 t[9];
#pragma unroll
    for (int j2 = 0; j2 < 9; ++j2) t[j2] = v[j1 + 3 * j2];
    dft9(t);
#pragma unroll
    for (int k2 = 0; k2 < 9; ++k2) Y[j1][k2] = (j1 * k2 == 0) ? t[k2] : cm(t[k2], c_w27[j1 * k2]);
  }
#pragma unroll
  for (int k2 = 0; k2 < 9; ++k2) {
    double2 t[3] = {Y[0][k2], Y[1][k2], Y[2][k2]};
    dft<3>(t);
#pragma unroll
    for (int k1 = 0; k1 < 3; ++k1) v[9 * k1 + k2] = t[k1];
  }
}

template <int M>
__device__ __forceinline__ void dftM(double2* v) {
  static_assert(M == 15 || M == 11 || M == 27, "register FFT: M = 15 (N = 480), 11 (352), 27 (864)");
  if constexpr (M == 15)
    dft15(v);
  else if constexpr (M == 11)
    dft11(v);
  else
    dft27(v);
}

// forward DFT of the line whose element l + 32 j is v[j]; S: warp scratch (M x 33);
// tw: pd8-padded W_N^i table; out[g]: X[r + M (k' + 16 h)], k' < 16, for the row r = 16 g + lane/2
// (< M) of row group g (M <= 16: one group; M = 27: two, the second half-populated)
template <int M>
struct RegFFT {
  static constexpr int NG = (M + 15) / 16;
};
template <int M>
__device__ __forceinline__ void warp_fft_reg(double2* v, double2* S, const double2* tw, int lane,
                                             double2 (*out)[16]) {
  dftM<M>(v);
#pragma unroll
  for (int k1 = 1; k1 < M; ++k1) v[k1] = cm(v[k1], tw[pd8(lane * k1)]);
  __syncwarp();
#pragma unroll
  for (int k1 = 0; k1 < M; ++k1) S[k1 * 33 + lane] = v[k1];
  __syncwarp();
  const int h = lane & 1;
#pragma unroll
  for (int g = 0; g < RegFFT<M>::NG; ++g) {
    const int r = 16 * g + (lane >> 1);
    const int rr = r < M ? r : M - 1;
#pragma unroll
    for (int m = 0; m < 16; ++m) out[g][m] = S[rr * 33 + 2 * m + h];
  }
#pragma unroll
  for (int g = 0; g < RegFFT<M>::NG; ++g) {
    dft16(out[g]);
    // radix-2 combine across the lane pair: X[k'] = Y0 + W32^k' Y1, X[k'+16] = Y0 - W32^k' Y1
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const double2 t = (h && k) ? cm(out[g][k], c_w32[k]) : out[g][k];  // h = 1 holds Y1
      double2 p;
      p.x = __shfl_xor_sync(0xffffffffu, t.x, 1);
      p.y = __shfl_xor_sync(0xffffffffu, t.y, 1);
      out[g][k] = h ? sb(p, t) : ad(t, p);
    }
  }
}

// STAGE: the next column's nx input values of every channel are prefetched with cp.async into a
// shared-memory staging area while the current column is scaled and inverse-transformed, so the
// forward FFTs read shared memory instead of waiting on strided global loads (used when the
// extra NIN * nx * 16 bytes keep the kernel's CTAs per SM).
template <int KIND, bool HALF, int M, bool STAGE>
__global__ void __launch_bounds__(XR_THREADS, M == 27 ? 1 : 2) k_xreg(const XArgs a) {
  constexpr int N = 32 * M, LSR = M * 33;
  constexpr int NIN = KChan<KIND, HALF>::NIN, NOUT = KChan<KIND, HALF>::NOUT;
  constexpr int NL = NIN > NOUT ? NIN : NOUT, NW = XR_THREADS / 32;
  extern __shared__ double2 smem[];
  double2* lines = smem;            // [NL][LSR]: transpose scratch of the line's warp, then the channel line
  double2* tw = smem + NL * LSR;    // pd8-padded twiddles
  double2* stage = tw + padded_line(N);  // [NIN][nx] (STAGE)
  double* stab = reinterpret_cast<double*>(stage + NIN * a.nx);  // [2][N] table rows (STAGE)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < N; i += blockDim.x) tw[pd8(i)] = a.tw[i];
  const int n_items = a.py * a.nzh;
  const int p[3] = {a.px, a.py, a.pz};
  const int r = lane >> 1, h = lane & 1;
  auto prefetch = [&](int it) {
    if (it < n_items) {
      const int ky2 = it / a.nzh, kz2 = it - ky2 * a.nzh;
      // (channel-major loop: no per-element integer division; nx <= N)
      const double2* src = a.B + ((int64_t)ky2 * a.nx) * a.nzh + kz2;
      for (int x = tid; x < a.nx; x += blockDim.x) {
#pragma unroll
        for (int c = 0; c < NIN; ++c) cp_async16(&stage[c * a.nx + x], src + c * a.ch_stride + (int64_t)x * a.nzh);
      }
    }
    cp_async_commit();
  };
  // table rows of a column (its scaling phase), prefetched while the previous column is
  // inverse-transformed
  auto prefetch_tab = [&](int it) {
    if (it < n_items) {
      const int ky2 = it / a.nzh, kz2 = it - ky2 * a.nzh;
      const int64_t t0 = ((int64_t)ky2 * a.nzh + kz2) * N;
      for (int i = tid; i < N / 2; i += blockDim.x) {
        if (KIND != HS_ROTLET) cp_async16(&stab[2 * i], a.tabB + t0 + 2 * i);
        if (KIND == HS_ROTLET || HALF) cp_async16(&stab[N + 2 * i], a.tabH + t0 + 2 * i);
      }
    }
    cp_async_commit();
  };
  if (STAGE) {
    prefetch(blockIdx.x);
    prefetch_tab(blockIdx.x);
  }
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int ky = item / a.nzh;
    const int kzl = item - ky * a.nzh, kz = a.kz0 + kzl;  // local column, global wavenumber index
    HS_CHECK(ky < a.py && kzl < a.nzh && kz <= a.pz / 2 && a.nx <= N);
    if (STAGE) cp_async_wait_all();
    __syncthreads();  // previous item's lines consumed (and twiddles / staged inputs visible)
    for (int c = warp; c < NIN; c += NW) {
      double2 v[M], out[RegFFT<M>::NG][16];
      const double2* src = a.B + c * a.ch_stride + (int64_t)ky * a.nx * a.nzh + kzl;
#pragma unroll
      for (int j = 0; j < M; ++j) {
        const int x = lane + 32 * j;
        if (STAGE)
          v[j] = x < a.nx ? stage[c * a.nx + x] : make_double2(0.0, 0.0);
        else
          v[j] = x < a.nx ? src[(int64_t)x * a.nzh] : make_double2(0.0, 0.0);
      }
      double2* S = lines + c * LSR;
      warp_fft_reg<M>(v, S, tw, lane, out);
      __syncwarp();
#pragma unroll
      for (int g = 0; g < RegFFT<M>::NG; ++g) {
        const int rg = r + 16 * g;
        if (rg < M) {
#pragma unroll
          for (int k = 0; k < 16; ++k) S[rg + M * (k + 16 * h)] = out[g][k];
        }
      }
    }
    __syncthreads();
    if (STAGE) prefetch(item + gridDim.x);  // staging area free: the forward FFTs have read it
    // k-space scaling at every kx of the column (channel c of kx at lines[c * LSR + kx])
    for (int kx = tid; kx < N; kx += blockDim.x) {
      const int64_t ti = ((int64_t)ky * a.nzh + kzl) * N + kx;
      const double tB = (KIND == HS_ROTLET) ? 0.0 : (STAGE ? stab[kx] : a.tabB[ti]);
      const double tH = (KIND == HS_ROTLET || HALF) ? (STAGE ? stab[N + kx] : a.tabH[ti]) : 0.0;
      double2* col = lines + kx;
      if (2 * kx == N || 2 * ky == a.py || 2 * kz == a.pz) {
        scale_nyquist<KIND, HALF>(col, LSR, kx, ky, kz, p, a.kscale, a.ka, a.kb, a.inv_n, tB, tH);
        continue;
      }
      cplx C[NIN], outc[6];
#pragma unroll
      for (int c = 0; c < NIN; ++c) {
        const double2 vv = col[c * LSR];
        C[c] = {vv.x, vv.y};
      }
      const double s8 = 1.0 / (8.0 * kPi), s4 = 1.0 / (4.0 * kPi);
      const double kxv = kval(kx, N, a.kscale[0]), kyv = kval(ky, a.py, a.kscale[1]), kzv = kval(kz, a.pz, a.kscale[2]);
      const double k2 = kxv * kxv + kyv * kyv + kzv * kzv;
      const double E = exp(-a.ka * k2);
      const double G = (KIND == HS_ROTLET) ? tH * E * s4 * a.inv_n : tB * E * (1.0 + a.kb * k2) * s8 * a.inv_n;
      const double Fc = HALF ? tH * E * s4 * a.inv_n : 0.0;
      apply_multiplier<KIND, HALF>(kxv, kyv, kzv, G, Fc, C, outc);
      // inverse transform by conjugation: IFFT(y) = conj(FFT(conj(y))) (normalisation already in inv_n)
#pragma unroll
      for (int o = 0; o < NOUT; ++o) col[o * LSR] = make_double2(outc[o].re, -outc[o].im);
    }
    __syncthreads();
    if (STAGE) prefetch_tab(item + gridDim.x);  // table rows read by this column's scaling
    for (int o = warp; o < NOUT; o += NW) {
      double2 v[M], out[RegFFT<M>::NG][16];
      double2* S = lines + o * LSR;
#pragma unroll
      for (int j = 0; j < M; ++j) v[j] = S[lane + 32 * j];
      warp_fft_reg<M>(v, S, tw, lane, out);
      double2* dst = a.Bout + o * a.ch_stride + (int64_t)ky * a.nx * a.nzh + kzl;
#pragma unroll
      for (int g = 0; g < RegFFT<M>::NG; ++g) {
        const int rg = r + 16 * g;
        if (rg < M) {
#pragma unroll
          for (int k = 0; k < 16; ++k) {
            const int x = rg + M * (k + 16 * h);
            if (x < a.nx) xstore(a, &dst[(int64_t)x * a.nzh], make_double2(out[g][k].x, -out[g][k].y));
          }
        }
      }
    }
  }
}

// ---- register x-stage for N = 750 = 30 x 25 (cfg4's padded length) -------------------------
// Lanes l < 30 hold x[l + 30 j] (j < 25): DFT25 over j in registers, twiddle W750^{l k1}, one
// transpose through shared memory (S[k1][l], rows of 31), then lanes r < 25 each take row r and
// finish with a DFT30 (= 2 x DFT15) in registers, ending with X[r + 25 k2], k2 < 30.
__device__ __forceinline__ void dft25(double2* v) {
  double2 Y[5][5];
#pragma unroll
  for (int j1 = 0; j1 < 5; ++j1) {
    double2 t[5];
#pragma unroll
    for (int j2 = 0; j2 < 5; ++j2) t[j2] = v[j1 + 5 * j2];
    dft<5>(t);
#pragma unroll
    for (int k2 = 0; k2 < 5; ++k2) Y[j1][k2] = (j1 * k2 == 0) ? t[k2] : cm(t[k2], c_w25[j1 * k2]);
  }
#pragma unroll
  for (int k2 = 0; k2 < 5; ++k2) {
    double2 t[5] = {Y[0][k2], Y[1][k2], Y[2][k2], Y[3][k2], Y[4][k2]};
    dft<5>(t);
#pragma unroll
    for (int k1 = 0; k1 < 5; ++k1) v[5 * k1 + k2] = t[k1];
  }
}
constexpr int X750_L = 30, X750_M = 25, X750_RS = 31, X750_LS = X750_M * X750_RS;  // line slot >= 750
// forward DFT of the line with x[l + 30 j] in v[j] (lanes < 30); result X[kx] left in S[kx]
__device__ __forceinline__ void warp_fft750(double2* v, double2* S, const double2* tw, int lane) {
  if (lane < X750_L) {
    dft25(v);
#pragma unroll
    for (int k1 = 1; k1 < X750_M; ++k1) v[k1] = cm(v[k1], tw[pd8(lane * k1)]);
  }
  __syncwarp();
  if (lane < X750_L) {
#pragma unroll
    for (int k1 = 0; k1 < X750_M; ++k1) S[k1 * X750_RS + lane] = v[k1];
  }
  __syncwarp();
  // DFT30 of row r = lane as 2 x DFT15 (even / odd l), read straight into the two halves
  double2 e[15], o[15];
  const int rr = lane < X750_M ? lane : X750_M - 1;
#pragma unroll
  for (int m = 0; m < 15; ++m) {
    e[m] = S[rr * X750_RS + 2 * m];
    o[m] = S[rr * X750_RS + 2 * m + 1];
  }
  __syncwarp();
  dft15(e);
  dft15(o);
  if (lane < X750_M) {
#pragma unroll
    for (int k = 0; k < 15; ++k) {
      const double2 t = k == 0 ? o[0] : cm(o[k], c_w30[k]);
      S[lane + X750_M * k] = ad(e[k], t);
      S[lane + X750_M * (k + 15)] = sb(e[k], t);
    }
  }
  __syncwarp();
}

template <int KIND, bool HALF>
__global__ void __launch_bounds__(XF_THREADS, 2) k_x750(const XArgs a) {
  constexpr int N = 750, LSR = X750_LS;
  constexpr int NIN = KChan<KIND, HALF>::NIN, NOUT = KChan<KIND, HALF>::NOUT;
  constexpr int NL = NIN > NOUT ? NIN : NOUT, NW = XF_THREADS / 32;
  extern __shared__ double2 smem[];
  double2* lines = smem;          // [NL][LSR]
  double2* tw = smem + NL * LSR;  // pd8-padded W750^i
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < N; i += blockDim.x) tw[pd8(i)] = a.tw[i];
  const int n_items = a.py * a.nzh;
  const int p[3] = {a.px, a.py, a.pz};
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int ky = item / a.nzh;
    const int kzl = item - ky * a.nzh, kz = a.kz0 + kzl;
    __syncthreads();
    for (int c = warp; c < NIN; c += NW) {
      double2 v[X750_M];
      const double2* src = a.B + c * a.ch_stride + (int64_t)ky * a.nx * a.nzh + kzl;
#pragma unroll
      for (int j = 0; j < X750_M; ++j) {
        const int x = lane + X750_L * j;
        v[j] = (lane < X750_L && x < a.nx) ? src[(int64_t)x * a.nzh] : make_double2(0.0, 0.0);
      }
      warp_fft750(v, lines + c * LSR, tw, lane);
    }
    __syncthreads();
    for (int kx = tid; kx < N; kx += blockDim.x) {
      const int64_t ti = ((int64_t)ky * a.nzh + kzl) * N + kx;
      const double tB = (KIND == HS_ROTLET) ? 0.0 : a.tabB[ti];
      const double tH = (KIND == HS_ROTLET || HALF) ? a.tabH[ti] : 0.0;
      double2* col = lines + kx;
      if (2 * kx == N || 2 * ky == a.py || 2 * kz == a.pz) {
        scale_nyquist<KIND, HALF>(col, LSR, kx, ky, kz, p, a.kscale, a.ka, a.kb, a.inv_n, tB, tH);
        continue;
      }
      cplx C[NIN], outc[6];
#pragma unroll
      for (int c = 0; c < NIN; ++c) {
        const double2 vv = col[c * LSR];
        C[c] = {vv.x, vv.y};
      }
      const double s8 = 1.0 / (8.0 * kPi), s4 = 1.0 / (4.0 * kPi);
      const double kxv = kval(kx, N, a.kscale[0]), kyv = kval(ky, a.py, a.kscale[1]), kzv = kval(kz, a.pz, a.kscale[2]);
      const double k2 = kxv * kxv + kyv * kyv + kzv * kzv;
      const double E = exp(-a.ka * k2);
      const double G = (KIND == HS_ROTLET) ? tH * E * s4 * a.inv_n : tB * E * (1.0 + a.kb * k2) * s8 * a.inv_n;
      const double Fc = HALF ? tH * E * s4 * a.inv_n : 0.0;
      apply_multiplier<KIND, HALF>(kxv, kyv, kzv, G, Fc, C, outc);
#pragma unroll
      for (int o = 0; o < NOUT; ++o) col[o * LSR] = make_double2(outc[o].re, -outc[o].im);
    }
    __syncthreads();
    for (int o = warp; o < NOUT; o += NW) {
      double2 v[X750_M];
      double2* S = lines + o * LSR;
#pragma unroll
      for (int j = 0; j < X750_M; ++j) v[j] = lane < X750_L ? S[lane + X750_L * j] : make_double2(0.0, 0.0);
      warp_fft750(v, S, tw, lane);
      double2* dst = a.Bout + o * a.ch_stride + (int64_t)ky * a.nx * a.nzh + kzl;
      for (int x = lane; x < a.nx; x += 32) {
        const double2 w = S[x];
        xstore(a, &dst[(int64_t)x * a.nzh], make_double2(w.x, -w.y));
      }
    }
  }
}

template <int KIND, bool HALF>
static hs_status launch_x750_t(hs_ctx* ctx, const XArgs& a) {
  HS_TRY(xreg_constants());
  constexpr int NL = KChan<KIND, HALF>::NIN > KChan<KIND, HALF>::NOUT ? KChan<KIND, HALF>::NIN : KChan<KIND, HALF>::NOUT;
  const size_t smem = sizeof(double2) * ((size_t)NL * X750_LS + padded_line(750));
  auto kern = k_x750<KIND, HALF>;
  HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, XF_THREADS, smem));
  const int items = a.py * a.nzh;
  const int grid = std::max(1, std::min(items, ctx->sm_count * std::max(per_sm, 1) * 8));
  kern<<<grid, XF_THREADS, smem, ctx->stream>>>(a);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

template <int KIND, bool HALF, int M>
static hs_status launch_xreg_t(hs_ctx* ctx, const XArgs& a) {
  HS_TRY(xreg_constants());
  constexpr int NL = KChan<KIND, HALF>::NIN > KChan<KIND, HALF>::NOUT ? KChan<KIND, HALF>::NIN : KChan<KIND, HALF>::NOUT;
  const size_t smem0 = sizeof(double2) * ((size_t)NL * M * 33 + padded_line(32 * M));
  const size_t smem1 = smem0 + sizeof(double2) * (size_t)KChan<KIND, HALF>::NIN * a.nx + sizeof(double) * 2 * 32 * M;
  // staging only if the kernel keeps its CTAs per SM (2, or 1 for M = 27) and HS_XSTAGE_NOSTAGE unset
  static const bool nostage = getenv("HS_XSTAGE_NOSTAGE") != nullptr;
  const size_t budget = (M == 27 ? 227 : 113) * 1024;
  const bool use_stage = !nostage && smem1 <= budget;
  const size_t smem = use_stage ? smem1 : smem0;
  auto kern = use_stage ? k_xreg<KIND, HALF, M, true> : k_xreg<KIND, HALF, M, false>;
  HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, XR_THREADS, smem));
  const int items = a.py * a.nzh;
  const int grid = std::max(1, std::min(items, ctx->sm_count * std::max(per_sm, 1) * 8));
  kern<<<grid, XR_THREADS, smem, ctx->stream>>>(a);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

// ---- y stage (N = 32 M) with the register FFT ----------------------------------------------
// Lines along y of the [y][x][kz] channel layout: a CTA takes one x and 8 consecutive kz
// (one warp per kz line); rows of 8 kz (128 contiguous bytes) are staged through shared
// memory with cp.async (coalesced), each warp transforms its column in registers
// (warp_fft_reg), and the results leave through shared memory as coalesced rows again.
// Forward: only the ny nonzero input rows are read (input pruning).  Inverse
// (unnormalised, by conjugation): only the ny output rows that the z stage needs are
// written (output pruning); in place.
constexpr int YS_KB = 8, YS_RS = YS_KB + 1;  // kz per CTA, padded row length (bank spread)

#ifndef YS_INV_PREFETCH
#define YS_INV_PREFETCH 0
#endif
// PRE: the next item's input rows are prefetched into a separate staging area (always for the
// forward transform, whose ny input rows fit next to the row buffer at two CTAs per SM; for the
// inverse, all py rows, only with YS_INV_PREFETCH=1 at one CTA per SM)
template <int M, bool FWD>
__global__ void __launch_bounds__(256, (M == 27 || (!FWD && YS_INV_PREFETCH)) ? 1 : 2)
    k_ystage(const double2* __restrict__ in, double2* __restrict__ out, const double2* __restrict__ twg, int nx,
             int nzh, int ny) {
  constexpr bool PRE = FWD || YS_INV_PREFETCH;
  constexpr int N = 32 * M;
  extern __shared__ double2 smem[];
  double2* buf = smem;              // [N rows][YS_RS]; later per-warp transpose scratch (8 x M*33)
  double2* tw = smem + N * YS_RS;   // pd8-padded twiddles
  static_assert(8 * M * 33 <= N * YS_RS, "scratch fits the row buffer");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < N; i += blockDim.x) tw[pd8(i)] = twg[i];
  const int nkb = (nzh + YS_KB - 1) / YS_KB;
  const int n_items = nx * nkb;
  const int rows_in = FWD ? ny : N, rows_out = FWD ? N : ny;
  const int64_t rstride = (int64_t)nx * nzh;  // elements between rows (y)
  const int r = lane >> 1, h = lane & 1;
  // forward: the next item's ny input rows are prefetched into a separate staging area (pre)
  // while the current item is transformed and written (the inverse reads all N rows; its
  // staging would not fit two CTAs per SM)
  double2* pre = tw + padded_line(N);  // [rows_in][YS_RS] (PRE)
  auto load_rows = [&](int it, double2* dst) {
    if (it < n_items) {
      const int x2 = it / nkb, k02 = (it - x2 * nkb) * YS_KB;
      const int kb2 = min(YS_KB, nzh - k02);
      const int64_t b2 = (int64_t)x2 * nzh + k02;
      for (int i = tid; i < rows_in * YS_KB; i += blockDim.x) {
        const int row = i / YS_KB, k = i - row * YS_KB;
        if (k < kb2) cp_async16(&dst[row * YS_RS + k], in + b2 + row * rstride + k);
      }
    }
    cp_async_commit();
  };
  if (PRE) load_rows(blockIdx.x, pre);
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int x = item / nkb, kz0 = (item - x * nkb) * YS_KB;
    const int kbn = min(YS_KB, nzh - kz0);
    const int64_t base = (int64_t)x * nzh + kz0;
    __syncthreads();  // previous item done with buf
    if (!PRE) load_rows(item, buf);
    cp_async_wait_all();
    __syncthreads();
    const double2* src = PRE ? pre : buf;
    double2 v[M], o16[RegFFT<M>::NG][16];
#pragma unroll
    for (int j = 0; j < M; ++j) {
      const int row = lane + 32 * j;
      double2 e = row < rows_in ? src[row * YS_RS + warp] : make_double2(0.0, 0.0);
      if (!FWD) e.y = -e.y;
      v[j] = e;
    }
    __syncthreads();  // every column read: the buffer becomes transpose scratch
    if (PRE) load_rows(item + gridDim.x, pre);
    warp_fft_reg<M>(v, buf + warp * M * 33, tw, lane, o16);
    __syncthreads();  // scratch use finished: the buffer collects the output rows
#pragma unroll
    for (int g = 0; g < RegFFT<M>::NG; ++g) {
      const int rg = r + 16 * g;
      if (rg < M) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          const int row = rg + M * (k + 16 * h);
          double2 e = o16[g][k];
          if (!FWD) e.y = -e.y;
          if (row < rows_out) buf[row * YS_RS + warp] = e;
        }
      }
    }
    __syncthreads();
    for (int i = tid; i < rows_out * YS_KB; i += blockDim.x) {
      const int row = i / YS_KB, k = i - row * YS_KB;
      if (k < kbn) out[base + row * rstride + k] = buf[row * YS_RS + k];
    }
  }
}

// y stage for 750-point lines (cfg4): same row staging as k_ystage, the column FFT by
// warp_fft750 (its natural-order result is read back from the warp's scratch into registers
// before the buffer collects the output rows)
template <bool FWD>
__global__ void __launch_bounds__(256, 1) k_ystage750(const double2* __restrict__ in, double2* __restrict__ out,
                                                      const double2* __restrict__ twg, int nx, int nzh, int ny) {
  constexpr int N = 750, NR = (N + 31) / 32;
  extern __shared__ double2 smem[];
  double2* buf = smem;             // [N rows][YS_RS]; later per-warp FFT scratch (8 x X750_LS)
  double2* tw = smem + N * YS_RS;  // pd8-padded twiddles
  static_assert(8 * X750_LS <= N * YS_RS, "scratch fits the row buffer");
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < N; i += blockDim.x) tw[pd8(i)] = twg[i];
  const int nkb = (nzh + YS_KB - 1) / YS_KB;
  const int n_items = nx * nkb;
  const int rows_in = FWD ? ny : N, rows_out = FWD ? N : ny;
  const int64_t rstride = (int64_t)nx * nzh;
  double2* pre = tw + padded_line(N);  // [ny][YS_RS] (FWD)
  auto load_rows = [&](int it, double2* dst) {
    if (it < n_items) {
      const int x2 = it / nkb, k02 = (it - x2 * nkb) * YS_KB;
      const int kb2 = min(YS_KB, nzh - k02);
      const int64_t b2 = (int64_t)x2 * nzh + k02;
      for (int i = tid; i < rows_in * YS_KB; i += blockDim.x) {
        const int row = i / YS_KB, k = i - row * YS_KB;
        if (k < kb2) cp_async16(&dst[row * YS_RS + k], in + b2 + row * rstride + k);
      }
    }
    cp_async_commit();
  };
  if (FWD) load_rows(blockIdx.x, pre);
  for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
    const int x = item / nkb, kz0 = (item - x * nkb) * YS_KB;
    const int kbn = min(YS_KB, nzh - kz0);
    const int64_t base = (int64_t)x * nzh + kz0;
    __syncthreads();
    if (!FWD) load_rows(item, buf);
    cp_async_wait_all();
    __syncthreads();
    const double2* src = FWD ? pre : buf;
    double2 v[X750_M];
#pragma unroll
    for (int j = 0; j < X750_M; ++j) {
      const int row = lane + X750_L * j;
      double2 e = (lane < X750_L && row < rows_in) ? src[row * YS_RS + warp] : make_double2(0.0, 0.0);
      if (!FWD) e.y = -e.y;
      v[j] = e;
    }
    __syncthreads();  // every column read: the buffer becomes FFT scratch
    if (FWD) load_rows(item + gridDim.x, pre);
    double2* S = buf + warp * X750_LS;
    warp_fft750(v, S, tw, lane);
    double2 res[NR];
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int k = lane + 32 * i;
      res[i] = k < N ? S[k] : make_double2(0.0, 0.0);
    }
    __syncthreads();  // scratch use finished: the buffer collects the output rows
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int row = lane + 32 * i;
      double2 e = res[i];
      if (!FWD) e.y = -e.y;
      if (row < rows_out) buf[row * YS_RS + warp] = e;
    }
    __syncthreads();
    for (int i = tid; i < rows_out * YS_KB; i += blockDim.x) {
      const int row = i / YS_KB, k = i - row * YS_KB;
      if (k < kbn) out[base + row * rstride + k] = buf[row * YS_RS + k];
    }
  }
}

// y stage of one channel; false when the length has no register kernel (caller uses cuFFT)
bool ystage_supported(int py) { return py == 480 || py == 352 || py == 864 || py == 750; }
hs_status launch_ystage(hs_ctx* ctx, bool fwd, const double2* in, double2* out, const double2* tw, int py, int nx,
                        int nzh, int ny) {
  HS_TRY(xreg_constants());
  auto go = [&](auto kern, int M) -> hs_status {
    const size_t smem = sizeof(double2) * ((size_t)32 * M * YS_RS + padded_line(32 * M) +
                                           (fwd ? (size_t)ny * YS_RS
                                                : (YS_INV_PREFETCH ? (size_t)32 * M * YS_RS : 0)));  // prefetch rows
    HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int items = nx * ((nzh + YS_KB - 1) / YS_KB);
    const int grid = std::max(1, std::min(items, ctx->sm_count * 2 * 8));
    kern<<<grid, 256, smem, ctx->stream>>>(in, out, tw, nx, nzh, ny);
    HS_LAUNCHED(ctx);
    return HS_OK;
  };
  if (py == 480) return fwd ? go(k_ystage<15, true>, 15) : go(k_ystage<15, false>, 15);
  if (py == 352) return fwd ? go(k_ystage<11, true>, 11) : go(k_ystage<11, false>, 11);
  if (py == 864) return fwd ? go(k_ystage<27, true>, 27) : go(k_ystage<27, false>, 27);
  if (py == 750) {
    const size_t smem = sizeof(double2) * ((size_t)750 * YS_RS + padded_line(750) + (fwd ? (size_t)ny * YS_RS : 0));
    auto kern = fwd ? k_ystage750<true> : k_ystage750<false>;
    HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int items = nx * ((nzh + YS_KB - 1) / YS_KB);
    const int grid = std::max(1, std::min(items, ctx->sm_count * 8));
    kern<<<grid, 256, smem, ctx->stream>>>(in, out, tw, nx, nzh, ny);
    HS_LAUNCHED(ctx);
    return HS_OK;
  }
  return fail(HS_ERR_PARAMETER, "y stage: unsupported length");
}

// ---- register z stage for pz = 924 (the metric configuration) and 660 (cfg2 / cfg3) ---------
// A real line of pz = 2 N2 points is the N2-point complex transform of z[n] = x[2n] + i x[2n+1] plus
// one pass over (k, N2 - k) pairs.  N2 = 22 M (M = 21: 462; M = 15: 330): lanes l < 22 hold
// z[l + 22 j] (j < M), DFT-M (21 = 3 x 7; 15 = 3 x 5) over j in registers, twiddle W_N2^{l k1}, one
// transpose through shared memory (S[k1][l], rows of 23), then lanes r < M each take row r and
// finish with a DFT22 (= 2 x DFT11), ending with Z[r + M k2] in natural order in the warp's scratch.
//   forward (k_zfwd, replaces the cuFFT D2Z): one warp per line; only the nonzero inputs are read
//     (the zero padding of the source grids is never touched), N2 + 1 outputs written; optionally
//     applies the half-space reflection while loading (plan.cu k_mirror_z);
//   inverse (k_zinv, replaces the cuFFT Z2D + k_interleave): a CTA takes LPC lines, one warp per
//     (line, output channel); only the z < nz outputs are formed and they leave channel-interleaved
//     ([z][pitch], one contiguous block per line) for the gather.
// Unnormalised both ways, like cuFFT; the inverse ignores the imaginary parts of the k = 0 and
// Nyquist entries (Z2D semantics).
__constant__ double2 c_w7[7];   // exp(-2 pi i m / 7)
__constant__ double2 c_w21[21];  // exp(-2 pi i m / 21)
__constant__ double2 c_w22[11];  // exp(-2 pi i m / 22)
__constant__ double2 c_w24[24];  // exp(-2 pi i m / 24)
__constant__ double2 c_w28[28];  // exp(-2 pi i m / 28)
static bool g_z924_consts = false;
static hs_status z924_constants() {
  HS_TRY(xreg_constants());  // c_w11
  if (g_z924_consts) return HS_OK;
  const long double tp = 6.283185307179586476925286766559005768L;
  double2 w7[7], w21[21], w22[11], w24[24], w28[28];
  for (int m = 0; m < 24; ++m) w24[m] = make_double2((double)std::cos(tp * m / 24), (double)-std::sin(tp * m / 24));
  for (int m = 0; m < 28; ++m) w28[m] = make_double2((double)std::cos(tp * m / 28), (double)-std::sin(tp * m / 28));
  for (int m = 0; m < 7; ++m) w7[m] = make_double2((double)std::cos(tp * m / 7), (double)-std::sin(tp * m / 7));
  for (int m = 0; m < 21; ++m) w21[m] = make_double2((double)std::cos(tp * m / 21), (double)-std::sin(tp * m / 21));
  for (int m = 0; m < 11; ++m) w22[m] = make_double2((double)std::cos(tp * m / 22), (double)-std::sin(tp * m / 22));
  HS_CUDA(cudaMemcpyToSymbol(c_w7, w7, sizeof(w7)));
  HS_CUDA(cudaMemcpyToSymbol(c_w21, w21, sizeof(w21)));
  HS_CUDA(cudaMemcpyToSymbol(c_w22, w22, sizeof(w22)));
  HS_CUDA(cudaMemcpyToSymbol(c_w24, w24, sizeof(w24)));
  HS_CUDA(cudaMemcpyToSymbol(c_w28, w28, sizeof(w28)));
  g_z924_consts = true;
  return HS_OK;
}

// DFT-7 in place (direct, symmetric pairs: 3 cos/sin pairs per output)
__device__ __forceinline__ void dft7(double2* v) {
  double2 sp[3], sm[3];
#pragma unroll
  for (int m = 1; m <= 3; ++m) {
    sp[m - 1] = ad(v[m], v[7 - m]);
    sm[m - 1] = sb(v[m], v[7 - m]);
  }
  double2 y[7];
  y[0] = ad(ad(v[0], sp[0]), ad(sp[1], sp[2]));
#pragma unroll
  for (int k = 1; k <= 3; ++k) {
    double2 re = v[0], im = make_double2(0.0, 0.0);
#pragma unroll
    for (int m = 1; m <= 3; ++m) {
      const double2 w = c_w7[(m * k) % 7];  // (cos, -sin)
      re = make_double2(fma(w.x, sp[m - 1].x, re.x), fma(w.x, sp[m - 1].y, re.y));
      im = make_double2(fma(w.y, sm[m - 1].x, im.x), fma(w.y, sm[m - 1].y, im.y));
    }
    y[k] = make_double2(re.x - im.y, re.y + im.x);
    y[7 - k] = make_double2(re.x + im.y, re.y - im.x);
  }
#pragma unroll
  for (int k = 0; k < 7; ++k) v[k] = y[k];
}

// DFT-21 in place: j = j1 + 3 j2 (j2 < 7), k = 7 k1 + k2 (DFT7 over j2, twiddle W21^{j1 k2}, DFT3 over j1)
__device__ __forceinline__ void dft21(double2* v) {
  double2 Y[3][7];
#pragma unroll
  for (int j1 = 0; j1 < 3; ++j1) {
    double2 t[7];
#pragma unroll
    for (int j2 = 0; j2 < 7; ++j2) t[j2] = v[j1 + 3 * j2];
    dft7(t);
#pragma unroll
    for (int k2 = 0; k2 < 7; ++k2) Y[j1][k2] = (j1 * k2 == 0) ? t[k2] : cm(t[k2], c_w21[j1 * k2]);
  }
#pragma unroll
  for (int k2 = 0; k2 < 7; ++k2) {
    double2 t[3] = {Y[0][k2], Y[1][k2], Y[2][k2]};
    dft<3>(t);
#pragma unroll
    for (int k1 = 0; k1 < 3; ++k1) v[7 * k1 + k2] = t[k1];
  }
}

// DFT-24 in place: j = j1 + 3 j2 (j2 < 8), k = 8 k1 + k2 (DFT8 over j2, twiddle W24^{j1 k2}, DFT3 over j1)
__device__ __forceinline__ void dft24(double2* v) {
  double2 Y[3][8];
#pragma unroll
  for (int j1 = 0; j1 < 3; ++j1) {
    double2 t[8];
#pragma unroll
    for (int j2 = 0; j2 < 8; ++j2) t[j2] = v[j1 + 3 * j2];
    dft<8>(t);
#pragma unroll
    for (int k2 = 0; k2 < 8; ++k2) Y[j1][k2] = (j1 * k2 == 0) ? t[k2] : cm(t[k2], c_w24[j1 * k2]);
  }
#pragma unroll
  for (int k2 = 0; k2 < 8; ++k2) {
    double2 t[3] = {Y[0][k2], Y[1][k2], Y[2][k2]};
    dft<3>(t);
#pragma unroll
    for (int k1 = 0; k1 < 3; ++k1) v[8 * k1 + k2] = t[k1];
  }
}
// DFT-28 in place: j = j1 + 4 j2 (j2 < 7), k = 7 k1 + k2 (DFT7 over j2, twiddle W28^{j1 k2}, DFT4 over j1)
__device__ __forceinline__ void dft28(double2* v) {
  double2 Y[4][7];
#pragma unroll
  for (int j1 = 0; j1 < 4; ++j1) {
    double2 t[7];
#pragma unroll
    for (int j2 = 0; j2 < 7; ++j2) t[j2] = v[j1 + 4 * j2];
    dft7(t);
#pragma unroll
    for (int k2 = 0; k2 < 7; ++k2) Y[j1][k2] = (j1 * k2 == 0) ? t[k2] : cm(t[k2], c_w28[j1 * k2]);
  }
#pragma unroll
  for (int k2 = 0; k2 < 7; ++k2) {
    double2 t[4] = {Y[0][k2], Y[1][k2], Y[2][k2], Y[3][k2]};
    dft<4>(t);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) v[7 * k1 + k2] = t[k1];
  }
}

// geometry of the L x M scheme: N2 = L M complex points per line (pz = 2 N2 real points);
// L = 22 lanes for M = 21 (pz = 924, the metric configuration) and 15 (660: cfg2 / cfg3),
// L = 30 lanes for M = 7 (420: cfg1), 24 (1440: cfg4) and 28 (1680: cfg5)
template <int M>
struct ZR {
  static constexpr int L = (M == 21 || M == 15) ? 22 : 30, H = L / 2, RS = L + 1;
  static constexpr int N2 = L * M, LS = M * RS;                    // scratch LS >= N2
  static constexpr int NZH = N2 + 1, PZ = 2 * N2, KH = N2 / 2;    // KH: pairs (k, N2 - k), k <= KH
  static constexpr int NQ = (KH + 32) / 32;                        // lane rounds over k <= KH
};
template <int M>
__device__ __forceinline__ void dftZ(double2* v) {
  static_assert(M == 21 || M == 15 || M == 7 || M == 24 || M == 28, "register z stage: M in {21, 15, 7, 24, 28}");
  if constexpr (M == 21) dft21(v);
  else if constexpr (M == 15) dft15(v);
  else if constexpr (M == 7) dft7(v);
  else if constexpr (M == 24) dft24(v);
  else dft28(v);
}
// forward DFT of the L M-point line with z[l + L j] in v[j] (lanes < L); result Z[k] left in S[k].
// ALL: every output (false: only Z[k], k < N2 / 2, i.e. the first half of each row's DFT-L)
template <int M, bool ALL>
__device__ __forceinline__ void warp_fftz(double2* v, double2* S, const double2* tw, int lane) {
  constexpr int L = ZR<M>::L, H = ZR<M>::H, RS = ZR<M>::RS;
  if (lane < L) {
    dftZ<M>(v);
#pragma unroll
    for (int k1 = 1; k1 < M; ++k1) v[k1] = cm(v[k1], tw[pd8(lane * k1)]);
  }
  __syncwarp();
  if (lane < L) {
#pragma unroll
    for (int k1 = 0; k1 < M; ++k1) S[k1 * RS + lane] = v[k1];
  }
  __syncwarp();
  // DFT-L of row r = lane as 2 x DFT-(L/2) (even / odd l)
  double2 e[H], o[H];
  const int rr = lane < M ? lane : M - 1;
#pragma unroll
  for (int m = 0; m < H; ++m) {
    e[m] = S[rr * RS + 2 * m];
    o[m] = S[rr * RS + 2 * m + 1];
  }
  __syncwarp();
  if constexpr (H == 11) {
    dft11(e);
    dft11(o);
  } else {
    dft15(e);
    dft15(o);
  }
  if (lane < M) {
#pragma unroll
    for (int k = 0; k < H; ++k) {
      const double2 w = H == 11 ? c_w22[k] : c_w30[k];
      const double2 t = k == 0 ? o[0] : cm(o[k], w);
      S[lane + M * k] = ad(e[k], t);
      if (ALL) S[lane + M * (k + H)] = sb(e[k], t);
    }
  }
  __syncwarp();
}

constexpr int ZF_WARPS = 8;
template <int M>
__global__ void __launch_bounds__(ZF_WARPS * 32, 1)
    k_zfwd(const double* __restrict__ in, double2* __restrict__ out, const double2* __restrict__ twg, int64_t nlines,
              int nz, int mirror, double msign, int n0) {
  constexpr int Z9_N2 = ZR<M>::N2, Z9_L = ZR<M>::L, Z9_M = M, Z9_LS = ZR<M>::LS, Z9_NZH = ZR<M>::NZH, Z9_PZ = ZR<M>::PZ,
                ZF_STAGE = ZR<M>::KH, KH = ZR<M>::KH;
  extern __shared__ double2 smem[];
  double2* tw = smem;                               // pd8-padded W_N2^i
  double2* twh = tw + padded_line(Z9_N2);           // W_pz^k, k <= KH
  double2* S = twh + KH + 1 + (threadIdx.x >> 5) * Z9_LS;
  // the warp's next line is prefetched (cp.async) into its staging row while the current one
  // is transformed, so the loads of one line overlap the arithmetic of the previous
  double2* stage = twh + KH + 1 + ZF_WARPS * Z9_LS + (threadIdx.x >> 5) * ZF_STAGE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < Z9_N2; i += blockDim.x) tw[pd8(i)] = twg[i];
  for (int i = threadIdx.x; i <= KH; i += blockDim.x) twh[i] = twg[Z9_N2 + i];
  __syncthreads();
  const int nc = (nz + 1) >> 1;  // nonzero complex inputs (nz <= 432 -> <= 216 -> j <= 9)
  const int64_t lstep = (int64_t)gridDim.x * ZF_WARPS;
  auto prefetch = [&](int64_t line) {
    if (line < nlines) {
      const double2* src = reinterpret_cast<const double2*>(in + line * Z9_PZ);
      for (int n = n0 + lane; n < nc; n += 32) cp_async16(&stage[n], &src[n]);
    }
    cp_async_commit();
  };
  // complex inputs below n0 are known zeros (never written by the spread): not loaded
  for (int n = lane; n < n0; n += 32) stage[n] = make_double2(0.0, 0.0);
  int64_t line = (int64_t)blockIdx.x * ZF_WARPS + warp;
  prefetch(line);
  for (; line < nlines; line += lstep) {
    cp_async_wait_all();
    __syncwarp();
    double2 v[Z9_M];
#pragma unroll
    for (int j = 0; j < Z9_M; ++j) {
      v[j] = make_double2(0.0, 0.0);
      if (Z9_L * j < KH) {
        const int n = lane + Z9_L * j;
        if (lane < Z9_L && n < nc) {
          if (mirror == 0) {
            v[j] = stage[n];
          } else {
            // mirrored spreading fused in (plan.cu k_mirror_z): node k of the transformed line is
            // S[k] + msign S[nz - k] (kernel channels, mirror = 1) or S[nz - k] (wall channels,
            // mirror = 2); the mirror of node 0 lies outside the grid (0).  nz even here.
            const double* sd = reinterpret_cast<const double*>(stage);
            const int k0 = 2 * n, k1 = 2 * n + 1;
            const double a0 = sd[k0], a1 = sd[k1];
            const double b0 = k0 == 0 ? 0.0 : sd[nz - k0], b1 = sd[nz - k1];
            v[j] = mirror == 1 ? make_double2(fma(msign, b0, a0), fma(msign, b1, a1)) : make_double2(b0, b1);
          }
          if (2 * n + 1 >= nz) v[j].y = 0.0;  // odd nz: the last pair's second entry is padding
        }
      }
    }
    __syncwarp();
    prefetch(line + lstep);
    warp_fftz<M, true>(v, S, tw, lane);
    // X[k] = E + W_pz^k O, X[N2 - k] = conj(E - W_pz^k O); E = (Z[k] + conj Z[N2-k]) / 2,
    // O = (Z[k] - conj Z[N2-k]) / (2 i)
    double2* dst = out + line * Z9_NZH;
#pragma unroll
    for (int q = 0; q < ZR<M>::NQ; ++q) {
      const int k = lane + 32 * q;
      if (k <= KH) {
        const double2 zk = S[k], zm = S[k == 0 ? 0 : Z9_N2 - k];
        const double2 E = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
        const double2 O = make_double2(0.5 * (zk.y + zm.y), -0.5 * (zk.x - zm.x));
        const double2 t = cm(O, twh[k]);
        dst[k] = ad(E, t);
        const double2 m = sb(E, t);
        dst[Z9_N2 - k] = make_double2(m.x, -m.y);
      }
    }
    __syncwarp();
  }
  cp_async_wait_all();
}

// LPC lines per CTA, NOUT channels: warp w -> (line w / NOUT, channel w % NOUT)
template <int M, int NOUT, int PITCH, int LPC>
__global__ void __launch_bounds__(NOUT * LPC * 32, 1)
    k_zinv(const double2* __restrict__ spec, int64_t ch_stride, double* __restrict__ gout,
              const double2* __restrict__ twg, int64_t nlines, int nz) {
  constexpr int Z9_N2 = ZR<M>::N2, Z9_L = ZR<M>::L, Z9_M = M, Z9_LS = ZR<M>::LS, Z9_NZH = ZR<M>::NZH, Z9_PZ = ZR<M>::PZ,
                KH = ZR<M>::KH;
  extern __shared__ double2 smem[];
  constexpr int NW = NOUT * LPC;
  double2* tw = smem;
  double2* twh = tw + padded_line(Z9_N2);
  double2* S = twh + KH + 1 + (threadIdx.x >> 5) * Z9_LS;
  double* obuf = reinterpret_cast<double*>(twh + KH + 1 + NW * Z9_LS);  // [LPC][nz][PITCH]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lc = warp / NOUT, c = warp - lc * NOUT;
  for (int i = threadIdx.x; i < Z9_N2; i += blockDim.x) tw[pd8(i)] = twg[i];
  for (int i = threadIdx.x; i <= KH; i += blockDim.x) twh[i] = twg[Z9_N2 + i];
  if (PITCH > NOUT)
    for (int i = threadIdx.x; i < LPC * nz * PITCH; i += blockDim.x) obuf[i] = 0.0;  // padding channels stay 0
  __syncthreads();
  const int nc = (nz + 1) >> 1;
  for (int64_t l0 = (int64_t)blockIdx.x * LPC; l0 < nlines; l0 += (int64_t)gridDim.x * LPC) {
    const int64_t line = l0 + lc;
    if (line < nlines) {
      const double2* X = spec + (int64_t)c * ch_stride + line * Z9_NZH;
      // conj(Z[k]), Z[k] = E[k] + i O[k], E = X[k] + conj X[N2-k], O = (X[k] - conj X[N2-k]) conj(W_pz^k);
      // Z[N2-k] = conj E + i conj O
#pragma unroll
      for (int q = 0; q < ZR<M>::NQ; ++q) {
        const int k = lane + 32 * q;
        if (k <= KH) {
          double2 xk = X[k], xm = X[Z9_N2 - k];
          if (k == 0) xk.y = xm.y = 0.0;
          const double2 E = make_double2(xk.x + xm.x, xk.y - xm.y);
          const double2 D = make_double2(xk.x - xm.x, xk.y + xm.y);
          const double2 w = twh[k];
          const double2 O = make_double2(fma(D.x, w.x, D.y * w.y), fma(D.y, w.x, -D.x * w.y));  // D conj(w)
          // Z[k] = (E.x - O.y, E.y + O.x): conj -> (E.x - O.y, -E.y - O.x)
          // Z[N2-k] = (E.x + O.y, -E.y + O.x): conj -> (E.x + O.y, E.y - O.x)
          if (k > 0) S[Z9_N2 - k] = make_double2(E.x + O.y, E.y - O.x);
          S[k] = make_double2(E.x - O.y, -E.y - O.x);
        }
      }
      __syncwarp();
      double2 v[Z9_M];
#pragma unroll
      for (int j = 0; j < Z9_M; ++j) v[j] = lane < Z9_L ? S[lane + Z9_L * j] : make_double2(0.0, 0.0);
      __syncwarp();
      warp_fftz<M, false>(v, S, tw, lane);  // z[n] = conj(S[n]), n < N2 / 2 >= nc
      double* ob = obuf + (size_t)lc * nz * PITCH + c;
#pragma unroll
      for (int q = 0; q < ZR<M>::NQ; ++q) {
        const int n = lane + 32 * q;
        if (n < nc) {
          const double2 f = S[n];
          ob[(2 * n) * PITCH] = f.x;
          if (2 * n + 1 < nz) ob[(2 * n + 1) * PITCH] = -f.y;
        }
      }
    }
    __syncthreads();
    // one contiguous [nz][PITCH] block per line
    const int per = nz * PITCH / 2;  // double2 per line (nz * PITCH even)
    for (int i = threadIdx.x; i < LPC * per; i += blockDim.x) {
      const int ll = i / per, r = i - ll * per;
      if (l0 + ll < nlines)
        reinterpret_cast<double2*>(gout + (l0 + ll) * (int64_t)PITCH * Z9_PZ)[r] =
            reinterpret_cast<const double2*>(obuf + (size_t)ll * nz * PITCH)[r];
    }
    __syncthreads();
  }
}

// (pz, nz) the register z stage handles: nz even, at most half the padded length
static int zstage_m(int pz) {
  switch (pz) {
    case ZR<21>::PZ: return 21;
    case ZR<15>::PZ: return 15;
    case ZR<7>::PZ: return 7;
    case ZR<24>::PZ: return 24;
    case ZR<28>::PZ: return 28;
    default: return 0;
  }
}
bool zstage_supported(int pz, int nz) { return zstage_m(pz) != 0 && nz <= pz / 2 && nz % 2 == 0; }
// twiddle table of the z stage: W_{N2}^i (N2 = pz / 2 entries) then W_{pz}^k (k <= N2 / 2)
int zstage_twiddle_count(int pz) { return pz / 2 + pz / 4 + 1; }
hs_status make_zstage_twiddles(int pz, double2* d_tw, cudaStream_t st) {
  const int n2 = pz / 2, kh = n2 / 2;
  std::vector<double2> tw(n2 + kh + 1);
  const long double tp = 6.283185307179586476925286766559005768L;
  for (int j = 0; j < n2; ++j) tw[j] = make_double2((double)std::cos(tp * j / n2), (double)-std::sin(tp * j / n2));
  for (int j = 0; j <= kh; ++j) tw[n2 + j] = make_double2((double)std::cos(tp * j / pz), (double)-std::sin(tp * j / pz));
  HS_CUDA(cudaMemcpyAsync(d_tw, tw.data(), sizeof(double2) * tw.size(), cudaMemcpyHostToDevice, st));
  HS_CUDA(cudaStreamSynchronize(st));
  return HS_OK;
}
// forward z of one channel: lines of pitch pz (nz nonzero values) -> nzh = pz / 2 + 1 spectrum entries
// mirror: 0 plain; 1 / 2: the half-space reflection of a kernel / wall channel applied while
// loading (nz even), msign = the kernel channel's image sign
// zero_below: nodes k < zero_below of every line are known to be zero and are not read
template <int M>
static hs_status launch_zfwd_t(hs_ctx* ctx, const double* in, double2* out, const double2* tw, int64_t nlines, int nz,
                               int mirror, double msign, int zero_below) {
  const size_t smem = sizeof(double2) * (padded_line(ZR<M>::N2) + ZR<M>::KH + 1 + (size_t)ZF_WARPS * (ZR<M>::LS + ZR<M>::KH));
  HS_CUDA(cudaFuncSetAttribute(k_zfwd<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 1;
  HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_zfwd<M>, ZF_WARPS * 32, smem));
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nlines, ZF_WARPS),
                                                               (int64_t)ctx->sm_count * std::max(per_sm, 1)));
  k_zfwd<M><<<grid, ZF_WARPS * 32, smem, ctx->stream>>>(in, out, tw, nlines, nz, mirror, msign,
                                                         std::max(0, std::min(zero_below, nz)) / 2);
  HS_LAUNCHED(ctx);
  return HS_OK;
}
hs_status launch_zfwd(hs_ctx* ctx, int pz, const double* in, double2* out, const double2* tw, int64_t nlines, int nz,
                      int mirror, double msign, int zero_below) {
  if (!zstage_supported(pz, nz)) return fail(HS_ERR_PARAMETER, "z stage: unsupported length");
  if (mirror && (nz & 1)) return fail(HS_ERR_PARAMETER, "z stage: fused mirror needs an even nz");
  HS_TRY(z924_constants());
  switch (zstage_m(pz)) {
    case 21: return launch_zfwd_t<21>(ctx, in, out, tw, nlines, nz, mirror, msign, zero_below);
    case 15: return launch_zfwd_t<15>(ctx, in, out, tw, nlines, nz, mirror, msign, zero_below);
    case 7: return launch_zfwd_t<7>(ctx, in, out, tw, nlines, nz, mirror, msign, zero_below);
    case 24: return launch_zfwd_t<24>(ctx, in, out, tw, nlines, nz, mirror, msign, zero_below);
    default: return launch_zfwd_t<28>(ctx, in, out, tw, nlines, nz, mirror, msign, zero_below);
  }
}
// inverse z of all n_out channels (channel stride ch_stride in `spec`), outputs z < nz interleaved
// into gout ([line][pz][pitch] storage, z < nz written)
template <int M>
static hs_status launch_zinv_t(hs_ctx* ctx, const double2* spec, int64_t ch_stride, int n_out, int pitch, double* gout,
                               const double2* tw, int64_t nlines, int nz) {
  auto go = [&](auto kern, int nw, int lpc) -> hs_status {
    const size_t smem = sizeof(double2) * (padded_line(ZR<M>::N2) + ZR<M>::KH + 1 + (size_t)nw * ZR<M>::LS) +
                        sizeof(double) * (size_t)lpc * nz * pitch;
    HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, nw * 32, smem));
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nlines, lpc),
                                                                 (int64_t)ctx->sm_count * std::max(per_sm, 1)));
    kern<<<grid, nw * 32, smem, ctx->stream>>>(spec, ch_stride, gout, tw, nlines, nz);
    HS_LAUNCHED(ctx);
    return HS_OK;
  };
  // 12 warps per CTA; 6 for the long lines (M >= 24: 28 complex registers per lane need the
  // 255-register budget of a 192-thread CTA)
  constexpr int NW = M >= 24 ? 6 : 12;
  if (n_out == 6 && pitch == 6) return go(k_zinv<M, 6, 6, NW / 6>, NW, NW / 6);
  if (n_out == 3 && pitch == 4) return go(k_zinv<M, 3, 4, NW / 3>, NW, NW / 3);
  if (n_out == 1 && pitch == 1) return go(k_zinv<M, 1, 1, NW>, NW, NW);  // one channel, not interleaved
  return fail(HS_ERR_PARAMETER, "z stage: unsupported channel layout");
}
hs_status launch_zinv_interleaved(hs_ctx* ctx, int pz, const double2* spec, int64_t ch_stride, int n_out, int pitch,
                                  double* gout, const double2* tw, int64_t nlines, int nz) {
  if (!zstage_supported(pz, nz)) return fail(HS_ERR_PARAMETER, "z stage: unsupported length");
  HS_TRY(z924_constants());
  switch (zstage_m(pz)) {
    case 21: return launch_zinv_t<21>(ctx, spec, ch_stride, n_out, pitch, gout, tw, nlines, nz);
    case 15: return launch_zinv_t<15>(ctx, spec, ch_stride, n_out, pitch, gout, tw, nlines, nz);
    case 7: return launch_zinv_t<7>(ctx, spec, ch_stride, n_out, pitch, gout, tw, nlines, nz);
    case 24: return launch_zinv_t<24>(ctx, spec, ch_stride, n_out, pitch, gout, tw, nlines, nz);
    default: return launch_zinv_t<28>(ctx, spec, ch_stride, n_out, pitch, gout, tw, nlines, nz);
  }
}

template <int KIND, bool HALF, int KB, class FFT>
static hs_status launch_xfused_t(hs_ctx* ctx, const XArgs& a) {
  constexpr int NL = KChan<KIND, HALF>::NIN > KChan<KIND, HALF>::NOUT ? KChan<KIND, HALF>::NIN
                                                                       : KChan<KIND, HALF>::NOUT;
  const size_t smem = sizeof(double2) * ((size_t)NL * KB * padded_line(a.plan.n) + a.plan.n);
  if (smem > 227 * 1024) return fail(HS_ERR_PARAMETER, "x-stage shared memory exceeds 227 KB");
  auto kern = k_xfused<KIND, HALF, KB, FFT>;
  HS_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int per_sm = 0;
  HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, XF_THREADS, smem));
  const int nkb = (a.nzh + KB - 1) / KB;
  const int items = a.py * nkb;
  const int grid = std::max(1, std::min(items, ctx->sm_count * std::max(per_sm, 1) * 8));
  kern<<<grid, XF_THREADS, smem, ctx->stream>>>(a);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

// FFT-length specialisations for the BASELINE configurations (cfg1 240, cfg2/3 352,
// HL 480, cfg4 750, cfg5 864); any other 11-smooth length <= 1024 uses AnyFFT.
template <int KIND, bool HALF, int KB>
static hs_status launch_xfused_len(hs_ctx* ctx, const XArgs& a) {
  switch (a.plan.n) {
    case 240: return launch_xfused_t<KIND, HALF, KB, FixedFFT<8, 2, 3, 5>>(ctx, a);
    case 352: {
      static const bool stockham = getenv("HS_XSTAGE_STOCKHAM") != nullptr;
      if (!stockham) return launch_xreg_t<KIND, HALF, 11>(ctx, a);
      return launch_xfused_t<KIND, HALF, KB, FixedFFT<8, 4, 11>>(ctx, a);
    }
    case 480: {
      static const bool stockham = getenv("HS_XSTAGE_STOCKHAM") != nullptr;  // previous kernel (comparison)
      if (!stockham) return launch_xreg_t<KIND, HALF, 15>(ctx, a);
      return launch_xfused_t<KIND, HALF, KB, FixedFFT<8, 4, 3, 5>>(ctx, a);
    }
    case 750: {
      static const bool stockham = getenv("HS_XSTAGE_STOCKHAM") != nullptr;
      if (!stockham) return launch_x750_t<KIND, HALF>(ctx, a);
      return launch_xfused_t<KIND, HALF, KB, FixedFFT<2, 3, 5, 5, 5>>(ctx, a);
    }
    case 864: {
      static const bool stockham = getenv("HS_XSTAGE_STOCKHAM") != nullptr;
      if (!stockham) return launch_xreg_t<KIND, HALF, 27>(ctx, a);
      return launch_xfused_t<KIND, HALF, KB, FixedFFT<8, 4, 3, 3, 3>>(ctx, a);
    }
    default: return launch_xfused_t<KIND, HALF, KB, AnyFFT>(ctx, a);
  }
}

// kind HS_MIXED: the mixed plan's first channel group (kmult.cuh)
hs_status launch_xfused(hs_ctx* ctx, int kind, int half, const XArgs& a) {
  if (half) {
    if (kind == HS_STOKESLET) return launch_xfused_len<HS_STOKESLET, true, 1>(ctx, a);
    if (kind == HS_STRESSLET) return launch_xfused_len<HS_STRESSLET, true, 1>(ctx, a);
    if (kind == HS_MIXED) return launch_xfused_len<HS_MIXED, true, 1>(ctx, a);
    return launch_xfused_len<HS_ROTLET, true, 1>(ctx, a);
  }
  if (kind == HS_STOKESLET) return launch_xfused_len<HS_STOKESLET, false, 1>(ctx, a);
  if (kind == HS_STRESSLET) return launch_xfused_len<HS_STRESSLET, false, 1>(ctx, a);
  if (kind == HS_MIXED) return launch_xfused_len<HS_MIXED, false, 1>(ctx, a);
  return launch_xfused_len<HS_ROTLET, false, 1>(ctx, a);
}

// twiddles exp(-2 pi i j / n), computed in long double on the host
hs_status make_twiddles(int n, double2* d_tw, cudaStream_t st) {
  std::vector<double2> tw(n);
  for (int j = 0; j < n; ++j) {
    const long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)j / (long double)n;
    tw[j] = make_double2((double)std::cos(ang), (double)std::sin(ang));
  }
  HS_CUDA(cudaMemcpyAsync(d_tw, tw.data(), sizeof(double2) * n, cudaMemcpyHostToDevice, st));
  HS_CUDA(cudaStreamSynchronize(st));
  return HS_OK;
}

// half-spectrum table [kx][ky][kz] -> x-stage layout [ky][kz - kz0][kx], kz in [kz0, kz0 + nzl)
__global__ void k_table_to_xmajor(const double* __restrict__ in, int px, int py, int nzh, int kz0, int nzl,
                                  double* __restrict__ out) {
  const int64_t n = (int64_t)px * py * nzl;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int kx = (int)(i % px);
    const int64_t r = i / px;
    const int kzl = (int)(r % nzl), ky = (int)(r / nzl);
    out[i] = in[((int64_t)kx * py + ky) * nzh + kz0 + kzl];
  }
}

hs_status launch_table_to_xmajor(hs_ctx* ctx, const double* in, int px, int py, int nzh, double* out, int kz0,
                                 int nzl) {
  if (nzl < 0) nzl = nzh - kz0;
  if (kz0 < 0 || kz0 + nzl > nzh) return fail(HS_ERR_PARAMETER, "table kz slice out of range");
  const int64_t n = (int64_t)px * py * nzl;
  if (n == 0) return HS_OK;
  const int gs = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->sm_count * 16);
  k_table_to_xmajor<<<gs, 256, 0, ctx->stream>>>(in, px, py, nzh, kz0, nzl, out);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

HS_DEFINE_CHECK_COLLECT(fft)

}  // namespace hs

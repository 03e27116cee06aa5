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
#include "common.cuh"
#include "kernels.cuh"

namespace hs {

constexpr int PT_WARPS = 8;
constexpr int PT_G = 4;      // targets per warp per pass
constexpr int PT_K = 256;    // candidates staged per chunk
constexpr int PT_Q = 64;     // queue capacity per (warp, target)
constexpr int PT_MAXRUN = 25;

struct PairConst {
  double xi, xi2, c2xs;  // xi, xi^2, 2 xi / sqrt(pi)
};

// Accumulate one pair.  d = x - y (target minus source), r2 = |d|^2 (> 0).
// k[0..2]: kernel part (raw), c[0..2]: wall correction (raw, 4 pi G convention).
template <int KIND, bool SCREENED>
__device__ __forceinline__ void eval_pair(const PairConst& pc, double d0, double d1, double d2, double r2,
                                          double x2, const double4& S, const double4& A, const double4& B,
                                          bool image, double* k, double* c) {
  const double rn = sqrt(r2);
  const double ri = 1.0 / rn;
  const double ri2 = ri * ri;
  double C = 1.0, e = 0.0;
  if (SCREENED) {
    const double E = exp(-pc.xi2 * r2);
    C = erfc(pc.xi * rn);
    e = pc.c2xs * E;
  }
  const double c0 = C * ri;
  const double c1 = (c0 + e) * ri2;
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

__device__ __forceinline__ double exact_r2(double d0, double d1, double d2) {
  // numba: r2 = d0 * d0 + d1 * d1 + d2 * d2, each op rounded, left to right
  return __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
}

template <int KIND, bool HALF>
__global__ void __launch_bounds__(PT_WARPS * 32) k_pair(const PairArgs a) {
  __shared__ double4 sP[PT_K];
  __shared__ double4 sA[PT_K];
  __shared__ double4 sB[PT_K];
  __shared__ unsigned short sq[PT_WARPS][PT_G][PT_Q];
  __shared__ int run_beg[PT_MAXRUN];
  __shared__ int run_pre[PT_MAXRUN + 1];
  __shared__ int s_nrun;
  constexpr bool kNeedB = (KIND == HS_STRESSLET) || (KIND == HS_ROTLET && HALF);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const unsigned lt_mask = (1u << lane) - 1u;
  const int nx = a.dims[0], ny = a.dims[1], nz = a.dims[2];
  PairConst pc;
  pc.xi = a.xi;
  pc.xi2 = a.xi * a.xi;
  pc.c2xs = 2.0 * a.xi / kSqrtPi;
  const double norm_k = (KIND == HS_ROTLET) ? 1.0 / (4.0 * kPi) : 1.0 / (8.0 * kPi);
  const double norm_c = 1.0 / (4.0 * kPi);

  const int n_cells = *a.n_cells_d;
  for (int cb = blockIdx.x; cb < n_cells; cb += gridDim.x) {
    const int cell = a.cells[cb];
    const int cz = cell % nz, cy = (cell / nz) % ny, cx = cell / (ny * nz);
    __syncthreads();
    if (threadIdx.x == 0) {
      int nr = 0, tot = 0;
      const int zlo = max(cz - 2, 0), zhi = min(cz + 2, nz - 1);
      for (int ix = max(cx - 2, 0); ix <= min(cx + 2, nx - 1); ++ix)
        for (int iy = max(cy - 2, 0); iy <= min(cy + 2, ny - 1); ++iy) {
          const int f = (ix * ny + iy) * nz;
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
    const int t_beg = a.t_start[cell];
    const int t_cnt = a.t_start[cell + 1] - t_beg;

    for (int tb = 0; tb < t_cnt; tb += PT_WARPS * PT_G) {
      double tx[PT_G], ty[PT_G], tz[PT_G];
      long long tcol[PT_G];
      bool tvalid[PT_G];
      double acc[PT_G][6];
      int qlen[PT_G];
#pragma unroll
      for (int g = 0; g < PT_G; ++g) {
        const int ti = tb + warp * PT_G + g;
        tvalid[g] = ti < t_cnt;
        const double4 t = a.TP[t_beg + (tvalid[g] ? ti : 0)];
        tx[g] = t.x;
        ty[g] = t.y;
        tz[g] = t.z;
        tcol[g] = (long long)t.w;
        qlen[g] = 0;
#pragma unroll
        for (int q = 0; q < 6; ++q) acc[g][q] = 0.0;
      }
      bool singular = false;
      unsigned long long n_acc = 0, n_img = 0;

      for (int c0 = 0; c0 < ncand; c0 += PT_K) {
        __syncthreads();
        {
          const int j = threadIdx.x;
          const int v = c0 + j;
          if (j < PT_K) {
            if (v < ncand) {
              int r = 0;
              while (r + 1 < nrun && run_pre[r + 1] <= v) ++r;
              const int row = run_beg[r] + (v - run_pre[r]);
              sP[j] = a.P[row];
              sA[j] = a.A[row];
              if (kNeedB) sB[j] = a.B[row];
            }
          }
        }
        __syncthreads();
        const int nc = min(PT_K, ncand - c0);
        for (int j0 = 0; j0 < nc; j0 += 32) {
          const int j = j0 + lane;
          const bool have = j < nc;
          const double4 s = sP[have ? j : 0];
          const long long sid = (long long)s.w;
#pragma unroll
          for (int g = 0; g < PT_G; ++g) {
            const double d0 = __dsub_rn(tx[g], s.x), d1 = __dsub_rn(ty[g], s.y), d2 = __dsub_rn(tz[g], s.z);
            const double r2 = exact_r2(d0, d1, d2);
            bool ok = have && tvalid[g] && sid != tcol[g] && r2 <= a.rc2;
            if (ok && r2 == 0.0) {
              singular = true;
              ok = false;
            }
            const unsigned m = __ballot_sync(0xffffffffu, ok);
            if (ok) sq[warp][g][qlen[g] + __popc(m & lt_mask)] = (unsigned short)j;
            qlen[g] += __popc(m);
            n_acc += __popc(m);
            if (HALF) n_img += __popc(m & __ballot_sync(0xffffffffu, ok && sid >= a.n_real));
            if (qlen[g] >= 32) {
              __syncwarp();
              const int jj = sq[warp][g][qlen[g] - 32 + lane];
              const double4 S = sP[jj];
              const double4 A = sA[jj];
              const double4 B = kNeedB ? sB[jj] : make_double4(0, 0, 0, 0);
              const double e0 = tx[g] - S.x, e1 = ty[g] - S.y, e2 = tz[g] - S.z;
              const double rr = exact_r2(e0, e1, e2);
              const bool img = HALF && ((long long)S.w >= a.n_real);
              eval_pair<KIND, true>(pc, e0, e1, e2, rr, tz[g], S, A, B, img, &acc[g][0], &acc[g][3]);
              qlen[g] -= 32;
              __syncwarp();
            }
          }
        }
        // flush the partial queues before the chunk is overwritten
#pragma unroll
        for (int g = 0; g < PT_G; ++g) {
          __syncwarp();
          if (lane < qlen[g]) {
            const int jj = sq[warp][g][lane];
            const double4 S = sP[jj];
            const double4 A = sA[jj];
            const double4 B = kNeedB ? sB[jj] : make_double4(0, 0, 0, 0);
            const double e0 = tx[g] - S.x, e1 = ty[g] - S.y, e2 = tz[g] - S.z;
            const double rr = exact_r2(e0, e1, e2);
            const bool img = HALF && ((long long)S.w >= a.n_real);
            eval_pair<KIND, true>(pc, e0, e1, e2, rr, tz[g], S, A, B, img, &acc[g][0], &acc[g][3]);
          }
          qlen[g] = 0;
        }
      }
      if (singular) atomicOr(a.flags, FLAG_SINGULAR);
      if (a.counts && lane == 0) {
        atomicAdd(&a.counts[0], n_acc);
        atomicAdd(&a.counts[1], n_img);
      }
#pragma unroll
      for (int g = 0; g < PT_G; ++g) {
        double r[6];
#pragma unroll
        for (int q = 0; q < 6; ++q) r[q] = warp_sum(acc[g][q]);
        if (lane == 0 && tvalid[g]) {
          const int ti = t_beg + tb + warp * PT_G + g;
          const int o = a.torig[ti];
          double u[3];
#pragma unroll
          for (int q = 0; q < 3; ++q) u[q] = r[q] * norm_k + r[3 + q] * norm_c;
          if (KIND == HS_STOKESLET && a.self_f != nullptr && tcol[g] >= 0 && tcol[g] < a.n_real) {
            // self term -(4 xi/sqrt(pi)) f / (8 pi)   (ewald_real.py:446-449)
            const double sc = -(4.0 * a.xi / kSqrtPi);
#pragma unroll
            for (int q = 0; q < 3; ++q) u[q] += sc * a.self_f[3 * tcol[g] + q] / (8.0 * kPi);
          }
#pragma unroll
          for (int q = 0; q < 3; ++q) a.u[3 * o + q] = u[q];
          if (a.uk) {
#pragma unroll
            for (int q = 0; q < 3; ++q) a.uk[3 * o + q] = r[q] * norm_k;
          }
          if (a.uc) {
#pragma unroll
            for (int q = 0; q < 3; ++q) a.uc[3 * o + q] = r[3 + q] * norm_c;
          }
        }
      }
    }
  }
}

hs_status launch_pair(hs_ctx* ctx, const PairArgs& a) {
  if (a.n_cells == 0) return HS_OK;
  const bool half = a.n_real >= 0;  // always true; geometry decided by B/P content
  (void)half;
  dim3 grid(a.n_cells), block(PT_WARPS * 32);
  // HALF is encoded by the caller through a.kind >= 16
  const int kind = a.kind & 15;
  const bool is_half = (a.kind & 16) != 0;
#define HS_PAIR_CASE(K, H) k_pair<K, H><<<grid, block, 0, ctx->stream>>>(a)
  if (is_half) {
    if (kind == HS_STOKESLET) HS_PAIR_CASE(HS_STOKESLET, true);
    else if (kind == HS_STRESSLET) HS_PAIR_CASE(HS_STRESSLET, true);
    else HS_PAIR_CASE(HS_ROTLET, true);
  } else {
    if (kind == HS_STOKESLET) HS_PAIR_CASE(HS_STOKESLET, false);
    else if (kind == HS_STRESSLET) HS_PAIR_CASE(HS_STRESSLET, false);
    else HS_PAIR_CASE(HS_ROTLET, false);
  }
#undef HS_PAIR_CASE
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
      eval_pair<KIND, false>(pc, d0, d1, d2, r2, T.z, S, sA[i], sB[i], img, k, c);
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

}  // namespace hs

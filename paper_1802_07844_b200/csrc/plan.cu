// plan.cu -- one evaluation of ewald.ewald_sum (reference: ewald.py:46-80) on the GPU.
//
// The plan owns all device buffers of one configuration and runs, stream-ordered:
//   real space:  cell keys of [y; y^I] -> stable counting sort -> cell-sorted
//                source records (reflect + wall channels fused) -> target cell
//                sort -> pair kernel (+ normalisation + stokeslet self term)
//   Fourier:     bin-sort kernel sources [y; y^I] and images y^I -> spread into
//                zero-padded real grids -> batched cuFFT D2Z -> fused k-space
//                scale (one pass, in place) -> batched cuFFT Z2D -> gather at
//                targets, adding the real-space part.
// Phase times are CUDA events on the plan's stream.
#define HS_TU_ID 4  // checked build: source of a failing HS_CHECK
#include <cufft.h>

#include <cmath>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace hs {

#define HS_CUFFT(expr)                                                                  \
  do {                                                                                  \
    cufftResult _r = (expr);                                                            \
    if (_r != CUFFT_SUCCESS)                                                            \
      return ::hs::fail(HS_ERR_RESOURCE, std::string(#expr) + ": cuFFT error " + std::to_string((int)_r)); \
  } while (0)

// ---------------------------------------------------------------------------
// record builders

// pair records in cell order: order[k] = combined index i (i >= n -> image of i-n)
__global__ void k_pair_records(int kind, int half, const int* __restrict__ order, int n_comb, int n,
                               const double* __restrict__ pos, const double* __restrict__ sa,
                               const double* __restrict__ sb, double4* __restrict__ P, double4* __restrict__ A,
                               double4* __restrict__ B, double4* __restrict__ Cq, unsigned* __restrict__ flags) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_comb; k += gridDim.x * blockDim.x) {
    const int i = order[k];
    const bool img = half && i >= n;
    const int s = img ? i - n : i;
    const double m = img ? -1.0 : 1.0;  // MIRROR z
    // z + 0.0 maps -0.0 to +0.0: in the half space the sign bit of a record's z then tells
    // images (z <= -0.0) from sources (z >= +0.0), which k_pair_q uses instead of the index
    const double z = pos[3 * s + 2];
    if (half && z < 0.0) atomicOr(flags, FLAG_GEOMETRY);  // sources must lie in x3 >= 0 (system.py:77)
    P[k] = make_double4(pos[3 * s], pos[3 * s + 1], m * (z + 0.0), (double)i);
    const double a0 = sa[3 * s], a1 = sa[3 * s + 1], a2 = sa[3 * s + 2];
    if (kind == HS_STOKESLET || kind == HS_MIXED) {
      // combined_f = [f; -f^I], f^I = f * (1,1,-1)  (system.py:171-177)
      A[k] = img ? make_double4(-a0, -a1, a2, 0.0) : make_double4(a0, a1, a2, 0.0);
      if (kind == HS_MIXED) {  // + the stresslet's combined g, q (rows of sb: g0 g1 g2 q0 q1 q2)
        const double* gq = sb + 6 * (size_t)s;
        B[k] = make_double4(gq[0], gq[1], m * gq[2], 0.0);
        Cq[k] = make_double4(gq[3], gq[4], m * gq[5], 0.0);
      }
    } else {
      const double b0 = sb[3 * s], b1 = sb[3 * s + 1], b2 = sb[3 * s + 2];
      const double g0 = a0, g1 = a1, g2 = m * a2;  // g or g^I
      const double q0 = b0, q1 = b1, q2 = m * b2;  // q or q^I
      if (kind == HS_STRESSLET) {
        A[k] = make_double4(g0, g1, g2, 0.0);
        B[k] = make_double4(q0, q1, q2, 0.0);
      } else {
        const double sg = img ? -1.0 : 1.0;
        A[k] = make_double4(sg * (g1 * q2 - g2 * q1), sg * (g2 * q0 - g0 * q2), sg * (g0 * q1 - g1 * q0), 0.0);
        // image wall channel v = 4 (q3 g^I - g3 q^I), v3 = 0 (kernels_direct.py:123-127)
        if (img) B[k] = make_double4(4.0 * (b2 * g0 - a2 * q0), 4.0 * (b2 * g1 - a2 * q1), 0.0, 0.0);
        else B[k] = make_double4(0.0, 0.0, 0.0, 0.0);
      }
    }
  }
}

// target records in cell order: order[k] = target t
__global__ void k_target_records(const int* __restrict__ order, int nt, const double* __restrict__ tpos,
                                 const long long* __restrict__ tcols, int tcol_identity, double4* __restrict__ TP,
                                 int* __restrict__ torig) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nt; k += gridDim.x * blockDim.x) {
    const int t = order ? order[k] : k;
    const double tc = tcol_identity ? (double)t : (tcols ? (double)tcols[t] : -1.0);
    TP[k] = make_double4(tpos[3 * t], tpos[3 * t + 1], tpos[3 * t + 2], tc);
    torig[k] = t;
  }
}

// spread source records in bin order.  set 0: kernel sources [y; y^I]; set 1: images y^I
// with wall channels; set 2 (mirrored spreading, see k_mirror_z): the sources y themselves
// carrying their kernel channels followed by their images' wall channels.  W has nch
// doubles per row (see kspace.cu channel layout).
__global__ void k_spread_records(int kind, int half, int set, const int* __restrict__ order, int n_rows, int n,
                                 const double* __restrict__ pos, const double* __restrict__ sa,
                                 const double* __restrict__ sb, int nch, double4* __restrict__ P,
                                 double* __restrict__ W) {
  const int nk_m = kind == HS_STRESSLET ? 6 : 3;  // set 2: kernel channels before the wall channels
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n_rows; k += gridDim.x * blockDim.x) {
    const int i = order[k];
    if (kind == HS_MIXED) {
      // mixed stokeslet + stresslet (kmult.cuh layout): set 2 (half space, mirrored) at the sources
      // [F | S V0 V1 V2 M00 M01 M02 M11 M12 M22 | C00 C01 C02 C11 C12 C22]; set 0 (free) [F | C]
      const double y3 = pos[3 * i + 2];
      P[k] = make_double4(pos[3 * i], pos[3 * i + 1], y3, 0.0);
      double* w = W + (size_t)k * nch;
      const double f0 = sa[3 * i], f1 = sa[3 * i + 1], f2 = sa[3 * i + 2];
      const double* gq = sb + 6 * (size_t)i;
      const double g0 = gq[0], g1 = gq[1], g2 = gq[2], q0 = gq[3], q1 = gq[4], q2 = gq[5];
      w[0] = f0;
      w[1] = f1;
      w[2] = f2;
      double* c = w + 3;
      if (set == 2) {
        const double gi2 = -g2, qi2 = -q2;  // g^I, q^I
        w[3] = -f2;                                            // s = -f3 (stokeslet)
        w[4] = -y3 * f0;                                       // v = -y3 f^I (stokeslet)
        w[5] = -y3 * f1;
        w[6] = y3 * f2 + 2.0 * (g0 * q0 + g1 * q1 + gi2 * qi2);  // + v3 = 2 g^I.q^I (stresslet)
        w[7] = -y3 * 2.0 * g0 * q0;                            // M = -y3 (g^I q^I^T + q^I g^I^T)
        w[8] = -y3 * (g0 * q1 + q0 * g1);
        w[9] = -y3 * (g0 * qi2 + q0 * gi2);
        w[10] = -y3 * 2.0 * g1 * q1;
        w[11] = -y3 * (g1 * qi2 + q1 * gi2);
        w[12] = -y3 * 2.0 * gi2 * qi2;
        c = w + 13;
      }
      c[0] = g0 * q0;  // symmetric part of g (x) q (stresslet kernel, source sign +1)
      c[1] = 0.5 * (g0 * q1 + g1 * q0);
      c[2] = 0.5 * (g0 * q2 + g2 * q0);
      c[3] = g1 * q1;
      c[4] = 0.5 * (g1 * q2 + g2 * q1);
      c[5] = g2 * q2;
      continue;
    }
    const bool img = (set == 1) || (set == 0 && half && i >= n);
    const int s = (set == 0 && half && i >= n) ? i - n : i;
    const double m = img ? -1.0 : 1.0;
    const double y3 = pos[3 * s + 2];
    P[k] = make_double4(pos[3 * s], pos[3 * s + 1], m * y3, 0.0);
    double* w = W + (size_t)k * nch;
    for (int part = (set == 2 ? 0 : set); part <= (set == 2 ? 1 : set); ++part) {
    if (set == 2 && part == 1) w += nk_m;
    const double a0 = sa[3 * s], a1 = sa[3 * s + 1], a2 = sa[3 * s + 2];
    double b0 = 0, b1 = 0, b2 = 0;
    if (kind != HS_STOKESLET) {
      b0 = sb[3 * s];
      b1 = sb[3 * s + 1];
      b2 = sb[3 * s + 2];
    }
    if (part == 0) {
      if (kind == HS_STOKESLET) {  // _kernel_weights: combined_f (ewald_fourier.py:357-359)
        w[0] = img ? -a0 : a0;
        w[1] = img ? -a1 : a1;
        w[2] = a2;  // -(f^I)_3 = f_3
      } else {
        const double g0 = a0, g1 = a1, g2 = m * a2, q0 = b0, q1 = b1, q2 = m * b2;
        const double sg = img ? -1.0 : 1.0;
        if (kind == HS_STRESSLET) {  // symmetric part of sign * g (x) q
          w[0] = sg * g0 * q0;
          w[1] = sg * 0.5 * (g0 * q1 + g1 * q0);
          w[2] = sg * 0.5 * (g0 * q2 + g2 * q0);
          w[3] = sg * g1 * q1;
          w[4] = sg * 0.5 * (g1 * q2 + g2 * q1);
          w[5] = sg * g2 * q2;
        } else {  // sign * (g x q)
          w[0] = sg * (g1 * q2 - g2 * q1);
          w[1] = sg * (g2 * q0 - g0 * q2);
          w[2] = sg * (g0 * q1 - g1 * q0);
        }
      }
    } else {
      // _correction_weights (ewald_fourier.py:373-382) with phi_channels (kernels_direct.py:93-127)
      if (kind == HS_STOKESLET) {
        w[0] = -a2;        // s = -f3
        w[1] = -y3 * a0;   // v = -y3 f^I
        w[2] = -y3 * a1;
        w[3] = y3 * a2;
      } else if (kind == HS_STRESSLET) {
        const double g0 = a0, g1 = a1, g2 = -a2, q0 = b0, q1 = b1, q2 = -b2;  // g^I, q^I
        w[0] = 2.0 * (g0 * q0 + g1 * q1 + g2 * q2);  // v3
        w[1] = -y3 * 2.0 * g0 * q0;                   // M00
        w[2] = -y3 * (g0 * q1 + q0 * g1);             // M01
        w[3] = -y3 * (g0 * q2 + q0 * g2);             // M02
        w[4] = -y3 * 2.0 * g1 * q1;                   // M11
        w[5] = -y3 * (g1 * q2 + q1 * g2);             // M12
        w[6] = -y3 * 2.0 * g2 * q2;                   // M22
      } else {
        const double g0 = a0, g1 = a1, q0 = b0, q1 = b1;  // (g^I)_{0,1} = g_{0,1}
        w[0] = 4.0 * (b2 * g0 - a2 * q0);
        w[1] = 4.0 * (b2 * g1 - a2 * q1);
      }
    }
    }
  }
}

// Mirrored spreading (half space).  Grid node k of z sits at -Lt + k h, so node 2Mt - k is
// its mirror image through the wall.  An image source y^I = (y1, y2, -y3) carries the
// kernel channels of its source up to a per-channel sign sigma_c (exact sign flips of the
// same products; k_spread_records set 0): stokeslet -f^I = (-f1, -f2, f3), stresslet
// -(R g)(R q)^T, rotlet -(Rg x Rq) = R (g x q).  Its window is the mirror of the source's
// window (floor((-y3 - o)/h) = 2Mt - 1 - floor((y3 - o)/h) up to rounding at exact node
// hits, where the dropped edge weight is exp(-pi P c^2 / 2) ~ 1e-15 relative).  So with S the
// spread of the N sources only (kernel + wall channels at y),
//   kernel channels:  G_c(k) = S_c(k) + sigma_c S_c(2Mt - k)
//   wall channels:    G_c(k) = S_c(2Mt - k)           (spread at the images y^I only)
// which replaces spreading 2N kernel + N wall sources (10 N P^3 for the stokeslet) by N
// sources (7 N P^3) and one pass over the grid.  In place, one thread per mirror pair.
__global__ void k_mirror_z(double* __restrict__ grid, int nch, unsigned kern_mask, unsigned sigma_neg,
                           int64_t ch_stride, int64_t lines, int pz, int nz) {
  const int half_n = nz / 2;  // pairs (k, nz - k) for k = 1 .. nz/2 - 1, plus k = nz/2 and k = 0
  const int64_t per = lines * (half_n + 1);
  const int64_t n = per * nch;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / per);
    const int64_t r = i - c * per;
    const int64_t line = r / (half_n + 1);
    const int k = (int)(r - line * (half_n + 1));
    double* g = grid + c * ch_stride + line * pz;
    const bool kern = (kern_mask >> c) & 1u;
    const double sg = ((sigma_neg >> c) & 1u) ? -1.0 : 1.0;
    if (k == 0) {  // mirror of node 0 is node nz (outside the grid, where S = 0)
      if (!kern) g[0] = 0.0;
    } else if (k == half_n) {  // the wall plane is its own mirror
      const double v = g[k];
      g[k] = kern ? v + sg * v : v;
    } else {
      const int kk = nz - k;
      HS_CHECK(k > 0 && k < half_n && kk > half_n && kk < nz);
      const double a = g[k], b = g[kk];
      g[k] = kern ? a + sg * b : b;
      g[kk] = kern ? b + sg * a : a;
    }
  }
}

// stokeslet self term only (rc = 0 path): u[t] = -(4 xi/sqrt(pi)) f[tcol] / (8 pi)
__global__ void k_self_term(int nt, const double* __restrict__ tpos, const long long* __restrict__ tcols,
                            int tcol_identity, int n, double xi, const double* __restrict__ f, double* __restrict__ u) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nt; t += gridDim.x * blockDim.x) {
    const long long c = tcol_identity ? t : (tcols ? tcols[t] : -1);
    if (c >= 0 && c < n) {
      const double sc = -(4.0 * xi / kSqrtPi);
      for (int q = 0; q < 3; ++q) u[3 * t + q] = sc * f[3 * c + q] / (8.0 * kPi);
    }
  }
}

// grid_out[i * pitch + c] = tmp[c][i] for i < count (channel stride n)
__global__ void k_interleave(const double* __restrict__ tmp, int nch, int64_t n, int64_t count, int pitch,
                             double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double v[8];
#pragma unroll
    for (int c = 0; c < 8; ++c) v[c] = c < nch ? tmp[(int64_t)c * n + i] : 0.0;
    double2* o = reinterpret_cast<double2*>(out + i * pitch);
    for (int c = 0; c < pitch; c += 2) o[c / 2] = make_double2(v[c], v[c + 1]);
  }
}

// targets for the Fourier gather, in bin order
__global__ void k_gather_records(const int* __restrict__ order, int nt, const double* __restrict__ tpos,
                                 double4* __restrict__ TG, int* __restrict__ tg_orig) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < nt; k += gridDim.x * blockDim.x) {
    const int t = order[k];
    TG[k] = make_double4(tpos[3 * t], tpos[3 * t + 1], tpos[3 * t + 2], 0.0);
    tg_orig[k] = t;
  }
}

inline int grid_size(hs_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->sm_count * 8));
}

hs_status build_pair_records(hs_ctx* ctx, int kind, int half, const int* order, int n_comb, int n, const double* pos,
                             const double* sa, const double* sb, double4* P, double4* A, double4* B) {
  if (n_comb == 0) return HS_OK;
  if (kind == HS_MIXED) return fail(HS_ERR_PARAMETER, "mixed sources evaluate through a plan");
  k_pair_records<<<grid_size(ctx, n_comb), 256, 0, ctx->stream>>>(kind, half, order, n_comb, n, pos, sa, sb, P, A, B,
                                                                         nullptr, ctx->d_flags);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

hs_status build_target_records(hs_ctx* ctx, const int* order, int nt, const double* tpos, const long long* tcols,
                               int tcol_identity, double4* TP, int* torig) {
  if (nt == 0) return HS_OK;
  k_target_records<<<grid_size(ctx, nt), 256, 0, ctx->stream>>>(order, nt, tpos, tcols, tcol_identity, TP, torig);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

}  // namespace hs

using namespace hs;

struct DeviceBuf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct hs_plan {
  hs_ctx* ctx = nullptr;
  hs_params prm{};
  bool half = true;
  int n_comb = 0;       // sources in the real-space / kernel spread set
  int nk = 0, nc = 0;   // kernel / correction channels
  // source-grid channel groups: grid_in holds sg_cap channels; the channels [0, n_in) are
  // spread and forward-transformed group by group (mixed single-GPU plans: 13 + 6, so the
  // 19 source grids never coexist); kern_mask / sigma_neg: kernel channels and their image
  // signs for the mirrored spreading (bit c = channel c)
  int sg_cap = 0;
  int ngroup = 1, group_c0[3] = {0, 0, 0};
  unsigned kern_mask = 0, sigma_mask = 0;
  bool tmp_aliased = false;     // grid_tmp lives in grid_in (mixed): re-zero its z padding after use
  bool four = true;             // false: real-space-only plan (M = 0; real_space_sum)
  int n_in = 0, n_out = 0;
  CellGeom cg{};
  GridGeom gg{};        // padded real grids
  KGeom kg{};
  int64_t n_real_grid = 0, n_half = 0;
  int nbins = 0;
  std::vector<DeviceBuf> bufs;
  int64_t bytes = 0;
  // inputs (staging for host memory)
  double *d_pos = nullptr, *d_sa = nullptr, *d_sb = nullptr, *d_tgt = nullptr;
  long long* d_tcols = nullptr;
  // real space
  int *keys = nullptr, *order = nullptr, *start = nullptr, *work = nullptr;
  int *t_order = nullptr, *t_start = nullptr;
  int2* items = nullptr;
  double4 *P = nullptr, *A = nullptr, *B = nullptr, *Cq = nullptr, *TP = nullptr;
  int* torig = nullptr;
  // Fourier
  int *bk_order = nullptr, *bk_start = nullptr, *bc_order = nullptr, *bc_start = nullptr;
  int *bt_order = nullptr, *bt_start = nullptr;
  double4 *SPk = nullptr, *SPc = nullptr, *TG = nullptr;
  double *SWk = nullptr, *SWc = nullptr;
  int* tg_orig = nullptr;
  // pruned FFT pipeline (fft.cu): grid_in/out [y][x][pz] real per channel, A/spec [y|ky][x][kz] complex
  int64_t n_grid = 0;           // ny * nx * pz
  int64_t n_mixed = 0;          // py * nx * nzh
  double* grid_in = nullptr;    // n_in * n_grid (z-padding stays zero: the z-transform is out of place)
  double2* Amix = nullptr;      // n_mixed (rows y >= ny stay zero: the y-transform is out of place)
  double2* spec = nullptr;      // max(n_in, n_out) * n_mixed
  double* grid_out = nullptr;   // [y][x][z][out_pitch] (channel-interleaved)
  int out_pitch = 6;
  double* grid_tmp = nullptr;   // n_out * n_grid: inverse-z outputs before interleaving
  GridGeom go{};                // geometry of grid_out
  double* tabB = nullptr;       // x-stage layout [ky][kz][kx]
  double* tabH = nullptr;
  double2* tw = nullptr;        // px twiddles
  double2* ytw = nullptr;       // py twiddles of the register y stage (null: cuFFT y stage)
  double2* ztw = nullptr;       // twiddles of the register z stage (null: cuFFT z stage + k_interleave)
  FftPlan xplan{};
  bool have_B = false, have_H = false;
  cufftHandle zf = 0, yf = 0, zi = 0;
  void* fft_work = nullptr;
  // outputs
  double *u = nullptr, *u_real = nullptr, *u_four = nullptr, *uk = nullptr, *uc = nullptr;
  unsigned long long* pair_counts = nullptr;
  unsigned long long* audit = nullptr;  // hs_plan_pair_audit: per-target neighbour audit (3 x nt)
  cudaEvent_t ev[16] = {};
  // y-slab decomposition (hs_plan_create_slab; sharding.py).  slab.world == 0: whole grid.
  hs_slab slab{};
  int yo = 0;                   // owned y planes y1 - y0 (whole grid: ny)
  int nzs = 0;                  // kz columns held in the mixed spectra (whole grid: nzh)
  int64_t n_amix = 0;           // elements of Amix (slab: yo * nx * nzh z-stage outputs)
  int n_sel_k = 0, n_sel_c = 0; // slab: kernel / correction sources spread by this rank
  // device inputs of the current evaluation (slab stages keep them between calls)
  const double *cur_pos = nullptr, *cur_fa = nullptr, *cur_fb = nullptr, *cur_tp = nullptr;
  const long long* cur_tc = nullptr;
  int cur_tcol_identity = 0;
  bool pair_timed = false, spread_timed = false, gather_timed = false;
  bool mirror = false;          // half space: spread the N sources once and mirror (k_mirror_z)
  bool mirror_in_z = false;     // the reflection is applied by the register z stage while loading (no k_mirror_z pass)
  int spread_tz0 = 0;           // mirror_in_z: first z tile the spread launches (nodes below stay zero)
  // concurrent real-space / Fourier pipelines (hs_plan_execute): the Fourier side runs on its
  // own high-priority stream with its own sort buffers, joined before the gather
  cudaStream_t st_four = nullptr;
  cudaEvent_t ev_in = nullptr, ev_four = nullptr;
  int *keys_f = nullptr, *work_f = nullptr;
  int* sort_keys = nullptr;     // buffers the spread / gather sorts use (keys or keys_f)
  int* sort_work = nullptr;
};

namespace {

#ifndef HS_TARGET_SUB
#define HS_TARGET_SUB 32
#endif
constexpr int kTargetSub = HS_TARGET_SUB;  // z sub-slabs per cell in the pair-kernel target order

template <typename T>
hs_status palloc(hs_plan* p, size_t count, T** out, bool zero = false) {
  size_t bytes = std::max<size_t>(count, 1) * sizeof(T);
  void* ptr = nullptr;
  cudaError_t e = cudaMalloc(&ptr, bytes);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(HS_ERR_RESOURCE, "device allocation of " + std::to_string(bytes) + " bytes failed: " +
                                     cudaGetErrorString(e));
  }
  if (zero) HS_CUDA(cudaMemset(ptr, 0, bytes));
  p->bufs.push_back({ptr, bytes});
  p->bytes += (int64_t)bytes;
  *out = (T*)ptr;
  return HS_OK;
}

int table_needs(int kind, int half, int table_kind) {
  // table_kinds_for (ewald_fourier.py:281-290)
  if (table_kind == HS_BIHARMONIC) return kind != HS_ROTLET;
  return kind == HS_ROTLET || half;
}

}  // namespace

namespace hs {
hs_status plan_channels(int kind, int half, int* nk, int* nc) {
  if (kind == HS_STOKESLET) { *nk = 3; *nc = half ? 4 : 0; }
  else if (kind == HS_STRESSLET) { *nk = 6; *nc = half ? 7 : 0; }
  else if (kind == HS_ROTLET) { *nk = 3; *nc = half ? 2 : 0; }
  else if (kind == HS_MIXED) { *nk = 9; *nc = half ? 10 : 0; }  // kmult.cuh mixed layout
  else return fail(HS_ERR_PARAMETER, "unknown kernel kind");
  return HS_OK;
}
}  // namespace hs

static unsigned mirror_sigma_neg(int kind) {
  // channels whose image value is minus the source value (k_spread_records set 0)
  if (kind == HS_STOKESLET) return 0x3u;               // (-, -, +)
  if (kind == HS_STRESSLET) return 0x1u | 0x2u | 0x8u | 0x20u;  // 00 01 11 22 negative, 02 12 positive
  return 0x4u;                                          // rotlet (+, +, -)
}

static hs_status plan_create_impl(hs_ctx* ctx, const hs_params* prm, const hs_slab* slab, hs_plan** out) {
  if (!ctx || !prm || !out) return fail(HS_ERR_PARAMETER, "null argument");
  HS_CUDA(cudaSetDevice(ctx->device));
  hs_plan* p = new hs_plan();
  p->ctx = ctx;
  p->prm = *prm;
  if (slab) p->slab = *slab;
  const bool sl = slab != nullptr;
  p->half = prm->geometry == HS_HALF;
  hs_status st = HS_OK;
  auto bail = [&](hs_status s) {
    hs_plan_destroy(p);
    return s;
  };
  if (prm->n < 1 || prm->n_targets < 0 || prm->n > (1 << 29) || prm->n_targets > (1 << 30))
    return bail(fail(HS_ERR_PARAMETER, "unsupported source/target count"));
  if ((st = plan_channels(prm->kind, p->half, &p->nk, &p->nc)) != HS_OK) return bail(st);
  const int n = (int)prm->n, nt = (int)prm->n_targets;
  p->n_comb = p->half ? 2 * n : n;
  p->n_in = p->nk + p->nc;
  p->n_out = p->half ? 6 : 3;
  // ---- real-space cell geometry: build_cell_list(src, 0.5*rc, (lo, hi))  (ewald_real.py:415-430)
  const double L = prm->L;
  double lo[3] = {0.0, 0.0, p->half ? -L : 0.0}, hi[3] = {L, L, L};
  const bool do_real = prm->rc > 0;
  if (do_real) {
    if ((st = cell_geometry(0.5 * prm->rc, lo, hi, &p->cg)) != HS_OK) return bail(st);
  } else {
    p->cg.dims[0] = p->cg.dims[1] = p->cg.dims[2] = 1;
  }
  const int ncell = (int)p->cg.ncell();
  // ---- grid geometry (M = 0: a real-space-only plan, no grids, transforms or tables)
  p->four = prm->M > 0;
  GridGeom& g = p->gg;
  int64_t px = 0, py = 0, pz = 0, nxd = 0, nzh = 0;
  if (!p->four) {
    if (sl) return bail(fail(HS_ERR_PARAMETER, "slab plans need the Fourier part (M > 0)"));
    for (int k = 0; k < 3; ++k) g.dims[k] = 1;
    g.P = 1;
  } else {
    for (int k = 0; k < 3; ++k) {
      g.origin[k] = prm->origin[k];
      g.dims[k] = (int)prm->dims[k];
    }
    g.h = prm->h;
    g.P = (int)prm->P;
    g.alpha = 2.0 * prm->xi * prm->xi / prm->eta;
    g.pref = std::pow(2.0 * prm->xi * prm->xi / (kPi * prm->eta), 1.5);
    px = prm->padded[0];
    py = prm->padded[1];
    pz = prm->padded[2];
    nxd = prm->dims[0];
    nzh = pz / 2 + 1;
    int64_t nyd = prm->dims[1];
    p->yo = (int)nyd;
    p->nzs = (int)nzh;
    if (sl) {
      // owned planes [y0, y1) plus P - 1 ghost planes above (spread contributions for the next
      // rank, then the gather halo received from it); owned kz columns [kz0, kz1)
      const hs_slab& s = *slab;
      if (s.world < 1 || s.rank < 0 || s.rank >= s.world || s.y0 < 0 || s.y1 <= s.y0 || s.y1 > prm->dims[1] ||
          s.kz0 < 0 || s.kz1 <= s.kz0 || s.kz1 > nzh)
        return bail(fail(HS_ERR_PARAMETER, "invalid slab (rank, world, y range, kz range)"));
      if (s.rank + 1 < s.world && s.y1 - s.y0 < prm->P - 1)
        return bail(fail(HS_ERR_PARAMETER, "y slab thinner than P - 1 planes: use fewer ranks"));
      p->yo = (int)(s.y1 - s.y0);
      p->nzs = (int)(s.kz1 - s.kz0);
      nyd = p->yo + prm->P - 1;
      g.dims[1] = (int)nyd;
      g.yoff = (int)s.y0;
      g.sel = 1;
      g.sel_lo = 0;
      g.sel_hi = p->yo;
    }
    // grids are stored [y][x][z] with z-pitch pz (see fft.cu)
    g.stride[0] = pz;
    g.stride[1] = nxd * pz;
    g.stride[2] = 1;
    g.ch_stride = nyd * nxd * pz;
    p->n_grid = nyd * nxd * pz;
    p->n_mixed = py * nxd * p->nzs;
    p->n_amix = sl ? (int64_t)p->yo * nxd * nzh : p->n_mixed;
    p->n_real_grid = px * py * pz;
    p->n_half = px * py * nzh;
    if (px != py) return bail(fail(HS_ERR_PARAMETER, "padded x and y lengths must agree"));
    if ((st = make_fft_plan((int)px, &p->xplan)) != HS_OK) return bail(st);
    KGeom& kg = p->kg;
    kg.p[0] = (int)px;
    kg.p[1] = (int)py;
    kg.p[2] = (int)pz;
    kg.nzh = (int)(pz / 2 + 1);
    for (int k = 0; k < 3; ++k) kg.kscale[k] = 1.0 / ((double)prm->padded[k] * prm->h);
    kg.a = (1.0 - prm->eta) / (4.0 * prm->xi * prm->xi);
    kg.b = 1.0 / (4.0 * prm->xi * prm->xi);
    kg.inv_n = 1.0 / ((double)px * (double)py * (double)pz);
  }
  p->nbins = p->four ? sp_nbins(g, 0) * sp_nbins(g, 1) * sp_nbins(g, 2) : 1;
  const int nb = p->nbins;

  // ---- buffers
  const int maxn = std::max(p->n_comb, std::max(nt, n));
  const int maxb = std::max(std::max(ncell * kTargetSub, nb + 1), p->four ? gather_keys(g) : 1);
#define A_(cnt, ptr, ...) if ((st = palloc(p, (size_t)(cnt), &(ptr), ##__VA_ARGS__)) != HS_OK) return bail(st)
  const bool mixed = prm->kind == HS_MIXED;
  A_(3 * (size_t)n, p->d_pos);
  A_(3 * (size_t)n, p->d_sa);
  if (prm->kind != HS_STOKESLET) A_((mixed ? 6 : 3) * (size_t)n, p->d_sb);
  if (!prm->targets_are_sources) {
    A_(3 * (size_t)std::max(nt, 1), p->d_tgt);
    A_((size_t)std::max(nt, 1), p->d_tcols);
  }
  A_(maxn, p->keys);
  A_(maxn, p->order);
  A_(counting_sort_work_ints(maxn, maxb), p->work);
  A_(maxn, p->keys_f);
  A_(counting_sort_work_ints(maxn, maxb), p->work_f);
  p->sort_keys = p->keys;
  p->sort_work = p->work;
  A_(ncell + 1, p->start);
  A_(nt + 1, p->t_order);
  A_((size_t)ncell * kTargetSub + 1, p->t_start);
  A_((size_t)nt / 128 + (size_t)p->cg.dims[0] * p->cg.dims[1] + 2, p->items);
  A_(p->n_comb, p->P);
  A_(p->n_comb, p->A);
  A_(p->n_comb, p->B);
  if (mixed) A_(p->n_comb, p->Cq);
  A_(std::max(nt, 1), p->TP);
  A_(std::max(nt, 1), p->torig);
  if (p->four) {
    A_(p->n_comb, p->bk_order);
    A_(nb + 2, p->bk_start);  // + the slab plan's drop bin
    A_(n, p->bc_order);
    A_(nb + 2, p->bc_start);
    A_(std::max(nt, 1), p->bt_order);
    A_((size_t)gather_keys(g) + 1, p->bt_start);
    // mirrored spreading (half space; HS_SPREAD_IMAGES=1 spreads the images explicitly, comparison)
    p->mirror = p->half && (mixed || !getenv("HS_SPREAD_IMAGES"));
    // channel groups and mirror masks
    p->sg_cap = p->n_in;
    p->ngroup = 1;
    p->group_c0[1] = p->n_in;
    if (mixed) {
      p->kern_mask = p->half ? (0x7u | (0x3Fu << 13)) : 0x1FFu;
      p->sigma_mask = p->half ? (0x3u | (0x2Bu << 13)) : 0u;
      if (!sl) {  // one GPU: spread / transform 13 + 6 (half) or 3 + 6 (free) channels at a time
        p->ngroup = 2;
        p->group_c0[1] = p->half ? 13 : 3;
        p->group_c0[2] = p->n_in;
        p->sg_cap = p->half ? 13 : 6;
      }
    } else {
      p->kern_mask = (1u << p->nk) - 1u;
      p->sigma_mask = mirror_sigma_neg(prm->kind);
    }
    A_(p->n_comb, p->SPk);
    A_(std::max((size_t)p->n_comb * p->nk, (size_t)n * p->n_in), p->SWk);
    if (p->nc) {
      A_(n, p->SPc);
      A_((size_t)n * p->nc, p->SWc);
    }
    A_(std::max(nt, 1), p->TG);
    A_(std::max(nt, 1), p->tg_orig);
    A_((size_t)p->sg_cap * p->n_grid, p->grid_in, true);
    A_((size_t)p->n_amix, p->Amix, true);
    A_((size_t)std::max(p->n_in, p->n_out) * p->n_mixed, p->spec);
    p->out_pitch = p->half ? 6 : 4;
    A_((size_t)p->out_pitch * p->n_grid, p->grid_out, true);
    // register z stage (single-GPU plans): the inverse writes the interleaved output grids
    // directly, so no per-channel inverse buffer exists; env HS_ZSTAGE_CUFFT: cuFFT z stage +
    // k_interleave (comparison)
    // (y-slab plans keep the per-channel inverse buffer: their channels arrive one at a time from
    // the all-to-all, so each is inverse-transformed on its own and interleaved at the end)
    const bool zreg = zstage_supported((int)pz, (int)prm->dims[2]) && !getenv("HS_ZSTAGE_CUFFT");
    if (zreg) A_(zstage_twiddle_count((int)pz), p->ztw);
    // single-GPU plans: the forward z stage applies the half-space reflection while loading
    // (slab plans exchange ghost planes of the reflected grids, so they keep the k_mirror_z pass)
    p->mirror_in_z = p->mirror && zreg && !sl && (prm->dims[2] % 2 == 0);
    // sources lie above the wall (node nz / 2), so no window starts below nz/2 - P/2 (one node of
    // margin): those tiles are not launched; their nodes keep the zeros the grids were allocated
    // with (nothing else writes them once the mirror pass is gone)
    if (p->mirror_in_z) p->spread_tz0 = (int)std::max<int64_t>(0, (prm->dims[2] / 2 - prm->P / 2 - 1) / SP_TZ);
    if (zreg && !sl) {
    } else if (mixed && !sl && p->sg_cap >= p->n_out) {
      p->grid_tmp = p->grid_in;  // the source grids are dead once forward-transformed
      p->tmp_aliased = true;
    } else {
      A_((size_t)p->n_out * p->n_grid, p->grid_tmp, true);
    }
    p->go = p->gg;
    p->go.stride[0] = (int64_t)p->out_pitch * pz;
    p->go.stride[1] = (int64_t)p->out_pitch * nxd * pz;
    p->go.stride[2] = p->out_pitch;
    p->go.ch_stride = 1;
    // tables in x-stage layout, only the plan's kz columns
    const size_t ntab = (size_t)px * py * p->nzs;
    if (table_needs(prm->kind, p->half, HS_BIHARMONIC)) A_(ntab, p->tabB);
    if (table_needs(prm->kind, p->half, HS_HARMONIC)) A_(ntab, p->tabH);
    A_(px, p->tw);
    if ((st = make_twiddles((int)px, p->tw, ctx->stream)) != HS_OK) return bail(st);
    if (ystage_supported((int)py) && !getenv("HS_YSTAGE_CUFFT")) {  // env: cuFFT y stage (comparison)
      A_(py, p->ytw);
      if ((st = make_twiddles((int)py, p->ytw, ctx->stream)) != HS_OK) return bail(st);
    }
    if (p->ztw && (st = make_zstage_twiddles((int)pz, p->ztw, ctx->stream)) != HS_OK) return bail(st);
  }
  A_(3 * (size_t)std::max(nt, 1), p->u);
  A_(3 * (size_t)std::max(nt, 1), p->u_real, true);
  A_(3 * (size_t)std::max(nt, 1), p->u_four, true);
  A_(3 * (size_t)std::max(nt, 1), p->uk, true);
  A_(3, p->pair_counts, true);  // [pairs, image pairs, work-item counter]
  A_(3 * (size_t)std::max(nt, 1), p->uc, true);
#undef A_
  // ---- cuFFT plans (batched over channels, shared work area)
  if (p->four) {
    // 1-D batched cuFFT plans for the z and y stages (x is fused with the scaling, fft.cu)
    size_t w1 = 0, w2 = 0, w3 = 0;
    if (cufftCreate(&p->zf) != CUFFT_SUCCESS || cufftCreate(&p->yf) != CUFFT_SUCCESS ||
        cufftCreate(&p->zi) != CUFFT_SUCCESS)
      return bail(fail(HS_ERR_RESOURCE, "cufftCreate failed"));
    cufftSetAutoAllocation(p->zf, 0);
    cufftSetAutoAllocation(p->yf, 0);
    cufftSetAutoAllocation(p->zi, 0);
    long long nz1[1] = {pz}, nzh1[1] = {nzh}, ny1[1] = {py};
    const long long zlines = (long long)p->yo * nxd, ylines = nxd * p->nzs;  // z: owned planes only
    if (cufftMakePlanMany64(p->zf, 1, nz1, nz1, 1, pz, nzh1, 1, nzh, CUFFT_D2Z, zlines, &w1) != CUFFT_SUCCESS)
      return bail(fail(HS_ERR_RESOURCE, "cuFFT z D2Z plan failed"));
    if (cufftMakePlanMany64(p->yf, 1, ny1, ny1, ylines, 1, ny1, ylines, 1, CUFFT_Z2Z, ylines, &w2) != CUFFT_SUCCESS)
      return bail(fail(HS_ERR_RESOURCE, "cuFFT y Z2Z plan failed"));
    if (cufftMakePlanMany64(p->zi, 1, nz1, nzh1, 1, nzh, nz1, 1, pz, CUFFT_Z2D, zlines, &w3) != CUFFT_SUCCESS)
      return bail(fail(HS_ERR_RESOURCE, "cuFFT z Z2D plan failed"));
    const size_t ws = std::max(w1, std::max(w2, w3));
    char* wsp = nullptr;
    if ((st = palloc(p, std::max<size_t>(ws, 16), &wsp)) != HS_OK) return bail(st);
    p->fft_work = wsp;
    cufftSetWorkArea(p->zf, wsp);
    cufftSetWorkArea(p->yf, wsp);
    cufftSetWorkArea(p->zi, wsp);
  }
  for (auto& e : p->ev) HS_CUDA(cudaEventCreate(&e));
  {
    int lo_prio = 0, hi_prio = 0;
    HS_CUDA(cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio));
    HS_CUDA(cudaStreamCreateWithPriority(&p->st_four, cudaStreamNonBlocking, hi_prio));
    HS_CUDA(cudaEventCreateWithFlags(&p->ev_in, cudaEventDisableTiming));
    HS_CUDA(cudaEventCreateWithFlags(&p->ev_four, cudaEventDisableTiming));
  }
  *out = p;
  return HS_OK;
}

extern "C" hs_status hs_plan_create(hs_ctx* ctx, const hs_params* prm, hs_plan** out) {
  return plan_create_impl(ctx, prm, nullptr, out);
}

extern "C" hs_status hs_plan_create_slab(hs_ctx* ctx, const hs_params* prm, const hs_slab* slab, hs_plan** out) {
  if (!slab) return fail(HS_ERR_PARAMETER, "null slab");
  return plan_create_impl(ctx, prm, slab, out);
}

extern "C" hs_status hs_plan_destroy(hs_plan* p) {
  if (!p) return HS_OK;
  if (p->zf) cufftDestroy(p->zf);
  if (p->yf) cufftDestroy(p->yf);
  if (p->zi) cufftDestroy(p->zi);
  for (auto& e : p->ev)
    if (e) cudaEventDestroy(e);
  if (p->ev_in) cudaEventDestroy(p->ev_in);
  if (p->ev_four) cudaEventDestroy(p->ev_four);
  if (p->st_four) cudaStreamDestroy(p->st_four);
  for (auto& b : p->bufs) cudaFree(b.p);
  delete p;
  return HS_OK;
}

extern "C" int64_t hs_plan_bytes(const hs_plan* p) { return p ? p->bytes : 0; }

extern "C" hs_status hs_plan_fft_counts(const hs_plan* p, int* n_fft, int* n_ifft) {
  if (!p) return fail(HS_ERR_PARAMETER, "null plan");
  if (n_fft) *n_fft = p->four ? p->n_in : 0;
  if (n_ifft) *n_ifft = p->four ? p->n_out : 0;
  return HS_OK;
}

extern "C" hs_status hs_plan_real_parts(hs_plan* p, double* kernel_part, double* correction_part, int mem) {
  if (!p) return fail(HS_ERR_PARAMETER, "null plan");
  const size_t bytes = 24 * (size_t)p->prm.n_targets;
  const cudaMemcpyKind k = mem == HS_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (bytes && kernel_part) HS_CUDA(cudaMemcpyAsync(kernel_part, p->uk, bytes, k, p->ctx->stream));
  if (bytes && correction_part) HS_CUDA(cudaMemcpyAsync(correction_part, p->uc, bytes, k, p->ctx->stream));
  HS_CUDA(cudaStreamSynchronize(p->ctx->stream));
  return HS_OK;
}

static int table_kz0(const hs_plan* p) { return p->slab.world > 0 ? (int)p->slab.kz0 : 0; }

extern "C" hs_status hs_plan_set_table(hs_plan* p, int table_kind, const double* samples, int mem) {
  if (!p || !samples) return fail(HS_ERR_PARAMETER, "null argument");
  if (!p->four) return fail(HS_ERR_CONFIG, "real-space-only plan (M = 0) has no tables");
  double* dst = table_kind == HS_BIHARMONIC ? p->tabB : p->tabH;
  if (!dst) return HS_OK;  // not needed by this kind/geometry
  hs_ctx* ctx = p->ctx;
  const int64_t pd[3] = {p->prm.padded[0], p->prm.padded[1], p->prm.padded[2]};
  const size_t full = (size_t)pd[0] * pd[1] * pd[2];
  const double* src = samples;
  // staging in the (idle) spectrum buffer when it is large enough, else stream-ordered allocations
  const size_t spec_bytes = sizeof(double2) * (size_t)std::max(p->n_in, p->n_out) * p->n_mixed;
  const size_t half_b = ((size_t)p->n_half * sizeof(double) + 255) & ~(size_t)255;
  const size_t full_b = (mem == HS_MEM_HOST) ? full * sizeof(double) : 0;
  const bool in_spec = half_b + full_b <= spec_bytes;
  HS_CUDA(cudaStreamSynchronize(ctx->stream));
  double* tmp = nullptr;
  double* half = nullptr;
  if (in_spec) {
    half = (double*)p->spec;
    if (full_b) tmp = (double*)((char*)p->spec + half_b);
  } else {
    HS_CUDA(cudaMallocAsync(&half, (size_t)p->n_half * sizeof(double), ctx->stream));
    if (full_b) HS_CUDA(cudaMallocAsync(&tmp, full_b, ctx->stream));
  }
  if (mem == HS_MEM_HOST) {
    HS_CUDA(cudaMemcpyAsync(tmp, samples, full * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
    src = tmp;
  }
  hs_status st = launch_take_half(ctx, src, pd, half);
  if (st == HS_OK)
    st = launch_table_to_xmajor(ctx, half, (int)pd[0], (int)pd[1], (int)(pd[2] / 2 + 1), dst, table_kz0(p), p->nzs);
  if (!in_spec) {
    cudaFreeAsync(half, ctx->stream);
    if (tmp) cudaFreeAsync(tmp, ctx->stream);
  }
  HS_TRY(st);
  HS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (table_kind == HS_BIHARMONIC) p->have_B = true;
  else p->have_H = true;
  return HS_OK;
}

namespace hs {
// precompute_greens into a half-spectrum real table (ewald_fourier.py:207-244)
static hs_status greens_half_table_full(hs_ctx* ctx, int kind, double R, double h, const int64_t big[3],
                                        const int64_t dims[3], const int64_t guards[3], const int64_t pd[3],
                                        double* half_out);

// Separable, pruned precompute (kspace.cu k_hat_lines / k_sep_scatter / k_sep_crop): the
// oversampled grid never exists; three batched 1-D C2R stages (z, y, x) keep only the
// real-space nodes 0..k_i of the crop after each stage.  Peak memory at cfg5 (big
// (1432,1432,2864)): ~12 GB of intermediates + the pd-sized crop and its spectrum, instead
// of 94 GB.  HS_TABLE_FULL=1 selects the 3-D big-grid transform (comparison).
hs_status greens_half_table(hs_ctx* ctx, int kind, double R, double h, const int64_t big[3], const int64_t dims[3],
                            const int64_t guards[3], const int64_t pd[3], double* half_out, void* scratch,
                            size_t scratch_bytes) {
  if (getenv("HS_TABLE_FULL")) return greens_half_table_full(ctx, kind, R, h, big, dims, guards, pd, half_out);
  cudaStream_t st = ctx->stream;
  const int64_t n[3] = {big[0], big[1], big[2]};
  const int64_t hh[3] = {n[0] / 2 + 1, n[1] / 2 + 1, n[2] / 2 + 1};
  int64_t k[3], kp[3];
  for (int d = 0; d < 3; ++d) {
    k[d] = dims[d] + guards[d];
    kp[d] = k[d] + 1;
    if (2 * k[d] != pd[d] || 2 * k[d] > n[d]) return fail(HS_ERR_PARAMETER, "precompute: crop does not match the grids");
  }
  const double scale = 1.0 / ((double)n[0] * (double)n[1] * (double)n[2]);
  const int64_t lt1 = hh[0] * hh[1], lt2 = kp[2] * hh[0], lt3 = kp[1] * kp[2];
  // lines per chunk: ~512 MB of line buffers per stage
  auto chunk = [](int64_t len_in_c, int64_t len_out_r, int64_t ltot) {
    const int64_t per = 16 * len_in_c + 8 * len_out_r;
    return std::max<int64_t>(1, std::min<int64_t>(ltot, ((int64_t)512 << 20) / per));
  };
  const int64_t B1 = chunk(hh[2], n[2], lt1), B2 = chunk(hh[1], n[1], lt2), B3 = chunk(hh[0], n[0], lt3);
  double2 *lin = nullptr, *A2 = nullptr, *A3 = nullptr, *spec = nullptr;
  double *lout = nullptr, *F = nullptr, *crop = nullptr;
  void* ws = nullptr;
  cufftHandle pl[3] = {0, 0, 0}, pf = 0;
  hs_status rs = HS_OK;
  // intermediates come from the caller's idle scratch (a plan's spectrum buffer) while it lasts
  // (bump allocation, 256-byte aligned), then from cudaMalloc; release() frees only the latter
  char* arena = (char*)scratch;
  size_t arena_used = 0;
  std::vector<void*> owned;
  auto alloc = [&](void** ptr, size_t bytes) {
    bytes = (std::max<size_t>(bytes, 16) + 255) & ~(size_t)255;
    if (arena && arena_used + bytes <= scratch_bytes) {
      *ptr = arena + arena_used;
      arena_used += bytes;
      return true;
    }
    if (cudaMalloc(ptr, bytes) != cudaSuccess) {
      cudaGetLastError();
      *ptr = nullptr;
      return false;
    }
    owned.push_back(*ptr);
    return true;
  };
  auto release = [&](void* ptr) {
    for (auto& o : owned)
      if (o == ptr && o) {
        cudaFree(o);
        o = nullptr;
      }
  };
  auto cleanup = [&]() {
    for (auto& q : pl)
      if (q) cufftDestroy(q);
    if (pf) cufftDestroy(pf);
    for (auto& o : owned)
      if (o) cudaFree(o);
  };
  do {
    const size_t lin_b = 16 * (size_t)std::max(B1 * hh[2], 1L), lout_b = 8 * (size_t)std::max(B1 * n[2], 1L);
    const size_t lin2 = 16 * (size_t)std::max(B2 * hh[1], B3 * hh[0]), lout2 = 8 * (size_t)std::max(B2 * n[1], B3 * n[0]);
    if (!alloc((void**)&lin, std::max(lin_b, lin2)) || !alloc((void**)&lout, std::max(lout_b, lout2)) ||
        !alloc((void**)&A2, 16 * (size_t)(lt2 + B2) * hh[1])) {
      rs = fail(HS_ERR_RESOURCE, "precompute: intermediate allocation failed");
      break;
    }
    // batched 1-D C2R plans (contiguous lines), one shared work area
    size_t wsz[3] = {0, 0, 0};
    const int64_t Bs[3] = {B1, B2, B3}, len[3] = {n[2], n[1], n[0]}, hin[3] = {hh[2], hh[1], hh[0]};
    bool ok = true;
    for (int s = 0; s < 3 && ok; ++s) {
      long long nn[1] = {len[s]}, ni[1] = {hin[s]}, no[1] = {len[s]};
      ok = cufftCreate(&pl[s]) == CUFFT_SUCCESS && cufftSetAutoAllocation(pl[s], 0) == CUFFT_SUCCESS &&
           cufftMakePlanMany64(pl[s], 1, nn, ni, 1, hin[s], no, 1, len[s], CUFFT_Z2D, Bs[s], &wsz[s]) == CUFFT_SUCCESS;
    }
    if (!ok) {
      rs = fail(HS_ERR_RESOURCE, "precompute: cuFFT C2R plan failed");
      break;
    }
    const size_t wmax = std::max(wsz[0], std::max(wsz[1], wsz[2]));
    if (!alloc(&ws, wmax)) {
      rs = fail(HS_ERR_RESOURCE, "precompute: cuFFT work area allocation failed");
      break;
    }
    for (auto& q : pl) {
      cufftSetWorkArea(q, ws);
      cufftSetStream(q, st);
    }
    // stage 1 (z): lines (kx, ky), generated on the fly
    for (int64_t l0 = 0; l0 < lt1 && rs == HS_OK; l0 += B1) {
      if ((rs = launch_hat_lines(ctx, kind, R, h, big, l0, B1, hh[1], hh[2], lt1, lin)) != HS_OK) break;
      if (cufftExecZ2D(pl[0], (cufftDoubleComplex*)lin, lout) != CUFFT_SUCCESS) {
        rs = fail(HS_ERR_CUDA, "precompute: z C2R failed");
        break;
      }
      rs = launch_sep_scatter(ctx, lout, l0, B1, lt1, n[2], kp[2], hh[0], hh[1], 1.0, A2, nullptr);
    }
    if (rs != HS_OK) break;
    if (!alloc((void**)&A3, 16 * (size_t)(lt3 + B3) * hh[0])) {
      rs = fail(HS_ERR_RESOURCE, "precompute: intermediate allocation failed");
      break;
    }
    // stage 2 (y): rows (z, kx) of A2
    for (int64_t l0 = 0; l0 < lt2 && rs == HS_OK; l0 += B2) {
      if (cufftExecZ2D(pl[1], (cufftDoubleComplex*)(A2 + l0 * hh[1]), lout) != CUFFT_SUCCESS) {
        rs = fail(HS_ERR_CUDA, "precompute: y C2R failed");
        break;
      }
      rs = launch_sep_scatter(ctx, lout, l0, B2, lt2, n[1], kp[1], kp[2], hh[0], 1.0, A3, nullptr);
    }
    if (rs != HS_OK) break;
    HS_CUDA(cudaStreamSynchronize(st));
    release(A2);
    A2 = nullptr;
    if (!alloc((void**)&F, 8 * (size_t)lt3 * kp[0])) {
      rs = fail(HS_ERR_RESOURCE, "precompute: intermediate allocation failed");
      break;
    }
    // stage 3 (x): rows (y, z) of A3
    for (int64_t l0 = 0; l0 < lt3 && rs == HS_OK; l0 += B3) {
      if (cufftExecZ2D(pl[2], (cufftDoubleComplex*)(A3 + l0 * hh[0]), lout) != CUFFT_SUCCESS) {
        rs = fail(HS_ERR_CUDA, "precompute: x C2R failed");
        break;
      }
      rs = launch_sep_scatter(ctx, lout, l0, B3, lt3, n[0], kp[0], 0, 0, scale, nullptr, F);
    }
    if (rs != HS_OK) break;
    HS_CUDA(cudaStreamSynchronize(st));
    for (auto& q : pl) {
      cufftDestroy(q);
      q = 0;
    }
    release(A3);
    A3 = nullptr;
    release(lin);
    lin = nullptr;
    release(lout);
    lout = nullptr;
    release(ws);
    ws = nullptr;
    // crop (evenness) and the forward transform on the padded grid
    const size_t ncrop = (size_t)pd[0] * pd[1] * pd[2], nch = (size_t)pd[0] * pd[1] * (pd[2] / 2 + 1);
    if (!alloc((void**)&crop, 8 * ncrop) || !alloc((void**)&spec, 16 * nch)) {
      rs = fail(HS_ERR_RESOURCE, "precompute: padded-grid allocation failed");
      break;
    }
    if ((rs = launch_sep_crop(ctx, F, k, crop)) != HS_OK) break;
    long long np[3] = {pd[0], pd[1], pd[2]};
    size_t w2 = 0;
    if (cufftCreate(&pf) != CUFFT_SUCCESS || cufftSetAutoAllocation(pf, 0) != CUFFT_SUCCESS ||
        cufftMakePlanMany64(pf, 3, np, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, 1, &w2) != CUFFT_SUCCESS) {
      rs = fail(HS_ERR_RESOURCE, "precompute: cuFFT D2Z plan failed");
      break;
    }
    if (!alloc(&ws, w2)) {
      rs = fail(HS_ERR_RESOURCE, "precompute: cuFFT work area allocation failed");
      break;
    }
    cufftSetWorkArea(pf, ws);
    cufftSetStream(pf, st);
    if (cufftExecD2Z(pf, crop, (cufftDoubleComplex*)spec) != CUFFT_SUCCESS) {
      rs = fail(HS_ERR_CUDA, "precompute: D2Z failed");
      break;
    }
    if ((rs = launch_real_part(ctx, spec, (int64_t)nch, half_out)) != HS_OK) break;
    if (cudaStreamSynchronize(st) != cudaSuccess) {
      rs = fail(HS_ERR_CUDA, "precompute: stream sync failed");
      break;
    }
  } while (false);
  cleanup();
  return rs;
}

static hs_status greens_half_table_full(hs_ctx* ctx, int kind, double R, double h, const int64_t big[3],
                                        const int64_t dims[3], const int64_t guards[3], const int64_t pd[3],
                                        double* half_out) {
  cudaStream_t st = ctx->stream;
  const int64_t nzb = big[2] / 2 + 1;
  const size_t nbh = (size_t)big[0] * big[1] * nzb, nbr = (size_t)big[0] * big[1] * big[2];
  const size_t ncrop = (size_t)pd[0] * pd[1] * pd[2], nch = (size_t)pd[0] * pd[1] * (pd[2] / 2 + 1);
  double2* hat = nullptr;
  double* field = nullptr;
  void* ws = nullptr;
  cufftHandle pb = 0, pf = 0;
  hs_status rs = HS_OK;
  auto cleanup = [&]() {
    if (pb) cufftDestroy(pb);
    if (pf) cufftDestroy(pf);
    if (hat) cudaFree(hat);
    if (field) cudaFree(field);
    if (ws) cudaFree(ws);
  };
  do {
    if (cudaMalloc(&hat, std::max(nbh * sizeof(double2), ncrop * sizeof(double))) != cudaSuccess ||
        cudaMalloc(&field, std::max(nbr, nch * 2) * sizeof(double)) != cudaSuccess) {
      cudaGetLastError();
      rs = fail(HS_ERR_RESOURCE, "precompute: big-grid allocation failed");
      break;
    }
    if ((rs = launch_greens_hat(ctx, kind, R, h, big, hat)) != HS_OK) break;
    long long nb[3] = {big[0], big[1], big[2]};
    size_t w1 = 0, w2 = 0;
    cufftCreate(&pb);
    cufftSetAutoAllocation(pb, 0);
    if (cufftMakePlanMany64(pb, 3, nb, nullptr, 1, 0, nullptr, 1, 0, CUFFT_Z2D, 1, &w1) != CUFFT_SUCCESS) {
      rs = fail(HS_ERR_RESOURCE, "precompute: cuFFT Z2D plan failed");
      break;
    }
    long long np[3] = {pd[0], pd[1], pd[2]};
    cufftCreate(&pf);
    cufftSetAutoAllocation(pf, 0);
    if (cufftMakePlanMany64(pf, 3, np, nullptr, 1, 0, nullptr, 1, 0, CUFFT_D2Z, 1, &w2) != CUFFT_SUCCESS) {
      rs = fail(HS_ERR_RESOURCE, "precompute: cuFFT D2Z plan failed");
      break;
    }
    if (cudaMalloc(&ws, std::max<size_t>(std::max(w1, w2), 16)) != cudaSuccess) {
      cudaGetLastError();
      rs = fail(HS_ERR_RESOURCE, "precompute: cuFFT work area allocation failed");
      break;
    }
    cufftSetWorkArea(pb, ws);
    cufftSetWorkArea(pf, ws);
    cufftSetStream(pb, st);
    cufftSetStream(pf, st);
    if (cufftExecZ2D(pb, (cufftDoubleComplex*)hat, field) != CUFFT_SUCCESS) {
      rs = fail(HS_ERR_RESOURCE, "precompute: Z2D failed");
      break;
    }
    // irfftn normalisation 1/prod(big); crop to the guarded torus (keep d+g per side)
    int64_t keep[3];
    for (int k = 0; k < 3; ++k) keep[k] = dims[k] + guards[k];
    const double scale = 1.0 / ((double)big[0] * (double)big[1] * (double)big[2]);
    double* crop = (double*)hat;  // reuse
    if ((rs = launch_crop(ctx, field, big, keep, scale, crop)) != HS_OK) break;
    double2* cs = (double2*)field;
    if (cufftExecD2Z(pf, crop, (cufftDoubleComplex*)cs) != CUFFT_SUCCESS) {
      rs = fail(HS_ERR_RESOURCE, "precompute: D2Z failed");
      break;
    }
    if ((rs = launch_real_part(ctx, cs, (int64_t)nch, half_out)) != HS_OK) break;
    if (cudaStreamSynchronize(st) != cudaSuccess) {
      rs = fail(HS_ERR_CUDA, "precompute: stream sync failed");
      break;
    }
  } while (false);
  cleanup();
  return rs;
}
HS_DEFINE_CHECK_COLLECT(plan)

}  // namespace hs

extern "C" hs_status hs_plan_build_tables(hs_plan* p, const int64_t big[3], double R, const int64_t guards[3]) {
  if (!p) return fail(HS_ERR_PARAMETER, "null plan");
  if (!p->four) return fail(HS_ERR_CONFIG, "real-space-only plan (M = 0) has no tables");
  const int64_t pd[3] = {p->prm.padded[0], p->prm.padded[1], p->prm.padded[2]};
  hs_ctx* ctx = p->ctx;
  // the spectrum buffer is idle outside an evaluation: it holds the half table and the
  // precompute's intermediates as far as it goes (the cfg5-size plans leave too little free
  // device memory for separate ones)
  const size_t spec_bytes = sizeof(double2) * (size_t)std::max(p->n_in, p->n_out) * p->n_mixed;
  const size_t half_bytes = ((size_t)p->n_half * sizeof(double) + 255) & ~(size_t)255;
  double* half = nullptr;
  char* scr = nullptr;
  size_t scr_bytes = 0;
  bool own_half = false;
  HS_CUDA(cudaStreamSynchronize(ctx->stream));
  if (spec_bytes >= half_bytes) {
    half = (double*)p->spec;
    scr = (char*)p->spec + half_bytes;
    scr_bytes = spec_bytes - half_bytes;
  } else {
    HS_CUDA(cudaMalloc(&half, (size_t)p->n_half * sizeof(double)));
    own_half = true;
  }
  hs_status st = HS_OK;
  for (int kind = 0; kind < 2 && st == HS_OK; ++kind) {
    double* dst = kind == HS_BIHARMONIC ? p->tabB : p->tabH;
    if (!dst) continue;
    st = greens_half_table(ctx, kind, R, p->prm.h, big, p->prm.dims, guards, pd, half, scr, scr_bytes);
    if (st == HS_OK)
      st = launch_table_to_xmajor(ctx, half, (int)pd[0], (int)pd[1], (int)(pd[2] / 2 + 1), dst, table_kz0(p), p->nzs);
    if (st == HS_OK && cudaStreamSynchronize(ctx->stream) != cudaSuccess) st = fail(HS_ERR_CUDA, "table build");
    if (st == HS_OK) (kind == HS_BIHARMONIC ? p->have_B : p->have_H) = true;
  }
  if (own_half) cudaFree(half);
  return st;
}

namespace {

hs_status sort_points_by_cell(hs_plan* p, const double* pos, int n_src, int n_total, int mirror, int check,
                              int* order, int* start, int sub = 1) {
  hs_ctx* ctx = p->ctx;
  HS_TRY(launch_cell_keys(ctx, pos, n_src, n_total, mirror, p->cg, check, p->keys, sub));
  return counting_sort(ctx, p->keys, n_total, (int)p->cg.ncell() * sub, order, start, p->work);
}

hs_status sort_points_by_bin(hs_plan* p, const double* pos, int n_src, int n_total, int mode, int* order,
                             int* start) {
  hs_ctx* ctx = p->ctx;
  HS_TRY(launch_grid_keys(ctx, pos, n_src, n_total, mode, p->gg, p->sort_keys));
  // slab plans: spread keys of sources owned by another rank are the extra bin nbins (not
  // ranked, never read)
  if (!(mode & 8) && p->slab.world > 0)
    return counting_sort(ctx, p->sort_keys, n_total, p->nbins + 1, order, start, p->sort_work, p->nbins);
  const int nb = (mode & 8) ? gather_keys(p->gg) : p->nbins;
  return counting_sort(ctx, p->sort_keys, n_total, nb, order, start, p->sort_work);
}

}  // namespace

namespace {

// device views of the caller's inputs (mem == HOST: staged through the plan's buffers)
hs_status stage_inputs(hs_plan* p, const double* positions, const double* sa, const double* sb,
                       const double* targets, const int64_t* tcols, int mem) {
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const hs_params& prm = p->prm;
  const int n = (int)prm.n, nt = (int)prm.n_targets;
  const int kind = prm.kind;
  if (!positions || !sa) return fail(HS_ERR_PARAMETER, "null argument");
  if (kind != HS_STOKESLET && !sb) return fail(HS_ERR_PARAMETER, "stresslet/rotlet need q (mixed: g and q)");
  if (!prm.targets_are_sources && nt > 0 && !targets) return fail(HS_ERR_PARAMETER, "targets required");
  const double *pos = positions, *fa = sa, *fb = sb, *tp = targets;
  const long long* tc = (const long long*)tcols;
  if (mem == HS_MEM_HOST) {
    HS_CUDA(cudaMemcpyAsync(p->d_pos, positions, 24 * (size_t)n, cudaMemcpyHostToDevice, st));
    HS_CUDA(cudaMemcpyAsync(p->d_sa, sa, 24 * (size_t)n, cudaMemcpyHostToDevice, st));
    pos = p->d_pos;
    fa = p->d_sa;
    if (kind != HS_STOKESLET) {
      HS_CUDA(cudaMemcpyAsync(p->d_sb, sb, (kind == HS_MIXED ? 48 : 24) * (size_t)n, cudaMemcpyHostToDevice, st));
      fb = p->d_sb;
    }
    if (!prm.targets_are_sources && nt > 0) {
      HS_CUDA(cudaMemcpyAsync(p->d_tgt, targets, 24 * (size_t)nt, cudaMemcpyHostToDevice, st));
      tp = p->d_tgt;
      if (tcols) {
        HS_CUDA(cudaMemcpyAsync(p->d_tcols, tcols, 8 * (size_t)nt, cudaMemcpyHostToDevice, st));
        tc = p->d_tcols;
      }
    }
  }
  if (prm.targets_are_sources) tp = pos;
  p->cur_pos = pos;
  p->cur_fa = fa;
  p->cur_fb = fb;
  p->cur_tp = tp;
  p->cur_tc = tc;
  p->cur_tcol_identity = prm.targets_are_sources ? 1 : 0;
  return HS_OK;
}

// real-space sums (ewald_real.py:381-455) of the plan's targets into u_real / uk / uc
hs_status stage_real(hs_plan* p, bool want) {
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const hs_params& prm = p->prm;
  const int n = (int)prm.n, nt = (int)prm.n_targets, kind = prm.kind;
  const double *pos = p->cur_pos, *fa = p->cur_fa, *fb = p->cur_fb, *tp = p->cur_tp;
  const long long* tc = p->cur_tc;
  const int tcol_identity = p->cur_tcol_identity;
  const bool do_real = want && prm.rc > 0;
  if (do_real) {
    HS_TRY(sort_points_by_cell(p, pos, n, p->n_comb, p->half ? 1 : 0, 1, p->order, p->start));
    k_pair_records<<<grid_size(ctx, p->n_comb), 256, 0, st>>>(kind, p->half, p->order, p->n_comb, n, pos, fa, fb,
                                                              p->P, p->A, p->B, p->Cq, ctx->d_flags);
    HS_LAUNCHED(ctx);
    if (nt > 0) {
      // targets: reference cells, ordered by z sub-slab inside each cell (compact warps)
      HS_TRY(sort_points_by_cell(p, tp, nt, nt, 0, 0, p->t_order, p->t_start, kTargetSub));
      k_target_records<<<grid_size(ctx, nt), 256, 0, st>>>(p->t_order, nt, tp, tc, tcol_identity, p->TP, p->torig);
      HS_LAUNCHED(ctx);
      const int ncol = (int)(p->cg.dims[0] * p->cg.dims[1]);
      const int* n_items_d = nullptr;
      HS_TRY(build_pair_items(ctx, p->t_start, ncol, (int)p->cg.dims[2] * kTargetSub, p->work, p->items,
                              &n_items_d));
      PairArgs a{};
      a.P = p->P;
      a.A = p->A;
      a.B = p->B;
      a.C = p->Cq;
      a.start = p->start;
      a.TP = p->TP;
      a.torig = p->torig;
      a.t_start = p->t_start;
      a.t_sub = kTargetSub;
      a.items = p->items;
      a.max_items = nt / 128 + ncol + 1;
      a.n_items_d = n_items_d;
      for (int k = 0; k < 3; ++k) a.dims[k] = (int)p->cg.dims[k];
      a.cz_lo = p->cg.lo[2];
      a.cz_edge = p->cg.edge[2];
      a.xi = prm.xi;
      a.rc2 = prm.rc * prm.rc;
      {
        // FP32 prefilter bound: relative FP32 coordinates err by < 2^-22 * (box size); keep a wide margin
        const double box = 3.0 * prm.L;
        const double rch = prm.rc * (1.0 + 1e-4) + box * std::ldexp(1.0, -20);
        a.rc2_hi = (float)(rch * rch) * (1.0f + 1e-6f);
        const double rcl = prm.rc * (1.0 - 1e-4) - box * std::ldexp(1.0, -20);
        a.rc2_lo = rcl > 0 ? (float)(rcl * rcl) * (1.0f - 1e-6f) : 0.0f;
      }
      a.n_real = n;
      a.kind = kind | (p->half ? 16 : 0);
      a.self_f = (kind == HS_STOKESLET || kind == HS_MIXED) ? fa : nullptr;
      a.u = p->u_real;
      a.uk = p->uk;
      a.uc = p->uc;
      a.flags = ctx->d_flags;
      a.counts = p->pair_counts;
      a.work = reinterpret_cast<int*>(p->pair_counts + 2);
      a.audit = p->audit;
      HS_CUDA(cudaMemsetAsync(p->pair_counts, 0, 3 * sizeof(unsigned long long), st));
      HS_CUDA(cudaEventRecord(p->ev[9], st));
      HS_TRY(launch_pair(ctx, a));
      HS_CUDA(cudaEventRecord(p->ev[10], st));
      p->pair_timed = true;
    }
  } else if (nt > 0) {
    HS_CUDA(cudaMemsetAsync(p->u_real, 0, 24 * (size_t)nt, st));
    HS_CUDA(cudaMemsetAsync(p->uk, 0, 24 * (size_t)nt, st));
    HS_CUDA(cudaMemsetAsync(p->uc, 0, 24 * (size_t)nt, st));
    if (want && (kind == HS_STOKESLET || kind == HS_MIXED)) {
      // rc = 0: no pairs, but the self term is still added (ewald_real.py:444-449)
      k_self_term<<<grid_size(ctx, nt), 256, 0, st>>>(nt, tp, tc, tcol_identity, n, prm.xi, fa, p->u_real);
      HS_LAUNCHED(ctx);
    }
  }
  return HS_OK;
}


// half space: spread the N sources with kernel + wall channels, then mirror (k_mirror_z).
// group gi: channels [group_c0[gi], group_c0[gi+1]) into grid_in channels 0.. (the sort and
// the records are made with group 0; later groups reuse them and the spread's window tables)
hs_status stage_spread_group(hs_plan* p, int gi) {
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int c0 = p->group_c0[gi], c1 = p->group_c0[gi + 1], cn = c1 - c0;
  if (gi > 0) {
    HS_CUDA(cudaEventRecord(p->ev[11], st));
    HS_TRY(launch_spread(ctx, p->SPk, p->SWk + c0, p->n_sel_k, cn, p->bk_start, p->gg, p->grid_in, p->n_in,
                         p->ngroup > 1, p->spread_tz0));
    if (p->mirror && !p->mirror_in_z) {
      const int64_t lines = (int64_t)p->gg.dims[1] * p->gg.dims[0];
      const int nz = p->gg.dims[2];
      k_mirror_z<<<grid_size(ctx, lines * (nz / 2 + 1) * cn), 256, 0, st>>>(
          p->grid_in, cn, p->kern_mask >> c0, p->sigma_mask >> c0, p->gg.ch_stride, lines, p->kg.p[2], nz);
      HS_LAUNCHED(ctx);
    }
    HS_CUDA(cudaEventRecord(p->ev[12], st));
    return HS_OK;
  }
  return HS_OK;
}

hs_status stage_spread_mirrored(hs_plan* p) {
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const hs_params& prm = p->prm;
  const int n = (int)prm.n, kind = prm.kind;
  HS_TRY(sort_points_by_bin(p, p->cur_pos, n, n, 0, p->bk_order, p->bk_start));
  int n_sel = n;
  if (p->slab.world > 0) {
    HS_CUDA(cudaMemcpyAsync(&n_sel, p->bk_start + p->nbins, sizeof(int), cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
  }
  p->n_sel_k = n_sel;
  p->n_sel_c = 0;
  if (n_sel > 0) {
    k_spread_records<<<grid_size(ctx, n_sel), 256, 0, st>>>(kind, 1, 2, p->bk_order, n_sel, n, p->cur_pos, p->cur_fa,
                                                            p->cur_fb, p->n_in, p->SPk, p->SWk);
    HS_LAUNCHED(ctx);
  }
  HS_CUDA(cudaEventRecord(p->ev[11], st));
  const int cn = p->group_c0[1];
  HS_TRY(launch_spread(ctx, p->SPk, p->SWk, n_sel, cn, p->bk_start, p->gg, p->grid_in, p->n_in, false,
                       p->spread_tz0));
  if (!p->mirror_in_z) {
    const int64_t lines = (int64_t)p->gg.dims[1] * p->gg.dims[0];
    const int nz = p->gg.dims[2];
    k_mirror_z<<<grid_size(ctx, lines * (nz / 2 + 1) * cn), 256, 0, st>>>(
        p->grid_in, cn, p->kern_mask, p->sigma_mask, p->gg.ch_stride, lines, p->kg.p[2], nz);
    HS_LAUNCHED(ctx);
  }
  HS_CUDA(cudaEventRecord(p->ev[12], st));
  p->spread_timed = true;
  return HS_OK;
}

// spreading of kernel sources [y; y^I] (or y) and wall-correction sources y^I into grid_in
// (ewald_fourier.py:319-332,353-382); a slab plan keeps the sources whose y window starts
// in its slab (k_grid_keys drop bin)
hs_status stage_spread(hs_plan* p) {
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const hs_params& prm = p->prm;
  const int n = (int)prm.n, kind = prm.kind;
  const double *pos = p->cur_pos, *fa = p->cur_fa, *fb = p->cur_fb;
  const bool sl = p->slab.world > 0;
  if (p->mirror) return stage_spread_mirrored(p);
  HS_TRY(sort_points_by_bin(p, pos, n, p->n_comb, p->half ? 1 : 0, p->bk_order, p->bk_start));
  if (p->nc) HS_TRY(sort_points_by_bin(p, pos, n, n, 2, p->bc_order, p->bc_start));
  int nk_sel = p->n_comb, nc_sel = n;
  if (sl) {
    // selected sources lead the bin order: their count is the start of the drop bin
    int cnt[2] = {0, 0};
    HS_CUDA(cudaMemcpyAsync(&cnt[0], p->bk_start + p->nbins, sizeof(int), cudaMemcpyDeviceToHost, st));
    if (p->nc) HS_CUDA(cudaMemcpyAsync(&cnt[1], p->bc_start + p->nbins, sizeof(int), cudaMemcpyDeviceToHost, st));
    HS_CUDA(cudaStreamSynchronize(st));
    nk_sel = cnt[0];
    nc_sel = cnt[1];
  }
  if (nk_sel > 0) {
    k_spread_records<<<grid_size(ctx, nk_sel), 256, 0, st>>>(kind, p->half, 0, p->bk_order, nk_sel, n, pos, fa, fb,
                                                             p->nk, p->SPk, p->SWk);
    HS_LAUNCHED(ctx);
  }
  if (kind == HS_MIXED) {  // free space: group 0 = F now, the stresslet channels by stage_spread_group
    p->n_sel_k = nk_sel;
    p->n_sel_c = 0;
    HS_CUDA(cudaEventRecord(p->ev[11], st));
    HS_TRY(launch_spread(ctx, p->SPk, p->SWk, nk_sel, p->group_c0[1], p->bk_start, p->gg, p->grid_in, p->nk));
    HS_CUDA(cudaEventRecord(p->ev[12], st));
    p->spread_timed = true;
    return HS_OK;
  }
  if (p->nc && nc_sel > 0) {
    k_spread_records<<<grid_size(ctx, nc_sel), 256, 0, st>>>(kind, p->half, 1, p->bc_order, nc_sel, n, pos, fa, fb,
                                                             p->nc, p->SPc, p->SWc);
    HS_LAUNCHED(ctx);
  }
  p->n_sel_k = nk_sel;
  p->n_sel_c = nc_sel;
  HS_CUDA(cudaEventRecord(p->ev[11], st));
  HS_TRY(launch_spread(ctx, p->SPk, p->SWk, nk_sel, p->nk, p->bk_start, p->gg, p->grid_in));
  if (p->nc)
    HS_TRY(launch_spread(ctx, p->SPc, p->SWc, nc_sel, p->nc, p->bc_start, p->gg, p->grid_in + (size_t)p->nk * p->n_grid));
  HS_CUDA(cudaEventRecord(p->ev[12], st));
  p->spread_timed = true;
  return HS_OK;
}

void set_fft_streams(hs_plan* p) {
  cufftSetStream(p->zf, p->ctx->stream);
  cufftSetStream(p->yf, p->ctx->stream);
  cufftSetStream(p->zi, p->ctx->stream);
}

// forward y transform of one channel: rows y < ny of `in` ([py][nx][nzs]) -> spec channel c
hs_status stage_yfwd(hs_plan* p, double2* in, int c) {
  double2* out = p->spec + (size_t)c * p->n_mixed;
  if (p->ytw)
    return launch_ystage(p->ctx, true, in, out, p->ytw, p->kg.p[1], p->gg.dims[0], p->nzs, (int)p->prm.dims[1]);
  if (cufftExecZ2Z(p->yf, (cufftDoubleComplex*)in, (cufftDoubleComplex*)out, CUFFT_FORWARD) != CUFFT_SUCCESS)
    return fail(HS_ERR_CUDA, "cuFFT y Z2Z failed");
  return HS_OK;
}

// inverse y transform of output channel o: rows y < ny written to `out` ([ny][nx][nzs] rows)
hs_status stage_yinv(hs_plan* p, int o, double2* out) {
  double2* so = p->spec + (size_t)o * p->n_mixed;
  const int ny = (int)p->prm.dims[1];
  if (p->ytw) return launch_ystage(p->ctx, false, so, out, p->ytw, p->kg.p[1], p->gg.dims[0], p->nzs, ny);
  if (cufftExecZ2Z(p->yf, (cufftDoubleComplex*)so, (cufftDoubleComplex*)so, CUFFT_INVERSE) != CUFFT_SUCCESS)
    return fail(HS_ERR_CUDA, "cuFFT y^-1 failed");
  if (out != so)
    HS_CUDA(cudaMemcpyAsync(out, so, sizeof(double2) * (size_t)ny * p->gg.dims[0] * p->nzs, cudaMemcpyDeviceToDevice,
                            p->ctx->stream));
  return HS_OK;
}

hs_status stage_xstage(hs_plan* p) {
  XArgs xa{};
  xa.B = p->spec;
  xa.Bout = p->spec;
  xa.accum = 0;
  xa.ch_stride = p->n_mixed;
  xa.tabB = p->tabB;
  xa.tabH = p->tabH;
  xa.tw = p->tw;
  xa.plan = p->xplan;
  xa.px = p->kg.p[0];
  xa.py = p->kg.p[1];
  xa.pz = p->kg.p[2];
  xa.nzh = p->nzs;
  xa.kz0 = p->slab.world > 0 ? (int)p->slab.kz0 : 0;
  xa.nx = p->gg.dims[0];
  for (int k = 0; k < 3; ++k) xa.kscale[k] = p->kg.kscale[k];
  xa.ka = p->kg.a;
  xa.kb = p->kg.b;
  xa.inv_n = p->kg.inv_n;
  HS_TRY(launch_xfused(p->ctx, p->prm.kind, p->half, xa));
  if (p->prm.kind == HS_MIXED) {
    // second channel group (kmult.cuh): the stresslet kernel channels, scaled without wall
    // channels, added to T1 (spec channels 0..2, the first pass's outputs)
    xa.B = p->spec + (size_t)(p->half ? 13 : 3) * p->n_mixed;
    xa.accum = 1;
    HS_TRY(launch_xfused(p->ctx, HS_STRESSLET, 0, xa));
  }
  return HS_OK;
}

// Fourier gather at the plan's targets: u_four, and u = u_real + u_four (ewald_fourier.py:626-630)
hs_status stage_gather(hs_plan* p) {
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int nt = (int)p->prm.n_targets;
  if (nt == 0) return HS_OK;
  HS_TRY(sort_points_by_bin(p, p->cur_tp, nt, nt, 8, p->bt_order, p->bt_start));
  k_gather_records<<<grid_size(ctx, nt), 256, 0, st>>>(p->bt_order, nt, p->cur_tp, p->TG, p->tg_orig);
  HS_LAUNCHED(ctx);
  HS_CUDA(cudaEventRecord(p->ev[13], st));
  HS_TRY(launch_gather_fourier(ctx, p->TG, p->tg_orig, nt, p->half ? 1 : 0, p->go, p->grid_out, p->u_four, p->u,
                               p->u_real, p->bt_start));
  HS_CUDA(cudaEventRecord(p->ev[14], st));
  p->gather_timed = true;
  return HS_OK;
}

hs_status stage_outputs(hs_plan* p, double* u, double* u_real, double* u_fourier, int mem) {
  cudaStream_t st = p->ctx->stream;
  const int nt = (int)p->prm.n_targets;
  const cudaMemcpyKind ok = mem == HS_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (nt > 0) {
    HS_CUDA(cudaMemcpyAsync(u, p->u, 24 * (size_t)nt, ok, st));
    if (u_real) HS_CUDA(cudaMemcpyAsync(u_real, p->u_real, 24 * (size_t)nt, ok, st));
    if (u_fourier) HS_CUDA(cudaMemcpyAsync(u_fourier, p->u_four, 24 * (size_t)nt, ok, st));
  }
  return HS_OK;
}

void fill_times(hs_plan* p, double* times, bool overlapped = false) {
  cudaEvent_t* ev = p->ev;
  float ms[9] = {0};
  for (int k = 0; k < 8; ++k) cudaEventElapsedTime(&ms[k], ev[k], ev[k + 1]);
  float tot = 0;
  cudaEventElapsedTime(&tot, ev[0], ev[8]);
  float fourier = 0;
  cudaEventElapsedTime(&fourier, ev[2], ev[7]);
  if (overlapped) {
    // both pipelines start at ev[1]: real = ev1 -> ev2 (context stream), gridding = ev1 -> ev3
    // (Fourier stream), gather = join -> ev7; the phases overlap, so they no longer sum to total
    cudaEventElapsedTime(&ms[2], ev[1], ev[3]);
    float g0 = 0;
    cudaEventElapsedTime(&g0, ev[6], ev[7]);
    float r = 0;
    cudaEventElapsedTime(&r, ev[1], ev[2]);
    ms[1] = r;
    float lastjoin = 0;  // gather proper: from the later of (real end, Fourier end)
    cudaEventElapsedTime(&lastjoin, ev[2], ev[7]);
    ms[6] = std::min(g0, lastjoin);
    cudaEventElapsedTime(&fourier, ev[1], ev[7]);
  }
  // [gridding, fft, scale, ifft, gather, real, fourier, prep, total, io]
  times[0] = ms[2];
  times[1] = ms[3];
  times[2] = ms[4];
  times[3] = ms[5];
  times[4] = ms[6];
  times[5] = ms[1];
  times[6] = fourier;
  times[7] = ms[0];
  times[8] = tot;
  times[9] = ms[7] + ms[0];
  float kp = 0, ks = 0, kg = 0;
  if (p->pair_timed) cudaEventElapsedTime(&kp, ev[9], ev[10]);
  if (p->spread_timed) cudaEventElapsedTime(&ks, ev[11], ev[12]);
  if (p->gather_timed) cudaEventElapsedTime(&kg, ev[13], ev[14]);
  // kernel-only times: [10] pair, [11] spread, [12] gather, [13] scale
  times[10] = kp;
  times[11] = ks;
  times[12] = kg;
  times[13] = ms[4];
  unsigned long long cnt[2] = {0, 0};
  if (p->pair_timed) cudaMemcpy(cnt, p->pair_counts, sizeof(cnt), cudaMemcpyDeviceToHost);
  times[14] = (double)cnt[0];  // accepted pairs
  times[15] = (double)cnt[1];  // accepted image pairs
}

hs_status begin_eval(hs_plan* p) {
  HS_CUDA(cudaSetDevice(p->ctx->device));
  HS_TRY(ctx_reset_flags(p->ctx));
  p->pair_timed = p->spread_timed = p->gather_timed = false;
  return HS_OK;
}

}  // namespace

extern "C" hs_status hs_plan_execute(hs_plan* p, const double* positions, const double* sa, const double* sb,
                                     const double* targets, const int64_t* tcols, double* u, double* u_real,
                                     double* u_fourier, int mem, int what, double* times) {
  if (!p || !positions || !sa || !u) return fail(HS_ERR_PARAMETER, "null argument");
  if (p->slab.world > 0) return fail(HS_ERR_PARAMETER, "slab plans evaluate through the hs_slab_* stages");
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int nt = (int)p->prm.n_targets;
  if ((what & 2) && !p->four) return fail(HS_ERR_CONFIG, "real-space-only plan (M = 0): no Fourier part");
  if ((what & 2) && (p->tabB && !p->have_B)) return fail(HS_ERR_CONFIG, "missing biharmonic table");
  if ((what & 2) && (p->tabH && !p->have_H)) return fail(HS_ERR_CONFIG, "missing harmonic table");
  HS_TRY(begin_eval(p));
  cudaEvent_t* ev = p->ev;
  HS_CUDA(cudaEventRecord(ev[0], st));
  HS_TRY(stage_inputs(p, positions, sa, sb, targets, tcols, mem));
  HS_CUDA(cudaEventRecord(ev[1], st));
  // The real-space pipeline (FP64 pair kernel) and the Fourier pipeline up to the gather are
  // independent: with both requested, the Fourier side is issued on the plan's high-priority
  // stream (its own sort buffers; the context stream is switched while its launches are
  // issued) and runs concurrently with the pair kernel, filling the SM slots and pipes the
  // pair kernel leaves idle; the gather, which adds u_real, waits for both.
  // HS_NO_OVERLAP=1: one stream (comparison).
  static const bool overlap_env = getenv("HS_NO_OVERLAP") == nullptr;
  const bool two = overlap_env && (what & 3) == 3 && !(what & 4);  // what bit 2: serialise (kernel timing)
  auto fourier_to_gather = [&]() -> hs_status {
    HS_TRY(stage_spread(p));
    HS_CUDA(cudaEventRecord(ev[3], ctx->stream));
    set_fft_streams(p);
    // forward z (D2Z) and y stages, one source channel at a time through the shared A buffer;
    // channel groups (mixed): spread the next group into the freed source grids
    for (int gi = 0; gi < p->ngroup; ++gi) {
      if (gi > 0) HS_TRY(stage_spread_group(p, gi));
      for (int c = p->group_c0[gi]; c < p->group_c0[gi + 1]; ++c) {
        const double* gin = p->grid_in + (size_t)(c - p->group_c0[gi]) * p->n_grid;
        if (p->ztw) {
          const int mir = !p->mirror_in_z ? 0 : (((p->kern_mask >> c) & 1u) ? 1 : 2);
          HS_TRY(launch_zfwd(ctx, p->kg.p[2], gin, p->Amix, p->ztw, (int64_t)p->gg.dims[1] * p->gg.dims[0], p->gg.dims[2], mir,
                             ((p->sigma_mask >> c) & 1u) ? -1.0 : 1.0, p->spread_tz0 * SP_TZ));
        }
        else if (cufftExecD2Z(p->zf, (double*)gin, (cufftDoubleComplex*)p->Amix) != CUFFT_SUCCESS)
          return fail(HS_ERR_CUDA, "cuFFT z D2Z failed");
        HS_TRY(stage_yfwd(p, p->Amix, c));
      }
    }
    HS_CUDA(cudaEventRecord(ev[4], ctx->stream));
    HS_TRY(stage_xstage(p));
    HS_CUDA(cudaEventRecord(ev[5], ctx->stream));
    for (int o = 0; o < p->n_out; ++o) {
      double2* so = p->spec + (size_t)o * p->n_mixed;
      HS_TRY(stage_yinv(p, o, so));
      if (!p->ztw &&
          cufftExecZ2D(p->zi, (cufftDoubleComplex*)so, p->grid_tmp + (size_t)o * p->n_grid) != CUFFT_SUCCESS)
        return fail(HS_ERR_CUDA, "cuFFT z Z2D failed");
    }
    if (p->ztw) {
      // inverse z of all output channels, written channel-interleaved (z < nz) for the gather
      HS_TRY(launch_zinv_interleaved(ctx, p->kg.p[2], p->spec, (int64_t)p->n_mixed, p->n_out, p->out_pitch, p->grid_out, p->ztw,
                                     (int64_t)p->gg.dims[1] * p->gg.dims[0], p->gg.dims[2]));
    } else {
      // channel-interleave the (y < ny, x < nx, z < nz) outputs for the broadcast gather
      k_interleave<<<grid_size(ctx, p->n_grid / 2), 256, 0, ctx->stream>>>(p->grid_tmp, p->n_out, p->n_grid,
                                                                           p->n_grid, p->out_pitch, p->grid_out);
      HS_LAUNCHED(ctx);
    }
    if (p->tmp_aliased) {
      // the inverse z transforms wrote whole pz lines into the source grids: restore their zero
      // z padding (the next spread writes z < nz only)
      const int nz = p->gg.dims[2], pz = p->kg.p[2];
      const size_t lines = (size_t)p->gg.dims[1] * p->gg.dims[0];
      HS_CUDA(cudaMemset2DAsync(p->grid_in + nz, sizeof(double) * pz, 0, sizeof(double) * (pz - nz),
                                lines * p->n_out, ctx->stream));
    }
    HS_CUDA(cudaEventRecord(ev[6], ctx->stream));
    return HS_OK;
  };
  // HS_OVERLAP_FOURIER_HI=1: the Fourier side on the high-priority stream (default: the
  // real-space side there, so the pair kernel keeps its slots and the Fourier kernels fill in)
  static const bool fourier_hi = getenv("HS_OVERLAP_FOURIER_HI") != nullptr;
  hs_status fst = HS_OK;
  if (two) {
    HS_CUDA(cudaStreamWaitEvent(p->st_four, ev[1], 0));
    ctx->stream = p->st_four;
    if (fourier_hi) {
      p->sort_keys = p->keys_f;
      p->sort_work = p->work_f;
      fst = fourier_to_gather();
    } else {
      fst = stage_real(p, (what & 1) != 0);
      if (fst == HS_OK && cudaEventRecord(ev[2], p->st_four) != cudaSuccess) fst = fail(HS_ERR_CUDA, "event");
    }
    if (fst == HS_OK && cudaEventRecord(p->ev_four, p->st_four) != cudaSuccess) fst = fail(HS_ERR_CUDA, "event");
    ctx->stream = st;
    p->sort_keys = p->keys;
    p->sort_work = p->work;
    set_fft_streams(p);
    HS_TRY(fst);
    if (!fourier_hi) {
      p->sort_keys = p->keys_f;
      p->sort_work = p->work_f;
      fst = fourier_to_gather();
      p->sort_keys = p->keys;
      p->sort_work = p->work;
      HS_TRY(fst);
    }
  }
  if (!two || fourier_hi) {
    HS_TRY(stage_real(p, (what & 1) != 0));
    HS_CUDA(cudaEventRecord(ev[2], st));
  }
  if (what & 2) {
    if (two) HS_CUDA(cudaStreamWaitEvent(st, p->ev_four, 0));
    else HS_TRY(fourier_to_gather());
    HS_TRY(stage_gather(p));
  } else {
    for (int k = 3; k <= 6; ++k) HS_CUDA(cudaEventRecord(ev[k], st));
    if (nt > 0) {
      HS_CUDA(cudaMemsetAsync(p->u_four, 0, 24 * (size_t)nt, st));
      HS_CUDA(cudaMemcpyAsync(p->u, p->u_real, 24 * (size_t)nt, cudaMemcpyDeviceToDevice, st));
    }
  }
  HS_CUDA(cudaEventRecord(ev[7], st));
  HS_TRY(stage_outputs(p, u, u_real, u_fourier, mem));
  HS_CUDA(cudaEventRecord(ev[8], st));
  HS_CUDA(cudaStreamSynchronize(st));
  HS_TRY(ctx_check_flags(ctx, "hs_plan_execute"));
  if (times) fill_times(p, times, two);
  return HS_OK;
}

// ---------------------------------------------------------------------------
// y-slab stages (see hsewald_b200.h).  Every stage is stream-ordered on the context's
// stream; the caller's exchanges must be ordered on the same stream (sharding.py binds
// the context to torch's current stream).

extern "C" hs_status hs_plan_pair_audit(hs_plan* p, const double* positions, const double* sa, const double* sb,
                                        const double* targets, const int64_t* tcols, uint64_t* audit, int mem) {
  if (!p || !positions || !sa || !audit) return fail(HS_ERR_PARAMETER, "null argument");
  if (!(p->prm.rc > 0)) return fail(HS_ERR_PARAMETER, "pair audit needs rc > 0");
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const size_t nt = (size_t)p->prm.n_targets, bytes = 3 * sizeof(unsigned long long) * std::max<size_t>(nt, 1);
  HS_TRY(begin_eval(p));
  HS_TRY(stage_inputs(p, positions, sa, sb, targets, tcols, mem));
  unsigned long long* buf = nullptr;
  if (mem == HS_MEM_DEVICE) buf = (unsigned long long*)audit;
  else HS_CUDA(cudaMallocAsync(&buf, bytes, st));
  HS_CUDA(cudaMemsetAsync(buf, 0, bytes, st));
  p->audit = buf;
  hs_status rs = stage_real(p, true);
  p->audit = nullptr;
  if (rs == HS_OK && mem == HS_MEM_HOST && nt)
    if (cudaMemcpyAsync(audit, buf, 3 * sizeof(unsigned long long) * nt, cudaMemcpyDeviceToHost, st) != cudaSuccess)
      rs = fail(HS_ERR_CUDA, "audit copy");
  if (mem == HS_MEM_HOST) cudaFreeAsync(buf, st);
  HS_TRY(rs);
  HS_CUDA(cudaStreamSynchronize(st));
  return ctx_check_flags(ctx, "hs_plan_pair_audit");
}

namespace {

// kz split / merge between the z-stage layout [rows][nzh] and per-rank blocks [W][rows][kz_s]
// (the all-to-all send / receive layout).  dir 0: split (lines -> blocks), 1: merge.
struct KzSplit {
  int w;
  int b[65];
};
__global__ void k_kz_exchange(double2* __restrict__ lines, double2* __restrict__ blocks, int64_t rows, int nzh,
                              KzSplit ks, int dir) {
  const int64_t n = rows * nzh;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / nzh;
    const int kz = (int)(i - r * nzh);
    int s = 0;
    while (s + 1 < ks.w && kz >= ks.b[s + 1]) ++s;
    const int w = ks.b[s + 1] - ks.b[s];
    const int64_t bi = (int64_t)ks.b[s] * rows + r * w + (kz - ks.b[s]);  // block s starts at rows * b[s]
    if (dir == 0) blocks[bi] = lines[i];
    else lines[i] = blocks[bi];
  }
}

// grid[c][y < P-1][x][z < nz] += ghost[c][y][x][z]
__global__ void k_ghost_add(double* __restrict__ grid, const double* __restrict__ ghost, int nch, int planes, int nx,
                            int nz, int pz, int64_t ch_stride) {
  const int64_t per = (int64_t)planes * nx * nz, n = per * nch;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int c = (int)(i / per);
    const int64_t r = i - c * per;
    const int64_t line = r / nz;
    const int z = (int)(r - line * nz);
    grid[c * ch_stride + line * pz + z] += ghost[i];
  }
}

KzSplit kz_split_of(const hs_plan* p) {
  KzSplit ks{};
  ks.w = (int)p->slab.world;
  for (int s = 0; s <= ks.w; ++s) ks.b[s] = (int)p->slab.kz_split[s];
  return ks;
}

hs_status check_slab(const hs_plan* p) {
  if (!p) return fail(HS_ERR_PARAMETER, "null plan");
  if (p->slab.world <= 0) return fail(HS_ERR_PARAMETER, "not a slab plan");
  return HS_OK;
}

}  // namespace

extern "C" hs_status hs_slab_sizes(const hs_plan* p, int64_t sizes[8]) {
  HS_TRY(check_slab(p));
  const int64_t nx = p->gg.dims[0], nz = p->prm.dims[2], P1 = p->prm.P - 1;
  const int64_t nzh = p->kg.nzh;
  sizes[0] = (int64_t)p->n_in * P1 * nx * nz;
  sizes[1] = 2 * (int64_t)p->yo * nx * nzh;
  sizes[2] = 2 * (int64_t)p->kg.p[1] * nx * p->nzs;
  sizes[3] = 2 * p->prm.dims[1] * nx * p->nzs;
  sizes[4] = P1 * nx * nz * p->out_pitch;
  sizes[5] = p->n_in;
  sizes[6] = p->n_out;
  sizes[7] = p->out_pitch;
  return HS_OK;
}

extern "C" hs_status hs_slab_begin(hs_plan* p, const double* positions, const double* sa, const double* sb,
                                   const double* targets, const int64_t* tcols, int mem, double* ghost_out) {
  HS_TRY(check_slab(p));
  if (!ghost_out) return fail(HS_ERR_PARAMETER, "null ghost buffer");
  if ((p->tabB && !p->have_B) || (p->tabH && !p->have_H)) return fail(HS_ERR_CONFIG, "missing Green's table");
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  HS_TRY(begin_eval(p));
  cudaEvent_t* ev = p->ev;
  HS_CUDA(cudaEventRecord(ev[0], st));
  HS_TRY(stage_inputs(p, positions, sa, sb, targets, tcols, mem));
  HS_CUDA(cudaEventRecord(ev[1], st));
  HS_TRY(stage_real(p, true));
  HS_CUDA(cudaEventRecord(ev[2], st));
  HS_TRY(stage_spread(p));
  // ghost planes [yo, yo + P - 1) of every channel, z compacted to nz
  const int64_t nx = p->gg.dims[0], nz = p->prm.dims[2], pz = p->kg.p[2], P1 = p->prm.P - 1;
  for (int c = 0; c < p->n_in; ++c)
    HS_CUDA(cudaMemcpy2DAsync(ghost_out + (size_t)c * P1 * nx * nz, nz * 8,
                              p->grid_in + (size_t)c * p->n_grid + (size_t)p->yo * nx * pz, pz * 8, nz * 8, P1 * nx,
                              cudaMemcpyDeviceToDevice, st));
  HS_CUDA(cudaEventRecord(ev[3], st));
  return HS_OK;
}

// Channel-range forms of the middle stages, so a caller can overlap the all-to-all of channel
// c with the transforms of channel c+1 (sharding.py issues the collectives asynchronously).
extern "C" hs_status hs_slab_forward_range(hs_plan* p, const double* ghost_in, double* send, int c0, int c1) {
  HS_TRY(check_slab(p));
  if (!send) return fail(HS_ERR_PARAMETER, "null send buffer");
  if (c0 < 0 || c1 > p->n_in || c0 > c1) return fail(HS_ERR_PARAMETER, "channel range");
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t nx = p->gg.dims[0], nz = p->prm.dims[2], pz = p->kg.p[2], P1 = p->prm.P - 1;
  if (c0 == 0 && ghost_in && P1 > 0) {
    k_ghost_add<<<grid_size(ctx, p->n_in * P1 * nx * nz), 256, 0, st>>>(p->grid_in, ghost_in, p->n_in, (int)P1,
                                                                        (int)nx, (int)nz, (int)pz, p->gg.ch_stride);
    HS_LAUNCHED(ctx);
  }
  set_fft_streams(p);
  const KzSplit ks = kz_split_of(p);
  const int64_t rows = (int64_t)p->yo * nx;
  for (int c = c0; c < c1; ++c) {
    if (p->ztw)
      HS_TRY(launch_zfwd(ctx, (int)pz, p->grid_in + (size_t)c * p->n_grid, p->Amix, p->ztw, rows, (int)nz));
    else if (cufftExecD2Z(p->zf, p->grid_in + (size_t)c * p->n_grid, (cufftDoubleComplex*)p->Amix) != CUFFT_SUCCESS)
      return fail(HS_ERR_CUDA, "cuFFT z D2Z failed");
    k_kz_exchange<<<grid_size(ctx, rows * p->kg.nzh), 256, 0, st>>>(
        p->Amix, (double2*)send + (size_t)c * p->n_amix, rows, p->kg.nzh, ks, 0);
    HS_LAUNCHED(ctx);
  }
  return HS_OK;
}

extern "C" hs_status hs_slab_forward(hs_plan* p, const double* ghost_in, double* send) {
  HS_TRY(check_slab(p));
  return hs_slab_forward_range(p, ghost_in, send, 0, p->n_in);
}

// part 0: y transforms of input channels [c0, c1) from recv; part 1: the x stage (c0, c1
// ignored); part 2: inverse y transforms of output channels [c0, c1) into back
extern "C" hs_status hs_slab_kspace_part(hs_plan* p, int part, const double* recv, double* back, int c0, int c1) {
  HS_TRY(check_slab(p));
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  set_fft_streams(p);
  if (part == 0) {
    if (!recv || c0 < 0 || c1 > p->n_in || c0 > c1) return fail(HS_ERR_PARAMETER, "kspace part 0 arguments");
    for (int c = c0; c < c1; ++c) HS_TRY(stage_yfwd(p, (double2*)recv + (size_t)c * p->n_mixed, c));
    if (c1 == p->n_in) HS_CUDA(cudaEventRecord(p->ev[4], st));
    return HS_OK;
  }
  if (part == 1) {
    HS_TRY(stage_xstage(p));
    HS_CUDA(cudaEventRecord(p->ev[5], st));
    return HS_OK;
  }
  if (part != 2 || !back || c0 < 0 || c1 > p->n_out || c0 > c1) return fail(HS_ERR_PARAMETER, "kspace part arguments");
  const size_t back_ch = (size_t)p->prm.dims[1] * p->gg.dims[0] * p->nzs;
  for (int o = c0; o < c1; ++o) HS_TRY(stage_yinv(p, o, (double2*)back + o * back_ch));
  return HS_OK;
}

extern "C" hs_status hs_slab_kspace(hs_plan* p, const double* recv, double* back) {
  HS_TRY(check_slab(p));
  if (!recv || !back) return fail(HS_ERR_PARAMETER, "null exchange buffer");
  // phase events: fft = z + exchange + y, scale = x stage, ifft = y^-1 + exchange + z^-1
  HS_TRY(hs_slab_kspace_part(p, 0, recv, back, 0, p->n_in));
  HS_TRY(hs_slab_kspace_part(p, 1, recv, back, 0, 0));
  return hs_slab_kspace_part(p, 2, recv, back, 0, p->n_out);
}

// inverse z transforms of output channels [o0, o1); the call with o1 == n_out also interleaves
// the owned planes and writes the halo for rank r-1
extern "C" hs_status hs_slab_backward_range(hs_plan* p, const double* recv_back, double* halo_out, int o0, int o1) {
  HS_TRY(check_slab(p));
  if (!recv_back || (o1 == p->n_out && !halo_out)) return fail(HS_ERR_PARAMETER, "null exchange buffer");
  if (o0 < 0 || o1 > p->n_out || o0 > o1) return fail(HS_ERR_PARAMETER, "channel range");
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  set_fft_streams(p);
  const int64_t nx = p->gg.dims[0], nz = p->prm.dims[2], pz = p->kg.p[2], P1 = p->prm.P - 1;
  const KzSplit ks = kz_split_of(p);
  const int64_t rows = (int64_t)p->yo * nx;
  for (int o = o0; o < o1; ++o) {
    k_kz_exchange<<<grid_size(ctx, rows * p->kg.nzh), 256, 0, st>>>(
        p->Amix, (double2*)recv_back + (size_t)o * p->n_amix, rows, p->kg.nzh, ks, 1);
    HS_LAUNCHED(ctx);
    if (p->ztw)  // one channel, plain lines of pitch pz (z < nz written; the padding stays zero)
      HS_TRY(launch_zinv_interleaved(ctx, (int)pz, p->Amix, 0, 1, 1, p->grid_tmp + (size_t)o * p->n_grid, p->ztw, rows, (int)nz));
    else if (cufftExecZ2D(p->zi, (cufftDoubleComplex*)p->Amix, p->grid_tmp + (size_t)o * p->n_grid) != CUFFT_SUCCESS)
      return fail(HS_ERR_CUDA, "cuFFT z Z2D failed");
  }
  if (o1 < p->n_out) return HS_OK;
  // interleave the owned planes; the ghost planes are filled by hs_slab_finish
  const int64_t n_owned = rows * pz;
  k_interleave<<<grid_size(ctx, n_owned / 2), 256, 0, st>>>(p->grid_tmp, p->n_out, p->n_grid, n_owned,
                                                            p->out_pitch, p->grid_out);
  HS_LAUNCHED(ctx);
  // halo for rank r-1: output planes [0, P-1), z compacted
  const int pitch = p->out_pitch;
  HS_CUDA(cudaMemcpy2DAsync(halo_out, nz * pitch * 8, p->grid_out, pz * pitch * 8, nz * pitch * 8, P1 * nx,
                            cudaMemcpyDeviceToDevice, st));
  HS_CUDA(cudaEventRecord(p->ev[6], st));
  return HS_OK;
}

extern "C" hs_status hs_slab_backward(hs_plan* p, const double* recv_back, double* halo_out) {
  HS_TRY(check_slab(p));
  return hs_slab_backward_range(p, recv_back, halo_out, 0, p->n_out);
}

extern "C" hs_status hs_slab_finish(hs_plan* p, const double* halo_in, double* u, double* u_real, double* u_fourier,
                                    int mem, double* times) {
  HS_TRY(check_slab(p));
  if (!u) return fail(HS_ERR_PARAMETER, "null output");
  hs_ctx* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  const int64_t nx = p->gg.dims[0], nz = p->prm.dims[2], pz = p->kg.p[2], P1 = p->prm.P - 1;
  const int pitch = p->out_pitch;
  double* ghost = p->grid_out + (size_t)p->yo * nx * pz * pitch;
  if (halo_in)
    HS_CUDA(cudaMemcpy2DAsync(ghost, pz * pitch * 8, halo_in, nz * pitch * 8, nz * pitch * 8, P1 * nx,
                              cudaMemcpyDeviceToDevice, st));
  else
    HS_CUDA(cudaMemsetAsync(ghost, 0, sizeof(double) * (size_t)P1 * nx * pz * pitch, st));
  HS_TRY(stage_gather(p));
  HS_CUDA(cudaEventRecord(p->ev[7], st));
  HS_TRY(stage_outputs(p, u, u_real, u_fourier, mem));
  HS_CUDA(cudaEventRecord(p->ev[8], st));
  HS_CUDA(cudaStreamSynchronize(st));
  HS_TRY(ctx_check_flags(ctx, "hs_slab_finish"));
  if (times) fill_times(p, times);
  return HS_OK;
}

// gridding.cu -- Gaussian spreading and gathering on the extended grid
// (reference: _gridding.py:21-89, ewald_fourier.py:319-346,626-630).
//
// Spreading is owner-computes and atomic-free: one CTA owns a 16x16x8 tile of
// grid nodes, each thread one (x,y) column of 8 z-nodes for every channel in
// registers.  The CTA streams the sources whose P^3 support can reach the
// tile (sources are bin-sorted by the tile of their window-centre cell, so
// the candidates are 3x3 (x,y) runs of 5 z-bins), stages per-source window
// slices restricted to the tile in shared memory, and every warp (a 4x8
// (x,y) patch) skips sources whose support misses its patch (warp-uniform
// branch).  Each grid value is written exactly once, deterministically,
// without FP64 shared-memory atomics (a CAS loop on sm_100a).
//
// Gathering: one warp per target, lanes over the P z-nodes of one (x,y)
// support column (coalesced 8*P-byte reads), loop over the P*P columns,
// shuffle reduction over lanes.
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace hs {

__global__ void k_grid_keys(const double* __restrict__ pos, int n_src, int n, int mode, GridGeom g, int nbx,
                            int nby, int nbz, int* __restrict__ keys, unsigned* __restrict__ flags,
                            bool gather_v5_keys) {
  const bool fine = (mode & 8) != 0;  // gather targets: (8x8 column, z cell) order
  mode &= 7;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int s = (mode == 1 && i >= n_src) ? i - n_src : i;
    const bool mir = (mode == 2) || (mode == 1 && i >= n_src);
    const double pc[3] = {pos[3 * s], pos[3 * s + 1], mir ? -pos[3 * s + 2] : pos[3 * s + 2]};
    int b[3], cc[3];
    bool drop = false;  // y-slab plan: window starts in another rank's slab
    const int tsz[3] = {SP_TX, SP_TY, SP_TZ};
    const int nb[3] = {nbx, nby, nbz};
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int64_t lo = g_lo(g, k, pc[k]);
      bad |= (lo < 0) || (lo + g.P > g.dims[k]);
      if (k == 1 && g.sel && !fine) drop = lo < g.sel_lo || lo >= g.sel_hi;
      int64_t c = lo + g.P / 2 - 1;  // window-centre cell i0
      c = c < 0 ? 0 : (c >= g.dims[k] ? g.dims[k] - 1 : c);
      int bb = (int)(c / tsz[k]);
      b[k] = bb >= nb[k] ? nb[k] - 1 : bb;
      cc[k] = (int)c;
    }
    if (drop) {
      keys[i] = nbx * nby * nbz;  // one extra bin past the spread bins: never read
      continue;
    }
    if (bad) atomicOr(flags, FLAG_OUT_OF_GRID);
    if (fine && gather_v5_keys) {
      // gather v5: warps of 32 consecutive targets share one 8x8 (x,y) column and a few z cells
      const int n8y = (g.dims[1] + 7) / 8;
      keys[i] = ((cc[0] >> 3) * n8y + (cc[1] >> 3)) * g.dims[2] + cc[2];
    } else if (fine) {
      // gather v7: (4x4 (x,y) column, z node): 8 consecutive targets span a 4x4 footprint
      // and ~5 z nodes (union ~(P+3)^2 columns x (P+5) nodes)
      const int n4y = (g.dims[1] + 3) / 4;
      keys[i] = ((cc[0] >> 2) * n4y + (cc[1] >> 2)) * g.dims[2] + cc[2];
    } else {
      keys[i] = (b[0] * nby + b[1]) * nbz + b[2];
    }
  }
}

hs_status launch_grid_keys(hs_ctx* ctx, const double* pos, int n_src, int n, int mode, const GridGeom& g,
                           int* keys) {
  if (n == 0) return HS_OK;
  const int gs = (int)std::min<int64_t>(ceil_div(n, 256), ctx->sm_count * 8);
  k_grid_keys<<<gs, 256, 0, ctx->stream>>>(pos, n_src, n, mode, g, sp_nbins(g, 0), sp_nbins(g, 1), sp_nbins(g, 2),
                                           keys, ctx->d_flags, gather_v5());
  HS_LAUNCHED(ctx);
  return HS_OK;
}

// ---------------------------------------------------------------------------
// Spreading.  Per source, the window along each axis is
//   w[a] = exp(-alpha (d0 - a h)^2) = E1 * E2^a * E3[a],
//   E1 = exp(-alpha d0^2), E2 = exp(2 alpha d0 h), E3[a] = exp(-alpha h^2 a^2)
// (d0 = distance to the first support node, _gridding.py:24-29), so a tile's
// window slice costs two multiplies per node instead of one exp; E1/E2 are
// computed once per source (k_spread_windows).
constexpr int SP_CHUNK = 96;   // sources staged per round
constexpr int SP_MAXCH = 4;    // channels per launch (register budget)
constexpr int SP_MAXP = 64;

struct WinConst {
  double e3[SP_MAXP];
};

__global__ void k_spread_windows(const double4* __restrict__ pts, int n, GridGeom g, int4* __restrict__ lo,
                                 double4* __restrict__ wxy, double2* __restrict__ wz) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double4 p = pts[i];
    const double pc[3] = {p.x, p.y, p.z};
    int l[3];
    double e1[3], e2[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int64_t lk = g_lo(g, k, pc[k]);
      l[k] = (int)lk;
      const double d0 = g_d(g, k, pc[k], lk);
      e1[k] = exp(-g.alpha * d0 * d0);
      e2[k] = exp(2.0 * g.alpha * d0 * g.h);
    }
    lo[i] = make_int4(l[0], l[1], l[2], 0);
    wxy[i] = make_double4(e1[0] * g.pref, e2[0], e1[1], e2[1]);  // pref folded into the x factor
    wz[i] = make_double2(e1[2], e2[2]);
  }
}

// window slice of length L starting at grid node `node0`, support start lo
template <int L>
__device__ __forceinline__ void window_slice(int node0, int lo, int P, double e1, double e2, const double* e3,
                                             double* out) {
#pragma unroll
  for (int i = 0; i < L; ++i) out[i] = 0.0;
  const int i0 = max(0, lo - node0);   // first slice index inside the support
  const int a0 = node0 + i0 - lo;      // its support offset (>= 0)
  if (i0 >= L || a0 >= P) return;
  // e2^a0 by binary exponentiation, then 4 independent chains with step e2^4
  double pw = 1.0, b = e2;
  for (int m = a0; m; m >>= 1) {
    if (m & 1) pw *= b;
    b *= b;
  }
  const double e22 = e2 * e2, e24 = e22 * e22;
  double p[4] = {e1 * pw, e1 * pw * e2, e1 * pw * e22, e1 * pw * e22 * e2};
#pragma unroll
  for (int j = 0; j < (L + 3) / 4; ++j) {
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int i = i0 + 4 * j + k, aa = a0 + 4 * j + k;
      if (i < L && aa < P) out[i] = p[k] * e3[aa];
      p[k] *= e24;
    }
  }
}

template <int NCH>
__global__ void __launch_bounds__(256, 2) k_spread(const int4* __restrict__ lo4, const double4* __restrict__ wxy,
                                                const double2* __restrict__ wzp, const double* __restrict__ w,
                                                int ldw, const int* __restrict__ bin_start, GridGeom g,
                                                WinConst wc, int nbx, int nby, int nbz, double* __restrict__ grids) {
  // rows padded by one double so the per-source staging writes do not share banks
  __shared__ double s_wx[SP_CHUNK][SP_TX + 1];
  __shared__ double s_wy[SP_CHUNK][SP_TY + 1];
  __shared__ double s_wz[SP_CHUNK][SP_TZ + 1];
  __shared__ double s_q[SP_CHUNK][NCH | 1];
  __shared__ unsigned s_mask[SP_CHUNK];
  __shared__ double s_e3[SP_MAXP];
  __shared__ int run_beg[9], run_pre[10];
  __shared__ int s_nrun;

  const int tz = blockIdx.x % nbz;
  const int ty = (blockIdx.x / nbz) % nby;
  const int tx = blockIdx.x / (nbz * nby);
  const int x0 = tx * SP_TX, y0 = ty * SP_TY, z0 = tz * SP_TZ;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  // warp patch: 4 (x) x 8 (y); 8 warps tile 16 x 16
  const int xo = (warp & 3) * 4 + (lane & 3), yo = (warp >> 2) * 8 + (lane >> 2);
  const int P = g.P;

  for (int i = threadIdx.x; i < P; i += blockDim.x) s_e3[i] = wc.e3[i];
  if (threadIdx.x == 0) {
    int nr = 0, tot = 0;
    const int zlo = max(tz - 2, 0), zhi = min(tz + 2, nbz - 1);
    for (int bx = max(tx - 1, 0); bx <= min(tx + 1, nbx - 1); ++bx)
      for (int by = max(ty - 1, 0); by <= min(ty + 1, nby - 1); ++by) {
        const int f = (bx * nby + by) * nbz;
        const int b = bin_start[f + zlo], e = bin_start[f + zhi + 1];
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
  const int nrun = s_nrun, ncand = run_pre[nrun];

  double acc[NCH][SP_TZ];
#pragma unroll
  for (int c = 0; c < NCH; ++c)
#pragma unroll
    for (int j = 0; j < SP_TZ; ++j) acc[c][j] = 0.0;

  // staging roles are warp-uniform (no intra-warp divergence): warps 0-1 x windows,
  // 2-3 y windows, 4-5 z windows + warp masks, 6-7 channel weights; 2 sources per thread.
  // The global records of chunk c+1 are loaded into registers while chunk c is computed.
  const int role = warp >> 1;
  int4 pl[2];
  double4 pe[2];
  double pq[2][NCH];
  auto prefetch = [&](int cbase) {
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int sidx = (warp & 1) * 32 + lane + 64 * k;
      const int v = cbase + sidx;
      if (sidx < SP_CHUNK && v < ncand) {
        int r = 0;
        while (r + 1 < nrun && run_pre[r + 1] <= v) ++r;
        const int row = run_beg[r] + (v - run_pre[r]);
        if (role <= 2) pl[k] = lo4[row];
        if (role <= 1) pe[k] = wxy[row];
        if (role == 2) {
          const double2 e = wzp[row];
          pe[k] = make_double4(e.x, e.y, 0.0, 0.0);
        }
        if (role == 3) {
#pragma unroll
          for (int c = 0; c < NCH; ++c) pq[k][c] = w[(size_t)row * ldw + c];
        }
      }
    }
  };
  if (ncand > 0) prefetch(0);
  for (int c0 = 0; c0 < ncand; c0 += SP_CHUNK) {
    const int nc = min(SP_CHUNK, ncand - c0);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2; ++k) {
      const int s = (warp & 1) * 32 + lane + 64 * k;
      if (s < nc) {
        const int4 l = pl[k];
        if (role == 0) {
          window_slice<SP_TX>(x0, l.x, P, pe[k].x, pe[k].y, s_e3, s_wx[s]);
        } else if (role == 1) {
          window_slice<SP_TY>(y0, l.y, P, pe[k].z, pe[k].w, s_e3, s_wy[s]);
        } else if (role == 2) {
          window_slice<SP_TZ>(z0, l.z, P, pe[k].x, pe[k].y, s_e3, s_wz[s]);
          // which warps' 4x8 (x,y) patches does the support reach? (z overlap is CTA-wide)
          unsigned m = 0;
          if (l.z < z0 + SP_TZ && l.z + P > z0) {
#pragma unroll
            for (int wq = 0; wq < 8; ++wq) {
              const int px = x0 + (wq & 3) * 4, py = y0 + (wq >> 2) * 8;
              if (l.x < px + 4 && l.x + P > px && l.y < py + 8 && l.y + P > py) m |= 1u << wq;
            }
          }
          s_mask[s] = m;
        } else {
#pragma unroll
          for (int c = 0; c < NCH; ++c) s_q[s][c] = pq[k][c];
        }
      }
    }
    __syncthreads();
    if (c0 + SP_CHUNK < ncand) prefetch(c0 + SP_CHUNK);
    for (int base = 0; base < nc; base += 32) {
      unsigned m = __ballot_sync(0xffffffffu, base + lane < nc && ((s_mask[base + lane] >> warp) & 1u));
      while (m) {
        const int s = base + __ffs(m) - 1;
        m &= m - 1;
        const double cxy = s_wx[s][xo] * s_wy[s][yo];
        double wz[SP_TZ];
#pragma unroll
        for (int j = 0; j < SP_TZ; ++j) wz[j] = s_wz[s][j];
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const double q = s_q[s][c] * cxy;
#pragma unroll
          for (int j = 0; j < SP_TZ; ++j) acc[c][j] = fma(q, wz[j], acc[c][j]);
        }
      }
    }
  }
  const int x = x0 + xo, y = y0 + yo;
  if (x < g.dims[0] && y < g.dims[1]) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      double* dst = grids + c * g.ch_stride + x * g.stride[0] + y * g.stride[1];
#pragma unroll
      for (int j = 0; j < SP_TZ; ++j) {
        const int z = z0 + j;
        if (z < g.dims[2]) dst[z * g.stride[2]] = acc[c][j];
      }
    }
  }
}

// Tensor-core variant: the per-warp accumulation is the small GEMM
//   C[(x,y) position p][z node n] += sum_s A[p][s] B[s][n],
//   A[p][s] = q_s wx_s(x_p) wy_s(y_p),  B[s][n] = wz_s(z_n),
// evaluated with FP64 DMMA (mma.sync m8n8k4; there is no FP64 tcgen05 kind) over groups
// of 4 hitting sources: the warp's 32 (x,y) positions are 4 row blocks of 8, the tile's
// 8 z nodes are the 8 columns.  One DMMA replaces 8 warp-wide DFMAs plus their operand
// traffic; the staging and hit masks are those of k_spread.
__device__ __forceinline__ void dmma_884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// Spread v3 (default): the DMMA accumulation of k_spread_mma, with the per-tile staging
// replaced by asynchronous copies.  k_spread_wtab evaluates every source's full window
// once (exp(-alpha d^2) per node, _gridding.py:21-30; the normalisation folded into the
// x factor) into zero-padded rows; a tile then copies (cp.async, 16-byte chunks) the
// slices it needs into a double-buffered shared-memory chunk while the warps accumulate
// the previous chunk -- one barrier per chunk, no window arithmetic in the tile loop.
struct WTab {                              // row layout of one source (doubles)
  int wx, wy, wz, stride;                  // padded row lengths and their sum
  __host__ __device__ static WTab make(int P) {
    WTab t;
    t.wx = (2 * SP_TX + P + 1) & ~1;
    t.wy = (2 * SP_TY + P + 1) & ~1;
    t.wz = (2 * SP_TZ + P + 1) & ~1;
    t.stride = t.wx + t.wy + t.wz;
    return t;
  }
};

__global__ void k_spread_wtab(const double4* __restrict__ pts, int n, GridGeom g, WTab wt, int4* __restrict__ lo,
                              double* __restrict__ tab) {
  // one warp per (source, axis) row; lanes write consecutive entries (coalesced)
  const int P = g.P;
  const int lane = threadIdx.x & 31;
  const int64_t nrow = (int64_t)n * 3;
  for (int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; r < nrow;
       r += ((int64_t)gridDim.x * blockDim.x) >> 5) {
    const int s = (int)(r / 3), k = (int)(r - 3 * (int64_t)s);
    const double4 p = pts[s];
    const double pc = k == 0 ? p.x : (k == 1 ? p.y : p.z);
    const int64_t l = g_lo(g, k, pc);
    const int pad = k == 0 ? SP_TX : (k == 1 ? SP_TY : SP_TZ);
    const int len = k == 0 ? wt.wx : (k == 1 ? wt.wy : wt.wz);
    double* row = tab + (int64_t)s * wt.stride + (k == 0 ? 0 : (k == 1 ? wt.wx : wt.wx + wt.wy));
    const double scale = k == 0 ? g.pref : 1.0;
    for (int j = lane; j < len; j += 32) {
      const int a = j - pad;
      double v = 0.0;
      if (a >= 0 && a < P) {
        const double d = g_d(g, k, pc, l + a);
        v = scale * exp(-g.alpha * d * d);
      }
      row[j] = v;
    }
    if (k == 0 && lane == 0)
      lo[s] = make_int4((int)l, (int)g_lo(g, 1, p.y), (int)g_lo(g, 2, p.z), 0);
  }
}

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "HS_WAIT_%=:\n"
      " mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra HS_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// bulk global -> shared copy (16-byte aligned, size a multiple of 16) completing on `bar`
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void cpa16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cpa8(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gmem));
}

// Warp-specialised pipeline: warp 8 produces chunks of SW_CH candidate sources into a
// ring of SW_K shared-memory buffers (hit masks, slice parities and weights by plain
// stores; the x / y / z window slices by bulk asynchronous copies from the window table,
// completing on the buffer's `full` mbarrier), warps 0-7 consume them (DMMA) and release
// the buffer on its `empty` mbarrier.  Consumers never wait for staging and may run up
// to SW_K chunks ahead of each other, so per-chunk load imbalance averages out.
#ifndef SW_CH_DEF
#define SW_CH_DEF 32
#define SW_K_DEF 8
#endif
constexpr int SW_CH = SW_CH_DEF, SW_K = SW_K_DEF, SW_H = SW_CH_DEF / 32, SW_RX = SP_TX + 2, SW_RY = SP_TY + 2, SW_RZ = SP_TZ + 2;
// producer warps (8, 9, ...): producer p stages the chunks c = p mod SW_NP, so the SW_K ring
// slots of one producer are fixed (SW_K % SW_NP == 0) and one warp's staging rate no longer
// bounds the eight consumers
#ifndef SW_NP_DEF
#define SW_NP_DEF 2
#endif
constexpr int SW_NP = SW_NP_DEF, SW_THREADS = (8 + SW_NP) * 32;
static_assert(SW_K % SW_NP == 0, "ring slots must divide among the producers");
template <int NCH>
struct SwBuf {
  static constexpr int RQ = NCH | 1;
  static constexpr int DOUBLES = SW_CH * (SW_RX + SW_RY + SW_RZ + RQ + 1);
};

// FLY (HS_SPREAD_FLY=1, comparison): the producers compute each source's window slices for the tile from its
// position (two exps per axis, then the Gaussian ratio recurrence w_{a+1} = w_a r_a,
// r_{a+1} = r_a exp(-2 alpha h^2); ~4e-15 relative after <= 18 steps) instead of copying them
// from the per-source window table: every source's slices were re-read by the ~25 tiles its
// support touches (11 GB of DRAM reads per channel group at HL), now only its 32-byte record
// and weights are -- but the producers' dependent recurrence chains then bound the consumers
// (24.4 vs 18.1 ms at HL), so !FLY (window tables + cp.async) is the default.
// NCW consumer warps: 8 (warp patch 4x8 (x,y) x 8 z, 2 CTAs/SM) or 16 (patch 4x4 x 8, 1 CTA/SM,
// a 16-deep ring): the smaller patch cuts the y padding of the DMMA work (window rows outside a
// warp's patch) from (24+7)/24 to (24+3)/24, and with all channels in one launch the producers
// stage every source once instead of once per channel group.
template <int NCH, bool FLY, int NCW = 8>
__global__ void __launch_bounds__((NCW + SW_NP) * 32, NCW == 8 ? 2 : 1) k_spread_mma4(const int4* __restrict__ lo4, const double* __restrict__ tab,
                                                       WTab wt, const double4* __restrict__ pts,
                                                       const double* __restrict__ w, int ldw,
                                                       const int* __restrict__ bin_start, GridGeom g, int nbx,
                                                       int nby, int nbz, double* __restrict__ grids) {
  constexpr int RX = SW_RX, RY = SW_RY, RZ = SW_RZ, RQ = SwBuf<NCH>::RQ, PER = SwBuf<NCH>::DOUBLES;
  extern __shared__ __align__(16) double sm_dyn[];
  constexpr int K = NCW == 16 ? 16 * 32 / SW_CH : SW_K;  // ring depth (16 slots of 32 sources)
  constexpr int PY = 64 / NCW, RB = PY / 2;  // warp patch rows, row blocks of 8 positions
  constexpr int PB = NCW;                    // mask bit of the window-slice parities
  __shared__ __align__(8) uint64_t full_bar[K], empty_bar[K];
  __shared__ int run_beg[9], run_pre[10];
  __shared__ int s_nrun;
  auto bx_ = [&](int b) { return reinterpret_cast<double(*)[RX]>(sm_dyn + b * PER); };
  auto by_ = [&](int b) { return reinterpret_cast<double(*)[RY]>(sm_dyn + b * PER + SW_CH * RX); };
  auto bz_ = [&](int b) { return reinterpret_cast<double(*)[RZ]>(sm_dyn + b * PER + SW_CH * (RX + RY)); };
  auto bq_ = [&](int b) { return reinterpret_cast<double(*)[RQ]>(sm_dyn + b * PER + SW_CH * (RX + RY + RZ)); };
  auto bm_ = [&](int b) { return reinterpret_cast<unsigned*>(sm_dyn + b * PER + SW_CH * (RX + RY + RZ + RQ)); };

  const int tz = blockIdx.x % nbz;
  const int ty = (blockIdx.x / nbz) % nby;
  const int tx = blockIdx.x / (nbz * nby);
  const int x0 = tx * SP_TX, y0 = ty * SP_TY, z0 = tz * SP_TZ;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int P = g.P;

  if (threadIdx.x == 0) {
    int nr = 0, tot = 0;
    const int zlo = max(tz - 2, 0), zhi = min(tz + 2, nbz - 1);
    for (int bx = max(tx - 1, 0); bx <= min(tx + 1, nbx - 1); ++bx)
      for (int by = max(ty - 1, 0); by <= min(ty + 1, nby - 1); ++by) {
        const int f = (bx * nby + by) * nbz;
        const int b = bin_start[f + zlo], e = bin_start[f + zhi + 1];
        if (e > b) {
          run_beg[nr] = b;
          run_pre[nr] = tot;
          tot += e - b;
          ++nr;
        }
      }
    run_pre[nr] = tot;
    s_nrun = nr;
#pragma unroll
    for (int k = 0; k < K; ++k) {
      mbar_init(&full_bar[k], 64);          // producer lanes: stores released + their cp.async completed
      mbar_init(&empty_bar[k], NCW * 32);   // every consumer thread
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int nrun = s_nrun, ncand = run_pre[nrun];
  const int nchunk = (ncand + SW_CH - 1) / SW_CH;

  if (warp >= NCW) {
    // ---------------- producers ----------------
    const int pid = warp - NCW;
    // rows / windows starts / weights of chunk c+1 and c+2 are in flight (registers) while
    // chunk c is staged, so the producer runs at one chunk per staging pass, not per load latency
    struct Pre {
      int4 lo[SW_H];
      int row[SW_H];
      double q[SW_H][NCH];
      double p[SW_H][3];
    };
    const double rq2 = exp(-2.0 * g.alpha * g.h * g.h);  // ratio of successive window ratios
    // dst[j] = window value of node a = a0 + j (relative to the window start lo), 0 outside [0, P)
    auto fill = [&](double* dst, int n, double pos, int k, int lo_local, int a0, double scale) {
      const int as = max(a0, 0);
      const double d = g_d(g, k, pos, lo_local + as);
      double wv = scale * exp(-g.alpha * d * d);
      double r = exp(g.alpha * g.h * (2.0 * d - g.h));
      for (int j = 0; j < n; ++j) {
        const int a = a0 + j;
        double v = 0.0;
        if (a >= as && a < P) {
          v = wv;
          wv *= r;
          r *= rq2;
        }
        dst[j] = v;
      }
    };
    // stride permutation of the candidate list (as in the pair kernel): candidates are in bin
    // order, so consecutive chunks would come from ONE neighbour bin and hit only the warp
    // patches on that side of the tile, leaving the other consumers idle while the ring fills;
    // permuted, every chunk samples all bins and the per-chunk work is even across warps
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
    auto fetch = [&](int c, Pre& f) {
#pragma unroll
      for (int h = 0; h < SW_H; ++h) {
        const int v0 = c * SW_CH + lane + 32 * h;
        f.row[h] = -1;
        if (c < nchunk && v0 < ncand) {
          const int v = (int)(((long long)v0 * pstride) % ncand);
          int r = 0, rhi = nrun - 1;  // last run with run_pre[r] <= v
          while (r < rhi) {
            const int mid = (r + rhi + 1) >> 1;
            if (run_pre[mid] <= v) r = mid;
            else rhi = mid - 1;
          }
          const int row = run_beg[r] + (v - run_pre[r]);
          f.row[h] = row;
          if (FLY) {
            const double4 pp = pts[row];
            f.p[h][0] = pp.x;
            f.p[h][1] = pp.y;
            f.p[h][2] = pp.z;
            f.lo[h] = make_int4((int)g_lo(g, 0, pp.x), (int)g_lo(g, 1, pp.y), (int)g_lo(g, 2, pp.z), 0);
          } else {
            f.lo[h] = lo4[row];
          }
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) f.q[h][ch] = w[(int64_t)row * ldw + ch];
        }
      }
    };
    Pre f1, f2;
    fetch(pid, f1);
    fetch(pid + SW_NP, f2);
    for (int c = pid; c < nchunk; c += SW_NP) {
      const int b = c % K;
      const Pre cur = f1;
      f1 = f2;
      fetch(c + 2 * SW_NP, f2);
      if (c >= K) mbar_wait(&empty_bar[b], ((c / K) - 1) & 1);
      unsigned m[SW_H];
      int ex[SW_H], ey[SW_H], ez[SW_H];
#pragma unroll
      for (int h = 0; h < SW_H; ++h) {
        const int sl = lane + 32 * h;
        ex[h] = ey[h] = ez[h] = 0;
        m[h] = 0u;
        if (cur.row[h] >= 0) {
          const int4 l = cur.lo[h];
          if (l.z < z0 + SP_TZ && l.z + P > z0) {
#pragma unroll
            for (int wq = 0; wq < NCW; ++wq) {
              const int px = x0 + (wq & 3) * 4, py = y0 + (wq >> 2) * PY;
              if (l.x < px + 4 && l.x + P > px && l.y < py + PY && l.y + P > py) m[h] |= 1u << wq;
            }
          }
          ex[h] = SP_TX + (x0 - l.x);
          ey[h] = SP_TY + (y0 - l.y);
          ez[h] = SP_TZ + (z0 - l.z);
          if (m[h]) {
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) bq_(b)[sl][ch] = cur.q[h][ch];
          }
        }
        bm_(b)[sl] = m[h] | (m[h] ? ((unsigned)(ex[h] & 1) << PB) | ((unsigned)(ey[h] & 1) << (PB + 1)) |
                                        ((unsigned)(ez[h] & 1) << (PB + 2))
                                  : 0u);
      }
      mbar_arrive(&full_bar[b]);  // masks / weights (plain stores) released
      if (FLY) {
#pragma unroll
        for (int h = 0; h < SW_H; ++h) {
          if (m[h]) {
            const int sl = lane + 32 * h;
            const int4 l = cur.lo[h];
            fill(bx_(b)[sl], RX, cur.p[h][0], 0, l.x, (ex[h] & ~1) - SP_TX, g.pref);
            fill(by_(b)[sl], RY, cur.p[h][1], 1, l.y, (ey[h] & ~1) - SP_TY, 1.0);
            fill(bz_(b)[sl], RZ, cur.p[h][2], 2, l.z, (ez[h] & ~1) - SP_TZ, 1.0);
          }
        }
        mbar_arrive(&full_bar[b]);  // window slices (plain stores) released
        continue;
      }
      // window slices: 16-byte cp.async chunks, completion tracked by the same barrier
#pragma unroll
      for (int h = 0; h < SW_H; ++h) {
        if (m[h]) {
          const int sl = lane + 32 * h;
          const double* src = tab + (int64_t)cur.row[h] * wt.stride;
          const double* sx = src + (ex[h] & ~1);
          const double* sy = src + wt.wx + (ey[h] & ~1);
          const double* sz = src + wt.wx + wt.wy + (ez[h] & ~1);
#pragma unroll
          for (int j = 0; j < RX / 2; ++j) cpa16(&bx_(b)[sl][2 * j], sx + 2 * j);
#pragma unroll
          for (int j = 0; j < RY / 2; ++j) cpa16(&by_(b)[sl][2 * j], sy + 2 * j);
#pragma unroll
          for (int j = 0; j < RZ / 2; ++j) cpa16(&bz_(b)[sl][2 * j], sz + 2 * j);
        }
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(&full_bar[b])) : "memory");
    }
    return;
  }

  // ---------------- consumers (warps 0 .. NCW-1) ----------------
  const int wx0 = (warp & 3) * 4, wy0 = (warp >> 2) * PY;  // warp patch origin inside the tile
  const int kq = lane & 3;   // k index (source slot) of this lane's A and B fragments
  const int rq = lane >> 2;  // A row / B column / C row of this lane
  double acc[RB][NCH][2];
#pragma unroll
  for (int rb = 0; rb < RB; ++rb)
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[rb][c][0] = acc[rb][c][1] = 0.0;
  for (int c = 0; c < nchunk; ++c) {
    const int b = c % K;
    const int nc = min(SW_CH, ncand - c * SW_CH);
    mbar_wait(&full_bar[b], (c / K) & 1);
    double(*s_wx)[RX] = bx_(b);
    double(*s_wy)[RY] = by_(b);
    double(*s_wz)[RZ] = bz_(b);
    double(*s_q)[RQ] = bq_(b);
    const unsigned* s_mask = bm_(b);
    for (int base = 0; base < nc; base += 32) {
      const unsigned mk = base + lane < nc ? s_mask[base + lane] : 0u;
      unsigned m = __ballot_sync(0xffffffffu, (mk >> warp) & 1u);
      while (m) {
        int sk = -1;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int sb = m ? base + __ffs(m) - 1 : -1;
          if (m) m &= m - 1;
          if (k == kq) sk = sb;
        }
        double bz = 0.0, q[NCH], cxy[RB];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) q[ch] = 0.0;
#pragma unroll
        for (int rb = 0; rb < RB; ++rb) cxy[rb] = 0.0;
        if (sk >= 0) {
          const unsigned par = s_mask[sk];
          const int pxo = (par >> PB) & 1, pyo = (par >> (PB + 1)) & 1, pzo = (par >> (PB + 2)) & 1;
          bz = s_wz[sk][pzo + rq];  // B[k][n] = wz_{s_k}(z_n), n = rq
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) q[ch] = s_q[sk][ch];
#pragma unroll
          for (int rb = 0; rb < RB; ++rb) {
            const int p = rb * 8 + rq;  // position of A row rq in row block rb
            cxy[rb] = s_wx[sk][pxo + wx0 + (p & 3)] * s_wy[sk][pyo + wy0 + (p >> 2)];
          }
        }
        // the weight goes into the B operand (wz q_c, one product per channel) so A = wx wy is
        // shared by the channels
        double bq[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) bq[ch] = bz * q[ch];
#pragma unroll
        for (int rb = 0; rb < RB; ++rb)
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) dmma_884(acc[rb][ch][0], acc[rb][ch][1], cxy[rb], bq[ch]);
      }
    }
    mbar_arrive(&empty_bar[b]);
  }
  // C fragment: row rq of row block rb = position p, columns z = 2 kq, 2 kq + 1
#pragma unroll
  for (int rb = 0; rb < RB; ++rb) {
    const int p = rb * 8 + rq;
    const int x = x0 + wx0 + (p & 3), y = y0 + wy0 + (p >> 2);
    if (x < g.dims[0] && y < g.dims[1]) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        double* dst = grids + c * g.ch_stride + x * g.stride[0] + y * g.stride[1];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int z = z0 + 2 * kq + i;
          if (z < g.dims[2]) dst[z * g.stride[2]] = acc[rb][c][i];
        }
      }
    }
  }
}

template <int NCH, int CH>
__global__ void __launch_bounds__(256, 2) k_spread_mma(const int4* __restrict__ lo4, const double4* __restrict__ wxy,
                                                      const double2* __restrict__ wzp, const double* __restrict__ w,
                                                      int ldw, const int* __restrict__ bin_start, GridGeom g,
                                                      WinConst wc, int nbx, int nby, int nbz,
                                                      double* __restrict__ grids) {
  extern __shared__ double sm_dyn[];  // CH-source staging (dynamic: CH * ~50 doubles)
  double(*s_wx)[SP_TX + 1] = reinterpret_cast<double(*)[SP_TX + 1]>(sm_dyn);
  double(*s_wy)[SP_TY + 1] = reinterpret_cast<double(*)[SP_TY + 1]>(sm_dyn + CH * (SP_TX + 1));
  double(*s_wz)[SP_TZ + 1] = reinterpret_cast<double(*)[SP_TZ + 1]>(sm_dyn + CH * (SP_TX + SP_TY + 2));
  double(*s_q)[NCH | 1] = reinterpret_cast<double(*)[NCH | 1]>(sm_dyn + CH * (SP_TX + SP_TY + SP_TZ + 3));
  unsigned* s_mask = reinterpret_cast<unsigned*>(sm_dyn + CH * (SP_TX + SP_TY + SP_TZ + 3 + (NCH | 1)));
  __shared__ double s_e3[SP_MAXP];
  __shared__ int run_beg[9], run_pre[10];
  __shared__ int s_nrun;

  const int tz = blockIdx.x % nbz;
  const int ty = (blockIdx.x / nbz) % nby;
  const int tx = blockIdx.x / (nbz * nby);
  const int x0 = tx * SP_TX, y0 = ty * SP_TY, z0 = tz * SP_TZ;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wx0 = (warp & 3) * 4, wy0 = (warp >> 2) * 8;  // warp patch origin inside the tile
  const int P = g.P;
  const int kq = lane & 3;   // k index (source slot) of this lane's A and B fragments
  const int rq = lane >> 2;  // A row / B column / C row of this lane

  for (int i = threadIdx.x; i < P; i += blockDim.x) s_e3[i] = wc.e3[i];
  if (threadIdx.x == 0) {
    int nr = 0, tot = 0;
    const int zlo = max(tz - 2, 0), zhi = min(tz + 2, nbz - 1);
    for (int bx = max(tx - 1, 0); bx <= min(tx + 1, nbx - 1); ++bx)
      for (int by = max(ty - 1, 0); by <= min(ty + 1, nby - 1); ++by) {
        const int f = (bx * nby + by) * nbz;
        const int b = bin_start[f + zlo], e = bin_start[f + zhi + 1];
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
  const int nrun = s_nrun, ncand = run_pre[nrun];

  double acc[4][NCH][2];
#pragma unroll
  for (int rb = 0; rb < 4; ++rb)
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[rb][c][0] = acc[rb][c][1] = 0.0;

  const int role = warp >> 1;
  constexpr int KPT = CH / 64;  // sources per staging thread
  int4 pl[KPT];
  double4 pe[KPT];
  double pq[KPT][NCH];
  auto prefetch = [&](int cbase) {
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int sidx = (warp & 1) * 32 + lane + 64 * k;
      const int v = cbase + sidx;
      if (v < ncand) {
        int r = 0;
        while (r + 1 < nrun && run_pre[r + 1] <= v) ++r;
        const int row = run_beg[r] + (v - run_pre[r]);
        if (role <= 2) pl[k] = lo4[row];
        if (role <= 1) pe[k] = wxy[row];
        if (role == 2) {
          const double2 e = wzp[row];
          pe[k] = make_double4(e.x, e.y, 0.0, 0.0);
        }
        if (role == 3) {
#pragma unroll
          for (int c = 0; c < NCH; ++c) pq[k][c] = w[(size_t)row * ldw + c];
        }
      }
    }
  };
  if (ncand > 0) prefetch(0);
  for (int c0 = 0; c0 < ncand; c0 += CH) {
    const int nc = min(CH, ncand - c0);
    __syncthreads();
#pragma unroll
    for (int k = 0; k < KPT; ++k) {
      const int s = (warp & 1) * 32 + lane + 64 * k;
      if (s < nc) {
        const int4 l = pl[k];
        if (role == 0) {
          window_slice<SP_TX>(x0, l.x, P, pe[k].x, pe[k].y, s_e3, s_wx[s]);
        } else if (role == 1) {
          window_slice<SP_TY>(y0, l.y, P, pe[k].z, pe[k].w, s_e3, s_wy[s]);
        } else if (role == 2) {
          window_slice<SP_TZ>(z0, l.z, P, pe[k].x, pe[k].y, s_e3, s_wz[s]);
          unsigned m = 0;
          if (l.z < z0 + SP_TZ && l.z + P > z0) {
#pragma unroll
            for (int wq = 0; wq < 8; ++wq) {
              const int px = x0 + (wq & 3) * 4, py = y0 + (wq >> 2) * 8;
              if (l.x < px + 4 && l.x + P > px && l.y < py + 8 && l.y + P > py) m |= 1u << wq;
            }
          }
          s_mask[s] = m;
        } else {
#pragma unroll
          for (int c = 0; c < NCH; ++c) s_q[s][c] = pq[k][c];
        }
      }
    }
    __syncthreads();
    if (c0 + CH < ncand) prefetch(c0 + CH);
    for (int base = 0; base < nc; base += 32) {
      unsigned m = __ballot_sync(0xffffffffu, base + lane < nc && ((s_mask[base + lane] >> warp) & 1u));
      while (m) {
        // next group of up to 4 hitting sources; this lane's slot kq
        int sk = -1;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int sb = m ? base + __ffs(m) - 1 : -1;
          if (m) m &= m - 1;
          if (k == kq) sk = sb;
        }
        const double bz = sk >= 0 ? s_wz[sk][rq] : 0.0;  // B[k][n] = wz_{s_k}(z_n), n = rq
        double q[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) q[c] = sk >= 0 ? s_q[sk][c] : 0.0;
#pragma unroll
        for (int rb = 0; rb < 4; ++rb) {
          const int p = rb * 8 + rq;  // position of A row rq in row block rb
          const double cxy = sk >= 0 ? s_wx[sk][wx0 + (p & 3)] * s_wy[sk][wy0 + (p >> 2)] : 0.0;
#pragma unroll
          for (int c = 0; c < NCH; ++c) dmma_884(acc[rb][c][0], acc[rb][c][1], cxy * q[c], bz);
        }
      }
    }
  }
  // C fragment: row rq of row block rb = position p, columns z = 2 kq, 2 kq + 1
#pragma unroll
  for (int rb = 0; rb < 4; ++rb) {
    const int p = rb * 8 + rq;
    const int x = x0 + wx0 + (p & 3), y = y0 + wy0 + (p >> 2);
    if (x < g.dims[0] && y < g.dims[1]) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        double* dst = grids + c * g.ch_stride + x * g.stride[0] + y * g.stride[1];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const int z = z0 + 2 * kq + i;
          if (z < g.dims[2]) dst[z * g.stride[2]] = acc[rb][c][i];
        }
      }
    }
  }
}

// Warp-independent variant (no CTA barriers): every warp streams the tile's candidate
// list itself, 32 sources at a time (lane = source), keeps the sources whose support
// reaches its own 4x8 (x,y) patch and the tile's z-range (ballot), builds their window
// slices for ITS 4 x-nodes, 8 y-nodes and 8 z-nodes in warp-private shared memory and
// accumulates them.  The z-slices are recomputed per warp (cheap: a few multiplies per
// node); in exchange no warp ever waits for another.
constexpr int SW_STRIDE = 4 + 8 + 8 + 1;  // wx[4] wy[8] wz[8] + pad (odd stride: conflict-free)

template <int NCH>
__global__ void __launch_bounds__(256, 2) k_spread2(const int4* __restrict__ lo4, const double4* __restrict__ wxy,
                                                   const double2* __restrict__ wzp, const double* __restrict__ w,
                                                   int ldw, const int* __restrict__ bin_start, GridGeom g,
                                                   WinConst wc, int nbx, int nby, int nbz,
                                                   double* __restrict__ grids) {
  extern __shared__ double sw_dyn[];  // [8 warps][32 * SW_STRIDE] windows, then [8][32 * (NCH|1)] weights
  __shared__ double s_e3[SP_MAXP];
  __shared__ int run_beg[9], run_pre[10];
  __shared__ int s_nrun;

  const int tz = blockIdx.x % nbz;
  const int ty = (blockIdx.x / nbz) % nby;
  const int tx = blockIdx.x / (nbz * nby);
  const int x0 = tx * SP_TX, y0 = ty * SP_TY, z0 = tz * SP_TZ;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int px0 = x0 + (warp & 3) * 4, py0 = y0 + (warp >> 2) * 8;  // this warp's patch
  const int xi = lane & 3, yi = lane >> 2;
  const int P = g.P;
  constexpr int QS = NCH | 1;
  double* win = sw_dyn + warp * 32 * SW_STRIDE;
  double* qw = sw_dyn + 8 * 32 * SW_STRIDE + warp * 32 * QS;

  for (int i = threadIdx.x; i < P; i += blockDim.x) s_e3[i] = wc.e3[i];
  if (threadIdx.x == 0) {
    int nr = 0, tot = 0;
    const int zlo = max(tz - 2, 0), zhi = min(tz + 2, nbz - 1);
    for (int bx = max(tx - 1, 0); bx <= min(tx + 1, nbx - 1); ++bx)
      for (int by = max(ty - 1, 0); by <= min(ty + 1, nby - 1); ++by) {
        const int f = (bx * nby + by) * nbz;
        const int b = bin_start[f + zlo], e = bin_start[f + zhi + 1];
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
  const int nrun = s_nrun, ncand = run_pre[nrun];

  double acc[NCH][SP_TZ];
#pragma unroll
  for (int c = 0; c < NCH; ++c)
#pragma unroll
    for (int j = 0; j < SP_TZ; ++j) acc[c][j] = 0.0;

  int r = 0;  // current run (candidates are visited in increasing order)
  for (int c0 = 0; c0 < ncand; c0 += 32) {
    const int v = c0 + lane;
    bool hit = false;
    int4 l = make_int4(0, 0, 0, 0);
    int row = 0;
    if (v < ncand) {
      while (r + 1 < nrun && run_pre[r + 1] <= c0) ++r;
      int rr = r;
      while (rr + 1 < nrun && run_pre[rr + 1] <= v) ++rr;
      row = run_beg[rr] + (v - run_pre[rr]);
      l = lo4[row];
      hit = (l.x < px0 + 4) && (l.x + P > px0) && (l.y < py0 + 8) && (l.y + P > py0) && (l.z < z0 + SP_TZ) &&
            (l.z + P > z0);
    }
    unsigned m = __ballot_sync(0xffffffffu, hit);
    if (!m) continue;
    if (hit) {
      const double4 e = wxy[row];
      const double2 ez = wzp[row];
      double* ws = win + lane * SW_STRIDE;
      window_slice<4>(px0, l.x, P, e.x, e.y, s_e3, ws);
      window_slice<8>(py0, l.y, P, e.z, e.w, s_e3, ws + 4);
      window_slice<SP_TZ>(z0, l.z, P, ez.x, ez.y, s_e3, ws + 12);
#pragma unroll
      for (int c = 0; c < NCH; ++c) qw[lane * QS + c] = w[(size_t)row * ldw + c];
    }
    __syncwarp();
    while (m) {
      const int sl = __ffs(m) - 1;
      m &= m - 1;
      const double* ws = win + sl * SW_STRIDE;
      const double cxy = ws[xi] * ws[4 + yi];
      double wz[SP_TZ];
#pragma unroll
      for (int j = 0; j < SP_TZ; ++j) wz[j] = ws[12 + j];
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        const double q = qw[sl * QS + c] * cxy;
#pragma unroll
        for (int j = 0; j < SP_TZ; ++j) acc[c][j] = fma(q, wz[j], acc[c][j]);
      }
    }
    __syncwarp();
  }
  const int x = px0 + xi, y = py0 + yi;
  if (x < g.dims[0] && y < g.dims[1]) {
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      double* dst = grids + c * g.ch_stride + x * g.stride[0] + y * g.stride[1];
#pragma unroll
      for (int j = 0; j < SP_TZ; ++j) {
        const int z = z0 + j;
        if (z < g.dims[2]) dst[z * g.stride[2]] = acc[c][j];
      }
    }
  }
}

hs_status launch_spread(hs_ctx* ctx, const double4* pts, const double* w, int n, int nch, const int* bin_start,
                        const GridGeom& g, double* grids, int ldw, bool reuse_wtab) {
  if (ldw <= 0) ldw = nch;  // weights row stride (a channel group of wider rows: ldw > nch)
  if (g.P > SP_MAXP) return fail(HS_ERR_PARAMETER, "spread supports window support P <= 64");
  const int nbx = sp_nbins(g, 0), nby = sp_nbins(g, 1), nbz = sp_nbins(g, 2);
  // default: v3 (window tables + cp.async staging + DMMA); HS_SPREAD_V0 = DMMA with in-tile window
  // arithmetic, HS_SPREAD_V1 = scalar DFMA, HS_SPREAD_V2 = warp-independent (comparison only)
  static const int variant = getenv("HS_SPREAD_V0") ? 0 : getenv("HS_SPREAD_V1") ? 1 : getenv("HS_SPREAD_V2") ? 2 : 3;
  // window tables + cp.async (default); HS_SPREAD_FLY=1: producers compute the slices (comparison:
  // 24.4 vs 18.1 ms at HL -- the producers' recurrence chains then bound the consumers, while the
  // table re-reads, 11 GB per channel group, run at ~1.2 TB/s off the critical path)
  static const bool tables = getenv("HS_SPREAD_FLY") == nullptr;
  if (variant == 3) {
    const WTab wt = WTab::make(g.P);
    void* scr3 = nullptr;
    const size_t nn = (size_t)std::max(n, 1);
    int4* lo = nullptr;
    double* tab = nullptr;
    if (tables) {
      HS_TRY(ctx_scratch(ctx, nn * (sizeof(int4) + sizeof(double) * wt.stride), &scr3));
      lo = (int4*)scr3;
      tab = (double*)(lo + nn);
    }
    if (n > 0 && tables && !reuse_wtab) {  // (reuse: same sources, tables of the previous call intact)
      const int gs = (int)std::min<int64_t>(ceil_div((int64_t)n * 3 * 32, 256), ctx->sm_count * 16);
      k_spread_wtab<<<gs, 256, 0, ctx->stream>>>(pts, n, g, wt, lo, tab);
      HS_LAUNCHED(ctx);
    }
    dim3 grid(nbx * nby * nbz);
    // default: 16 consumer warps (4x4 patches), up to 7 channels per launch, groups balanced
    // (7 -> 7, 13 -> 7 + 6); HS_SPREAD_W8=1: 8 warps (4x8 patches), 4 channels per launch
    static const bool w8 = getenv("HS_SPREAD_W8") != nullptr;
    if (tables && !w8 && nch >= 3) {
      const int ngroup = (nch + 6) / 7;
      for (int gi = 0, c0 = 0; gi < ngroup; ++gi) {
        const int cn = (nch - c0) / (ngroup - gi);
        double* gout = grids + (size_t)c0 * g.ch_stride;
        const double* wc0 = w + c0;
        switch (cn) {
#define HS_SP16(N)                                                                                                 \
  case N: {                                                                                                        \
    const size_t smm = sizeof(double) * (16 * 32 / SW_CH) * SwBuf<N>::DOUBLES;                                     \
    HS_CUDA(cudaFuncSetAttribute(k_spread_mma4<N, false, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,        \
                                 (int)smm));                                                                       \
    k_spread_mma4<N, false, 16><<<grid, (16 + SW_NP) * 32, smm, ctx->stream>>>(lo, tab, wt, pts, wc0, ldw,         \
                                                                             bin_start, g, nbx, nby, nbz, gout);   \
  } break;
          HS_SP16(3) HS_SP16(4) HS_SP16(5) HS_SP16(6) HS_SP16(7)
#undef HS_SP16
          default: return fail(HS_ERR_PARAMETER, "spread channel group");
        }
        HS_LAUNCHED(ctx);
        c0 += cn;
      }
      return HS_OK;
    }
    for (int c0 = 0; c0 < nch; c0 += SP_MAXCH) {
      const int cn = std::min(SP_MAXCH, nch - c0);
      double* gout = grids + (size_t)c0 * g.ch_stride;
      const double* wc0 = w + c0;
      switch (cn) {
#define HS_SP3(N)                                                                                                    \
  case N: {                                                                                                          \
    const size_t smm = sizeof(double) * SW_K * SwBuf<N>::DOUBLES;                                                    \
    if (tables) {                                                                                                    \
      HS_CUDA(cudaFuncSetAttribute(k_spread_mma4<N, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smm)); \
      k_spread_mma4<N, false><<<grid, SW_THREADS, smm, ctx->stream>>>(lo, tab, wt, pts, wc0, ldw, bin_start, g, nbx, \
                                                                      nby, nbz, gout);                               \
    } else {                                                                                                         \
      HS_CUDA(cudaFuncSetAttribute(k_spread_mma4<N, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smm));  \
      k_spread_mma4<N, true><<<grid, SW_THREADS, smm, ctx->stream>>>(lo, tab, wt, pts, wc0, ldw, bin_start, g, nbx,  \
                                                                     nby, nbz, gout);                                \
    }                                                                                                                \
  } break;
        HS_SP3(1) HS_SP3(2) HS_SP3(3) HS_SP3(4)
#undef HS_SP3
      }
      HS_LAUNCHED(ctx);
    }
    return HS_OK;
  }
  void* scr = nullptr;
  const size_t per = sizeof(int4) + sizeof(double4) + sizeof(double2);
  HS_TRY(ctx_scratch(ctx, per * (size_t)std::max(n, 1), &scr));
  int4* lo = (int4*)scr;
  double4* wxy = (double4*)(lo + std::max(n, 1));
  double2* wz = (double2*)(wxy + std::max(n, 1));
  if (n > 0) {
    const int gs = (int)std::min<int64_t>(ceil_div(n, 256), ctx->sm_count * 8);
    k_spread_windows<<<gs, 256, 0, ctx->stream>>>(pts, n, g, lo, wxy, wz);
    HS_LAUNCHED(ctx);
  }
  WinConst wc{};
  for (int a = 0; a < g.P; ++a) wc.e3[a] = std::exp(-g.alpha * (g.h * a) * (g.h * a));
  dim3 grid(nbx * nby * nbz), block(256);
  for (int c0 = 0; c0 < nch; c0 += SP_MAXCH) {
    const int cn = std::min(SP_MAXCH, nch - c0);
    double* gout = grids + (size_t)c0 * g.ch_stride;
    const double* wc0 = w + c0;
    switch (cn) {
#define HS_SP(N)                                                                                              \
  case N:                                                                                                     \
    if (variant == 0) {                                                                                       \
      constexpr int CHM = 64;                                                                                 \
      const size_t smm = sizeof(double) * CHM * (SP_TX + SP_TY + SP_TZ + 3 + (N | 1)) + sizeof(unsigned) * CHM; \
      HS_CUDA(cudaFuncSetAttribute(k_spread_mma<N, CHM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smm)); \
      k_spread_mma<N, CHM><<<grid, block, smm, ctx->stream>>>(lo, wxy, wz, wc0, nch, bin_start, g, wc, nbx, nby, nbz, \
                                                              gout);                                          \
    } else if (variant == 1)                                                                                  \
      k_spread<N><<<grid, block, 0, ctx->stream>>>(lo, wxy, wz, wc0, nch, bin_start, g, wc, nbx, nby, nbz, gout); \
    else {                                                                                                    \
      const size_t sm2 = sizeof(double) * 8 * 32 * (SW_STRIDE + (N | 1));                                     \
      HS_CUDA(cudaFuncSetAttribute(k_spread2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));     \
      k_spread2<N><<<grid, block, sm2, ctx->stream>>>(lo, wxy, wz, wc0, nch, bin_start, g, wc, nbx, nby, nbz, gout); \
    }                                                                                                         \
    break;
      HS_SP(1) HS_SP(2) HS_SP(3) HS_SP(4)
#undef HS_SP
    }
    HS_LAUNCHED(ctx);
  }
  return HS_OK;
}

// ---------------------------------------------------------------------------
// Gather: warp per point, lanes over z.  MODE 0: generic channels -> out[perm[i]*ldo + c]
// (ewald_fourier.gather); MODE 1: half/free Fourier velocity with T1 (3) and T2 (3).
template <int NCH, int MODE>
__global__ void __launch_bounds__(256) k_gather(const double4* __restrict__ pts, const int* __restrict__ perm,
                                                int n, GridGeom g, const double* __restrict__ grids,
                                                double* __restrict__ out, int ldo, double scale,
                                                double* __restrict__ u_total, const double* __restrict__ u_real,
                                                unsigned* __restrict__ flags) {
  __shared__ double s_w[8][2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int P = g.P;
  for (int i = blockIdx.x * 8 + warp; i < n; i += gridDim.x * 8) {
    const double4 p = pts[i];
    const int64_t lx = g_lo(g, 0, p.x);
    const int64_t ly = g_lo(g, 1, p.y);
    const int64_t lz = g_lo(g, 2, p.z);
    const bool bad = lx < 0 || ly < 0 || lz < 0 || lx + P > g.dims[0] || ly + P > g.dims[1] || lz + P > g.dims[2];
    double acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = 0.0;
    if (!bad) {
      __syncwarp();
      if (lane < P) {
        const double dx = g_d(g, 0, p.x, lx + lane);
        const double dy = g_d(g, 1, p.y, ly + lane);
        s_w[warp][0][lane] = exp(-g.alpha * dx * dx);
        s_w[warp][1][lane] = exp(-g.alpha * dy * dy);
      }
      double wz = 0.0;
      if (lane < P) {
        const double dz = g_d(g, 2, p.z, lz + lane);
        wz = exp(-g.alpha * dz * dz);
      }
      __syncwarp();
      const int zi = lane < P ? lane : 0;
      const double* base = grids + lx * g.stride[0] + ly * g.stride[1] + (lz + zi) * g.stride[2];
      for (int a = 0; a < P; ++a) {
        const double wxa = g.pref * s_w[warp][0][a];
        for (int b = 0; b < P; ++b) {
          const double wv = (wxa * s_w[warp][1][b]) * wz;
          const double* q = base + a * g.stride[0] + b * g.stride[1];
#pragma unroll
          for (int c = 0; c < NCH; ++c) acc[c] = fma(__ldg(q + c * g.ch_stride), wv, acc[c]);
        }
      }
    } else if (lane == 0) {
      atomicOr(flags, FLAG_OUT_OF_GRID);
    }
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = warp_sum(acc[c]);
    if (lane == 0) {
      const int o = perm ? perm[i] : i;
      const double h3 = g.h * g.h * g.h;
      if (MODE == 0) {
#pragma unroll
        for (int c = 0; c < NCH; ++c) out[(size_t)o * ldo + c] = acc[c] * h3 * scale;
      } else {
        // u_F = h^3 sum w T1 - x3 h^3 sum w T2   (ewald_fourier.py:626-630)
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          double v = acc[q] * h3;
          if (NCH == 6) v -= p.z * (acc[3 + q] * h3);
          if (out) out[3 * (size_t)o + q] = v;
          if (u_total) u_total[3 * (size_t)o + q] = (u_real ? u_real[3 * (size_t)o + q] : 0.0) + v;
        }
      }
    }
  }
}

hs_status launch_gather(hs_ctx* ctx, const double4* pts, const int* perm, int n, int nch, const GridGeom& g,
                        const double* grids, double* out, int ldo, double scale) {
  if (n == 0) return HS_OK;
  if (g.P > 32) return fail(HS_ERR_PARAMETER, "gather supports window support P <= 32");
  const int gs = (int)std::min<int64_t>(ceil_div(n, 8), ctx->sm_count * 64);
  switch (nch) {
#define HS_GA(N)                                                                                               \
  case N:                                                                                                      \
    k_gather<N, 0><<<gs, 256, 0, ctx->stream>>>(pts, perm, n, g, grids, out, ldo, scale, nullptr, nullptr,   \
                                                ctx->d_flags);                                               \
    break;
    HS_GA(1) HS_GA(2) HS_GA(3) HS_GA(4) HS_GA(5) HS_GA(6) HS_GA(7) HS_GA(8)
#undef HS_GA
    default:
      return fail(HS_ERR_PARAMETER, "gather supports 1..8 channels per launch");
  }
  HS_LAUNCHED(ctx);
  return HS_OK;
}

// ---------------------------------------------------------------------------
// Fourier gather of the half-space pipeline (ewald_fourier.py:626-630):
//   u_F(t) = h^3 [ sum_p w_t(p) T1(p) - x3_t sum_p w_t(p) T2(p) ]
// A CTA owns GA_T consecutive targets of the 4x4x4-sub-tile order (spatially compact).
// It walks the x-planes of the union of their supports; each plane slab
// (y-range x z-range x channels) is staged in shared memory by the whole CTA
// (coalesced rows of the channel-interleaved output grid), then every warp
// (lanes = 32 targets) accumulates its targets from broadcast shared-memory reads.
// Window factors come from the Gaussian recurrence w(n+1) = w(n) r(n),
// r(n+1) = r(n) q (q = e^{-2 alpha h^2}) started at each lane's first support node.
constexpr int GA_T = 256;                 // targets (threads) per CTA
constexpr int GA_SMEM_DOUBLES = 9216;     // 72 KB plane slab
constexpr int GA_ZM = 32;                 // register z-window length (fast path)

template <int NCH, int PITCH>
__global__ void __launch_bounds__(GA_T, 2) k_gather3(const double4* __restrict__ pts, const int* __restrict__ orig,
                                                    int n, GridGeom g, const double* __restrict__ T,
                                                    double* __restrict__ u_four, double* __restrict__ u_tot,
                                                    const double* __restrict__ u_real, unsigned* __restrict__ flags) {
  extern __shared__ __align__(16) double slab[];  // GA_SMEM_DOUBLES
  __shared__ int s_box[6];
  const int lane = threadIdx.x & 31;
  const int P = g.P;
  const double q = exp(-2.0 * g.alpha * g.h * g.h);
  for (int base = blockIdx.x * GA_T; base < n; base += gridDim.x * GA_T) {
    const int t = base + threadIdx.x;
    const bool valid = t < n;
    const double4 pt = pts[valid ? t : base];
    const double pc[3] = {pt.x, pt.y, pt.z};
    int lo[3];
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int64_t l = g_lo(g, k, pc[k]);
      bad |= (l < 0) || (l + P > g.dims[k]);
      lo[k] = (int)l;
    }
    if (valid && bad) atomicOr(flags, FLAG_OUT_OF_GRID);
    const bool act = valid && !bad;
    // warp and CTA union boxes
    int W0[3], W1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      W0[k] = (int)__reduce_min_sync(0xffffffffu, (unsigned)(act ? lo[k] : 0x7fffffff));
      W1[k] = (int)__reduce_max_sync(0xffffffffu, (unsigned)(act ? lo[k] + P : 0));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      s_box[0] = s_box[1] = s_box[2] = 0x7fffffff;
      s_box[3] = s_box[4] = s_box[5] = 0;
    }
    __syncthreads();
    if (lane == 0 && W1[0] > 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        atomicMin(&s_box[k], W0[k]);
        atomicMax(&s_box[3 + k], W1[k]);
      }
    }
    __syncthreads();
    const int X0 = s_box[0], Y0 = s_box[1], Z0 = s_box[2], X1 = s_box[3], Y1 = s_box[4], Z1 = s_box[5];
    double acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = 0.0;
    if (X1 > X0) {
      double w0[3], r0[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double d = g_d(g, k, pc[k], lo[k]);
        w0[k] = act ? exp(-g.alpha * d * d) : 0.0;
        r0[k] = exp(g.alpha * (2.0 * d * g.h - g.h * g.h));
      }
      w0[2] *= g.pref;
      // per-lane z window over this warp's z range, zero outside the lane's support
      const int nzw = W1[2] - W0[2];
      const bool zfast = nzw <= GA_ZM;
      double wzv[GA_ZM];
      {
        double wz = w0[2], rz = r0[2];
#pragma unroll
        for (int i = 0; i < GA_ZM; ++i) {
          const int z = W0[2] + i;
          const bool inz = z >= lo[2] && z < lo[2] + P;
          wzv[i] = inz ? wz : 0.0;
          if (inz) {
            wz *= rz;
            rz *= q;
          }
        }
      }
      const int nzu = Z1 - Z0;
      const int rowlen = nzu * PITCH;                       // doubles per staged row
      const int ychunk = max(1, min(Y1 - Y0, GA_SMEM_DOUBLES / rowlen));
      double wx = w0[0], rx = r0[0];
      for (int x = X0; x < X1; ++x) {
        const bool inx = x >= lo[0] && x < lo[0] + P;
        const double wxe = inx ? wx : 0.0;
        if (inx) {
          wx *= rx;
          rx *= q;
        }
        const bool warp_x = __any_sync(0xffffffffu, wxe != 0.0);
        double wy = w0[1], ry = r0[1];
        for (int yc = Y0; yc < Y1; yc += ychunk) {
          const int yn = min(ychunk, Y1 - yc);
          __syncthreads();
          // stage rows y in [yc, yc+yn) of plane x: contiguous (z, channel) runs
          {
            const int nvec = rowlen / 2;  // double2 per row
            for (int i = threadIdx.x; i < yn * nvec; i += GA_T) {
              const int r = i / nvec, v = i - r * nvec;
              const double* src = T + (int64_t)x * g.stride[0] + (int64_t)(yc + r) * g.stride[1] +
                                  (int64_t)Z0 * PITCH + 2 * v;
              reinterpret_cast<double2*>(slab)[r * nvec + v] = __ldg(reinterpret_cast<const double2*>(src));
            }
          }
          __syncthreads();
          if (!warp_x) continue;
          const int ya = max(yc, W0[1]), yb = min(yc + yn, W1[1]);
          for (int y = yc; y < ya; ++y) {  // advance the y recurrence through rows before this warp's range
            if (y >= lo[1] && y < lo[1] + P) {
              wy *= ry;
              ry *= q;
            }
          }
          for (int y = ya; y < yb; ++y) {
            const bool iny = y >= lo[1] && y < lo[1] + P;
            const double wye = iny ? wy : 0.0;
            if (iny) {
              wy *= ry;
              ry *= q;
            }
            const double cxy = wxe * wye;
            if (!__any_sync(0xffffffffu, cxy != 0.0)) continue;
            const double* row = slab + (y - yc) * rowlen;
            if (zfast) {
              // fast path: per-lane z window in registers, 6 FMAs + broadcast loads per node
              double S[NCH];
#pragma unroll
              for (int c = 0; c < NCH; ++c) S[c] = 0.0;
              const double* pz0 = row + (W0[2] - Z0) * PITCH;
#pragma unroll
              for (int i = 0; i < GA_ZM; ++i) {
                const int ii = min(i, nzw - 1);
                double v[PITCH];
#pragma unroll
                for (int c = 0; c < PITCH; c += 2) {
                  const double2 vv = *reinterpret_cast<const double2*>(pz0 + ii * PITCH + c);
                  v[c] = vv.x;
                  v[c + 1] = vv.y;
                }
#pragma unroll
                for (int c = 0; c < NCH; ++c) S[c] = fma(wzv[i], v[c], S[c]);
              }
#pragma unroll
              for (int c = 0; c < NCH; ++c) acc[c] = fma(cxy, S[c], acc[c]);
              continue;
            }
            double wz = w0[2] * cxy, rz = r0[2];
            for (int z = W0[2]; z < W1[2]; ++z) {
              const bool inz = z >= lo[2] && z < lo[2] + P;
              const double we = inz ? wz : 0.0;
              if (inz) {
                wz *= rz;
                rz *= q;
              }
              const double* pz = row + (z - Z0) * PITCH;
              double v[PITCH];
#pragma unroll
              for (int c = 0; c < PITCH; c += 2) {
                const double2 vv = *reinterpret_cast<const double2*>(pz + c);
                v[c] = vv.x;
                v[c + 1] = vv.y;
              }
#pragma unroll
              for (int c = 0; c < NCH; ++c) acc[c] = fma(we, v[c], acc[c]);
            }
          }
          for (int y = yb; y < yc + yn; ++y) {  // rows after this warp's range (keep the recurrence in step)
            if (y >= lo[1] && y < lo[1] + P) {
              wy *= ry;
              ry *= q;
            }
          }
        }
      }
    }
    if (act) {
      const int o = orig[t];
      const double h3 = g.h * g.h * g.h;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double v = acc[k] * h3;
        if (NCH == 6) v -= pt.z * (acc[3 + k] * h3);
        if (u_four) u_four[3 * (size_t)o + k] = v;
        if (u_tot) u_tot[3 * (size_t)o + k] = (u_real ? u_real[3 * (size_t)o + k] : 0.0) + v;
      }
    }
  }
}

// Barrier-free gather: lanes = 32 nearby targets (one warp is independent of the others).
// The warp walks the (x,y) columns of its targets' union; each column's z-range (<= GA_ZM
// nodes x 6 channels, 1.5 KB) is loaded cooperatively (one 48-byte node per lane, fully
// coalesced) into a warp-private, double-buffered shared-memory slot one column ahead, and
// consumed with broadcast 128-bit reads against the per-lane register z-window.
template <int NCH, int PITCH>
__global__ void __launch_bounds__(256, 2) k_gather5(const double4* __restrict__ pts, const int* __restrict__ orig,
                                                   int n, GridGeom g, const double* __restrict__ T,
                                                   double* __restrict__ u_four, double* __restrict__ u_tot,
                                                   const double* __restrict__ u_real, unsigned* __restrict__ flags) {
  __shared__ __align__(16) double s_col[8][2][GA_ZM * PITCH];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = gridDim.x * (blockDim.x >> 5);
  const int P = g.P;
  const double q = exp(-2.0 * g.alpha * g.h * g.h);
  for (int wbase = (blockIdx.x * (blockDim.x >> 5) + warp) * 32; wbase < n; wbase += nwarps * 32) {
    const int t = wbase + lane;
    const bool valid = t < n;
    const double4 pt = pts[valid ? t : wbase];
    const double pc[3] = {pt.x, pt.y, pt.z};
    int lo[3];
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int64_t l = g_lo(g, k, pc[k]);
      bad |= (l < 0) || (l + P > g.dims[k]);
      lo[k] = (int)l;
    }
    if (valid && bad) atomicOr(flags, FLAG_OUT_OF_GRID);
    const bool act = valid && !bad;
    int W0[3], W1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      W0[k] = (int)__reduce_min_sync(0xffffffffu, (unsigned)(act ? lo[k] : 0x7fffffff));
      W1[k] = (int)__reduce_max_sync(0xffffffffu, (unsigned)(act ? lo[k] + P : 0));
    }
    double acc[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) acc[c] = 0.0;
    const int nzw = W1[2] - W0[2];
    if (W1[0] > W0[0] && nzw <= GA_ZM) {
      double w0[3], r0[3];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double d = g_d(g, k, pc[k], lo[k]);
        w0[k] = act ? exp(-g.alpha * d * d) : 0.0;
        r0[k] = exp(g.alpha * (2.0 * d * g.h - g.h * g.h));
      }
      w0[2] *= g.pref;
      double wzv[GA_ZM];
      {
        double wz = w0[2], rz = r0[2];
#pragma unroll
        for (int i = 0; i < GA_ZM; ++i) {
          const int z = W0[2] + i;
          const bool inz = z >= lo[2] && z < lo[2] + P;
          wzv[i] = inz ? wz : 0.0;
          if (inz) {
            wz *= rz;
            rz *= q;
          }
        }
      }
      const int ny_u = W1[1] - W0[1];
      const int ncol = (W1[0] - W0[0]) * ny_u;
      const int zl = min(lane, nzw - 1);  // node this lane loads (clamped; wzv is 0 beyond nzw)
      auto load_col = [&](int ci, double2* r) {
        const int x = W0[0] + ci / ny_u, y = W0[1] + ci % ny_u;
        const double* src = T + (int64_t)x * g.stride[0] + (int64_t)y * g.stride[1] + (int64_t)(W0[2] + zl) * PITCH;
#pragma unroll
        for (int c = 0; c < PITCH / 2; ++c) r[c] = __ldg(reinterpret_cast<const double2*>(src) + c);
      };
      double2 nxt[PITCH / 2];
      load_col(0, nxt);
      double wx = w0[0], rx = r0[0], wy = w0[1], ry = r0[1], wxe = 0.0;
      for (int ci = 0; ci < ncol; ++ci) {
        const int buf = ci & 1;
        double2* dst = reinterpret_cast<double2*>(s_col[warp][buf]) + lane * (PITCH / 2);
#pragma unroll
        for (int c = 0; c < PITCH / 2; ++c) dst[c] = nxt[c];
        __syncwarp();
        if (ci + 1 < ncol) load_col(ci + 1, nxt);
        // window factors of column (x, y) (x-major, y-minor traversal)
        const int yy = ci % ny_u;
        if (yy == 0) {
          const int x = W0[0] + ci / ny_u;
          const bool inx = x >= lo[0] && x < lo[0] + P;
          wxe = inx ? wx : 0.0;
          if (inx) {
            wx *= rx;
            rx *= q;
          }
          wy = w0[1];
          ry = r0[1];
        }
        const int y = W0[1] + yy;
        const bool iny = y >= lo[1] && y < lo[1] + P;
        const double cxy = wxe * (iny ? wy : 0.0);
        if (iny) {
          wy *= ry;
          ry *= q;
        }
        if (__any_sync(0xffffffffu, cxy != 0.0)) {
          const double* colp = s_col[warp][buf];
          double S[NCH];
#pragma unroll
          for (int c = 0; c < NCH; ++c) S[c] = 0.0;
#pragma unroll
          for (int i = 0; i < GA_ZM; ++i) {
            double v[PITCH];
#pragma unroll
            for (int c = 0; c < PITCH; c += 2) {
              const double2 vv = *reinterpret_cast<const double2*>(colp + i * PITCH + c);
              v[c] = vv.x;
              v[c + 1] = vv.y;
            }
#pragma unroll
            for (int c = 0; c < NCH; ++c) S[c] = fma(wzv[i], v[c], S[c]);
          }
#pragma unroll
          for (int c = 0; c < NCH; ++c) acc[c] = fma(cxy, S[c], acc[c]);
        }
      }
    } else if (W1[0] > W0[0]) {
      // sparse warp (z range wider than the register window): each lane sums its own support
      if (act) {
        double ws[3][GA_ZM];
        for (int k = 0; k < 3; ++k)
          for (int a2 = 0; a2 < P; ++a2) {
            const double d = g_d(g, k, pc[k], lo[k] + a2);
            ws[k][a2] = exp(-g.alpha * d * d);
          }
        for (int a2 = 0; a2 < P; ++a2)
          for (int b2 = 0; b2 < P; ++b2) {
            const double cxy = g.pref * ws[0][a2] * ws[1][b2];
            const double* src = T + (int64_t)(lo[0] + a2) * g.stride[0] + (int64_t)(lo[1] + b2) * g.stride[1] +
                                (int64_t)lo[2] * PITCH;
            for (int c2 = 0; c2 < P; ++c2) {
              const double wv = cxy * ws[2][c2];
#pragma unroll
              for (int c = 0; c < NCH; ++c) acc[c] = fma(wv, __ldg(src + c2 * PITCH + c), acc[c]);
            }
          }
      }
    }
    if (act) {
      const int o = orig[t];
      const double h3 = g.h * g.h * g.h;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double v = acc[k] * h3;
        if (NCH == 6) v -= pt.z * (acc[3 + k] * h3);
        if (u_four) u_four[3 * (size_t)o + k] = v;
        if (u_tot) u_tot[3 * (size_t)o + k] = (u_real ? u_real[3 * (size_t)o + k] : 0.0) + v;
      }
    }
  }
}

// Gather v7 (default).  Targets are sorted by (4x4 (x,y) block, z node) of their window
// centre and cut into RUNS of <= G7_TG targets of one block whose windows start within
// 32 - P z nodes of each other, and ITEMS of <= G7_WARPS runs of one block
// (k_g7_items).  A CTA takes an item, one warp per run; the warp's lanes are 32
// consecutive z nodes.  The CTA walks the (x,y) columns of the item's union (a (P+3)^2
// square), staging each column's z-range once through a cp.async ring; every lane takes
// ITS node of the column (all channels) and accumulates, per target t and channel c,
//   E_l[t][c] += wx_t(x) wy_t(y) G_c(x, y, z_l)
// so each shared-memory value feeds G7_TG fused multiply-adds from registers (no
// broadcast reads).  The z factor is applied once at the end, u_t,c = sum_l wz_t(z_l)
// E_l[t][c] (warp reduction).  The x/y factors of a run live in warp-private tables.
// Windows are evaluated directly, exp(-alpha d^2), as in the reference (_gridding.py:21-30).
#ifndef G7_STEP_DEF
#define G7_STEP_DEF 4
#endif
#ifndef G7_ZC_DEF
#define G7_ZC_DEF 48
#endif
// columns per barrier step (G7_STEP) and ring slots (3 steps in flight), static shared memory
constexpr int G7_TG = 8, G7_GW = 32, G7_WARPS = 4, G7_ZC = G7_ZC_DEF, G7_STEP = G7_STEP_DEF, G7_R = 3 * G7_STEP;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// runs and items of one 4x4 block's targets [b, e) (z-sorted); emit == nullptr: count only
__device__ int g7_cut(const double4* __restrict__ pts, int b, int e, const GridGeom& g, int4* emit) {
  int nitem = 0, i = b;
  while (i < e) {
    const int ib = i;
    int nrun = 0;
    int lens = 0;
    const int64_t zi0 = g_lo(g, 2, pts[i].z);
    while (i < e && nrun < G7_WARPS) {
      const int64_t zr0 = g_lo(g, 2, pts[i].z);
      if (zr0 - zi0 > G7_ZC - g.P) break;
      int len = 1;
      ++i;
      while (i < e && len < G7_TG) {
        const int64_t z = g_lo(g, 2, pts[i].z);
        if (z - zr0 > 32 - g.P || z - zi0 > G7_ZC - g.P) break;
        ++len;
        ++i;
      }
      lens |= len << (8 * nrun);
      ++nrun;
    }
    if (emit) emit[nitem] = make_int4(ib, i - ib, lens, 0);
    ++nitem;
  }
  return nitem;
}

__global__ void k_g7_count(const double4* __restrict__ pts, const int* __restrict__ bstart, int nblk, int nz,
                           GridGeom g, int* __restrict__ cnt) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nblk; c += gridDim.x * blockDim.x)
    cnt[c] = g7_cut(pts, bstart[c * nz], bstart[(c + 1) * nz], g, nullptr);
}

__global__ void k_g7_fill(const double4* __restrict__ pts, const int* __restrict__ bstart, int nblk, int nz,
                          GridGeom g, const int* __restrict__ istart, int4* __restrict__ items) {
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < nblk; c += gridDim.x * blockDim.x)
    g7_cut(pts, bstart[c * nz], bstart[(c + 1) * nz], g, items + istart[c]);
}

template <int NCH, int PITCH>
__global__ void __launch_bounds__(G7_WARPS * 32, 2) k_gather7(const double4* __restrict__ pts,
                                                             const int* __restrict__ orig, const int4* __restrict__ items,
                                                             const int* __restrict__ n_items_d, GridGeom g,
                                                             const double* __restrict__ T,
                                                             double* __restrict__ u_four, double* __restrict__ u_tot,
                                                             const double* __restrict__ u_real,
                                                             unsigned* __restrict__ flags) {
  constexpr int TG = G7_TG, GW = G7_GW, NT = G7_WARPS * 32, CPN = PITCH / 2;  // 16-byte chunks per node
  __shared__ double s_w[G7_WARPS][2][TG][GW];
  __shared__ __align__(16) double s_ring[G7_R][G7_ZC * PITCH];
  __shared__ int s_u[G7_WARPS][6];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int P = g.P;
  double(*wx_tab)[GW] = s_w[warp][0];
  double(*wy_tab)[GW] = s_w[warp][1];
  const int n_items = *n_items_d;
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int4 item = items[it];
    int rb = item.x;
#pragma unroll
    for (int w = 0; w < G7_WARPS; ++w)
      if (w < warp) rb += (item.z >> (8 * w)) & 0xff;
    const int rlen = (item.z >> (8 * warp)) & 0xff;
    const int t = rb + lane;
    const bool valid = lane < rlen;
    const double4 pt = pts[valid ? t : item.x];
    const double pc[3] = {pt.x, pt.y, pt.z};
    int lo[3];
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const int64_t l = g_lo(g, k, pc[k]);
      bad |= (l < 0) || (l + P > g.dims[k]);
      lo[k] = (int)l;
    }
    if (valid && bad) atomicOr(flags, FLAG_OUT_OF_GRID);
    const bool act = valid && !bad;
    const unsigned amask = __ballot_sync(0xffffffffu, act);
    int W0[3], W1[3];
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      W0[k] = (int)__reduce_min_sync(0xffffffffu, (unsigned)(act ? lo[k] : 0x7fffffff));
      W1[k] = (int)__reduce_max_sync(0xffffffffu, (unsigned)(act ? lo[k] + P : 0));
    }
    __syncthreads();  // previous item done with s_u / ring / tables
    if (lane == 0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        s_u[warp][k] = amask ? W0[k] : 0x7fffffff;
        s_u[warp][3 + k] = amask ? W1[k] : (int)0x80000000;
      }
    }
    __syncthreads();
    int C0[3] = {0x7fffffff, 0x7fffffff, 0x7fffffff}, C1[3] = {(int)0x80000000, (int)0x80000000, (int)0x80000000};
#pragma unroll
    for (int w = 0; w < G7_WARPS; ++w)
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        C0[k] = min(C0[k], s_u[w][k]);
        C1[k] = max(C1[k], s_u[w][3 + k]);
      }
    // no active target in the item (all out of the grid): C0 = INT_MAX and C1 - C0 would wrap
    if (C0[0] == 0x7fffffff) continue;
    const int nxu = C1[0] - C0[0], nyu = C1[1] - C0[1], nzu = C1[2] - C0[2];
    // limits exceeded (only with out-of-grid targets, an error anyway)
    if (nxu <= 0 || nxu > GW || nyu > GW || nzu > G7_ZC) continue;
    double res[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) res[c] = 0.0;
    // x / y window tables of this warp's run (0 outside a target's support)
#pragma unroll
    for (int tt = 0; tt < TG; ++tt) {
      const bool tin = (amask >> tt) & 1u;
      const double px = __shfl_sync(0xffffffffu, pc[0], tt), py = __shfl_sync(0xffffffffu, pc[1], tt);
      const int lx = __shfl_sync(0xffffffffu, lo[0], tt), ly = __shfl_sync(0xffffffffu, lo[1], tt);
      double vx = 0.0, vy = 0.0;
      const int x = C0[0] + lane, y = C0[1] + lane;
      if (tin && lane < nxu && x >= lx && x < lx + P) {
        const double d = g_d(g, 0, px, x);
        vx = exp(-g.alpha * d * d);
      }
      if (tin && lane < nyu && y >= ly && y < ly + P) {
        const double d = g_d(g, 1, py, y);
        vy = exp(-g.alpha * d * d);
      }
      wx_tab[tt][lane] = vx;
      wy_tab[tt][lane] = vy;
    }
    __syncwarp();
    const int ncol = nxu * nyu, nchunk = nzu * CPN;
    // cp.async issue state: this thread's 16-byte chunks k = tid + NT j of every column
    const double* colp = T + (int64_t)C0[0] * g.stride[0] + (int64_t)C0[1] * g.stride[1] + (int64_t)C0[2] * PITCH +
                         2 * threadIdx.x;
    const int64_t row_wrap = g.stride[0] - (int64_t)nyu * g.stride[1];
    int iy = 0, nissued = 0;
    auto issue_step = [&](int step) {
#pragma unroll
      for (int j = 0; j < G7_STEP; ++j) {
        if (nissued < ncol) {
          double* dst = s_ring[(step * G7_STEP + j) % G7_R] + 2 * threadIdx.x;
#pragma unroll
          for (int q = 0; q < (G7_ZC * CPN + NT - 1) / NT; ++q)
            if ((int)threadIdx.x + q * NT < nchunk) cp_async16(dst + 2 * q * NT, colp + 2 * q * NT);
          ++nissued;
          colp += g.stride[1];
          if (++iy == nyu) {
            iy = 0;
            colp += row_wrap;
          }
        }
      }
      cp_async_commit();
    };
    issue_step(0);
    issue_step(1);
    const int zn = min(W0[2] - C0[2] + lane, nzu - 1);  // this lane's node in the staged column
    double E[TG][NCH];
#pragma unroll
    for (int tt = 0; tt < TG; ++tt)
#pragma unroll
      for (int c = 0; c < NCH; ++c) E[tt][c] = 0.0;
    int cx = 0, cy = 0, slot = 0;
    // one column: node values and window factors, then the FMAs
    auto column = [&](int sl) {
      const double2* src = reinterpret_cast<const double2*>(&s_ring[sl][zn * PITCH]);
      double v[PITCH], cxy[TG];
#pragma unroll
      for (int c = 0; c < CPN; ++c) {
        const double2 q2 = src[c];
        v[2 * c] = q2.x;
        v[2 * c + 1] = q2.y;
      }
#pragma unroll
      for (int tt = 0; tt < TG; ++tt) cxy[tt] = wx_tab[tt][cx] * wy_tab[tt][cy];
      if (++cy == nyu) {
        cy = 0;
        ++cx;
      }
#pragma unroll
      for (int tt = 0; tt < TG; ++tt)
#pragma unroll
        for (int c = 0; c < NCH; ++c) E[tt][c] = fma(cxy[tt], v[c], E[tt][c]);
    };
    const int nfull = ncol / G7_STEP, nrem = ncol - nfull * G7_STEP;
    for (int sidx = 0; sidx < nfull; ++sidx) {
      cp_async_wait<1>();
      __syncthreads();
      issue_step(sidx + 2);
      if (amask) {
#pragma unroll
        for (int j = 0; j < G7_STEP; ++j) column(slot + j);
      }
      slot = slot + G7_STEP == G7_R ? 0 : slot + G7_STEP;
    }
    if (nrem) {  // ragged last step (already issued)
      cp_async_wait<1>();
      __syncthreads();
      if (amask)
        for (int j = 0; j < nrem; ++j) column(slot + j);
    }
    cp_async_wait<0>();
    if (amask) {
      // z factors of this lane's node, reduce over the warp; lane t accumulates target t
      const int z = W0[2] + lane;
#pragma unroll
      for (int tt = 0; tt < TG; ++tt) {
        const double pz = __shfl_sync(0xffffffffu, pc[2], tt);
        const int lz = __shfl_sync(0xffffffffu, lo[2], tt);
        double wz = 0.0;
        if (((amask >> tt) & 1u) && z >= lz && z < lz + P) {
          const double d = g_d(g, 2, pz, z);
          wz = exp(-g.alpha * d * d);
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          const double sum = warp_sum(wz * E[tt][c]);
          if (lane == tt) res[c] = sum;
        }
      }
    }
    if (act) {
      const int o = orig[t];
      const double h3p = g.h * g.h * g.h * g.pref;
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        double v = res[k] * h3p;
        if (NCH == 6) v -= pt.z * (res[3 + k] * h3p);
        if (u_four) u_four[3 * (size_t)o + k] = v;
        if (u_tot) u_tot[3 * (size_t)o + k] = (u_real ? u_real[3 * (size_t)o + k] : 0.0) + v;
      }
    }
  }
}

bool gather_v5() {
  static const bool v5 = getenv("HS_GATHER_V5") != nullptr;  // previous default (comparison)
  return v5;
}

hs_status launch_gather_fourier(hs_ctx* ctx, const double4* pts, const int* orig, int n, int half, const GridGeom& g,
                                const double* T, double* u_fourier, double* u_total, const double* u_real,
                                const int* bstart) {
  if (n == 0) return HS_OK;
  static const bool v1 = getenv("HS_GATHER_V1") != nullptr;  // debugging aid: warp-per-target gather
  if (v1) {
    const int gs1 = (int)std::min<int64_t>(ceil_div(n, 8), ctx->sm_count * 64);
    if (half)
      k_gather<6, 1><<<gs1, 256, 0, ctx->stream>>>(pts, orig, n, g, T, u_fourier, 3, 1.0, u_total, u_real,
                                                   ctx->d_flags);
    else
      k_gather<3, 1><<<gs1, 256, 0, ctx->stream>>>(pts, orig, n, g, T, u_fourier, 3, 1.0, u_total, u_real,
                                                   ctx->d_flags);
    HS_LAUNCHED(ctx);
    return HS_OK;
  }
  if (g.P > GA_ZM) return fail(HS_ERR_PARAMETER, "window support P > 32 is not supported by the gather");
  static const bool v3 = getenv("HS_GATHER_V3") != nullptr;  // CTA-staged variant (comparison)
  if (!v3 && !gather_v5()) {
    if (!bstart) return fail(HS_ERR_PARAMETER, "gather v7 needs the block order");
    if (g.P > 32 || g.P > G7_ZC) return fail(HS_ERR_PARAMETER, "window support P > 32 is not supported by the gather");
    // items (worst case one per target): count per 4x4 block, scan, fill
    const int nb4 = ((g.dims[0] + 3) / 4) * ((g.dims[1] + 3) / 4);
    void* scr = nullptr;
    const size_t bytes = sizeof(int4) * (size_t)n + sizeof(int) * (3 * (size_t)nb4 + 8);
    HS_TRY(ctx_scratch(ctx, bytes, &scr));
    int4* items = (int4*)scr;
    int* cnt = (int*)(items + n);
    int* istart = cnt + nb4;  // nb4 + 1
    int* sc = istart + nb4 + 1;
    const int gsb = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nb4, 128), ctx->sm_count * 4));
    k_g7_count<<<gsb, 128, 0, ctx->stream>>>(pts, bstart, nb4, g.dims[2], g, cnt);
    HS_LAUNCHED(ctx);
    HS_TRY(exclusive_scan(ctx, cnt, nb4, istart, sc));
    k_g7_fill<<<gsb, 128, 0, ctx->stream>>>(pts, bstart, nb4, g.dims[2], g, istart, items);
    HS_LAUNCHED(ctx);
    const int gs7 = (int)std::min<int64_t>(n, (int64_t)ctx->sm_count * 2);
    if (half)
      k_gather7<6, 6><<<gs7, G7_WARPS * 32, 0, ctx->stream>>>(pts, orig, items, istart + nb4, g, T, u_fourier,
                                                             u_total, u_real, ctx->d_flags);
    else
      k_gather7<3, 4><<<gs7, G7_WARPS * 32, 0, ctx->stream>>>(pts, orig, items, istart + nb4, g, T, u_fourier,
                                                             u_total, u_real, ctx->d_flags);
    HS_LAUNCHED(ctx);
    return HS_OK;
  }
  if (!v3) {
    const int gs5 = (int)std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->sm_count * 32);
    if (half)
      k_gather5<6, 6><<<gs5, 256, 0, ctx->stream>>>(pts, orig, n, g, T, u_fourier, u_total, u_real, ctx->d_flags);
    else
      k_gather5<3, 4><<<gs5, 256, 0, ctx->stream>>>(pts, orig, n, g, T, u_fourier, u_total, u_real, ctx->d_flags);
    HS_LAUNCHED(ctx);
    return HS_OK;
  }
  const int gs = (int)std::min<int64_t>(ceil_div(n, GA_T), (int64_t)ctx->sm_count * 32);
  const size_t smem = sizeof(double) * GA_SMEM_DOUBLES;
  if (half) {
    HS_CUDA(cudaFuncSetAttribute(k_gather3<6, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_gather3<6, 6><<<gs, GA_T, smem, ctx->stream>>>(pts, orig, n, g, T, u_fourier, u_total, u_real, ctx->d_flags);
  } else {
    HS_CUDA(cudaFuncSetAttribute(k_gather3<3, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_gather3<3, 4><<<gs, GA_T, smem, ctx->stream>>>(pts, orig, n, g, T, u_fourier, u_total, u_real, ctx->d_flags);
  }
  HS_LAUNCHED(ctx);
  return HS_OK;
}

}  // namespace hs

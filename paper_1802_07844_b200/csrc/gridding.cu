// gridding.cu -- Gaussian spreading and gathering on the extended grid
// (reference: _gridding.py:21-89, ewald_fourier.py:319-346,626-630).
//
// Spreading (k_spread_wtab + k_spread_mma4) is owner-computes and atomic-free: one CTA owns a
// 16x16x8 tile of grid nodes; producer warps stream the sources whose P^3 support can reach
// the tile (bin-sorted by the tile of their window-centre cell: 3x3 (x,y) runs of 5 z-bins)
// and stage their window slices (cp.async from per-source window rows) and weights into an
// mbarrier ring; 16 consumer warps, one 4x4 (x,y) x 8 z patch each, accumulate with FP64
// DMMA in registers.  Each grid value is written exactly once, deterministically, without
// FP64 shared-memory atomics (a CAS loop on sm_100a).
//
// Gathering: k_gather8 in the plan (runs of <= 8 targets of one 4x4 block, columns staged by
// cp.async, the z contraction on the FP64 tensor pipe); k_gather (warp per target, lanes over
// the z nodes of one support column) for the stand-alone API and window supports P > 29.
#define HS_TU_ID 2  // checked build: source of a failing HS_CHECK
#include <cmath>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace hs {

__global__ void k_grid_keys(const double* __restrict__ pos, int n_src, int n, int mode, GridGeom g, int nbx,
                            int nby, int nbz, int* __restrict__ keys, unsigned* __restrict__ flags) {
  const bool fine = (mode & 8) != 0;  // gather targets: (4x4 column, z node) order
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
    if (fine) {
      // gather (k_gather8): (4x4 (x,y) column, z node): 8 consecutive targets span a 4x4 footprint
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
                                           keys, ctx->d_flags);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

// ---------------------------------------------------------------------------
constexpr int SP_MAXP = 64;

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
                              double* __restrict__ tab, int zlo_min, unsigned* __restrict__ flags) {
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
    if (k == 0 && lane == 0) {
      const int lz = (int)g_lo(g, 2, p.z);
      lo[s] = make_int4((int)l, (int)g_lo(g, 1, p.y), lz, 0);
      // a window below the first launched z tile (a source at or below the wall of a mirrored
      // half-space plan) would be dropped silently: flag it like a window leaving the grid
      if (lz < zlo_min) atomicOr(flags, FLAG_OUT_OF_GRID);
    }
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
#ifndef SP_STRIP
#define SP_STRIP 2  // tile-order strip width in x (0: plain x-major order)
#endif
constexpr int SW_IDQ = 64;  // consumer id FIFO capacity (>= 3 leftovers + SW_CH hits, power of two)
template <int NCH>
struct SwBuf {
  static constexpr int RQ = NCH | 1;
  static constexpr int DOUBLES = SW_CH * (SW_RX + SW_RY + SW_RZ + RQ + 1);
};

// Window slices come from the per-source window table (k_spread_wtab) by cp.async; computing
// them in the producers instead (the Gaussian ratio recurrence from each source's position)
// removes the table re-reads but measured slower (24.4 vs 18.1 ms at HL):
// the producers' dependent recurrence chains then bound the consumers.
// NCW consumer warps: 8 (warp patch 4x8 (x,y) x 8 z, 2 CTAs/SM) or 16 (patch 4x4 x 8, 1 CTA/SM,
// a 16-deep ring): the smaller patch cuts the y padding of the DMMA work (window rows outside a
// warp's patch) from (24+7)/24 to (24+3)/24, and with all channels in one launch the producers
// stage every source once instead of once per channel group.
template <int NCH, int NCW = 8>
__global__ void __launch_bounds__((NCW + SW_NP) * 32, NCW == 8 ? 2 : 1) k_spread_mma4(const int4* __restrict__ lo4, const double* __restrict__ tab,
                                                       WTab wt, const double4* __restrict__ pts,
                                                       const double* __restrict__ w, int ldw,
                                                       const int* __restrict__ bin_start, GridGeom g, int nbx,
                                                       int nby, int nbz, double* __restrict__ grids, int tz0) {
  constexpr int RX = SW_RX, RY = SW_RY, RZ = SW_RZ, RQ = SwBuf<NCH>::RQ, PER = SwBuf<NCH>::DOUBLES;
  extern __shared__ __align__(16) double sm_dyn[];
  constexpr int K = NCW == 16 ? 16 * 32 / SW_CH : SW_K;  // ring depth (16 slots of 32 sources)
  constexpr int PY = 64 / NCW, RB = PY / 2;  // warp patch rows, row blocks of 8 positions
  constexpr int PB = NCW;                    // mask bit of the window-slice parities
  __shared__ __align__(8) uint64_t full_bar[K], empty_bar[K];
  __shared__ int run_beg[9], run_pre[10];
  __shared__ int s_nrun;
  __shared__ unsigned short s_ids[NCW][SW_IDQ];  // per-warp FIFO of hit ids (consumers)
  auto bx_ = [&](int b) { return reinterpret_cast<double(*)[RX]>(sm_dyn + b * PER); };
  auto by_ = [&](int b) { return reinterpret_cast<double(*)[RY]>(sm_dyn + b * PER + SW_CH * RX); };
  auto bz_ = [&](int b) { return reinterpret_cast<double(*)[RZ]>(sm_dyn + b * PER + SW_CH * (RX + RY)); };
  auto bq_ = [&](int b) { return reinterpret_cast<double(*)[RQ]>(sm_dyn + b * PER + SW_CH * (RX + RY + RZ)); };
  auto bm_ = [&](int b) { return reinterpret_cast<unsigned*>(sm_dyn + b * PER + SW_CH * (RX + RY + RZ + RQ)); };

  // Tile order: strips of SP_STRIP tile columns in x; within a strip y-major, then the strip's x
  // columns, z fastest.  Consecutively launched tiles then share their candidate bins (a source's
  // window rows are re-read by the ~25 tiles its support touches): the live set is 3 y-columns x
  // (SP_STRIP + 2) x-columns of sources, which the L2 holds, instead of whole x-slabs.
  // (only the z tiles tz0 .. nbz - 1 are launched: a mirrored half-space plan never spreads below
  // the wall, and its forward z stage reads those nodes as the zeros they were allocated with)
  int tx, ty, tz;
  const int nzl = nbz - tz0;  // launched z tiles per column
  if (SP_STRIP > 0) {
    const int per_strip = SP_STRIP * nby * nzl;
    const int sidx = blockIdx.x / per_strip, r = blockIdx.x - sidx * per_strip;
    const int kk = min(SP_STRIP, nbx - sidx * SP_STRIP);  // width of this strip
    ty = r / (kk * nzl);
    const int r2 = r - ty * kk * nzl;
    tx = sidx * SP_STRIP + r2 / nzl;
    tz = tz0 + r2 - (r2 / nzl) * nzl;
  } else {
    tz = tz0 + blockIdx.x % nzl;
    ty = (blockIdx.x / nzl) % nby;
    tx = blockIdx.x / (nzl * nby);
  }
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
          f.lo[h] = lo4[row];
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
      // window slices: 16-byte cp.async chunks, completion tracked by the same barrier
#pragma unroll
      for (int h = 0; h < SW_H; ++h) {
        if (m[h]) {
          const int sl = lane + 32 * h;
          const double* src = tab + (int64_t)cur.row[h] * wt.stride;
          const double* sx = src + (ex[h] & ~1);
          const double* sy = src + wt.wx + (ey[h] & ~1);
          const double* sz = src + wt.wx + wt.wy + (ez[h] & ~1);
          // the tile's slices lie inside the source's zero-padded window rows
          HS_CHECK((ex[h] & ~1) >= 0 && (ex[h] & ~1) + RX <= wt.wx && (ey[h] & ~1) >= 0 &&
                   (ey[h] & ~1) + RY <= wt.wy && (ez[h] & ~1) >= 0 && (ez[h] & ~1) + RZ <= wt.wz);
          HS_CHECK(b < K && sl < SW_CH && cur.row[h] >= 0);
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
  // K-slot carry: the m8n8k4 contraction takes 4 sources, and the sources a warp patch meets in
  // one chunk rarely come in multiples of 4.  Every chunk's hits are appended (one ballot, one
  // store per hit lane) to a per-warp FIFO of ring ids (buffer * SW_CH + slot); groups of 4 are
  // taken from its head, so the < 4 leftover ids of a chunk head the first group of the next one
  // (their buffer is released one chunk later) and every group but a tile's last is full --
  // ~15 % fewer DMMAs than a zero-padded group per chunk end, and no serial bit-extraction
  // chain per group.
  unsigned short* ids = s_ids[warp];
  int head = 0, tail = 0;  // warp-uniform
  const unsigned lanes_lt = (1u << lane) - 1u;
  // fragments of one group for this lane: A = wx wy at its row's position (per row block), B = wz q_c
  struct Ops {
    double cxy[RB], bq[NCH];
  };
  // id = ring id | slice parities << 9 (appended by the hit lane, so no mask re-read here)
  auto load_ops = [&](int gid) {
    Ops o;
    double bz = 0.0, q[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) q[ch] = 0.0;
#pragma unroll
    for (int rb = 0; rb < RB; ++rb) o.cxy[rb] = 0.0;
    if (gid >= 0) {
      const int gb = (gid >> 5) & 15, sk = gid & 31;
      const int pxo = (gid >> 9) & 1, pyo = (gid >> 10) & 1, pzo = (gid >> 11) & 1;
      HS_CHECK(gb < K && pzo + rq < RZ && pxo + wx0 + 3 < RX && pyo + wy0 + PY - 1 < RY);
      bz = bz_(gb)[sk][pzo + rq];  // B[k][n] = wz_{s_k}(z_n), n = rq
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) q[ch] = bq_(gb)[sk][ch];
#pragma unroll
      for (int rb = 0; rb < RB; ++rb) {
        const int p = rb * 8 + rq;  // position of A row rq in row block rb
        o.cxy[rb] = bx_(gb)[sk][pxo + wx0 + (p & 3)] * by_(gb)[sk][pyo + wy0 + (p >> 2)];
      }
    }
    // the weight goes into the B operand (wz q_c, one product per channel) so A = wx wy is
    // shared by the channels
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) o.bq[ch] = bz * q[ch];
    return o;
  };
  auto mma = [&](const Ops& o) {
#pragma unroll
    for (int rb = 0; rb < RB; ++rb)
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) dmma_884(acc[rb][ch][0], acc[rb][ch][1], o.cxy[rb], o.bq[ch]);
  };
  static_assert(SW_CH == 32 && K <= 16, "one ballot per chunk; id = 4 buffer bits | 5 slot bits | 3 parity bits");
  for (int c = 0; c < nchunk; ++c) {
    const int b = c % K;
    const int nc = min(SW_CH, ncand - c * SW_CH);
    mbar_wait(&full_bar[b], (c / K) & 1);
    const unsigned mk = lane < nc ? bm_(b)[lane] : 0u;
    const bool hit = (mk >> warp) & 1u;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    const bool had_left = tail > head;  // ids of chunk c - 1
    if (hit)
      ids[(tail + __popc(m & lanes_lt)) & (SW_IDQ - 1)] =
          (unsigned short)(b * SW_CH + lane + (((mk >> PB) & 7u) << 9));
    tail += __popc(m);
    __syncwarp();
    HS_CHECK(tail - head <= 3 + SW_CH);
    if (had_left && tail - head < 4) {
      // too few hits to complete the group: fire it partly filled, so that a leftover never
      // outlives the chunk after its own
      const int gid = head + kq < tail ? ids[(head + kq) & (SW_IDQ - 1)] : -1;
      head = tail;
      mma(load_ops(gid));
    }
    while (tail - head >= 4) {
      const int gid = ids[(head + kq) & (SW_IDQ - 1)];
      head += 4;
      mma(load_ops(gid));
    }
    if (c > 0) mbar_arrive(&empty_bar[(c - 1) % K]);  // the previous chunk's leftovers are consumed
  }
  if (tail > head) mma(load_ops(head + kq < tail ? ids[(head + kq) & (SW_IDQ - 1)] : -1));
  if (nchunk > 0) mbar_arrive(&empty_bar[(nchunk - 1) % K]);
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

hs_status launch_spread(hs_ctx* ctx, const double4* pts, const double* w, int n, int nch, const int* bin_start,
                        const GridGeom& g, double* grids, int ldw, bool reuse_wtab, int tz_begin) {
  if (ldw <= 0) ldw = nch;  // weights row stride (a channel group of wider rows: ldw > nch)
  if (g.P > SP_MAXP) return fail(HS_ERR_PARAMETER, "spread supports window support P <= 64");
  const int nbx = sp_nbins(g, 0), nby = sp_nbins(g, 1), nbz = sp_nbins(g, 2);
  const WTab wt = WTab::make(g.P);
  void* scr = nullptr;
  const size_t nn = (size_t)std::max(n, 1);
  HS_TRY(ctx_scratch(ctx, nn * (sizeof(int4) + sizeof(double) * wt.stride), &scr));
  int4* lo = (int4*)scr;
  double* tab = (double*)(lo + nn);
  if (n > 0 && !reuse_wtab) {  // (reuse: same sources, tables of the previous call intact)
    const int gs = (int)std::min<int64_t>(ceil_div((int64_t)n * 3 * 32, 256), ctx->sm_count * 16);
    k_spread_wtab<<<gs, 256, 0, ctx->stream>>>(pts, n, g, wt, lo, tab,
                                               std::max(0, std::min(tz_begin, nbz - 1)) * SP_TZ, ctx->d_flags);
    HS_LAUNCHED(ctx);
  }
  const int tz0 = std::max(0, std::min(tz_begin, nbz - 1));
  dim3 grid(nbx * nby * (nbz - tz0));
  if (nch >= 3) {
    // 16 consumer warps (4x4 patches), up to 7 channels per launch, groups balanced
    // (7 -> 7, 13 -> 7 + 6, 19 -> 7 + 6 + 6)
    const int ngroup = (nch + 6) / 7;
    for (int gi = 0, c0 = 0; gi < ngroup; ++gi) {
      const int cn = (nch - c0) / (ngroup - gi);
      double* gout = grids + (size_t)c0 * g.ch_stride;
      const double* wc0 = w + c0;
      switch (cn) {
#define HS_SP16(N)                                                                                             \
  case N: {                                                                                                    \
    const size_t smm = sizeof(double) * (16 * 32 / SW_CH) * SwBuf<N>::DOUBLES;                                 \
    HS_CUDA(cudaFuncSetAttribute(k_spread_mma4<N, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smm)); \
    k_spread_mma4<N, 16><<<grid, (16 + SW_NP) * 32, smm, ctx->stream>>>(lo, tab, wt, pts, wc0, ldw, bin_start, g, \
                                                                        nbx, nby, nbz, gout, tz0);            \
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
  // 1 or 2 channels (stand-alone spread API): 8 consumer warps (4x8 patches)
  switch (nch) {
#define HS_SP8(N)                                                                                            \
  case N: {                                                                                                  \
    const size_t smm = sizeof(double) * SW_K * SwBuf<N>::DOUBLES;                                            \
    HS_CUDA(cudaFuncSetAttribute(k_spread_mma4<N, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smm)); \
    k_spread_mma4<N, 8><<<grid, SW_THREADS, smm, ctx->stream>>>(lo, tab, wt, pts, w, ldw, bin_start, g, nbx, nby, \
                                                               nbz, grids, tz0);                             \
  } break;
    HS_SP8(1) HS_SP8(2)
#undef HS_SP8
    default: return fail(HS_ERR_PARAMETER, "spread channel count");
  }
  HS_LAUNCHED(ctx);
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
// Gather (k_gather8).  Targets are sorted by (4x4 (x,y) block, z node) of their window
// centre and cut into RUNS of <= G7_TG targets of one block whose windows start within
// 32 - P z nodes of each other, and ITEMS of <= G7_WARPS runs of one block whose windows start
// within G7_ZC - P nodes (k_g7_count / k_g7_fill).  A CTA takes an item, one warp per run.
// The CTA walks the (x,y) columns of the item's union (a (P+3)^2 square), staging each
// column's z-range (<= G7_ZC nodes, all channels) once through a cp.async ring, G7_STEP columns
// per barrier; each warp contracts the staged columns with its run's window factors on the
// FP64 tensor pipe (see k_gather8).  The x/y factors of a run live in warp-private tables.
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

// runs and items of one 4x4 block's targets [b, e) (z-sorted), by one warp; emit == nullptr: count
// only.  The cut is a sequential scan over the targets' z window starts: a run takes up to G7_TG
// targets whose starts stay within 32 - P nodes of its first, an item up to G7_WARPS runs within
// G7_ZC - P nodes of its first target.  Lanes load 32 window starts at a time; every lane then
// steps the same (warp-uniform) state machine over the shuffled values, lane 0 emits.
__device__ int g7_cut(const double4* __restrict__ pts, int b, int e, const GridGeom& g, int4* emit, int lane) {
  int nitem = 0;
  bool item_open = false, in_run = false;
  int ib = 0, nrun = 0, lens = 0, len = 0;
  int64_t zi0 = 0, zr0 = 0;
  const int run_span = 32 - g.P, item_span = G7_ZC - g.P;
  for (int base = b; base < e; base += 32) {
    const int64_t zl = base + lane < e ? g_lo(g, 2, pts[base + lane].z) : 0;
    const int nk = min(32, e - base);
    for (int k = 0; k < nk; ++k) {
      const int64_t z = __shfl_sync(0xffffffffu, zl, k);
      const int i = base + k;
      if (in_run) {
        if (len < G7_TG && z - zr0 <= run_span && z - zi0 <= item_span) {
          ++len;
          continue;
        }
        lens |= len << (8 * nrun);
        ++nrun;
        in_run = false;
      }
      if (item_open && !(nrun < G7_WARPS && z - zi0 <= item_span)) {
        if (emit && lane == 0) emit[nitem] = make_int4(ib, i - ib, lens, 0);
        ++nitem;
        item_open = false;
      }
      if (!item_open) {
        ib = i;
        nrun = 0;
        lens = 0;
        zi0 = z;
        item_open = true;
      }
      zr0 = z;
      len = 1;
      in_run = true;
    }
  }
  if (in_run) lens |= len << (8 * nrun);
  if (item_open) {
    if (emit && lane == 0) emit[nitem] = make_int4(ib, e - ib, lens, 0);
    ++nitem;
  }
  return nitem;
}

__global__ void k_g7_count(const double4* __restrict__ pts, const int* __restrict__ bstart, int nblk, int nz,
                           GridGeom g, int* __restrict__ cnt) {
  const int lane = threadIdx.x & 31;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nblk; c += (gridDim.x * blockDim.x) >> 5) {
    const int n = g7_cut(pts, bstart[c * nz], bstart[(c + 1) * nz], g, nullptr, lane);
    if (lane == 0) cnt[c] = n;
  }
}

__global__ void k_g7_fill(const double4* __restrict__ pts, const int* __restrict__ bstart, int nblk, int nz,
                          GridGeom g, const int* __restrict__ istart, int4* __restrict__ items) {
  const int lane = threadIdx.x & 31;
  for (int c = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < nblk; c += (gridDim.x * blockDim.x) >> 5)
    g7_cut(pts, bstart[c * nz], bstart[(c + 1) * nz], g, items + istart[c], lane);
}

// Gather on the FP64 tensor pipe (k_gather8).  Items, runs, the column staging ring and the
// x / y window tables as described above; the per-column contraction over z is a DMMA: for a run of <= 8 targets t and its 32-node z window,
//   D[t][n] += A[t][k] B[k][n],   A[t][k] = wz_t(z0 + 4 s + k),   B[k][n] = G_c(col, z0 + 4 s + k)
// with n = (column of the 4-column step, channel of a channel pair), 8 k-steps of 4 nodes; then
// u_t,c += wx_t(col) wy_t(col) D[t][n].  One m8n8k4 DMMA does 256 FMAs where the previous
// DFMA form (lanes = z nodes, E[t][c] += wx wy G in registers) issued 8 targets x 6 channels
// DFMAs per lane per column: ~5x fewer instructions per useful FMA, 93 registers instead of
// 200, 16.5 -> 11.6-11.9 ms at HL (profiles/r02/experiments/bench_gather_*).  (Fragments of mma.m8n8k4.f64: A[lane/4][lane%4],
// B[lane%4][lane/4], C/D[lane/4][2 (lane%4) + {0,1}].)

template <int NCH, int PITCH>
__global__ void __launch_bounds__(G7_WARPS * 32) k_gather8(const double4* __restrict__ pts,
                                                          const int* __restrict__ orig, const int4* __restrict__ items,
                                                          const int* __restrict__ n_items_d, int* __restrict__ work,
                                                          GridGeom g,
                                                          const double* __restrict__ T,
                                                          double* __restrict__ u_four, double* __restrict__ u_tot,
                                                          const double* __restrict__ u_real,
                                                          unsigned* __restrict__ flags) {
  constexpr int TG = G7_TG, GW = G7_GW, NT = G7_WARPS * 32, CPN = PITCH / 2;  // 16-byte chunks per node
  constexpr int NCP = (NCH + 1) / 2;  // channel pairs
  static_assert(G7_STEP == 4, "one DMMA n-block = 4 columns x a channel pair");
  __shared__ double s_w[G7_WARPS][2][TG][GW];
  // (a ring row pitch padded so the 4 columns' B fragments fall in distinct banks measured equal)
  __shared__ __align__(16) double s_ring[G7_R][G7_ZC * PITCH];
  __shared__ int s_u[G7_WARPS][6];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int P = g.P;
  const int ft = lane >> 2, fk = lane & 3;  // fragment row (target) / k index; B: n = ft
  double(*wx_tab)[GW] = s_w[warp][0];
  double(*wy_tab)[GW] = s_w[warp][1];
  const int n_items = *n_items_d;
  // items are drawn from a global counter (no static share per CTA: no tail behind the slowest one)
  __shared__ int s_item;
  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_item = atomicAdd(work, 1);
    __syncthreads();
    const int it = s_item;
    if (it >= n_items) break;
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
    if (C0[0] == 0x7fffffff) continue;  // no active target in the item
    const int nxu = C1[0] - C0[0], nyu = C1[1] - C0[1], nzu = C1[2] - C0[2];
    if (nxu <= 0 || nxu > GW || nyu > GW || nzu > G7_ZC) continue;  // (out-of-grid targets only)
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
    // A fragments: wz of fragment row ft (target ft of the run) at nodes W0z + 4 s + fk
    double a[8];
    {
      const bool tin = (amask >> ft) & 1u;
      const double pz = __shfl_sync(0xffffffffu, pc[2], ft);
      const int lz = __shfl_sync(0xffffffffu, lo[2], ft);
#pragma unroll
      for (int sk = 0; sk < 8; ++sk) {
        const int z = W0[2] + 4 * sk + fk;
        double v = 0.0;
        if (tin && z >= lz && z < lz + P) {
          const double d = g_d(g, 2, pz, z);
          v = exp(-g.alpha * d * d);
        }
        a[sk] = v;
      }
    }
    // B rows: staged node of k-step sk for this lane's k (clamped into the staged range, where
    // every target's A is zero anyway)
    const int zoff = W0[2] - C0[2];
    HS_CHECK(!amask || (zoff >= 0 && zoff < G7_ZC && nzu <= G7_ZC));  // (idle warps skip the steps)
    // k-steps that reach a target's window: the run's z extent W1 - W0 <= 31 (7 steps for 88 %
    // of the runs at HL)
    const int nks = min(8, (W1[2] - W0[2] + 3) >> 2);
    __syncwarp();
    const int ncol = nxu * nyu, nchunk = nzu * CPN;
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
    double acc[2 * NCP];
#pragma unroll
    for (int c = 0; c < 2 * NCP; ++c) acc[c] = 0.0;
    // column index of this lane's D column (fk) in the current step, and of its B column (ft/2)
    int colD = fk;
    // one step of (up to) 4 staged columns from ring slot sl: 8 k-steps x NCP channel pairs
    auto step = [&](int sl, int ncols) {
      const int cb = ft >> 1;                 // B: column of the step
      const bool bval = cb < ncols;
      const double* bcol = s_ring[sl + (bval ? cb : 0)] + (ft & 1);
      // (two accumulator sets for even / odd k-steps measured slower: 12.4 vs 11.9 ms)
      double d[NCP][2];
#pragma unroll
      for (int cp = 0; cp < NCP; ++cp) d[cp][0] = d[cp][1] = 0.0;
#pragma unroll
      for (int sk = 0; sk < 8; ++sk) {
        if (sk < nks) {  // warp-uniform
          const int zi = min(zoff + 4 * sk + fk, nzu - 1);
#pragma unroll
          for (int cp = 0; cp < NCP; ++cp) {
            const double b = bval ? bcol[zi * PITCH + 2 * cp] : 0.0;
            dmma_884(d[cp][0], d[cp][1], a[sk], b);
          }
        }
      }
      // epilogue: D[ft][2 fk + j] belongs to column fk of the step, channels 2 cp + j
      double w = 0.0;
      if (fk < ncols && colD < ncol) {
        const int cx = colD / nyu, cy = colD - cx * nyu;
        HS_CHECK(cx < GW && cy < GW);
        w = wx_tab[ft][cx] * wy_tab[ft][cy];
      }
#pragma unroll
      for (int cp = 0; cp < NCP; ++cp) {
        acc[2 * cp] = fma(w, d[cp][0], acc[2 * cp]);
        acc[2 * cp + 1] = fma(w, d[cp][1], acc[2 * cp + 1]);
      }
      colD += G7_STEP;
    };
    int slot = 0;
    const int nfull = ncol / G7_STEP, nrem = ncol - nfull * G7_STEP;
    for (int sidx = 0; sidx < nfull; ++sidx) {
      cp_async_wait<1>();
      __syncthreads();
      issue_step(sidx + 2);
      if (amask) step(slot, G7_STEP);
      slot = slot + G7_STEP == G7_R ? 0 : slot + G7_STEP;
    }
    if (nrem) {  // ragged last step (already issued)
      cp_async_wait<1>();
      __syncthreads();
      if (amask) step(slot, nrem);
    }
    cp_async_wait<0>();
    // the 4 lanes of a target hold its sums over the columns = fk (mod 4): reduce, then lane
    // tt takes target tt's result from lane 4 tt
    double res[NCH];
#pragma unroll
    for (int c = 0; c < 2 * NCP; ++c) {
      double v = acc[c];
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      const double r = __shfl_sync(0xffffffffu, v, (lane & 7) * 4);
      if (c < NCH) res[c] = r;
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

hs_status launch_gather_fourier(hs_ctx* ctx, const double4* pts, const int* orig, int n, int half, const GridGeom& g,
                                const double* T, double* u_fourier, double* u_total, const double* u_real,
                                const int* bstart) {
  if (n == 0) return HS_OK;
  if (g.P > 32) return fail(HS_ERR_PARAMETER, "window support P > 32 is not supported by the gather");
  // k_gather8: an item's x / y window union is at most P + 3 nodes wide (targets of one 4x4
  // block), which must fit the GW = 32 lanes of its tables; wider supports (P = 30 .. 32) take
  // the warp-per-target gather
  if (g.P + 3 > G7_GW || g.P > G7_ZC) {
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
  if (!bstart) return fail(HS_ERR_PARAMETER, "gather needs the block order");
  // items (worst case one per target): count per 4x4 block, scan, fill
  const int nb4 = ((g.dims[0] + 3) / 4) * ((g.dims[1] + 3) / 4);
  void* scr = nullptr;
  const size_t bytes = sizeof(int4) * (size_t)n + sizeof(int) * (3 * (size_t)nb4 + 8 + 4);
  HS_TRY(ctx_scratch(ctx, bytes, &scr));
  int4* items = (int4*)scr;
  int* cnt = (int*)(items + n);
  int* istart = cnt + nb4;  // nb4 + 1
  int* sc = istart + nb4 + 1;
  int* work = cnt + 3 * (size_t)nb4 + 8;  // work-item counter of the gather kernel
  HS_CUDA(cudaMemsetAsync(work, 0, sizeof(int), ctx->stream));
  const int gsb = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(nb4, 4), ctx->sm_count * 16));  // warp per block
  k_g7_count<<<gsb, 128, 0, ctx->stream>>>(pts, bstart, nb4, g.dims[2], g, cnt);
  HS_LAUNCHED(ctx);
  HS_TRY(exclusive_scan(ctx, cnt, nb4, istart, sc));
  k_g7_fill<<<gsb, 128, 0, ctx->stream>>>(pts, bstart, nb4, g.dims[2], g, istart, items);
  HS_LAUNCHED(ctx);
  int per_sm = 0;
  HS_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, half ? k_gather8<6, 6> : k_gather8<3, 4>,
                                                        G7_WARPS * 32, 0));
  const int gs8 = (int)std::min<int64_t>(n, (int64_t)ctx->sm_count * std::max(per_sm, 1));
  if (half)
    k_gather8<6, 6><<<gs8, G7_WARPS * 32, 0, ctx->stream>>>(pts, orig, items, istart + nb4, work, g, T, u_fourier,
                                                           u_total, u_real, ctx->d_flags);
  else
    k_gather8<3, 4><<<gs8, G7_WARPS * 32, 0, ctx->stream>>>(pts, orig, items, istart + nb4, work, g, T, u_fourier,
                                                           u_total, u_real, ctx->d_flags);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

HS_DEFINE_CHECK_COLLECT(gridding)

}  // namespace hs

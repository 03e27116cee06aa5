// sort.cu -- deterministic stable counting sort of small integer keys on the GPU.
//
// Used for (a) the real-space cell list, bit-exact with the reference's
// `np.argsort(flat, kind="stable")` + `cumsum(bincount)` (ewald_real.py:246-250),
// and (b) binning sources/targets by grid tile for spreading and gathering.
//
// Algorithm: histogram (int atomics) -> exclusive scan -> atomic scatter into
// each key's segment (arbitrary order) -> per-segment rank sort by original
// index.  Since a stable argsort orders equal keys by ascending index, ranking
// every element of a segment by its value reproduces it exactly, independent
// of the scatter order.
#define HS_TU_ID 5  // checked build: source of a failing HS_CHECK
#include "common.cuh"
#include "kernels.cuh"

namespace hs {

__global__ void k_histogram(const int* __restrict__ keys, int n, int nb, int* __restrict__ counts) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    HS_CHECK(keys[i] >= 0 && keys[i] < nb);
    atomicAdd(&counts[keys[i]], 1);
  }
}

// Single-CTA exclusive scan of counts[0..nb) into start[0..nb] (start[nb] = total).
// Also copies start into cursor for the scatter pass and records the largest bin.
__global__ void k_scan(const int* __restrict__ counts, int nb, int* __restrict__ start,
                       int* __restrict__ cursor, int* __restrict__ max_count) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  if (threadIdx.x == 0) carry = 0;
  int local_max = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int base = 0; base < nb; base += blockDim.x) {
    int i = base + threadIdx.x;
    int v = i < nb ? counts[i] : 0;
    local_max = max(local_max, v);
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) warp_sums[warp] = x;
    __syncthreads();
    if (warp == 0) {
      int w = lane < (blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      warp_sums[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    int excl = carry + (warp > 0 ? warp_sums[warp - 1] : 0) + x - v;
    if (i < nb) {
      start[i] = excl;
      cursor[i] = excl;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) start[nb] = carry;
  // block max
  for (int o = 16; o > 0; o >>= 1) local_max = max(local_max, __shfl_xor_sync(0xffffffffu, local_max, o));
  if (lane == 0) atomicMax(max_count, local_max);
}

// Multi-CTA exclusive scan for large key ranges (the gather's (4x4 block, z node) keys reach
// ~1.3 M bins at HL, where the single-CTA scan above took 0.2 ms per sort):
// tile sums -> single-CTA scan of the tile sums -> per-tile rescan with the tile offset.
constexpr int SCAN_T = 1024, SCAN_TILE = 2 * SCAN_T;
__device__ __forceinline__ int block_excl_scan(int v, int* ws, int* total) {
  // exclusive scan of v over the CTA (SCAN_T threads); *total = CTA sum (smem broadcast)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = ws[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    ws[lane] = w;
  }
  __syncthreads();
  const int r = (warp > 0 ? ws[warp - 1] : 0) + x - v;
  *total = ws[31];
  __syncthreads();
  return r;
}
__global__ void __launch_bounds__(SCAN_T) k_scan_tiles(const int* __restrict__ counts, int nb, int* __restrict__ sums,
                                                       int* __restrict__ max_count) {
  __shared__ int ws[32];
  const int i = blockIdx.x * SCAN_TILE + 2 * threadIdx.x;
  const int a = i < nb ? counts[i] : 0, b = i + 1 < nb ? counts[i + 1] : 0;
  int tot;
  block_excl_scan(a + b, ws, &tot);
  if (threadIdx.x == 0) sums[blockIdx.x] = tot;
  int m = max(a, b);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(max_count, m);
}
__global__ void __launch_bounds__(SCAN_T) k_scan_apply(const int* __restrict__ counts, int nb,
                                                       const int* __restrict__ off, int ntile, int* __restrict__ start,
                                                       int* __restrict__ cursor) {
  __shared__ int ws[32];
  const int i = blockIdx.x * SCAN_TILE + 2 * threadIdx.x;
  const int a = i < nb ? counts[i] : 0, b = i + 1 < nb ? counts[i + 1] : 0;
  int tot;
  const int e = off[blockIdx.x] + block_excl_scan(a + b, ws, &tot);
  if (i < nb) start[i] = cursor[i] = e;
  if (i + 1 < nb) start[i + 1] = cursor[i + 1] = e + a;
  if (blockIdx.x == 0 && threadIdx.x == 0) start[nb] = off[ntile];
}

__global__ void k_scatter(const int* __restrict__ keys, int n, int* __restrict__ cursor,
                          int* __restrict__ tmp) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    int p = atomicAdd(&cursor[keys[i]], 1);
    HS_CHECK(p >= 0 && p < n);
    tmp[p] = i;
  }
}

// One warp per segment: rank = #{elements in the segment smaller than me}.
__global__ void k_segment_rank_warp(const int* __restrict__ start, int nb, const int* __restrict__ tmp,
                                    int* __restrict__ order, int limit) {
  const int lane = threadIdx.x & 31;
  const int warps_per_block = blockDim.x >> 5;
  for (int b = blockIdx.x * warps_per_block + (threadIdx.x >> 5); b < nb; b += gridDim.x * warps_per_block) {
    const int s = start[b], len = start[b + 1] - s;
    if (len == 0 || len > limit) continue;
    if (len == 1) {
      if (lane == 0) order[s] = tmp[s];
      continue;
    }
    for (int i = lane; i < len; i += 32) {
      const int e = tmp[s + i];
      int r = 0;
      for (int j = 0; j < len; ++j) r += (__ldg(&tmp[s + j]) < e);
      HS_CHECK(r < len);
      order[s + r] = e;
    }
  }
}

// One CTA per large segment, tiles of the segment staged through shared memory.
__global__ void k_segment_rank_block(const int* __restrict__ start, const int* __restrict__ big_bins,
                                     const int* __restrict__ n_big, const int* __restrict__ tmp,
                                     int* __restrict__ order) {
  __shared__ int tile[1024];
  for (int bi = blockIdx.x; bi < *n_big; bi += gridDim.x) {
  const int b = big_bins[bi];
  const int s = start[b], len = start[b + 1] - s;
  for (int i0 = 0; i0 < len; i0 += blockDim.x) {
    const int i = i0 + threadIdx.x;
    const int e = i < len ? tmp[s + i] : 0x7fffffff;
    int r = 0;
    for (int j0 = 0; j0 < len; j0 += 1024) {
      __syncthreads();
      for (int j = threadIdx.x; j < 1024; j += blockDim.x) tile[j] = (j0 + j < len) ? tmp[s + j0 + j] : 0x7fffffff;
      __syncthreads();
      const int m = min(1024, len - j0);
      for (int j = 0; j < m; ++j) r += (tile[j] < e);
    }
    HS_CHECK(i >= len || r < len);
    if (i < len) order[s + r] = e;
  }
  __syncthreads();
  }
}

__global__ void k_find_big(const int* __restrict__ start, int nb, int limit, int* __restrict__ big_bins,
                           int* __restrict__ n_big) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < nb; b += gridDim.x * blockDim.x)
    if (start[b + 1] - start[b] > limit) big_bins[atomicAdd(n_big, 1)] = b;
}

// keys[n] in [0, nb): writes order[n] (stable argsort) and start[nb+1].
// Scratch: counts/cursor (2*nb+4 ints) + tmp (n ints).
hs_status counting_sort(hs_ctx* ctx, const int* keys, int n, int nb, int* order, int* start, int* work,
                        int nb_rank) {
  // nb_rank < nb: segments >= nb_rank are left unranked (their order entries undefined)
  if (nb_rank < 0 || nb_rank > nb) nb_rank = nb;
  cudaStream_t st = ctx->stream;
  int* counts = work;              // nb
  int* cursor = work + nb;         // nb
  int* maxc = work + 2 * nb;       // 1 (largest segment, diagnostics)
  int* nbig = work + 2 * nb + 1;   // 1
  int* tmp = work + 2 * nb + 4;    // n
  HS_CUDA(cudaMemsetAsync(counts, 0, sizeof(int) * nb, st));
  HS_CUDA(cudaMemsetAsync(maxc, 0, sizeof(int) * 2, st));
  const int gs = (int)std::min<int64_t>(ceil_div(std::max(n, 1), 256), ctx->sm_count * 8);
  if (n > 0) {
    k_histogram<<<gs, 256, 0, st>>>(keys, n, nb, counts);
    HS_LAUNCHED(ctx);
  }
  if (nb <= 4 * SCAN_TILE) {
    k_scan<<<1, 1024, 0, st>>>(counts, nb, start, cursor, maxc);
    HS_LAUNCHED(ctx);
  } else {
    const int ntile = (int)ceil_div(nb, SCAN_TILE);
    int* sums = work + 2 * nb + 4 + n;   // counting_sort_work_ints: + 2 ntile + 8
    int* off = sums + ntile;              // ntile + 1
    int* junk = off + ntile + 1;          // cursor of the tile-sum scan (ntile) and its max
    k_scan_tiles<<<ntile, SCAN_T, 0, st>>>(counts, nb, sums, maxc);
    HS_LAUNCHED(ctx);
    k_scan<<<1, 1024, 0, st>>>(sums, ntile, off, junk, junk + ntile);
    HS_LAUNCHED(ctx);
    k_scan_apply<<<ntile, SCAN_T, 0, st>>>(counts, nb, off, ntile, start, cursor);
    HS_LAUNCHED(ctx);
  }
  if (n == 0) return HS_OK;
  k_scatter<<<gs, 256, 0, st>>>(keys, n, cursor, tmp);
  HS_LAUNCHED(ctx);
  const int kWarpLimit = 2048;
  if (nb_rank == 0) return HS_OK;
  const int wb = (int)std::min<int64_t>(ceil_div(nb_rank, 8), ctx->sm_count * 16);
  k_segment_rank_warp<<<wb, 256, 0, st>>>(start, nb_rank, tmp, order, kWarpLimit);
  HS_LAUNCHED(ctx);
  // segments longer than kWarpLimit (clustered or degenerate cell lists): one CTA each
  int* big = cursor;  // cursor is dead after the scatter
  k_find_big<<<(int)ceil_div(nb_rank, 256), 256, 0, st>>>(start, nb_rank, kWarpLimit, big, nbig);
  HS_LAUNCHED(ctx);
  k_segment_rank_block<<<ctx->sm_count, 1024, 0, st>>>(start, big, nbig, tmp, order);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

hs_status exclusive_scan(hs_ctx* ctx, const int* in, int n, int* out, int* scratch) {
  HS_CUDA(cudaMemsetAsync(scratch + n, 0, sizeof(int), ctx->stream));
  k_scan<<<1, 1024, 0, ctx->stream>>>(in, n, out, scratch, scratch + n);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

HS_DEFINE_CHECK_COLLECT(sort)

}  // namespace hs

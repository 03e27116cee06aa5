// api.cu -- context management and the stand-alone C-ABI entry points
// (cell list, spread, gather, Green's-table precompute, direct sum).
#define HS_TU_ID 8  // checked build: source of a failing HS_CHECK
#include <cufft.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"

namespace hs {

static thread_local std::string t_last_error;

void set_error(const std::string& msg) { t_last_error = msg; }

hs_status fail(hs_status s, const std::string& msg) {
  t_last_error = msg;
  return s;
}

hs_status ctx_scratch(hs_ctx* ctx, size_t bytes, void** out) {
  if (bytes > ctx->scratch_bytes) {
    if (ctx->scratch) {
      HS_CUDA(cudaStreamSynchronize(ctx->stream));
      cudaFree(ctx->scratch);
      ctx->scratch = nullptr;
      ctx->scratch_bytes = 0;
    }
    cudaError_t e = cudaMalloc(&ctx->scratch, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(HS_ERR_RESOURCE, "scratch allocation of " + std::to_string(bytes) + " bytes failed");
    }
    ctx->scratch_bytes = bytes;
  }
  *out = ctx->scratch;
  return HS_OK;
}

hs_status ctx_reset_flags(hs_ctx* ctx) {
  HS_CUDA(cudaMemsetAsync(ctx->d_flags, 0, sizeof(unsigned), ctx->stream));
  return HS_OK;
}

hs_status ctx_check_flags(hs_ctx* ctx, const char* where) {
  HS_CUDA(cudaMemcpyAsync(ctx->h_flags, ctx->d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, ctx->stream));
  HS_CUDA(cudaStreamSynchronize(ctx->stream));
  const unsigned f = *ctx->h_flags;
  if (f & FLAG_GEOMETRY) return fail(HS_ERR_GEOMETRY, std::string(where) + ": points outside the box (cell-list bounds, or a source below the wall)");
  if (f & FLAG_OUT_OF_GRID) return fail(HS_ERR_OUT_OF_GRID, std::string(where) + ": window support leaves the grid");
  if (f & FLAG_SINGULAR) return fail(HS_ERR_SINGULAR, std::string(where) + ": coincident target and source");
  return HS_OK;
}

// device staging helper: returns a device pointer for `bytes` of caller data
struct Staged {
  void* d = nullptr;
  bool owned = false;
  ~Staged() {
    if (owned && d) cudaFree(d);
  }
};

static hs_status stage_in(hs_ctx* ctx, const void* src, size_t bytes, int mem, Staged* s) {
  if (mem == HS_MEM_DEVICE || bytes == 0) {
    s->d = const_cast<void*>(src);
    return HS_OK;
  }
  HS_CUDA(cudaMalloc(&s->d, std::max<size_t>(bytes, 8)));
  s->owned = true;
  HS_CUDA(cudaMemcpyAsync(s->d, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
  return HS_OK;
}

static hs_status alloc_dev(size_t bytes, Staged* s) {
  HS_CUDA(cudaMalloc(&s->d, std::max<size_t>(bytes, 8)));
  s->owned = true;
  return HS_OK;
}

__global__ void k_to_double4(const double* __restrict__ p, int n, double4* __restrict__ out, double w) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    out[i] = make_double4(p[3 * i], p[3 * i + 1], p[3 * i + 2], w);
}

// rows of (points, weights[:, c0:c0+cn]) in sorted order
__global__ void k_permute_rows(const int* __restrict__ ord, int n, const double* __restrict__ p,
                               const double* __restrict__ w, int nch, int c0, int cn, double4* __restrict__ P4,
                               double* __restrict__ W) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    const int i = ord[k];
    P4[k] = make_double4(p[3 * i], p[3 * i + 1], p[3 * i + 2], 0.0);
    for (int c = 0; c < cn; ++c) W[(size_t)k * cn + c] = w[(size_t)i * nch + c0 + c];
  }
}

__global__ void k_i32_to_i64(const int* __restrict__ a, int n, long long* __restrict__ b) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) b[i] = a[i];
}

// channel-first (nch, nx, ny, nz) grids with a compact layout
static GridGeom compact_grid(const double origin[3], double h, const int64_t dims[3], int P, double xi, double eta) {
  GridGeom g{};
  for (int k = 0; k < 3; ++k) {
    g.origin[k] = origin[k];
    g.dims[k] = (int)dims[k];
  }
  g.h = h;
  g.P = P;
  g.alpha = 2.0 * xi * xi / eta;
  g.pref = std::pow(2.0 * xi * xi / (kPi * eta), 1.5);
  g.stride[0] = dims[1] * dims[2];
  g.stride[1] = dims[2];
  g.stride[2] = 1;
  g.ch_stride = dims[0] * dims[1] * dims[2];
  return g;
}

static inline int gsz(hs_ctx* ctx, int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, 256), (int64_t)ctx->sm_count * 8));
}

#define HS_TU_DECL(NAME) void chk_collect_##NAME(unsigned long long*, unsigned long long*, int);
HS_TU_DECL(pair)
HS_TU_DECL(gridding)
HS_TU_DECL(fft)
HS_TU_DECL(plan)
HS_TU_DECL(sort)
HS_TU_DECL(kspace)
HS_TU_DECL(cell_list)
#undef HS_TU_DECL
HS_DEFINE_CHECK_COLLECT(api)

}  // namespace hs

using namespace hs;

extern "C" {

hs_status hs_debug_checks(uint64_t* first_failure, uint64_t* failures, int reset) {
  if (!first_failure || !failures) return fail(HS_ERR_PARAMETER, "null output");
#ifdef HS_CHECKED
  unsigned long long f = 0, c = 0;
  HS_CUDA(cudaDeviceSynchronize());
  chk_collect_pair(&f, &c, reset);
  chk_collect_gridding(&f, &c, reset);
  chk_collect_fft(&f, &c, reset);
  chk_collect_plan(&f, &c, reset);
  chk_collect_sort(&f, &c, reset);
  chk_collect_kspace(&f, &c, reset);
  chk_collect_cell_list(&f, &c, reset);
  chk_collect_api(&f, &c, reset);
  *first_failure = f;
  *failures = c;
  return HS_OK;
#else
  (void)reset;
  *first_failure = 0;
  *failures = 0;
  return fail(HS_ERR_CONFIG, "not a checked build (make -C paper_1802_07844_b200/csrc checked)");
#endif
}

const char* hs_last_error(void) { return t_last_error.c_str(); }

hs_status hs_ctx_create(int device, hs_ctx** out) {
  if (!out) return fail(HS_ERR_PARAMETER, "null output");
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count == 0) {
    cudaGetLastError();
    return fail(HS_ERR_CUDA, "no CUDA device available (this library has no CPU fallback)");
  }
  if (device < 0 || device >= count) return fail(HS_ERR_PARAMETER, "device index out of range");
  HS_CUDA(cudaSetDevice(device));
  cudaDeviceProp prop;
  HS_CUDA(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10) return fail(HS_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100-class");
  hs_ctx* c = new hs_ctx();
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  if (cudaMalloc(&c->d_flags, sizeof(unsigned)) != cudaSuccess ||
      cudaMallocHost(&c->h_flags, sizeof(unsigned)) != cudaSuccess) {
    delete c;
    return fail(HS_ERR_CUDA, "context allocation failed");
  }
  cudaMemset(c->d_flags, 0, sizeof(unsigned));
  *out = c;
  return HS_OK;
}

hs_status hs_ctx_destroy(hs_ctx* ctx) {
  if (!ctx) return HS_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  if (ctx->scratch) cudaFree(ctx->scratch);
  if (ctx->d_flags) cudaFree(ctx->d_flags);
  if (ctx->h_flags) cudaFreeHost(ctx->h_flags);
  delete ctx;
  return HS_OK;
}

hs_status hs_ctx_set_stream(hs_ctx* ctx, void* stream) {
  if (!ctx) return fail(HS_ERR_PARAMETER, "null context");
  ctx->stream = (cudaStream_t)stream;
  return HS_OK;
}

int64_t hs_ctx_launch_count(const hs_ctx* ctx) { return ctx ? ctx->launches : 0; }

hs_status hs_cell_dims(double rc, const double lo[3], const double hi[3], int64_t dims[3], double edge[3]) {
  CellGeom g;
  HS_TRY(cell_geometry(rc, lo, hi, &g));
  for (int k = 0; k < 3; ++k) {
    dims[k] = g.dims[k];
    edge[k] = g.edge[k];
  }
  return HS_OK;
}

hs_status hs_cell_list(hs_ctx* ctx, const double* points, int64_t n, double rc, const double lo[3],
                       const double hi[3], int64_t* order, int64_t* start, int mem) {
  if (!ctx || (n > 0 && (!points || !order)) || !start) return fail(HS_ERR_PARAMETER, "null argument");
  if (n > (1 << 30)) return fail(HS_ERR_PARAMETER, "too many points");
  HS_CUDA(cudaSetDevice(ctx->device));
  CellGeom g;
  HS_TRY(cell_geometry(rc, lo, hi, &g));
  const int ni = (int)n, nb = (int)g.ncell();
  Staged pts, keys, ord, st, work, o64, s64;
  HS_TRY(stage_in(ctx, points, 24 * (size_t)n, mem, &pts));
  HS_TRY(alloc_dev(4 * (size_t)n, &keys));
  HS_TRY(alloc_dev(4 * (size_t)n, &ord));
  HS_TRY(alloc_dev(4 * ((size_t)nb + 1), &st));
  HS_TRY(alloc_dev(4 * counting_sort_work_ints(ni, nb), &work));
  HS_TRY(ctx_reset_flags(ctx));
  HS_TRY(launch_cell_keys(ctx, (const double*)pts.d, ni, ni, 0, g, 1, (int*)keys.d));
  HS_TRY(counting_sort(ctx, (const int*)keys.d, ni, nb, (int*)ord.d, (int*)st.d, (int*)work.d));
  long long* d_order = (long long*)order;
  long long* d_start = (long long*)start;
  if (mem == HS_MEM_HOST) {
    HS_TRY(alloc_dev(8 * (size_t)std::max(n, (int64_t)1), &o64));
    HS_TRY(alloc_dev(8 * ((size_t)nb + 1), &s64));
    d_order = (long long*)o64.d;
    d_start = (long long*)s64.d;
  }
  if (ni > 0) {
    k_i32_to_i64<<<gsz(ctx, ni), 256, 0, ctx->stream>>>((const int*)ord.d, ni, d_order);
    HS_LAUNCHED(ctx);
  }
  k_i32_to_i64<<<gsz(ctx, nb + 1), 256, 0, ctx->stream>>>((const int*)st.d, nb + 1, d_start);
  HS_LAUNCHED(ctx);
  if (mem == HS_MEM_HOST) {
    if (ni > 0) HS_CUDA(cudaMemcpyAsync(order, d_order, 8 * (size_t)n, cudaMemcpyDeviceToHost, ctx->stream));
    HS_CUDA(cudaMemcpyAsync(start, d_start, 8 * ((size_t)nb + 1), cudaMemcpyDeviceToHost, ctx->stream));
  }
  return ctx_check_flags(ctx, "build_cell_list");
}

hs_status hs_spread(hs_ctx* ctx, const double* points, const double* weights, int64_t n, int nch,
                    const double origin[3], double h, const int64_t dims[3], int P, double xi, double eta,
                    double* grids, int mem) {
  if (!ctx || !grids || (n > 0 && (!points || !weights))) return fail(HS_ERR_PARAMETER, "null argument");
  if (nch < 1) return fail(HS_ERR_PARAMETER, "need at least one channel");
  if (P > std::min(dims[0], std::min(dims[1], dims[2])))
    return fail(HS_ERR_PARAMETER, "window support exceeds grid extent");
  HS_CUDA(cudaSetDevice(ctx->device));
  GridGeom g = compact_grid(origin, h, dims, P, xi, eta);
  const int ni = (int)n;
  const int nb = sp_nbins(g, 0) * sp_nbins(g, 1) * sp_nbins(g, 2);
  const size_t gbytes = 8 * (size_t)nch * g.ch_stride;
  Staged pts, w, keys, ord, st, work, P4, W, out;
  HS_TRY(stage_in(ctx, points, 24 * (size_t)n, mem, &pts));
  HS_TRY(stage_in(ctx, weights, 8 * (size_t)n * nch, mem, &w));
  HS_TRY(alloc_dev(4 * (size_t)n, &keys));
  HS_TRY(alloc_dev(4 * (size_t)n, &ord));
  HS_TRY(alloc_dev(4 * ((size_t)nb + 1), &st));
  HS_TRY(alloc_dev(4 * counting_sort_work_ints(ni, nb), &work));
  HS_TRY(alloc_dev(32 * (size_t)n, &P4));
  HS_TRY(alloc_dev(8 * (size_t)n * nch, &W));
  double* d_grids = grids;
  if (mem == HS_MEM_HOST) {
    HS_TRY(alloc_dev(gbytes, &out));
    d_grids = (double*)out.d;
  }
  HS_TRY(ctx_reset_flags(ctx));
  HS_TRY(launch_grid_keys(ctx, (const double*)pts.d, ni, ni, 0, g, (int*)keys.d));
  HS_TRY(counting_sort(ctx, (const int*)keys.d, ni, nb, (int*)ord.d, (int*)st.d, (int*)work.d));
  // permute points/weights into bin order (channel groups of <= 8 per launch)
  for (int c0 = 0; c0 < nch; c0 += 8) {
    const int cn = std::min(8, nch - c0);
    if (ni > 0) {
      k_permute_rows<<<gsz(ctx, ni), 256, 0, ctx->stream>>>((const int*)ord.d, ni, (const double*)pts.d,
                                                            (const double*)w.d, nch, c0, cn, (double4*)P4.d,
                                                            (double*)W.d);
      HS_LAUNCHED(ctx);
    }
    HS_TRY(launch_spread(ctx, (const double4*)P4.d, (const double*)W.d, ni, cn, (const int*)st.d, g,
                         d_grids + (size_t)c0 * g.ch_stride));
  }
  if (mem == HS_MEM_HOST) HS_CUDA(cudaMemcpyAsync(grids, d_grids, gbytes, cudaMemcpyDeviceToHost, ctx->stream));
  return ctx_check_flags(ctx, "spread");
}

hs_status hs_gather(hs_ctx* ctx, const double* grids, int nch, const double* points, int64_t n,
                    const double origin[3], double h, const int64_t dims[3], int P, double xi, double eta,
                    double* out, int mem) {
  if (!ctx || !grids || (n > 0 && (!points || !out))) return fail(HS_ERR_PARAMETER, "null argument");
  HS_CUDA(cudaSetDevice(ctx->device));
  GridGeom g = compact_grid(origin, h, dims, P, xi, eta);
  const int ni = (int)n;
  Staged gr, pts, P4, o;
  HS_TRY(stage_in(ctx, grids, 8 * (size_t)nch * g.ch_stride, mem, &gr));
  HS_TRY(stage_in(ctx, points, 24 * (size_t)n, mem, &pts));
  HS_TRY(alloc_dev(32 * (size_t)n, &P4));
  double* d_out = out;
  if (mem == HS_MEM_HOST) {
    HS_TRY(alloc_dev(8 * (size_t)n * nch, &o));
    d_out = (double*)o.d;
  }
  HS_TRY(ctx_reset_flags(ctx));
  if (ni > 0) {
    k_to_double4<<<gsz(ctx, ni), 256, 0, ctx->stream>>>((const double*)pts.d, ni, (double4*)P4.d, 0.0);
    HS_LAUNCHED(ctx);
  }
  for (int c0 = 0; c0 < nch; c0 += 8) {
    const int cn = std::min(8, nch - c0);
    // out columns c0.. of a (n, nch) row-major array: ldo = nch
    HS_TRY(launch_gather(ctx, (const double4*)P4.d, nullptr, ni, cn, g, (const double*)gr.d + (size_t)c0 * g.ch_stride,
                         d_out + c0, nch, 1.0));
  }
  if (mem == HS_MEM_HOST && ni > 0)
    HS_CUDA(cudaMemcpyAsync(out, d_out, 8 * (size_t)n * nch, cudaMemcpyDeviceToHost, ctx->stream));
  return ctx_check_flags(ctx, "gather");
}

hs_status hs_precompute_greens(hs_ctx* ctx, int kind, double R, double h, const int64_t big[3],
                               const int64_t dims[3], const int64_t guards[3], double* samples, int mem) {
  if (!ctx || !samples) return fail(HS_ERR_PARAMETER, "null argument");
  HS_CUDA(cudaSetDevice(ctx->device));
  int64_t pd[3];
  for (int k = 0; k < 3; ++k) pd[k] = 2 * (dims[k] + guards[k]);
  const size_t nhalf = (size_t)pd[0] * pd[1] * (pd[2] / 2 + 1), nfull = (size_t)pd[0] * pd[1] * pd[2];
  Staged half, full, cs;
  HS_TRY(alloc_dev(8 * nhalf, &half));
  HS_TRY(hs::greens_half_table(ctx, kind, R, h, big, dims, guards, pd, (double*)half.d));
  // expand: the table is real and even, so the half spectrum determines it
  HS_TRY(alloc_dev(16 * nhalf, &cs));  // (re, unused) pairs for the expansion kernel
  double* d_full = samples;
  if (mem == HS_MEM_HOST) {
    HS_TRY(alloc_dev(8 * nfull, &full));
    d_full = (double*)full.d;
  }
  HS_CUDA(cudaMemcpy2DAsync(cs.d, 16, half.d, 8, 8, nhalf, cudaMemcpyDeviceToDevice, ctx->stream));
  HS_TRY(launch_expand_half(ctx, (const double2*)cs.d, pd, d_full));
  if (mem == HS_MEM_HOST) HS_CUDA(cudaMemcpyAsync(samples, d_full, 8 * nfull, cudaMemcpyDeviceToHost, ctx->stream));
  HS_CUDA(cudaStreamSynchronize(ctx->stream));
  return HS_OK;
}

hs_status hs_direct_sum(hs_ctx* ctx, int kind, int geometry, int64_t n, const double* positions, const double* sa,
                        const double* sb, int64_t n_targets, const double* targets, const int64_t* tcols,
                        double* u, int mem) {
  if (!ctx || !positions || !sa || !u) return fail(HS_ERR_PARAMETER, "null argument");
  if (kind != HS_STOKESLET && !sb) return fail(HS_ERR_PARAMETER, "stresslet/rotlet need q");
  HS_CUDA(cudaSetDevice(ctx->device));
  const int ni = (int)n, nt = (int)n_targets;
  const int half = geometry == HS_HALF;
  const int n_src = half ? 2 * ni : ni;
  Staged pos, a, b, tg, tc, order, P, A, B, TP, torig, uo;
  HS_TRY(stage_in(ctx, positions, 24 * (size_t)n, mem, &pos));
  HS_TRY(stage_in(ctx, sa, 24 * (size_t)n, mem, &a));
  if (kind != HS_STOKESLET) HS_TRY(stage_in(ctx, sb, 24 * (size_t)n, mem, &b));
  HS_TRY(stage_in(ctx, targets, 24 * (size_t)nt, mem, &tg));
  if (tcols) HS_TRY(stage_in(ctx, tcols, 8 * (size_t)nt, mem, &tc));
  HS_TRY(alloc_dev(4 * (size_t)n_src, &order));
  HS_TRY(alloc_dev(32 * (size_t)n_src, &P));
  HS_TRY(alloc_dev(32 * (size_t)n_src, &A));
  HS_TRY(alloc_dev(32 * (size_t)n_src, &B));
  HS_TRY(alloc_dev(32 * (size_t)nt, &TP));
  HS_TRY(alloc_dev(4 * (size_t)nt, &torig));
  double* d_u = u;
  if (mem == HS_MEM_HOST) {
    HS_TRY(alloc_dev(24 * (size_t)nt, &uo));
    d_u = (double*)uo.d;
  }
  {
    std::vector<int> iota(n_src);
    for (int i = 0; i < n_src; ++i) iota[i] = i;
    HS_CUDA(cudaMemcpyAsync(order.d, iota.data(), 4 * (size_t)n_src, cudaMemcpyHostToDevice, ctx->stream));
    HS_CUDA(cudaStreamSynchronize(ctx->stream));
  }
  HS_TRY(ctx_reset_flags(ctx));
  HS_TRY(build_pair_records(ctx, kind, half, (const int*)order.d, n_src, ni, (const double*)pos.d,
                            (const double*)a.d, (const double*)b.d, (double4*)P.d, (double4*)A.d, (double4*)B.d));
  HS_TRY(build_target_records(ctx, nullptr, nt, (const double*)tg.d, (const long long*)tc.d, 0, (double4*)TP.d,
                              (int*)torig.d));
  HS_TRY(launch_direct(ctx, kind, half, ni, n_src, (const double4*)P.d, (const double4*)A.d, (const double4*)B.d, nt,
                       (const double4*)TP.d, d_u));
  if (mem == HS_MEM_HOST && nt > 0)
    HS_CUDA(cudaMemcpyAsync(u, d_u, 24 * (size_t)nt, cudaMemcpyDeviceToHost, ctx->stream));
  return ctx_check_flags(ctx, "direct_sum");
}

}  // extern "C"

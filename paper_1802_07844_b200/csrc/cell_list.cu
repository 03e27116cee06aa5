// cell_list.cu -- bit-exact real-space cell list (reference: ewald_real.py:192-251).
//
// The flat cell id of every point is computed with the reference's exact
// IEEE-754 operation sequence (subtract, divide, truncate toward zero, clip,
// (cx*ny + cy)*nz + cz) using explicitly rounded intrinsics so that no FMA
// contraction can move a point across a cell face; the stable argsort is the
// deterministic counting sort in sort.cu.
#define HS_TU_ID 7  // checked build: source of a failing HS_CHECK
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace hs {

hs_status cell_geometry(double rc, const double lo[3], const double hi[3], CellGeom* g) {
  if (!(rc > 0)) return fail(HS_ERR_PARAMETER, "build_cell_list requires rc > 0");
  for (int k = 0; k < 3; ++k) {
    g->lo[k] = lo[k];
    g->hi[k] = hi[k];
    double extent = hi[k] - lo[k];
    double q = extent / rc;                       // (extent / rc).astype(int64)
    int64_t d = (int64_t)q;
    if (d < 1) d = 1;                             // np.maximum(1, ...)
    g->dims[k] = d;
    g->edge[k] = extent / (double)d;              // extent / dims
  }
  if (g->ncell() > (int64_t)1 << 30) return fail(HS_ERR_RESOURCE, "cell list too fine (more than 2^30 cells)");
  return HS_OK;
}

struct KeyGeom {
  double lo[3], lo_m[3], hi_p[3], edge[3];
  int64_t dims[3];
};

__global__ void k_cell_keys(const double* __restrict__ pos, int n_src, int n_total, int mirror, KeyGeom g,
                            int check_bounds, int* __restrict__ keys, unsigned* __restrict__ flags, int sub) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_total; i += gridDim.x * blockDim.x) {
    const int s = i < n_src ? i : i - n_src;
    double p[3] = {pos[3 * s], pos[3 * s + 1], pos[3 * s + 2]};
    if (mirror && i >= n_src) p[2] = -p[2];  // y * MIRROR (system.py:168-169)
    int64_t c[3];
    double vz = 0.0;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      bad |= (p[k] < g.lo_m[k]) || (p[k] > g.hi_p[k]);
      double v = __ddiv_rn(__dsub_rn(p[k], g.lo[k]), g.edge[k]);
      int64_t ci = (int64_t)v;  // astype(int64) truncates toward zero
      ci = ci < 0 ? 0 : ci;
      ci = ci > g.dims[k] - 1 ? g.dims[k] - 1 : ci;
      c[k] = ci;
      if (k == 2) vz = v;
    }
    if (check_bounds && bad) atomicOr(flags, FLAG_GEOMETRY);
    const int flat = (int)((c[0] * g.dims[1] + c[1]) * g.dims[2] + c[2]);
    if (sub > 1) {
      int sl = (int)((vz - (double)c[2]) * sub);
      sl = sl < 0 ? 0 : (sl > sub - 1 ? sub - 1 : sl);
      keys[i] = flat * sub + sl;
    } else {
      keys[i] = flat;
    }
  }
}

hs_status launch_cell_keys(hs_ctx* ctx, const double* pos, int n_src, int n_total, int mirror,
                           const CellGeom& cg, int check_bounds, int* keys, int sub) {
  KeyGeom g;
  for (int k = 0; k < 3; ++k) {
    g.lo[k] = cg.lo[k];
    g.lo_m[k] = cg.lo[k] - 1e-12;  // np.any(points < lo - 1e-12)
    g.hi_p[k] = cg.hi[k] + 1e-12;
    g.edge[k] = cg.edge[k];
    g.dims[k] = cg.dims[k];
  }
  if (n_total == 0) return HS_OK;
  int gs = (int)std::min<int64_t>(ceil_div(n_total, 256), ctx->sm_count * 8);
  k_cell_keys<<<gs, 256, 0, ctx->stream>>>(pos, n_src, n_total, mirror, g, check_bounds, keys, ctx->d_flags,
                                           sub);
  HS_LAUNCHED(ctx);
  return HS_OK;
}

HS_DEFINE_CHECK_COLLECT(cell_list)

}  // namespace hs

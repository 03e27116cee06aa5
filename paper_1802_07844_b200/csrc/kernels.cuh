// kernels.cuh -- internal launcher interfaces shared by the .cu translation units.
#pragma once
#include "common.cuh"

namespace hs {

// sort.cu
hs_status counting_sort(hs_ctx* ctx, const int* keys, int n, int nb, int* order, int* start, int* work,
                        int nb_rank = -1);
inline size_t counting_sort_work_ints(int n, int nb) {
  return (size_t)2 * nb + 4 + (size_t)n + 3 * (size_t)ceil_div(nb, 2048) + 8;  // + multi-CTA scan scratch
}
// exclusive scan of in[0..n) into out[0..n] (out[n] = total); scratch: n + 2 ints
hs_status exclusive_scan(hs_ctx* ctx, const int* in, int n, int* out, int* scratch);

// ---------------------------------------------------------------------------
// cell lists (cell_list.cu)
struct CellGeom {
  double lo[3], hi[3], edge[3];
  int64_t dims[3];
  int64_t ncell() const { return dims[0] * dims[1] * dims[2]; }
};
// dims/edge exactly as numpy computes them (ewald_real.py:241-243)
hs_status cell_geometry(double rc, const double lo[3], const double hi[3], CellGeom* g);
// keys for n_total points: point i < n_src is pos[i]; i >= n_src is pos[i-n_src]
// mirrored through z=0 when `mirror` (ImageSystem.combined_positions, system.py:164-191).
// sub > 1: key = flat * sub + z sub-slab (ordering only; the cell itself is reference-exact)
hs_status launch_cell_keys(hs_ctx* ctx, const double* pos, int n_src, int n_total, int mirror,
                           const CellGeom& g, int check_bounds, int* keys, int sub = 1);

// ---------------------------------------------------------------------------
// spreading / gathering (gridding.cu)
struct GridGeom {
  double origin[3];
  double h, alpha, pref;   // alpha = 2 xi^2/eta, pref = (2 xi^2/(pi eta))^{3/2}
  int dims[3];             // nx, ny, nz (region holding data)
  int P;
  int64_t stride[3];       // element strides of the storage layout (x, y, z)
  int64_t ch_stride;       // element stride between channels
  // y-slab decomposition (sharding.py): stored node (i,j,k) is global node (i, j + yoff, k);
  // window starts are computed from the GLOBAL geometry (bit-identical on every rank) and
  // shifted.  sel: spreading keeps only points whose local y window start is in [sel_lo, sel_hi)
  int yoff;
  int sel, sel_lo, sel_hi;
};
// window start / node distance in the grid's local node numbering (yoff = 0: _gridding.py:24-29);
// only y is ever offset, so x / z (k a compile-time constant at every call) cost nothing extra
__device__ __forceinline__ int64_t g_lo(const GridGeom& g, int k, double pos) {
  const int64_t l = window_lo(pos, g.origin[k], g.h, g.P);
  return k == 1 ? l - g.yoff : l;
}
__device__ __forceinline__ double g_d(const GridGeom& g, int k, double pos, int64_t local_idx) {
  return window_d(pos, g.origin[k], g.h, k == 1 ? local_idx + g.yoff : local_idx);
}
constexpr int SP_TX = 16, SP_TY = 16, SP_TZ = 8;  // spread tile / bin shape
// gather target order: (4x4 (x,y) column, z node) of the window-centre node
inline int gather_keys(const GridGeom& g) {
  return ((g.dims[0] + 3) / 4) * ((g.dims[1] + 3) / 4) * g.dims[2];
}
inline int sp_nbins(const GridGeom& g, int k) {
  const int t[3] = {SP_TX, SP_TY, SP_TZ};
  return (int)ceil_div(g.dims[k], t[k]);
}
// Bin keys of spreading/gathering points by the grid tile holding their window
// centre cell; flags FLAG_OUT_OF_GRID if a window leaves the grid (_gridding.py:50-52).
// point i of a set: mode 0 -> pos[i]; mode 1 -> combined [y; y^I] (n_total = 2 n_src);
// mode 2 -> images y^I only (n_total = n_src).
hs_status launch_grid_keys(hs_ctx* ctx, const double* pos, int n_src, int n_total, int mode, const GridGeom& g,
                           int* keys);
// sorted spread: pts/weights already in bin order; bin_start[nbins+1]
hs_status launch_spread(hs_ctx* ctx, const double4* pts, const double* w, int n, int nch,
                        const int* bin_start, const GridGeom& g, double* grids, int ldw = 0,
                        bool reuse_wtab = false, int tz_begin = 0);  // tz_begin: first z tile launched
// gather: nch channels (<= 8) at n points (any order); out[i*ldo + ch] (times h^3 * scale)
hs_status launch_gather(hs_ctx* ctx, const double4* pts, const int* perm, int n, int nch,
                        const GridGeom& g, const double* grids, double* out, int ldo, double scale);
// half-space Fourier gather: u[orig] (+)= h^3 (T1 . w - x3 T2 . w) (ewald_fourier.py:626-630)
// bstart: start of every gather-order key (the (4x4 block, z node) sort of the targets)
hs_status launch_gather_fourier(hs_ctx* ctx, const double4* pts, const int* orig, int n, int half,
                                const GridGeom& g, const double* T, double* u_fourier, double* u_total,
                                const double* u_real, const int* bstart);

// ---------------------------------------------------------------------------
// real space (pair.cu)
struct PairArgs {
  const double4* P;   // cell-sorted combined sources: x, y, z, original combined index
  const double4* A;   // strength a: f (stokeslet), g (stresslet), sign*(g x q) (rotlet)
  const double4* B;   // strength b: q (stresslet), image wall channel v1,v2 (rotlet), g (mixed)
  const double4* C;   // mixed only: q
  const int* start;   // src cell start, ncell+1
  const double4* TP;  // cell-sorted targets: x, y, z, tcol
  const int* torig;   // output row of each sorted target
  const int* t_start; // target (cell, z sub-slab) start, ncell*t_sub+1
  int t_sub;          // z sub-slabs per cell in the target order
  const int2* items;  // work items (cell column, first sorted target)
  int max_items;      // launch bound (>= actual count)
  const int* n_items_d;  // actual count (device)
  int dims[3];
  double cz_lo, cz_edge;  // z cell geometry: cz = clamp(trunc((z - cz_lo)/cz_edge))
  __device__ __forceinline__ int cell_z(double z) const {
    long long c = (long long)__ddiv_rn(__dsub_rn(z, cz_lo), cz_edge);
    c = c < 0 ? 0 : c;
    return (int)(c > dims[2] - 1 ? dims[2] - 1 : c);
  }
  double xi, rc2;
  float rc2_hi;       // FP32 prefilter bound: (rc (1+1e-4) + 2^-20 box)^2, conservative
  float rc2_lo;       // FP32 sure-accept bound: (rc (1-1e-4) - 2^-20 box)^2 (0 if negative)
  int n_real;         // combined index >= n_real -> image
  int kind;
  const double* self_f;  // stokeslet self term strengths (original f) or null
  double* u;          // (nt,3) real-space velocity (normalised)
  double* uk;         // optional (nt,3) kernel part
  double* uc;         // optional (nt,3) correction part
  unsigned* flags;
  unsigned long long* counts;  // [accepted pairs, accepted image pairs] (optional)
  int* work;          // zeroed work-item counter: CTAs take items dynamically (null: static round robin)
  // neighbour audit (hs_plan_pair_audit; null in production launches): per original target
  // [accepted pairs, accepted image pairs, sum of splitmix64(combined source id) mod 2^64]
  unsigned long long* audit;
};
hs_status launch_pair(hs_ctx* ctx, const PairArgs& a);
hs_status build_pair_items(hs_ctx* ctx, const int* t_start, int ncol, int nz, int* work, int2* items,
                           const int** n_items_d);
hs_status launch_direct(hs_ctx* ctx, int kind, int half, int n_real, int n_src, const double4* P,
                        const double4* A, const double4* B, int nt, const double4* TP, double* u);

// ---------------------------------------------------------------------------
// k-space (kspace.cu)
struct KGeom {
  int p[3];          // padded dims
  int nzh;           // p[2]/2 + 1 (half spectrum)
  double kscale[3];  // 1/(p_i h) (numpy fftfreq spacing)
  double a, b;       // (1-eta)/4xi^2, 1/4xi^2
  double inv_n;      // 1/(px py pz) (scipy ifftn normalisation)
};
// channel layout per kind (see plan.cu); spectra: (nch, px, py, nzh) complex
hs_status launch_kscale(hs_ctx* ctx, int kind, int half, const KGeom& k, const double* tabB,
                        const double* tabH, double2* spec, int64_t ch_stride);
// Green's table precompute (ewald_fourier.py:154-174,207-244)
hs_status launch_greens_hat(hs_ctx* ctx, int kind, double R, double h, const int64_t big[3],
                            double2* out);
// separable table precompute pieces (kspace.cu)
hs_status launch_hat_lines(hs_ctx* ctx, int kind, double R, double h, const int64_t big[3], int64_t l0, int64_t nl,
                           int64_t h1, int64_t h2, int64_t ltot, double2* out);
hs_status launch_sep_scatter(hs_ctx* ctx, const double* src, int64_t l0, int64_t nl, int64_t ltot, int64_t n,
                             int64_t kp, int64_t na, int64_t nb, double scale, double2* dst, double* dst_real);
hs_status launch_sep_crop(hs_ctx* ctx, const double* F, const int64_t k[3], double* crop);
hs_status launch_crop(hs_ctx* ctx, const double* field, const int64_t big[3], const int64_t keep[3], double scale,
                      double* crop);
hs_status launch_real_part(hs_ctx* ctx, const double2* spec, int64_t n, double* out);
hs_status launch_expand_half(hs_ctx* ctx, const double2* half_spec, const int64_t p[3], double* full);
hs_status launch_take_half(hs_ctx* ctx, const double* full, const int64_t p[3], double* half);

// ---------------------------------------------------------------------------
// fused x-stage of the pruned FFT pipeline (fft.cu)
struct FftPlan {
  static constexpr int kMaxPass = 12;
  int n, npass;
  int radix[kMaxPass];
};
struct XArgs {
  double2* B;            // channel-major spectra, each [ky < py][x < nx][kz < nzh]
  double2* Bout;         // output channels (same layout; B for the in-place pass)
  int accum;             // 1: outputs are added to Bout (a second channel group's pass)
  int64_t ch_stride;     // complex elements between channels
  const double* tabB;    // biharmonic table, x-stage layout [ky][kz][kx] (or null)
  const double* tabH;    // harmonic table, same layout (or null)
  const double2* tw;     // px twiddles exp(-2 pi i j/px)
  FftPlan plan;          // radix plan of px
  int px, py, pz, nzh, nx;
  int kz0;               // global kz of local column 0 (y-slab plans own kz columns [kz0, kz0 + nzh))
  double kscale[3];      // 1/(p_i h)
  double ka, kb;         // (1-eta)/4xi^2, 1/4xi^2
  double inv_n;          // 1/(px py pz)
};
hs_status make_fft_plan(int n, FftPlan* pl);
hs_status make_twiddles(int n, double2* d_tw, cudaStream_t st);
hs_status launch_xfused(hs_ctx* ctx, int kind, int half, const XArgs& a);
// y stage with the register FFT (py = 480 or 352): forward reads rows y < ny, writes all py rows;
// inverse reads all py rows, writes rows y < ny (in place allowed)
bool ystage_supported(int py);
hs_status launch_ystage(hs_ctx* ctx, bool fwd, const double2* in, double2* out, const double2* tw, int py, int nx,
                        int nzh, int ny);
// register z stage (pz = 924 or 660): forward replaces the cuFFT D2Z, inverse the cuFFT Z2D + channel interleave
bool zstage_supported(int pz, int nz);
int zstage_twiddle_count(int pz);
hs_status make_zstage_twiddles(int pz, double2* d_tw, cudaStream_t st);
hs_status launch_zfwd(hs_ctx* ctx, int pz, const double* in, double2* out, const double2* tw, int64_t nlines, int nz,
                      int mirror = 0, double msign = 1.0, int zero_below = 0);
hs_status launch_zinv_interleaved(hs_ctx* ctx, int pz, const double2* spec, int64_t ch_stride, int n_out, int pitch,
                                  double* gout, const double2* tw, int64_t nlines, int nz);
// kz columns [kz0, kz0 + nzl) only (a y-slab plan's share; full table: kz0 = 0, nzl = nzh)
hs_status launch_table_to_xmajor(hs_ctx* ctx, const double* in, int px, int py, int nzh, double* out, int kz0 = 0,
                                 int nzl = -1);

// plan.cu helpers reused by the stand-alone API
hs_status greens_half_table(hs_ctx* ctx, int kind, double R, double h, const int64_t big[3], const int64_t dims[3],
                            const int64_t guards[3], const int64_t pd[3], double* half_out,
                            void* scratch = nullptr, size_t scratch_bytes = 0);
hs_status build_pair_records(hs_ctx* ctx, int kind, int half, const int* order, int n_comb, int n, const double* pos,
                             const double* sa, const double* sb, double4* P, double4* A, double4* B);
hs_status build_target_records(hs_ctx* ctx, const int* order, int nt, const double* tpos, const long long* tcols,
                               int tcol_identity, double4* TP, int* torig);

}  // namespace hs

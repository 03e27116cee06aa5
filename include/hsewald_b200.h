/*
 * hsewald_b200.h -- C ABI of the B200-native half-space Spectral-Ewald hot path.
 *
 * Drop-in boundary for the reference package `hsewald` (arXiv:1802.07844,
 * /root/reference/pkg/src/hsewald).  The reference has no FFI of its own: its
 * evaluation entry points are plain Python functions over NumPy float64 /
 * int64 arrays.  Each entry point below replaces one of them (file:line cited)
 * and keeps its argument meaning and error behaviour; the Python package
 * `paper_1802_07844_b200` binds these with ctypes (INTEGRATION.md shows the
 * binding a maintainer of the reference would add).
 *
 * Conventions
 *   - All arrays are float64 / int64, C-contiguous, row-major, exactly the
 *     shapes the reference uses ((n,3) points, (n,nch) weights, channel-first
 *     grids (nch,nx,ny,nz), ...).
 *   - `mem` selects where the caller's array pointers live: HS_MEM_DEVICE
 *     (cudaMalloc'ed / torch CUDA tensors on the context's device) or
 *     HS_MEM_HOST (pageable or pinned host memory; the library stages the
 *     copies on the context's stream and returns after they complete).
 *   - Every call returns an hs_status.  Non-zero statuses map one-to-one onto
 *     the reference's exception classes (errors.py:4-29); hs_last_error()
 *     returns a message for the calling thread's last failure.
 *   - A context is bound to one device and one CUDA stream; calls on one
 *     context are stream-ordered and must not be issued concurrently from
 *     several host threads.  No CPU fallback exists: with no usable device,
 *     hs_ctx_create fails with HS_ERR_CUDA.
 */
#ifndef HSEWALD_B200_H
#define HSEWALD_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HS_OK = 0,
  HS_ERR_SINGULAR = 1,        /* SingularityError  (ewald_real.py:298-299,440-441) */
  HS_ERR_OUT_OF_GRID = 2,     /* GeometryError: window leaves grid (_gridding.py:50-52) */
  HS_ERR_CONFIG = 3,          /* ConfigError: grid/table mismatch (ewald_fourier.py:493-503) */
  HS_ERR_RESOURCE = 4,        /* ResourceError: allocation / budget (ewald_fourier.py:221-224) */
  HS_ERR_CUDA = 5,            /* CUDA / cuFFT failure (no reference counterpart) */
  HS_ERR_GEOMETRY = 6,        /* GeometryError: cell-list bounds (ewald_real.py:239-240) */
  HS_ERR_PARAMETER = 7        /* ParameterError (ewald_real.py:237-238, ewald_fourier.py:323-324) */
} hs_status;

enum { HS_MEM_DEVICE = 0, HS_MEM_HOST = 1 };
enum { HS_STOKESLET = 0, HS_STRESSLET = 1, HS_ROTLET = 2 };   /* _KIND_ID, ewald_real.py:29 */
/* Mixed stokeslet + stresslet sources sharing one set of positions (BASELINE configs[4]):
 * one evaluation equals the sum of the reference's two ewald_sum calls (ref:ewald.py:46-80),
 * with the two kinds' kernel and wall channels summed in k-space before the inverse
 * transforms.  Strengths: sa = f (n,3), sb = [g | q] (n,6) rows g0 g1 g2 q0 q1 q2. */
enum { HS_MIXED = 3 };
enum { HS_FREE = 0, HS_HALF = 1 };                            /* system.py:25-27 */
enum { HS_HARMONIC = 0, HS_BIHARMONIC = 1 };                  /* _KIND_BYTE, ewald_fourier.py:40 */

typedef struct hs_ctx hs_ctx;
typedef struct hs_plan hs_plan;

/* ---- context ---------------------------------------------------------- */
hs_status hs_ctx_create(int device, hs_ctx** out);
hs_status hs_ctx_destroy(hs_ctx* ctx);
/* Bind the context to a CUDA stream (cudaStream_t passed as void*; NULL = legacy default). */
hs_status hs_ctx_set_stream(hs_ctx* ctx, void* stream);
const char* hs_last_error(void);
/* Number of kernels this library launched since the context was created (for bench accounting). */
int64_t hs_ctx_launch_count(const hs_ctx* ctx);

/* ---- cell list: replaces ewald_real.build_cell_list (ewald_real.py:228-251) ----
 * points (n,3); bounds lo/hi (3,) host; rc > 0.  Outputs: order int64[n] (stable
 * argsort of the flat cell id), start int64[ncell+1], dims int64[3] (host),
 * edge double[3] (host).  ncell = prod(dims) is known to the caller through
 * hs_cell_dims() before allocating `start`. */
hs_status hs_cell_dims(double rc, const double lo[3], const double hi[3], int64_t dims[3], double edge[3]);
hs_status hs_cell_list(hs_ctx* ctx, const double* points, int64_t n, double rc, const double lo[3],
                       const double hi[3], int64_t* order, int64_t* start, int mem);

/* ---- gridding: replaces ewald_fourier.spread / gather (ewald_fourier.py:319-346,
 * _gridding.py:33-89).  grids are channel-first (nch,nx,ny,nz); gather returns
 * (n,nch) already multiplied by h^3 like ewald_fourier.gather. */
hs_status hs_spread(hs_ctx* ctx, const double* points, const double* weights, int64_t n, int nch,
                    const double origin[3], double h, const int64_t dims[3], int P, double xi,
                    double eta, double* grids, int mem);
hs_status hs_gather(hs_ctx* ctx, const double* grids, int nch, const double* points, int64_t n,
                    const double origin[3], double h, const int64_t dims[3], int P, double xi,
                    double eta, double* out, int mem);

/* ---- Green's tables: replaces ewald_fourier.precompute_greens (ewald_fourier.py:207-244).
 * kind HS_HARMONIC / HS_BIHARMONIC; big (3,) = oversampled grid; dims, guards (3,);
 * samples: real array of shape padded_dims = 2*(dims+guards). */
hs_status hs_precompute_greens(hs_ctx* ctx, int kind, double R, double h, const int64_t big[3],
                               const int64_t dims[3], const int64_t guards[3], double* samples, int mem);

/* ---- the whole evaluation ---------------------------------------------
 * A plan owns every device buffer of one (kind, geometry, grid, n, n_targets)
 * configuration: cell lists, channel grids, spectra, cuFFT plans, tables.
 * hs_params mirrors ewald.EwaldParams + GridSpec (ewald.py:17-43,
 * ewald_fourier.py:58-147); derived grid quantities are passed in so the host
 * mirror stays the single source of truth for them. */
typedef struct {
  int kind;               /* HS_STOKESLET / HS_STRESSLET / HS_ROTLET */
  int geometry;           /* HS_HALF / HS_FREE */
  double L;               /* box edge */
  double xi, rc;          /* Ewald split */
  int64_t M, P;           /* grid count (after the M+P parity bump) and window support */
  double h, eta;          /* GridSpec.h, GridSpec.eta */
  double origin[3];       /* GridSpec.origin */
  int64_t dims[3];        /* GridSpec.dims */
  int64_t padded[3];      /* GridSpec.padded_dims */
  int64_t n;              /* sources */
  int64_t n_targets;      /* targets (== n when targets are the sources) */
  int targets_are_sources;/* 1: targets=None semantics (target_indices = arange(n)) */
} hs_params;

/* params.M == 0 creates a real-space-only plan (real_space_sum, ewald_real.py:381-455): no grids,
 * transforms or tables are allocated; hs_plan_execute then accepts what = 1 only. */
hs_status hs_plan_create(hs_ctx* ctx, const hs_params* params, hs_plan** out);
hs_status hs_plan_destroy(hs_plan* plan);
/* Device bytes the plan holds. */
int64_t hs_plan_bytes(const hs_plan* plan);
/* Load one reference-layout table (GreensTable.samples, shape padded_dims). */
hs_status hs_plan_set_table(hs_plan* plan, int table_kind, const double* samples, int mem);
/* Build the tables this plan needs on the GPU (precompute_greens for each of
 * table_kinds_for(kind, geometry), ewald_fourier.py:281-290). */
hs_status hs_plan_build_tables(hs_plan* plan, const int64_t big[3], double R, const int64_t guards[3]);

/* Evaluate ewald.ewald_sum (ewald.py:46-80) for one set of strengths.
 *   positions (n,3); sa = f (stokeslet) or g; sb = q (stresslet/rotlet) or NULL;
 *   targets (n_targets,3) or NULL when targets_are_sources;
 *   tcols int64[n_targets] = target_indices (or NULL: -1 for all, no self term);
 *   u (n_targets,3) = real + fourier; u_real / u_fourier optional (NULL).
 *   times (optional, 16 doubles, milliseconds, CUDA events):
 *     [gridding, fft, scale, ifft, gather, real, fourier, h2d, total, io,
 *      k_pair, k_spread, k_gather, k_scale (kernel-only), accepted pairs, accepted image pairs]
 *   what: bit 0 = real part, bit 1 = Fourier part (3 = full sum); bit 2 = run the two parts
 *   one after the other on the context stream (by default the real-space part runs on a second,
 *   high-priority stream concurrently with the Fourier part up to the gather; serialised runs
 *   give undisturbed per-kernel times). */
hs_status hs_plan_execute(hs_plan* plan, const double* positions, const double* sa, const double* sb,
                          const double* targets, const int64_t* tcols, double* u, double* u_real,
                          double* u_fourier, int mem, int what, double* times);

/* Real-space parts of the last execute (ewald_real.py:450-452 `parts`): kernel
 * uk/(8pi|4pi) and correction uc/(4pi), each (n_targets,3). */
hs_status hs_plan_real_parts(hs_plan* plan, double* kernel_part, double* correction_part, int mem);

/* Neighbour audit of the real-space pair pass (ewald_real.py:277-299): evaluates the
 * real-space part for the given inputs (same arguments as hs_plan_execute) and writes, per
 * target, [accepted pairs, accepted image pairs, sum over the accepted combined source ids j
 * (j >= n: image of j - n) of splitmix64(j) mod 2^64] into audit (n_targets x 3 uint64).
 * The reference keeps a pair when ids[p] != tcols[t] and r2 = d0*d0 + d1*d1 + d2*d2 <= rc^2
 * over the 5x5x5 half-cells around the target's cell; the audit proves the CUDA pass keeps
 * exactly those sets (tests/test_gpu_parity.py, against oracle/ and tests/golden/). */
hs_status hs_plan_pair_audit(hs_plan* plan, const double* positions, const double* sa, const double* sb,
                             const double* targets, const int64_t* tcols, uint64_t* audit, int mem);

/* Number of forward / inverse 3-D transforms one execute performs. */
hs_status hs_plan_fft_counts(const hs_plan* plan, int* n_fft, int* n_ifft);

/* ---- y-slab decomposition of one evaluation over W ranks (multi-GPU) ----
 * The reference is single-process (ewald_fourier.py:486-636); this is the
 * sharded form of the same ewald_sum.  Rank r owns grid planes y in [y0, y1)
 * (all x, z) and half-spectrum columns kz in [kz0, kz1) (all kx, ky).  Its plan
 * holds ALL sources (real-space neighbours and images are global) and only
 * its own targets: those whose gather window starts in [y0, y1) (the caller
 * partitions them, see sharding.py).  One evaluation is five stages with four
 * exchanges the caller performs (torch.distributed / NCCL, or copies when all
 * ranks live in one process):
 *   hs_slab_begin     real-space sums of the rank's targets; spread of the
 *                     sources whose y window starts in the slab into planes
 *                     [y0, y1 + P - 1); ghost_out <- planes [y1, y1+P-1) of
 *                     every channel, layout [n_in][P-1][nx][nz]
 *   (send ghost_out to rank r+1)
 *   hs_slab_forward   ghost_in (from r-1, or NULL) added to planes [y0, y0+P-1);
 *                     z D2Z on owned planes; send <- per channel c the kz
 *                     blocks of every destination, layout [n_in][W][y1-y0][nx][kz1_s-kz0_s]
 *   (per channel: all-to-all send[c] -> recv[c]; recv layout [n_in][py][nx][kz1-kz0],
 *    block s = rows [y0_s, y1_s); rows >= ny must be zero)
 *   hs_slab_kspace    y transform, fused x transform + k-space scaling, inverse y;
 *                     back <- [n_out][ny][nx][kz1-kz0]
 *   (per channel: all-to-all back[c] rows [y0_s, y1_s) -> recv_back[c] block s,
 *    recv_back layout [n_out][W][y1-y0][nx][kz1_s-kz0_s])
 *   hs_slab_backward  inverse z on owned planes; halo_out <- output planes
 *                     [y0, y0+P-1), layout [P-1][nx][nz][pitch]
 *   (send halo_out to rank r-1)
 *   hs_slab_finish    halo_in (from r+1, or NULL) fills planes [y1, y1+P-1);
 *                     gather at the rank's targets; u = real + Fourier.
 * All exchange buffers are device memory on the plan's device; sizes come from
 * hs_slab_sizes.  Pointers passed to hs_slab_begin (inputs) must stay valid
 * until hs_slab_finish returns. */
typedef struct {
  int64_t rank, world;
  int64_t y0, y1;         /* owned grid planes */
  int64_t kz0, kz1;       /* owned half-spectrum columns */
  int64_t kz_split[65];   /* column boundaries of all ranks: rank s owns [kz_split[s], kz_split[s+1]) */
  int64_t y_split[65];    /* plane boundaries of all ranks */
} hs_slab;

/* Sizes of the exchange buffers, in doubles (complex values count 2):
 *   [0] ghost: n_in (P-1) nx nz             [1] send / recv_back, per channel: 2 (y1-y0) nx nzh
 *   [2] recv, per channel: 2 py nx (kz1-kz0)  [3] back, per channel: 2 ny nx (kz1-kz0)
 *   [4] halo: (P-1) nx nz pitch             [5] n_in   [6] n_out   [7] pitch */
hs_status hs_plan_create_slab(hs_ctx* ctx, const hs_params* params, const hs_slab* slab, hs_plan** out);
hs_status hs_slab_sizes(const hs_plan* plan, int64_t sizes[8]);
hs_status hs_slab_begin(hs_plan* plan, const double* positions, const double* sa, const double* sb,
                        const double* targets, const int64_t* tcols, int mem, double* ghost_out);
hs_status hs_slab_forward(hs_plan* plan, const double* ghost_in, double* send);
hs_status hs_slab_kspace(hs_plan* plan, const double* recv, double* back);
hs_status hs_slab_backward(hs_plan* plan, const double* recv_back, double* halo_out);
hs_status hs_slab_finish(hs_plan* plan, const double* halo_in, double* u, double* u_real, double* u_fourier,
                         int mem, double* times);
/* Channel-range forms of the middle stages, so the all-to-all of channel c can run (on the
 * collective's own stream) while channel c+1 is transformed:
 *   hs_slab_forward_range: as hs_slab_forward for input channels [c0, c1) (ghost add with c0 == 0);
 *   hs_slab_kspace_part:   part 0 = y transforms of input channels [c0, c1) from recv,
 *                          part 1 = the x stage, part 2 = inverse y of output channels [c0, c1);
 *   hs_slab_backward_range: inverse z of output channels [c0, c1); the call with c1 == n_out
 *                          also interleaves and writes halo_out. */
hs_status hs_slab_forward_range(hs_plan* plan, const double* ghost_in, double* send, int c0, int c1);
hs_status hs_slab_kspace_part(hs_plan* plan, int part, const double* recv, double* back, int c0, int c1);
hs_status hs_slab_backward_range(hs_plan* plan, const double* recv_back, double* halo_out, int c0, int c1);

/* ---- direct O(N Nt) half-space/free-space sum on the GPU (kernels_direct.py:211-371).
 * Same argument meaning as hs_plan_execute's strengths; returns physically
 * normalised velocities. */
hs_status hs_direct_sum(hs_ctx* ctx, int kind, int geometry, int64_t n, const double* positions,
                        const double* sa, const double* sb, int64_t n_targets, const double* targets,
                        const int64_t* tcols, double* u, int mem);

/* ---- debugging: device-side checks of the checked build (libhsewald_b200_checked.so, built
 * with -DHS_CHECKED; HSEWALD_CHECKED=1 selects it in the Python package).  Every kernel's ring,
 * queue and staging indices and its global stores are bounds-checked; the first failing check
 * ((translation unit << 32) | source line) and the failure count since the last reset are
 * returned.  The production library returns HS_ERR_CONFIG. */
hs_status hs_debug_checks(uint64_t* first_failure, uint64_t* failures, int reset);

#ifdef __cplusplus
}
#endif
#endif /* HSEWALD_B200_H */

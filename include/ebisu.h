/*
 * ebisu.h -- C ABI of the B200-native iterated Jacobi sweep (libebisu.so).
 *
 * This is the drop-in boundary for the reference's hot path.  The reference
 * (stencilplan, pure Python/NumPy) exposes the path as three Python calls;
 * each entry point below replaces one of them and keeps its contract:
 *
 *   ebisu_run_host / ebisu_run_device
 *     replace  stencilplan.grid.reference_run(grid, stencil, t) -> Grid
 *              (pkg/src/stencilplan/grid.py:106-113, per-step body
 *               reference_step grid.py:96-103, tap sum apply_taps :76-93)
 *     and the engine registry entries
 *              planner._ENGINES[scheme](grid, stencil, params) -> (Grid, trace)
 *              (planner.py:219,227; run_sm_tiling engine/sm.py:51,
 *               run_device_tiling engine/device.py:55)
 *     The result equals reference_run(grid, stencil, steps): bitwise when
 *     params.exact != 0 (one IEEE binary64 rounding per multiply and per add,
 *     taps summed in the order given), within 1e-12 relative otherwise.
 *     The input is never modified (reference purity, test_grid.py:152-157).
 *
 *   ebisu_run_host_f32 / ebisu_run_device_f32
 *     the same contract in binary32 (no reference counterpart: Grid forces
 *     float64, grid.py:38); the north-star fp32 mode, within 1e-5 relative
 *     of reference_run.
 *
 *   ebisu_random_grid_device
 *     replaces stencilplan.grid.random_grid / rng.uniform_array
 *              (grid.py:56-60, rng.py:31-46), bit-identical draws.
 *
 *   ebisu_compare_device
 *     replaces the planner's parity check np.array_equal + first mismatch
 *              (planner.py:227-232) on device-resident grids.
 *
 *   ebisu_check_compatible
 *     replaces grid._check_compatible (grid.py:63-73) and
 *     TilingParams.validate (engine/params.py:52-90); same messages.
 *
 * Conventions: plain C types only; no exceptions cross the ABI; every call
 * returns an ebisu_status and, on failure, leaves a thread-local message for
 * ebisu_last_error().  Grids are dense C-order float64 (or, for the _f32
 * entry points, float32) arrays, axis 0 slowest
 * (the streaming axis).  The caller owns every buffer it passes; the library
 * owns only device scratch it allocates itself and the pinned host slots it
 * stages pageable host buffers through (both released by
 * ebisu_release_scratch).  Calls are reentrant; one CUDA stream per call.
 */
#ifndef EBISU_H
#define EBISU_H

#include <stdint.h>

#if defined(EBISU_BUILD) && defined(__GNUC__)
#define EBISU_API __attribute__((visibility("default")))
#else
#define EBISU_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define EBISU_ABI_VERSION 3  /* 2: ebisu_params.frame_ready, fp32 entry points;
                                 3: ebisu_params.reserve_sms, trace.cluster_ctas */
#define EBISU_MAX_DIMS 3
#define EBISU_MAX_TAPS 128

typedef enum ebisu_status {
  EBISU_OK = 0,
  EBISU_ERR_VALUE = 1,       /* reference ValueError (grid/stencil mismatch)   */
  EBISU_ERR_PARAM = 2,       /* reference engine.ParamError (bad TilingParams) */
  EBISU_ERR_CUDA = 3,        /* CUDA runtime / driver failure                   */
  EBISU_ERR_UNSUPPORTED = 4, /* no kernel for this request (never a fallback)   */
  EBISU_ERR_NO_DEVICE = 5    /* no CUDA device visible                          */
} ebisu_status;

/* Scheme selector; mirrors engine/params.py:12-14 plus the GPU-only choices. */
typedef enum ebisu_scheme {
  EBISU_SCHEME_AUTO = 0,          /* planner picks (temporal blocking when possible) */
  EBISU_SCHEME_NAIVE = 1,         /* one sm_100a launch per time step (yardstick)    */
  EBISU_SCHEME_SM_TILING = 2,     /* overlapped streaming tiles, "sm-tiling"        */
  EBISU_SCHEME_DEVICE_TILING = 3, /* halo-exchange tiles, "device-tiling"           */
  EBISU_SCHEME_RESIDENT = 4       /* resident tiles, runtime taps: any stencil (AUTO
                                     uses it for shapes without a specialised kernel,
                                     e.g. 1-D and user tap sets, when the cost model
                                     beats one launch per step)                      */
} ebisu_scheme;

/* Stencil shape: reference StencilShape (shapes.py:27-56).  offsets holds
 * ntaps*dims ints, tap-major, axis 0 first, in the order the taps are summed. */
typedef struct ebisu_stencil {
  int32_t dims;            /* 1..3 */
  int32_t ntaps;           /* 1..EBISU_MAX_TAPS */
  const int32_t* offsets;  /* [ntaps][dims] */
  const double* coeffs;    /* [ntaps] */
} ebisu_stencil;

/* Tiling parameters: reference TilingParams (engine/params.py:18-38). */
typedef struct ebisu_params {
  int32_t scheme;            /* ebisu_scheme */
  int32_t t;                 /* temporal depth per HBM round trip (0 = auto) */
  int32_t tile[2];           /* reference tile extents over tiled axes (validated,
                                0 = auto); the GPU tile is chosen by the planner */
  int32_t device_tile_grid[2];
  int32_t lazy;              /* accepted for parity; the GPU kernels sync once per advance */
  int32_t exact;             /* 1: bitwise (no FMA contraction); 0: tolerance mode
                                (1e-12 relative): FMA chains, or for uniform
                                coefficients reassociated sums (see below)         */
  int32_t persistent;        /* 1: one cooperative launch, grid sync between epochs */
  int32_t validate_tile;     /* 1: apply the reference TilingParams.validate rules  */
  int32_t lane_cells;        /* cells per lane along the fastest axis (0 = planner) */
  int32_t seg_rows;          /* rows per work unit along axis 0 (0 = planner)       */
  int32_t variant;           /* n-th registered kernel for (shape, t) (0 = default) */
  int32_t per_tap_products;  /* 1: never share products between taps (see below)   */
  int32_t out_planes[2];     /* write only output planes [lo, hi) along axis 0; {0,0}
                                = all.  Needs a single fused epoch (steps <= t): the
                                multi-GPU driver computes its boundary band first,
                                sends it, and computes the interior while NCCL runs */
  int32_t frame_ready;       /* 1: d_out (and d_scratch) already hold the input's
                                Dirichlet frame, skip the frame pre-copy (repeated
                                epochs into the same buffers) */
  int32_t reserve_sms;       /* leave this many SMs free of the sweep's persistent
                                grid (0 = none): kernels issued concurrently on
                                other streams -- the multi-GPU driver's NCCL halo
                                exchange -- then run beside the interior instead
                                of queueing behind it */
} ebisu_params;
/* Shared products: when every coefficient of the stencil is bitwise equal (the
 * catalog default 1/|taps|, shapes.py:148-157), term_k = RN(c*x_k) depends on
 * the cell only, so the kernels compute it once per cell and level and every
 * tap reuses it.  The sums keep the reference order, so the result is still
 * bitwise equal to reference_run; only the DMUL count drops (13 -> 7 DP ops
 * per j3d7pt cell-step).  per_tap_products=1 forces the per-tap kernels.
 *
 * Reassociated sums (exact = 0, uniform coefficients): sum_k c*x_k is computed
 * as c * (regrouped sum) -- separable column/row sums shared between
 * neighbouring targets -- within the north star's 1e-12 relative tolerance:
 * j3d27pt 27 -> ~6 DP per cell-step, j2d25pt 25 -> ~6, j2ds25pt 25 -> ~12. */

/* Closed-form execution counters of the GPU run (reference ExecutionTrace,
 * engine/trace.py:25-40), plus GPU facts. */
typedef struct ebisu_trace {
  uint64_t gm_loads;         /* cells loaded from HBM by TMA (incl. overlap halos) */
  uint64_t gm_stores;        /* cells stored                                       */
  uint64_t gm_halo_loads;
  uint64_t gm_halo_stores;
  uint64_t syncs_block;
  uint64_t syncs_device;     /* grid-wide barriers                                 */
  uint64_t cells_computed;   /* lane-steps issued                                  */
  uint64_t cells_valid;      /* stored cells x depth                               */
  uint64_t device_tiles;     /* work units (strip x segment) processed             */
  uint64_t kernel_launches;
  double elapsed_ms;         /* device time of the sweep (CUDA events)             */
  int32_t kernel_id;         /* which kernel family ran (see ebisu_kernel_name)    */
  int32_t t_used;            /* temporal depth actually fused                      */
  int32_t grid_ctas;
  int32_t warps_per_cta;
  int32_t arith;             /* EBISU_ARITH_*: arithmetic of the main stage        */
  int32_t cluster_ctas;      /* CTAs per cluster tile (device tile) of the main stage */
  int32_t reserved[2];
} ebisu_trace;

/* ebisu_trace.arith */
#define EBISU_ARITH_SHARED_PRODUCTS 0 /* bitwise: RN(c*x) once per cell, tap-order adds */
#define EBISU_ARITH_PER_TAP_EXACT 1   /* bitwise: RN(ck*xk) per tap, tap-order adds     */
#define EBISU_ARITH_PER_TAP_FMA 2     /* tolerance: FMA chain in tap order              */
#define EBISU_ARITH_REASSOCIATED 3    /* tolerance: c * (regrouped sum), uniform coeffs */

/* Library / device facts. */
EBISU_API int32_t ebisu_abi_version(void);
EBISU_API const char* ebisu_last_error(void);
EBISU_API const char* ebisu_kernel_name(int32_t kernel_id);
EBISU_API int32_t ebisu_device_count(void);

/* Validation only (no GPU needed): reference _check_compatible + validate. */
EBISU_API int32_t ebisu_check_compatible(const ebisu_stencil* stencil, int32_t ndim,
                               const int64_t* extents, const ebisu_params* params);

/* Host buffers in/out: H2D, sweep, D2H on the current device.  in/out may
 * alias only if identical (in-place on the host side is allowed). */
EBISU_API int32_t ebisu_run_host(const ebisu_stencil* stencil, int32_t ndim,
                       const int64_t* extents, const double* in, double* out,
                       int64_t steps, const ebisu_params* params,
                       ebisu_trace* trace /* nullable */);

/* Device buffers: d_in is read only; d_out receives the result; d_scratch is
 * an optional grid-sized device buffer (NULL: library arena).  stream is a
 * cudaStream_t (NULL = legacy default stream).  Asynchronous unless trace is
 * non-NULL (then the call waits to fill elapsed_ms). */
EBISU_API int32_t ebisu_run_device(const ebisu_stencil* stencil, int32_t ndim,
                         const int64_t* extents, const double* d_in, double* d_out,
                         double* d_scratch, int64_t steps,
                         const ebisu_params* params, void* stream,
                         ebisu_trace* trace /* nullable */);

/* fp32 sweeps (north-star tolerance mode, 1e-5 relative to the fp64
 * reference): same contract with float buffers; arithmetic in binary32 with
 * the same operation order (coefficients rounded to float once).  The fast
 * path needs the last extent to be a multiple of 4 (16-byte TMA rows). */
EBISU_API int32_t ebisu_run_host_f32(const ebisu_stencil* stencil, int32_t ndim,
                           const int64_t* extents, const float* in, float* out,
                           int64_t steps, const ebisu_params* params,
                           ebisu_trace* trace /* nullable */);
EBISU_API int32_t ebisu_run_device_f32(const ebisu_stencil* stencil, int32_t ndim,
                             const int64_t* extents, const float* d_in, float* d_out,
                             float* d_scratch, int64_t steps,
                             const ebisu_params* params, void* stream,
                             ebisu_trace* trace /* nullable */);

/* SplitMix64 uniforms [0,1): d_out[i] = draw i of SplitMix64(seed) for
 * i in [start, start+n). Bit-identical to rng.uniform_array. */
EBISU_API int32_t ebisu_random_grid_device(uint64_t seed, int64_t start, int64_t n,
                                 double* d_out, void* stream);

/* Device-side parity check of two float64 arrays: number of bitwise
 * mismatches, first mismatch index (-1 if none), max |a-b| and max |b|. */
EBISU_API int32_t ebisu_compare_device(const double* d_a, const double* d_b, int64_t n,
                             int64_t* mismatches, int64_t* first_mismatch,
                             double* max_abs_diff, double* max_abs_ref,
                             void* stream);

/* Free the library's device scratch arena for the current device and the
 * pinned host slots of the pageable-buffer path. */
EBISU_API int32_t ebisu_release_scratch(void);

#ifdef __cplusplus
}
#endif
#endif /* EBISU_H */

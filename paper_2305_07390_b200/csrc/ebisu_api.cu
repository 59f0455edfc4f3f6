// ebisu_api.cu -- the C ABI (include/ebisu.h): validation with the
// reference's messages, shape matching, kernel planning, epoch chaining,
// TMA descriptor encoding, and the host<->device wrappers.
//
// Reference call sites replaced (see include/ebisu.h for the full map):
//   grid.reference_run        pkg/src/stencilplan/grid.py:106-113
//   grid._check_compatible    grid.py:63-73
//   engine.params.validate    engine/params.py:52-90
//   planner._ENGINES[...]     planner.py:219,227
#include <cudaTypedefs.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>

#include <algorithm>
#include <array>
#include <cmath>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "ebisu_internal.h"
#include "ebisu_common.cuh"
#include "ebisu_shapes.cuh"
#include "ebisu_stream2d.cuh"

namespace ebisu {
namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(EBISU_ERR_CUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define EB_CUDA(call)                                  \
  do {                                                 \
    cudaError_t _e = (call);                           \
    if (_e != cudaSuccess) return cuda_fail(_e, #call); \
  } while (0)

// ---- shape matching -------------------------------------------------------
template <class SH>
bool match_shape(const ebisu_stencil* s) {
  if (s->dims != SH::dims || s->ntaps != SH::NT) return false;
  for (int i = 0; i < SH::NT; ++i) {
    const Off o = SH::tap(i);
    const int* p = s->offsets + i * s->dims;
    if (p[0] != o.d0) return false;
    if (s->dims >= 2 && p[1] != o.d1) return false;
    if (s->dims >= 3 && p[2] != o.d2) return false;
  }
  return true;
}

int identify_shape(const ebisu_stencil* s) {
  if (match_shape<StarShape<2, 1>>(s)) return SHAPE_J2D5PT;
  if (match_shape<StarShape<2, 2>>(s)) return SHAPE_J2D9PT;
  if (match_shape<BoxShape<2, 1>>(s)) return SHAPE_J2D9PT_GOL;
  if (match_shape<BoxShape<2, 2>>(s)) return SHAPE_J2D25PT;
  if (match_shape<StarShape<2, 3>>(s)) return SHAPE_J2D13PT;
  if (match_shape<StarShape<2, 6>>(s)) return SHAPE_J2DS25PT;
  if (match_shape<StarShape<3, 1>>(s)) return SHAPE_J3D7PT;
  if (match_shape<StarShape<3, 2>>(s)) return SHAPE_J3D13PT;
  if (match_shape<NoCornerShape3<true>>(s)) return SHAPE_J3D17PT;
  if (match_shape<BoxShape<3, 1>>(s)) return SHAPE_J3D27PT;
  if (match_shape<NoCornerShape3<false>>(s)) return SHAPE_POISSON;
  if (match_shape<StarShape<1, 1>>(s)) return SHAPE_J1D3PT;
  return SHAPE_GENERIC;
}

// ---- validation (reference messages) -------------------------------------
int validate(const ebisu_stencil* st, int ndim, const int64_t* ext, const ebisu_params* prm,
             ProblemDesc* out) {
  if (!st || !ext) return fail(EBISU_ERR_VALUE, "null stencil or extents");
  if (st->dims < 1 || st->dims > EBISU_MAX_DIMS)
    return fail(EBISU_ERR_VALUE, "stencil dims %d not supported (1..3)", st->dims);
  if (st->ntaps < 1) return fail(EBISU_ERR_VALUE, "tap set is empty");
  if (st->ntaps > EBISU_MAX_TAPS)
    return fail(EBISU_ERR_VALUE, "%d taps exceed the supported %d", st->ntaps, EBISU_MAX_TAPS);
  if (!st->offsets || !st->coeffs) return fail(EBISU_ERR_VALUE, "null offsets or coefficients");
  // grid._check_compatible (grid.py:63-73)
  if (ndim != st->dims)
    return fail(EBISU_ERR_VALUE, "grid is %d-D but stencil is %d-D", ndim, st->dims);
  int rad = 0;
  bool has_zero = false;
  for (int t = 0; t < st->ntaps; ++t) {
    bool zero = true;
    for (int d = 0; d < st->dims; ++d) {
      const int v = st->offsets[t * st->dims + d];
      rad = std::max(rad, v < 0 ? -v : v);
      zero = zero && v == 0;
    }
    has_zero = has_zero || zero;
  }
  if (!has_zero) return fail(EBISU_ERR_VALUE, "tap set must contain the zero offset");
  for (int d = 0; d < ndim; ++d) {
    if (ext[d] <= 2 * rad)
      return fail(EBISU_ERR_VALUE, "extent %lld too small for radius %d (need > %d)",
                  (long long)ext[d], rad, 2 * rad);
  }
  long long total = 1;
  for (int d = 0; d < ndim; ++d) total *= ext[d];
  if (total >= (1ll << 40)) return fail(EBISU_ERR_VALUE, "grid too large");
  out->dims = st->dims;
  out->ntaps = st->ntaps;
  out->rad = rad;
  for (int d = 0; d < 3; ++d) out->ext[d] = d < ndim ? ext[d] : 1;
  out->offsets = st->offsets;
  out->coeffs = st->coeffs;
  out->shape_id = identify_shape(st);
  if (prm) {
    if (prm->scheme < EBISU_SCHEME_AUTO || prm->scheme > EBISU_SCHEME_RESIDENT)
      return fail(EBISU_ERR_PARAM, "unknown scheme %d", prm->scheme);
    if (prm->t < 0) return fail(EBISU_ERR_PARAM, "temporal depth must be >= 1");
    if (prm->reserve_sms < 0) return fail(EBISU_ERR_PARAM, "reserve_sms must be >= 0");
    if (prm->out_planes[1] != 0 &&
        (prm->out_planes[0] < 0 || prm->out_planes[0] >= prm->out_planes[1] ||
         prm->out_planes[1] > ext[0]))
      return fail(EBISU_ERR_PARAM, "output-plane range [%d, %d) outside [0, %lld)",
                  prm->out_planes[0], prm->out_planes[1], (long long)ext[0]);
    if (prm->validate_tile && prm->t >= 1) {
      // engine/params.py:52-90 (reference TilingParams.validate)
      const int t = prm->t;
      int axes[3], nax = 0;
      if (st->dims == 1) {
        axes[nax++] = 0;
      } else if (st->dims == 2 && prm->scheme == EBISU_SCHEME_DEVICE_TILING) {
        axes[nax++] = 0;
        axes[nax++] = 1;
      } else {
        for (int a = 1; a < st->dims; ++a) axes[nax++] = a;
      }
      if (prm->scheme == EBISU_SCHEME_SM_TILING) {
        for (int i = 0; i < nax && i < 2; ++i) {
          const int w = prm->tile[i];
          if (w - 2 * rad * t <= 0)
            return fail(EBISU_ERR_PARAM,
                        "tile extent %d leaves no valid core at depth %d (needs > %d)", w, t,
                        2 * rad * t);
        }
      } else if (prm->scheme == EBISU_SCHEME_DEVICE_TILING) {
        const int halo = rad * t;
        for (int i = 0; i < nax && i < 2; ++i) {
          const int g = prm->device_tile_grid[i] ? prm->device_tile_grid[i] : 1;
          const int w = prm->tile[i];
          if (g < 1) return fail(EBISU_ERR_PARAM, "device tile grid entries must be >= 1");
          const long long interior = ext[axes[i]] - 2 * rad;
          const long long loaded = (long long)g * w;
          if (loaded < interior && loaded + 2 * halo > ext[axes[i]])
            return fail(EBISU_ERR_PARAM,
                        "device tile of %lld cells plus 2*%d halo exceeds extent %lld on axis %d",
                        loaded, halo, (long long)ext[axes[i]], axes[i]);
          if (loaded - 2 * halo <= 0 && loaded < interior)
            return fail(EBISU_ERR_PARAM, "device tile of %lld cells has no core at depth %d",
                        loaded, t);
        }
      }
    }
  }
  return EBISU_OK;
}

// ---- device facts ----------------------------------------------------------
struct DevInfo {
  int sms = 0;
  bool coop = false;
};

int device_info(DevInfo* di) {
  int dev = 0;
  EB_CUDA(cudaGetDevice(&dev));
  static std::mutex mu;
  static std::vector<DevInfo> cache;
  std::lock_guard<std::mutex> lk(mu);
  if ((int)cache.size() <= dev) cache.resize(dev + 1);
  if (cache[dev].sms == 0) {
    int v = 0;
    EB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
    cache[dev].sms = v;
    EB_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrCooperativeLaunch, dev));
    cache[dev].coop = v != 0;
    // Keep freed scratch in the stream-ordered pool (8 GiB grids reuse it).
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
  }
  *di = cache[dev];
  return EBISU_OK;
}

// ---- TMA descriptors ---------------------------------------------------------
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

int encode_map(CUtensorMap* m, const void* base, int rank, const long long* dims_fast_first,
               const int* box_fast_first, int elem, long long row_pitch) {
  auto enc = get_encode();
  if (!enc) return fail(EBISU_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t gdim[3], gstride[2];
  cuuint32_t box[3], estr[3];
  // byte strides of dims 1.. : the innermost row pitch may exceed the extent
  // (padded rows of an odd last extent; TMA needs 16-byte strides)
  long long pitch = (long long)elem * row_pitch;
  for (int i = 0; i < rank; ++i) {
    gdim[i] = (cuuint64_t)dims_fast_first[i];
    box[i] = (cuuint32_t)box_fast_first[i];
    estr[i] = 1;
    if (i + 1 < rank) {
      gstride[i] = (cuuint64_t)pitch;
      pitch *= dims_fast_first[i + 1];
    }
  }
  CUresult r = enc(m, elem == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64,
                   (cuuint32_t)rank, const_cast<void*>(base), gdim,
                   gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(EBISU_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return EBISU_OK;
}

// ---- planning -----------------------------------------------------------------
enum KernelId : int {
  KID_NONE = 0,
  KID_NAIVE = 1,
  KID_STREAM2D = 2,
  KID_STREAM3D = 3,
  KID_HALO2D = 4,
  KID_GENERIC = 5,
  KID_GENERIC_S3D = 6,
};

// First registered kernel for (shape, depth, exactness) -- the registry lists
// the planner's default lane width first -- or the one with lane width C.
// Kernel family for a request: shared-product kernels (uni) are bitwise exact,
// so they serve both exact and FMA requests when the coefficients are uniform.
// Tolerance requests (exact = 0) with uniform coefficients prefer the
// reassociated kernels (uni && !exact) and fall back to the bitwise ones.
bool family_ok(const TbKernel& k, bool exact, bool uni, int family, int elem) {
  if (k.family != family || k.elem != elem) return false;
  if (uni) return k.uni != 0 && (exact ? k.exact != 0 : true);
  return k.uni == 0 && (k.exact != 0) == exact;
}

const TbKernel* find_tb(int shape_id, int dims, int T, bool exact, bool uni, int family,
                        int elem, int C = 0, int variant = 0) {
  int n = 0;
  const TbKernel* ks = tb_kernels(&n);
  // tolerance + uniform: reassociated kernels (exact == 0) first, then the
  // bitwise shared-product ones; variants are numbered across both passes
  const bool tol = uni && !exact;
  for (int pass = tol ? 0 : 1; pass < 2; ++pass)
    for (int i = 0; i < n; ++i) {
      if (!(ks[i].shape_id == shape_id && ks[i].dims == dims && ks[i].T == T &&
            family_ok(ks[i], exact, uni, family, elem) && (C == 0 || ks[i].C == C)))
        continue;
      if (tol && (ks[i].exact == 0) != (pass == 0)) continue;
      if (variant-- == 0) return &ks[i];
    }
  return nullptr;
}

// largest instantiated depth <= tmax for this shape
int best_depth_leq(int shape_id, int dims, int tmax, bool exact, bool uni, int family,
                   int elem) {
  int n = 0, best = 0;
  const TbKernel* ks = tb_kernels(&n);
  for (int i = 0; i < n; ++i)
    if (ks[i].shape_id == shape_id && ks[i].dims == dims &&
        family_ok(ks[i], exact, uni, family, elem) && ks[i].T <= tmax)
      best = std::max(best, ks[i].T);
  return best;
}

// Scheme -> kernel family.  sm-tiling: overlapped warp strips; device-tiling:
// CTA strips with per-level halo exchange.  AUTO: overlapped for every shape
// -- measured faster on B200 even for the large-halo stars (DESIGN.md §3.3:
// j2ds25pt 199 vs 146, j2d13pt 486 vs 352 GCells/s at 8192^2).
int pick_family(int scheme, int shape_id, int dims) {
  (void)shape_id;
  if (dims != 2) return 0;
  return scheme == EBISU_SCHEME_DEVICE_TILING ? 1 : 0;
}

// Every coefficient bitwise equal (the catalog default, shapes.py:156-157)?
bool uniform_coeffs(const ProblemDesc& p) {
  for (int i = 1; i < p.ntaps; ++i)
    if (memcmp(&p.coeffs[i], &p.coeffs[0], sizeof(double)) != 0) return false;
  return true;
}

// Default fused depth (measured sweet spot on B200).
// Tolerance mode with uniform coefficients (reassociated kernels): the
// measured-best depth per shape where it differs from the bitwise one
// (8192^2 x 96 / 512^3 x 500: j2d13pt t=2 601 vs t=3 , j2d9pt t=3 848 vs t=4 spills)
int default_depth_tol(int shape_id, int exact_default) {
  switch (shape_id) {
    case SHAPE_J2D13PT: return 2;
    default: return exact_default;
  }
}

int default_depth(int shape_id) {
  switch (shape_id) {
    case SHAPE_J2D5PT: return 8;
    case SHAPE_J2D9PT_GOL: return 6;
    case SHAPE_J2D9PT: return 4;
    case SHAPE_J2D25PT: return 2;  // t=1/2/3/4: 293/330/248/202 (tools/tune_depths.py)
    case SHAPE_J2D13PT: return 3;
    case SHAPE_J2DS25PT: return 1;
    case SHAPE_J3D7PT: return 4;
    case SHAPE_J3D13PT: return 2;
    case SHAPE_J3D27PT: return 2;
    case SHAPE_J3D17PT: return 2;
    case SHAPE_POISSON: return 2;
    default: return 4;
  }
}

struct Stage {
  int kind;            // KID_*
  const TbKernel* k;   // for TB stages
  int epochs;          // fused epochs (TB) or steps (naive)
  int T = 0;           // KID_GENERIC: levels per epoch
};

struct Counters {
  uint64_t gm_loads = 0, gm_stores = 0, cells_computed = 0, device_tiles = 0, syncs_device = 0,
           syncs_block = 0, launches = 0, halo_loads = 0, halo_stores = 0;
  int grid = 0, nw = 0, t_used = 0, kid = KID_NONE;
  int cluster = 1;  // CTAs per cluster tile of the main stage
  int arith = -1;  // EBISU_ARITH_* of the first (main) stage
};

// arithmetic family of a kernel (ebisu_trace.arith)
inline int arith_of(const TbKernel* k) {
  if (k->uni) return k->exact ? EBISU_ARITH_SHARED_PRODUCTS : EBISU_ARITH_REASSOCIATED;
  return k->exact ? EBISU_ARITH_PER_TAP_EXACT : EBISU_ARITH_PER_TAP_FMA;
}

inline int stream3d_advances_host(int ka, int r1, int TZ, int WN) {
  const int n = r1 + TZ - ka;
  return (n + WN - 1) / WN * WN;
}

// Row (axis-0) segmentation of the work units.  Every unit pays a pipeline
// warm-up of `warm` advances; units are handed out dynamically to `slots`
// concurrent workers, so an epoch takes about units*(len+warm)/slots plus a
// tail of up to one unit.  Minimise that estimate.
void plan_segments(int n0, long long tiles, long long slots, int warm, int min_len,
                   int* nseg_out, int* seg_len_out) {
  double best = 1e300;
  int best_len = n0;
  for (int nseg = 1; nseg <= 4096 && nseg <= n0; ++nseg) {
    const int len = (n0 + nseg - 1) / nseg;
    if (len < min_len && nseg > 1) break;
    const int ns = (n0 + len - 1) / len;
    const double units = (double)tiles * ns;
    const double unit_cost = (double)(len + warm);
    const double cost = std::max(units / (double)slots, 1.0) * unit_cost + 0.5 * unit_cost;
    if (cost < best * 0.999) {
      best = cost;
      best_len = len;
    }
  }
  *seg_len_out = best_len;
  *nseg_out = (n0 + best_len - 1) / best_len;
}

// Guided segment list over output rows/planes [z_lo, z_hi): start with the
// balanced length and halve it once the remaining work is under two rounds of
// units, so the epoch tail (the grid.sync wait) is made of short units; never
// below min_len (short segments pay the per-unit warm-up in full).
std::vector<int> guided_segments(int z_lo, int z_hi, long long tiles, long long slots,
                                 int seg_len, int min_len, int seg_rows_req) {
  std::vector<int> seg_start;
  if (seg_rows_req > 0) {
    for (int r = z_lo; r < z_hi; r += seg_rows_req) seg_start.push_back(r);
  } else {
    int cur = std::max(seg_len, min_len), pos = z_lo;
    while (pos < z_hi) {
      const long long rem = z_hi - pos;
      while (cur > min_len && rem * tiles < 2ll * cur * slots) cur = std::max(min_len, cur / 2);
      seg_start.push_back(pos);
      pos += (int)std::min<long long>(cur, rem);
    }
  }
  if ((int)seg_start.size() > EBISU_MAX_SEGS) {
    const int len = (z_hi - z_lo + EBISU_MAX_SEGS - 1) / EBISU_MAX_SEGS;
    seg_start.clear();
    for (int r = z_lo; r < z_hi; r += len) seg_start.push_back(r);
  }
  seg_start.push_back(z_hi);
  return seg_start;
}

// Dataflow epochs (per-unit completion flags instead of grid.sync between
// epochs); EBISU_DATAFLOW=0 restores the grid-wide barrier (A/B measurement).
bool dataflow_epochs() {
  static const bool on = [] {
    const char* v = getenv("EBISU_DATAFLOW");
    return !(v && v[0] == '0');
  }();
  return on;
}

// Per-epoch dynamic-scheduling counters for one stage (zeroed on `st`).
int alloc_work(int epochs, cudaStream_t st, int** out) {
  EB_CUDA(cudaMallocAsync((void**)out, sizeof(int) * (size_t)std::max(epochs, 1), st));
  EB_CUDA(cudaMemsetAsync(*out, 0, sizeof(int) * (size_t)std::max(epochs, 1), st));
  return EBISU_OK;
}

int run_tb2d_stage(const ProblemDesc& p, const TbKernel* k, int epochs, int first_src,
                   int first_dst, void* bufs[3], const CUtensorMap maps[3], bool coop_req,
                   int seg_rows_req, const DevInfo& di, cudaStream_t st, Counters* ctr) {
  const int n0 = (int)p.ext[0], n1 = (int)p.ext[1];
  const int T = k->T, R = p.rad;
  int per_sm = 0;
  EB_CUDA(cudaFuncSetAttribute(k->func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               k->smem_bytes));
  EB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k->func, k->NW * 32,
                                                        (size_t)k->smem_bytes));
  if (per_sm < 1) return fail(EBISU_ERR_CUDA, "stream2d kernel cannot be resident (T=%d)", T);
  const int max_ctas = per_sm * di.sms;
  const int total_warps = max_ctas * k->NW;
  const int VW = k->valid_x;
  const int LC = k->box0, HX = (LC - VW) / 2;
  int aligned = 0;
  const int nstrips = stream2d_nstrips(n1, LC, VW, HX, R, k->C, &aligned, 16 / p.elem);
  const int span = p.z_hi - p.z_lo;  // output rows of this call
  int nseg = 1, seg_len = span;
  plan_segments(span, nstrips, total_warps, 2 * T * R, std::max(16, 2 * T * R), &nseg, &seg_len);
  // Persistent multi-epoch launches: uniform segments (the guided schedule
  // measured 3 % slower there: dataflow epochs already hide the tail and the
  // extra warm-ups cost more).  Single-epoch launches (the multi-GPU driver's
  // per-epoch calls, one launch per epoch) end in a real tail: guided
  // segments, shortest last.  EBISU_SEG2D=uniform|guided forces one (A/B).
  const bool multi = coop_req && di.coop && epochs > 1;
  bool guided = !multi;
  if (const char* v = getenv("EBISU_SEG2D")) guided = strcmp(v, "guided") == 0;
  const std::vector<int> seg_start =
      guided_segments(p.z_lo, p.z_hi, nstrips, total_warps, seg_len,
                      guided ? std::max(16, 2 * T * R) : seg_len,
                      seg_rows_req > 0 ? seg_rows_req : (guided ? 0 : seg_len));
  nseg = (int)seg_start.size() - 1;
  const long long units = (long long)nstrips * nseg;
  // every resident warp pulls units dynamically
  int grid = (int)std::min<long long>(max_ctas, (units + k->NW - 1) / k->NW);
  if (grid < 1) grid = 1;
  const bool coop = coop_req && di.coop && epochs > 1;

  TbLaunch L{};
  L.n0 = n0;
  L.n1 = n1;
  L.nstrips = nstrips;
  L.nseg = nseg;
  L.seg_len = seg_len;
  L.seg_start = seg_start.data();
  L.z_lo = p.z_lo;
  L.z_hi = p.z_hi;
  L.first_src = first_src;
  L.first_dst = first_dst;
  L.aligned = aligned;
  L.pitch = (int)(p.pitch ? p.pitch : p.ext[1]);
  for (int i = 0; i < 3; ++i) L.buf[i] = bufs[i];
  L.maps = maps;
  L.coeffs = p.coeffs;
  L.grid = grid;
  L.stream = st;
  long long* clk = nullptr;
  const char* clk_path = getenv("EBISU_UNIT_CLOCK");
  if (clk_path && *clk_path) {
    EB_CUDA(cudaMallocAsync((void**)&clk, sizeof(long long) * 2 * units, st));
    EB_CUDA(cudaMemsetAsync(clk, 0, sizeof(long long) * 2 * units, st));
    L.unit_clock = clk;
  }
  int* work = nullptr;
  if (int rc = alloc_work(epochs, st, &work)) return rc;
  int* flags = nullptr;
  if (coop && dataflow_epochs()) {
    EB_CUDA(cudaMallocAsync((void**)&flags, sizeof(int) * (size_t)units, st));
    EB_CUDA(cudaMemsetAsync(flags, 0, sizeof(int) * (size_t)units, st));
  }
  if (coop) {
    L.epochs = epochs;
    L.cooperative = true;
    L.work = work;
    L.flags = flags;
    EB_CUDA(k->launch(L));
    ctr->launches += 1;
    // dataflow epochs replace the grid-wide barrier by per-unit flag waits
    if (!flags) ctr->syncs_device += (uint64_t)(epochs - 1);
  } else {
    int src = first_src, dst = first_dst;
    for (int e = 0; e < epochs; ++e) {
      L.epochs = 1;
      L.first_src = src;
      L.first_dst = dst;
      L.cooperative = false;
      L.work = work + e;
      EB_CUDA(k->launch(L));
      ctr->launches += 1;
      src = dst;
      dst = (dst == BUF_OUT) ? BUF_SCR : BUF_OUT;
    }
  }
  cudaFreeAsync(work, st);
  if (flags) cudaFreeAsync(flags, st);
  if (clk) {
    std::vector<long long> h(2 * units);
    EB_CUDA(cudaMemcpyAsync(h.data(), clk, sizeof(long long) * 2 * units,
                            cudaMemcpyDeviceToHost, st));
    EB_CUDA(cudaStreamSynchronize(st));
    cudaFreeAsync(clk, st);
    if (FILE* f = fopen(clk_path, "w")) {
      fprintf(f, "unit,strip,seg,start_ns,end_ns\n");
      for (long long u = 0; u < units; ++u)
        fprintf(f, "%lld,%lld,%lld,%lld,%lld\n", u, u % nstrips, u / nstrips, h[2 * u],
                h[2 * u + 1]);
      fclose(f);
    }
  }
  // closed-form counters (reference ExecutionTrace semantics, trace.py:1-17)
  uint64_t loads = 0, adv = 0;
  for (int g = 0; g < nseg; ++g) {
    const int r0 = seg_start[g], r1 = seg_start[g + 1];
    const int ka = std::max(0, r0 - T * R), kb = std::min(n0, r1 + T * R);
    loads += (uint64_t)(kb - ka);
    adv += (uint64_t)(r1 + T * R - ka);
  }
  ctr->gm_loads += (uint64_t)epochs * loads * (uint64_t)(32 * k->C) * (uint64_t)nstrips;
  ctr->gm_stores += (uint64_t)epochs * (uint64_t)span * (uint64_t)n1;
  ctr->cells_computed +=
      (uint64_t)epochs * adv * (uint64_t)T * (uint64_t)(32 * k->C) * (uint64_t)nstrips;
  ctr->device_tiles += (uint64_t)epochs * (uint64_t)units;
  ctr->grid = grid;
  ctr->nw = k->NW;
  ctr->t_used = std::max(ctr->t_used, T);
  if (ctr->arith < 0) ctr->arith = arith_of(k);
  if (ctr->kid == KID_NONE) ctr->kid = KID_STREAM2D;  // the first (main) stage names the run
  return EBISU_OK;
}

int run_halo2d_stage(const ProblemDesc& p, const TbKernel* k, int epochs, int first_src,
                     int first_dst, void* bufs[3], const CUtensorMap maps[3], bool coop_req,
                     int seg_rows_req, int cl_req, const DevInfo& di, cudaStream_t st,
                     Counters* ctr) {
  const int n0 = (int)p.ext[0], n1 = (int)p.ext[1];
  const int T = k->T, R = p.rad;
  int per_sm = 0;
  EB_CUDA(cudaFuncSetAttribute(k->func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               k->smem_bytes));
  EB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k->func, k->NW * 32,
                                                        (size_t)k->smem_bytes));
  if (per_sm < 1) return fail(EBISU_ERR_CUDA, "halo2d kernel cannot be resident (T=%d)", T);
  const int LW = k->wn, VW = k->valid_x, HX = (LW - VW) / 2, Z = k->z;
  // Device tile = a cluster of CL CTA strips side by side (the reference's
  // device_tile_grid, engine/device.py:91-93): only the tile's outer edges
  // carry the t*R margin, the CL-1 seams exchange edges through DSMEM.  One
  // tile spanning the whole width has no margin at all.
  auto strips_for = [&](int cl, int* aligned) {
    const int LWc = cl * LW, VWc = LWc - 2 * HX;
    if (LWc >= n1) {
      *aligned = 0;
      return 1;
    }
    *aligned = n1 >= 2 * LWc ? 1 : 0;
    if (*aligned) {
      const int mid = strip_last_x0(n1, LWc, 2) - VWc;
      return 2 + (mid > 0 ? (mid + VWc - 1) / VWc : 0);
    }
    return (n1 + VWc - 1) / VWc;
  };
  // reassociated (tolerance) kernels exchange once per block of advances:
  // single-CTA tiles only
  const bool ra = k->uni && !k->exact;
  // the cluster-tile twin of this kernel (same shape, depth, lanes, arithmetic)
  const TbKernel* kc = nullptr;
  if (!ra) {
    int nk = 0;
    const TbKernel* ks = tb_kernels(&nk);
    for (int i = 0; i < nk && !kc; ++i)
      if (ks[i].max_clusters_n && ks[i].shape_id == k->shape_id && ks[i].T == T &&
          ks[i].C == k->C && ks[i].exact == k->exact && ks[i].uni == k->uni &&
          ks[i].elem == k->elem && ks[i].family == 1)
        kc = &ks[i];
  }
  int cl = 1, max_ctas = per_sm * di.sms;
  // (no cluster-tile twin for this stencil / depth / arithmetic: the device
  // tile is one CTA -- the same result, device_tile_grid only shapes the run)
  if (kc) {
    double best = -1;
    // requested: that many CTAs (portable cluster sizes 1..8); AUTO: 1/2/4/8
    const int req = std::min(cl_req, 8);
    const int cands[4] = {1, 2, 4, 8};
    for (int i = 0; i < (req > 0 ? 1 : 4); ++i) {
      const int c = req > 0 ? req : cands[i];
      int slots = per_sm * di.sms;
      if (c > 1) {
        int ncl = 0;
        EB_CUDA(kc->max_clusters_n(c, &ncl));
        slots = std::min(ncl * c, per_sm * di.sms / c * c);  // (reserve_sms)
      }
      if (slots < c) continue;
      int al = 0;
      // CTA strips of work per row over the resident CTAs (lower is better)
      const double cost = (double)strips_for(c, &al) * c / slots;
      if (best < 0 || cost < best * 0.99) {
        best = cost;
        cl = c;
        max_ctas = slots;
      }
    }
    if (best < 0)
      return fail(EBISU_ERR_UNSUPPORTED, "no resident cluster of %d halo-exchange CTAs", cl_req);
    if (cl > 1) k = kc;
  }
  int aligned = 0;
  const int nstrips = strips_for(cl, &aligned);
  const int span = p.z_hi - p.z_lo;
  int nseg = 1, seg_len = span;
  plan_segments(span, nstrips, max_ctas / cl, T * (R + Z), std::max(16, 2 * T * Z), &nseg,
                &seg_len);
  if (seg_rows_req > 0) {
    seg_len = seg_rows_req;
    nseg = (span + seg_len - 1) / seg_len;
  }
  const long long units = (long long)nstrips * nseg;
  int grid = (int)std::min<long long>(max_ctas / cl, units) * cl;
  if (grid < cl) grid = cl;
  const bool coop = coop_req && di.coop && epochs > 1;
  TbLaunch L{};
  L.n0 = n0;
  L.n1 = n1;
  L.nstrips = nstrips;
  L.nseg = nseg;
  L.seg_len = seg_len;
  L.z_lo = p.z_lo;
  L.z_hi = p.z_hi;
  L.aligned = aligned;
  L.pitch = (int)(p.pitch ? p.pitch : p.ext[1]);
  for (int i = 0; i < 3; ++i) L.buf[i] = bufs[i];
  L.maps = maps;
  L.coeffs = p.coeffs;
  L.grid = grid;
  L.stream = st;
  L.cluster = cl;
  int* work = nullptr;
  if (int rc = alloc_work(epochs, st, &work)) return rc;
  if (coop) {
    L.epochs = epochs;
    L.first_src = first_src;
    L.first_dst = first_dst;
    L.cooperative = true;
    L.work = work;
    EB_CUDA(k->launch(L));
    ctr->launches += 1;
    ctr->syncs_device += (uint64_t)(epochs - 1);
  } else {
    int src = first_src, dst = first_dst;
    for (int e = 0; e < epochs; ++e) {
      L.epochs = 1;
      L.first_src = src;
      L.first_dst = dst;
      L.cooperative = false;
      L.work = work + e;
      EB_CUDA(k->launch(L));
      ctr->launches += 1;
      src = dst;
      dst = (dst == BUF_OUT) ? BUF_SCR : BUF_OUT;
    }
  }
  cudaFreeAsync(work, st);
  // closed-form counters: every advance loads one row per warp; halo traffic
  // = 2R edge values per produced row per warp and level (shared memory and,
  // across the cluster seams, DSMEM)
  uint64_t adv = 0;
  const int Wr = Z + R + 1;
  for (int g = 0; g < nseg; ++g) {
    const int r0 = p.z_lo + g * seg_len, r1 = std::min(p.z_hi, r0 + seg_len);
    const int ka = std::max(0, r0 - T * R);
    adv += (uint64_t)((r1 + T * Z - ka + Wr - 1) / Wr * Wr);
  }
  const uint64_t cols = (uint64_t)LW * cl * nstrips;
  ctr->gm_loads += (uint64_t)epochs * adv * cols;
  ctr->gm_stores += (uint64_t)epochs * (uint64_t)span * (uint64_t)n1;
  ctr->cells_computed += (uint64_t)epochs * adv * (uint64_t)T * cols;
  ctr->halo_stores += (uint64_t)epochs * adv * (uint64_t)T * 2ull * R * k->NW * cl * nstrips;
  ctr->halo_loads += (uint64_t)epochs * adv * (uint64_t)T * 2ull * R * k->NW * cl * nstrips;
  ctr->syncs_block += (uint64_t)epochs * adv * (uint64_t)nstrips * cl;
  ctr->device_tiles += (uint64_t)epochs * (uint64_t)units;
  ctr->grid = grid;
  ctr->nw = k->NW;
  ctr->cluster = cl;
  ctr->t_used = std::max(ctr->t_used, T);
  if (ctr->arith < 0) ctr->arith = arith_of(k);
  if (ctr->kid == KID_NONE) ctr->kid = KID_HALO2D;
  return EBISU_OK;
}

int run_tb3d_stage(const ProblemDesc& p, const TbKernel* k, int epochs, int first_src,
                   int first_dst, void* bufs[3], const CUtensorMap maps[3], bool coop_req,
                   int seg_rows_req, const DevInfo& di, cudaStream_t st, Counters* ctr) {
  const int n0 = (int)p.ext[0], n1 = (int)p.ext[1], n2 = (int)p.ext[2];
  const int T = k->T, R = p.rad;
  int per_sm = 0;
  EB_CUDA(cudaFuncSetAttribute(k->func, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               k->smem_bytes));
  EB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k->func, k->NW * 32,
                                                        (size_t)k->smem_bytes));
  if (per_sm < 1) return fail(EBISU_ERR_CUDA, "stream3d kernel cannot be resident (T=%d)", T);
  int max_ctas = per_sm * di.sms;
  const int cl = k->cluster;  // CTAs per tile (2: cluster pair along axis 1)
  if (cl > 1) {
    int nclusters = 0;
    EB_CUDA(k->max_clusters(&nclusters));
    if (nclusters < 1) return fail(EBISU_ERR_CUDA, "cluster kernel cannot be resident (T=%d)", T);
    max_ctas = std::min(nclusters * cl, std::max(cl, max_ctas / cl * cl));  // (reserve_sms)
  }
  // edge-aligned tiles when two fit along an axis (stream2d_strip geometry)
  auto tiles_along = [](int n, int L, int V, int* aligned, int AL) {
    if (n >= 2 * L) {
      *aligned = 1;
      const int mid = strip_last_x0(n, L, AL) - V;
      return 2 + (mid > 0 ? (mid + V - 1) / V : 0);
    }
    *aligned = 0;
    return (n + V - 1) / V;
  };
  int aligned_x = 0, aligned_y = 0;
  const int ntx = tiles_along(n2, k->box0, k->valid_x, &aligned_x, 16 / p.elem);
  const int nty = tiles_along(n1, k->box1 * cl, k->valid_y, &aligned_y, 1);
  const long long tiles = (long long)ntx * nty;
  const int span = p.z_hi - p.z_lo;  // output planes of this call
  int nseg = 1, seg_len = span;
  plan_segments(span, tiles, max_ctas / cl, 3 * T * R, std::max(8, 2 * T * R), &nseg, &seg_len);
  // (never below 4x the per-unit warm-up, which short segments pay in full;
  // EBISU_SEG3D=uniform: the balanced uniform length, for A/B measurement)
  const char* seg_mode = getenv("EBISU_SEG3D");
  const bool uniform = seg_mode && strcmp(seg_mode, "uniform") == 0;
  int min_len = std::max(std::max(8, 2 * T * R), 4 * (T * R + T * k->z));
  if (const char* v = getenv("EBISU_SEGMIN3D")) min_len = std::max(8, atoi(v));  // tuning
  const std::vector<int> seg_start =
      guided_segments(p.z_lo, p.z_hi, tiles, max_ctas / cl, seg_len,
                      uniform ? std::max(seg_len, min_len) : min_len,
                      (uniform && seg_rows_req <= 0) ? std::max(seg_len, min_len) : seg_rows_req);
  nseg = (int)seg_start.size() - 1;
  const long long units = tiles * nseg;
  int grid = (int)std::min<long long>(max_ctas, units * cl);
  if (grid < cl) grid = cl;
  const bool coop = coop_req && di.coop && epochs > 1;
  TbLaunch L{};
  L.n0 = n0;
  L.n1 = n1;
  L.n2 = n2;
  L.pitch = (int)(p.pitch ? p.pitch : p.ext[2]);
  L.ntx = ntx;
  L.nty = nty;
  L.aligned_x = aligned_x;
  L.aligned_y = aligned_y;
  L.nseg = nseg;
  L.seg_len = seg_len;
  L.seg_start = seg_start.data();
  for (int i = 0; i < 3; ++i) L.buf[i] = bufs[i];
  L.maps = maps;
  L.coeffs = p.coeffs;
  L.grid = grid;
  L.stream = st;
  int* work = nullptr;
  if (int rc = alloc_work(epochs, st, &work)) return rc;
  if (coop) {
    L.epochs = epochs;
    L.first_src = first_src;
    L.first_dst = first_dst;
    L.cooperative = true;
    L.work = work;
    EB_CUDA(k->launch(L));
    ctr->launches += 1;
    ctr->syncs_device += (uint64_t)(epochs - 1);
  } else {
    int src = first_src, dst = first_dst;
    for (int e = 0; e < epochs; ++e) {
      L.epochs = 1;
      L.first_src = src;
      L.first_dst = dst;
      L.cooperative = false;
      L.work = work + e;
      EB_CUDA(k->launch(L));
      ctr->launches += 1;
      src = dst;
      dst = (dst == BUF_OUT) ? BUF_SCR : BUF_OUT;
    }
  }
  cudaFreeAsync(work, st);
  uint64_t loads = 0, adv = 0;
  const int WN = k->wn;
  for (int g = 0; g < nseg; ++g) {
    const int r0 = seg_start[g], r1 = seg_start[g + 1];
    const int ka = std::max(0, r0 - T * R);
    const int n = stream3d_advances_host(ka, r1, T * k->z, WN);
    loads += (uint64_t)n;  // every advance loads one plane (TMA zero-fills past n0)
    adv += (uint64_t)n;
  }
  ctr->cluster = std::max(ctr->cluster, cl);
  const uint64_t tile_cells = (uint64_t)k->box0 * (uint64_t)k->box1 * (uint64_t)cl;
  ctr->gm_loads += (uint64_t)epochs * loads * tile_cells * (uint64_t)ntx * nty;
  ctr->gm_stores += (uint64_t)epochs * (uint64_t)span * n1 * n2;
  ctr->cells_computed += (uint64_t)epochs * adv * (uint64_t)T * tile_cells * (uint64_t)ntx * nty;
  ctr->device_tiles += (uint64_t)epochs * (uint64_t)units;
  ctr->syncs_block += (uint64_t)epochs * adv * (uint64_t)ntx * nty * (uint64_t)cl;
  ctr->grid = grid;
  ctr->nw = k->NW;
  ctr->t_used = std::max(ctr->t_used, T);
  if (ctr->arith < 0) ctr->arith = arith_of(k);
  if (ctr->kid == KID_NONE) ctr->kid = KID_STREAM3D;
  return EBISU_OK;
}

// ---- resident-tile kernel (any tap set): tile shape and depth ----------------
// Tile-shape cost model in SM clocks (the grid's tiles spread over all SMs):
//   compute  per level: the level's region x (ntaps loads + 1 store) x elem /
//            128 B/clk of shared memory / kSmemEff, plus kLevelLatency
//   HBM      (loaded + core) x elem / kHbmBytesPerClkSm + kTileLatency,
//            overlapped with the other CTA's compute at 2 CTAs per SM
// (B200: 7.7 TB/s / 148 SMs / 1.9 GHz ~ 27 B/clk; 23 sustained.)
constexpr double kHbmBytesPerClkSm = 23.0;
constexpr double kSmemEff = 0.45;      // measured share of the shared-memory rate
constexpr double kTileLatency = 2500;  // clocks: tile load round trip + store drain
constexpr double kLevelLatency = 300;  // clocks: per-level barrier and pipeline drain
constexpr int kGenSmemBytes = 227 * 1024;

// resident CTAs per SM (EBISU_GEN_CTAS, measurement knob): 1 = one 227 KB
// tile per SM, 2 = two half-size tiles whose load and compute phases overlap
int gen_ctas_per_sm() {
  static const int v = [] {
    const char* e = getenv("EBISU_GEN_CTAS");
    const int n = e ? atoi(e) : 2;
    return n == 1 ? 1 : 2;
  }();
  return v;
}

struct GenPlan {
  GenArgs a;
  double clk_per_cell_step;  // whole-GPU estimate (all SMs)
  int grid;
  int smem;
  int threads;
};

bool gen_plan(const ProblemDesc& p, int T, int sms, GenPlan* out) {
  const int D = p.dims, R = p.rad;
  if (T < 1 || T > EBISU_GEN_MAXT) return false;
  GenArgs a;
  memset(&a, 0, sizeof(a));
  for (int ax = 0; ax < 3; ++ax) a.ext[ax] = 1;
  for (int d = 0; d < D; ++d) a.ext[3 - D + d] = p.ext[d];
  a.pitch = p.pitch ? p.pitch : p.ext[D - 1];
  a.zaxis = 3 - D;
  a.z_lo = p.z_lo;
  a.z_hi = p.z_hi;
  a.T = T;
  long long span[3];
  for (int ax = 0; ax < 3; ++ax) {
    const bool present = ax >= 3 - D;
    a.H[ax] = present ? T * R : 0;
    a.RA[ax] = present ? R : 0;
    a.F[ax] = present ? R : 0;
    span[ax] = ax == a.zaxis ? (long long)(p.z_hi - p.z_lo) : a.ext[ax];
  }
  // per-CTA budget: 228 KB per SM less 1 KB reserved per resident CTA
  const long long budget = std::min(kGenSmemBytes, 228 * 1024 / gen_ctas_per_sm() - 1024);
  const long long cap = budget / (2 * p.elem) - 128;  // + 128 pad elements per buffer
  static const int cand[] = {16, 24, 32, 48, 64, 96, 128, 160, 192, 256, 320, 384, 512,
                             768, 1024, 1536, 2048, 4096, 8192, 16384, 32768};
  // candidate extents of one axis: the list plus "whole span", <= limit
  auto axis_cands = [&](int ax, long long limit, std::vector<int>& v) {
    v.clear();
    const long long whole = span[ax] + 2LL * a.H[ax];
    for (int c : cand)
      if (c > 2 * a.H[ax] && c < whole && c <= limit) v.push_back(c);
    if (whole <= limit) v.push_back((int)whole);
    if (v.empty() && limit > 2 * a.H[ax] && limit < whole) v.push_back((int)limit);
  };
  // measured: the kernel sustains ~45 % of the shared-memory rate (1-D j1d3pt
  // t=16 499 GCells/s, 2-D j2d5pt-order-reversed t=8 273 GCells/s)
  const double per_cell_smem = (double)(p.ntaps + 1) * p.elem / 128.0 / kSmemEff;
  double best = 1e300;
  GenArgs bestA = a;
  std::vector<int> c2, c1, c0;
  axis_cands(2, cap, c2);
  for (int L2 : c2) {
    axis_cands(1, cap / L2, c1);
    if (D < 2) c1.assign(1, 1);
    for (int L1 : c1) {
      if ((long long)L1 * L2 > cap) continue;
      long long lim0 = cap / ((long long)L1 * L2);
      int L0;
      if (D < 3) {
        L0 = 1;
      } else {
        L0 = (int)std::min<long long>(lim0, span[0] + 2LL * a.H[0]);
        if (L0 <= 2 * a.H[0]) continue;
      }
      const int L[3] = {L0, L1, L2};
      int V[3];
      long long nt[3];
      bool ok = true;
      for (int ax = 0; ax < 3; ++ax) {
        V[ax] = L[ax] - 2 * a.H[ax];
        if (V[ax] <= 0) ok = false;
        nt[ax] = ok ? (span[ax] + V[ax] - 1) / V[ax] : 0;
      }
      if (!ok) continue;
      double comp = 0;
      for (int s = 1; s <= T; ++s) {
        const long long w0 = L0 - 2LL * s * a.RA[0], w1 = L1 - 2LL * s * a.RA[1];
        const long long w2 = L2 - 2LL * s * a.RA[2];
        comp += (double)(w0 * w1) * (double)((w2 + 127) / 128 * 128) * per_cell_smem;
      }
      const double cells_l = (double)L0 * L1 * L2, cells_v = (double)V[0] * V[1] * V[2];
      // HBM bytes plus the exposed load round trip (~kTileLatency clocks)
      const double mem = (cells_l + cells_v) * p.elem / kHbmBytesPerClkSm + kTileLatency;
      comp += T * kLevelLatency;  // barrier + pipeline drain per level
      const long long ntiles = nt[0] * nt[1] * nt[2];
      if (ntiles > (1LL << 31)) continue;
      const int cps = gen_ctas_per_sm();
      const double waves = std::ceil((double)ntiles / (sms * cps)) * cps;
      // two CTAs per SM overlap one tile's HBM phase with the other's compute
      const double total = cps > 1 ? waves / cps * std::max(2 * comp, comp + mem)
                                   : waves * (comp + mem);
      const double cells = (double)span[0] * span[1] * span[2] * T;
      const double cost = total / cells;
      if (cost < best) {
        best = cost;
        for (int ax = 0; ax < 3; ++ax) {
          bestA.L[ax] = L[ax];
          bestA.V[ax] = V[ax];
          bestA.nt[ax] = (int)nt[ax];
        }
      }
    }
  }
  if (best >= 1e300) return false;
  a = bestA;
  a.ntaps = p.ntaps;
  for (int lv = 1; lv <= T; ++lv) {  // the kernel's per-level row/chunk divisors
    const int w1 = a.L[1] - 2 * lv * a.RA[1], w2 = a.L[2] - 2 * lv * a.RA[2];
    a.lvl_cpr[lv - 1] = gen_div((uint32_t)std::max(1, (w2 + 127) / 128));
    a.lvl_w1[lv - 1] = gen_div((uint32_t)std::max(1, w1));
  }
  for (int k = 0; k < p.ntaps; ++k) {
    const int* o = p.offsets + k * D;
    int off[3] = {0, 0, 0};
    for (int d = 0; d < D; ++d) off[3 - D + d] = o[d];
    a.lin[k] = (off[0] * a.L[1] + off[1]) * a.L[2] + off[2];
    a.coef[k] = p.coeffs[k];
  }
  out->a = a;
  out->clk_per_cell_step = best;
  const long long ntiles = (long long)a.nt[0] * a.nt[1] * a.nt[2];
  out->grid = (int)std::min<long long>(ntiles, (long long)sms * gen_ctas_per_sm());
  out->smem = 2 * (a.L[0] * a.L[1] * a.L[2] + 128) * p.elem;  // kGenPad per buffer
  out->threads = generic_threads() / gen_ctas_per_sm();
  return true;
}

// Depth for the resident-tile kernel: the requested one (else the deepest
// below it that fits); AUTO uses the kernel only where it measured faster than
// one launch per step.  Measured on B200 (tools/gen_bench.py, 64 steps):
//   1-D j1d3pt 2^25 cells   resident t=16 539 GCells/s vs naive 364
//   2-D 8192^2, 5/9/13 taps resident t=8 273/208/131 vs naive 338/287/215
//   3-D 512^3, 7/27 taps    resident t=2 84/50 vs naive 182/84
// (the kernel sustains ~45 % of the shared-memory rate with runtime taps:
// no register reuse between taps).  Forced (scheme RESIDENT) without a depth:
// the measured-best depth per dimensionality.
int gen_pick_depth(const ProblemDesc& p, int t_req, int sms, bool forced) {
  if (!forced && p.dims >= 2) return 0;  // 2-D/3-D: one launch per step is faster
  int want = std::min(t_req, EBISU_GEN_MAXT);
  if (want <= 0) want = p.dims == 1 ? 16 : (p.dims == 2 ? 8 : 2);
  for (int T = want; T >= 1; --T) {
    GenPlan g;
    if (gen_plan(p, T, sms, &g)) return T;
  }
  return 0;
}

int run_generic_stage(const ProblemDesc& p, int T, int epochs, int first_src, int first_dst,
                      void* bufs[3], bool exact, const DevInfo& di, cudaStream_t st,
                      Counters* ctr) {
  GenPlan g;
  if (!gen_plan(p, T, di.sms, &g))
    return fail(EBISU_ERR_UNSUPPORTED, "no resident tile fits depth %d at radius %d", T, p.rad);
  int src = first_src, dst = first_dst;
  for (int e = 0; e < epochs; ++e) {
    g.a.in = bufs[src];
    g.a.out = bufs[dst];
    EB_CUDA(launch_generic_tb(g.a, p.elem, exact, g.grid, g.threads, g.smem, st));
    ctr->launches += 1;
    src = dst;
    dst = (dst == BUF_OUT) ? BUF_SCR : BUF_OUT;
  }
  // closed-form counters
  const GenArgs& a = g.a;
  const uint64_t ntiles = (uint64_t)a.nt[0] * a.nt[1] * a.nt[2];
  uint64_t comp = 0;
  for (int s = 1; s <= T; ++s)
    comp += (uint64_t)(a.L[0] - 2 * s * a.RA[0]) * (uint64_t)(a.L[1] - 2 * s * a.RA[1]) *
            (uint64_t)(a.L[2] - 2 * s * a.RA[2]);
  uint64_t span = 1;
  for (int ax = 0; ax < 3; ++ax)
    span *= (uint64_t)(ax == a.zaxis ? (a.z_hi - a.z_lo) : a.ext[ax]);
  ctr->gm_loads += (uint64_t)epochs * ntiles * (uint64_t)a.L[0] * a.L[1] * a.L[2];
  ctr->gm_stores += (uint64_t)epochs * span;
  ctr->cells_computed += (uint64_t)epochs * ntiles * comp;
  ctr->device_tiles += (uint64_t)epochs * ntiles;
  ctr->syncs_block += (uint64_t)epochs * ntiles * (uint64_t)(T + 2);
  ctr->grid = g.grid;
  ctr->nw = g.threads / 32;
  ctr->t_used = std::max(ctr->t_used, T);
  if (ctr->arith < 0) ctr->arith = exact ? EBISU_ARITH_PER_TAP_EXACT : EBISU_ARITH_PER_TAP_FMA;
  if (ctr->kid == KID_NONE) ctr->kid = KID_GENERIC;
  return EBISU_OK;
}

// ---- one-step 3-D streaming for any tap set (k_generic_s3d) -------------------
// Plan: 128 x 16 output tiles (64-wide when the ring would not fit), z
// segments so that every resident CTA has units (>= 4 (2R+1) planes each: the
// 2R-plane prologue is the per-unit overhead); false when no tile fits.
constexpr int kS3DPrefetch = 1;  // = kGenS3DPrefetch (ebisu_generic.cu)
constexpr int kS3DTileY = 16;
bool s3d_plan(const ProblemDesc& p, int sms, GenS3DArgs* a, int* grid, int* smem) {
  if (p.dims != 3) return false;
  const int R = p.rad;
  memset(a, 0, sizeof(*a));
  a->R = R;
  a->LY = kS3DTileY;
  a->LX = 128;
  auto bytes = [&](int ly, int lx) {  // 2R+1 planes + kS3DPrefetch in flight
    return (2 * R + 1 + kS3DPrefetch) * (ly + 2 * R) * (lx + 2 * R) * p.elem;
  };
  if (bytes(a->LY, a->LX) > kGenSmemBytes) a->LX = 64;
  if (bytes(a->LY, a->LX) > kGenSmemBytes) return false;
  *smem = bytes(a->LY, a->LX);
  a->n0 = p.ext[0];
  a->n1 = p.ext[1];
  a->n2 = p.ext[2];
  a->pitch = p.pitch ? p.pitch : p.ext[2];
  a->z_lo = p.z_lo;
  a->z_hi = p.z_hi;
  a->nty = (int)((p.ext[1] + a->LY - 1) / a->LY);
  a->ntx = (int)((p.ext[2] + a->LX - 1) / a->LX);
  const long long tiles = (long long)a->nty * a->ntx;
  const int per_sm = std::max(1, 228 * 1024 / (*smem + 1024));
  const long long slots = (long long)sms * std::min(per_sm, 8);
  const long long span = p.z_hi - p.z_lo;
  long long nseg = std::max<long long>(1, (2 * slots + tiles - 1) / tiles);
  const long long min_len = 4LL * (2 * R + 1);
  nseg = std::min(nseg, std::max<long long>(1, span / min_len));
  a->seg_len = (int)((span + nseg - 1) / nseg);
  a->nseg = (int)((span + a->seg_len - 1) / a->seg_len);
  const long long units = tiles * a->nseg;
  *grid = (int)std::min<long long>(units, slots);
  a->ntaps = p.ntaps;
  const int PX = a->LX + 2 * R;
  for (int k = 0; k < p.ntaps; ++k) {
    const int* o = p.offsets + 3 * k;
    a->dz[k] = o[0];
    a->lin[k] = o[1] * PX + o[2];
    a->coef[k] = p.coeffs[k];
  }
  return true;
}

int run_device_impl(const ProblemDesc& p0, const void* d_in, void* d_out, void* d_scr,
                    long long steps, const ebisu_params* prm, cudaStream_t st, Counters* ctr) {
  ProblemDesc p = p0;
  const bool ranged = prm && prm->out_planes[1] > 0;
  p.z_lo = ranged ? prm->out_planes[0] : 0;
  p.z_hi = ranged ? prm->out_planes[1] : (int)p.ext[0];
  DevInfo di;
  int rc = device_info(&di);
  if (rc) return rc;
  // SMs left free for concurrent kernels on other streams (at least one SM
  // stays with the sweep)
  if (prm && prm->reserve_sms > 0) di.sms = std::max(1, di.sms - prm->reserve_sms);
  const long long total = p.ext[0] * p.ext[1] * p.ext[2];
  const size_t bytes = (size_t)total * (size_t)p.elem;
  if (steps == 0) {
    if (d_out != d_in) EB_CUDA(cudaMemcpyAsync(d_out, d_in, bytes, cudaMemcpyDeviceToDevice, st));
    return EBISU_OK;
  }
  const bool exact = prm ? prm->exact != 0 : true;
  const int scheme = prm ? prm->scheme : EBISU_SCHEME_AUTO;
  const bool coop = prm ? prm->persistent != 0 : true;

  // ---- plan the stage list ----------------------------------------------------
  std::vector<Stage> stages;
  const int D = p.dims;
  const bool uni = uniform_coeffs(p) && !(prm && prm->per_tap_products);
  // TMA needs 16-byte row strides (last extent a multiple of 16 bytes) and
  // 16-byte aligned bases.  Otherwise the TB kernels run on row-padded copies
  // (pitch rounded up to 16 bytes; TMA maps keep the true extent, so the pad
  // is never read): one strided copy in, one out -- two grid passes per sweep
  // instead of falling back to one-launch-per-step.
  const bool force_gen = scheme == EBISU_SCHEME_RESIDENT;
  const bool tb_shape = (D == 2 || D == 3) && p.shape_id != SHAPE_GENERIC &&
                        scheme != EBISU_SCHEME_NAIVE && !force_gen;
  const bool tma_direct = ((p.ext[D - 1] * p.elem) % 16 == 0) &&
                          (reinterpret_cast<uintptr_t>(d_in) % 16 == 0) &&
                          (reinterpret_cast<uintptr_t>(d_out) % 16 == 0) &&
                          (!d_scr || reinterpret_cast<uintptr_t>(d_scr) % 16 == 0);
  bool pitched = tb_shape && !tma_direct && !ranged && !(prm && prm->frame_ready);
  bool tb_ok = tb_shape && (tma_direct || pitched);
  if (tb_ok) {
    int t = (prm && prm->t > 0) ? prm->t : default_depth(p.shape_id);
    if (!(prm && prm->t > 0) && uni && !exact) t = default_depth_tol(p.shape_id, t);
    // fp32 windows cost half the registers: the 2-D star runs deeper
    if (!(prm && prm->t > 0) && p.elem == 4 && p.shape_id == SHAPE_J2D5PT) t = 16;
    const int want_c = prm ? prm->lane_cells : 0;
    const int want_v = prm ? prm->variant : 0;
    int fam = pick_family(scheme, p.shape_id, D);
    // no halo-exchange instantiation for this stencil/arithmetic: the
    // overlapped kernels compute the identical result
    if (fam == 1 && best_depth_leq(p.shape_id, D, 64, exact, uni, 1, p.elem) == 0) fam = 0;
    const TbKernel* k = find_tb(p.shape_id, D, t, exact, uni, fam, p.elem, want_c, want_v);
    // 3-D device tiles of several CTAs (device_tile_grid[0] >= 2 along axis
    // 1): the 2-CTA cluster tile exchanging its seam rows through DSMEM
    // (ebisu_stream3d_cl.cuh; engine/device.py:292-389's multi-block streamed
    // tile), where one is instantiated for this stencil and depth
    if (D == 3 && scheme == EBISU_SCHEME_DEVICE_TILING && !want_c && !want_v && prm &&
        prm->device_tile_grid[0] >= 2) {
      int nk = 0;
      const TbKernel* ks = tb_kernels(&nk);
      for (int i = 0; i < nk; ++i)
        if (ks[i].cluster == 2 && ks[i].shape_id == p.shape_id && ks[i].dims == 3 &&
            ks[i].T == t && family_ok(ks[i], exact, uni, 0, p.elem)) {
          k = &ks[i];
          break;
        }
    }
    if (!k && (want_c || want_v))
      return fail(EBISU_ERR_UNSUPPORTED, "no kernel with depth %d, %d cells per lane, variant %d",
                  t, want_c, want_v);
    if (!k && fam == 1) {
      // no halo-exchange kernel of this depth: the overlapped kernel of the
      // same depth computes the identical result
      const TbKernel* k0 = find_tb(p.shape_id, D, t, exact, uni, 0, p.elem);
      if (k0 && best_depth_leq(p.shape_id, D, t, exact, uni, 1, p.elem) == 0) {
        fam = 0;
        k = k0;
      }
    }
    if (!k) {
      // depth not instantiated: compose the sweep from the deepest kernel
      // below it (epochs compose bitwise, test_grid.py:94-117)
      t = best_depth_leq(p.shape_id, D, t, exact, uni, fam, p.elem);
      k = t ? find_tb(p.shape_id, D, t, exact, uni, fam, p.elem) : nullptr;
    }
    if (!k) {
      tb_ok = false;
    } else {
      long long full = steps / t;
      long long rem = steps % t;
      const int kid = D == 3 ? KID_STREAM3D : (fam == 1 ? KID_HALO2D : KID_STREAM2D);
      if (full > 0) stages.push_back({kid, k, (int)full});
      while (rem > 0) {
        // remainder epochs: the deepest kernel <= rem of this family, else of
        // the overlapped family (identical results), else the naive kernel
        int f2 = fam;
        int t2 = best_depth_leq(p.shape_id, D, (int)rem, exact, uni, f2, p.elem);
        if (t2 == 0 && fam != 0) {
          f2 = 0;
          t2 = best_depth_leq(p.shape_id, D, (int)rem, exact, uni, f2, p.elem);
        }
        if (t2 == 0) {
          stages.push_back({KID_NAIVE, nullptr, (int)rem});
          break;
        }
        const long long e2 = rem / t2;
        const int kid2 = D == 3 ? KID_STREAM3D : (f2 == 1 ? KID_HALO2D : KID_STREAM2D);
        stages.push_back({kid2, find_tb(p.shape_id, D, t2, exact, uni, f2, p.elem), (int)e2});
        rem -= e2 * t2;
      }
    }
  }
  // a padded sweep is all-TB (the naive kernel works on the caller's layout)
  if (pitched)
    for (auto& s : stages) tb_ok = tb_ok && s.kind != KID_NAIVE;
  if (!tb_ok) {
    // no specialised kernel (1-D, user tap sets, or forced): the resident-tile
    // kernel for any tap set when its cost model beats one launch per step
    pitched = false;
    stages.clear();
    const int tg = scheme == EBISU_SCHEME_NAIVE
                       ? 0
                       : gen_pick_depth(p, (prm && prm->t > 0) ? prm->t : 0, di.sms, force_gen);
    if (tg > 0) {
      const long long full = steps / tg, rem = steps % tg;
      if (full > 0) stages.push_back({KID_GENERIC, nullptr, (int)full, tg});
      if (rem > 0) stages.push_back({KID_GENERIC, nullptr, 1, (int)rem});
    } else {
      stages.push_back({KID_NAIVE, nullptr, (int)steps});
    }
  }

  // ---- buffers: every stage writes a full grid (frame included) -----------------
  long long nwrites = 0;  // number of grid writes
  for (auto& s : stages) nwrites += s.epochs;
  if (ranged && nwrites != 1)
    return fail(EBISU_ERR_PARAM,
                "output-plane range needs a single fused epoch (steps <= t with a kernel of "
                "that depth), got %lld writes",
                nwrites);
  void* scr = d_scr;
  bool own_scr = false;
  void* pad[3] = {nullptr, nullptr, nullptr};  // padded in / out / scratch
  const long long Xn = p.ext[D - 1];
  const long long rows = total / Xn;
  if (pitched) {
    const long long al = 16 / p.elem;
    p.pitch = (Xn + al - 1) / al * al;
    const size_t pbytes = (size_t)(rows * p.pitch) * (size_t)p.elem;
    for (int b = 0; b < 3; ++b) {
      if (b == BUF_SCR && nwrites <= 1) continue;
      cudaError_t e = cudaMallocAsync(&pad[b], pbytes, st);
      if (e != cudaSuccess) {
        for (int j = 0; j < b; ++j)
          if (pad[j]) cudaFreeAsync(pad[j], st);
        return cuda_fail(e, "cudaMallocAsync(padded buffer)");
      }
    }
    cudaError_t e = cudaMemcpy2DAsync(pad[BUF_IN], (size_t)(p.pitch * p.elem), d_in,
                                      (size_t)(Xn * p.elem), (size_t)(Xn * p.elem), (size_t)rows,
                                      cudaMemcpyDeviceToDevice, st);
    if (e != cudaSuccess) {
      for (void* q : pad)
        if (q) cudaFreeAsync(q, st);
      return cuda_fail(e, "padded input copy");
    }
  } else if (nwrites > 1 && !scr) {
    EB_CUDA(cudaMallocAsync(&scr, bytes, st));
    own_scr = true;
  }
  void* bufs[3] = {const_cast<void*>(d_in), d_out, scr};
  if (pitched)
    for (int b = 0; b < 3; ++b) bufs[b] = pad[b];
  CUtensorMap maps[3];
  // Shared-product kernels never store frame cells (their windows hold
  // products, not values); the frame is constant, so copy it once into both
  // ping-pong buffers (a shell of 2R planes/rows/columns, not the grid).
  bool any_uni = false;
  for (auto& s : stages) any_uni = any_uni || (s.k && s.k->uni);
  if (any_uni) {
    for (int b = BUF_OUT; b <= BUF_SCR; ++b) {
      if (!bufs[b]) continue;
      // frame_ready vouches for the caller's buffers only: scratch the
      // library just allocated holds no frame yet
      if (prm && prm->frame_ready && !(b == BUF_SCR && own_scr)) continue;
      cudaError_t e = launch_frame_copy(p, bufs[BUF_IN], bufs[b], st, di.sms);
      if (e != cudaSuccess) {
        if (own_scr) cudaFreeAsync(scr, st);
        for (void* q : pad)
          if (q) cudaFreeAsync(q, st);
        return cuda_fail(e, "frame copy launch");
      }
      ctr->launches += 1;
    }
  }

  // write w (0-based) goes to OUT iff (nwrites-1-w) is even
  long long w = 0;
  int src = BUF_IN;
  int result = EBISU_OK;
  for (auto& s : stages) {
    const int dst = ((nwrites - 1 - w) % 2 == 0) ? BUF_OUT : BUF_SCR;
    if (s.kind == KID_NAIVE) {
      int cs = src, cd = dst;
      // 3-D steps without a temporal-blocking kernel (user tap sets,
      // remainders): the streaming one-step kernel unless the naive
      // yardstick was asked for
      GenS3DArgs sa;
      int s3_grid = 0, s3_smem = 0;
      const bool s3d = scheme != EBISU_SCHEME_NAIVE && s3d_plan(p, di.sms, &sa, &s3_grid, &s3_smem);
      for (int i = 0; i < s.epochs; ++i) {
        cudaError_t e;
        if (s3d) {
          sa.in = bufs[cs];
          sa.out = bufs[cd];
          e = launch_generic_s3d(sa, p.elem, exact, s3_grid, s3_smem, st);
        } else {
          e = launch_naive_step(p, bufs[cs], bufs[cd], exact, st, di.sms);
        }
        if (e != cudaSuccess) {
          result = cuda_fail(e, "naive step launch");
          break;
        }
        ctr->launches += 1;
        cs = cd;
        cd = (cd == BUF_OUT) ? BUF_SCR : BUF_OUT;
      }
      if (result) break;
      ctr->gm_loads += (uint64_t)s.epochs * (uint64_t)total;
      ctr->gm_stores += (uint64_t)s.epochs * (uint64_t)total;
      ctr->cells_computed += (uint64_t)s.epochs * (uint64_t)total;
      if (ctr->arith < 0) ctr->arith = exact ? EBISU_ARITH_PER_TAP_EXACT : EBISU_ARITH_PER_TAP_FMA;
      if (ctr->kid == KID_NONE) ctr->kid = s3d ? KID_GENERIC_S3D : KID_NAIVE;
      ctr->t_used = std::max(ctr->t_used, 1);
      src = (s.epochs % 2 == 1) ? dst : (dst == BUF_OUT ? BUF_SCR : BUF_OUT);
    } else if (s.kind == KID_GENERIC) {
      result = run_generic_stage(p, s.T, s.epochs, src, dst, bufs, exact, di, st, ctr);
      if (result) break;
      src = (s.epochs % 2 == 1) ? dst : (dst == BUF_OUT ? BUF_SCR : BUF_OUT);
    } else {
      {
        // 2-D: one 32*C-column row per TMA box; 3-D: one LY x LX tile plane
        const long long dims_ff[3] = {p.ext[D - 1], p.ext[D - 2], D == 3 ? p.ext[0] : 1};
        const int box[3] = {s.k->box0, s.k->box1, 1};
        for (int i = 0; i < 3 && !result; ++i) {
          if (!bufs[i]) {
            memset(&maps[i], 0, sizeof(CUtensorMap));
            continue;
          }
          result = encode_map(&maps[i], bufs[i], D, dims_ff, box, p.elem,
                              p.pitch ? p.pitch : p.ext[D - 1]);
        }
        if (result) break;
      }
      if (D == 2 && s.kind == KID_HALO2D)
        result = run_halo2d_stage(p, s.k, s.epochs, src, dst, bufs, maps, coop,
                                  prm ? prm->seg_rows : 0, prm ? prm->device_tile_grid[1] : 0,
                                  di, st, ctr);
      else if (D == 2)
        result = run_tb2d_stage(p, s.k, s.epochs, src, dst, bufs, maps, coop,
                                prm ? prm->seg_rows : 0, di, st, ctr);
      else
        result = run_tb3d_stage(p, s.k, s.epochs, src, dst, bufs, maps, coop,
                                prm ? prm->seg_rows : 0, di, st, ctr);
      if (result) break;
      src = (s.epochs % 2 == 1) ? dst : (dst == BUF_OUT ? BUF_SCR : BUF_OUT);
    }
    w += s.epochs;
  }
  if (own_scr) cudaFreeAsync(scr, st);
  if (pitched) {
    if (!result) {
      cudaError_t e = cudaMemcpy2DAsync(d_out, (size_t)(Xn * p.elem), pad[BUF_OUT],
                                        (size_t)(p.pitch * p.elem), (size_t)(Xn * p.elem),
                                        (size_t)rows, cudaMemcpyDeviceToDevice, st);
      if (e != cudaSuccess) result = cuda_fail(e, "padded output copy");
    }
    for (void* q : pad)
      if (q) cudaFreeAsync(q, st);
  }
  return result;
}

}  // namespace
}  // namespace ebisu

using namespace ebisu;

extern "C" {

int32_t ebisu_abi_version(void) { return EBISU_ABI_VERSION; }

const char* ebisu_last_error(void) { return g_err.c_str(); }

const char* ebisu_kernel_name(int32_t id) {
  switch (id) {
    case KID_NAIVE: return "naive_step";
    case KID_STREAM2D: return "stream2d_tb";
    case KID_STREAM3D: return "stream3d_tb";
    case KID_HALO2D: return "halo2d_tb";
    case KID_GENERIC: return "resident_tb";
    case KID_GENERIC_S3D: return "stream3d_step";
    default: return "none";
  }
}

int32_t ebisu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int32_t ebisu_check_compatible(const ebisu_stencil* stencil, int32_t ndim, const int64_t* extents,
                               const ebisu_params* params) {
  ProblemDesc p;
  g_err.clear();
  return validate(stencil, ndim, extents, params, &p);
}

static void fill_trace(ebisu_trace* tr, const ProblemDesc& p, long long steps, const Counters& c,
                       float ms) {
  if (!tr) return;
  memset(tr, 0, sizeof(*tr));
  long long interior = 1;
  for (int d = 0; d < p.dims; ++d) interior *= (p.ext[d] - 2 * p.rad);
  tr->gm_loads = c.gm_loads;
  tr->gm_stores = c.gm_stores;
  tr->gm_halo_loads = c.halo_loads;
  tr->gm_halo_stores = c.halo_stores;
  tr->syncs_device = c.syncs_device;
  tr->syncs_block = c.syncs_block;
  tr->cells_computed = c.cells_computed;
  tr->cells_valid = (uint64_t)interior * (uint64_t)steps;
  tr->device_tiles = c.device_tiles;
  tr->kernel_launches = c.launches;
  tr->elapsed_ms = ms;
  tr->kernel_id = c.kid;
  tr->t_used = c.t_used;
  tr->grid_ctas = c.grid;
  tr->warps_per_cta = c.nw;
  tr->cluster_ctas = c.cluster;
  tr->arith = c.arith < 0 ? EBISU_ARITH_SHARED_PRODUCTS : c.arith;
}

static int32_t run_device_entry(const ebisu_stencil* stencil, int32_t ndim,
                                const int64_t* extents, const void* d_in, void* d_out,
                                void* d_scratch, int64_t steps, const ebisu_params* params,
                                void* stream, ebisu_trace* trace, int elem) {
  g_err.clear();
  if (steps < 0) return fail(EBISU_ERR_VALUE, "step count must be >= 0");
  if (steps > INT32_MAX)
    return fail(EBISU_ERR_VALUE, "step count %lld exceeds 2^31-1", (long long)steps);
  ProblemDesc p;
  int rc = validate(stencil, ndim, extents, params, &p);
  if (rc) return rc;
  p.elem = elem;
  if (!d_in || !d_out) return fail(EBISU_ERR_VALUE, "null device buffer");
  if (d_in == d_out && steps > 0)
    return fail(EBISU_ERR_VALUE, "d_in and d_out must be distinct (the input is read only)");
  if (ebisu_device_count() == 0) return fail(EBISU_ERR_NO_DEVICE, "no CUDA device visible");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (trace) {
    EB_CUDA(cudaEventCreate(&e0));
    EB_CUDA(cudaEventCreate(&e1));
    EB_CUDA(cudaEventRecord(e0, st));
  }
  Counters c;
  rc = run_device_impl(p, d_in, d_out, d_scratch, steps, params, st, &c);
  float ms = 0.f;
  if (trace) {
    if (!rc) {
      cudaError_t e = cudaEventRecord(e1, st);
      if (e == cudaSuccess) e = cudaEventSynchronize(e1);
      if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
      if (e != cudaSuccess) rc = cuda_fail(e, "timing events");
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  }
  if (!rc) fill_trace(trace, p, steps, c, ms);
  return rc;
}

// ---- pageable host buffers: staged copies ---------------------------------------
// The drop-in reference_run hands over pageable numpy arrays.  The driver's
// pageable copies run single-threaded through its own bounce buffer, and a
// fresh output array takes its page faults inside the D2H copy (measured:
// 512 MiB H2D 48 ms, D2H 30 ms prefaulted / ~120 ms fresh, vs 10 + 10 ms
// pinned).  Instead: a process-wide ring of pinned slots (256 MiB); host threads
// copy chunks between the caller's array and the slots (faulting fresh pages
// in parallel) while the DMA engine moves the previous group of slots.
namespace staging {
constexpr size_t kRingBytes = 256u << 20;  // pinned ring: 2K slots of kRingBytes/(2K)
struct Pool {
  std::mutex mu;  // one staged transfer at a time (concurrent calls queue here)
  std::vector<void*> slots;
  std::vector<cudaEvent_t> done;
  int dev = -1;
};
Pool& pool() {
  static Pool p;
  return p;
}
int threads() {
  static const int n = [] {
    if (const char* e = getenv("EBISU_STAGING_THREADS")) {  // measurement knob
      const int v = atoi(e);
      if (v >= 1 && v <= 64) return v;
    }
    // one copy thread per host core, up to 16 (512 MiB each way, fresh
    // output: 8 threads 87 ms per 8192^2 reference_run call, 16 threads 82)
    const unsigned hw = std::thread::hardware_concurrency();
    return (int)std::max(2u, std::min(16u, hw ? hw : 2u));
  }();
  return n;
}
size_t chunk_bytes() { return kRingBytes / (2 * (size_t)threads()); }
bool pageable(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return true;
  }
  return a.type == cudaMemoryTypeUnregistered;
}
// (caller holds the pool lock) ensure 2*K pinned slots on the current device
cudaError_t ensure(Pool& P, int K) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (P.dev != dev) {
    for (void* q : P.slots) cudaFreeHost(q);
    for (cudaEvent_t ev : P.done) cudaEventDestroy(ev);
    P.slots.clear();
    P.done.clear();
    P.dev = dev;
  }
  while ((int)P.slots.size() < 2 * K) {
    void* q = nullptr;
    cudaEvent_t ev;
    if ((e = cudaMallocHost(&q, chunk_bytes())) != cudaSuccess) return e;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) {
      cudaFreeHost(q);
      return e;
    }
    P.slots.push_back(q);
    P.done.push_back(ev);
  }
  return cudaSuccess;
}
// parallel memcpy of up to K (dst, src, len) jobs; no exception crosses the
// C ABI: a job whose thread cannot be created runs on the calling thread
void par_copy(const std::vector<std::array<size_t, 3>>& jobs) {
  auto run = [&jobs](size_t i) {
    memcpy((void*)jobs[i][0], (const void*)jobs[i][1], jobs[i][2]);
  };
  std::vector<std::thread> th;
  for (size_t i = 1; i < jobs.size(); ++i) {
    try {
      th.emplace_back(run, i);
    } catch (...) {
      run(i);
    }
  }
  if (!jobs.empty()) run(0);
  for (auto& t : th) t.join();
}
// free the pinned slots (ebisu_release_scratch)
void release() {
  Pool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  for (cudaEvent_t ev : P.done) cudaEventSynchronize(ev);
  for (void* q : P.slots) cudaFreeHost(q);
  for (cudaEvent_t ev : P.done) cudaEventDestroy(ev);
  P.slots.clear();
  P.done.clear();
  P.dev = -1;
}
cudaError_t h2d(void* d, const void* h, size_t bytes, cudaStream_t st) {
  Pool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  const int K = threads();
  cudaError_t e = ensure(P, K);
  if (e != cudaSuccess) return e;
  const size_t kChunk = chunk_bytes();
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  for (size_t g = 0; g < nch; g += K) {
    std::vector<std::array<size_t, 3>> jobs;
    for (size_t c = g; c < std::min(nch, g + K); ++c) {
      const int slot = (int)(c % (2 * K));
      // the slot's previous DMA (2K chunks ago) must have drained
      if ((e = cudaEventSynchronize(P.done[slot])) != cudaSuccess) return e;
      const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      jobs.push_back({(size_t)P.slots[slot], (size_t)h + off, len});
    }
    par_copy(jobs);
    for (size_t c = g; c < std::min(nch, g + K); ++c) {
      const int slot = (int)(c % (2 * K));
      const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      if ((e = cudaMemcpyAsync((char*)d + off, P.slots[slot], len, cudaMemcpyHostToDevice, st)) !=
          cudaSuccess)
        return e;
      if ((e = cudaEventRecord(P.done[slot], st)) != cudaSuccess) return e;
    }
  }
  // the slots stay referenced by queued DMA: drain before releasing the pool
  for (cudaEvent_t ev : P.done)
    if ((e = cudaEventSynchronize(ev)) != cudaSuccess) return e;
  return cudaSuccess;
}
cudaError_t d2h(void* h, const void* d, size_t bytes, cudaStream_t st) {
  Pool& P = pool();
  std::lock_guard<std::mutex> lk(P.mu);
  const int K = threads();
  cudaError_t e = ensure(P, K);
  if (e != cudaSuccess) return e;
  const size_t kChunk = chunk_bytes();
  const size_t nch = (bytes + kChunk - 1) / kChunk;
  auto issue = [&](size_t g) -> cudaError_t {
    for (size_t c = g; c < std::min(nch, g + K); ++c) {
      const int slot = (int)(c % (2 * K));
      const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      cudaError_t r = cudaMemcpyAsync(P.slots[slot], (const char*)d + off, len,
                                      cudaMemcpyDeviceToHost, st);
      if (r == cudaSuccess) r = cudaEventRecord(P.done[slot], st);
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  };
  if (nch > 0 && (e = issue(0)) != cudaSuccess) return e;
  for (size_t g = 0; g < nch; g += K) {
    // DMA of the next group into the other half of the ring overlaps the
    // host copies of this one
    if (g + K < nch && (e = issue(g + K)) != cudaSuccess) return e;
    std::vector<std::array<size_t, 3>> jobs;
    for (size_t c = g; c < std::min(nch, g + K); ++c) {
      const int slot = (int)(c % (2 * K));
      if ((e = cudaEventSynchronize(P.done[slot])) != cudaSuccess) return e;
      const size_t off = c * kChunk, len = std::min(kChunk, bytes - off);
      jobs.push_back({(size_t)h + off, (size_t)P.slots[slot], len});
    }
    par_copy(jobs);
  }
  return cudaSuccess;
}
}  // namespace staging

static int32_t run_host_entry(const ebisu_stencil* stencil, int32_t ndim,
                              const int64_t* extents, const void* in, void* out, int64_t steps,
                              const ebisu_params* params, ebisu_trace* trace, int elem) {
  g_err.clear();
  if (steps < 0) return fail(EBISU_ERR_VALUE, "step count must be >= 0");
  if (steps > INT32_MAX)
    return fail(EBISU_ERR_VALUE, "step count %lld exceeds 2^31-1", (long long)steps);
  ProblemDesc p;
  int rc = validate(stencil, ndim, extents, params, &p);
  if (rc) return rc;
  if (!in || !out) return fail(EBISU_ERR_VALUE, "null host buffer");
  if (ebisu_device_count() == 0) return fail(EBISU_ERR_NO_DEVICE, "no CUDA device visible");
  const size_t bytes = (size_t)(p.ext[0] * p.ext[1] * p.ext[2]) * (size_t)elem;
  cudaStream_t st = cudaStreamPerThread;
  void *d_in = nullptr, *d_out = nullptr;
  EB_CUDA(cudaMallocAsync(&d_in, bytes, st));
  cudaError_t e = cudaMallocAsync(&d_out, bytes, st);
  if (e != cudaSuccess) {
    cudaFreeAsync(d_in, st);
    return cuda_fail(e, "cudaMallocAsync(out)");
  }
  // pageable (e.g. numpy) buffers: staged through pinned slots by host threads
  const bool stage_in = staging::pageable(in), stage_out = staging::pageable(out);
  e = stage_in ? staging::h2d(d_in, in, bytes, st)
               : cudaMemcpyAsync(d_in, in, bytes, cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    rc = run_device_entry(stencil, ndim, extents, d_in, d_out, nullptr, steps, params, st, trace,
                          elem);
    if (!rc)
      e = stage_out ? staging::d2h(out, d_out, bytes, st)
                    : cudaMemcpyAsync(out, d_out, bytes, cudaMemcpyDeviceToHost, st);
  }
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  cudaFreeAsync(d_in, st);
  cudaFreeAsync(d_out, st);
  if (rc) return rc;
  if (e != cudaSuccess) return cuda_fail(e, "host<->device copy");
  return EBISU_OK;
}

int32_t ebisu_run_device(const ebisu_stencil* stencil, int32_t ndim, const int64_t* extents,
                         const double* d_in, double* d_out, double* d_scratch, int64_t steps,
                         const ebisu_params* params, void* stream, ebisu_trace* trace) {
  return run_device_entry(stencil, ndim, extents, d_in, d_out, d_scratch, steps, params, stream,
                          trace, 8);
}

int32_t ebisu_run_device_f32(const ebisu_stencil* stencil, int32_t ndim, const int64_t* extents,
                             const float* d_in, float* d_out, float* d_scratch, int64_t steps,
                             const ebisu_params* params, void* stream, ebisu_trace* trace) {
  return run_device_entry(stencil, ndim, extents, d_in, d_out, d_scratch, steps, params, stream,
                          trace, 4);
}

int32_t ebisu_run_host(const ebisu_stencil* stencil, int32_t ndim, const int64_t* extents,
                       const double* in, double* out, int64_t steps, const ebisu_params* params,
                       ebisu_trace* trace) {
  return run_host_entry(stencil, ndim, extents, in, out, steps, params, trace, 8);
}

int32_t ebisu_run_host_f32(const ebisu_stencil* stencil, int32_t ndim, const int64_t* extents,
                           const float* in, float* out, int64_t steps, const ebisu_params* params,
                           ebisu_trace* trace) {
  return run_host_entry(stencil, ndim, extents, in, out, steps, params, trace, 4);
}

int32_t ebisu_random_grid_device(uint64_t seed, int64_t start, int64_t n, double* d_out,
                                 void* stream) {
  g_err.clear();
  if (n < 0 || start < 0) return fail(EBISU_ERR_VALUE, "negative range");
  DevInfo di;
  int rc = device_info(&di);
  if (rc) return rc;
  EB_CUDA(launch_splitmix(seed, start, n, d_out, reinterpret_cast<cudaStream_t>(stream), di.sms));
  return EBISU_OK;
}

int32_t ebisu_compare_device(const double* d_a, const double* d_b, int64_t n, int64_t* mismatches,
                             int64_t* first_mismatch, double* max_abs_diff, double* max_abs_ref,
                             void* stream) {
  g_err.clear();
  DevInfo di;
  int rc = device_info(&di);
  if (rc) return rc;
  long long m = 0, f = -1;
  double mx = 0, mr = 0;
  EB_CUDA(launch_compare(d_a, d_b, n, &m, &f, &mx, &mr, reinterpret_cast<cudaStream_t>(stream),
                         di.sms));
  if (mismatches) *mismatches = m;
  if (first_mismatch) *first_mismatch = f;
  if (max_abs_diff) *max_abs_diff = mx;
  if (max_abs_ref) *max_abs_ref = mr;
  return EBISU_OK;
}

int32_t ebisu_release_scratch(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return fail(EBISU_ERR_NO_DEVICE, "no device");
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) cudaMemPoolTrimTo(pool, 0);
  staging::release();  // pinned host slots of the pageable-buffer path
  return EBISU_OK;
}

}  // extern "C"

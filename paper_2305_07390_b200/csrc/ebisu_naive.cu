// ebisu_naive.cu -- one launch per time step, runtime tap list.
//
// Direct restatement of reference_step (grid.py:96-103): every interior cell
// gets the tap sum in tap order (apply_taps, grid.py:76-93), frame cells are
// copied.  It serves three roles: the naive-HBM-roofline yardstick
// (16 B/cell-step), the path for arbitrary user stencils that match no
// specialised kernel, and the remainder steps of a sweep when T is not a
// multiple of the fused depth and no matching depth was instantiated.
#include <type_traits>

#include "ebisu_common.cuh"
#include "ebisu_internal.h"
#include "ebisu_shapes.cuh"

namespace ebisu {

// Geometry of one naive step: the grid as P planes x Y rows x X cells (1-D:
// P = Y = 1; 2-D: P = 1), rows [row_lo, row_hi) written.  A row is the unit of
// work: a CTA owns CPT*BS consecutive cells of one row, so every index is a
// row base plus a lane offset -- no per-cell 64-bit division -- and each
// thread keeps CPT independent cells (CPT*ntaps independent loads) in flight.
struct NaiveGeom {
  long long P, Y, X;
  long long row_lo, row_hi;
  int R0, R1, R2;     // frame widths along the three padded axes
  int chunks;         // CTAs per row
};

struct NaiveTaps {
  int ntaps;
  long long lin[EBISU_MAX_TAPS];  // linear offsets
  double coef[EBISU_MAX_TAPS];
};

constexpr int kNaiveBS = 256;  // threads per CTA
constexpr int kNaiveCPT = 4;   // cells per thread (strided by kNaiveBS: coalesced)

// Compile-time tap pattern (catalog shapes, ebisu_shapes.cuh) or runtime taps
// (SH = void: any stencil, any order).  EXACT: one rounding per multiply and
// per add in tap order (bitwise equal to apply_taps, grid.py:76-93).
template <class SH, bool EXACT, class E>
__global__ void __launch_bounds__(kNaiveBS) k_naive_step(const E* __restrict__ in,
                                                         E* __restrict__ out,
                                                         const __grid_constant__ NaiveGeom g,
                                                         const __grid_constant__ NaiveTaps tp) {
  const long long row = g.row_lo + (long long)(blockIdx.x / (unsigned)g.chunks);
  const int chunk = (int)(blockIdx.x % (unsigned)g.chunks);
  if (row >= g.row_hi) return;
  const long long p = row / g.Y, y = row - p * g.Y;
  const E* src = in + row * g.X;
  E* dst = out + row * g.X;
  const long long x0 = (long long)chunk * (kNaiveBS * kNaiveCPT) + threadIdx.x;
  const bool frame_row = (p < g.R0) || (p >= g.P - g.R0) || (y < g.R1) || (y >= g.Y - g.R1);
  if (frame_row) {
#pragma unroll
    for (int k = 0; k < kNaiveCPT; ++k) {
      const long long x = x0 + k * kNaiveBS;
      if (x < g.X) dst[x] = src[x];
    }
    return;
  }
  E acc[kNaiveCPT];
  bool live[kNaiveCPT], inner[kNaiveCPT];
#pragma unroll
  for (int k = 0; k < kNaiveCPT; ++k) {
    const long long x = x0 + k * kNaiveBS;
    live[k] = x < g.X;
    inner[k] = (x >= g.R2) && (x < g.X - g.R2);
  }
  if constexpr (!std::is_void_v<SH>) {
    // catalog shape: every tap's offset is a compile-time (d0, d1, d2) over
    // runtime strides; all NT*CPT loads are independent of the sums
    const long long plane = g.Y * g.X;
    static_for<SH::NT>([&](auto iI) {
      constexpr int i = decltype(iI)::value;
      constexpr Off o = SH::tap(i);
      long long lin;
      if constexpr (SH::dims == 3)
        lin = o.d0 * plane + o.d1 * g.X + o.d2;
      else if constexpr (SH::dims == 2)
        lin = o.d0 * g.X + o.d1;
      else
        lin = o.d0;
      const E c = (E)tp.coef[i];
#pragma unroll
      for (int k = 0; k < kNaiveCPT; ++k) {
        const long long x = x0 + k * kNaiveBS;
        const E v = inner[k] ? __ldg(src + x + lin) : (E)0;
        if constexpr (i == 0)
          acc[k] = tap_first<EXACT, E>(c, v);
        else
          acc[k] = tap_next<EXACT, E>(acc[k], c, v);
      }
    });
  } else {
#pragma unroll
    for (int k = 0; k < kNaiveCPT; ++k) {
      const long long x = x0 + k * kNaiveBS;
      acc[k] = tap_first<EXACT, E>((E)tp.coef[0], inner[k] ? __ldg(src + x + tp.lin[0]) : (E)0);
    }
    for (int t = 1; t < tp.ntaps; ++t) {
      const long long lin = tp.lin[t];
      const E c = (E)tp.coef[t];
#pragma unroll
      for (int k = 0; k < kNaiveCPT; ++k) {
        const long long x = x0 + k * kNaiveBS;
        acc[k] = tap_next<EXACT, E>(acc[k], c, inner[k] ? __ldg(src + x + lin) : (E)0);
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kNaiveCPT; ++k) {
    const long long x = x0 + k * kNaiveBS;
    if (live[k]) dst[x] = inner[k] ? acc[k] : src[x];
  }
}

template <class SH, class E>
cudaError_t launch_naive_typed(const E* in, E* out, const NaiveGeom& g, const NaiveTaps& tp,
                               bool exact, long long blocks, cudaStream_t st) {
  if (exact)
    k_naive_step<SH, true, E><<<(unsigned)blocks, kNaiveBS, 0, st>>>(in, out, g, tp);
  else
    k_naive_step<SH, false, E><<<(unsigned)blocks, kNaiveBS, 0, st>>>(in, out, g, tp);
  return cudaGetLastError();
}

template <class E>
cudaError_t launch_naive_shape(int shape_id, const E* in, E* out, const NaiveGeom& g,
                               const NaiveTaps& tp, bool exact, long long blocks,
                               cudaStream_t st) {
  switch (shape_id) {
    case SHAPE_J2D5PT: return launch_naive_typed<StarShape<2, 1>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_J2D9PT: return launch_naive_typed<StarShape<2, 2>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_J2D9PT_GOL:
      return launch_naive_typed<BoxShape<2, 1>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_J2D25PT: return launch_naive_typed<BoxShape<2, 2>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_J2D13PT: return launch_naive_typed<StarShape<2, 3>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_J2DS25PT:
      return launch_naive_typed<StarShape<2, 6>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_J3D7PT: return launch_naive_typed<StarShape<3, 1>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_J3D13PT: return launch_naive_typed<StarShape<3, 2>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_J3D17PT:
      return launch_naive_typed<NoCornerShape3<true>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_J3D27PT: return launch_naive_typed<BoxShape<3, 1>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_POISSON:
      return launch_naive_typed<NoCornerShape3<false>>(in, out, g, tp, exact, blocks, st);
    case SHAPE_J1D3PT: return launch_naive_typed<StarShape<1, 1>>(in, out, g, tp, exact, blocks, st);
    default: return launch_naive_typed<void>(in, out, g, tp, exact, blocks, st);
  }
}

cudaError_t launch_naive_step(const ProblemDesc& p, const void* in, void* out,
                              bool exact, cudaStream_t st, int num_sms) {
  (void)num_sms;
  NaiveGeom g{};
  NaiveTaps tp{};
  tp.ntaps = p.ntaps;
  g.P = p.dims == 3 ? p.ext[0] : 1;
  g.Y = p.dims == 3 ? p.ext[1] : (p.dims == 2 ? p.ext[0] : 1);
  g.X = p.ext[p.dims - 1];
  g.R0 = p.dims == 3 ? p.rad : 0;
  g.R1 = p.dims >= 2 ? p.rad : 0;
  g.R2 = p.rad;
  const long long z_hi = p.z_hi > 0 ? p.z_hi : p.ext[0];
  const long long per = p.dims == 3 ? g.Y : 1;  // rows per axis-0 index
  g.row_lo = p.dims == 1 ? 0 : (long long)p.z_lo * per;
  g.row_hi = p.dims == 1 ? 1 : z_hi * per;
  g.chunks = (int)((g.X + kNaiveBS * kNaiveCPT - 1) / (kNaiveBS * kNaiveCPT));
  const long long plane = g.Y * g.X;
  for (int t = 0; t < p.ntaps; ++t) {
    const int* o = p.offsets + t * p.dims;
    long long l;
    if (p.dims == 3)
      l = o[0] * plane + (long long)o[1] * g.X + o[2];
    else if (p.dims == 2)
      l = (long long)o[0] * g.X + o[1];
    else
      l = o[0];
    tp.lin[t] = l;
    tp.coef[t] = p.coeffs[t];
  }
  const long long blocks = (g.row_hi - g.row_lo) * g.chunks;
  if (blocks <= 0) return cudaSuccess;
  if (blocks > 0x7fffffffll) return cudaErrorInvalidValue;
  if (p.elem == 4)
    return launch_naive_shape<float>(p.shape_id, static_cast<const float*>(in),
                                     static_cast<float*>(out), g, tp, exact, blocks, st);
  return launch_naive_shape<double>(p.shape_id, static_cast<const double*>(in),
                                    static_cast<double*>(out), g, tp, exact, blocks, st);
}

// ---- frame pre-copy -----------------------------------------------------------
// Copies the Dirichlet frame (cells within R of any face, common.py:96-112)
// from `in` to `out`.  One warp per row of the fastest axis: frame rows are
// copied whole, other rows only their first and last R cells.
template <class E>
__global__ void __launch_bounds__(256) k_frame_copy(const E* __restrict__ in,
                                                    E* __restrict__ out, long long P,
                                                    long long Y, long long X, long long pitch,
                                                    int R0, int R1, int R2, long long row_lo,
                                                    long long row_hi) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long row = row_lo + (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
       row < row_hi; row += warps) {
    const long long pp = row / Y, y = row % Y;
    const E* src = in + row * pitch;
    E* dst = out + row * pitch;
    if (pp < R0 || pp >= P - R0 || y < R1 || y >= Y - R1) {
      for (long long j = lane; j < X; j += 32) dst[j] = src[j];
    } else {
      for (int j = lane; j < 2 * R2; j += 32) {
        const long long x = j < R2 ? j : X - 2 * R2 + j;
        dst[x] = src[x];
      }
    }
  }
}

cudaError_t launch_frame_copy(const ProblemDesc& p, const void* in, void* out,
                              cudaStream_t st, int num_sms) {
  long long P = 1, Y = 1, X = p.ext[0];
  int R0 = 0, R1 = 0;
  if (p.dims == 2) {
    Y = p.ext[0];
    X = p.ext[1];
    R1 = p.rad;
  } else if (p.dims == 3) {
    P = p.ext[0];
    Y = p.ext[1];
    X = p.ext[2];
    R0 = R1 = p.rad;
  }
  // rows of the output-plane range only (axis 0 = planes in 3-D, rows in 2-D)
  const long long z_hi = p.z_hi > 0 ? p.z_hi : p.ext[0];
  const long long per = p.dims == 3 ? Y : 1;
  long long row_lo = (long long)p.z_lo * per, row_hi = z_hi * per;
  if (p.dims == 1) row_lo = 0, row_hi = 1;
  const long long rows = row_hi - row_lo;
  const long long pitch = p.pitch ? p.pitch : X;
  long long blocks = (rows + 7) / 8;
  const long long cap = (long long)num_sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (p.elem == 4)
    k_frame_copy<float><<<(unsigned)blocks, 256, 0, st>>>(
        static_cast<const float*>(in), static_cast<float*>(out), P, Y, X, pitch, R0, R1, p.rad,
        row_lo, row_hi);
  else
    k_frame_copy<double><<<(unsigned)blocks, 256, 0, st>>>(
        static_cast<const double*>(in), static_cast<double*>(out), P, Y, X, pitch, R0, R1, p.rad,
        row_lo, row_hi);
  return cudaGetLastError();
}

// ---- SplitMix64 uniforms, bit-identical to rng.uniform_array ---------------
__global__ void __launch_bounds__(256) k_splitmix_uniform(unsigned long long seed,
                                                          long long start, long long n,
                                                          double* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    unsigned long long z = seed + (unsigned long long)(start + i + 1) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z = z ^ (z >> 31);
    // (z >> 11) < 2^53 converts exactly; the scale by 2^-53 is exact.
    out[i] = (double)(z >> 11) * 0x1.0p-53;
  }
}

cudaError_t launch_splitmix(unsigned long long seed, long long start, long long n, double* out,
                            cudaStream_t st, int num_sms) {
  if (n <= 0) return cudaSuccess;
  long long blocks = (n + 255) / 256;
  const long long cap = (long long)num_sms * 16;
  if (blocks > cap) blocks = cap;
  k_splitmix_uniform<<<(unsigned)blocks, 256, 0, st>>>(seed, start, n, out);
  return cudaGetLastError();
}

// ---- device-side comparison ------------------------------------------------
struct CompareOut {
  unsigned long long mismatches;
  long long first;
  unsigned long long max_abs_bits;  // non-negative doubles order like their bits
  unsigned long long max_ref_bits;
};

__global__ void __launch_bounds__(256) k_compare(const double* __restrict__ a,
                                                 const double* __restrict__ b, long long n,
                                                 CompareOut* o) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  unsigned long long mism = 0;
  long long first = -1;
  double mx = 0.0, mr = 0.0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const double x = a[i], y = b[i];
    if (__double_as_longlong(x) != __double_as_longlong(y)) {
      ++mism;
      if (first < 0) first = i;
    }
    const double d = fabs(x - y);
    mx = (d > mx || d != d) ? d : mx;
    mr = fmax(mr, fabs(y));
  }
  for (int off = 16; off; off >>= 1) {
    mism += __shfl_down_sync(kFullMask, mism, off);
    const long long f2 = __shfl_down_sync(kFullMask, first, off);
    if (f2 >= 0 && (first < 0 || f2 < first)) first = f2;
    const double m2 = __shfl_down_sync(kFullMask, mx, off);
    mx = (m2 > mx || m2 != m2) ? m2 : mx;
    mr = fmax(mr, __shfl_down_sync(kFullMask, mr, off));
  }
  if ((threadIdx.x & 31) == 0) {
    if (mism) atomicAdd(&o->mismatches, mism);
    if (first >= 0) {
      // first mismatch = minimum index; ordered as unsigned after a bias
      atomicMin(reinterpret_cast<unsigned long long*>(&o->first),
                (unsigned long long)first);
    }
    atomicMax(&o->max_abs_bits, (unsigned long long)__double_as_longlong(mx));
    atomicMax(&o->max_ref_bits, (unsigned long long)__double_as_longlong(mr));
  }
}

cudaError_t launch_compare(const double* a, const double* b, long long n, long long* mism,
                           long long* first, double* max_abs, double* max_ref, cudaStream_t st,
                           int num_sms) {
  CompareOut* d = nullptr;
  cudaError_t err = cudaMallocAsync(&d, sizeof(CompareOut), st);
  if (err != cudaSuccess) return err;
  CompareOut init{0ull, (long long)-1, 0ull, 0ull};
  // first = -1 == 0xffff...: atomicMin on unsigned keeps the smallest index.
  err = cudaMemcpyAsync(d, &init, sizeof(init), cudaMemcpyHostToDevice, st);
  if (err == cudaSuccess && n > 0) {
    long long blocks = (n + 255) / 256;
    const long long cap = (long long)num_sms * 8;
    if (blocks > cap) blocks = cap;
    k_compare<<<(unsigned)blocks, 256, 0, st>>>(a, b, n, d);
    err = cudaGetLastError();
  }
  CompareOut h{};
  if (err == cudaSuccess) err = cudaMemcpyAsync(&h, d, sizeof(h), cudaMemcpyDeviceToHost, st);
  if (err == cudaSuccess) err = cudaStreamSynchronize(st);
  cudaFreeAsync(d, st);
  if (err != cudaSuccess) return err;
  *mism = (long long)h.mismatches;
  *first = h.first;
  *max_abs = __longlong_as_double_host((long long)h.max_abs_bits);
  *max_ref = __longlong_as_double_host((long long)h.max_ref_bits);
  return cudaSuccess;
}

}  // namespace ebisu

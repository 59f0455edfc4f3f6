// ebisu_naive.cu -- one launch per time step, runtime tap list.
//
// Direct restatement of reference_step (grid.py:96-103): every interior cell
// gets the tap sum in tap order (apply_taps, grid.py:76-93), frame cells are
// copied.  It serves three roles: the naive-HBM-roofline yardstick
// (16 B/cell-step), the path for arbitrary user stencils that match no
// specialised kernel, and the remainder steps of a sweep when T is not a
// multiple of the fused depth and no matching depth was instantiated.
#include "ebisu_common.cuh"
#include "ebisu_internal.h"

namespace ebisu {

struct NaiveTaps {
  int ntaps;
  int rad;
  int dims;
  long long n0, n1, n2;  // extents (unused axes = 1)
  long long z_lo, z_hi;  // output planes [z_lo, z_hi) along axis 0
  long long lin[EBISU_MAX_TAPS];  // linear offsets
  double coef[EBISU_MAX_TAPS];
};

template <bool EXACT, class E>
__global__ void __launch_bounds__(256) k_naive_step(const E* __restrict__ in,
                                                    E* __restrict__ out,
                                                    const __grid_constant__ NaiveTaps tp) {
  const long long plane = tp.n1 * tp.n2;
  const long long base = tp.z_lo * plane;
  const long long total = (tp.z_hi - tp.z_lo) * plane;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long idx = base + (long long)blockIdx.x * blockDim.x + threadIdx.x;
       idx < base + total; idx += stride) {
    const long long i2 = idx % tp.n2;
    const long long r = idx / tp.n2;
    const long long i1 = r % tp.n1;
    const long long i0 = r / tp.n1;
    const int R = tp.rad;
    bool frame = (i0 < R) || (i0 >= tp.n0 - R);
    if (tp.dims >= 2) frame |= (i1 < R) || (i1 >= tp.n1 - R);
    if (tp.dims >= 3) frame |= (i2 < R) || (i2 >= tp.n2 - R);
    E v;
    if (frame) {
      v = in[idx];
    } else {
      v = tap_first<EXACT, E>((E)tp.coef[0], __ldg(in + idx + tp.lin[0]));
      for (int t = 1; t < tp.ntaps; ++t)
        v = tap_next<EXACT, E>(v, (E)tp.coef[t], __ldg(in + idx + tp.lin[t]));
    }
    out[idx] = v;
  }
}

cudaError_t launch_naive_step(const ProblemDesc& p, const void* in, void* out,
                              bool exact, cudaStream_t st, int num_sms) {
  NaiveTaps tp{};
  tp.ntaps = p.ntaps;
  tp.rad = p.rad;
  tp.dims = p.dims;
  tp.n0 = p.ext[0];
  tp.n1 = p.dims >= 2 ? p.ext[1] : 1;
  tp.n2 = p.dims >= 3 ? p.ext[2] : 1;
  tp.z_lo = p.z_lo;
  tp.z_hi = p.z_hi > 0 ? p.z_hi : p.ext[0];
  for (int t = 0; t < p.ntaps; ++t) {
    const int* o = p.offsets + t * p.dims;
    long long l = o[0];
    if (p.dims >= 2) l = l * tp.n1 + o[1];
    if (p.dims >= 3) l = l * tp.n2 + o[2];
    tp.lin[t] = l;
    tp.coef[t] = p.coeffs[t];
  }
  const long long total = (tp.z_hi - tp.z_lo) * tp.n1 * tp.n2;
  long long blocks = (total + 255) / 256;
  const long long cap = (long long)num_sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (p.elem == 4) {
    const float* fi = static_cast<const float*>(in);
    float* fo = static_cast<float*>(out);
    if (exact)
      k_naive_step<true, float><<<(unsigned)blocks, 256, 0, st>>>(fi, fo, tp);
    else
      k_naive_step<false, float><<<(unsigned)blocks, 256, 0, st>>>(fi, fo, tp);
  } else {
    const double* di = static_cast<const double*>(in);
    double* dout = static_cast<double*>(out);
    if (exact)
      k_naive_step<true, double><<<(unsigned)blocks, 256, 0, st>>>(di, dout, tp);
    else
      k_naive_step<false, double><<<(unsigned)blocks, 256, 0, st>>>(di, dout, tp);
  }
  return cudaGetLastError();
}

// ---- frame pre-copy -----------------------------------------------------------
// Copies the Dirichlet frame (cells within R of any face, common.py:96-112)
// from `in` to `out`.  One warp per row of the fastest axis: frame rows are
// copied whole, other rows only their first and last R cells.
template <class E>
__global__ void __launch_bounds__(256) k_frame_copy(const E* __restrict__ in,
                                                    E* __restrict__ out, long long P,
                                                    long long Y, long long X, int R0, int R1,
                                                    int R2, long long row_lo, long long row_hi) {
  const int lane = threadIdx.x & 31;
  const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
  for (long long row = row_lo + (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
       row < row_hi; row += warps) {
    const long long pp = row / Y, y = row % Y;
    const E* src = in + row * X;
    E* dst = out + row * X;
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
  long long blocks = (rows + 7) / 8;
  const long long cap = (long long)num_sms * 8;
  if (blocks > cap) blocks = cap;
  if (blocks < 1) blocks = 1;
  if (p.elem == 4)
    k_frame_copy<float><<<(unsigned)blocks, 256, 0, st>>>(
        static_cast<const float*>(in), static_cast<float*>(out), P, Y, X, R0, R1, p.rad, row_lo,
        row_hi);
  else
    k_frame_copy<double><<<(unsigned)blocks, 256, 0, st>>>(
        static_cast<const double*>(in), static_cast<double*>(out), P, Y, X, R0, R1, p.rad, row_lo,
        row_hi);
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

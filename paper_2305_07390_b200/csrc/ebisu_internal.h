// ebisu_internal.h -- internal interfaces between the C-ABI driver
// (ebisu_api.cu) and the kernel translation units.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#include "../../include/ebisu.h"

namespace ebisu {

inline double __longlong_as_double_host(long long v) {
  double d;
  memcpy(&d, &v, sizeof(d));
  return d;
}

// Validated problem (host side).
struct ProblemDesc {
  int dims;
  int ntaps;
  int rad;
  long long ext[3];
  const int* offsets;    // [ntaps][dims]
  const double* coeffs;  // [ntaps]
  int shape_id;          // ShapeId or SHAPE_GENERIC
  int z_lo = 0, z_hi = 0;  // output planes [z_lo, z_hi) along axis 0 (set by the driver)
  int elem = 8;            // element bytes: 8 (fp64) or 4 (fp32)
  long long pitch = 0;     // row pitch of the kernel buffers (elements; 0 = last extent)
};

cudaError_t launch_naive_step(const ProblemDesc& p, const void* in, void* out, bool exact,
                              cudaStream_t st, int num_sms);  // writes planes [z_lo, z_hi)
cudaError_t launch_frame_copy(const ProblemDesc& p, const void* in, void* out,
                              cudaStream_t st, int num_sms);  // both buffers at p.pitch
cudaError_t launch_splitmix(unsigned long long seed, long long start, long long n, double* out,
                            cudaStream_t st, int num_sms);
cudaError_t launch_compare(const double* a, const double* b, long long n, long long* mism,
                           long long* first, double* max_abs, double* max_ref, cudaStream_t st,
                           int num_sms);

// ---- resident-tile temporal blocking for any tap set (ebisu_generic.cu) ----
// The grid is viewed as (planes, rows, cols) = ext[0..2]: 1-D (1, 1, n),
// 2-D (1, n0, n1), 3-D (n0, n1, n2); grid axis 0 sits at tile axis zaxis.
// magic numbers of an unsigned division by d (GenArgs per-level divisors)
struct GenDiv {
  uint32_t m, s1, s2;
};
__host__ __device__ inline GenDiv gen_div(uint32_t d) {
  uint32_t l = 0;
  while ((1u << l) < d) ++l;  // l = ceil(log2 d)
  GenDiv g;
  g.m = (uint32_t)((((unsigned long long)1 << 32) * (((unsigned long long)1 << l) - d)) / d) + 1;
  g.s1 = l > 0 ? 1 : 0;
  g.s2 = l > 0 ? l - 1 : 0;
  return g;
}
#define EBISU_GEN_MAXT 32  // levels per resident-tile launch

struct GenArgs {
  long long ext[3];
  long long pitch;       // row pitch (elements)
  int zaxis;             // 3 - dims
  long long z_lo, z_hi;  // output range along grid axis 0
  int L[3], V[3], H[3];  // loaded / core / halo extents per tile axis
  int RA[3];             // shrink per level (R on present axes, 0 on absent)
  int F[3];              // frame width per axis
  int nt[3];             // tiles per axis
  int T;                 // fused levels of this launch (<= EBISU_GEN_MAXT)
  GenDiv lvl_cpr[EBISU_GEN_MAXT];  // level s: row chunks per region row
  GenDiv lvl_w1[EBISU_GEN_MAXT];   // level s: region rows per plane
  int ntaps;
  int lin[EBISU_MAX_TAPS];  // tile-linear tap offsets
  double coef[EBISU_MAX_TAPS];
  const void* in;
  void* out;
};
cudaError_t launch_generic_tb(const GenArgs& a, int elem, bool exact, int grid, int threads,
                              int smem, cudaStream_t st);

// ---- one-step 2.5-D streaming for any 3-D tap set (ebisu_generic.cu) ----------
// CTA = LY x LX output tile streamed along axis 0 through a ring of
// 2R+2 shared-memory planes (each plane loaded once, with its R-wide ring).
struct GenS3DArgs {
  long long n0, n1, n2;
  long long pitch;          // row pitch (elements)
  long long z_lo, z_hi;     // output planes
  int R, LY, LX;            // radius, core tile
  int nty, ntx, nseg, seg_len;
  int ntaps;
  int dz[EBISU_MAX_TAPS];   // axis-0 offset of tap k
  int lin[EBISU_MAX_TAPS];  // in-plane offset dy*(LX+2R) + dx
  double coef[EBISU_MAX_TAPS];
  const void* in;
  void* out;
};
cudaError_t launch_generic_s3d(const GenS3DArgs& a, int elem, bool exact, int grid, int smem,
                               cudaStream_t st);
constexpr int kGenS3DThreads = 256;
int generic_threads();

// ---- temporal-blocking kernel registry -------------------------------------
struct TbLaunch {
  // geometry
  int n0, n1, n2;  // extents (2-D: n2 unused)
  int nstrips, nseg, seg_len;  // 2-D decomposition
  int z_lo, z_hi;              // output rows/planes [z_lo, z_hi) along axis 0
  int aligned;                 // 2-D: edge-aligned strips
  int pitch;                   // row pitch of every buffer (elements; n_last or padded)
  int ntx, nty;                // 3-D decomposition (tiles along axis 2 / axis 1)
  int aligned_x, aligned_y;    // 3-D: edge-aligned tiles along axis 2 / axis 1
  const int* seg_start;        // 3-D: nseg+1 segment bounds along axis 0 (guided)
  int epochs;
  int first_src, first_dst;
  void* buf[3];  // element type of the stage's kernel
  const CUtensorMap* maps;  // host copies [3]
  const double* coeffs;
  int grid;
  bool cooperative;
  cudaStream_t stream;
  long long* unit_clock;  // optional per-unit timing (profiling)
  int* work;              // per-epoch dynamic-scheduling counters (device)
  int* flags;             // per-unit completed-epoch flags (dataflow epochs) or null
  int cluster = 1;        // halo2d: CTAs per cluster tile along axis 1 (device tile grid)
};

struct TbKernel {
  int shape_id;
  int dims;
  int T;         // fused depth
  int C;         // cells per lane along the fastest axis
  int NW;        // warps per CTA
  int S;         // ring slots
  int exact;
  int uni;       // shared-product kernel (uniform coefficients; bitwise exact)
  int smem_bytes;
  int box0, box1, box2;  // TMA box (elements) fastest first
  int valid_x;           // valid columns per warp strip (2-D) or per tile (3-D, axis 2)
  int valid_y;           // 3-D: valid rows per tile (axis 1)
  int z;                 // 3-D: level skew along axis 0 (advances per level)
  int wn;                // 3-D: window planes (advance-loop unroll)
  const void* func;      // kernel symbol (occupancy queries / attributes)
  cudaError_t (*launch)(const TbLaunch&);
  int family;            // 0: overlapped (sm-tiling), 1: halo exchange (device-tiling)
  int elem;              // element bytes: 8 (fp64) or 4 (fp32)
  int cluster = 1;       // CTAs per cluster along axis 1 (2: one tile over two SMs, DSMEM seam)
  cudaError_t (*max_clusters)(int*) = nullptr;  // resident clusters (cluster kernels)
  cudaError_t (*max_clusters_n)(int, int*) = nullptr;  // halo2d: resident clusters of size n
};

// All instantiated temporal-blocking kernels (ebisu_registry.cu).
const TbKernel* tb_kernels(int* count);

}  // namespace ebisu

// ebisu_generic.cu -- temporal blocking for ANY tap set (runtime taps),
// 1-D, 2-D and 3-D, sm_100a.
//
// The specialised kernels (k_stream2d / k_stream3d / k_halo2d) bake the tap
// pattern into register windows at compile time, so they cover the catalog
// shapes (shapes.py:60-157) only.  The reference accepts any StencilShape
// (shapes.py:27-56: arbitrary offsets, arbitrary order, any radius) and its
// engines tile it the same way (engine/device.py:214-261, the lazy resident
// tile: a block loads its region plus rad*t, runs t steps on chip, stores the
// core).  This kernel is that scheme on B200 for an arbitrary tap list:
//
//  * Work unit = one resident tile of L0 x L1 x L2 cells (axes absent in
//    lower dimensions have extent 1) = core V + halo H = T*R per side on
//    every tiled axis.  Tiles cover the grid (or the output-plane range
//    [z_lo, z_hi) along axis 0) with their cores; a persistent grid strides
//    over them.
//  * The tile lives in shared memory as two ping-pong buffers (2 CTAs x 512
//    threads x ~113 KB per SM); level s computes the region shrunk by s*R
//    per side from the level s-1 buffer.  Taps are tile-linear offsets in the
//    kernel parameter space (uniform across the warp: constant-bank
//    broadcast; unrolled for up to 27 taps); every lane owns 4 cells of a
//    128-cell row chunk (4 independent sums in flight).
//  * Frame cells (distance < R from a face, common.py:96-112) and cells
//    outside the domain carry their value; a computed interior cell reads only
//    cells within R, all inside the domain, so the zero-filled outside is
//    never read by a stored cell.
//  * The stored core includes frame cells, so every output cell is written
//    by exactly one tile (no frame pre-copy, no scratch assumptions).
//  * Arithmetic: taps in the given order, one rounding per multiply and per
//    add (EXACT) -> bitwise equal to apply_taps (grid.py:76-93); FMA chain in
//    tolerance mode.
//  * Per cell-step cost: NT shared loads + 1 shared store (no register
//    reuse: the pattern is not known at compile time); the host planner
//    (ebisu_api.cu gen_plan) picks the tile shape from that cost and the HBM
//    round trip.  Measured, it wins over one launch per step in 1-D only, so
//    AUTO runs 1-D tap sets here (t = 16), 2-D ones on the naive kernel and
//    3-D ones on k_generic_s3d below (gen_pick_depth).
//
// k_generic_s3d: one step of any 3-D tap set, 2.5-D streaming through a
// shared-memory plane ring (see the kernel's comment).
#include "ebisu_common.cuh"
#include "ebisu_internal.h"
#include "ebisu_shapes.cuh"  // static_for

namespace ebisu {

constexpr int kGenThreads = 1024;

// cp.async of one element, zero-filled when !pred (src-size 0)
template <class E>
__device__ __forceinline__ void cp_async_zfill(E* dst, const E* src, bool pred) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_u32(dst)), "l"(src),
               "n"((int)sizeof(E)), "r"(pred ? (int)sizeof(E) : 0)
               : "memory");
}
constexpr int kGenCPL = 4;  // cells per lane per row chunk
constexpr int kGenPad = 32 * kGenCPL;  // elements after each buffer (idle lanes read there)

// n / d for 0 <= n < 2^31 by a block-uniform d >= 1 (Granlund-Montgomery:
// one mul.hi, an add and two shifts instead of the ~20-instruction division);
// the per-level divisors come precomputed from the host (GenArgs.lvl_*), the
// per-tile ones are derived once per tile
struct FastDiv {
  uint32_t m, s1, s2;
  __device__ __forceinline__ explicit FastDiv(const GenDiv& g) : m(g.m), s1(g.s1), s2(g.s2) {}
  __device__ __forceinline__ explicit FastDiv(uint32_t dv) {
    const GenDiv g = gen_div(dv);
    m = g.m;
    s1 = g.s1;
    s2 = g.s2;
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const {
    const uint32_t t = __umulhi(n, m);
    return (t + ((n - t) >> s1)) >> s2;
  }
};
constexpr int kGenMaxNT = 27;  // tap counts with an unrolled kernel (3x3x3 box); more: runtime loop

// Tap k of the list: compile-time index when NT > 0 (uniform registers,
// loaded once), runtime index otherwise.
template <int NT>
struct TapLoop {
  template <class F>
  __device__ __forceinline__ static void run(int, F&& f) {
    static_for<NT - 1>([&](auto kI) { f(decltype(kI)::value + 1); });
  }
};
template <>
struct TapLoop<0> {
  template <class F>
  __device__ __forceinline__ static void run(int ntaps, F&& f) {
#pragma unroll 1
    for (int k = 1; k < ntaps; ++k) f(k);
  }
};

template <class E, bool EXACT, int NT>
__global__ void __launch_bounds__(kGenThreads, 1) k_generic_tb(const __grid_constant__ GenArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int L0 = a.L[0], L1 = a.L[1], L2 = a.L[2];
  const int ncell = L0 * L1 * L2;
  E* const b0 = reinterpret_cast<E*>(smem);
  E* const b1 = b0 + ncell + kGenPad;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int NW = blockDim.x >> 5;
  constexpr int CH = 32 * kGenCPL;  // cells per row chunk
  const long long ext0 = a.ext[0], ext1 = a.ext[1], ext2 = a.ext[2];
  const E* __restrict__ in = static_cast<const E*>(a.in);
  E* __restrict__ out = static_cast<E*>(a.out);
  const long long ntiles = (long long)a.nt[0] * a.nt[1] * a.nt[2];
  const int ntaps = NT > 0 ? NT : a.ntaps;

  for (long long tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int t2 = (int)(tile % a.nt[2]);
    const int t1 = (int)((tile / a.nt[2]) % a.nt[1]);
    const int t0 = (int)(tile / ((long long)a.nt[2] * a.nt[1]));
    // core origin per axis (axis a.zaxis starts at z_lo) and loaded origin
    const long long c0 = (a.zaxis == 0 ? a.z_lo : 0) + (long long)t0 * a.V[0];
    const long long c1 = (a.zaxis == 1 ? a.z_lo : 0) + (long long)t1 * a.V[1];
    const long long c2 = (a.zaxis == 2 ? a.z_lo : 0) + (long long)t2 * a.V[2];
    const long long o0 = c0 - a.H[0], o1 = c1 - a.H[1], o2 = c2 - a.H[2];
    // computable cells (inside the domain, outside the frame) in tile
    // coordinates: [flo_a, fhi_a) per axis
    auto clampi = [](long long v, int hi) { return (int)max(0LL, min(v, (long long)hi)); };
    const int flo0 = clampi(a.F[0] - o0, L0), fhi0 = clampi(ext0 - a.F[0] - o0, L0);
    const int flo1 = clampi(a.F[1] - o1, L1), fhi1 = clampi(ext1 - a.F[1] - o1, L1);
    const int flo2 = clampi(a.F[2] - o2, L2), fhi2 = clampi(ext2 - a.F[2] - o2, L2);

    // ---- load the tile (zero outside the domain) ----------------------------
    {
      const int cpr = (L2 + 31) / 32;
      const int nch = L0 * L1 * cpr;
      const FastDiv dcpr((uint32_t)cpr), dL1((uint32_t)L1);
      for (int c = warp; c < nch; c += NW) {
        const int row = (int)dcpr.div((uint32_t)c);
        const int x = (c - row * cpr) * 32 + lane;
        if (x >= L2) continue;
        const int i0 = (int)dL1.div((uint32_t)row), i1 = row - i0 * L1;
        const long long g0 = o0 + i0, g1 = o1 + i1, g2 = o2 + x;
        const bool inside = g0 >= 0 && g0 < ext0 && g1 >= 0 && g1 < ext1 && g2 >= 0 && g2 < ext2;
        // asynchronous copy (LDGSTS), zero fill outside the domain: every
        // warp keeps all its row chunks in flight
        cp_async_zfill(b0 + row * L2 + x, inside ? in + (g0 * ext1 + g1) * a.pitch + g2 : in,
                       inside);
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    }
    __syncthreads();

    // ---- T levels on chip -------------------------------------------------------
    E* cur = b0;
    E* nxt = b1;
    for (int s = 1; s <= a.T; ++s) {
      const int lo0 = s * a.RA[0], hi0 = L0 - s * a.RA[0];
      const int lo1 = s * a.RA[1], hi1 = L1 - s * a.RA[1];
      const int lo2 = s * a.RA[2], hi2 = L2 - s * a.RA[2];
      const int w1 = hi1 - lo1, w2 = hi2 - lo2;
      const int cpr = (w2 + CH - 1) / CH;
      const int nch = (hi0 - lo0) * w1 * cpr;
      const FastDiv dcpr(a.lvl_cpr[s - 1]), dw1(a.lvl_w1[s - 1]);
      for (int c = warp; c < nch; c += NW) {
        const int row = (int)dcpr.div((uint32_t)c);
        const int xb = lo2 + (c - row * cpr) * CH + lane;
        const int r0 = (int)dw1.div((uint32_t)row);
        const int i0 = lo0 + r0, i1 = lo1 + (row - r0 * w1);
        const bool crow = i0 >= flo0 && i0 < fhi0 && i1 >= flo1 && i1 < fhi1;
        // lanes past the region (x >= hi2) compute from the padding and
        // store nothing: every address is base + 32j + tap offset
        const E* __restrict__ p = cur + (i0 * L1 + i1) * L2 + xb;
        E acc[kGenCPL];
        {
          const E cf = (E)a.coef[0];
          const int off = a.lin[0];
#pragma unroll
          for (int j = 0; j < kGenCPL; ++j) acc[j] = tap_first<EXACT, E>(cf, p[32 * j + off]);
        }
        TapLoop<NT>::run(ntaps, [&](int k) {
          const E cf = (E)a.coef[k];
          const int off = a.lin[k];
#pragma unroll
          for (int j = 0; j < kGenCPL; ++j) acc[j] = tap_next<EXACT, E>(acc[j], cf, p[32 * j + off]);
        });
        E* __restrict__ q = nxt + (p - cur);
#pragma unroll
        for (int j = 0; j < kGenCPL; ++j) {
          const int x = xb + 32 * j;
          if (x < hi2) q[32 * j] = (crow && x >= flo2 && x < fhi2) ? acc[j] : p[32 * j];
        }
      }
      __syncthreads();
      E* tmp = cur;
      cur = nxt;
      nxt = tmp;
    }

    // ---- store the core (clipped to the domain / output range) -----------------
    {
      const long long zend = a.z_hi;
      const long long e0 = a.zaxis == 0 ? zend : ext0;
      const long long e1 = a.zaxis == 1 ? zend : ext1;
      const long long e2 = a.zaxis == 2 ? zend : ext2;
      const int v0 = (int)min((long long)a.V[0], e0 - c0);
      const int v1 = (int)min((long long)a.V[1], e1 - c1);
      const int v2 = (int)min((long long)a.V[2], e2 - c2);
      const int cpr = (v2 + 31) / 32;
      const int nch = v0 * v1 * cpr;
      const FastDiv dcpr((uint32_t)cpr), dv1((uint32_t)max(v1, 1));
      for (int c = warp; c < nch; c += NW) {
        const int row = (int)dcpr.div((uint32_t)c);
        const int x = (c - row * cpr) * 32 + lane;
        if (x >= v2) continue;
        const int r0 = (int)dv1.div((uint32_t)row), r1 = row - r0 * v1;
        const int idx = ((a.H[0] + r0) * L1 + (a.H[1] + r1)) * L2 + a.H[2] + x;
        out[((c0 + r0) * ext1 + (c1 + r1)) * a.pitch + (c2 + x)] = cur[idx];
      }
    }
    __syncthreads();  // the next tile's load overwrites b0
  }
}

// ---- one step, any 3-D tap set: 2.5-D streaming through a plane ring ----------
// The one-launch-per-step naive kernel reads the z+-R planes of every cell
// from L2/HBM (512^3 j3d7pt-order-reversed: 180 GCells/s, 0.44 of the naive
// roofline); here a CTA streams an LY x LX tile along axis 0 and keeps the
// last 2R+1 planes (with their R-wide ring) in shared memory, so every input
// cell is loaded once per tile (plus the ring) and every tap is a shared-
// memory read.  The next plane's cp.async overlaps the current plane's sums.
constexpr int kGenS3DPrefetch = 1;  // planes in flight (measured: 2 or 3 with 8-row tiles were slower: fewer CTAs per SM)

template <class E, bool EXACT, int NT>
__global__ void __launch_bounds__(kGenS3DThreads) k_generic_s3d(const __grid_constant__ GenS3DArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  E* const ring = reinterpret_cast<E*>(smem);
  const int R = a.R, LY = a.LY, LX = a.LX;
  const int PY = LY + 2 * R, PX = LX + 2 * R, PL = PY * PX;
  constexpr int PD = kGenS3DPrefetch;  // planes in flight ahead of the sums
  const int K = 2 * R + 1 + PD;        // ring slots
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = kGenS3DThreads / 32;
  const long long n0 = a.n0, n1 = a.n1, n2 = a.n2;
  const E* __restrict__ in = static_cast<const E*>(a.in);
  E* __restrict__ out = static_cast<E*>(a.out);
  const int ntaps = NT > 0 ? NT : a.ntaps;
  const long long units = (long long)a.nty * a.ntx * a.nseg;

  for (long long u = blockIdx.x; u < units; u += gridDim.x) {
    const int tx = (int)(u % a.ntx);
    const int ty = (int)((u / a.ntx) % a.nty);
    const int sg = (int)(u / ((long long)a.ntx * a.nty));
    const long long Y0 = (long long)ty * LY, X0 = (long long)tx * LX;
    const long long za = a.z_lo + (long long)sg * a.seg_len;
    const long long zb = min(a.z_hi, za + a.seg_len);
    // load plane z (ring slot z mod K), zero outside the domain
    // in-domain columns of the loaded plane, tile coordinates [clo, chi);
    // stored columns [0, ohi) and computed (non-frame) ones [clo_f, chi_f)
    const int clo = (int)max(0LL, (long long)R - X0);
    const int chi = (int)min((long long)PX, n2 - X0 + R);
    const int ohi = (int)min((long long)LX, n2 - X0);
    const int clo_f = (int)max(0LL, (long long)R - X0);
    const int chi_f = (int)min((long long)LX, n2 - R - X0);
    auto load = [&](long long z) {
      E* dst = ring + (int)(((z % K) + K) % K) * PL;
      const bool zin = z >= 0 && z < n0;
      for (int r = warp; r < PY; r += NW) {
        const long long y = Y0 - R + r;
        const bool yin = zin && y >= 0 && y < n1;
        // row base at tile column 0 (only dereferenced for in-domain columns)
        const E* src = in + ((z * n1 + y) * a.pitch + X0 - R);
        E* d = dst + r * PX;
        for (int c = lane; c < PX; c += 32) {
          const bool ok = yin && c >= clo && c < chi;
          cp_async_zfill(d + c, ok ? src + c : in, ok);
        }
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    // prologue: planes za-R .. za+R-1+PD (one commit group each)
    for (long long z = za - R; z < za + R + PD; ++z) load(z);
    for (long long z = za; z < zb; ++z) {
      // plane z+R is in (at most PD-1 younger groups pending) and every
      // thread is done with plane z-1, so the slot of plane z-R-1 takes
      // plane z+R+PD, in flight during the next PD planes' sums
      asm volatile("cp.async.wait_group %0;" ::"n"(PD - 1) : "memory");
      __syncthreads();
      if (z + PD < zb) {
        load(z + R + PD);
      } else {
        asm volatile("cp.async.commit_group;" ::: "memory");  // keep the group count
      }
      const bool fz = z < R || z >= n0 - R;
      const int zs = (int)(z % K);  // ring slot of plane z (z >= 0 here)
      // ring offset of every tap for this plane (slot of plane z+dz, plus the
      // in-plane offset): registers when the tap count is a template constant
      int toff[NT > 0 ? NT : 1];
      if constexpr (NT > 0) {
#pragma unroll
        for (int k = 0; k < NT; ++k) {
          int slot = zs + a.dz[k];
          slot += slot < 0 ? K : 0;
          slot -= slot >= K ? K : 0;
          toff[k] = slot * PL + a.lin[k];
        }
      }
      for (int r = warp; r < LY; r += NW) {
        const long long y = Y0 + r;
        if (y >= n1) break;
        const bool fy = fz || y < R || y >= n1 - R;
        const int base = (r + R) * PX + R;
        E* const orow = out + (z * n1 + y) * a.pitch + X0;
        for (int c0 = 0; c0 < LX; c0 += 128) {
          E acc[4];
          bool live[4], comp[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const int c = c0 + lane + 32 * j;  // tile column (32-bit tests)
            live[j] = c < ohi;
            comp[j] = !fy && c >= clo_f && c < chi_f;
          }
          const E* pc = ring + base + c0 + lane;
          auto tap = [&](int k) -> const E* {
            if constexpr (NT > 0) {
              return pc + toff[k];
            } else {
              int slot = zs + a.dz[k];
              slot += slot < 0 ? K : 0;
              slot -= slot >= K ? K : 0;
              return pc + slot * PL + a.lin[k];
            }
          };
          {
            const E* p = tap(0);
            const E cf = (E)a.coef[0];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = tap_first<EXACT, E>(cf, p[32 * j]);
          }
          TapLoop<NT>::run(ntaps, [&](int k) {
            const E* p = tap(k);
            const E cf = (E)a.coef[k];
#pragma unroll
            for (int j = 0; j < 4; ++j) acc[j] = tap_next<EXACT, E>(acc[j], cf, p[32 * j]);
          });
          const E* ctr = ring + zs * PL + base + c0 + lane;
          E* o = orow + c0 + lane;
#pragma unroll
          for (int j = 0; j < 4; ++j)
            if (live[j]) o[32 * j] = comp[j] ? acc[j] : ctr[32 * j];
        }
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    __syncthreads();  // the next unit's prologue overwrites the ring
  }
}

template <class E, bool EXACT, int N = 1>
const void* s3d_kernel_for(int ntaps) {
  if constexpr (N > kGenMaxNT) {
    return (const void*)k_generic_s3d<E, EXACT, 0>;
  } else {
    if (ntaps == N) return (const void*)k_generic_s3d<E, EXACT, N>;
    return s3d_kernel_for<E, EXACT, N + 1>(ntaps);
  }
}

cudaError_t launch_generic_s3d(const GenS3DArgs& a, int elem, bool exact, int grid, int smem,
                               cudaStream_t st) {
  const void* fn;
  if (elem == 4)
    fn = exact ? s3d_kernel_for<float, true>(a.ntaps) : s3d_kernel_for<float, false>(a.ntaps);
  else
    fn = exact ? s3d_kernel_for<double, true>(a.ntaps) : s3d_kernel_for<double, false>(a.ntaps);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  void* args[] = {const_cast<GenS3DArgs*>(&a)};
  e = cudaLaunchKernel(fn, dim3(grid), dim3(kGenS3DThreads), args, (size_t)smem, st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

// kernel for (E, EXACT, ntaps): unrolled for 1..kGenMaxNT taps
template <class E, bool EXACT, int N = 1>
const void* generic_kernel_for(int ntaps) {
  if constexpr (N > kGenMaxNT) {
    return (const void*)k_generic_tb<E, EXACT, 0>;
  } else {
    if (ntaps == N) return (const void*)k_generic_tb<E, EXACT, N>;
    return generic_kernel_for<E, EXACT, N + 1>(ntaps);
  }
}

template <class E>
cudaError_t launch_generic_typed(const GenArgs& a, bool exact, int grid, int threads, int smem,
                                 cudaStream_t st) {
  const void* fn = exact ? generic_kernel_for<E, true>(a.ntaps) : generic_kernel_for<E, false>(a.ntaps);
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  void* args[] = {const_cast<GenArgs*>(&a)};
  e = cudaLaunchKernel(fn, dim3(grid), dim3(threads), args, (size_t)smem, st);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

cudaError_t launch_generic_tb(const GenArgs& a, int elem, bool exact, int grid, int threads,
                              int smem, cudaStream_t st) {
  if (elem == 4) return launch_generic_typed<float>(a, exact, grid, threads, smem, st);
  return launch_generic_typed<double>(a, exact, grid, threads, smem, st);
}

int generic_threads() { return kGenThreads; }

}  // namespace ebisu

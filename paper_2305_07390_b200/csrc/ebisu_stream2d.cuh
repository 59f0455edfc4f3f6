// ebisu_stream2d.cuh -- 2-D temporal-blocking sweep for sm_100a.
//
// Replaces the reference's overlapped-tiling engine (engine/sm.py:95-206,
// "SM tiling": each block loads core + rad*t per tiled side, streams axis 0
// through a circular multi-queue, fuses t levels, stores only the core) with
// a B200 design:
//
//  * Work unit = (warp strip, row segment).  A warp strip is 32*C columns
//    loaded, VW = 32*C - 2*T*R of them valid after T fused levels; row
//    segments split axis 0 so that >= 148 SMs x resident warps have work
//    (SURVEY.md §7 hard part 3).  Every warp is an autonomous overlapped
//    tile: no __syncthreads and no cross-warp traffic inside an epoch.
//  * Rows move HBM -> shared memory by TMA (cp.async.bulk.tensor.2d, one
//    32*C-double box per row; out-of-bounds columns are zero-filled) into a
//    per-warp S-slot mbarrier ring: the circular multi-queue of
//    multiqueue.py:103-211 with power-of-two slots and mask addressing.
//  * Each lane owns C consecutive columns.  The T levels are kept as
//    register windows of 2R+1 rows per level (the "RST" register streaming
//    of engine/rst.py, taken to its limit): level s at advance k consumes
//    rows k-(s+1)R .. k-(s-1)R of level s-1 and emits row k-sR.  The advance
//    loop is unrolled by 2R+1 so window slots are compile-time registers
//    (no moves).  Horizontal neighbours outside the lane come from warp
//    shuffles.
//  * Dirichlet frame (distance < R from a face): a frame cell at level s
//    equals its value at level s-1, i.e. the centre of the window -- no
//    stored copy of the input is needed (common.py:96-112 semantics).
//  * Level T rows are stored straight to HBM for the valid core columns.
//  * Epochs (T fused steps each) run inside one cooperative launch separated
//    by grid.sync(), or one launch per epoch.
//
// Exactness: taps are summed in catalog order with __dmul_rn/__dadd_rn
// (EXACT) -> bitwise equal to reference_run (grid.py:76-113).
#pragma once

#include <cooperative_groups.h>

#include "ebisu_common.cuh"
#include "ebisu_shapes.cuh"

namespace ebisu {

struct Stream2DArgs {
  int n0, n1;        // extents (axis 0 rows, axis 1 columns); row pitch = n1
  int nstrips;       // warp strips along axis 1
  int nseg;          // row segments along axis 0
  int seg_len;       // rows per segment
  int epochs;        // fused epochs in this launch
  int first_src;     // BufId of epoch 0's source
  int first_dst;     // BufId of epoch 0's destination
  double* buf[3];    // device pointers by BufId
};

template <class SH, int T, int C, int NW, int S>
struct Stream2DCfg {
  static constexpr int R = SH::R;
  static constexpr int W = 2 * R + 1;       // window rows per level
  static constexpr int LC = 32 * C;         // loaded columns per warp
  // Column halo rounded up to even: a TMA box must start on a 16-byte
  // boundary in the innermost dimension (2 doubles).
  static constexpr int HX = (T * R + 1) & ~1;
  static constexpr int VW = LC - 2 * HX;    // valid columns per warp (even)
  static constexpr int ROW_BYTES = LC * 8;
  static constexpr int RING_BYTES = S * ROW_BYTES;
  static constexpr int SMEM_BYTES = NW * RING_BYTES + NW * S * 8;
  static_assert(VW > 0, "tile leaves no valid core");
  static_assert((S & (S - 1)) == 0, "ring slots must be a power of two");
  static_assert(LC <= 256, "TMA box inner dimension is limited to 256 elements");
};

// Does any tap in row dy have a nonzero column offset?
template <class SH>
__host__ __device__ constexpr bool row_has_halo(int dy) {
  for (int i = 0; i < SH::NT; ++i)
    if (SH::tap(i).d0 == dy && SH::tap(i).d1 != 0) return true;
  return false;
}

template <int W>
__host__ __device__ constexpr int pmod(int a) {
  return ((a % W) + W) % W;
}

// One work unit (warp strip x row segment) of one epoch.  EDGE = the unit
// owns frame cells (top/bottom segment, first/last strip): only then are the
// frame-row branches and frame-column selects compiled in; interior units run
// the pure tap pipeline.
template <class SH, int T, int C, int S, bool EXACT, bool EDGE>
__device__ __forceinline__ void stream2d_unit(const CUtensorMap* tm, double* __restrict__ out,
                                              double* ring, uint64_t* bars, uint32_t ring_cnt,
                                              int lane, int n0, int n1, int X0, int r0, int r1,
                                              const Coefs<SH::NT>& cf) {
  constexpr int R = SH::R;
  constexpr int W = 2 * R + 1;
  constexpr int LC = 32 * C;
  constexpr int ROW_BYTES = LC * 8;
  constexpr int TR = T * R;
  constexpr int HX = (TR + 1) & ~1;
  constexpr int VW = LC - 2 * HX;

  const int ka = max(0, r0 - TR);
  const int kb = min(n0, r1 + TR);
  const int kend = r1 + TR;

  // Prologue: fill the ring S rows ahead.
  if (lane == 0) {
    for (int i = 0; i < S && ka + i < kb; ++i) {
      const uint32_t slot = (ring_cnt + i) & (S - 1);
      mbar_arrive_expect_tx(&bars[slot], ROW_BYTES);
      tma_load_2d(ring + slot * LC, tm, X0, ka + i, &bars[slot]);
    }
  }

  bool fcol[C];   // frame column (EDGE only)
  bool stcol[C];  // stored (valid core) column
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int lc = lane * C + c;
    const int x = X0 + lc;
    fcol[c] = EDGE && ((x < R) || (x >= n1 - R));
    stcol[c] = (lc >= HX) && (lc < HX + VW) && (x < n1);
  }

  double win[T][W][C];
#pragma unroll
  for (int s = 0; s < T; ++s)
#pragma unroll
    for (int w = 0; w < W; ++w)
#pragma unroll
      for (int c = 0; c < C; ++c) win[s][w][c] = 0.0;

  for (int kbase = ka; kbase < kend; kbase += W) {
#pragma unroll
    for (int uu = 0; uu < W; ++uu) {
      const int k = kbase + uu;
      // ---- level 0: next input row from the TMA ring ----------------------
      // (the select keeps the window write unconditional, so the dead oldest
      // row never stays live across the advance)
      {
        double v[C];
        if (k < kb) {
          const uint32_t pos = ring_cnt + (uint32_t)(k - ka);
          const uint32_t slot = pos & (S - 1);
          mbar_wait(&bars[slot], (pos / S) & 1);
          // Refill the slot consumed one advance ago: its LDS results have
          // been used by now, so the async-proxy write cannot overtake the
          // generic-proxy read (no proxy fence on the hot path).
          if (lane == 0 && k > ka && k - 1 + S < kb) {
            const uint32_t ps = (pos - 1) & (S - 1);
            mbar_arrive_expect_tx(&bars[ps], ROW_BYTES);
            tma_load_2d(ring + ps * LC, tm, X0, k - 1 + S, &bars[ps]);
          }
          const double* rowp = ring + slot * LC + lane * C;
          if constexpr (C % 2 == 0) {
#pragma unroll
            for (int c = 0; c < C; c += 2) {
              const double2 t2 = *reinterpret_cast<const double2*>(rowp + c);
              v[c] = t2.x;
              v[c + 1] = t2.y;
            }
          } else {
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = rowp[c];
          }
        } else {
#pragma unroll
          for (int c = 0; c < C; ++c) v[c] = 0.0;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) win[0][uu][c] = v[c];
      }
      // ---- levels 1..T ----------------------------------------------------
      // Every level runs every advance.  During pipeline warm-up a level's
      // target row is not yet valid (it depends on rows before ka) and it
      // computes values that no valid row ever consumes: level s row q is
      // valid iff q >= ka + s*R (or the segment starts at the top frame), and
      // level s+1 only reads rows >= q' - R of it.
      static_for<T>([&](auto sI) {
        constexpr int s = decltype(sI)::value + 1;  // level being produced
        const int q = k - s * R;                    // its target row
        double nv[C];
        bool frame_row = false;
        if constexpr (EDGE) frame_row = (q < R) || (q >= n0 - R);
        if (frame_row) {
          // frame row (or warm-up row outside the grid): value carries over
#pragma unroll
          for (int c = 0; c < C; ++c) nv[c] = win[s - 1][pmod<W>(uu - s * R)][c];
        } else {
          // horizontal halos (only rows whose taps leave the lane's columns)
          double hl[W][R], hr[W][R];
          static_for<W>([&](auto wI) {
            constexpr int dy = decltype(wI)::value - R;
            if constexpr (row_has_halo<SH>(dy)) {
              static_for<R>([&](auto jI) {
                constexpr int j = decltype(jI)::value;
                constexpr int ccl = -R + j;
                constexpr int dl = (-ccl + C - 1) / C;
                constexpr int coll = ccl + dl * C;
                constexpr int ccr = C + j;
                constexpr int dr = ccr / C;
                constexpr int colr = ccr - dr * C;
                const int sl = pmod<W>(uu - s * R + dy);
                hl[wI][j] = __shfl_up_sync(kFullMask, win[s - 1][sl][coll], dl);
                hr[wI][j] = __shfl_down_sync(kFullMask, win[s - 1][sl][colr], dr);
              });
            }
          });
#pragma unroll
          for (int c = 0; c < C; ++c) {
            double acc = 0.0;
            static_for<SH::NT>([&](auto iI) {
              constexpr int i = decltype(iI)::value;
              constexpr Off o = SH::tap(i);
              const int sl = pmod<W>(uu - s * R + o.d0);
              const int cc = c + o.d1;
              double x;
              if (cc < 0)
                x = hl[o.d0 + R][cc + R];
              else if (cc >= C)
                x = hr[o.d0 + R][cc - C];
              else
                x = win[s - 1][sl][cc];
              if constexpr (i == 0)
                acc = tap_first<EXACT>(cf.c[0], x);
              else
                acc = tap_next<EXACT>(acc, cf.c[i], x);
            });
            if constexpr (EDGE)
              nv[c] = fcol[c] ? win[s - 1][pmod<W>(uu - s * R)][c] : acc;
            else
              nv[c] = acc;
          }
        }
        if constexpr (s < T) {
#pragma unroll
          for (int c = 0; c < C; ++c) win[s][pmod<W>(uu - s * R)][c] = nv[c];
        } else {
          if (q >= r0 && q < r1) {
            double* orow = out + (size_t)q * (size_t)n1 + (X0 + lane * C);
#pragma unroll
            for (int c = 0; c < C; ++c)
              if (stcol[c]) orow[c] = nv[c];
          }
        }
      });
    }
  }
}

template <class SH, int T, int C, int NW, int S, bool EXACT, int MINB>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_stream2d(const __grid_constant__ TmapSet maps, const Stream2DArgs a,
               const __grid_constant__ Coefs<SH::NT> cf) {
  using Cfg = Stream2DCfg<SH, T, C, NW, S>;
  constexpr int R = Cfg::R;
  constexpr int VW = Cfg::VW;
  constexpr int TR = T * R;
  constexpr int HX = Cfg::HX;

  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  double* ring = reinterpret_cast<double*>(smem + warp * Cfg::RING_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + NW * Cfg::RING_BYTES) + warp * S;

  if (lane == 0) {
#pragma unroll
    for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
    fence_mbarrier_init();
    prefetch_tmap(&maps.m[0]);
    prefetch_tmap(&maps.m[1]);
    prefetch_tmap(&maps.m[2]);
  }
  __syncwarp();

  const int n0 = a.n0, n1 = a.n1;
  const int gwarp = blockIdx.x * NW + warp;
  const int nwarps = gridDim.x * NW;
  const int units = a.nstrips * a.nseg;
  uint32_t ring_cnt = 0;  // rows consumed so far by this warp (ring position)

  int src = a.first_src, dst = a.first_dst;
  for (int e = 0; e < a.epochs; ++e) {
    const CUtensorMap* tm = &maps.m[src];
    double* __restrict__ out = (dst == BUF_OUT) ? a.buf[BUF_OUT] : a.buf[BUF_SCR];

    for (int u = gwarp; u < units; u += nwarps) {
      const int strip = u % a.nstrips;
      const int seg = u / a.nstrips;
      const int X0 = strip * VW - HX;  // global column of loaded column 0 (even)
      const int r0 = seg * a.seg_len;
      const int r1 = min(n0, r0 + a.seg_len);
      const int ka = max(0, r0 - TR);
      const int kb = min(n0, r1 + TR);
      // Frame cells inside this unit's dependency cone (valid range +- T*R)?
      // Only then must frame rows/columns be carried instead of computed.
      const bool edge = (r0 - TR < R) || (r1 + TR > n0 - R) || (strip * VW - TR < R) ||
                        ((strip + 1) * VW + TR > n1 - R);
      if (__shfl_sync(kFullMask, edge, 0))
        stream2d_unit<SH, T, C, S, EXACT, true>(tm, out, ring, bars, ring_cnt, lane, n0, n1,
                                                X0, r0, r1, cf);
      else
        stream2d_unit<SH, T, C, S, EXACT, false>(tm, out, ring, bars, ring_cnt, lane, n0, n1,
                                                 X0, r0, r1, cf);
      ring_cnt += (uint32_t)(kb - ka);
    }

    if (e + 1 < a.epochs) {
      // Make this epoch's generic-proxy stores visible to the next epoch's
      // TMA (async-proxy) loads issued by other CTAs.
      fence_proxy_async_global();
      __threadfence();
      cooperative_groups::this_grid().sync();
      fence_proxy_async_global();
    }
    const int nsrc = dst;
    dst = (dst == BUF_OUT) ? BUF_SCR : BUF_OUT;
    src = nsrc;
  }
}

}  // namespace ebisu

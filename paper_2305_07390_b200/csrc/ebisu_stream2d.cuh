// ebisu_stream2d.cuh -- 2-D temporal-blocking sweep for sm_100a.
//
// Replaces the reference's overlapped-tiling engine (engine/sm.py:95-206,
// "SM tiling": each block loads core + rad*t per tiled side, streams axis 0
// through a circular multi-queue, fuses t levels, stores only the core) with
// a B200 design:
//
//  * Work unit = (warp strip, row segment).  A warp strip is LC = 32*C
//    columns loaded, VW = LC - 2*HX of them valid after T fused levels
//    (HX = T*R rounded up to even); row segments split axis 0 so that every
//    resident warp has work (SURVEY.md §7 hard part 3).  Every warp is an
//    autonomous overlapped tile: no __syncthreads, no cross-warp traffic
//    inside an epoch.
//  * Rows move HBM -> shared memory by TMA (cp.async.bulk.tensor.2d, one
//    LC-double box per row; out-of-bounds columns are zero-filled) into a
//    per-warp S-slot mbarrier ring: the circular multi-queue of
//    multiqueue.py:103-211 with power-of-two slots and mask addressing.
//  * Each lane owns C consecutive columns.  The T levels are register
//    windows of 2R+1 rows per level (the "RST" register streaming of
//    engine/rst.py, taken to its limit): level s at advance k consumes rows
//    k-(s+1)R .. k-(s-1)R of level s-1 and emits row k-sR.  The advance loop
//    is unrolled by 2R+1 so window slots are compile-time registers.
//    Horizontal neighbours outside the lane come from warp shuffles.
//  * Dirichlet frame (distance < R from a face): a frame cell at level s
//    equals its value at level s-1 (the window centre), common.py:96-112.
//    Strip geometry is aligned to the domain edges -- strip 0 starts at
//    column 0, the last strip ends at column n1 -- so frame columns only ever
//    sit in lane 0's first R cells or lane 31's last R cells (2R predicated
//    selects per level, edge strips only); frame rows only occur in the
//    first/last unrolled blocks of the top/bottom segment, which run a
//    select variant of the block.  Interior work carries no frame logic, so
//    edge units cost the same as interior ones and no epoch waits on them.
//  * Level T rows are stored straight to HBM for the unit's valid columns.
//  * Epochs (T fused steps each) run inside one cooperative launch separated
//    by grid.sync(), or one launch per epoch.
//
// Exactness: taps are summed in catalog order with __dmul_rn/__dadd_rn
// (EXACT) -> bitwise equal to reference_run (grid.py:76-113).
#pragma once

#include <cooperative_groups.h>

#include <type_traits>

#include "ebisu_common.cuh"
#include "ebisu_shapes.cuh"

namespace ebisu {

struct Stream2DArgs {
  int n0, n1;        // extents (axis 0 rows, axis 1 columns); row pitch = n1
  int nstrips;       // warp strips along axis 1
  int nseg;          // row segments along axis 0
  int seg_len;       // rows per segment
  int z_lo, z_hi;    // output rows [z_lo, z_hi) (segments tile this range)
  // row segment j = [seg_start[j], seg_start[j+1]); guided schedule (long
  // segments handed out first, short ones at the epoch tail), as in 3-D
  int seg_start[EBISU_MAX_SEGS + 1];
  int epochs;        // fused epochs in this launch
  int first_src;     // BufId of epoch 0's source
  int first_dst;     // BufId of epoch 0's destination
  int aligned;       // 1: edge-aligned strips (n1 >= 2*LC); 0: generic strips
  int pitch;         // row pitch of every buffer (elements, >= n1; > n1 = padded rows)
  void* buf[3];      // device pointers by BufId (element type E of the kernel)
  long long* unit_clock;  // optional profiling: [units][2] start/end globaltimer (ns)
  int* work;         // per-epoch unit counters (dynamic scheduling), zeroed by the host
  // Dataflow epochs (non-null, cooperative launch): flags[u] = epochs unit u
  // has completed.  A unit of epoch e waits only for the epoch-(e-1) units
  // whose outputs it reads (its strip +-2, the segments within T*R rows) --
  // the same units that read what it overwrites, so RAW and WAR are both
  // covered -- instead of a grid-wide barrier: warps that finish an epoch
  // early start the next one (no epoch tail).  Deadlock-free: units are
  // claimed epoch by epoch, so every dependency is held by a resident warp.
  int* flags;
};

template <class SH, int T, int C, int NW, int S, class E = double>
struct Stream2DCfg {
  static constexpr int R = SH::R;
  static constexpr int W = 2 * R + 1;       // window rows per level
  static constexpr int LC = 32 * C;         // loaded columns per warp
  // Column halo rounded up to even: a TMA box must start on a 16-byte
  // boundary in the innermost dimension (2 doubles / 4 floats).
  static constexpr int AL = 16 / (int)sizeof(E);
  static constexpr int HX = (T * R + AL - 1) / AL * AL;
  static constexpr int VW = LC - 2 * HX;    // valid columns per warp (even)
  static constexpr int ROW_BYTES = LC * (int)sizeof(E);
  static constexpr int RING_BYTES = S * ROW_BYTES;
  static constexpr int SMEM_BYTES = NW * RING_BYTES + NW * S * 8;
  static_assert(VW > 0, "tile leaves no valid core");
  static_assert((S & (S - 1)) == 0, "ring slots must be a power of two");
  static_assert(LC <= 256, "TMA box inner dimension is limited to 256 elements");
};

// Strip geometry shared by host and device.  Aligned mode (n1 >= 2*LC):
//   strip 0      X0 = 0,          valid [0, VW+HX)
//   strip j      X0 = j*VW,       valid [j*VW+HX, (j+1)*VW+HX) clipped at xl
//   last strip   X0 = xlast,      valid [xl, n1),  xl = xlast+HX
//                (xlast = n1-LC rounded up to the TMA alignment)
// Generic mode: X0 = j*VW-HX, valid [j*VW, (j+1)*VW) clipped at n1.
struct StripGeom {
  int X0, vlo, vhi;
  int fc;  // frame columns: 0 none, 1 lane-0 left, 2 lane-31 right, 3 generic
};

// Start of the last strip in aligned mode: n1 - LC rounded UP to the TMA
// alignment AL (elements per 16 bytes; 1 for axes other than the innermost).
// With an even last extent that is n1 - LC exactly; with a padded odd extent
// the last strip overhangs the domain by < AL columns (TMA zero-fills them;
// they feed no stored cell: frame columns only carry their value).
__host__ __device__ inline int strip_last_x0(int n1, int LC, int AL) {
  return (n1 - LC + AL - 1) / AL * AL;
}

__host__ __device__ inline int stream2d_nstrips(int n1, int LC, int VW, int HX, int R, int C,
                                                int* aligned, int AL = 1) {
  if (n1 >= 2 * LC && R <= C) {
    *aligned = 1;
    // columns [VW+HX, xlast+HX) for middle strips
    const int mid = strip_last_x0(n1, LC, AL) - VW;
    return 2 + (mid > 0 ? (mid + VW - 1) / VW : 0);
  }
  *aligned = 0;
  return (n1 + VW - 1) / VW;
}

__host__ __device__ inline StripGeom stream2d_strip(int j, int nstrips, int aligned, int n1,
                                                    int LC, int VW, int HX, int AL = 1) {
  StripGeom g;
  if (aligned) {
    const int xlast = strip_last_x0(n1, LC, AL);
    const int xl = xlast + HX;
    if (j == nstrips - 1) {
      g.X0 = xlast;
      g.vlo = xl;
      g.vhi = n1;
      // frame columns in lane 31's last R cells only when the strip ends at n1
      g.fc = xlast == n1 - LC ? 2 : 3;
    } else {
      g.X0 = j * VW;
      g.vlo = j == 0 ? 0 : j * VW + HX;
      g.vhi = min((j + 1) * VW + HX, xl);
      g.fc = j == 0 ? 1 : 0;
    }
  } else {
    g.X0 = j * VW - HX;
    g.vlo = j * VW;
    g.vhi = min((j + 1) * VW, n1);
    g.fc = 3;
  }
  return g;
}

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


// ---- tolerance mode (exact = 0, uniform coefficients): reassociated sums ----
// sum_k c*x_k = c * sum_k x_k may be regrouped within the north star's fp64
// tolerance (1e-12 relative).  Stars: sum = column sum over 2R+1 rows + row
// sum over 2R+1 columns - centre; boxes: row sum of the column sums.  Both
// are sliding sums of K = 2R+1 terms for 4 consecutive outputs (4 target
// rows of a block, 4 cells of a lane), computed with shared partial sums:
// K + 4 adds for 4 outputs instead of 4(K-1), no subtraction, no drift.
// j2ds25pt: 11.5 DP per cell-step instead of 25.
template <class SH>
__host__ __device__ constexpr bool ra2d_star() {
  // star pattern in reference order: column -R..R then row offsets
  if (!SH::kStar || SH::dims != 2) return false;
  return true;
}
template <class SH>
__host__ __device__ constexpr bool ra2d_box() {
  return !SH::kStar && SH::dims == 2 && SH::NT == (2 * SH::R + 1) * (2 * SH::R + 1);
}
template <class SH>
__host__ __device__ constexpr bool ra2d_eligible() {
  return ra2d_star<SH>() || ra2d_box<SH>();
}
// pairwise sum of a[0..N-1] (short dependency chains)
template <int N, class E>
__device__ __forceinline__ E tree_sum(const E* a) {
  E part[N];
#pragma unroll
  for (int j = 0; j < N; ++j) part[j] = a[j];
#pragma unroll
  for (int w = 1; w < N; w *= 2)
#pragma unroll
    for (int j = 0; j + w < N; j += 2 * w) part[j] = add_rn<E>(part[j], part[j + w]);
  return part[0];
}
// o[i] = a[i] + ... + a[i+K-1], i = 0..1 (a has K+1 entries): K adds
template <int K, class E>
__device__ __forceinline__ void slide2(const E* a, E* o) {
  const E core = tree_sum<K - 1>(a + 1);
  o[0] = add_rn<E>(a[0], core);
  o[1] = add_rn<E>(core, a[K]);
}
// o[i] = a[i] + ... + a[i+K-1], i = 0..3 (a has K+3 entries)
template <int K, class E>
__device__ __forceinline__ void slide4(const E* a, E* o) {
  static_assert(K >= 3, "window of at least 3");
  E core = E(0);
  if constexpr (K > 3) {
    // a[3..K-1], pairwise (short dependency chains)
    E part[(K - 3 + 1) / 2];
#pragma unroll
    for (int j = 0; j < (K - 3) / 2; ++j) part[j] = add_rn<E>(a[3 + 2 * j], a[4 + 2 * j]);
    if constexpr ((K - 3) % 2) part[(K - 3) / 2] = a[K - 1];
    constexpr int NP = (K - 3 + 1) / 2;
#pragma unroll
    for (int w = 1; w < NP; w *= 2)
#pragma unroll
      for (int j = 0; j + w < NP; j += 2 * w) part[j] = add_rn<E>(part[j], part[j + w]);
    core = part[0];
  }
  const E l1 = K > 3 ? add_rn<E>(core, a[2]) : a[2];
  const E l2 = add_rn<E>(l1, a[1]);
  o[0] = add_rn<E>(l2, a[0]);
  o[1] = add_rn<E>(l2, a[K]);
  const E p = add_rn<E>(a[K], a[K + 1]);
  o[2] = add_rn<E>(l1, p);
  o[3] = add_rn<E>(K > 3 ? add_rn<E>(core, p) : p, a[K + 2]);
}
template <int K, int N, class E>
__device__ __forceinline__ void slide_n(const E* a, E* o) {
  static_assert(N == 2 || N == 4, "2 or 4 outputs");
  if constexpr (N == 2)
    slide2<K>(a, o);
  else
    slide4<K>(a, o);
}

// One work unit (warp strip x row segment) of one epoch.  FC selects the
// frame-column handling (see StripGeom); frame rows are handled per block.
template <class SH, int T, int C, int S, bool EXACT, bool UNI, int FC, class E, int SHIFT = 0>
__device__ __forceinline__ int stream2d_unit(const CUtensorMap* tm, E* __restrict__ out,
                                              E* ring, uint64_t* bars, uint32_t ring_cnt,
                                              int lane, int n0, int n1, int pitch, const StripGeom& g,
                                              int r0, int r1, const Coefs<SH::NT, E>& cf) {
  constexpr int R = SH::R;
  constexpr int W = 2 * R + 1;
  constexpr int LC = 32 * C;
  constexpr int ROW_BYTES = LC * (int)sizeof(E);
  constexpr int TR = T * R;
  static_assert(FC == 0 || FC == 3 || R <= C, "frame columns must fit in one lane");

  const int X0 = g.X0;
  const int ka = max(0, r0 - TR);
  const int kend = r1 + TR;
  // rows [ka, kload) are all loaded (whole unrolled blocks): TMA zero-fills
  // rows >= n0, and rows >= r1 + T*R only feed target rows >= r1, which are
  // never stored -- so the level-0 read needs no branch
  constexpr int UWC = SHIFT ? SHIFT : 2 * R + 1;
  const int kload = ka + (kend - ka + UWC - 1) / UWC * UWC;

  // Prologue: fill the ring S rows ahead.
  if (lane == 0) {
    for (int i = 0; i < S && ka + i < kload; ++i) {
      const uint32_t slot = (ring_cnt + i) & (S - 1);
      mbar_arrive_expect_tx(&bars[slot], ROW_BYTES);
      tma_load_2d(ring + slot * LC, tm, X0, ka + i, &bars[slot]);
    }
  }

  bool fcol[C];   // this lane's frame columns
  bool stcol[C];  // stored (valid) columns
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int x = X0 + lane * C + c;
    if constexpr (FC == 1)
      fcol[c] = (c < R) && (lane == 0);
    else if constexpr (FC == 2)
      fcol[c] = (c >= C - R) && (lane == 31);
    else if constexpr (FC == 3)
      fcol[c] = (x < R) || (x >= n1 - R);
    else
      fcol[c] = false;
    stcol[c] = (x >= g.vlo) && (x < g.vhi);
  }
  // compile-time: which columns may hold frame cells
  auto col_may_frame = [](int c) constexpr {
    return FC == 3 || (FC == 1 && c < R) || (FC == 2 && c >= C - R);
  };

  // SHIFT = U > 0: W + U - 1 slots per level (the W - 1 carried rows and the
  // U rows produced by one unrolled block)
  constexpr int WS = SHIFT ? W + SHIFT - 1 : W;
  E win[T][WS][C];
#pragma unroll
  for (int s = 0; s < T; ++s)
#pragma unroll
    for (int w = 0; w < WS; ++w)
#pragma unroll
      for (int c = 0; c < C; ++c) win[s][w][c] = 0.0;

  // One unrolled block of UW advances.  FROWS: some target row in this block
  // may be a frame row (only near the top/bottom of the grid).
  //   rotating windows (SHIFT = 0): UW = W advances per block, row q+dy of
  //     level s-1 sits in slot (k - s*R + dy) mod W, a compile-time register;
  //   shifted windows (SHIFT = U, large radii): UW = U advances per block;
  //     inner advance uu writes its row to slot W-1+uu and reads row q+dy
  //     from slot R+dy+uu; after the block the window shifts down by U
  //     ((W-1)*C register moves per U advances).  The code is W/U times
  //     smaller than the rotating version, which for W = 13 keeps the loop in
  //     the instruction cache (the rotating kernel measured 11.6 %
  //     no-instruction stalls at R = 6).
  constexpr int UW = SHIFT ? SHIFT : W;
  // tolerance mode (exact = 0, uniform coefficients): reassociated sums
  constexpr bool RA = UNI && !EXACT;
  static_assert(!RA || C == 4, "reassociated kernels: 4 cells per lane");
  auto slot_of = [](int uu, int s, int dy) {
    return SHIFT ? R + dy + uu : pmod<W>(uu - s * R + dy);
  };
  auto put = [&](auto lvl_tag, int uu, const E (&v)[C]) {
    constexpr int L = decltype(lvl_tag)::value;
    if constexpr (SHIFT) {
#pragma unroll
      for (int c = 0; c < C; ++c) win[L][W - 1 + uu][c] = v[c];
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c) win[L][pmod<W>(uu - L * R)][c] = v[c];
    }
  };
  auto block = [&](int kbase, auto frows_tag) {
    constexpr bool FROWS = decltype(frows_tag)::value;
#pragma unroll
    for (int uu = 0; uu < UW; ++uu) {
      const int k = kbase + uu;
      // ---- level 0: next input row from the TMA ring ----------------------
      // (the select keeps the window write unconditional, so the dead oldest
      // row never stays live across the advance)
      {
        E v[C];
        {
          const uint32_t pos = ring_cnt + (uint32_t)(k - ka);
          const uint32_t slot = pos & (S - 1);
          mbar_wait(&bars[slot], (pos / S) & 1);
          // Refill the slot consumed one advance ago: its LDS results have
          // been used by now, so the async-proxy write cannot overtake the
          // generic-proxy read (no proxy fence on the hot path).
          if (lane == 0 && k > ka && k - 1 + S < kload) {
            const uint32_t ps = (pos - 1) & (S - 1);
            mbar_arrive_expect_tx(&bars[ps], ROW_BYTES);
            tma_load_2d(ring + ps * LC, tm, X0, k - 1 + S, &bars[ps]);
          }
          const E* rowp = ring + slot * LC + lane * C;
          if constexpr (C % 2 == 0) {
#pragma unroll
            for (int c = 0; c < C; c += 2) {
              const vec2_t<E> t2 = *reinterpret_cast<const vec2_t<E>*>(rowp + c);
              v[c] = t2.x;
              v[c + 1] = t2.y;
            }
          } else {
#pragma unroll
            for (int c = 0; c < C; ++c) v[c] = rowp[c];
          }
        }
        // UNI: the window holds products y = c*x (one DMUL per cell per level)
#pragma unroll
        for (int c = 0; c < C; ++c) v[c] = UNI ? mul_rn<E>(cf.c[0], v[c]) : v[c];
        put(std::integral_constant<int, 0>{}, uu, v);
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
        // horizontal halos (only rows whose taps leave the lane's columns)
        E hl[W][R], hr[W][R];
        static_for<W>([&](auto wI) {
          constexpr int dy = decltype(wI)::value - R;
          if constexpr (!RA && row_has_halo<SH>(dy)) {
            static_for<R>([&](auto jI) {
              constexpr int j = decltype(jI)::value;
              constexpr int ccl = -R + j;
              constexpr int dl = (-ccl + C - 1) / C;
              constexpr int coll = ccl + dl * C;
              constexpr int ccr = C + j;
              constexpr int dr = ccr / C;
              constexpr int colr = ccr - dr * C;
              const int sl = slot_of(uu, s, dy);
              hl[wI][j] = __shfl_up_sync(kFullMask, win[s - 1][sl][coll], dl);
              hr[wI][j] = __shfl_down_sync(kFullMask, win[s - 1][sl][colr], dr);
            });
          }
        });
        // tap-major order: the C per-column chains are independent
        E acc[C];
        if constexpr (RA) {
          // tolerance mode: column sums over the 2R+1 window rows (pairwise),
          // then 2R+1-column row sums of the centre row (stars, + column sum
          // - centre) or of the column sums (boxes), see slide4
          E b[2 * R + C];
#pragma unroll
          for (int c = 0; c < C; ++c) {
            E part[W];
#pragma unroll
            for (int j = 0; j < W; ++j) part[j] = win[s - 1][slot_of(uu, s, j - R)][c];
#pragma unroll
            for (int w = 1; w < W; w *= 2)
#pragma unroll
              for (int j = 0; j + w < W; j += 2 * w) part[j] = add_rn<E>(part[j], part[j + w]);
            acc[c] = part[0];
            b[R + c] = ra2d_box<SH>() ? part[0] : win[s - 1][slot_of(uu, s, 0)][c];
          }
          static_for<R>([&](auto jI) {
            constexpr int j = decltype(jI)::value;
            constexpr int ccl = -R + j;
            constexpr int dl = (-ccl + C - 1) / C;
            constexpr int coll = ccl + dl * C;
            constexpr int ccr = C + j;
            constexpr int dr = ccr / C;
            constexpr int colr = ccr - dr * C;
            b[j] = __shfl_up_sync(kFullMask, b[R + coll], dl);
            b[R + C + j] = __shfl_down_sync(kFullMask, b[R + colr], dr);
          });
          E h[4];
          slide4<W>(b, h);
#pragma unroll
          for (int c = 0; c < C; ++c)
            acc[c] = ra2d_box<SH>() ? h[c] : add_rn<E>(acc[c], sub_rn<E>(h[c], b[R + c]));
        } else
        static_for<SH::NT>([&](auto iI) {
          constexpr int i = decltype(iI)::value;
          constexpr Off o = SH::tap(i);
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const int sl = slot_of(uu, s, o.d0);
            const int cc = c + o.d1;
            E x;
            if (cc < 0)
              x = hl[o.d0 + R][cc + R];
            else if (cc >= C)
              x = hr[o.d0 + R][cc - C];
            else
              x = win[s - 1][sl][cc];
            if constexpr (UNI)
              acc[c] = (i == 0) ? x : add_rn<E>(acc[c], x);
            else if constexpr (i == 0)
              acc[c] = tap_first<EXACT>(cf.c[0], x);
            else
              acc[c] = tap_next<EXACT>(acc[c], cf.c[i], x);
          }
        });
        // frame cells carry level s-1's centre (branch-free selects); in UNI
        // mode the carried centre is the product c*x, which is the frame's
        // product at every level, and level T never stores frame cells (the
        // host pre-copies the frame into both ping-pong buffers)
        E nv[C];
        bool frow = false;
        if constexpr (FROWS) frow = (q < R) || (q >= n0 - R);
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const E centre = win[s - 1][slot_of(uu, s, 0)][c];
          const E val = (UNI && s < T) ? mul_rn<E>(cf.c[0], acc[c]) : acc[c];
          if (FROWS && col_may_frame(c))
            nv[c] = (frow || fcol[c]) ? centre : val;
          else if (FROWS)
            nv[c] = frow ? centre : val;
          else if (col_may_frame(c))
            nv[c] = fcol[c] ? centre : val;
          else
            nv[c] = val;
        }
        if constexpr (s < T) {
          put(std::integral_constant<int, s>{}, uu, nv);
        } else {
          if (q >= r0 && q < r1) {
            E* orow = out + (size_t)q * (size_t)pitch + (X0 + lane * C);
            bool st[C];
#pragma unroll
            for (int c = 0; c < C; ++c) {
              st[c] = stcol[c];
              if constexpr (UNI) {
                if (FROWS) st[c] = st[c] && !frow;
                if (col_may_frame(c)) st[c] = st[c] && !fcol[c];
              }
            }
            if constexpr (C % 2 == 0) {
              // 16-byte stores (branch free; a pair is split only at strip edges)
#pragma unroll
              for (int c = 0; c < C; c += 2) st_pair_if(orow + c, nv[c], nv[c + 1], st[c], st[c + 1]);
            } else {
#pragma unroll
              for (int c = 0; c < C; ++c)
                if (st[c]) orow[c] = nv[c];
            }
          }
        }
      });
    }
    if constexpr (SHIFT) {
      // keep the W-1 newest rows of every level for the next block
#pragma unroll
      for (int L = 0; L < T; ++L)
#pragma unroll
        for (int w = 0; w + 1 < W; ++w)
#pragma unroll
          for (int c = 0; c < C; ++c) win[L][w][c] = win[L][w + SHIFT][c];
    }
  };

  // Tolerance mode with shifted windows (large radii): level-major blocks of
  // U = 4 advances -- level 0 loads the block's 4 rows, then each level
  // completes its 4 target rows from the window (the same rows the
  // advance-major order uses), sharing the column sums of the 4 targets.
  auto block_ra = [&](int kbase, auto frows_tag) {
    constexpr bool FROWS = decltype(frows_tag)::value;
    static_assert(!(RA && SHIFT) || SHIFT == 4, "level-major blocks of 4 rows");
#pragma unroll
    for (int uu = 0; uu < UW; ++uu) {
      const int k = kbase + uu;
      const uint32_t pos = ring_cnt + (uint32_t)(k - ka);
      const uint32_t slot = pos & (S - 1);
      mbar_wait(&bars[slot], (pos / S) & 1);
      if (lane == 0 && k > ka && k - 1 + S < kload) {
        const uint32_t ps = (pos - 1) & (S - 1);
        mbar_arrive_expect_tx(&bars[ps], ROW_BYTES);
        tma_load_2d(ring + ps * LC, tm, X0, k - 1 + S, &bars[ps]);
      }
      const E* rowp = ring + slot * LC + lane * C;
#pragma unroll
      for (int c = 0; c < C; c += 2) {
        const vec2_t<E> t2 = *reinterpret_cast<const vec2_t<E>*>(rowp + c);
        win[0][W - 1 + uu][c] = mul_rn<E>(cf.c[0], t2.x);
        win[0][W - 1 + uu][c + 1] = mul_rn<E>(cf.c[0], t2.y);
      }
    }
    static_for<T>([&](auto sI) {
      constexpr int s = decltype(sI)::value + 1;
      E acc[UW][C];
      // column sums of the 4 targets (window slots uu .. uu+2R)
      E V[UW][C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        E a[W + 3], o[4];
#pragma unroll
        for (int j = 0; j < W + 3; ++j) a[j] = win[s - 1][j][c];
        slide4<W>(a, o);
#pragma unroll
        for (int uu = 0; uu < UW; ++uu) V[uu][c] = o[uu];
      }
#pragma unroll
      for (int uu = 0; uu < UW; ++uu) {
        // row sums over 2R+1 columns of the centre row (stars) or of the
        // column sums (boxes); neighbours outside the lane by shuffles
        E b[2 * R + C];
#pragma unroll
        for (int c = 0; c < C; ++c) b[R + c] = ra2d_box<SH>() ? V[uu][c] : win[s - 1][R + uu][c];
        static_for<R>([&](auto jI) {
          constexpr int j = decltype(jI)::value;
          constexpr int ccl = -R + j;
          constexpr int dl = (-ccl + C - 1) / C;
          constexpr int coll = ccl + dl * C;
          constexpr int ccr = C + j;
          constexpr int dr = ccr / C;
          constexpr int colr = ccr - dr * C;
          b[j] = __shfl_up_sync(kFullMask, b[R + coll], dl);
          b[R + C + j] = __shfl_down_sync(kFullMask, b[R + colr], dr);
        });
        E h[4];
        slide4<W>(b, h);
#pragma unroll
        for (int c = 0; c < C; ++c)
          acc[uu][c] = ra2d_box<SH>() ? h[c]
                                      : add_rn<E>(V[uu][c], sub_rn<E>(h[c], win[s - 1][R + uu][c]));
      }
#pragma unroll
      for (int uu = 0; uu < UW; ++uu) {
        const int q = kbase + uu - s * R;
        bool frow = false;
        if constexpr (FROWS) frow = (q < R) || (q >= n0 - R);
        E nv[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const E centre = win[s - 1][R + uu][c];
          const E val = s < T ? mul_rn<E>(cf.c[0], acc[uu][c]) : acc[uu][c];
          bool f = frow;
          if (col_may_frame(c)) f = f || fcol[c];
          nv[c] = f ? centre : val;
        }
        if constexpr (s < T) {
#pragma unroll
          for (int c = 0; c < C; ++c) win[s][W - 1 + uu][c] = nv[c];
        } else if (q >= r0 && q < r1 && !frow) {
          E* orow = out + (size_t)q * (size_t)pitch + (X0 + lane * C);
#pragma unroll
          for (int c = 0; c < C; c += 2) {
            const bool s0 = stcol[c] && !(col_may_frame(c) && fcol[c]);
            const bool s1 = stcol[c + 1] && !(col_may_frame(c + 1) && fcol[c + 1]);
            st_pair_if(orow + c, nv[c], nv[c + 1], s0, s1);
          }
        }
      }
    });
#pragma unroll
    for (int L = 0; L < T; ++L)
#pragma unroll
      for (int w = 0; w + 1 < W; ++w)
#pragma unroll
        for (int c = 0; c < C; ++c) win[L][w][c] = win[L][w + SHIFT][c];
  };

  for (int kbase = ka; kbase < kend; kbase += UW) {
    // target rows of this block: [kbase - TR, kbase + UW - 1 - R]
    const bool frows = (kbase - TR < R) || (kbase + UW - 1 >= n0);
    if constexpr (RA && SHIFT) {
      if (frows)
        block_ra(kbase, std::true_type{});
      else
        block_ra(kbase, std::false_type{});
    } else {
      if (frows)
        block(kbase, std::true_type{});
      else
        block(kbase, std::false_type{});
    }
  }
  return kload - ka;
}

// Warp-wide atomic grab of the next work unit (lane 0 increments).
__device__ __forceinline__ int next_unit(int* counter, int lane) {
  int u = 0;
  if (lane == 0) u = atomicAdd(counter, 1);
  return __shfl_sync(kFullMask, u, 0);
}

template <class SH, int T, int C, int NW, int S, bool EXACT, bool UNI, int MINB, class E = double,
          int SHIFT = 0>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_stream2d(const __grid_constant__ TmapSet maps, const Stream2DArgs a,
               const __grid_constant__ Coefs<SH::NT, E> cf) {
  using Cfg = Stream2DCfg<SH, T, C, NW, S, E>;
  constexpr int R = Cfg::R;
  constexpr int TR = T * R;
  // the dataflow dependency scan visits strips +-2: enough only while a
  // strip's loaded columns overlap at most its two neighbours on each side
  static_assert(3 * Cfg::HX <= Cfg::LC, "dependency scan needs HX <= VW");

  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  E* ring = reinterpret_cast<E*>(smem + warp * Cfg::RING_BYTES);
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
  const int units = a.nstrips * a.nseg;
  uint32_t ring_cnt = 0;  // rows consumed so far by this warp (ring position)

  int src = a.first_src, dst = a.first_dst;
  for (int e = 0; e < a.epochs; ++e) {
    const CUtensorMap* tm = &maps.m[src];
    E* __restrict__ out = static_cast<E*>((dst == BUF_OUT) ? a.buf[BUF_OUT] : a.buf[BUF_SCR]);

    // Dynamic unit distribution: a warp grabs the next unit when it finishes
    // one, so warps the scheduler favours take more units and the epoch tail
    // is at most one unit (static assignment left SMs half idle).
    for (int u = next_unit(a.work + e, lane); u < units; u = next_unit(a.work + e, lane)) {
      const int strip = u % a.nstrips;
      const int seg = u / a.nstrips;
      const StripGeom g =
          stream2d_strip(strip, a.nstrips, a.aligned, n1, Cfg::LC, Cfg::VW, Cfg::HX, Cfg::AL);
      const int r0 = a.seg_start[seg];
      const int r1 = a.seg_start[seg + 1];
      if (a.flags && e > 0) {
        // wait for the previous epoch's units that wrote our input region
        // (rows [r0-TR, r1+TR), columns [X0, X0+LC)); lanes split the checks
        int lo_seg = seg, hi_seg = seg;
        while (lo_seg > 0 && a.seg_start[lo_seg] > r0 - TR) --lo_seg;
        while (hi_seg + 1 < a.nseg && a.seg_start[hi_seg + 1] < r1 + TR) ++hi_seg;
        const int nseg_dep = hi_seg - lo_seg + 1;
        for (int d = lane; d < 5 * nseg_dep; d += 32) {
          const int js = strip - 2 + d % 5;
          if (js < 0 || js >= a.nstrips) continue;
          const StripGeom gj =
              stream2d_strip(js, a.nstrips, a.aligned, n1, Cfg::LC, Cfg::VW, Cfg::HX, Cfg::AL);
          // RAW: js wrote what we read; WAR: js reads what we overwrite
          const bool raw = gj.vlo < g.X0 + Cfg::LC && gj.vhi > g.X0;
          const bool war = gj.X0 < g.vhi && gj.X0 + Cfg::LC > g.vlo;
          if (!raw && !war) continue;
          wait_flag_geq(a.flags + (lo_seg + d / 5) * a.nstrips + js, e);
        }
        __syncwarp();
        fence_proxy_async_global();  // the TMA loads below see those stores
      }
      long long t_start = 0;
      if (a.unit_clock && e == 0 && lane == 0)
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
      int used;
      if constexpr (R > C) {
        // generic strips; those clear of the frame columns skip the masks
        if (g.X0 >= R && g.X0 + Cfg::LC <= n1 - R)
          used = stream2d_unit<SH, T, C, S, EXACT, UNI, 0, E, SHIFT>(tm, out, ring, bars, ring_cnt,
                                                                     lane, n0, n1, a.pitch, g, r0, r1, cf);
        else
          used = stream2d_unit<SH, T, C, S, EXACT, UNI, 3, E, SHIFT>(tm, out, ring, bars, ring_cnt,
                                                                     lane, n0, n1, a.pitch, g, r0, r1, cf);
      } else switch (g.fc) {
        case 0:
          used = stream2d_unit<SH, T, C, S, EXACT, UNI, 0, E, SHIFT>(tm, out, ring, bars, ring_cnt,
                                                                     lane, n0, n1, a.pitch, g, r0, r1, cf);
          break;
        case 1:
          used = stream2d_unit<SH, T, C, S, EXACT, UNI, 1, E, SHIFT>(tm, out, ring, bars, ring_cnt,
                                                                     lane, n0, n1, a.pitch, g, r0, r1, cf);
          break;
        case 2:
          used = stream2d_unit<SH, T, C, S, EXACT, UNI, 2, E, SHIFT>(tm, out, ring, bars, ring_cnt,
                                                                     lane, n0, n1, a.pitch, g, r0, r1, cf);
          break;
        default:
          used = stream2d_unit<SH, T, C, S, EXACT, UNI, 3, E, SHIFT>(tm, out, ring, bars, ring_cnt,
                                                                     lane, n0, n1, a.pitch, g, r0, r1, cf);
          break;
      }
      ring_cnt += (uint32_t)used;
      if (a.flags) {
        // publish: every lane's stores, then the flag (release)
        fence_proxy_async_global();
        __threadfence();
        __syncwarp();
        if (lane == 0) st_release_gpu(a.flags + u, e + 1);
      }
      if (a.unit_clock && e == 0 && lane == 0) {
        long long t_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        a.unit_clock[2 * u] = t_start;
        a.unit_clock[2 * u + 1] = t_end;
      }
    }

    if (e + 1 < a.epochs && !a.flags) {
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

// ebisu_halo2d.cuh -- 2-D temporal blocking with per-level halo exchange
// ("device tiling"), sm_100a.
//
// Replaces the reference's device-tiling engine (engine/device.py:55-389:
// a device tile of g x w blocks that exchange their per-level halos through a
// staging buffer and a device barrier, Listing 3 order) with a CTA-level
// design:
//
//  * Work unit = (CTA strip, row segment).  The CTA is the device tile: NW
//    warps side by side, warp w owning LC = 32*C columns of a strip of
//    LW = NW*LC columns.  Only the strip carries an overlapped margin of
//    HX = T*R columns per side; inside the strip, warps exchange the edge
//    columns of every produced row, so no column is computed twice.  With
//    LW = 1024 the valid fraction at t=2, R=6 is 0.977, against 0.81 for a
//    128-column overlapped warp strip (the paper's argument for halo exchange
//    on large halos, Table 1 / SURVEY §7 step 6).
//  * Rows arrive per warp by TMA into an S-slot mbarrier ring (as in
//    k_stream2d).  Levels are register windows; x-neighbours inside a warp come
//    from shuffles, across warps from a small shared-memory edge buffer:
//    xh[level][slot][warp][side][R] -- the leftmost and rightmost R values of
//    every row a warp produces.
//  * Level skew Z = max(R, 2) for stars (only the centre row needs
//    x-neighbours, and it was produced Z advances earlier) and R+1 for boxes
//    (every window row does; the newest was produced one advance earlier).
//    Every exchanged value is thus at least DR advances old (DR = Z for
//    stars, 1 for boxes), so split-phase mbarriers order the exchange: each
//    warp arrives after its advance, and an advance waits only for the phase
//    DR advances back.  Warps drift up to DR advances apart and never drain
//    at a block-wide barrier (measured: the drift-1 version spent 20% of its
//    stall samples waiting on the barrier).
//  * Dirichlet frame, exact / shared-product arithmetic: as k_stream2d.
#pragma once

#include <cooperative_groups.h>

#include <type_traits>

#include "ebisu_common.cuh"
#include "ebisu_shapes.cuh"
#include "ebisu_stream2d.cuh"

namespace ebisu {

template <class SH, int T, int C, int NW, int S>
struct Halo2DCfg {
  static constexpr int R = SH::R;
  // level skew (advances).  Stars need x-neighbours of the centre row only,
  // produced Z advances earlier, so warps may drift DR = Z advances apart;
  // radius-1 stars use Z = 2 to get that slack.  Boxes read rows up to one
  // advance old: Z = R + 1, DR = 1.
  static constexpr int Z = SH::kStar ? (R < 2 ? 2 : R) : R + 1;
  static constexpr int DR = SH::kStar ? Z : 1;
  static constexpr int LAG = SH::kStar ? Z : Z + R;  // oldest exchanged row read
  static constexpr int W = Z + R + 1;                 // window rows per level
  static constexpr int LC = 32 * C;                   // columns per warp
  static constexpr int LW = NW * LC;                  // columns per CTA strip
  static constexpr int HX = (T * R + 1) & ~1;         // strip margin (even: TMA)
  static constexpr int VW = LW - 2 * HX;              // valid columns per strip
  static constexpr int NBMIN = DR + LAG;  // writers may run DR advances ahead
  static constexpr int NB = NBMIN <= 2 ? 2 : (NBMIN <= 4 ? 4 : (NBMIN <= 8 ? 8 : 16));
  static constexpr int ROW_BYTES = LC * 8;
  static constexpr int RING_BYTES = NW * S * ROW_BYTES;
  // edge buffer columns: 0 = left neighbour CTA's last warp (cluster),
  // 1..NW = this CTA's warps, NW+1 = right neighbour CTA's first warp
  static constexpr int XCOLS = NW + 2;
  static constexpr int XH_DOUBLES = T * NB * XCOLS * 2 * R;  // levels 0..T-1
  // mbarriers: TMA ring (NW*S), advance barriers (DR), foreign-edge receive
  // barriers fullL/fullR and slot-release barriers emptyL/emptyR (NB each),
  // then the unit id
  static constexpr int BAR_OFF = RING_BYTES + XH_DOUBLES * 8;
  static constexpr int SMEM_BYTES = BAR_OFF + (NW * S + DR + 4 * NB) * 8 + 16;
  static_assert(VW > 0, "strip leaves no valid core");
  static_assert(NB >= NBMIN, "edge-buffer slots must cover lag + drift");
  static_assert((S & (S - 1)) == 0, "ring slots must be a power of two");
  static_assert(LC <= 256, "TMA box inner dimension is limited to 256 elements");
  static_assert(R <= LC, "halo must fit in one neighbouring warp");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
};

struct Halo2DArgs {
  int n0, n1;
  int nstrips, nseg, seg_len;
  int z_lo, z_hi;  // output rows [z_lo, z_hi)
  int epochs;
  int first_src, first_dst;
  int aligned;  // edge-aligned strips (n1 >= 2*LW)
  int pitch;    // row pitch of every buffer (elements, >= n1)
  double* buf[3];
  int* work;
};

// Cluster context of a CTA: rank and size of the device tile (CL CTA strips
// side by side along axis 1, exchanging their outer warps' edge columns
// through DSMEM).  Remote addresses are formed on use (mapa): the same
// shared-memory offsets in the neighbour CTA.
struct Halo2DCluster {
  int rank, n;
  __device__ __forceinline__ bool has_l() const { return rank > 0; }
  __device__ __forceinline__ bool has_r() const { return rank < n - 1; }
};

// One unit: CTA strip x row segment.  EDGE: the strip touches a frame column.
template <class SH, int T, int C, int NW, int S, bool EXACT, bool UNI, bool EDGE, int SHIFT,
          bool CLU>
__device__ __forceinline__ int halo2d_unit(const CUtensorMap* tm, double* __restrict__ out,
                                           double* ring, uint64_t* bars, double* xh,
                                           uint64_t* advbar, const Halo2DCluster& cc,
                                           uint32_t ring_cnt, uint32_t& adv,
                                           int warp, int lane, int n0, int n1, int pitch, int X0, int vlo,
                                           int vhi, int r0, int r1, const Coefs<SH::NT>& cf) {
  using Cfg = Halo2DCfg<SH, T, C, NW, S>;
  constexpr int R = Cfg::R, Z = Cfg::Z, W = Cfg::W, NB = Cfg::NB, LC = Cfg::LC;
  constexpr int ROW_BYTES = Cfg::ROW_BYTES;
  constexpr int TZ = T * Z;

  const int ka = max(0, r0 - T * R);
  // SHIFT = U > 0: shifted windows, U advances per block (see stream2d_unit)
  constexpr int UW = SHIFT ? SHIFT : W;
  constexpr int WS = SHIFT ? W + SHIFT - 1 : W;
  const int nadv = (r1 + TZ - ka + UW - 1) / UW * UW;  // whole unrolled blocks
  const int kend = ka + nadv;
  const int XW = X0 + warp * LC;  // this warp's first column

  // per-warp ring: rows [ka, kend); TMA zero-fills rows >= n0, rows >= r1+T*R
  // only feed targets >= r1 (never stored)
  if (lane == 0) {
    for (int i = 0; i < S && i < nadv; ++i) {
      const uint32_t slot = (ring_cnt + i) & (S - 1);
      mbar_arrive_expect_tx(&bars[slot], ROW_BYTES);
      tma_load_2d(ring + slot * LC, tm, XW, ka + i, &bars[slot]);
    }
  }

  uint32_t fmask = 0, stmask = 0;
#pragma unroll
  for (int c = 0; c < C; ++c) {
    const int x = XW + lane * C + c;
    const bool f = EDGE && ((x < R) || (x >= n1 - R));
    bool st = (x >= vlo) && (x < vhi);
    if (UNI) st = st && !f;
    fmask |= (uint32_t)f << c;
    stmask |= (uint32_t)st << c;
  }

  double win[T][WS][C];
#pragma unroll
  for (int s = 0; s < T; ++s)
#pragma unroll
    for (int w = 0; w < WS; ++w)
#pragma unroll
      for (int c = 0; c < C; ++c) win[s][w][c] = 0.0;

  // edge buffer of (level, slot, warp, side)
  constexpr int XCOLS = Cfg::XCOLS;
  uint64_t* const fullL = advbar + Cfg::DR;  // receive barriers (kernel layout)
  uint64_t* const fullR = fullL + NB;
  uint64_t* const emptyL = fullR + NB;       // slot releases by the neighbours
  uint64_t* const emptyR = emptyL + NB;
  auto xoff = [&](int level, int slot, int w, int side) -> int {
    return (((level * NB + slot) * XCOLS + w) * 2 + side) * R;
  };
  auto xrow = [&](int level, int slot, int w, int side) -> double* {
    return xh + xoff(level, slot, w, side);
  };
  // push the warp's leftmost / rightmost R values of a produced row:
  // predicated stores, only the edge lanes' predicates are on (no branch)
  auto push = [&](int level, int slot, const double (&v)[C]) {
    double* L = xrow(level, slot, warp + 1, 0);
    double* Rt = xrow(level, slot, warp + 1, 1);
#pragma unroll
    for (int c = 0; c < C; ++c) {
      const int col = lane * C + c;
      if (c < R) st_shared_if(L + min(col, R - 1), v[c], col < R);
      if (C - c <= R) st_shared_if(Rt + max(col - (LC - R), 0), v[c], col >= LC - R);
    }
    // the tile's outer warps also hand their outer edge to the neighbour CTA
    // of the cluster: st.async into its xh, completing 8 bytes each on its
    // receive barrier for this advance (no fence: the TMA-style handshake)
    if (CLU && warp == 0 && cc.has_l() && lane * C < R) {
      // left CTA: its right-foreign column (NW+1), completing on its fullR
      const uint32_t dst = mapa_shared(xrow(level, slot, NW + 1, 0), cc.rank - 1);
      const uint32_t bar = mapa_shared(fullR + slot, cc.rank - 1);
#pragma unroll
      for (int c = 0; c < C && c < R; ++c)
        if (lane * C + c < R) st_async_f64(dst + 8u * (lane * C + c), v[c], bar);
    }
    if (CLU && warp == NW - 1 && cc.has_r() && lane * C + C > LC - R) {
      // right CTA: its left-foreign column (0), completing on its fullL
      const uint32_t dst = mapa_shared(xrow(level, slot, 0, 1), cc.rank + 1);
      const uint32_t bar = mapa_shared(fullL + slot, cc.rank + 1);
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (lane * C + c >= LC - R) st_async_f64(dst + 8u * (lane * C + c - (LC - R)), v[c], bar);
    }
  };
  // edge-buffer columns of the left / right neighbour of this warp (the outer
  // warps of a cluster tile read never-written zeros: invalid margin)
  const int wl = warp;
  const int wr = warp + 2;
  // foreign edges of advance a (outer warps with a neighbour CTA): wait for
  // the neighbour's st.async bytes of that advance
  auto wait_foreign = [&](uint32_t a) {
    if (CLU && (warp == 0 && cc.has_l()) || (warp == NW - 1 && cc.has_r()))
      mbar_wait(&(warp == 0 ? fullL : fullR)[a & (NB - 1)], (a / NB) & 1);
  };
  // before an outer warp pushes advance a into the neighbour's slot, the
  // neighbour must have released the slot's previous use (advance a - NB)
  auto wait_slot_free = [&](uint32_t a) {
    if (CLU && a >= (uint32_t)NB && ((warp == 0 && cc.has_l()) || (warp == NW - 1 && cc.has_r())))
      mbar_wait(&(warp == 0 ? emptyL : emptyR)[a & (NB - 1)], ((a / NB) - 1) & 1);
  };
  // the last read of a foreign slot is LAG advances after it was produced:
  // release it to the producer (relaxed: the values are in registers)
  auto release_slot = [&](uint32_t a) {
    if (CLU && lane == 0 && a >= (uint32_t)Cfg::LAG) {
      const uint32_t j = (a - Cfg::LAG) & (NB - 1);
      if (warp == 0 && cc.has_l())
        mbar_arrive_remote_relaxed(mapa_shared(emptyR + j, cc.rank - 1));
      if (warp == NW - 1 && cc.has_r())
        mbar_arrive_remote_relaxed(mapa_shared(emptyL + j, cc.rank + 1));
    }
  };
  // arm this advance's receive barriers (one arrival + the expected bytes)
  auto arm_foreign = [&](uint32_t a) {
    if (CLU && lane == 0 && ((warp == 0 && cc.has_l()) || (warp == NW - 1 && cc.has_r())))
      mbar_arrive_expect_tx(&(warp == 0 ? fullL : fullR)[a & (NB - 1)], T * R * 8);
  };
  // advance done: local arrival; outer warps release the foreign slot whose
  // last reader this advance was
  auto arrive_adv = [&](uint32_t a) {
    if (lane == 0) mbar_arrive(&advbar[a % Cfg::DR]);
    release_slot(a);
  };

  auto block = [&](int kbase, auto frows_tag) {
    constexpr bool FROWS = decltype(frows_tag)::value;
#pragma unroll
    for (int uu = 0; uu < UW; ++uu) {
      const int k = kbase + uu;
      const int bk = adv & (NB - 1);  // edge-buffer slot of this advance
      arm_foreign(adv);
      wait_slot_free(adv);
      // (DR barriers round robin: advance a arrives on advbar[a % DR] as its
      // phase a / DR; waiting for advance adv-DR is then unambiguous)
      if (adv >= (uint32_t)Cfg::DR) {
        const uint32_t a = adv - Cfg::DR;
        mbar_wait(&advbar[a % Cfg::DR], (a / Cfg::DR) & 1);
      }
      // ---- level 0 --------------------------------------------------------
      {
        const uint32_t pos = ring_cnt + (uint32_t)(k - ka);
        const uint32_t slot = pos & (S - 1);
        mbar_wait(&bars[slot], (pos / S) & 1);
        if (lane == 0 && k > ka && k - 1 + S < kend) {
          const uint32_t ps = (pos - 1) & (S - 1);
          mbar_arrive_expect_tx(&bars[ps], ROW_BYTES);
          tma_load_2d(ring + ps * LC, tm, XW, k - 1 + S, &bars[ps]);
        }
        const double* rowp = ring + slot * LC + lane * C;
        double v[C];
#pragma unroll
        for (int c = 0; c < C; c += 2) {
          const double2 t2 = *reinterpret_cast<const double2*>(rowp + c);
          v[c] = UNI ? __dmul_rn(cf.c[0], t2.x) : t2.x;
          v[c + 1] = UNI ? __dmul_rn(cf.c[0], t2.y) : t2.y;
        }
#pragma unroll
        for (int c = 0; c < C; ++c) {
          if constexpr (SHIFT)
            win[0][W - 1 + uu][c] = v[c];
          else
            win[0][uu][c] = v[c];
        }
        push(0, bk, v);
      }
      // ---- levels 1..T --------------------------------------------------------
      static_for<T>([&](auto sI) {
        constexpr int s = decltype(sI)::value + 1;
        const int q = k - s * Z;
        double hl[2 * R + 1][R], hr[2 * R + 1][R];
        static_for<2 * R + 1>([&](auto dI) {
          constexpr int dy = decltype(dI)::value - R;
          if constexpr (row_has_halo<SH>(dy)) {
            const int sl = SHIFT ? R + dy + uu : pmod<W>(uu - s * Z + dy);
            const uint32_t ap = adv - (uint32_t)(Z - dy);  // advance that produced the row
            const int xs = ap & (NB - 1);
            if (CLU && adv >= (uint32_t)(Z - dy)) wait_foreign(ap);
            const double* Lb = xrow(s - 1, xs, wr, 0);   // right neighbour's left edge
            const double* Rb = xrow(s - 1, xs, wl, 1);   // left neighbour's right edge
            static_for<R>([&](auto jI) {
              constexpr int j = decltype(jI)::value;
              constexpr int ccl = -R + j;
              constexpr int dl = (-ccl + C - 1) / C;
              constexpr int coll = ccl + dl * C;
              constexpr int ccr = C + j;
              constexpr int dr = ccr / C;
              constexpr int colr = ccr - dr * C;
              double a = __shfl_up_sync(kFullMask, win[s - 1][sl][coll], dl);
              double b = __shfl_down_sync(kFullMask, win[s - 1][sl][colr], dr);
              // lanes whose neighbour column lies in the next warp (branch
              // free: every lane loads from a clamped in-range address)
              a = ld_shared_if(Rb + max(R + lane * C + ccl, 0), lane < dl, a);
              b = ld_shared_if(Lb + min(max(lane * C + ccr - LC, 0), R - 1), lane > 31 - dr, b);
              hl[dI][j] = a;
              hr[dI][j] = b;
            });
          }
        });
        double acc[C];
        static_for<SH::NT>([&](auto iI) {
          constexpr int i = decltype(iI)::value;
          constexpr Off o = SH::tap(i);
#pragma unroll
          for (int c = 0; c < C; ++c) {
            const int sl = SHIFT ? R + o.d0 + uu : pmod<W>(uu - s * Z + o.d0);
            const int cc = c + o.d1;
            double x;
            if (cc < 0)
              x = hl[o.d0 + R][cc + R];
            else if (cc >= C)
              x = hr[o.d0 + R][cc - C];
            else
              x = win[s - 1][sl][cc];
            if constexpr (UNI)
              acc[c] = (i == 0) ? x : __dadd_rn(acc[c], x);
            else if constexpr (i == 0)
              acc[c] = tap_first<EXACT>(cf.c[0], x);
            else
              acc[c] = tap_next<EXACT>(acc[c], cf.c[i], x);
          }
        });
        bool frow = false;
        if constexpr (FROWS) frow = (q < R) || (q >= n0 - R);
        double nv[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const double centre = win[s - 1][SHIFT ? R + uu : pmod<W>(uu - s * Z)][c];
          const double val = (UNI && s < T) ? __dmul_rn(cf.c[0], acc[c]) : acc[c];
          if constexpr (EDGE || FROWS) {
            bool f = frow;
            if constexpr (EDGE) f = f || ((fmask >> c) & 1u);
            nv[c] = f ? centre : val;
          } else {
            nv[c] = val;
          }
        }
        if constexpr (s < T) {
#pragma unroll
          for (int c = 0; c < C; ++c) {
            if constexpr (SHIFT)
              win[s][W - 1 + uu][c] = nv[c];
            else
              win[s][pmod<W>(uu - s * Z)][c] = nv[c];
          }
          push(s, bk, nv);
        } else {
          bool qok = (q >= r0) && (q < r1);
          if (UNI && FROWS) qok = qok && !frow;
          if (qok) {
            double* orow = out + (size_t)q * (size_t)pitch + (XW + lane * C);
#pragma unroll
            for (int c = 0; c < C; ++c)
              if ((stmask >> c) & 1u) orow[c] = nv[c];
          }
        }
      });
      __syncwarp();
      arrive_adv(adv);  // (release covers the warp)
      ++adv;
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

  // Tolerance mode (exact = 0, uniform coefficients), stars with Z = R >= U:
  // level-major blocks of U advances (see stream2d_unit's block_ra) -- the
  // column sums of a level's U targets share partial sums (slide4), the row
  // sums of each centre row are sliding sums over the lane's C cells plus the
  // exchanged halo.  Every exchanged centre row is >= Z - U + 1 advances old,
  // so one barrier wait per block (for advance adv + U - 1 - DR) covers it.
  constexpr bool RA = UNI && !EXACT;
  static_assert(!RA || (SHIFT == 4 && SH::kStar && Z >= SHIFT), "tolerance halo kernel: stars, Z >= U");
  auto block_ra = [&](int kbase, auto frows_tag) {
    constexpr bool FROWS = decltype(frows_tag)::value;
    constexpr int U = SHIFT;
    if (adv + U - 1 >= (uint32_t)Cfg::DR) {
      const uint32_t a = adv + U - 1 - Cfg::DR;
      mbar_wait(&advbar[a % Cfg::DR], (a / Cfg::DR) & 1);
    }
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
      const int k = kbase + uu;
      const uint32_t pos = ring_cnt + (uint32_t)(k - ka);
      const uint32_t slot = pos & (S - 1);
      mbar_wait(&bars[slot], (pos / S) & 1);
      if (lane == 0 && k > ka && k - 1 + S < kend) {
        const uint32_t ps = (pos - 1) & (S - 1);
        mbar_arrive_expect_tx(&bars[ps], ROW_BYTES);
        tma_load_2d(ring + ps * LC, tm, XW, k - 1 + S, &bars[ps]);
      }
      const double* rowp = ring + slot * LC + lane * C;
      double v[C];
#pragma unroll
      for (int c = 0; c < C; c += 2) {
        const double2 t2 = *reinterpret_cast<const double2*>(rowp + c);
        v[c] = __dmul_rn(cf.c[0], t2.x);
        v[c + 1] = __dmul_rn(cf.c[0], t2.y);
      }
#pragma unroll
      for (int c = 0; c < C; ++c) win[0][W - 1 + uu][c] = v[c];
      push(0, (adv + uu) & (NB - 1), v);
    }
    static_for<T>([&](auto sI) {
      constexpr int s = decltype(sI)::value + 1;
      double V[U][C];
#pragma unroll
      for (int c = 0; c < C; ++c) {
        double a[W + 3], o[4];
#pragma unroll
        for (int j = 0; j < W + 3; ++j) a[j] = win[s - 1][j][c];
        slide4<W>(a, o);
#pragma unroll
        for (int uu = 0; uu < U; ++uu) V[uu][c] = o[uu];
      }
#pragma unroll
      for (int uu = 0; uu < U; ++uu) {
        const int k = kbase + uu;
        const int q = k - s * Z;
        // centre row q of level s-1 with R columns each side: in-warp by
        // shuffles, across warps from the neighbours' edge buffers
        double b[2 * R + C];
#pragma unroll
        for (int c = 0; c < C; ++c) b[R + c] = win[s - 1][R + uu][c];
        const int xs = (adv + uu - Z) & (NB - 1);
        const double* Lb = xrow(s - 1, xs, wr, 0);
        const double* Rb = xrow(s - 1, xs, wl, 1);
        static_for<R>([&](auto jI) {
          constexpr int j = decltype(jI)::value;
          constexpr int ccl = -R + j;
          constexpr int dl = (-ccl + C - 1) / C;
          constexpr int coll = ccl + dl * C;
          constexpr int ccr = C + j;
          constexpr int dr = ccr / C;
          constexpr int colr = ccr - dr * C;
          double x0 = __shfl_up_sync(kFullMask, b[R + coll], dl);
          double x1 = __shfl_down_sync(kFullMask, b[R + colr], dr);
          b[j] = ld_shared_if(Rb + max(R + lane * C + ccl, 0), lane < dl, x0);
          b[R + C + j] = ld_shared_if(Lb + min(max(lane * C + ccr - LC, 0), R - 1), lane > 31 - dr, x1);
        });
        double h[C];
        slide_n<W, C>(b, h);
        bool frow = false;
        if constexpr (FROWS) frow = (q < R) || (q >= n0 - R);
        double nv[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
          const double centre = b[R + c];
          const double acc = __dadd_rn(V[uu][c], __dsub_rn(h[c], centre));
          const double val = s < T ? __dmul_rn(cf.c[0], acc) : acc;
          bool f = frow;
          if constexpr (EDGE) f = f || ((fmask >> c) & 1u);
          nv[c] = f ? centre : val;
        }
        if constexpr (s < T) {
#pragma unroll
          for (int c = 0; c < C; ++c) win[s][W - 1 + uu][c] = nv[c];
          push(s, (adv + uu) & (NB - 1), nv);
        } else if (q >= r0 && q < r1 && !frow) {
          double* orow = out + (size_t)q * (size_t)pitch + (XW + lane * C);
#pragma unroll
          for (int c = 0; c < C; c += 2)
            st_pair_if(orow + c, nv[c], nv[c + 1], (stmask >> c) & 1u, (stmask >> (c + 1)) & 1u);
        }
      }
    });
    __syncwarp();
    if (lane == 0)
#pragma unroll
      for (int uu = 0; uu < U; ++uu) mbar_arrive(&advbar[(adv + uu) % Cfg::DR]);
    adv += U;
#pragma unroll
    for (int L = 0; L < T; ++L)
#pragma unroll
      for (int w = 0; w + 1 < W; ++w)
#pragma unroll
        for (int c = 0; c < C; ++c) win[L][w][c] = win[L][w + U][c];
  };

  for (int kbase = ka; kbase < kend; kbase += UW) {
    // target rows of this block: [kbase - TZ, kbase + UW - 1 - Z]
    const bool frows = (kbase - TZ < R) || (kbase + UW - 1 - Z >= n0 - R);
    if constexpr (RA) {
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
  return nadv;
}

template <class SH, int T, int C, int NW, int S, bool EXACT, bool UNI, int MINB,
          int SHIFT = 0, bool CLU = false>
__global__ void __launch_bounds__(NW * 32, MINB)
    k_halo2d(const __grid_constant__ TmapSet maps, const Halo2DArgs a,
             const __grid_constant__ Coefs<SH::NT> cf) {
  using Cfg = Halo2DCfg<SH, T, C, NW, S>;
  constexpr int NB = Cfg::NB;
  extern __shared__ __align__(1024) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* ring = reinterpret_cast<double*>(smem + warp * S * Cfg::ROW_BYTES);
  double* xh = reinterpret_cast<double*>(smem + Cfg::RING_BYTES);
  uint64_t* bars_all = reinterpret_cast<uint64_t*>(smem + Cfg::BAR_OFF);
  uint64_t* bars = bars_all + warp * S;
  uint64_t* advbar = bars_all + NW * S;
  uint64_t* fullL = advbar + Cfg::DR;  // then fullR, emptyL, emptyR (NB each)
  int* s_unit = reinterpret_cast<int*>(fullL + 4 * NB);

  // cluster = device tile of CL CTA strips side by side (CL = 1: a lone CTA)
  // (CLU = false: compiled for single-CTA tiles, no cluster code)
  const int rank = CLU ? (int)cluster_ctarank() : 0;
  const int CL = CLU ? (int)cluster_nctarank() : 1;
  Halo2DCluster cc;
  cc.rank = rank;
  cc.n = CL;

  if (threadIdx.x == 0) {
    for (int i = 0; i < NW * S; ++i) mbar_init(&bars_all[i], 1);
    for (int i = 0; i < Cfg::DR; ++i) mbar_init(&advbar[i], NW);
    // receive (our outer warp's expect_tx + the neighbour's bytes) and slot
    // release (the neighbour's outer warp) barriers, NB each per side
    for (int i = 0; i < 4 * NB; ++i) mbar_init(&fullL[i], 1);
    fence_mbarrier_init();
    prefetch_tmap(&maps.m[0]);
    prefetch_tmap(&maps.m[1]);
    prefetch_tmap(&maps.m[2]);
  }
  // the edge buffers of the tile's outer warps are read but never written
  for (int i = threadIdx.x; i < Cfg::XH_DOUBLES; i += NW * 32) xh[i] = 0.0;
  __syncthreads();
  // the neighbours' barriers must be initialised before anyone touches them
  if (CL > 1) cluster_sync_all();

  const int n0 = a.n0, n1 = a.n1;
  const int units = a.nstrips * a.nseg;
  const int LWc = CL * Cfg::LW;  // cluster tile width
  uint32_t ring_cnt = 0, adv = 0;
  int src = a.first_src, dst = a.first_dst;
  for (int e = 0; e < a.epochs; ++e) {
    const CUtensorMap* tm = &maps.m[src];
    double* __restrict__ out = (dst == BUF_OUT) ? a.buf[BUF_OUT] : a.buf[BUF_SCR];
    for (;;) {
      // rank 0 claims the next unit for the whole cluster tile
      if (threadIdx.x == 0 && rank == 0) {
        const int u = atomicAdd(a.work + e, 1);
        *s_unit = u;
        for (int r = 1; r < CL; ++r) st_cluster_u32(mapa_shared(s_unit, r), (uint32_t)u);
      }
      if (CL > 1)
        cluster_sync_all();
      else
        __syncthreads();
      const int u = *s_unit;
      if (CL > 1)
        cluster_sync_all();  // every rank has read it: the next claim may overwrite
      else
        __syncthreads();
      if (u >= units) break;
      const int strip = u % a.nstrips;
      const int seg = u / a.nstrips;
      StripGeom g;
      if (a.nstrips == 1 && LWc >= n1) {  // one tile spans the width: no margin
        g.X0 = 0;
        g.vlo = 0;
        g.vhi = n1;
      } else {
        g = stream2d_strip(strip, a.nstrips, a.aligned, n1, LWc, LWc - 2 * Cfg::HX, Cfg::HX, 2);
      }
      const int X0 = g.X0 + rank * Cfg::LW;
      const int vlo = max(g.vlo, X0), vhi = min(g.vhi, X0 + Cfg::LW);
      const int r0 = a.z_lo + seg * a.seg_len;
      const int r1 = min(a.z_hi, r0 + a.seg_len);
      const bool edge = (X0 < Cfg::R) || (X0 + Cfg::LW > n1 - Cfg::R);
      int used;
      if (edge)
        used = halo2d_unit<SH, T, C, NW, S, EXACT, UNI, true, SHIFT, CLU>(
            tm, out, ring, bars, xh, advbar, cc, ring_cnt, adv, warp, lane, n0, n1, a.pitch, X0,
            vlo, vhi, r0, r1, cf);
      else
        used = halo2d_unit<SH, T, C, NW, S, EXACT, UNI, false, SHIFT, CLU>(
            tm, out, ring, bars, xh, advbar, cc, ring_cnt, adv, warp, lane, n0, n1, a.pitch, X0,
            vlo, vhi, r0, r1, cf);
      ring_cnt += (uint32_t)used;
    }
    if (e + 1 < a.epochs) {
      fence_proxy_async_global();
      __threadfence();
      cooperative_groups::this_grid().sync();
      fence_proxy_async_global();
    }
    const int nsrc = dst;
    dst = (dst == BUF_OUT) ? BUF_SCR : BUF_OUT;
    src = nsrc;
  }
  // no CTA may exit while a neighbour can still write its shared memory
  if (CL > 1) cluster_sync_all();
}

}  // namespace ebisu

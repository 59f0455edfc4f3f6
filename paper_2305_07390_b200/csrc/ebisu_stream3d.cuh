// ebisu_stream3d.cuh -- 3-D (2.5-D streaming) temporal-blocking sweep, sm_100a.
//
// Replaces the reference's 3-D engines (engine/sm.py:95-206 plane pipeline
// over a circular multi-queue; engine/device.py:292-389 streamed device
// tiles with per-level halo exchange and a barrier per advance) with:
//
//  * Work unit = (tile ty, tile tx, z segment).  The CTA owns an LY x LX
//    in-plane tile (LY = NWY*CY rows along axis 1, LX = 32*CX columns along
//    axis 2) and streams it along axis 0.  Planes arrive by TMA
//    (cp.async.bulk.tensor.3d, box {LX, LY, 1}, out-of-bounds zero fill) in an
//    S-slot mbarrier ring.
//  * Thread (warp w, lane l) owns the CY x CX block rows w*CY.., columns
//    l*CX..; its z-window of every level lives in registers (RST register
//    streaming).  In-plane neighbours come from a per-level shared-memory
//    plane buffer that each level writes once per advance ("push halo"), read
//    one or more advances later ("pull halo"), with ONE __syncthreads per
//    advance (the reference's lazy mode: one barrier per advance,
//    device.py:381-387).
//  * Skew Z between levels: level s at advance k emits plane k - s*Z.  For
//    stars only the centre plane needs in-plane neighbours, so Z = R; for
//    boxes every plane does, so Z = R + 1.  Either way every in-plane value a
//    level reads was produced in an earlier advance.
//  * Frame cells carry the previous level's centre (EDGE units only).
//  * Exact mode: __dmul_rn/__dadd_rn in catalog tap order (bitwise).
#pragma once

#include <cooperative_groups.h>

#include "ebisu_common.cuh"
#include "ebisu_shapes.cuh"
#include "ebisu_stream2d.cuh"  // StripGeom / stream2d_strip (tile geometry)

namespace ebisu {

// Tile geometry along one in-plane axis (stream2d_strip's arithmetic for an
// aligned width, without the frame-column class the 3-D kernels do not use).
// Kept separate on purpose: the AL-generic 2-D version perturbs ptxas's
// register allocation of the 3-D kernels (248 vs 254 registers, j3d7pt 512^3
// 693 vs 733 GCells/s measured A/B on one box).
__host__ __device__ inline StripGeom tile3d_strip(int j, int ntiles, int aligned, int n, int L,
                                                  int V, int H) {
  StripGeom g;
  g.fc = 0;
  if (aligned) {
    const int xl = n - L + H;
    if (j == ntiles - 1) {
      g.X0 = n - L;
      g.vlo = xl;
      g.vhi = n;
    } else {
      g.X0 = j * V;
      g.vlo = j == 0 ? 0 : j * V + H;
      g.vhi = min((j + 1) * V + H, xl);
    }
  } else {
    g.X0 = j * V - H;
    g.vlo = j * V;
    g.vhi = min((j + 1) * V, n);
  }
  return g;
}

struct Stream3DArgs {
  int n0, n1, n2;   // extents
  int pitch;        // row pitch of every buffer (elements, >= n2); plane pitch n1*pitch
  int nty, ntx;     // tiles along axis 1 / axis 2
  int aligned_y, aligned_x;  // edge-aligned tiles along axis 1 / axis 2
  int nseg;         // z segments
  int seg_len;      // (planner's nominal length; the real bounds are seg_start)
  int z_lo, z_hi;   // output planes [z_lo, z_hi) (informational: seg_start tiles it)
  // z segment j covers planes [seg_start[j], seg_start[j+1]).  Guided
  // schedule: segments shrink toward the end of the list, and units are
  // handed out segment-major, so the epoch tail is made of short units.
  int seg_start[EBISU_MAX_SEGS + 1];
  int epochs;
  int first_src, first_dst;
  void* buf[3];  // element type E of the kernel
  int* work;  // per-epoch unit counters (dynamic scheduling), zeroed by the host
};

// Does tap set need in-plane neighbours on planes other than the centre?
template <class SH>
__host__ __device__ constexpr bool offcentre_inplane() {
  for (int i = 0; i < SH::NT; ++i)
    if (SH::tap(i).d0 != 0 && (SH::tap(i).d1 != 0 || SH::tap(i).d2 != 0)) return true;
  return false;
}

// DEC = decoupled levels: skew R+1 even for stars, so that within one
// advance no level consumes another level's output (T independent chains).
// Which planes (dz) of the window need values outside the thread's block?
template <class SH>
__host__ __device__ constexpr bool plane_needs_inplane(int dz) {
  for (int i = 0; i < SH::NT; ++i)
    if (SH::tap(i).d0 == dz && (SH::tap(i).d1 != 0 || SH::tap(i).d2 != 0)) return true;
  return false;
}

// Does extended row ey (relative to the block, in [-R, CY+R)) of plane dz
// need x-halo values (some tap reaches (ey, outside the lane's columns))?
template <class SH>
__host__ __device__ constexpr bool row_needs_x_halo(int dz, int ey, int CY) {
  for (int i = 0; i < SH::NT; ++i) {
    const Off o = SH::tap(i);
    if (o.d0 != dz || o.d2 == 0) continue;
    // cell rows cy in [0, CY) reach ey = cy + d1
    if (ey - o.d1 >= 0 && ey - o.d1 < CY) return true;
  }
  return false;
}

template <class SH, int T, int CY, int CX, int NWY, int S, int FL = 0, class E = double>
struct Stream3DCfg {
  static constexpr int R = SH::R;
  static constexpr int Z = (offcentre_inplane<SH>() || (FL & 1)) ? R + 1 : R;  // level skew
  static constexpr int WN = 2 * R + (Z - R) + 1;                   // window planes
  static constexpr int NB = offcentre_inplane<SH>() ? Z + R + 1 : Z + 1;  // halo buffers
  static constexpr int LY = NWY * CY;
  static constexpr int LX = 32 * CX;
  static constexpr int HY = T * R;
  static constexpr int AL = 16 / (int)sizeof(E);
  static constexpr int HX = (T * R + AL - 1) / AL * AL;  // TMA: 16-byte aligned box start
  static constexpr int VY = LY - 2 * HY;
  static constexpr int VX = LX - 2 * HX;
  // Halo buffer: per warp, its top R and bottom R rows of a level's plane
  // ("push halo"); neighbours along axis 2 come from warp shuffles.
  static constexpr int HROWW = 2 * R;                 // rows per warp
  static constexpr int HPLANE = NWY * HROWW * LX;     // doubles per halo buffer
  static constexpr int RING_PLANE = LY * LX;          // elements per ring slot
  static constexpr int RING_BYTES = S * RING_PLANE * (int)sizeof(E);
  static constexpr int HALO_BYTES = T * NB * HPLANE * (int)sizeof(E);
  static constexpr int SMEM_BYTES = RING_BYTES + HALO_BYTES + S * 8;
  static_assert(CY >= R, "a warp's rows must cover the radius");
  static_assert(VY > 0 && VX > 0, "tile leaves no valid core");
  static_assert(LX <= 256 && LY <= 256, "TMA box dims are limited to 256");
  static_assert((S & (S - 1)) == 0, "ring slots must be a power of two");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
};

// Advances of a unit: [ka, ka + nadv), nadv rounded up to a multiple of WN so
// the unrolled loop never runs past the planes it loaded.  Planes >= n0 come
// back zero-filled from TMA; planes in [r1 + T*R, ka + nadv) only feed target
// planes >= r1, which are never stored.
template <int WN>
__host__ __device__ inline int stream3d_advances(int ka, int r1, int TZ) {
  const int n = r1 + TZ - ka;
  return (n + WN - 1) / WN * WN;
}

// One work unit (tile x z segment) of one epoch.  EDGE: the tile touches the
// frame along axis 1 or 2 (per-cell frame masks); frame planes along axis 0
// are handled per block of WN advances (FPL), so z-edge segments cost the same
// as interior ones outside their first and last blocks.  Returns the planes
// consumed from the ring.
template <class SH, int T, int CY, int CX, int NWY, int S, int FL, bool EXACT, bool UNI, bool EDGE,
          class E>
__device__ __forceinline__ int stream3d_unit(const CUtensorMap* tm, E* __restrict__ out,
                                             E* ring, E* halo, uint64_t* bars,
                                             uint32_t ring_cnt, int warp, int lane, int n0,
                                             int n1, int n2, int rp, int X0, int Y0, int xlo, int xhi,
                                             int ylo, int yhi, int r0, int r1,
                                             const Coefs<SH::NT, E>& cf) {
  using Cfg = Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>;
  constexpr int R = Cfg::R, Z = Cfg::Z, WN = Cfg::WN, NB = Cfg::NB;
  constexpr int LY = Cfg::LY, LX = Cfg::LX;
  constexpr int PLANE_BYTES = LY * LX * (int)sizeof(E);
  constexpr int TZ = T * Z;  // pipeline depth along z
  static_assert(CY * CX <= 32, "cell masks are 32-bit");

  const int ka = max(0, r0 - T * R);
  const int nadv = stream3d_advances<WN>(ka, r1, TZ);
  const int kend = ka + nadv;
  const int tid = warp * 32 + lane;
  const int ty0 = warp * CY;  // tile row of this thread's first row
  const int tx0 = lane * CX;  // tile column of this thread's first column

  if (tid == 0) {
    for (int i = 0; i < S && i < nadv; ++i) {
      const uint32_t slot = (ring_cnt + i) & (S - 1);
      mbar_arrive_expect_tx(&bars[slot], PLANE_BYTES);
      tma_load_3d(ring + slot * Cfg::RING_PLANE, tm, X0, Y0, ka + i, &bars[slot]);
    }
  }

  // per-cell masks, bit cy*CX+cx: frame cells (EDGE tiles) and stored cells
  uint32_t fmask = 0, stmask = 0;
#pragma unroll
  for (int cy = 0; cy < CY; ++cy)
#pragma unroll
    for (int cx = 0; cx < CX; ++cx) {
      const int yy = Y0 + ty0 + cy, xx = X0 + tx0 + cx;
      const bool f = EDGE && ((yy < R) || (yy >= n1 - R) || (xx < R) || (xx >= n2 - R));
      bool st = (yy >= ylo) && (yy < yhi) && (xx >= xlo) && (xx < xhi);
      if (UNI) st = st && !f;  // shared-product levels hold products; frame pre-copied
      fmask |= (uint32_t)f << (cy * CX + cx);
      stmask |= (uint32_t)st << (cy * CX + cx);
    }

  E win[T][WN][CY][CX];
#pragma unroll
  for (int s = 0; s < T; ++s)
#pragma unroll
    for (int w = 0; w < WN; ++w)
#pragma unroll
      for (int cy = 0; cy < CY; ++cy)
#pragma unroll
        for (int cx = 0; cx < CX; ++cx) win[s][w][cy][cx] = 0.0;

  // Halo buffer (level, b): warp-major [NWY][2R][LX]; this thread's columns.
  auto hrow = [&](int level, int b, int w, int r) -> E* {
    return halo + (size_t)(level * NB + b) * Cfg::HPLANE + (size_t)(w * 2 * R + r) * LX + tx0;
  };
  // push: top R rows and bottom R rows of this thread's block
  auto push = [&](int level, int b, const E (&v)[CY][CX]) {
    static_for<2 * R>([&](auto rI) {
      constexpr int r = decltype(rI)::value;
      constexpr int cy = r < R ? r : CY - 2 * R + r;
      E* d = hrow(level, b, warp, r);
      if constexpr (CX % 2 == 0) {
#pragma unroll
        for (int cx = 0; cx < CX; cx += 2)
          *reinterpret_cast<vec2_t<E>*>(d + cx) = make_v2<E>(v[cy][cx], v[cy][cx + 1]);
      } else {
#pragma unroll
        for (int cx = 0; cx < CX; ++cx) d[cx] = v[cy][cx];
      }
    });
  };
  // pull: rows above (the warp above's bottom rows) and below (the warp
  // below's top rows).  Edge warps of the tile read their own buffer rows:
  // those cells lie outside the tile's valid core anyway.
  const int wa = warp > 0 ? warp - 1 : warp;
  const int wbl = warp < NWY - 1 ? warp + 1 : warp;

  // output pointer of this thread's first cell in plane q = k - T*Z
  const long long plane = (long long)n1 * (long long)rp;
  E* obase = out + ((long long)(Y0 + ty0) * rp + (X0 + tx0));

  auto block = [&](int kbase, auto fpl_tag) {
    constexpr bool FPL = decltype(fpl_tag)::value;  // a target plane may be a frame plane
#pragma unroll
    for (int uu = 0; uu < WN; ++uu) {
      const int k = kbase + uu;
      const int bk = k % NB;  // halo buffer written this advance
      // ---- level 0 ----------------------------------------------------------
      {
        E v[CY][CX];
        const uint32_t pos = ring_cnt + (uint32_t)(k - ka);
        const uint32_t slot = pos & (S - 1);
        mbar_wait(&bars[slot], (pos / S) & 1);
        const E* p = ring + slot * Cfg::RING_PLANE + ty0 * LX + tx0;
#pragma unroll
        for (int cy = 0; cy < CY; ++cy) {
          if constexpr (CX % 2 == 0) {
#pragma unroll
            for (int cx = 0; cx < CX; cx += 2) {
              const vec2_t<E> t2 = *reinterpret_cast<const vec2_t<E>*>(p + cy * LX + cx);
              v[cy][cx] = t2.x;
              v[cy][cx + 1] = t2.y;
            }
          } else {
#pragma unroll
            for (int cx = 0; cx < CX; ++cx) v[cy][cx] = p[cy * LX + cx];
          }
        }
        // UNI: windows and halos carry products y = c*x (one DMUL per cell)
        if constexpr (UNI) {
#pragma unroll
          for (int cy = 0; cy < CY; ++cy)
#pragma unroll
            for (int cx = 0; cx < CX; ++cx) v[cy][cx] = mul_rn<E>(cf.c[0], v[cy][cx]);
        }
#pragma unroll
        for (int cy = 0; cy < CY; ++cy)
#pragma unroll
          for (int cx = 0; cx < CX; ++cx) win[0][uu][cy][cx] = v[cy][cx];
        push(0, bk, v);
      }
      // ---- levels 1..T --------------------------------------------------------
      static_for<T>([&](auto sI) {
        constexpr int s = decltype(sI)::value + 1;
        const int q = k - s * Z;  // target plane of level s
        bool fpl = false;         // frame plane: every cell carries level s-1
        if constexpr (FPL) fpl = (q < R) || (q >= n0 - R);
        E nv[CY][CX];
        {
          // extended neighbourhood of the planes that need in-plane values:
          // ext[dz][cy+R][cx+R], cy in [-R, CY+R), cx in [-R, CX+R)
          E ext[2 * R + 1][CY + 2 * R][CX + 2 * R];
          static_for<2 * R + 1>([&](auto zI) {
            constexpr int dz = decltype(zI)::value - R;
            if constexpr (plane_needs_inplane<SH>(dz)) {
              const int sl = pmod<WN>(uu - s * Z + dz);
              const int b = (k - Z + dz + NB * 4) % NB;  // written at advance k - Z + dz
#pragma unroll
              for (int cy = 0; cy < CY; ++cy)
#pragma unroll
                for (int cx = 0; cx < CX; ++cx) ext[zI][cy + R][cx + R] = win[s - 1][sl][cy][cx];
              // rows above / below from the halo buffer
#pragma unroll
              for (int r = 0; r < R; ++r) {
                const E* up = hrow(s - 1, b, wa, warp > 0 ? R + r : r);
                const E* dn = hrow(s - 1, b, wbl, warp < NWY - 1 ? r : R + r);
                if constexpr (CX % 2 == 0) {
#pragma unroll
                  for (int cx = 0; cx < CX; cx += 2) {
                    const vec2_t<E> a2 = *reinterpret_cast<const vec2_t<E>*>(up + cx);
                    const vec2_t<E> b2 = *reinterpret_cast<const vec2_t<E>*>(dn + cx);
                    ext[zI][r][cx + R] = a2.x;
                    ext[zI][r][cx + 1 + R] = a2.y;
                    ext[zI][CY + R + r][cx + R] = b2.x;
                    ext[zI][CY + R + r][cx + 1 + R] = b2.y;
                  }
                } else {
#pragma unroll
                  for (int cx = 0; cx < CX; ++cx) {
                    ext[zI][r][cx + R] = up[cx];
                    ext[zI][CY + R + r][cx + R] = dn[cx];
                  }
                }
              }
              // columns left / right from the neighbouring lanes
#pragma unroll
              for (int ey = 0; ey < CY + 2 * R; ++ey) {
                if (!row_needs_x_halo<SH>(dz, ey - R, CY)) continue;
#pragma unroll
                for (int j = 0; j < R; ++j) {
                  const int ccl = -R + j;
                  const int dl = (-ccl + CX - 1) / CX;
                  const int coll = ccl + dl * CX;
                  ext[zI][ey][j] = __shfl_up_sync(kFullMask, ext[zI][ey][coll + R], dl);
                  const int ccr = CX + j;
                  const int dr = ccr / CX;
                  const int colr = ccr - dr * CX;
                  ext[zI][ey][CX + R + j] = __shfl_down_sync(kFullMask, ext[zI][ey][colr + R], dr);
                }
              }
            }
          });
          // tap-major: CY*CX independent chains interleave in the instruction stream
          E acc[CY][CX];
          static_for<SH::NT>([&](auto iI) {
            constexpr int i = decltype(iI)::value;
            constexpr Off o = SH::tap(i);
#pragma unroll
            for (int cy = 0; cy < CY; ++cy) {
#pragma unroll
              for (int cx = 0; cx < CX; ++cx) {
                E x;
                if constexpr (plane_needs_inplane<SH>(o.d0))
                  x = ext[o.d0 + R][cy + o.d1 + R][cx + o.d2 + R];
                else
                  x = win[s - 1][pmod<WN>(uu - s * Z + o.d0)][cy][cx];
                if constexpr (UNI)
                  acc[cy][cx] = (i == 0) ? x : add_rn<E>(acc[cy][cx], x);
                else if constexpr (i == 0)
                  acc[cy][cx] = tap_first<EXACT>(cf.c[0], x);
                else
                  acc[cy][cx] = tap_next<EXACT>(acc[cy][cx], cf.c[i], x);
              }
            }
          });
#pragma unroll
          for (int cy = 0; cy < CY; ++cy)
#pragma unroll
            for (int cx = 0; cx < CX; ++cx) {
              // UNI: levels < T carry products; a frame cell's product never
              // changes, and level T skips frame cells (host pre-copies them)
              const E val =
                  (UNI && s < T) ? mul_rn<E>(cf.c[0], acc[cy][cx]) : acc[cy][cx];
              if constexpr (EDGE || FPL) {
                bool f = fpl;
                if constexpr (EDGE) f = f || ((fmask >> (cy * CX + cx)) & 1u);
                nv[cy][cx] = f ? win[s - 1][pmod<WN>(uu - s * Z)][cy][cx] : val;
              } else {
                nv[cy][cx] = val;
              }
            }
        }
        if constexpr (s < T) {
#pragma unroll
          for (int cy = 0; cy < CY; ++cy)
#pragma unroll
            for (int cx = 0; cx < CX; ++cx) win[s][pmod<WN>(uu - s * Z)][cy][cx] = nv[cy][cx];
          push(s, bk, nv);
        } else {
          bool qok = (q >= r0) && (q < r1);
          if (UNI && FPL) qok = qok && !fpl;
          if (qok) {
            E* o = obase + (long long)q * plane;
#pragma unroll
            for (int cy = 0; cy < CY; ++cy)
#pragma unroll
              for (int cx = 0; cx < CX; ++cx)
                if ((stmask >> (cy * CX + cx)) & 1u) o[(long long)cy * rp + cx] = nv[cy][cx];
          }
        }
      });
      // one barrier per advance: halo pushes visible, ring slot k consumed
      __syncthreads();
      if (tid == 0 && k + S < kend) {
        const uint32_t slot = (ring_cnt + (uint32_t)(k - ka)) & (S - 1);
        mbar_arrive_expect_tx(&bars[slot], PLANE_BYTES);
        tma_load_3d(ring + slot * Cfg::RING_PLANE, tm, X0, Y0, k + S, &bars[slot]);
      }
    }
  };

  for (int kbase = ka; kbase < kend; kbase += WN) {
    // target planes of this block: [kbase - TZ, kbase + WN - 1 - Z]
    if ((kbase - TZ < R) || (kbase + WN - 1 - Z >= n0 - R))
      block(kbase, std::true_type{});
    else
      block(kbase, std::false_type{});
  }
  return nadv;
}

// Radius-1 stars in catalog order ((-1,0,0), (0,0,0), (1,0,0), then in-plane
// taps of the centre plane): the z window of 3 planes per level collapses to 2
// values per cell -- the partial sum P = t(-1) + t(0) of the next target and
// the newest plane Y (the next target's centre).  Same operations in the same
// order, one third fewer window registers, no rotating window (unroll 1).
template <class SH>
__host__ __device__ constexpr bool ps_eligible() {
  if (!(SH::kStar && SH::R == 1 && SH::dims == 3)) return false;
  if (SH::tap(0).d0 != -1 || SH::tap(1).d0 != 0 || SH::tap(2).d0 != 1) return false;
  for (int i = 0; i < 3; ++i)
    if (SH::tap(i).d1 != 0 || SH::tap(i).d2 != 0) return false;
  for (int i = 3; i < SH::NT; ++i)
    if (SH::tap(i).d0 != 0) return false;
  return true;
}

template <class SH, int T, int CY, int CX, int NWY, int S, int FL, bool EXACT, bool UNI, bool EDGE,
          class E>
__device__ __forceinline__ int stream3d_unit_ps(const CUtensorMap* tm, E* __restrict__ out,
                                                E* ring, E* halo, uint64_t* bars,
                                                uint32_t ring_cnt, int warp, int lane, int n0,
                                                int n1, int n2, int rp, int X0, int Y0, int xlo,
                                                int xhi, int ylo, int yhi, int r0, int r1,
                                                const Coefs<SH::NT, E>& cf) {
  using Cfg = Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>;
  static_assert(ps_eligible<SH>(), "partial-sum path needs a radius-1 star in catalog order");
  constexpr int NB = Cfg::NB;
  constexpr int LY = Cfg::LY, LX = Cfg::LX;
  constexpr int PLANE_BYTES = LY * LX * (int)sizeof(E);
  static_assert(Cfg::Z == 1 && NB >= 2, "star skew");
  static_assert(CY * CX <= 32, "cell masks are 32-bit");

  const int ka = max(0, r0 - T);
  // level T emits plane k - T; advances run in pairs (the rolling Y/P state
  // then alternates between two register sets instead of being moved), and
  // an extra trailing advance only targets planes >= r1
  const int nadv = (r1 + T - ka + 1) & ~1;
  const int kend = ka + nadv;
  const int tid = warp * 32 + lane;
  const int ty0 = warp * CY;
  const int tx0 = lane * CX;

  if (tid == 0) {
    for (int i = 0; i < S && i < nadv; ++i) {
      const uint32_t slot = (ring_cnt + i) & (S - 1);
      mbar_arrive_expect_tx(&bars[slot], PLANE_BYTES);
      tma_load_3d(ring + slot * Cfg::RING_PLANE, tm, X0, Y0, ka + i, &bars[slot]);
    }
  }

  uint32_t fmask = 0, stmask = 0;
#pragma unroll
  for (int cy = 0; cy < CY; ++cy)
#pragma unroll
    for (int cx = 0; cx < CX; ++cx) {
      const int yy = Y0 + ty0 + cy, xx = X0 + tx0 + cx;
      const bool f = EDGE && ((yy < 1) || (yy >= n1 - 1) || (xx < 1) || (xx >= n2 - 1));
      bool st = (yy >= ylo) && (yy < yhi) && (xx >= xlo) && (xx < xhi);
      if (UNI) st = st && !f;
      fmask |= (uint32_t)f << (cy * CX + cx);
      stmask |= (uint32_t)st << (cy * CX + cx);
    }

  // Y[s]: newest plane of level s; P[s]: partial sum (taps 0 and 1) of level
  // s+1's next target.  Level s+1 at advance k targets q = k-s-1, whose centre
  // is Y[s] (produced last advance) and whose z+1 plane is produced now.
  E Y[T][CY][CX], P[T][CY][CX];
#pragma unroll
  for (int s = 0; s < T; ++s)
#pragma unroll
    for (int cy = 0; cy < CY; ++cy)
#pragma unroll
      for (int cx = 0; cx < CX; ++cx) Y[s][cy][cx] = P[s][cy][cx] = 0.0;

  auto hrow = [&](int level, int b, int w, int r) -> E* {
    return halo + (size_t)(level * NB + b) * Cfg::HPLANE + (size_t)(w * 2 + r) * LX + tx0;
  };
  auto push = [&](int level, int b, const E (&v)[CY][CX]) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int cy = r == 0 ? 0 : CY - 1;
      E* d = hrow(level, b, warp, r);
#pragma unroll
      for (int cx = 0; cx < CX; cx += 2)
        *reinterpret_cast<vec2_t<E>*>(d + cx) = make_v2<E>(v[cy][cx], v[cy][cx + 1]);
    }
  };
  const int wa = warp > 0 ? warp - 1 : warp;
  const int wbl = warp < NWY - 1 ? warp + 1 : warp;
  const long long plane = (long long)n1 * (long long)rp;
  E* obase = out + ((long long)(Y0 + ty0) * rp + (X0 + tx0));

  auto advance = [&](int k, auto fpl_tag) {
    constexpr bool FPL = decltype(fpl_tag)::value;
    const int bk = k & (NB - 1);        // halo buffer written this advance
    const int bp = (k - 1) & (NB - 1);  // centre planes were pushed last advance
    E nw[CY][CX];                  // newest plane of the level below
    {
      const uint32_t pos = ring_cnt + (uint32_t)(k - ka);
      const uint32_t slot = pos & (S - 1);
      mbar_wait(&bars[slot], (pos / S) & 1);
      const E* p = ring + slot * Cfg::RING_PLANE + ty0 * LX + tx0;
#pragma unroll
      for (int cy = 0; cy < CY; ++cy)
#pragma unroll
        for (int cx = 0; cx < CX; cx += 2) {
          const vec2_t<E> t2 = *reinterpret_cast<const vec2_t<E>*>(p + cy * LX + cx);
          nw[cy][cx] = UNI ? mul_rn<E>(cf.c[0], t2.x) : t2.x;
          nw[cy][cx + 1] = UNI ? mul_rn<E>(cf.c[0], t2.y) : t2.y;
        }
      push(0, bk, nw);
    }
    static_for<T>([&](auto sI) {
      constexpr int s = decltype(sI)::value + 1;  // level produced
      const int q = k - s;
      bool fpl = false;
      if constexpr (FPL) fpl = (q < 1) || (q >= n0 - 1);
      // centre plane of level s-1 with its in-plane halo
      E ext[CY + 2][CX + 2];
#pragma unroll
      for (int cy = 0; cy < CY; ++cy)
#pragma unroll
        for (int cx = 0; cx < CX; ++cx) ext[cy + 1][cx + 1] = Y[s - 1][cy][cx];
      {
        const E* up = hrow(s - 1, bp, wa, warp > 0 ? 1 : 0);
        const E* dn = hrow(s - 1, bp, wbl, warp < NWY - 1 ? 0 : 1);
#pragma unroll
        for (int cx = 0; cx < CX; cx += 2) {
          const vec2_t<E> a2 = *reinterpret_cast<const vec2_t<E>*>(up + cx);
          const vec2_t<E> b2 = *reinterpret_cast<const vec2_t<E>*>(dn + cx);
          ext[0][cx + 1] = a2.x;
          ext[0][cx + 2] = a2.y;
          ext[CY + 1][cx + 1] = b2.x;
          ext[CY + 1][cx + 2] = b2.y;
        }
      }
#pragma unroll
      for (int cy = 1; cy <= CY; ++cy) {
        ext[cy][0] = __shfl_up_sync(kFullMask, ext[cy][CX], 1);
        ext[cy][CX + 1] = __shfl_down_sync(kFullMask, ext[cy][1], 1);
      }
      E nv[CY][CX];
#pragma unroll
      for (int cy = 0; cy < CY; ++cy)
#pragma unroll
        for (int cx = 0; cx < CX; ++cx) {
          E acc;
          if constexpr (UNI)
            acc = add_rn<E>(P[s - 1][cy][cx], nw[cy][cx]);
          else
            acc = tap_next<EXACT>(P[s - 1][cy][cx], cf.c[2], nw[cy][cx]);
          static_for<SH::NT - 3>([&](auto iI) {
            constexpr int i = decltype(iI)::value + 3;
            constexpr Off o = SH::tap(i);
            const E x = ext[cy + 1 + o.d1][cx + 1 + o.d2];
            if constexpr (UNI)
              acc = add_rn<E>(acc, x);
            else
              acc = tap_next<EXACT>(acc, cf.c[i], x);
          });
          const E val = (UNI && s < T) ? mul_rn<E>(cf.c[0], acc) : acc;
          if constexpr (EDGE || FPL) {
            bool f = fpl;
            if constexpr (EDGE) f = f || ((fmask >> (cy * CX + cx)) & 1u);
            nv[cy][cx] = f ? Y[s - 1][cy][cx] : val;
          } else {
            nv[cy][cx] = val;
          }
        }
      // roll level s-1's state: next target's first two taps, newest plane
#pragma unroll
      for (int cy = 0; cy < CY; ++cy)
#pragma unroll
        for (int cx = 0; cx < CX; ++cx) {
          if constexpr (UNI)
            P[s - 1][cy][cx] = add_rn<E>(Y[s - 1][cy][cx], nw[cy][cx]);
          else
            P[s - 1][cy][cx] = tap_next<EXACT>(tap_first<EXACT>(cf.c[0], Y[s - 1][cy][cx]),
                                               cf.c[1], nw[cy][cx]);
          Y[s - 1][cy][cx] = nw[cy][cx];
          nw[cy][cx] = nv[cy][cx];
        }
      if constexpr (s < T) {
        push(s, bk, nv);
      } else {
        bool qok = (q >= r0) && (q < r1);
        if (UNI && FPL) qok = qok && !fpl;
        if (qok) {
          E* o = obase + (long long)q * plane;
#pragma unroll
          for (int cy = 0; cy < CY; ++cy)
#pragma unroll
            for (int cx = 0; cx < CX; ++cx)
              if ((stmask >> (cy * CX + cx)) & 1u) o[(long long)cy * rp + cx] = nv[cy][cx];
        }
      }
    });
    __syncthreads();
    if (tid == 0 && k + S < kend) {
      const uint32_t slot = (ring_cnt + (uint32_t)(k - ka)) & (S - 1);
      mbar_arrive_expect_tx(&bars[slot], PLANE_BYTES);
      tma_load_3d(ring + slot * Cfg::RING_PLANE, tm, X0, Y0, k + S, &bars[slot]);
    }
  };

  for (int k = ka; k < kend; k += 2) {
    // target planes of these two advances: [k - T, k]
    if ((k - T < 1) || (k >= n0 - 1)) {
      advance(k, std::true_type{});
      advance(k + 1, std::true_type{});
    } else {
      advance(k, std::false_type{});
      advance(k + 1, std::false_type{});
    }
  }
  return nadv;
}

// Plane-major radius-1 stencils (j3d27pt, j3d17pt, poisson: taps sorted by
// axis-0 offset, the catalog's lexicographic order): each plane of the level
// below is gathered with its in-plane neighbourhood ONCE and feeds the three
// targets it touches -- the z+1 taps of target c-1 (completing it), the z taps
// of target c, the z-1 taps of target c+1 -- as consecutive runs of the
// reference order.  A level keeps two partial sums, the plane it will consume
// next and the plane it consumed last (frame carry): no 3-plane neighbourhood
// per advance, a third of the shuffles and halo loads of the window path.

// ---- tolerance mode (exact = 0, uniform coefficients): reassociated sums ----
// With one coefficient c for every tap, sum_k c*x_k = c * sum_k x_k, and the
// sum may be regrouped: the north star's fp64 tolerance (1e-12 relative)
// admits any order.  A plane's in-plane taps are then a "pattern" sum that
// is the same for every target the plane feeds (j3d27pt: the 3x3 box for all
// three targets), computed ONCE per plane as separable column sums: 6 DP per
// j3d27pt cell-step instead of 27.
//   pat3_mask(dz): 9-bit mask of the in-plane offsets (d1, d2) with d0 = dz
//   pat3_col(dz, dx): 3-bit set of rows d1 in column d2 = dx of that pattern
template <class SH>
__host__ __device__ constexpr uint32_t pat3_mask(int dz) {
  uint32_t m = 0;
  for (int i = 0; i < SH::NT; ++i)
    if (SH::tap(i).d0 == dz) m |= 1u << ((SH::tap(i).d1 + 1) * 3 + (SH::tap(i).d2 + 1));
  return m;
}
template <class SH>
__host__ __device__ constexpr int pat3_col(int dz, int dx) {
  int s = 0;
  for (int dy = -1; dy <= 1; ++dy)
    if ((pat3_mask<SH>(dz) >> ((dy + 1) * 3 + (dx + 1))) & 1u) s |= 1 << (dy + 1);
  return s;
}
// column sum over row set RS needed at all / needed in a neighbour column
template <class SH>
__host__ __device__ constexpr bool pat3_rs_used(int rs, bool shifted) {
  for (int dz = -1; dz <= 1; ++dz)
    for (int dx = -1; dx <= 1; ++dx)
      if (pat3_col<SH>(dz, dx) == rs && (!shifted || dx != 0)) return true;
  return false;
}
// first dz with the same pattern (pattern sums are computed once)
template <class SH>
__host__ __device__ constexpr int pat3_canon(int dz) {
  for (int d = -1; d < dz; ++d)
    if (pat3_mask<SH>(d) == pat3_mask<SH>(dz)) return d;
  return dz;
}

template <class SH>
__host__ __device__ constexpr bool pm_eligible() {
  if (SH::dims != 3 || SH::R != 1 || SH::kStar) return false;
  for (int i = 1; i < SH::NT; ++i)
    if (SH::tap(i).d0 < SH::tap(i - 1).d0) return false;
  return true;
}

template <class SH, int T, int CY, int CX, int NWY, int S, int FL, bool EXACT, bool UNI, bool EDGE,
          class E>
__device__ __forceinline__ int stream3d_unit_pm(const CUtensorMap* tm, E* __restrict__ out,
                                                E* ring, E* halo, uint64_t* bars,
                                                uint32_t ring_cnt, int warp, int lane, int n0,
                                                int n1, int n2, int rp, int X0, int Y0, int xlo,
                                                int xhi, int ylo, int yhi, int r0, int r1,
                                                const Coefs<SH::NT, E>& cf) {
  using Cfg = Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>;
  static_assert(pm_eligible<SH>(), "plane-major path needs sorted radius-1 taps");
  constexpr int NB = Cfg::NB;
  constexpr int LY = Cfg::LY, LX = Cfg::LX;
  constexpr int PLANE_BYTES = LY * LX * (int)sizeof(E);
  static_assert(NB >= 2, "halo slots");
  static_assert(CY * CX <= 32, "cell masks are 32-bit");
  static_assert(CX % 2 == 0, "vec2_t<E> rows");

  const int ka = max(0, r0 - T);
  // level s emits plane k - 2s; advances in pairs (register sets alternate)
  const int nadv = (r1 + 2 * T - ka + 1) & ~1;
  const int kend = ka + nadv;
  const int tid = warp * 32 + lane;
  const int ty0 = warp * CY;
  const int tx0 = lane * CX;

  if (tid == 0) {
    for (int i = 0; i < S && i < nadv; ++i) {
      const uint32_t slot = (ring_cnt + i) & (S - 1);
      mbar_arrive_expect_tx(&bars[slot], PLANE_BYTES);
      tma_load_3d(ring + slot * Cfg::RING_PLANE, tm, X0, Y0, ka + i, &bars[slot]);
    }
  }

  uint32_t fmask = 0, stmask = 0;
#pragma unroll
  for (int cy = 0; cy < CY; ++cy)
#pragma unroll
    for (int cx = 0; cx < CX; ++cx) {
      const int yy = Y0 + ty0 + cy, xx = X0 + tx0 + cx;
      const bool f = EDGE && ((yy < 1) || (yy >= n1 - 1) || (xx < 1) || (xx >= n2 - 1));
      bool st = (yy >= ylo) && (yy < yhi) && (xx >= xlo) && (xx < xhi);
      if (UNI) st = st && !f;
      fmask |= (uint32_t)f << (cy * CX + cx);
      stmask |= (uint32_t)st << (cy * CX + cx);
    }

  // per level s (1..T), index s-1:  A = target c+1 after its z-1 taps,
  // B = target c after its z-1 and z taps, Yc = the level-below plane to
  // consume next advance, Yp = the one consumed last (frame carry)
  E A[T][CY][CX], B[T][CY][CX], Yc[T][CY][CX], Yp[T][CY][CX];
#pragma unroll
  for (int s = 0; s < T; ++s)
#pragma unroll
    for (int cy = 0; cy < CY; ++cy)
#pragma unroll
      for (int cx = 0; cx < CX; ++cx) A[s][cy][cx] = B[s][cy][cx] = Yc[s][cy][cx] = Yp[s][cy][cx] = 0.0;

  auto hrow = [&](int level, int b, int w, int r) -> E* {
    return halo + (size_t)(level * NB + b) * Cfg::HPLANE + (size_t)(w * 2 + r) * LX + tx0;
  };
  auto push = [&](int level, int b, const E (&v)[CY][CX]) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int cy = r == 0 ? 0 : CY - 1;
      E* d = hrow(level, b, warp, r);
#pragma unroll
      for (int cx = 0; cx < CX; cx += 2)
        *reinterpret_cast<vec2_t<E>*>(d + cx) = make_v2<E>(v[cy][cx], v[cy][cx + 1]);
    }
  };
  const int wa = warp > 0 ? warp - 1 : warp;
  const int wbl = warp < NWY - 1 ? warp + 1 : warp;
  const long long plane = (long long)n1 * (long long)rp;
  E* obase = out + ((long long)(Y0 + ty0) * rp + (X0 + tx0));

  // sum of the taps with axis-0 offset DZ over the gathered neighbourhood,
  // starting from `acc` (FIRST: the run opens the target's sum)
  auto run_taps = [&](auto dz_tag, auto first_tag, const E (&e)[CY + 2][CX + 2], int cy,
                      int cx, E acc) -> E {
    constexpr int DZ = decltype(dz_tag)::value;
    constexpr bool FIRST = decltype(first_tag)::value;
    static_for<SH::NT>([&](auto iI) {
      constexpr int i = decltype(iI)::value;
      constexpr Off o = SH::tap(i);
      if constexpr (o.d0 == DZ) {
        const E x = e[cy + 1 + o.d1][cx + 1 + o.d2];
        constexpr bool OPEN = FIRST && (i == 0 || SH::tap(i > 0 ? i - 1 : 0).d0 != DZ);
        if constexpr (UNI)
          acc = OPEN ? x : add_rn<E>(acc, x);
        else if constexpr (OPEN)
          acc = tap_first<EXACT>(cf.c[i], x);
        else
          acc = tap_next<EXACT>(acc, cf.c[i], x);
      }
    });
    return acc;
  };

  // Tolerance mode: level s consumes plane p (the level below, produced last
  // advance) through its pattern sums -- target c-1 gets pattern(+1) and
  // completes, target c gets pattern(0), target c+1 opens with pattern(-1).
  constexpr bool RA = UNI && !EXACT;
  int bk = 0, bp = 0;
  auto ra_level = [&](auto s_tag, int q, bool fpl, E (&nw)[CY][CX]) {
    constexpr int s = decltype(s_tag)::value;
    // plane rows -1..CY (halo rows from the warps above / below), own columns
    E e[CY + 2][CX];
#pragma unroll
    for (int cy = 0; cy < CY; ++cy)
#pragma unroll
      for (int cx = 0; cx < CX; ++cx) e[cy + 1][cx] = Yc[s - 1][cy][cx];
    {
      const E* up = hrow(s - 1, bp, wa, warp > 0 ? 1 : 0);
      const E* dn = hrow(s - 1, bp, wbl, warp < NWY - 1 ? 0 : 1);
#pragma unroll
      for (int cx = 0; cx < CX; cx += 2) {
        const vec2_t<E> a2 = *reinterpret_cast<const vec2_t<E>*>(up + cx);
        const vec2_t<E> b2 = *reinterpret_cast<const vec2_t<E>*>(dn + cx);
        e[0][cx] = a2.x;
        e[0][cx + 1] = a2.y;
        e[CY + 1][cx] = b2.x;
        e[CY + 1][cx + 1] = b2.y;
      }
    }
    // column sums cs[rs][cy][cx + 1] over row set rs (bit dy+1), own columns;
    // neighbour columns -1 / CX by shuffles where a pattern reaches them
    E cs[8][CY][CX + 2];
    static_for<8>([&](auto rI) {
      constexpr int RS = decltype(rI)::value;
      if constexpr (RS != 0 && pat3_rs_used<SH>(RS, false)) {
#pragma unroll
        for (int cx = 0; cx < CX; ++cx) {
          if constexpr (RS == 7 && CY % 2 == 0) {
            // rows cy-1..cy+1: the pair (cy, cy+1) is shared by outputs cy, cy+1
#pragma unroll
            for (int cy = 0; cy < CY; cy += 2) {
              const E m = add_rn<E>(e[cy + 1][cx], e[cy + 2][cx]);
              cs[RS][cy][cx + 1] = add_rn<E>(e[cy][cx], m);
              cs[RS][cy + 1][cx + 1] = add_rn<E>(m, e[cy + 3][cx]);
            }
          } else {
#pragma unroll
            for (int cy = 0; cy < CY; ++cy) {
              E a = E(0);
              bool first = true;
#pragma unroll
              for (int dy = -1; dy <= 1; ++dy)
                if ((RS >> (dy + 1)) & 1) {
                  a = first ? e[cy + 1 + dy][cx] : add_rn<E>(a, e[cy + 1 + dy][cx]);
                  first = false;
                }
              cs[RS][cy][cx + 1] = a;
            }
          }
        }
        if constexpr (pat3_rs_used<SH>(RS, true)) {
#pragma unroll
          for (int cy = 0; cy < CY; ++cy) {
            cs[RS][cy][0] = __shfl_up_sync(kFullMask, cs[RS][cy][CX], 1);
            cs[RS][cy][CX + 1] = __shfl_down_sync(kFullMask, cs[RS][cy][1], 1);
          }
        }
      }
    });
    // pattern sums of dz = -1, 0, +1 (identical patterns computed once)
    E ps[3][CY][CX];
    static_for<3>([&](auto zI) {
      constexpr int dz = decltype(zI)::value - 1;
      if constexpr (pat3_canon<SH>(dz) == dz && pat3_mask<SH>(dz) != 0) {
        constexpr int c0 = pat3_col<SH>(dz, -1), c1 = pat3_col<SH>(dz, 0),
                      c2 = pat3_col<SH>(dz, 1);
#pragma unroll
        for (int cy = 0; cy < CY; ++cy) {
          if constexpr (c0 == 7 && c1 == 7 && c2 == 7 && CX % 2 == 0) {
#pragma unroll
            for (int cx = 0; cx < CX; cx += 2) {
              const E m = add_rn<E>(cs[7][cy][cx + 1], cs[7][cy][cx + 2]);
              ps[zI][cy][cx] = add_rn<E>(cs[7][cy][cx], m);
              ps[zI][cy][cx + 1] = add_rn<E>(m, cs[7][cy][cx + 3]);
            }
          } else {
#pragma unroll
            for (int cx = 0; cx < CX; ++cx) {
              E a = E(0);
              bool first = true;
              if constexpr (c1 != 0) {
                a = cs[c1][cy][cx + 1];
                first = false;
              }
              if constexpr (c0 != 0) {
                a = first ? cs[c0][cy][cx] : add_rn<E>(a, cs[c0][cy][cx]);
                first = false;
              }
              if constexpr (c2 != 0) a = first ? cs[c2][cy][cx + 2] : add_rn<E>(a, cs[c2][cy][cx + 2]);
              ps[zI][cy][cx] = a;
            }
          }
        }
      }
    });
    constexpr int zm = pat3_canon<SH>(-1) + 1, z0 = pat3_canon<SH>(0) + 1,
                  zp = pat3_canon<SH>(1) + 1;
    E nv[CY][CX];
#pragma unroll
    for (int cy = 0; cy < CY; ++cy)
#pragma unroll
      for (int cx = 0; cx < CX; ++cx) {
        const E Cq = pat3_mask<SH>(1) ? add_rn<E>(B[s - 1][cy][cx], ps[zp][cy][cx]) : B[s - 1][cy][cx];
        const E Bn = pat3_mask<SH>(0) ? add_rn<E>(A[s - 1][cy][cx], ps[z0][cy][cx]) : A[s - 1][cy][cx];
        const E An = pat3_mask<SH>(-1) ? ps[zm][cy][cx] : E(0);
        const E val = s < T ? mul_rn<E>(cf.c[0], Cq) : Cq;
        bool f = fpl;
        if constexpr (EDGE) f = f || ((fmask >> (cy * CX + cx)) & 1u);
        nv[cy][cx] = f ? Yp[s - 1][cy][cx] : val;
        A[s - 1][cy][cx] = An;
        B[s - 1][cy][cx] = Bn;
        Yp[s - 1][cy][cx] = Yc[s - 1][cy][cx];
        Yc[s - 1][cy][cx] = nw[cy][cx];
        nw[cy][cx] = nv[cy][cx];
      }
    if constexpr (s < T) {
      push(s, bk, nv);
    } else {
      if (q >= r0 && q < r1 && !fpl) {
        E* o = obase + (long long)q * plane;
#pragma unroll
        for (int cy = 0; cy < CY; ++cy)
#pragma unroll
          for (int cx = 0; cx < CX; ++cx)
            if ((stmask >> (cy * CX + cx)) & 1u) o[(long long)cy * rp + cx] = nv[cy][cx];
      }
    }
  };

  auto advance = [&](int k, auto fpl_tag) {
    constexpr bool FPL = decltype(fpl_tag)::value;
    bk = k & (NB - 1);
    bp = (k - 1) & (NB - 1);
    E nw[CY][CX];  // newest plane of the level below (produced this advance)
    {
      const uint32_t pos = ring_cnt + (uint32_t)(k - ka);
      const uint32_t slot = pos & (S - 1);
      mbar_wait(&bars[slot], (pos / S) & 1);
      const E* p = ring + slot * Cfg::RING_PLANE + ty0 * LX + tx0;
#pragma unroll
      for (int cy = 0; cy < CY; ++cy)
#pragma unroll
        for (int cx = 0; cx < CX; cx += 2) {
          const vec2_t<E> t2 = *reinterpret_cast<const vec2_t<E>*>(p + cy * LX + cx);
          nw[cy][cx] = UNI ? mul_rn<E>(cf.c[0], t2.x) : t2.x;
          nw[cy][cx + 1] = UNI ? mul_rn<E>(cf.c[0], t2.y) : t2.y;
        }
      push(0, bk, nw);
    }
    static_for<T>([&](auto sI) {
      constexpr int s = decltype(sI)::value + 1;
      const int q = k - 2 * s;  // target completed this advance (= consumed plane - 1)
      bool fpl = false;
      if constexpr (FPL) fpl = (q < 1) || (q >= n0 - 1);
      if constexpr (RA) {
        ra_level(std::integral_constant<int, s>{}, q, fpl, nw);
        return;
      }
      // gather the consumed plane (level s-1, produced last advance) once
      E e[CY + 2][CX + 2];
#pragma unroll
      for (int cy = 0; cy < CY; ++cy)
#pragma unroll
        for (int cx = 0; cx < CX; ++cx) e[cy + 1][cx + 1] = Yc[s - 1][cy][cx];
      {
        const E* up = hrow(s - 1, bp, wa, warp > 0 ? 1 : 0);
        const E* dn = hrow(s - 1, bp, wbl, warp < NWY - 1 ? 0 : 1);
#pragma unroll
        for (int cx = 0; cx < CX; cx += 2) {
          const vec2_t<E> a2 = *reinterpret_cast<const vec2_t<E>*>(up + cx);
          const vec2_t<E> b2 = *reinterpret_cast<const vec2_t<E>*>(dn + cx);
          e[0][cx + 1] = a2.x;
          e[0][cx + 2] = a2.y;
          e[CY + 1][cx + 1] = b2.x;
          e[CY + 1][cx + 2] = b2.y;
        }
      }
#pragma unroll
      for (int ey = 0; ey < CY + 2; ++ey) {
        e[ey][0] = __shfl_up_sync(kFullMask, e[ey][CX], 1);
        e[ey][CX + 1] = __shfl_down_sync(kFullMask, e[ey][1], 1);
      }
      E nv[CY][CX];
#pragma unroll
      for (int cy = 0; cy < CY; ++cy)
#pragma unroll
        for (int cx = 0; cx < CX; ++cx) {
          const E C = run_taps(std::integral_constant<int, 1>{}, std::false_type{}, e, cy,
                                    cx, B[s - 1][cy][cx]);
          const E Bn = run_taps(std::integral_constant<int, 0>{}, std::false_type{}, e,
                                     cy, cx, A[s - 1][cy][cx]);
          const E An = run_taps(std::integral_constant<int, -1>{}, std::true_type{}, e, cy,
                                     cx, 0.0);
          const E val = (UNI && s < T) ? mul_rn<E>(cf.c[0], C) : C;
          if constexpr (EDGE || FPL) {
            bool f = fpl;
            if constexpr (EDGE) f = f || ((fmask >> (cy * CX + cx)) & 1u);
            nv[cy][cx] = f ? Yp[s - 1][cy][cx] : val;
          } else {
            nv[cy][cx] = val;
          }
          A[s - 1][cy][cx] = An;
          B[s - 1][cy][cx] = Bn;
          Yp[s - 1][cy][cx] = Yc[s - 1][cy][cx];
          Yc[s - 1][cy][cx] = nw[cy][cx];
          nw[cy][cx] = nv[cy][cx];
        }
      if constexpr (s < T) {
        push(s, bk, nv);
      } else {
        bool qok = (q >= r0) && (q < r1);
        if (UNI && FPL) qok = qok && !fpl;
        if (qok) {
          E* o = obase + (long long)q * plane;
#pragma unroll
          for (int cy = 0; cy < CY; ++cy)
#pragma unroll
            for (int cx = 0; cx < CX; ++cx)
              if ((stmask >> (cy * CX + cx)) & 1u) o[(long long)cy * rp + cx] = nv[cy][cx];
        }
      }
    });
    __syncthreads();
    if (tid == 0 && k + S < kend) {
      const uint32_t slot = (ring_cnt + (uint32_t)(k - ka)) & (S - 1);
      mbar_arrive_expect_tx(&bars[slot], PLANE_BYTES);
      tma_load_3d(ring + slot * Cfg::RING_PLANE, tm, X0, Y0, k + S, &bars[slot]);
    }
  };

  for (int k = ka; k < kend; k += 2) {
    // targets of these two advances: [k - 2T, k - 1]
    if ((k - 2 * T < 1) || (k - 1 >= n0 - 1)) {
      advance(k, std::true_type{});
      advance(k + 1, std::true_type{});
    } else {
      advance(k, std::false_type{});
      advance(k + 1, std::false_type{});
    }
  }
  return nadv;
}

template <class SH, int T, int CY, int CX, int NWY, int S, int FL, bool EXACT, bool UNI, int MINB,
          class E = double>
__global__ void __launch_bounds__(NWY * 32, MINB)
    k_stream3d(const __grid_constant__ TmapSet maps, const Stream3DArgs a,
               const __grid_constant__ Coefs<SH::NT, E> cf) {
  using Cfg = Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>;
  constexpr int R = Cfg::R;
  extern __shared__ __align__(1024) unsigned char smem[];
  E* ring = reinterpret_cast<E*>(smem);
  E* halo = reinterpret_cast<E*>(smem + Cfg::RING_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::RING_BYTES + Cfg::HALO_BYTES);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
    fence_mbarrier_init();
    prefetch_tmap(&maps.m[0]);
    prefetch_tmap(&maps.m[1]);
    prefetch_tmap(&maps.m[2]);
  }
  __syncthreads();

  const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
  const int tiles = a.nty * a.ntx;
  const int units = tiles * a.nseg;
  uint32_t ring_cnt = 0;
  int src = a.first_src, dst = a.first_dst;
  for (int e = 0; e < a.epochs; ++e) {
    const CUtensorMap* tm = &maps.m[src];
    E* __restrict__ out = static_cast<E*>((dst == BUF_OUT) ? a.buf[BUF_OUT] : a.buf[BUF_SCR]);
    __shared__ int s_unit;
    for (;;) {
      // dynamic unit distribution across CTAs (tail <= one unit)
      if (threadIdx.x == 0) s_unit = atomicAdd(a.work + e, 1);
      __syncthreads();
      const int u = s_unit;
      if (u >= units) break;
      // segment-major order: the long segments are handed out first and the
      // short tail segments last (guided scheduling, see Stream3DArgs)
      const int j = u / tiles;
      const int tile = u - j * tiles;
      const int tx = tile % a.ntx;
      const int ty = tile / a.ntx;
      const int r0 = a.seg_start[j];
      const int r1 = a.seg_start[j + 1];
      // edge-aligned tiles (a.aligned_x/y): the first tile starts at the
      // domain edge and the last ends there -- the frame needs no halo, so
      // those tiles keep the margin on one side only (fewer tiles per axis)
      // (x geometry over the 16-byte-aligned width: with an odd, row-padded
      // last extent the last tile starts on a TMA-aligned column and may store
      // into the pad column, which is never read)
      const int n2g = (n2 + Cfg::AL - 1) / Cfg::AL * Cfg::AL;
      const StripGeom gx = tile3d_strip(tx, a.ntx, a.aligned_x, n2g, Cfg::LX, Cfg::VX, Cfg::HX);
      const StripGeom gy = tile3d_strip(ty, a.nty, a.aligned_y, n1, Cfg::LY, Cfg::VY, Cfg::HY);
      const int X0 = gx.X0, Y0 = gy.X0;
      const int TR = T * R;
      (void)TR;
      const bool edge = (X0 < R) || (X0 + Cfg::LX > n2 - R) || (Y0 < R) || (Y0 + Cfg::LY > n1 - R);
      int used;
      if constexpr (pm_eligible<SH>() && (FL & 1) == 0) {
        if (edge)
          used = stream3d_unit_pm<SH, T, CY, CX, NWY, S, FL, EXACT, UNI, true, E>(
              tm, out, ring, halo, bars, ring_cnt, warp, lane, n0, n1, n2, a.pitch, X0, Y0, gx.vlo, gx.vhi,
              gy.vlo, gy.vhi, r0, r1, cf);
        else
          used = stream3d_unit_pm<SH, T, CY, CX, NWY, S, FL, EXACT, UNI, false, E>(
              tm, out, ring, halo, bars, ring_cnt, warp, lane, n0, n1, n2, a.pitch, X0, Y0, gx.vlo, gx.vhi,
              gy.vlo, gy.vhi, r0, r1, cf);
      } else if constexpr (ps_eligible<SH>() && (FL & 1) == 0) {
        if (edge)
          used = stream3d_unit_ps<SH, T, CY, CX, NWY, S, FL, EXACT, UNI, true, E>(
              tm, out, ring, halo, bars, ring_cnt, warp, lane, n0, n1, n2, a.pitch, X0, Y0, gx.vlo, gx.vhi, gy.vlo, gy.vhi, r0, r1, cf);
        else
          used = stream3d_unit_ps<SH, T, CY, CX, NWY, S, FL, EXACT, UNI, false, E>(
              tm, out, ring, halo, bars, ring_cnt, warp, lane, n0, n1, n2, a.pitch, X0, Y0, gx.vlo, gx.vhi, gy.vlo, gy.vhi, r0, r1, cf);
      } else if (edge)
        used = stream3d_unit<SH, T, CY, CX, NWY, S, FL, EXACT, UNI, true, E>(
            tm, out, ring, halo, bars, ring_cnt, warp, lane, n0, n1, n2, a.pitch, X0, Y0, gx.vlo, gx.vhi, gy.vlo, gy.vhi, r0, r1, cf);
      else
        used = stream3d_unit<SH, T, CY, CX, NWY, S, FL, EXACT, UNI, false, E>(
            tm, out, ring, halo, bars, ring_cnt, warp, lane, n0, n1, n2, a.pitch, X0, Y0, gx.vlo, gx.vhi, gy.vlo, gy.vhi, r0, r1, cf);
      ring_cnt += (uint32_t)used;
      __syncthreads();  // halo buffers and s_unit are reused by the next unit
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
}

}  // namespace ebisu

// ebisu_stream3d_cl.cuh -- 3-D streaming temporal blocking over 2-CTA
// clusters (sm_100a thread-block clusters + distributed shared memory).
//
// Why: the overlapped 3-D tile is capped by ONE SM's register file (the T
// fused levels of a 32x64 tile fill 8 warps x 254 registers), and its valid
// fraction is (LY-2TR)(LX-2TR)/(LY*LX) = 0.656 at t=4.  A cluster of two CTAs
// on two SMs streams ONE 64x64 tile: rank 0 owns rows [0, 32), rank 1 rows
// [32, 64).  Only the pair's outer edges carry the t*R overlap halo; across
// the seam the two CTAs exchange, every advance and every level, the one row
// each side needs -- the reference device-tiling scheme's per-level halo
// exchange (engine/device.py:292-389, Listing 3), here between the
// shared memories of two SMs instead of through global memory.  Valid
// fraction 0.766 at t=4 (+17 %).
//
// Seam exchange (point to point, no cluster-wide barrier per advance):
//  * the seam warp of each rank (rank 0: its last warp; rank 1: warp 0)
//    writes its seam row of every level straight into the PEER's receive
//    ring xin[slot][level] with st.async (16 B per lane), each completing its
//    bytes on the peer's full[slot] mbarrier (complete_tx) -- the TMA-style
//    handshake: no release fence, so the producer never waits for its own
//    outstanding HBM stores (a release.cluster arrive compiles to
//    MEMBAR.ALL.GPU, and its acquire twin to an L1 invalidate: measured 2x
//    slower);
//  * at the next advance the peer's seam warp arms full[slot] with the
//    expected bytes, waits on it, reads its own xin[slot], and arrives
//    (relaxed, remote) on the producer's empty[slot] once the values are in
//    registers; the producer waits on empty[slot] before reusing that slot
//    NBX advances later.
//  Both ranks run the same unit sequence (rank 0 claims the unit and hands
//  it over through DSMEM behind a cluster barrier), so their advance
//  counters agree and the mbarrier phases line up.  Deadlock-free: an
//  advance's pushes wait only on the consumer's progress NBX-1 >= 1 advances
//  back.
//
// Everything else is the partial-sum radius-1-star kernel of
// ebisu_stream3d.cuh (stream3d_unit_ps): same operations in the same order,
// bitwise equal to reference_run.
#pragma once

#include <cooperative_groups.h>

#include "ebisu_common.cuh"
#include "ebisu_shapes.cuh"
#include "ebisu_stream2d.cuh"
#include "ebisu_stream3d.cuh"

namespace ebisu {

// (cluster / DSMEM primitives: ebisu_common.cuh)

// Seam area layout (after the one-CTA kernel's ring, halo buffers and ring
// barriers): receive ring xin[NBX][T][LX], full[NBX] (one mbarrier per slot:
// all T rows of an advance; per-level barriers measured slower, 538 vs 601
// GCells/s at t=3), empty[NBX], unit id.
template <int T, int LX, int NBX>
struct SeamBufs {
  static constexpr int XIN_DOUBLES = NBX * T * LX;
  static constexpr int FULL_OFF = XIN_DOUBLES * 8;
  static constexpr int EMPTY_OFF = FULL_OFF + NBX * 8;
  static constexpr int UNIT_OFF = EMPTY_OFF + NBX * 8;
  static constexpr int BYTES = UNIT_OFF + 16;
};

template <class SH, int T, int CY, int CX, int NWY, int S>
struct Stream3DClCfg {
  using Base = Stream3DCfg<SH, T, CY, CX, NWY, S, 0, double>;
  static constexpr int NBX = 4;  // seam receive slots (producer slack NBX-1 advances)
  static constexpr int LY = Base::LY;        // rows per CTA
  static constexpr int LY2 = 2 * LY;         // rows per cluster tile
  static constexpr int VY2 = LY2 - 2 * Base::HY;
  static constexpr int SEAM_OFF = Base::SMEM_BYTES;  // after ring + halo + ring barriers
  static constexpr int SMEM_BYTES = SEAM_OFF + SeamBufs<T, Base::LX, NBX>::BYTES;
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory budget");
  static_assert(ps_eligible<SH>(), "cluster kernel: radius-1 star in catalog order");
};

// One unit (cluster tile x z segment) on one rank.  acnt: running advance
// counter (identical on both ranks) driving the seam ring phases.
template <class SH, int T, int CY, int CX, int NWY, int S, bool UNI, bool EDGE, int RANK>
__device__ __forceinline__ int stream3d_unit_cl(
    const CUtensorMap* tm, double* __restrict__ out, uint32_t ring_cnt, uint32_t& acnt,
    int warp, int lane, int n0, int n1, int n2, int rp, int X0, int Y0, int xlo, int xhi, int ylo,
    int yhi, int r0, int r1, const Coefs<SH::NT, double>& cf) {
  using E = double;
  using ClCfg = Stream3DClCfg<SH, T, CY, CX, NWY, S>;
  using Cfg = typename ClCfg::Base;
  using SB = SeamBufs<T, Cfg::LX, ClCfg::NBX>;
  constexpr int NB = Cfg::NB;
  constexpr int NBX = ClCfg::NBX;
  constexpr int LY = Cfg::LY, LX = Cfg::LX;
  constexpr int PLANE_BYTES = LY * LX * 8;
  constexpr uint32_t SEAM_BYTES = T * LX * 8;  // the T seam rows of one advance
  constexpr uint32_t PEER = RANK ^ 1;
  static_assert(Cfg::Z == 1 && NB >= 2, "star skew");
  static_assert(CY * CX <= 32 && CX % 2 == 0, "cell masks / vector seam stores");
  // shared-memory carve-up at compile-time offsets (no pointer registers)
  extern __shared__ __align__(1024) unsigned char smem[];
  E* ring = reinterpret_cast<E*>(smem);
  E* halo = reinterpret_cast<E*>(smem + Cfg::RING_BYTES);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::RING_BYTES + Cfg::HALO_BYTES);
  E* xin = reinterpret_cast<E*>(smem + ClCfg::SEAM_OFF);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ClCfg::SEAM_OFF + SB::FULL_OFF);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + ClCfg::SEAM_OFF + SB::EMPTY_OFF);

  const int ka = max(0, r0 - T);
  const int nadv = (r1 + T - ka + 1) & ~1;
  const int kend = ka + nadv;
  const int tid = warp * 32 + lane;
  const int ty0 = warp * CY;
  const int tx0 = lane * CX;
  // the seam: rank 0's last warp sends its bottom row down, rank 1's warp 0
  // sends its top row up; each receives the other's row for its pull
  const bool seam = warp == (RANK == 0 ? NWY - 1 : 0);
  constexpr int seam_cy = RANK == 0 ? CY - 1 : 0;

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
  // push: the CTA-local halo rows, and on the seam warp the seam row into
  // the peer's receive slot `xs` (level `level`)
  auto push = [&](int level, int b, int xs, const E (&v)[CY][CX]) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      const int cy = r == 0 ? 0 : CY - 1;
      E* d = hrow(level, b, warp, r);
#pragma unroll
      for (int cx = 0; cx < CX; cx += 2)
        *reinterpret_cast<vec2_t<E>*>(d + cx) = make_v2<E>(v[cy][cx], v[cy][cx + 1]);
    }
    if (seam) {
      const uint32_t dst = mapa_shared(xin + ((xs * T + level) * LX + tx0), PEER);
      const uint32_t bar = mapa_shared(full + xs, PEER);
#pragma unroll
      for (int cx = 0; cx < CX; cx += 2)
        st_async_v2f64(dst + cx * 8, v[seam_cy][cx], v[seam_cy][cx + 1], bar);
    }
  };
  // neighbours inside the CTA; the seam side reads the receive ring instead
  const int wa = warp > 0 ? warp - 1 : warp;
  const int wbl = warp < NWY - 1 ? warp + 1 : warp;
  const long long plane = (long long)n1 * (long long)rp;
  E* obase = out + ((long long)(Y0 + ty0) * rp + (X0 + tx0));

  auto advance = [&](int k, auto fpl_tag) {
    constexpr bool FPL = decltype(fpl_tag)::value;
    const int bk = k & (NB - 1);
    const int bp = (k - 1) & (NB - 1);
    const uint32_t u = acnt;                 // this advance's global index
    const int xs = (int)(u % NBX);           // seam slot written this advance
    const int xr = (int)((u + NBX - 1) % NBX);  // slot holding the previous advance
    if (seam && u >= NBX) {
      // the peer has consumed what we wrote into slot xs NBX advances ago
      mbar_wait(&empty[xs], ((u / NBX) - 1) & 1);
    }
    E nw[CY][CX];
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
      push(0, bk, xs, nw);
    }
    static_for<T>([&](auto sI) {
      constexpr int s = decltype(sI)::value + 1;
      const int q = k - s;
      // the peer's seam rows of the previous advance: arm the slot with the
      // bytes it expects and wait for them (before the first level's pull)
      if constexpr (s == 1) {
        if (seam && u >= 1) {
          if (lane == 0) mbar_arrive_expect_tx(full + xr, SEAM_BYTES);
          mbar_wait(full + xr, ((u - 1) / NBX) & 1);
        }
      }
      bool fpl = false;
      if constexpr (FPL) fpl = (q < 1) || (q >= n0 - 1);
      E ext[CY + 2][CX + 2];
#pragma unroll
      for (int cy = 0; cy < CY; ++cy)
#pragma unroll
        for (int cx = 0; cx < CX; ++cx) ext[cy + 1][cx + 1] = Y[s - 1][cy][cx];
      {
        const E* up = hrow(s - 1, bp, wa, warp > 0 ? 1 : 0);
        const E* dn = hrow(s - 1, bp, wbl, warp < NWY - 1 ? 0 : 1);
        const E* xrow = xin + (size_t)((xr * T + (s - 1)) * LX + tx0);
        if (seam) {
          if constexpr (RANK == 0)
            dn = xrow;
          else
            up = xrow;
        }
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
            acc = tap_next<true>(P[s - 1][cy][cx], cf.c[2], nw[cy][cx]);
          static_for<SH::NT - 3>([&](auto iI) {
            constexpr int i = decltype(iI)::value + 3;
            constexpr Off o = SH::tap(i);
            const E x = ext[cy + 1 + o.d1][cx + 1 + o.d2];
            if constexpr (UNI)
              acc = add_rn<E>(acc, x);
            else
              acc = tap_next<true>(acc, cf.c[i], x);
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
#pragma unroll
      for (int cy = 0; cy < CY; ++cy)
#pragma unroll
        for (int cx = 0; cx < CX; ++cx) {
          if constexpr (UNI)
            P[s - 1][cy][cx] = add_rn<E>(Y[s - 1][cy][cx], nw[cy][cx]);
          else
            P[s - 1][cy][cx] = tap_next<true>(tap_first<true>(cf.c[0], Y[s - 1][cy][cx]),
                                              cf.c[1], nw[cy][cx]);
          Y[s - 1][cy][cx] = nw[cy][cx];
          nw[cy][cx] = nv[cy][cx];
        }
      if constexpr (s < T) {
        push(s, bk, xs, nv);
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
    if (seam && u >= 1) {
      // slot xr consumed (its values have fed this advance's sums)
      __syncwarp();
      if (lane == 0) mbar_arrive_remote_relaxed(mapa_shared(empty + xr, PEER));
    }
    __syncthreads();
    if (tid == 0 && k + S < kend) {
      const uint32_t slot = (ring_cnt + (uint32_t)(k - ka)) & (S - 1);
      mbar_arrive_expect_tx(&bars[slot], PLANE_BYTES);
      tma_load_3d(ring + slot * Cfg::RING_PLANE, tm, X0, Y0, k + S, &bars[slot]);
    }
    ++acnt;
  };

  for (int k = ka; k < kend; k += 2) {
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

// Cluster (2, 1, 1): blockIdx.x pairs (rank = %cluster_ctarank).  Units are
// (cluster tile, z segment); geometry along axis 1 uses the 2*LY-row tile.
template <class SH, int T, int CY, int CX, int NWY, int S, bool UNI, int MINB>
__global__ void __launch_bounds__(NWY * 32, MINB)
    k_stream3d_cl(const __grid_constant__ TmapSet maps, const Stream3DArgs a,
                  const __grid_constant__ Coefs<SH::NT, double> cf) {
  using ClCfg = Stream3DClCfg<SH, T, CY, CX, NWY, S>;
  using Cfg = typename ClCfg::Base;
  constexpr int NBX = ClCfg::NBX;
  extern __shared__ __align__(1024) unsigned char smem[];
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + Cfg::RING_BYTES + Cfg::HALO_BYTES);
  using SB = SeamBufs<T, Cfg::LX, NBX>;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ClCfg::SEAM_OFF + SB::FULL_OFF);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem + ClCfg::SEAM_OFF + SB::EMPTY_OFF);
  int* s_unit = reinterpret_cast<int*>(smem + ClCfg::SEAM_OFF + SB::UNIT_OFF);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int rank = (int)cluster_ctarank();
  const uint32_t peer = (uint32_t)(rank ^ 1);

  if (threadIdx.x == 0) {
#pragma unroll
    for (int i = 0; i < S; ++i) mbar_init(&bars[i], 1);
    for (int i = 0; i < NBX; ++i)
      mbar_init(&full[i], 1);   // our seam warp's expect_tx; the bytes come by st.async
    for (int i = 0; i < NBX; ++i)
      mbar_init(&empty[i], 1);  // the peer seam warp's consumed token
    fence_mbarrier_init();
    prefetch_tmap(&maps.m[0]);
    prefetch_tmap(&maps.m[1]);
    prefetch_tmap(&maps.m[2]);
  }
  // the peer's barriers must be initialised before anyone arrives on them
  cluster_sync_all();
  const uint32_t peer_unit = mapa_shared(s_unit, peer);

  const int n0 = a.n0, n1 = a.n1, n2 = a.n2;
  const int tiles = a.nty * a.ntx;
  const int units = tiles * a.nseg;
  uint32_t ring_cnt = 0, acnt = 0;
  int src = a.first_src, dst = a.first_dst;
  for (int e = 0; e < a.epochs; ++e) {
    const CUtensorMap* tm = &maps.m[src];
    double* __restrict__ out =
        static_cast<double*>((dst == BUF_OUT) ? a.buf[BUF_OUT] : a.buf[BUF_SCR]);
    for (;;) {
      // rank 0 claims the next unit for the pair; both ranks see it after the
      // cluster barrier (which also retires the previous unit on both SMs)
      if (rank == 0 && threadIdx.x == 0) {
        const int u = atomicAdd(a.work + e, 1);
        *s_unit = u;
        st_cluster_u32(peer_unit, (uint32_t)u);
      }
      cluster_sync_all();
      const int u = *s_unit;
      cluster_sync_all();  // both ranks have read it: the next claim may overwrite
      if (u >= units) break;
      const int j = u / tiles;
      const int tile = u - j * tiles;
      const int tx = tile % a.ntx;
      const int ty = tile / a.ntx;
      const int r0 = a.seg_start[j];
      const int r1 = a.seg_start[j + 1];
      const StripGeom gx = stream2d_strip(tx, a.ntx, a.aligned_x, n2, Cfg::LX, Cfg::VX, Cfg::HX,
                                          Cfg::AL);
      const StripGeom gy =
          stream2d_strip(ty, a.nty, a.aligned_y, n1, ClCfg::LY2, ClCfg::VY2, Cfg::HY);
      const int X0 = gx.X0, Y0 = gy.X0 + rank * Cfg::LY;  // this rank's rows of the pair tile
      constexpr int R = 1;
      const bool edge =
          (X0 < R) || (X0 + Cfg::LX > n2 - R) || (Y0 < R) || (Y0 + Cfg::LY > n1 - R);
      int used;
#define EBISU_CL_UNIT(EDGE_, RANK_)                                                          \
  stream3d_unit_cl<SH, T, CY, CX, NWY, S, UNI, EDGE_, RANK_>(tm, out, ring_cnt, acnt, warp,   \
                                                             lane, n0, n1, n2, a.pitch, X0, Y0, \
                                                             gx.vlo, gx.vhi, gy.vlo, gy.vhi,   \
                                                             r0, r1, cf)
      if (rank == 0)
        used = edge ? EBISU_CL_UNIT(true, 0) : EBISU_CL_UNIT(false, 0);
      else
        used = edge ? EBISU_CL_UNIT(true, 1) : EBISU_CL_UNIT(false, 1);
#undef EBISU_CL_UNIT
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
  // no CTA may exit while its peer can still touch its shared memory
  cluster_sync_all();
}

}  // namespace ebisu

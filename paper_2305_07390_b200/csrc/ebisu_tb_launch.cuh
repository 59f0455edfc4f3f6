// ebisu_tb_launch.cuh -- host launch wrappers + registry entries for the
// temporal-blocking kernel instantiations.
#pragma once

#include <string.h>

#include "ebisu_internal.h"
#include "ebisu_stream2d.cuh"
#include "ebisu_stream3d.cuh"
#include "ebisu_halo2d.cuh"
#include "ebisu_stream3d_cl.cuh"

namespace ebisu {

template <class SH, int T, int C, int NW, int S, bool EXACT, bool UNI, int MINB, class E,
          int SHIFT = 0>
cudaError_t launch_stream2d(const TbLaunch& L) {
  using Cfg = Stream2DCfg<SH, T, C, NW, S, E>;
  auto kern = k_stream2d<SH, T, C, NW, S, EXACT, UNI, MINB, E, SHIFT>;
  cudaError_t err =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (err != cudaSuccess) return err;
  TmapSet maps;
  memcpy(&maps.m[0], L.maps, 3 * sizeof(CUtensorMap));
  Stream2DArgs a;
  a.n0 = L.n0;
  a.n1 = L.n1;
  a.nstrips = L.nstrips;
  a.nseg = L.nseg;
  a.seg_len = L.seg_len;
  a.z_lo = L.z_lo;
  a.z_hi = L.z_hi;
  a.epochs = L.epochs;
  a.first_src = L.first_src;
  a.first_dst = L.first_dst;
  a.aligned = L.aligned;
  a.pitch = L.pitch;
  if (L.nseg > EBISU_MAX_SEGS) return cudaErrorInvalidValue;
  for (int j = 0; j <= L.nseg; ++j) a.seg_start[j] = L.seg_start[j];
  for (int i = 0; i < 3; ++i) a.buf[i] = L.buf[i];
  a.unit_clock = L.unit_clock;
  a.work = L.work;
  a.flags = L.flags;
  Coefs<SH::NT, E> cf;
  for (int i = 0; i < SH::NT; ++i) cf.c[i] = (E)L.coeffs[i];
  if (L.cooperative) {
    void* args[] = {(void*)&maps, (void*)&a, (void*)&cf};
    return cudaLaunchCooperativeKernel((const void*)kern, dim3(L.grid), dim3(NW * 32), args,
                                       (size_t)Cfg::SMEM_BYTES, L.stream);
  }
  kern<<<L.grid, NW * 32, Cfg::SMEM_BYTES, L.stream>>>(maps, a, cf);
  return cudaGetLastError();
}

// Register-budget heuristic: the windows hold T*(2R+1)*C doubles (2 registers
// each) plus ~64 registers of addressing, halos and accumulators.  (The old
// estimate 4*T*R*C+48 capped t=4..7 at 128/168 registers and spilled.)
#ifndef EBISU_MINB_BIAS
#define EBISU_MINB_BIAS 0
#endif
constexpr int s2d_minb(int T, int R, int C, int NW, int ebytes = 8) {
  const int est = ebytes / 4 * T * (2 * R + 1) * C + 64;
  int m = 65536 / (NW * 32 * (est < 64 ? 64 : est)) + EBISU_MINB_BIAS;
  return m < 1 ? 1 : (m > 8 ? 8 : m);
}

#define EBISU_S2D_ENTRY(SHAPE_ID, SH, T, C, NW, S, EX, UNI, E) \
  EBISU_S2D_ENTRY_SH(SHAPE_ID, SH, T, C, NW, S, EX, UNI, E, 0)
// SHIFT: 0 = rotating register windows, U > 0 = shifted windows with U
// advances per unrolled block (see stream2d_unit)
#define EBISU_S2D_ENTRY_SH(SHAPE_ID, SH, T, C, NW, S, EX, UNI, E, SHIFT)                       \
  TbKernel {                                                                                  \
    SHAPE_ID, 2, T, C, NW, S, EX, UNI, Stream2DCfg<SH, T, C, NW, S, E>::SMEM_BYTES, 32 * C, 1, \
        1, Stream2DCfg<SH, T, C, NW, S, E>::VW, 0, 0, 0,                                     \
        (const void*)&k_stream2d<SH, T, C, NW, S, (EX) != 0, (UNI) != 0,                      \
                                 s2d_minb(T, SH::R, C, NW, (int)sizeof(E)), E, SHIFT>,        \
        &launch_stream2d<SH, T, C, NW, S, (EX) != 0, (UNI) != 0,                              \
                         s2d_minb(T, SH::R, C, NW, (int)sizeof(E)), E, SHIFT>,                \
        0, (int)sizeof(E)                                                                     \
  }

// explicit MINB (CTAs per SM the register budget targets)
#define EBISU_S2D_ENTRY_M(SHAPE_ID, SH, T, C, NW, S, EX, UNI, E, SHIFT, MINB)                  \
  TbKernel {                                                                                  \
    SHAPE_ID, 2, T, C, NW, S, EX, UNI, Stream2DCfg<SH, T, C, NW, S, E>::SMEM_BYTES, 32 * C, 1, \
        1, Stream2DCfg<SH, T, C, NW, S, E>::VW, 0, 0, 0,                                     \
        (const void*)&k_stream2d<SH, T, C, NW, S, (EX) != 0, (UNI) != 0, MINB, E, SHIFT>,     \
        &launch_stream2d<SH, T, C, NW, S, (EX) != 0, (UNI) != 0, MINB, E, SHIFT>, 0,          \
        (int)sizeof(E)                                                                        \
  }

template <class SH, int T, int CY, int CX, int NWY, int S, int FL, bool EXACT, bool UNI, int MINB,
          class E>
cudaError_t launch_stream3d(const TbLaunch& L) {
  using Cfg = Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>;
  auto kern = k_stream3d<SH, T, CY, CX, NWY, S, FL, EXACT, UNI, MINB, E>;
  cudaError_t err =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (err != cudaSuccess) return err;
  TmapSet maps;
  memcpy(&maps.m[0], L.maps, 3 * sizeof(CUtensorMap));
  Stream3DArgs a;
  a.n0 = L.n0;
  a.n1 = L.n1;
  a.n2 = L.n2;
  a.pitch = L.pitch;
  a.nty = L.nty;
  a.ntx = L.ntx;
  a.aligned_x = L.aligned_x;
  a.aligned_y = L.aligned_y;
  a.nseg = L.nseg;
  a.seg_len = L.seg_len;
  a.z_lo = L.z_lo;
  a.z_hi = L.z_hi;
  if (L.nseg > EBISU_MAX_SEGS) return cudaErrorInvalidValue;
  for (int j = 0; j <= L.nseg; ++j) a.seg_start[j] = L.seg_start[j];
  a.epochs = L.epochs;
  a.first_src = L.first_src;
  a.first_dst = L.first_dst;
  for (int i = 0; i < 3; ++i) a.buf[i] = L.buf[i];
  a.work = L.work;
  Coefs<SH::NT, E> cf;
  for (int i = 0; i < SH::NT; ++i) cf.c[i] = (E)L.coeffs[i];
  if (L.cooperative) {
    void* args[] = {(void*)&maps, (void*)&a, (void*)&cf};
    return cudaLaunchCooperativeKernel((const void*)kern, dim3(L.grid), dim3(NWY * 32), args,
                                       (size_t)Cfg::SMEM_BYTES, L.stream);
  }
  kern<<<L.grid, NWY * 32, Cfg::SMEM_BYTES, L.stream>>>(maps, a, cf);
  return cudaGetLastError();
}

#define EBISU_S3D_ENTRY(SHAPE_ID, SH, T, CY, CX, NWY, S, FL, EX, UNI, MINB, E)                 \
  TbKernel {                                                                                  \
    SHAPE_ID, 3, T, CX, NWY, S, EX, UNI, Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>::SMEM_BYTES, \
        Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>::LX,                                        \
        Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>::LY, 1,                                     \
        Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>::VX,                                        \
        Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>::VY,                                        \
        Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>::Z,                                         \
        ((ps_eligible<SH>() || pm_eligible<SH>()) && ((FL) & 1) == 0)                        \
            ? 2                                                                               \
            : Stream3DCfg<SH, T, CY, CX, NWY, S, FL, E>::WN,                                  \
        (const void*)&k_stream3d<SH, T, CY, CX, NWY, S, FL, (EX) != 0, (UNI) != 0, MINB, E>,  \
        &launch_stream3d<SH, T, CY, CX, NWY, S, FL, (EX) != 0, (UNI) != 0, MINB, E>, 0,      \
        (int)sizeof(E)                                                                        \
  }

// 2-CTA cluster kernel (ebisu_stream3d_cl.cuh): cudaLaunchKernelEx with a
// (2, 1, 1) cluster, cooperative when the sweep has several epochs.
template <class SH, int T, int CY, int CX, int NWY, int S, bool UNI, int MINB>
cudaError_t launch_stream3d_cl(const TbLaunch& L) {
  using ClCfg = Stream3DClCfg<SH, T, CY, CX, NWY, S>;
  auto kern = k_stream3d_cl<SH, T, CY, CX, NWY, S, UNI, MINB>;
  cudaError_t err =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ClCfg::SMEM_BYTES);
  if (err != cudaSuccess) return err;
  TmapSet maps;
  memcpy(&maps.m[0], L.maps, 3 * sizeof(CUtensorMap));
  Stream3DArgs a;
  a.n0 = L.n0;
  a.n1 = L.n1;
  a.n2 = L.n2;
  a.pitch = L.pitch;
  a.nty = L.nty;
  a.ntx = L.ntx;
  a.aligned_x = L.aligned_x;
  a.aligned_y = L.aligned_y;
  a.nseg = L.nseg;
  a.seg_len = L.seg_len;
  a.z_lo = L.z_lo;
  a.z_hi = L.z_hi;
  if (L.nseg > EBISU_MAX_SEGS) return cudaErrorInvalidValue;
  for (int j = 0; j <= L.nseg; ++j) a.seg_start[j] = L.seg_start[j];
  a.epochs = L.epochs;
  a.first_src = L.first_src;
  a.first_dst = L.first_dst;
  for (int i = 0; i < 3; ++i) a.buf[i] = L.buf[i];
  a.work = L.work;
  Coefs<SH::NT, double> cf;
  for (int i = 0; i < SH::NT; ++i) cf.c[i] = L.coeffs[i];
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(L.grid);
  cfg.blockDim = dim3(NWY * 32);
  cfg.dynamicSmemBytes = (size_t)ClCfg::SMEM_BYTES;
  cfg.stream = L.stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = 2;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeCooperative;
  attrs[1].val.cooperative = L.cooperative ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  return cudaLaunchKernelEx(&cfg, kern, maps, a, cf);
}

// resident clusters of the cluster kernel (occupancy query for the planner)
template <class SH, int T, int CY, int CX, int NWY, int S, bool UNI, int MINB>
cudaError_t clusters_stream3d_cl(int* n) {
  using ClCfg = Stream3DClCfg<SH, T, CY, CX, NWY, S>;
  auto kern = k_stream3d_cl<SH, T, CY, CX, NWY, S, UNI, MINB>;
  cudaError_t err =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, ClCfg::SMEM_BYTES);
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(2);
  cfg.blockDim = dim3(NWY * 32);
  cfg.dynamicSmemBytes = (size_t)ClCfg::SMEM_BYTES;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = 2;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(n, (const void*)kern, &cfg);
}

#define EBISU_S3D_CL_ENTRY(SHAPE_ID, SH, T, CY, CX, NWY, S, UNI, MINB)                        \
  TbKernel {                                                                                  \
    SHAPE_ID, 3, T, CX, NWY, S, 1, UNI, Stream3DClCfg<SH, T, CY, CX, NWY, S>::SMEM_BYTES,     \
        Stream3DCfg<SH, T, CY, CX, NWY, S, 0, double>::LX,                                    \
        Stream3DCfg<SH, T, CY, CX, NWY, S, 0, double>::LY, 1,                                 \
        Stream3DCfg<SH, T, CY, CX, NWY, S, 0, double>::VX,                                    \
        Stream3DClCfg<SH, T, CY, CX, NWY, S>::VY2, 1, 2,                                      \
        (const void*)&k_stream3d_cl<SH, T, CY, CX, NWY, S, (UNI) != 0, MINB>,                 \
        &launch_stream3d_cl<SH, T, CY, CX, NWY, S, (UNI) != 0, MINB>, 0, 8, 2,                \
        &clusters_stream3d_cl<SH, T, CY, CX, NWY, S, (UNI) != 0, MINB>                        \
  }

template <class SH, int T, int C, int NW, int S, bool EXACT, bool UNI, int MINB, int SHIFT,
          bool CLU>
cudaError_t launch_halo2d(const TbLaunch& L) {
  using Cfg = Halo2DCfg<SH, T, C, NW, S>;
  auto kern = k_halo2d<SH, T, C, NW, S, EXACT, UNI, MINB, SHIFT, CLU>;
  if (!CLU && L.cluster != 1) return cudaErrorInvalidValue;
  cudaError_t err =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (err != cudaSuccess) return err;
  TmapSet maps;
  memcpy(&maps.m[0], L.maps, 3 * sizeof(CUtensorMap));
  Halo2DArgs a;
  a.n0 = L.n0;
  a.n1 = L.n1;
  a.nstrips = L.nstrips;
  a.nseg = L.nseg;
  a.seg_len = L.seg_len;
  a.z_lo = L.z_lo;
  a.z_hi = L.z_hi;
  a.epochs = L.epochs;
  a.first_src = L.first_src;
  a.first_dst = L.first_dst;
  a.aligned = L.aligned;
  a.pitch = L.pitch;
  for (int i = 0; i < 3; ++i) a.buf[i] = static_cast<double*>(L.buf[i]);
  a.work = L.work;
  Coefs<SH::NT> cf;
  for (int i = 0; i < SH::NT; ++i) cf.c[i] = L.coeffs[i];
  // clusters of L.cluster CTAs along x (the device tile), cooperative when
  // the sweep has several epochs
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(L.grid);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = (size_t)Cfg::SMEM_BYTES;
  cfg.stream = L.stream;
  cudaLaunchAttribute attrs[2];
  attrs[0].id = cudaLaunchAttributeClusterDimension;
  attrs[0].val.clusterDim.x = (unsigned)L.cluster;
  attrs[0].val.clusterDim.y = 1;
  attrs[0].val.clusterDim.z = 1;
  attrs[1].id = cudaLaunchAttributeCooperative;
  attrs[1].val.cooperative = L.cooperative ? 1 : 0;
  cfg.attrs = attrs;
  cfg.numAttrs = 2;
  if (L.cluster > 8) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return err;
  }
  return cudaLaunchKernelEx(&cfg, kern, maps, a, cf);
}

// resident clusters of n CTAs (occupancy query for the planner)
template <class SH, int T, int C, int NW, int S, bool EXACT, bool UNI, int MINB, int SHIFT>
cudaError_t max_clusters_halo2d(int n, int* out) {
  using Cfg = Halo2DCfg<SH, T, C, NW, S>;
  auto kern = k_halo2d<SH, T, C, NW, S, EXACT, UNI, MINB, SHIFT, true>;
  cudaError_t err =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (err != cudaSuccess) return err;
  if (n > 8) {
    err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (err != cudaSuccess) return err;
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(n * 64);
  cfg.blockDim = dim3(NW * 32);
  cfg.dynamicSmemBytes = (size_t)Cfg::SMEM_BYTES;
  cudaLaunchAttribute attr;
  attr.id = cudaLaunchAttributeClusterDimension;
  attr.val.clusterDim.x = (unsigned)n;
  attr.val.clusterDim.y = 1;
  attr.val.clusterDim.z = 1;
  cfg.attrs = &attr;
  cfg.numAttrs = 1;
  return cudaOccupancyMaxActiveClusters(out, (const void*)kern, &cfg);
}

// box0 = warp columns (TMA box), valid_x = valid columns per CTA strip, C =
// cells per lane, z = level skew, wn = strip columns (LW)
#define EBISU_H2D_ENTRY(SHAPE_ID, SH, T, C, NW, S, EX, UNI, MINB) \
  EBISU_H2D_ENTRY_SH(SHAPE_ID, SH, T, C, NW, S, EX, UNI, MINB, 0)
#define EBISU_H2D_ENTRY_SH(SHAPE_ID, SH, T, C, NW, S, EX, UNI, MINB, SHIFT)                    \
  TbKernel {                                                                                  \
    SHAPE_ID, 2, T, C, NW, S, EX, UNI, Halo2DCfg<SH, T, C, NW, S>::SMEM_BYTES, 32 * C, 1, 1,   \
        Halo2DCfg<SH, T, C, NW, S>::VW, 0, Halo2DCfg<SH, T, C, NW, S>::Z,                     \
        Halo2DCfg<SH, T, C, NW, S>::LW,                                                       \
        (const void*)&k_halo2d<SH, T, C, NW, S, (EX) != 0, (UNI) != 0, MINB, SHIFT, false>,   \
        &launch_halo2d<SH, T, C, NW, S, (EX) != 0, (UNI) != 0, MINB, SHIFT, false>, 1, 8      \
  }
// cluster-tile twin (device tile of several CTAs, DSMEM seam exchange):
// registered after the single-CTA kernels; the planner picks it when the
// device tile spans more than one CTA
#define EBISU_H2D_ENTRY_CL(SHAPE_ID, SH, T, C, NW, S, EX, UNI, MINB, SHIFT)                    \
  TbKernel {                                                                                  \
    SHAPE_ID, 2, T, C, NW, S, EX, UNI, Halo2DCfg<SH, T, C, NW, S>::SMEM_BYTES, 32 * C, 1, 1,   \
        Halo2DCfg<SH, T, C, NW, S>::VW, 0, Halo2DCfg<SH, T, C, NW, S>::Z,                     \
        Halo2DCfg<SH, T, C, NW, S>::LW,                                                       \
        (const void*)&k_halo2d<SH, T, C, NW, S, (EX) != 0, (UNI) != 0, MINB, SHIFT, true>,    \
        &launch_halo2d<SH, T, C, NW, S, (EX) != 0, (UNI) != 0, MINB, SHIFT, true>, 1, 8, 1,   \
        nullptr, &max_clusters_halo2d<SH, T, C, NW, S, (EX) != 0, (UNI) != 0, MINB, SHIFT>    \
  }

}  // namespace ebisu

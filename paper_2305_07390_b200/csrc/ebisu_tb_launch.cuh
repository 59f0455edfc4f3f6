// ebisu_tb_launch.cuh -- host launch wrappers + registry entries for the
// temporal-blocking kernel instantiations.
#pragma once

#include <string.h>

#include "ebisu_internal.h"
#include "ebisu_stream2d.cuh"
#include "ebisu_stream3d.cuh"

namespace ebisu {

template <class SH, int T, int C, int NW, int S, bool EXACT, int MINB>
cudaError_t launch_stream2d(const TbLaunch& L) {
  using Cfg = Stream2DCfg<SH, T, C, NW, S>;
  auto kern = k_stream2d<SH, T, C, NW, S, EXACT, MINB>;
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
  a.epochs = L.epochs;
  a.first_src = L.first_src;
  a.first_dst = L.first_dst;
  a.aligned = L.aligned;
  for (int i = 0; i < 3; ++i) a.buf[i] = L.buf[i];
  a.unit_clock = L.unit_clock;
  a.work = L.work;
  Coefs<SH::NT> cf;
  for (int i = 0; i < SH::NT; ++i) cf.c[i] = L.coeffs[i];
  if (L.cooperative) {
    void* args[] = {(void*)&maps, (void*)&a, (void*)&cf};
    return cudaLaunchCooperativeKernel((const void*)kern, dim3(L.grid), dim3(NW * 32), args,
                                       (size_t)Cfg::SMEM_BYTES, L.stream);
  }
  kern<<<L.grid, NW * 32, Cfg::SMEM_BYTES, L.stream>>>(maps, a, cf);
  return cudaGetLastError();
}

// Register-budget heuristic: the window holds ~T*2R*C doubles live.
#ifndef EBISU_MINB_BIAS
#define EBISU_MINB_BIAS 0
#endif
constexpr int s2d_minb(int T, int R, int C, int NW) {
  const int est = 4 * T * R * C + 48;
  int m = 65536 / (NW * 32 * (est < 64 ? 64 : est)) + EBISU_MINB_BIAS;
  return m < 1 ? 1 : (m > 8 ? 8 : m);
}

#define EBISU_S2D_ENTRY(SHAPE_ID, SH, T, C, NW, S, EX)                                         \
  TbKernel {                                                                                  \
    SHAPE_ID, 2, T, C, NW, S, EX, Stream2DCfg<SH, T, C, NW, S>::SMEM_BYTES, 32 * C, 1, 1,      \
        Stream2DCfg<SH, T, C, NW, S>::VW, 0,                                                  \
        (const void*)&k_stream2d<SH, T, C, NW, S, (EX) != 0, s2d_minb(T, SH::R, C, NW)>,      \
        &launch_stream2d<SH, T, C, NW, S, (EX) != 0, s2d_minb(T, SH::R, C, NW)>               \
  }

template <class SH, int T, int CY, int CX, int NWY, int S, bool DEC, bool EXACT, int MINB>
cudaError_t launch_stream3d(const TbLaunch& L) {
  using Cfg = Stream3DCfg<SH, T, CY, CX, NWY, S, DEC>;
  auto kern = k_stream3d<SH, T, CY, CX, NWY, S, DEC, EXACT, MINB>;
  cudaError_t err =
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
  if (err != cudaSuccess) return err;
  TmapSet maps;
  memcpy(&maps.m[0], L.maps, 3 * sizeof(CUtensorMap));
  Stream3DArgs a;
  a.n0 = L.n0;
  a.n1 = L.n1;
  a.n2 = L.n2;
  a.nty = L.nty;
  a.ntx = L.ntx;
  a.nseg = L.nseg;
  a.seg_len = L.seg_len;
  a.epochs = L.epochs;
  a.first_src = L.first_src;
  a.first_dst = L.first_dst;
  for (int i = 0; i < 3; ++i) a.buf[i] = L.buf[i];
  a.work = L.work;
  Coefs<SH::NT> cf;
  for (int i = 0; i < SH::NT; ++i) cf.c[i] = L.coeffs[i];
  if (L.cooperative) {
    void* args[] = {(void*)&maps, (void*)&a, (void*)&cf};
    return cudaLaunchCooperativeKernel((const void*)kern, dim3(L.grid), dim3(NWY * 32), args,
                                       (size_t)Cfg::SMEM_BYTES, L.stream);
  }
  kern<<<L.grid, NWY * 32, Cfg::SMEM_BYTES, L.stream>>>(maps, a, cf);
  return cudaGetLastError();
}

#define EBISU_S3D_ENTRY(SHAPE_ID, SH, T, CY, CX, NWY, S, DEC, EX, MINB)                         \
  TbKernel {                                                                                  \
    SHAPE_ID, 3, T, CX, NWY, S, EX, Stream3DCfg<SH, T, CY, CX, NWY, S, DEC>::SMEM_BYTES,       \
        Stream3DCfg<SH, T, CY, CX, NWY, S, DEC>::LX, Stream3DCfg<SH, T, CY, CX, NWY, S, DEC>::LY, \
        1, Stream3DCfg<SH, T, CY, CX, NWY, S, DEC>::VX,                                        \
        Stream3DCfg<SH, T, CY, CX, NWY, S, DEC>::VY,                                           \
        (const void*)&k_stream3d<SH, T, CY, CX, NWY, S, DEC, (EX) != 0, MINB>,                \
        &launch_stream3d<SH, T, CY, CX, NWY, S, DEC, (EX) != 0, MINB>                         \
  }

}  // namespace ebisu

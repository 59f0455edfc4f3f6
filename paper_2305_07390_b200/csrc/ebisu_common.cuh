// ebisu_common.cuh -- sm_100a PTX helpers shared by the sweep kernels:
// mbarrier ring, TMA (cp.async.bulk.tensor) loads, proxy fences, and the
// exact (one rounding per op) / contracted tap accumulation.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace ebisu {

constexpr unsigned kFullMask = 0xffffffffu;

// Upper bound on axis-0 segments of one sweep (kernel-parameter table).
#define EBISU_MAX_SEGS 96

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ---- mbarrier -------------------------------------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

__device__ __forceinline__ void fence_mbarrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Plain arrival (release at CTA scope): one per participating thread.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint32_t bar_addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(bar_addr), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t a = smem_u32(bar);
  while (!mbar_try_wait(a, parity)) {
  }
}

// ---- predicated shared-memory access (no divergent branch) ----------------
__device__ __forceinline__ void st_shared_if(double* p, double v, bool pred) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q st.shared.f64 [%0], %1;\n\t}" ::"r"(
          smem_u32(p)),
      "d"(v), "r"((int)pred)
      : "memory");
}
// returns *p if pred, else dflt
__device__ __forceinline__ double ld_shared_if(const double* p, bool pred, double dflt) {
  double r = dflt;
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.shared.f64 %0, [%1];\n\t}"
      : "+d"(r)
      : "r"(smem_u32(p)), "r"((int)pred)
      : "memory");
  return r;
}

// two adjacent cells to global memory, branch free: one 16-byte store when
// both are stored, else the single one (p must be 16-byte aligned)
__device__ __forceinline__ void st_pair_if(double* p, double a, double b, bool s0, bool s1) {
  asm volatile(
      "{\n\t.reg .pred p0, p1, pb, q0, q1;\n\t"
      "setp.ne.b32 p0, %3, 0;\n\tsetp.ne.b32 p1, %4, 0;\n\t"
      "and.pred pb, p0, p1;\n\txor.pred q0, p0, pb;\n\txor.pred q1, p1, pb;\n\t"
      "@pb st.global.v2.f64 [%0], {%1, %2};\n\t"
      "@q0 st.global.f64 [%0], %1;\n\t"
      "@q1 st.global.f64 [%0+8], %2;\n\t}" ::"l"(p),
      "d"(a), "d"(b), "r"((int)s0), "r"((int)s1)
      : "memory");
}
__device__ __forceinline__ void st_pair_if(float* p, float a, float b, bool s0, bool s1) {
  asm volatile(
      "{\n\t.reg .pred p0, p1, pb, q0, q1;\n\t"
      "setp.ne.b32 p0, %3, 0;\n\tsetp.ne.b32 p1, %4, 0;\n\t"
      "and.pred pb, p0, p1;\n\txor.pred q0, p0, pb;\n\txor.pred q1, p1, pb;\n\t"
      "@pb st.global.v2.f32 [%0], {%1, %2};\n\t"
      "@q0 st.global.f32 [%0], %1;\n\t"
      "@q1 st.global.f32 [%0+4], %2;\n\t}" ::"l"(p),
      "f"(a), "f"(b), "r"((int)s0), "r"((int)s1)
      : "memory");
}

// ---- epoch dataflow flags (gpu scope) --------------------------------------
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// spin until *p >= v (the producer's release pairs with this acquire)
__device__ __forceinline__ void wait_flag_geq(const int* p, int v) {
  while (ld_acquire_gpu(p) < v) __nanosleep(64);
}

// ---- proxy fences ---------------------------------------------------------
// Generic-proxy accesses -> later async-proxy (TMA) accesses.
__device__ __forceinline__ void fence_proxy_async_shared() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}

// ---- cluster / DSMEM primitives -----------------------------------------------
__device__ __forceinline__ uint32_t cluster_ctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of `local` (a shared::cta pointer) in CTA `rank`
__device__ __forceinline__ uint32_t mapa_shared(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(local)), "r"(rank));
  return r;
}
// asynchronous remote store completing 16 bytes on the destination CTA's mbarrier
__device__ __forceinline__ void st_async_v2f64(uint32_t addr, double a, double b,
                                               uint32_t remote_bar) {
  asm volatile(
      "st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(
          addr),
      "d"(a), "d"(b), "r"(remote_bar)
      : "memory");
}
// asynchronous remote store of one double completing 8 bytes on the
// destination CTA's mbarrier
__device__ __forceinline__ void st_async_f64(uint32_t addr, double v, uint32_t remote_bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];" ::"r"(
                   addr),
               "d"(v), "r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ uint32_t cluster_nctarank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void st_cluster_u32(uint32_t addr, uint32_t v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// relaxed arrive on an mbarrier in another CTA of the cluster (a flow-control
// token: the values it releases are already consumed into registers)
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t remote_bar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(remote_bar)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n"
               ::: "memory");
}

// ---- TMA tensor loads (global -> shared, completion on an mbarrier) -------
__device__ __forceinline__ void tma_load_2d(void* smem_dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* smem_dst, const CUtensorMap* map, int32_t c0,
                                            int32_t c1, int32_t c2, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(smem_dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

// ---- element type (fp64: the reference's arithmetic; fp32: the north-star
// 1e-5 mode) ------------------------------------------------------------------
template <class E>
struct Vec2;
template <>
struct Vec2<double> {
  using type = double2;
};
template <>
struct Vec2<float> {
  using type = float2;
};
template <class E>
using vec2_t = typename Vec2<E>::type;
template <class E>
__device__ __forceinline__ vec2_t<E> make_v2(E a, E b) {
  vec2_t<E> r;
  r.x = a;
  r.y = b;
  return r;
}

template <class E>
__device__ __forceinline__ E mul_rn(E a, E b);
template <>
__device__ __forceinline__ double mul_rn<double>(double a, double b) {
  return __dmul_rn(a, b);
}
template <>
__device__ __forceinline__ float mul_rn<float>(float a, float b) {
  return __fmul_rn(a, b);
}
template <class E>
__device__ __forceinline__ E add_rn(E a, E b);
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) {
  return __dadd_rn(a, b);
}
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) {
  return __fadd_rn(a, b);
}
template <class E>
__device__ __forceinline__ E sub_rn(E a, E b);
template <>
__device__ __forceinline__ double sub_rn<double>(double a, double b) {
  return __dsub_rn(a, b);
}
template <>
__device__ __forceinline__ float sub_rn<float>(float a, float b) {
  return __fsub_rn(a, b);
}
template <class E>
__device__ __forceinline__ E fma_rn(E a, E b, E c);
template <>
__device__ __forceinline__ double fma_rn<double>(double a, double b, double c) {
  return __fma_rn(a, b, c);
}
template <>
__device__ __forceinline__ float fma_rn<float>(float a, float b, float c) {
  return __fmaf_rn(a, b, c);
}

// ---- tap accumulation -----------------------------------------------------
// EXACT: acc = c0*x0; acc = acc + ck*xk -- each op separately rounded, i.e.
// exactly numpy's `term = c * cells[sl]; acc = acc + term` (grid.py:87-92).
// Not EXACT: contracted FMA chain (tolerance mode, 1e-12 relative).
template <bool EXACT, class E>
__device__ __forceinline__ E tap_first(E c, E x) {
  return mul_rn<E>(c, x);
}
template <bool EXACT, class E>
__device__ __forceinline__ E tap_next(E acc, E c, E x) {
  if constexpr (EXACT) {
    return add_rn<E>(acc, mul_rn<E>(c, x));
  } else {
    return fma_rn<E>(c, x, acc);
  }
}

// Coefficients travel in the kernel parameter space (constant bank), so the
// multiply operands come straight from c[0x0][...] without occupying
// registers.  fp32 kernels get the coefficients rounded to float once.
template <int NT, class E = double>
struct Coefs {
  E c[NT];
};

struct alignas(64) TmapSet {
  CUtensorMap m[3];  // [0] = input, [1] = output, [2] = scratch
};

enum BufId : int { BUF_IN = 0, BUF_OUT = 1, BUF_SCR = 2 };

}  // namespace ebisu

// nesa_ptx.cuh -- sm_100a PTX helpers: mbarrier, bulk async copy (TMA bulk
// engine, SASS UBLKCP), cp.async with mbarrier completion, named barriers.
#pragma once
#include <cstdint>

namespace nesa {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count)
               : "memory");
}

// Make barrier initialisation visible to the async proxy (bulk copies).
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(
                   smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}

// Bulk global -> shared copy completing on an mbarrier (tx bytes).
// src, dst and bytes must be 16-byte aligned / multiples of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, "
      "[%3];" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// L2 policy: evict-first (streamed-once operator data must not displace the
// far-field working set from L2).
__device__ __forceinline__ uint64_t l2_evict_first_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint64_t l2_evict_last_policy() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// 16-byte global store / load with an L2 cache-policy hint.
__device__ __forceinline__ void st16_hint(void* p, float4 v, uint64_t pol) {
  asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(p), "f"(v.x),
               "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
               : "memory");
}
__device__ __forceinline__ float4 ld16_hint(const void* p, uint64_t pol) {
  float4 v;
  asm volatile("ld.global.L2::cache_hint.v4.f32 {%0, %1, %2, %3}, [%4], %5;"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p), "l"(pol));
  return v;
}

// Bulk global -> shared copy with an L2 cache hint.
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
      "[%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// Ampere-style async copies of 4/8/16 bytes (LDGSTS).
template <int BYTES>
__device__ __forceinline__ void cp_async(void* dst, const void* src) {
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
                 : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "n"(BYTES)
                 : "memory");
  }
}

// Copy of BYTES (4, 8 or a multiple of 16) as one or more cp.async.
template <int BYTES>
__device__ __forceinline__ void cp_async_n(void* dst, const void* src) {
  if constexpr (BYTES <= 16) {
    cp_async<BYTES>(dst, src);
  } else {
    static_assert(BYTES % 16 == 0, "cp.async size");
#pragma unroll
    for (int i = 0; i < BYTES / 16; ++i)
      cp_async<16>(static_cast<char*>(dst) + 16 * i, static_cast<const char*>(src) + 16 * i);
  }
}

// cp.async of BYTES (4, 8, 16) that writes zeros instead when !valid.
template <int BYTES>
__device__ __forceinline__ void cp_async_zfill(void* dst, const void* src, bool valid) {
  const int n = valid ? BYTES : 0;
  if constexpr (BYTES == 16) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
                 "r"(n)
                 : "memory");
  } else {
    asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;" ::"r"(smem_u32(dst)), "l"(src),
                 "n"(BYTES), "r"(n)
                 : "memory");
  }
}

template <int BYTES>
__device__ __forceinline__ void cp_async_zfill_n(void* dst, const void* src, bool valid) {
  if constexpr (BYTES <= 16) {
    cp_async_zfill<BYTES>(dst, src, valid);
  } else {
#pragma unroll
    for (int i = 0; i < BYTES / 16; ++i)
      cp_async_zfill<16>(static_cast<char*>(dst) + 16 * i, static_cast<const char*>(src) + 16 * i,
                         valid);
  }
}

__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;" ::: "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

// Arrive on `bar` once all prior cp.async of this thread have landed.  The
// barrier's expected count must include this arrival (.noinc).
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

// Programmatic dependent launch: wait for the previous grid in the stream
// (no-op when launched without the attribute) / let the next one launch.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

// Paired FP32 FMA (Blackwell FFMA2): (c.x, c.y) += a * (x.x, x.y), each lane
// rounded exactly like fmaf, so results are bitwise those of two FFMAs.
__device__ __forceinline__ void ffma2(float& c0, float& c1, float a, float x0, float x1) {
  unsigned long long c, x, aa;
  asm("mov.b64 %0, {%1, %2};" : "=l"(c) : "f"(c0), "f"(c1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(x0), "f"(x1));
  asm("mov.b64 %0, {%1, %1};" : "=l"(aa) : "f"(a));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(c) : "l"(aa), "l"(x));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(c0), "=f"(c1) : "l"(c));
}
// elementwise a * b + c and a * b on float2 pairs (FFMA2 / FMUL2)
__device__ __forceinline__ float2 ffma2v(float2 a, float2 b, float2 c) {
  unsigned long long pa, pb, pc;
  asm("mov.b64 %0, {%1, %2};" : "=l"(pa) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(pb) : "f"(b.x), "f"(b.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(pc) : "f"(c.x), "f"(c.y));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(pc) : "l"(pa), "l"(pb));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(pc));
  return r;
}
__device__ __forceinline__ float2 fmul2v(float2 a, float2 b) {
  unsigned long long pa, pb, pc;
  asm("mov.b64 %0, {%1, %2};" : "=l"(pa) : "f"(a.x), "f"(a.y));
  asm("mov.b64 %0, {%1, %2};" : "=l"(pb) : "f"(b.x), "f"(b.y));
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(pc) : "l"(pa), "l"(pb));
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(pc));
  return r;
}
// complex z * w with the loop-invariant pairs W1 = (w.x, w.y), W2 = (-w.y, w.x):
// z.x W1 + z.y W2 (one FMUL2 + one FFMA2)
__device__ __forceinline__ float2 cmul_pk(float2 z, float2 W1, float2 W2) {
  return ffma2v(make_float2(z.y, z.y), W2, fmul2v(make_float2(z.x, z.x), W1));
}

// 8 x 4 register tile: acc[r][c] += m[r] x[c] (float: column pairs share one FFMA2)
template <typename T>
__device__ __forceinline__ void tile_fma8x4(T (&acc)[8][4], const T (&m0)[4], const T (&m1)[4],
                                            const T (&x)[4]) {
  if constexpr (sizeof(T) == 4) {
#pragma unroll
    for (int c = 0; c < 4; c += 2)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        ffma2(reinterpret_cast<float&>(acc[r][c]), reinterpret_cast<float&>(acc[r][c + 1]), float(m0[r]),
              float(x[c]), float(x[c + 1]));
        ffma2(reinterpret_cast<float&>(acc[r + 4][c]), reinterpret_cast<float&>(acc[r + 4][c + 1]),
              float(m1[r]), float(x[c]), float(x[c + 1]));
      }
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c)
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        acc[r][c] = fma(m0[r], x[c], acc[r][c]);
        acc[r + 4][c] = fma(m1[r], x[c], acc[r + 4][c]);
      }
  }
}

// acc[rr] += a * x[rr] for rr < R (float: paired FMAs; double: scalar)
template <typename T, int R>
__device__ __forceinline__ void fma_row(T (&acc)[R], T a, const T (&x)[R]) {
  if constexpr (sizeof(T) == 4 && R % 2 == 0) {
#pragma unroll
    for (int rr = 0; rr < R; rr += 2)
      ffma2(reinterpret_cast<float&>(acc[rr]), reinterpret_cast<float&>(acc[rr + 1]), float(a),
            float(x[rr]), float(x[rr + 1]));
  } else {
#pragma unroll
    for (int rr = 0; rr < R; ++rr) acc[rr] = fma(a, x[rr], acc[rr]);
  }
}

}  // namespace nesa

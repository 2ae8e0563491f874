// device.cuh — sm_100a device helpers shared by the tq kernels:
// int128 arithmetic, LSB-first bitmaps, the engine hashes (fnv1a64 of
// reference common.hpp:128-136, SplitMix64 of common.hpp:139-158), and the
// TMA bulk-copy / mbarrier primitives used to stage column tiles in smem.
#pragma once
#ifndef __CUDACC_RTC__
#include <cstdint>
#include <cuda_runtime.h>
#endif
#include "program_types.h"  // RTC builds: fixed-width integer typedefs

namespace tq {

using i128 = __int128;
using u128 = unsigned __int128;
using u64 = unsigned long long;
using u32 = unsigned int;

constexpr u32 kFull = 0xffffffffu;

// ------------------------------------------------------------------ int128
__device__ __forceinline__ i128 mk128(u64 lo, u64 hi) { return (i128)(((u128)hi << 64) | (u128)lo); }
__device__ __forceinline__ u64 lo64(i128 v) { return (u64)(u128)v; }
__device__ __forceinline__ u64 hi64(i128 v) { return (u64)((u128)v >> 64); }
__device__ __forceinline__ bool fits64(i128 v) { return hi64(v) == (u64)((long long)lo64(v) >> 63); }

// Wrapping 128-bit multiply with a 64x64->128 fast path (decimal(11,2)
// operands and their products almost always fit).
__device__ __forceinline__ bool fits32(i128 v) {
  const long long l = (long long)lo64(v);
  return hi64(v) == (u64)(l >> 63) && l == (long long)(int)l;
}
__device__ __forceinline__ i128 mul128(i128 a, i128 b) {
  if (fits32(a) && fits32(b)) return (i128)((long long)(int)lo64(a) * (long long)(int)lo64(b));
  if (fits64(a) && fits64(b)) {
    long long x = (long long)lo64(a), y = (long long)lo64(b);
    u64 lo = (u64)x * (u64)y;
    u64 hi = (u64)__mul64hi(x, y);
    return mk128(lo, hi);
  }
  return (i128)((u128)a * (u128)b);
}
__device__ __forceinline__ i128 add128(i128 a, i128 b) { return (i128)((u128)a + (u128)b); }
__device__ __forceinline__ i128 sub128(i128 a, i128 b) { return (i128)((u128)a - (u128)b); }
__device__ __forceinline__ i128 wrap64(i128 v) { return (i128)(long long)lo64(v); }

__device__ __forceinline__ double i128_to_f64(i128 v) {
  if (fits64(v)) return (double)(long long)lo64(v);
  return (double)v;
}

__device__ __forceinline__ i128 shfl_xor_i128(i128 v, int m) {
  u64 lo = __shfl_xor_sync(kFull, lo64(v), m);
  u64 hi = __shfl_xor_sync(kFull, hi64(v), m);
  return mk128(lo, hi);
}
__device__ __forceinline__ i128 warp_sum_i128(i128 v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v = add128(v, shfl_xor_i128(v, m));
  return v;
}
__device__ __forceinline__ double warp_sum_f64(double v) {
#pragma unroll
  for (int m = 16; m > 0; m >>= 1) v += __shfl_xor_sync(kFull, v, m);
  return v;
}

// Exact int128 accumulation with two 64-bit atomics (carry propagated):
// sum mod 2^128 is order independent, so results are bit-exact.
__device__ __forceinline__ void atomic_add_i128(u64* p, i128 v) {
  u64 lo = lo64(v), hi = hi64(v);
  u64 old = atomicAdd(&p[0], lo);
  u64 carry = (old + lo) < old ? 1ull : 0ull;
  u64 h = hi + carry;
  if (h) atomicAdd(&p[1], h);
}
__device__ __forceinline__ void atomic_minmax_i128(u128* p, i128 v, bool is_min) {
  u128 cur = *(volatile u128*)p;
  for (;;) {
    i128 c = (i128)cur;
    bool better = is_min ? (v < c) : (v > c);
    if (!better) return;
    u128 prev = atomicCAS(p, cur, (u128)v);
    if (prev == cur) return;
    cur = prev;
  }
}
__device__ __forceinline__ void atomic_minmax_f64(double* p, double v, bool is_min) {
  u64* q = (u64*)p;
  u64 cur = *(volatile u64*)q;
  for (;;) {
    double c = __longlong_as_double((long long)cur);
    bool better = is_min ? (v < c) : (v > c);
    if (!better) return;
    u64 prev = atomicCAS(q, cur, (u64)__double_as_longlong(v));
    if (prev == cur) return;
    cur = prev;
  }
}

// ------------------------------------------------------------------ bitmaps
__device__ __forceinline__ bool bm_get(const uint8_t* bm, u64 i) { return (bm[i >> 3] >> (i & 7)) & 1; }
__device__ __forceinline__ void bm_set_atomic(uint8_t* bm, u64 i) {
  // byte-address -> containing aligned 32-bit word
  uintptr_t a = (uintptr_t)(bm + (i >> 3));
  u32* w = (u32*)(a & ~(uintptr_t)3);
  u32 bit = (u32)((a & 3) * 8 + (i & 7));
  atomicOr(w, 1u << bit);
}

// ------------------------------------------------------------------ hashes
constexpr u64 kFnvBasis = 0xcbf29ce484222325ull;
constexpr u64 kFnvPrime = 0x100000001b3ull;
__device__ __forceinline__ u64 fnv_bytes(u64 h, u64 v, int nbytes) {
#pragma unroll 8
  for (int i = 0; i < nbytes; ++i) {
    h ^= (v >> (8 * i)) & 0xff;
    h *= kFnvPrime;
  }
  return h;
}
__host__ __device__ __forceinline__ u64 sm_mix(u64 z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
constexpr u64 kGamma = 0x9e3779b97f4a7c15ull;
// k-th output of SplitMix64(seed).next(), k >= 1 (counter-based form).
__host__ __device__ __forceinline__ u64 sm_nth(u64 seed, u64 k) { return sm_mix(seed + k * kGamma); }
// Internal table hash (join / group tables); NOT the partition hash.
// Multiplicative (Fibonacci) mixing per word, high bits folded down so the
// low bits used as the slot index see every key bit.
__device__ __forceinline__ u64 key_hash(const u64* w, int n) {
  u64 h = 0x12345678abcdefull;
#pragma unroll
  for (int i = 0; i < n; ++i) h = (h ^ w[i]) * kGamma;
  return h ^ (h >> 29) ^ (h >> 47);
}

// Blocked Bloom filter: 3 bits in one 32-bit word chosen by the high hash bits.
__device__ __forceinline__ u32 bloom_bits(u64 h) {
  return (1u << (h & 31)) | (1u << ((h >> 5) & 31)) | (1u << ((h >> 10) & 31));
}
__device__ __forceinline__ u64 bloom_word(u64 h, u64 mask) { return (h >> 32) & mask; }

// fnv1a64 mod 2^32 == 32-bit FNV-1a with basis 0x84222325 / prime 0x1b3
// (low words of the 64-bit constants): exact for power-of-two part counts.
__device__ __forceinline__ u32 fnv32_bytes(u32 h, u64 v, int nbytes) {
#pragma unroll 8
  for (int i = 0; i < nbytes; ++i) {
    h ^= (u32)(v >> (8 * i)) & 0xffu;
    h *= 0x1b3u;
  }
  return h;
}

// ------------------------------------------------------------------ mbarrier + TMA bulk copy
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, u32 count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, u32 bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint64_t* bar, u32 parity) {
  u32 ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, u32 parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// 1-D bulk async copy global -> shared, completion counted on `bar` (bytes).
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Same, with an L2 cache policy (streamed column tiles: evict_first, so
// hash tables and Bloom filters the kernel probes stay resident in L2).
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, u32 bytes, uint64_t* bar, u64 policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
__device__ __forceinline__ u64 l2_policy_evict_first() {
  u64 pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

// Bulk prefetch global -> L2 (no shared memory, no completion tracking).
__device__ __forceinline__ void bulk_prefetch_l2(const void* src, u32 bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}

// Acquire loads of a publication word (GPU scope, global / CTA scope, shared).
__device__ __forceinline__ u32 ld_acquire_gpu(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ u32 ld_acquire_cta_shared(const u32* p) {
  u32 v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}

__device__ __forceinline__ u32 lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ u32 lanemask_lt() {
  u32 m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

}  // namespace tq

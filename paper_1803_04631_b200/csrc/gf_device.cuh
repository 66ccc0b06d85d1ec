// gf_device.cuh -- device helpers: Philox4x32-10, warp scans, bitonic sort.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace gf {

constexpr unsigned kFull = 0xffffffffu;

// Philox4x32-10 (Salmon et al., SC'11; Random123 constants).  The oracle
// restates the same function (oracle/gf_oracle.c gfo_philox4x32_10) and the
// Random123 known-answer vectors pin both.
__device__ __forceinline__ uint4 philox4x32_10(uint4 c, uint2 k) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) { k.x += 0x9E3779B9u; k.y += 0xBB67AE85u; }
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = make_uint4(hi1 ^ c.y ^ k.x, lo1, hi0 ^ c.w ^ k.y, lo0);
    }
    return c;
}

// top 24 bits -> float in [0, 1), exact
__device__ __forceinline__ float u24(uint32_t r) { return __uint2float_rn(r >> 8) * 5.9604644775390625e-08f; }

__device__ __forceinline__ float warp_incl_scan(float x, int lane) {
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        float y = __shfl_up_sync(kFull, x, o);
        if (lane >= o) x = __fadd_rn(x, y);
    }
    return x;
}

__device__ __forceinline__ uint32_t warp_max_u32(uint32_t x) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(kFull, x, o));
    return x;
}

// ascending bitonic sort of one key per lane
__device__ __forceinline__ uint32_t warp_bitonic_sort(uint32_t key, int lane) {
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            uint32_t p = __shfl_xor_sync(kFull, key, j);
            bool up = (lane & k) == 0;
            bool lower = (lane & j) == 0;
            key = (lower == up) ? min(key, p) : max(key, p);
        }
    }
    return key;
}

// Transposed topic layout of K1's shared-memory p* table: topic t lives in
// float slot tpos(t) = (t % m) * 32 + t / m, m = ceil(K / 32), i.e. its bank
// is t / m (the topic's high bits).  A theta row is sorted by topic, so the
// lanes of one gather (entries 8 apart in the row) hit distinct banks; with
// the natural layout (bank = t % 32) they collide like random addresses.
// Theta entries store tpos(t) << 2 (a byte offset) in their low 16 bits.
// t / m is a multiply-high by magic = ceil(2^32 / m): exact for t, m < 2^16.
struct TPos {
    uint32_t m, magic;
};
__host__ __device__ inline uint32_t tpos_m(int K) { return (uint32_t)(K + 31) / 32u; }
__host__ __device__ inline uint32_t tpos_slots(int K) { return 32u * tpos_m(K); }
__host__ __device__ inline TPos tpos_geom(int K) {
    TPos g;
    g.m = tpos_m(K);
    g.magic = g.m > 1 ? (uint32_t)((0x100000000ULL + g.m - 1) / g.m) : 0u;
    return g;
}
__device__ __forceinline__ uint32_t tpos(uint32_t t, TPos g) {
    const uint32_t q = g.m > 1 ? __umulhi(t, g.magic) : t;
    return (t - q * g.m) * 32u + q;
}
__device__ __forceinline__ uint32_t tpos_inv(uint32_t p, TPos g) { return (p & 31u) * g.m + (p >> 5); }

__device__ __forceinline__ float prev_float(float x) { return __int_as_float(__float_as_int(x) - 1); }

// system-scope signalling between the GPUs of one node (peer-mapped memory)
__device__ __forceinline__ void st_release_sys(uint32_t* p, uint32_t v) {
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ unsigned long long now_ns() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// TMA bulk prefetch of [p, p + bytes) into L2 (16-byte aligned, bytes % 16 == 0)
__device__ __forceinline__ void prefetch_l2_bulk(const void* p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

// Shared-memory accesses on 32-bit shared-window addresses.  Through a
// generic pointer (e.g. a per-warp slice of an extern __shared__ array used
// with atomicAdd) the compiler re-derives the CTA's shared window at every
// access (S2UR SR_CgaCtaId + 4 uniform ops + LEA: ~6 extra issue slots per
// atomic, measured in K3's SASS); with the address converted once these are
// one LEA + the ATOMS / LDS.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void sh_red_add(uint32_t a, uint32_t v) {
    asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void sh_red_or(uint32_t a, uint32_t v) {
    asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t sh_exch(uint32_t a, uint32_t v) {
    uint32_t r;
    asm volatile("atom.shared.exch.b32 %0, [%1], %2;" : "=r"(r) : "r"(a), "r"(v) : "memory");
    return r;
}
__device__ __forceinline__ uint32_t sh_ld(uint32_t a) {
    uint32_t r;
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a) : "memory");
    return r;
}
__device__ __forceinline__ void sh_st(uint32_t a, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

// One-shot TMA bulk copy global -> this CTA's shared memory (16-byte
// aligned, bytes % 16 == 0) completing on an mbarrier: thread 0 arms the
// barrier and issues the copy, every thread waits on phase 0.  The caller
// passes a fresh __shared__ 8-byte barrier and synchronises the block between
// bulk_copy_issue and bulk_copy_wait (the barrier's init must be visible).
__device__ __forceinline__ void bulk_copy_issue(uint32_t bar, uint32_t dst, const void* src, uint32_t bytes) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(dst), "l"(src), "r"(bytes), "r"(bar) : "memory");
}
__device__ __forceinline__ void bulk_copy_wait(uint32_t bar) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        "WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
        " @!p bra WAIT_%=;\n"
        "}\n" ::"r"(bar)
        : "memory");
}

// Per-thread L2 prefetch of the 128-byte line holding p (no uniform operands:
// cp.async.bulk.prefetch takes its address and size in uniform registers, so
// with a different address in every lane the compiler serialises it into a
// 32-iteration loop per warp -- measured 13% of K1's instructions)
__device__ __forceinline__ void prefetch_l2_line(const void* p) {
    asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}

}  // namespace gf

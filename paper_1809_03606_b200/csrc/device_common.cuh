// device_common.cuh — device primitives shared by the stack (decode.cu) and
// list (list.cu) decoder kernels: min-sum f, exact g, HD helpers, the in-place
// BETA op on the flat beta, the re-encoding transform and warp key reductions.
// Product code only (the oracle has its own, independent implementation).
#pragma once
#include <cuda_runtime.h>

#include "internal.h"

#ifdef POLAR_DEBUG
#include <cassert>
#define POLAR_DCHECK(c) assert(c)
#else
#define POLAR_DCHECK(c) ((void)0)
#endif

namespace polar {

constexpr uint32_t FULL = 0xFFFFFFFFu;

// Eq. (1): sign(a) sign(b) min(|a|,|b|).  The sign is taken from
// the sign bits, so it differs from a comparison-based sign only when an input
// is -0, i.e. when the result is a zero: HD, |.|, the PM sums and every later
// f/g see +0 and -0 alike (reading R2), so bits, PMs and counts are unchanged.
// The sign is taken from the product a*b (IEEE: its sign bit is the XOR of the
// operands' sign bits, zeros and underflow included), so the sign costs one
// FMA-pipe multiply and the merge one logic op instead of two logic ops.  A
// NaN product needs inf * 0, and then m = 0: only a zero's sign can differ.
__device__ __forceinline__ float f_minsum(float a, float b) {
    const float m = fminf(fabsf(a), fabsf(b));
    const float p = __fmul_rn(a, b);
    return __uint_as_float(__float_as_uint(m) | (__float_as_uint(p) & 0x80000000u));
}
// corrected Eq. (2): g = a_hi + (1 - 2 beta) a_lo (reading R1); a_hi - a_lo is
// a_hi + (-a_lo) exactly, so flipping the sign bit of a_lo is exact.
__device__ __forceinline__ float g_exact(float lo, float hi, uint32_t bit) {
    return hi + __uint_as_float(__float_as_uint(lo) ^ (bit << 31));
}
__device__ __forceinline__ float negpart(float x) { return x < 0.f ? -x : 0.f; }
__device__ __forceinline__ float pospart(float x) { return x < 0.f ? 0.f : x; }

// BETA(lam, phi): beta[(phi-1)Lam + i] ^= beta[phi Lam + i] (Fig. 7d)
__device__ __forceinline__ void beta_op(uint32_t *beta, int lam, int phi, int lane) {
    const int Lam = 1 << lam;
    if (Lam >= 32) {
        const int wd = ((phi - 1) * Lam) >> 5, ws = (phi * Lam) >> 5, nwd = Lam >> 5;
        #pragma unroll 1
        for (int t_0 = 0; t_0 < (nwd); t_0 += 32) if (const int t = t_0 + lane; t < (nwd)) beta[wd + t] ^= beta[ws + t];
    } else if (lane == 0) {
        const int p = (phi - 1) * Lam;             // 2*Lam bits inside one word
        const int w = p >> 5, o = p & 31;
        const uint32_t x = beta[w];
        const uint32_t r = (x >> (o + Lam)) & ((1u << Lam) - 1u);
        beta[w] = x ^ (r << o);
    }
    __syncwarp();
}

// The same BETA op on a flat beta held in registers, word w in lane w
// (N <= 1024): whole words move by one shuffle, a sub-word level is one RMW in
// the owning lane
__device__ __forceinline__ void beta_op_reg(uint32_t &bw, int lam, int phi, int lane) {
    const int Lam = 1 << lam;
    if (Lam >= 32) {
        const int wd = ((phi - 1) * Lam) >> 5, nwd = Lam >> 5;
        const uint32_t x = __shfl_down_sync(FULL, bw, nwd);
        if (lane >= wd && lane < wd + nwd) bw ^= x;
    } else {
        const int p = (phi - 1) * Lam;             // 2*Lam bits inside one word
        const uint32_t r = (bw >> ((p & 31) + Lam)) & ((1u << Lam) - 1u);
        if (lane == (p >> 5)) bw ^= r << (p & 31);
    }
}

// u <- x F^{(x)n} on nw bit-packed words: the re-encoding of
// the root beta that gives u_hat in non-systematic mode
__device__ __forceinline__ void xform_words(uint32_t *w, int N, int nw, int lane) {
    const uint32_t masks[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
    #pragma unroll 1
    for (int j_0 = 0; j_0 < (nw); j_0 += 32) if (const int j = j_0 + lane; j < (nw)) {
        uint32_t x = w[j];
#pragma unroll
        for (int s = 0; s < 5; s++)
            if ((1 << s) < N) x ^= (x >> (1 << s)) & masks[s];
        w[j] = x;
    }
    __syncwarp();
    #pragma unroll 1
    for (int H = 1; H < nw; H <<= 1) {
        #pragma unroll 1
        for (int j_0 = 0; j_0 < (nw); j_0 += 32) if (const int j = j_0 + lane; j < (nw))
            if ((j & H) == 0) w[j] ^= w[j + H];
        __syncwarp();
    }
}

// Warp minimum of 64-bit keys (hi, lo) with unique lo among equal hi.
__device__ __forceinline__ void warp_min_key(uint32_t hi, uint32_t lo, uint32_t &mh, uint32_t &ml) {
    mh = __reduce_min_sync(FULL, hi);
    ml = __reduce_min_sync(FULL, hi == mh ? lo : 0xFFFFFFFFu);
}

__device__ __forceinline__ void top4_insert(unsigned long long key, unsigned long long &t0, unsigned long long &t1,
                                            unsigned long long &t2, unsigned long long &t3) {
    if (key < t3) {
        if (key < t2) {
            t3 = t2;
            if (key < t1) {
                t2 = t1;
                if (key < t0) { t1 = t0; t0 = key; } else t1 = key;
            } else t2 = key;
        } else t3 = key;
    }
}
__device__ __forceinline__ int bitlen(uint32_t x) { return 32 - __clz(x); }

// ---- streaming host pipeline (capi.cu, decode_host_stream): one launch over a
// batch whose LLR rows are still being copied in.  Chunk i (2^shift frames) may
// be read once ready[i] != 0, a flag written by a stream memory operation that
// follows the chunk's H2D copy on the copy stream.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t *p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Whole warp (every lane reads the flag; the loop condition is a warp
// reduction, so the wait keeps the warp provably converged — a lane-0 spin
// here made ptxas treat the whole decode loop as divergent).  A flag that
// never arrives (a failed copy) sets *err after about 2^26 sleeps of
// >= 256 ns (> 17 s) and lets the frame through, so the launch ends and the
// host reports it.  Once *err is set (by that timeout, or by the host
// releasing the launch after a failed copy) every later wait of the launch
// returns at once: a stalled batch costs one timeout, not one per frame.
__device__ __forceinline__ void wait_chunk_ready(const uint32_t *ready, uint32_t *err, unsigned long long f, int shift) {
    const uint32_t *fl = ready + (f >> shift);
    #pragma unroll 1
    for (uint32_t t = 0; !__reduce_or_sync(FULL, ld_acquire_u32(fl)); t++) {
        if (__reduce_or_sync(FULL, ld_acquire_u32(err))) return;
        if (t >> 26) {
            if ((threadIdx.x & 31) == 0) atomicExch(err, 1u);
            return;
        }
        __nanosleep(256);
    }
}

}  // namespace polar

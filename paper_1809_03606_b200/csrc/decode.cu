// decode.cu — the FSSCS-RM decode kernel for sm_100a.
//
// One warp decodes one frame at a time; a persistent grid pulls frames from a
// global queue so early-terminating frames free their warp.  Per warp, shared
// memory holds the channel LLRs (alpha_n), the single alpha memory (stage
// lambda = Lambda floats), the flat N-bit beta
// and the per-length counters.  The path-metric stack lives in
// registers: lane l owns entries l, l+32, ... (SLOTS = ceil(D/32) per lane) and
// selection / replacement use warp reductions (REDUX) — the paper's linear
// search done as a 32-wide parallel search.  Each stack entry
// references a snapshot slot holding the beta prefix of its fork plus a flip
// descriptor (paths store beta, not u_hat), so a path switch
// restores beta without repopulation and recomputes the alpha spine from the
// root (Alg. 4).
//
// Arithmetic is float32 with the operation order of the oracle (reading R3):
// f/g per Eq. (1) and corrected Eq. (2) (reading R1), tree-order sums, argmin
// keys (|alpha| bits, index), candidates sorted by (dPM, mask), stack order
// (PM, serial).  Built with -fmad=false; no fast-math.
#include <cuda_runtime.h>
#ifdef POLAR_TRACE_FRAME
#include <cstdio>
#endif

#include "device_common.cuh"

namespace polar {

#ifndef POLAR_BETA_REGS
#define POLAR_BETA_REGS 1      // 0: the flat beta in shared memory in every kernel (A/B builds).  Two or four
                               // words per lane for n = 11 / 12 measured slower (C4 2260 -> 2012, C5 2868 -> 2395)
#endif
#ifndef POLAR_UNR_BIG
#define POLAR_UNR_BIG 1        // the N = 2048 kernel unrolls the float4 stage loop too (C4 2203 -> 2263 Mbps; N = 4096: 2868 -> 2525, not done)
#endif
#ifndef POLAR_MERGE_FAST
#define POLAR_MERGE_FAST 0     // register stacks: the all-candidates-first merge as a shift (measured slower:
                               // C2 6702 -> 6654, C4 2264 -> 2203, C5 2872 -> 2822 Mbps)
#endif
#ifndef POLAR_MERGE_FAST_HOT
#define POLAR_MERGE_FAST_HOT 1 // the same for the D > 128 window (P 2838 -> 2870)
#endif
#ifndef POLAR_SNAP_SOFT
#define POLAR_SNAP_SOFT 32     // snapshot slots above this trigger an exact recount (lazy bitmaps); 1 << 30: never
#endif
#ifndef POLAR_CONST_AW
#define POLAR_CONST_AW 1       // specialised kernels: the alpha area's size as a compile-time constant
#endif
#ifndef POLAR_LEAN_WATCHDOG
#define POLAR_LEAN_WATCHDOG 1  // specialised (MODE >= 1) kernels: no pop-count watchdog
#endif
#ifndef POLAR_PREFETCH_SNAP
#define POLAR_PREFETCH_SNAP 0  // register beta: the switch's snapshot load issued right after the pop (measured slower: C2 6931 -> 6908, P 3012 -> 2965)
#endif
#ifndef POLAR_NOSER
#define POLAR_NOSER 0          // sorted register stacks without serial words: the order is the position
                               // (candidates carry the largest serials, so they follow equal PMs), the working
                               // path is a flag bit in its entry's jsm word.  Measured: C2 6942 -> 6956, C5 3117
                               // -> 3156, C4 2326 -> 2290 Mbps; with POLAR_R0_FAST ptxas no longer proves the
                               // CRC kernels' decode loop converged (C3 6490 -> 5956): not taken
#endif
// The next three: 0 off, 1 in the kernels where measured faster, 2 in every kernel (A/B and test builds)
#ifndef POLAR_R0_FAST
#define POLAR_R0_FAST 1        // sorted register stacks: an R0 node's single candidate inserted by one shift
                               // (n = 10, 11 kernels: C2 6937 -> 7113, C3 6480 -> 6661, C4 2326 -> 2394 Mbps with
                               // POLAR_SUM_FULL; n = 12: C5 3122 -> 3052, n = 7: C1 -12%: left off there)
#endif
#ifndef POLAR_REP_FAST
#define POLAR_REP_FAST 1       // the same for a REP node's two warp-uniform candidates (n = 10 kernels: C2 7125
                               // -> 7197; n = 11: C4 2394 -> 2338, n = 12: C5 3052 -> 2497: left off there)
#endif
#ifndef POLAR_SUM_FULL
#define POLAR_SUM_FULL 1       // R0 / REP nodes with Lambda <= 32: the full five-level shuffle tree, unrolled
                               // (n = 10, 11 kernels; C2 alone 6942 -> 6975)
#endif
#ifndef POLAR_BWPL
#define POLAR_BWPL 1           // register stages below 5 read the left sibling's beta from one shuffled word
#endif
#ifndef POLAR_SORTED_STACK
#define POLAR_SORTED_STACK 2   // 2: every register stack sorted; 1: D <= 32 only; 0: none (A/B builds)
#endif

constexpr uint32_t EMPTY = 0xFFFFFFFFu;
constexpr uint32_t NO_SNAP = 0xFFFFu;

// ALPHA(s, psi): alpha_s from alpha_{s+1} (Eq. 4, Alg. 1) for stages s >= 6
// (Lambda >= 64) held in shared memory at alpha[2^s, 2^{s+1}).  Stage n is the
// channel row: shared memory (CHAN_SMEM) or the LLR input read through L1/L2
// with coherent loads (never the non-coherent path: the streaming host
// pipeline lands rows while the kernel runs, ordered by the chunk flags).
template <bool CHAN_SMEM>
__device__ __forceinline__ float4 ld4(const float *p, bool) {
    return *reinterpret_cast<const float4 *>(p);
}
template <bool CHAN_SMEM>
__device__ __forceinline__ float ld1(const float *p, bool) {
    return *p;
}

// src: stage s+1 (or the channel row when s+1 == n); dst: stage s.  UNR:
// unroll the float4 loop (independent iterations; measured on n = 10 only).
// BR: the flat beta is held in registers, word w in lane w (bw), not in beta[]
template <bool CHAN_SMEM, bool UNR = false, bool BR = false>
__device__ __forceinline__ void alpha_stage(const float *src, float *dst, const uint32_t *beta, uint32_t bw,
                                            int n, int s, int psi, int lane) {
    const int Ls = 1 << s;
    const bool top = (s + 1 == n);
    const bool odd = (psi & 1) != 0;
    const int boff = (psi - 1) << s;                 // left sibling's segment of the flat beta
    if (Ls == 64) {
        // two elements per lane: lane and lane + 32
        const float lo0 = ld1<CHAN_SMEM>(src + lane, top), lo1 = ld1<CHAN_SMEM>(src + 32 + lane, top);
        const float hi0 = ld1<CHAN_SMEM>(src + 64 + lane, top), hi1 = ld1<CHAN_SMEM>(src + 96 + lane, top);
        if (odd) {
            const uint32_t w0 = BR ? __shfl_sync(FULL, bw, boff >> 5) : beta[boff >> 5];
            const uint32_t w1 = BR ? __shfl_sync(FULL, bw, (boff >> 5) + 1) : beta[(boff >> 5) + 1];
            dst[lane] = g_exact(lo0, hi0, (w0 >> lane) & 1u);
            dst[32 + lane] = g_exact(lo1, hi1, (w1 >> lane) & 1u);
        } else {
            dst[lane] = f_minsum(lo0, hi0);
            dst[32 + lane] = f_minsum(lo1, hi1);
        }
    } else {
        auto chunk = [&](int i) {
            const float4 lo = ld4<CHAN_SMEM>(src + i, top);
            const float4 hi = ld4<CHAN_SMEM>(src + Ls + i, top);
            float4 o;
            if (odd) {
                const uint32_t b = (BR ? __shfl_sync(FULL, bw, (boff + i) >> 5) : beta[(boff + i) >> 5]) >> ((boff + i) & 31);
                o.x = g_exact(lo.x, hi.x, b & 1); o.y = g_exact(lo.y, hi.y, (b >> 1) & 1);
                o.z = g_exact(lo.z, hi.z, (b >> 2) & 1); o.w = g_exact(lo.w, hi.w, (b >> 3) & 1);
            } else {
                o.x = f_minsum(lo.x, hi.x); o.y = f_minsum(lo.y, hi.y);
                o.z = f_minsum(lo.z, hi.z); o.w = f_minsum(lo.w, hi.w);
            }
            *reinterpret_cast<float4 *>(dst + i) = o;
        };
        // Ls >= 128: every lane runs Ls / 128 chunks.  With the register beta
        // (shuffles inside) the loop is written uniform so the warp stays
        // provably converged; the shared-memory form keeps the lane-strided loop
        // (measured faster there)
        if constexpr (BR && UNR) {
            #pragma unroll 4
            for (int k = 0; k < (Ls >> 7); k++) chunk(lane * 4 + (k << 7));
        } else if constexpr (BR) {
            #pragma unroll 1
            for (int k = 0; k < (Ls >> 7); k++) chunk(lane * 4 + (k << 7));
        } else if constexpr (UNR) {
            #pragma unroll 4
            for (int i = lane * 4; i < Ls; i += 128) chunk(i);
        } else {
            #pragma unroll 1
            for (int i = lane * 4; i < Ls; i += 128) chunk(i);
        }
    }
    __syncwarp();
}

// Stack entry packing: jsm = j (13 bits: decision-node ordinal = schedule
// progress) | snapshot slot << 13 | flip mask relative to the
// snapshot (4 bits).  Register stacks (D <= 128): 8-bit slot (0xFF none), mask
// at bit 21.  Global stacks (D > 128): 14-bit slot (0x3FFF none), mask at 27.
template <bool BIG>
struct Pk {
    static constexpr uint32_t NONE = BIG ? 0x3FFFu : 0xFFu;
    static constexpr int MSH = BIG ? 27 : 21;
    __device__ static __forceinline__ uint32_t j(uint32_t x) { return x & 0x1FFFu; }
    __device__ static __forceinline__ uint32_t snap(uint32_t x) { return (x >> 13) & NONE; }
    __device__ static __forceinline__ uint32_t mask(uint32_t x) { return (x >> MSH) & 0xFu; }
    __device__ static __forceinline__ uint32_t make(uint32_t jj, uint32_t sn, uint32_t m) {
        return jj | (sn << 13) | (m << MSH);
    }
};
__device__ __forceinline__ uint32_t jsm_j(uint32_t x) { return x & 0x1FFFu; }
__device__ __forceinline__ uint32_t jsm_snap(uint32_t x) { return Pk<false>::snap(x); }
__device__ __forceinline__ uint32_t jsm_mask(uint32_t x) { return Pk<false>::mask(x); }
__device__ __forceinline__ uint32_t jsm_make(uint32_t j, uint32_t snap, uint32_t mask) {
    return Pk<false>::make(j, snap, mask);
}
constexpr uint32_t SNAP_NONE = 0xFFu;

// first free snapshot slot: not referenced by a live entry (except `skip`),
// nor equal to `extra` (a slot still to be read)
template <int SLOTS>
__device__ __forceinline__ int alloc_snapshot(const uint32_t (&s_ser)[SLOTS], const uint32_t (&s_jsm)[SLOTS], int D,
                                              int skip_lane, int skip_slot, uint32_t extra, int lane) {
    int slot = -1;
#pragma unroll
    for (int w = 0; w < SLOTS; w++) {
        uint32_t used = 0;
#pragma unroll
        for (int s = 0; s < SLOTS; s++) {
            const uint32_t sn = jsm_snap(s_jsm[s]);
            const bool skip = (lane == skip_lane && s == skip_slot);
            if (s_ser[s] != EMPTY && !skip && sn != SNAP_NONE && (int)(sn >> 5) == w) used |= 1u << (sn & 31);
        }
        used = __reduce_or_sync(FULL, used);
        if (extra != SNAP_NONE && (int)(extra >> 5) == w) used |= 1u << (extra & 31);
        const int lim = D - w * 32;
        uint32_t freem = ~used;
        if (lim < 32) freem &= (1u << lim) - 1u;
        if (slot < 0 && freem) slot = w * 32 + __ffs(freem) - 1;
    }
    POLAR_DCHECK(slot >= 0 && slot < D);
    return slot;
}

// NL > 0: compile-time code length 2^NL (stage sizes and shifts fold to
// constants); NL = 0: any N at run time.
// Snapshot-slot allocation with a conservative used-bitmap (uniform across the
// warp): bits are set on allocation and only cleared by an exact recount from
// the live entries, done when the bitmap has no free slot left.
template <int SLOTS>
__device__ __forceinline__ int alloc_snapshot_lazy(uint32_t *used, const uint32_t (&s_ser)[SLOTS],
                                                   const uint32_t (&s_jsm)[SLOTS], int D, int skip_lane,
                                                   int skip_slot, uint32_t extra, int lane, int nlive = 0) {
    if (SLOTS == 1) return alloc_snapshot<SLOTS>(s_ser, s_jsm, D, skip_lane, skip_slot, extra, lane);  // 1 REDUX: exact
    int slot = -1;
#pragma unroll
    for (int w = 0; w < SLOTS; w++) {
        const int lim = D - w * 32;
        uint32_t freem = ~used[w];
        if (lim < 32) freem &= (lim > 0) ? ((1u << lim) - 1u) : 0u;
        if (slot < 0 && freem) slot = w * 32 + __ffs(freem) - 1;
    }
    // an exact recount also when the first free slot is above POLAR_SNAP_SOFT
    // + the live entries (so a recount always lands below the cap):
    // the slots in use stay compact, so the per-warp arena stays L2-resident
    if (slot < 0 || slot >= POLAR_SNAP_SOFT + nlive) {
        slot = -1;
#pragma unroll
        for (int w = 0; w < SLOTS; w++) {
            uint32_t u = 0;
#pragma unroll
            for (int s = 0; s < SLOTS; s++) {
                const uint32_t sn = jsm_snap(s_jsm[s]);
                const bool skip = (lane == skip_lane && s == skip_slot);
                if (s_ser[s] != EMPTY && !skip && sn != SNAP_NONE && (int)(sn >> 5) == w) u |= 1u << (sn & 31);
            }
            u = __reduce_or_sync(FULL, u);
            if (extra != SNAP_NONE && (int)(extra >> 5) == w) u |= 1u << (extra & 31);
            __syncwarp();
            if (lane == 0) used[w] = u;
        }
        __syncwarp();
#pragma unroll
        for (int w = 0; w < SLOTS; w++) {
            const int lim = D - w * 32;
            uint32_t freem = ~used[w];
            if (lim < 32) freem &= (lim > 0) ? ((1u << lim) - 1u) : 0u;
            if (slot < 0 && freem) slot = w * 32 + __ffs(freem) - 1;
        }
    }
    __syncwarp();
    if (lane == 0) used[slot >> 5] |= 1u << (slot & 31);
    __syncwarp();
    POLAR_DCHECK(slot >= 0 && slot < D);
    return slot;
}

// Global stack (D > 128): the same conservative bitmap over D slots, in
// shared memory (UW = ceil(D/32) words), searched from a hint word (every word
// below it is full); the exact recount scans the live entries of the global
// stack (all but entry `skip`) and marks `extra`.
// (hot: also the hot-window entry of this lane, hser / hjsm)
__device__ __forceinline__ int alloc_snapshot_big(uint32_t *used, int &uhint, const uint32_t *sjsm, int nS, int D,
                                                  int skip, uint32_t extra, int lane, bool hot = false,
                                                  uint32_t hser = 0xFFFFFFFFu, uint32_t hjsm = 0) {
    const int UW = (D + 31) >> 5;
    int slot = -1;
    // (pass 0 finds a slot above max(POLAR_SNAP_SOFT, 2 nS): recount, so the
    // slots in use stay compact and the arena L2-resident)
    const int soft = max(POLAR_SNAP_SOFT, 2 * nS + 64);
    #pragma unroll 1
    for (int pass = 0; pass < 2 && slot < 0; pass++) {
        if (pass == 1) {
            #pragma unroll 1
            for (int w_0 = 0; w_0 < (UW); w_0 += 32) if (const int w = w_0 + lane; w < (UW)) used[w] = 0u;
            __syncwarp();
            #pragma unroll 1
            for (int i_0 = 0; i_0 < (nS); i_0 += 32) if (const int i = i_0 + lane; i < (nS)) {
                const uint32_t sn = Pk<true>::snap(sjsm[i]);
                if (i != skip && sn != Pk<true>::NONE) atomicOr(used + (sn >> 5), 1u << (sn & 31));
            }
            if (hot && hser != 0xFFFFFFFFu) {
                const uint32_t sn = Pk<true>::snap(hjsm);
                if (sn != Pk<true>::NONE) atomicOr(used + (sn >> 5), 1u << (sn & 31));
            }
            __syncwarp();
            if (lane == 0 && extra != Pk<true>::NONE) used[extra >> 5] |= 1u << (extra & 31);
            __syncwarp();
            uhint = 0;
        }
        #pragma unroll 1
        for (int w0 = uhint; w0 < UW; w0 += 32) {
            const int wi = w0 + lane;
            uint32_t fm = 0;
            if (wi < UW) {
                fm = ~used[wi];
                const int lim = D - wi * 32;
                if (lim < 32) fm &= (1u << lim) - 1u;
            }
            const uint32_t b = __ballot_sync(FULL, fm != 0u);
            if (b) {
                const int fl = __ffs(b) - 1;
                const uint32_t fv = __shfl_sync(FULL, fm, fl);
                slot = 32 * (w0 + fl) + __ffs(fv) - 1;
                uhint = w0 + fl;
                if (pass == 0 && slot >= soft) slot = -1;
                break;
            }
        }
    }
    __syncwarp();
    if (lane == 0) used[slot >> 5] |= 1u << (slot & 31);
    __syncwarp();
    POLAR_DCHECK(slot >= 0 && slot < D);
    return slot;
}

// launch bound (CTAs of 4 warps per SM) per instantiation: register stacks
// of 2 or 4 entries per lane need more registers; the N = 2048 and N = 4096
// specialisations trade registers for warps (measured)
#ifndef POLAR_MB_PLAIN
#define POLAR_MB_PLAIN 9       // CTAs per SM of the no-CRC register-stack instances (A/B builds override)
#endif
#ifndef POLAR_MB_N11
#define POLAR_MB_N11 7         // CTAs per SM of the N = 2048 instances (7 x 29 KB shared memory fits)
#endif
#ifndef POLAR_MB_N12
#define POLAR_MB_N12 6         // CTAs per SM of the N = 4096 instances (80 registers, no spill: C5 2874 -> 3038 Mbps; 7: 2900)
#endif
#ifndef POLAR_MB_BIG
#define POLAR_MB_BIG kDecodeMinBlocks
#endif
#ifndef POLAR_MB_SL1
#define POLAR_MB_SL1 kDecodeMinBlocks
#endif
template <int SLOTS, int NL, bool NOCRC>
constexpr int kDecodeMinBlocksFor() {
    return NL == 11 ? POLAR_MB_N11 : (NL == 12 ? POLAR_MB_N12 : (SLOTS == 4 ? 3 : (SLOTS == 2 ? 5 : (NOCRC && SLOTS == 1 ? POLAR_MB_PLAIN : (SLOTS == 1 ? POLAR_MB_SL1 : (SLOTS == 0 ? POLAR_MB_BIG : kDecodeMinBlocks))))));
}

// SLOTS = 1, 2, 4: register stack of 32 SLOTS entries (D <= 128).  SLOTS = 0:
// global stack (D up to 8192, the paper's D = NL): dense unsorted arrays per
// warp in global memory (L2-resident in practice), scanned by the 32 lanes.
// MODE (compile time): 0 general; 1 systematic readout and more than one node
// (re-encoding and whole-code-node paths left out of the code); 2 as 1 and no
// CRC (the CRC path left out too)
// CNT: the instrumented instance behind polar_scs_decode_counts — the same
// decode, placement read from the parameters, and per frame the work it
// executed: f/g evaluations, BETA XOR bits, node elements, snapshot words
template <int SLOTS, bool SNAP_SMEM, bool CHAN_SMEM, int NL = 0, bool GA = false, int MODE = 0, bool CNT = false>
__global__ void __launch_bounds__(kDecodeWarps * 32, kDecodeMinBlocksFor<SLOTS, NL, MODE == 2>())
fsscs_decode_kernel(const DecodeParams P) {
    constexpr bool BIG = (SLOTS == 0);
    constexpr int SL = BIG ? 1 : SLOTS;       // register arrays (unused when BIG)
    // register stacks (D <= 128) are kept sorted by (PM, serial): position
    // p = 32 s + lane in slot s (position 0 = best): select reads the head,
    // insertion is one merge
    // D > 128 (HOT): a sorted 32-entry window in registers (the SLOTS = 1 stack)
    // holds the best entries, an unsorted global store (cold) the rest, with
    // hot keys <= cb < cold keys; GSCAN: the whole stack in global memory,
    // scanned on every pop
    constexpr bool HOT = BIG && (POLAR_BIG_HOT != 0);
    constexpr bool GSCAN = BIG && !HOT;
    constexpr bool SORTED = (!BIG && ((SLOTS == 1 && POLAR_SORTED_STACK >= 1) || POLAR_SORTED_STACK >= 2)) || HOT;
    // code-length-specialised kernels with N <= 1024: the flat beta (N/32 <= 32
    // words) lives in registers, word w in lane w (bw); beta[] in shared memory
    // only stages the output
    constexpr bool BREG = (NL == 10 || NL == 7) && (POLAR_BETA_REGS != 0);
    // NOSER: no serial word per entry (sorted register stacks): an entry is
    // live iff its PM word is not EMPTY (a NaN pattern no PM takes), and the
    // working path's entry carries WFLAG in its jsm word
    constexpr bool NOSER = SORTED && !BIG && (POLAR_NOSER != 0);
    constexpr uint32_t WFLAG = 1u << 25;
    // node-kind-specialised inserts and the full sum tree, per kernel as measured
    constexpr bool R0F = SORTED && !HOT && (POLAR_R0_FAST == 2 || (POLAR_R0_FAST == 1 && !CNT && (NL == 10 || NL == 11)));
    constexpr bool REPF = SORTED && !HOT && (POLAR_REP_FAST == 2 || (POLAR_REP_FAST == 1 && !CNT && NL == 10));
    constexpr bool SUMF = (POLAR_SUM_FULL == 2 || (POLAR_SUM_FULL == 1 && !CNT && (NL == 10 || NL == 11)));
    using PK = Pk<BIG>;
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31;
    // warp index as a warp reduction: ptxas then knows it (and every shared-
    // memory address derived from it) is warp-uniform, so branches on values
    // loaded from this warp's shared memory compile as uniform branches, with
    // no reconvergence barriers or divergence checks around the warp intrinsics
    const int warp = (int)__reduce_max_sync(FULL, threadIdx.x >> 5);
    const int n = (NL > 0) ? NL : P.n;
    const int N = 1 << n;
    const int nw = (NL > 0) ? (NL >= 5 ? (1 << NL) / 32 : 1) : P.nw;
    const int K = P.K, D = P.D, M = P.M;

    // per-depth records (host.cpp: node j and the node j-1 that ends a path of
    // depth j, unpacked), staged in shared memory when they fit; the schedule
    // walk between nodes is derived from them
    // (register-stack specialised kernels are only launched when they fit; the
    // global-stack kernel reads them through L1: their shared memory costs it a CTA)
    const bool recs_smem = (POLAR_RECS_SMEM && NL > 0 && !BIG) || P.sched_words > 0;
    if (recs_smem) {
        #pragma unroll 1
        for (int i = threadIdx.x; i < P.sched_words / 4; i += blockDim.x)
            reinterpret_cast<uint4 *>(smem)[i] = P.recs[i];
        __syncthreads();
    }
    auto rec_at = [&](int jj, int q) -> uint4 {
        return recs_smem ? reinterpret_cast<const uint4 *>(smem)[4 * jj + q] : __ldg(P.recs + 4 * jj + q);
    };
    uint32_t *wb = smem + P.sched_words + warp * P.warp_words;
    // BIG: the first KW stack keys live in shared memory (the rest in global)
    constexpr int KW = HOT ? 0 : 128;
    unsigned long long *wkey = reinterpret_cast<unsigned long long *>(wb);
    const bool chan_sm = CNT ? (P.chan_in_smem != 0) : CHAN_SMEM;
    const bool snap_sm = CNT ? (P.snap_in_smem != 0) : SNAP_SMEM;
    float *chan_s = reinterpret_cast<float *>(wb + P.win_words);   // channel row (chan_sm)
    float *alpha = chan_sm ? chan_s + N : chan_s;                  // stages >= 6 (+ scratch)
    // (code-length-specialised kernels without the L2 arena: alpha_words = N, a constant)
    uint32_t *beta = reinterpret_cast<uint32_t *>(alpha + ((POLAR_CONST_AW && NL > 0 && !GA && !CNT) ? (1 << NL) : P.alpha_words));
    // stage t lives at [2^t, 2^{t+1}) of the shared alpha memory, or of this
    // warp's global (L2) arena for t >= sg (sg = n: everything in shared memory)
    const int sg = P.sg;
    float *galpha = P.galpha ? P.galpha + (size_t)(blockIdx.x * kDecodeWarps + warp) * (size_t)N : alpha;
    auto SP = [&](int t) -> float * {
        if constexpr (GA || CNT) return (t >= sg ? galpha : alpha) + (1 << t);
        return alpha + (1 << t);
    };
    uint32_t *best = beta + nw;
    uint16_t *cnt = reinterpret_cast<uint16_t *>(best + nw);
    uint32_t *shdr = best + nw + P.cnt_words;                      // fork headers m1..m4, 2 words/slot (!BIG)
    uint32_t *snap_used = shdr + P.hdr_words;                      // snapshot-slot bitmap (used_words)
    uint32_t *uhat = snap_used + P.used_words;                     // nw words: u_hat (non-systematic)
    // snapshot slot k of this warp: shared memory, or global slot index snap0 + k
    uint32_t *snap_s = uhat + P.uhat_words;                        // (uhat_words = nw only when non-systematic)
    const uint32_t gwarp = (uint32_t)(blockIdx.x * kDecodeWarps + warp);
    const uint32_t snap0 = gwarp * (uint32_t)D;
    // global stack (BIG): keys (PM bits << 32 | serial: u64 order = (PM, serial)
    // order, reading R7) and jsm words; fork headers per slot
    unsigned long long *skey = BIG ? P.stack_keys + (size_t)gwarp * (size_t)(D + kColdPad) : nullptr;
    uint32_t *sjsm = BIG ? P.stack_jsm + (size_t)gwarp * (size_t)(D + kColdPad) : nullptr;
    uint2 *ghdr = BIG ? P.hdr_global + (size_t)gwarp * (size_t)D : nullptr;
    auto kget = [&](int i) -> unsigned long long { return i < KW ? wkey[i] : __ldcg(skey + i); };
    auto kset = [&](int i, unsigned long long k) {
        if (i < KW) wkey[i] = k;
        else skey[i] = k;
    };
    auto hdr_at = [&](int k) -> uint2 * { return BIG ? ghdr + k : reinterpret_cast<uint2 *>(shdr) + k; };
    const int sstride = (NL > 0) ? nw : P.snap_stride;
    auto snap_slot = [&](int k) -> uint32_t * {
        POLAR_DCHECK(k >= 0 && k < D);
        if (snap_sm) return snap_s + k * sstride;
        return P.snap_global + (size_t)(snap0 + (uint32_t)k) * (size_t)sstride;
    };

    // frame queue: each warp holds the frame it decodes and the next one it
    // claimed, whose LLR row is prefetched into L2 meanwhile
    unsigned long long f = 0, fnext = 0;
    if (lane == 0) { f = atomicAdd(P.queue, 1ull); fnext = atomicAdd(P.queue, 1ull); }
    f = __shfl_sync(FULL, f, 0);
    fnext = __shfl_sync(FULL, fnext, 0);
    const unsigned long long nfr = (unsigned long long)P.n_frames;

    #pragma unroll 1
    while (f < nfr) {
        if (P.ready) wait_chunk_ready(P.ready, P.err, f, P.chunk_shift);   // streaming: this frame's chunk has landed
        if (fnext < nfr && (!P.ready || __reduce_or_sync(FULL, ld_acquire_u32(P.ready + (fnext >> P.chunk_shift))))) {
            const char *nr = reinterpret_cast<const char *>(P.llr + (size_t)fnext * N);
            #pragma unroll 1
            for (int b = lane * 128; b < N * 4; b += 32 * 128)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(nr + b));
        }
        unsigned long long fnext2 = 0;
        if (lane == 0) fnext2 = atomicAdd(P.queue, 1ull);

        // ---- the channel row (the only mandatory HBM read) -----------------
        const float *row = P.llr + (size_t)f * N;
        const float *chan = chan_sm ? chan_s : row;
        if (chan_sm) {
            if (N >= 4) {
                #pragma unroll 1
                for (int i = lane * 4; i < N; i += 128)
                    *reinterpret_cast<float4 *>(chan_s + i) = __ldcs(reinterpret_cast<const float4 *>(row + i));
            } else if (lane < N) {
                chan_s[lane] = row[lane];
            }
        }
        #pragma unroll 1
        for (int i_0 = 0; i_0 < (P.cnt_words); i_0 += 32) if (const int i = i_0 + lane; i < (P.cnt_words)) reinterpret_cast<uint32_t *>(cnt)[i] = 0;
        __syncwarp();

        // ---- stack: root path (PM 0, serial 0, j 0) ------------------------
        uint32_t s_pm[SL], s_ser[SL], s_jsm[SL];
#pragma unroll
        for (int s = 0; s < SL; s++) { s_pm[s] = EMPTY; s_ser[s] = EMPTY; s_jsm[s] = PK::make(0, PK::NONE, 0); }
        if (lane == 0) { s_pm[0] = 0u; s_ser[0] = 0u; if (NOSER) s_jsm[0] |= WFLAG; }
        int nS = 1;
        int uhint = 0;
        int widx = 0;                     // BIG: index of the working path's entry (-1: not live)
        int nA = HOT ? 0 : 1, hole = -1;  // BIG: array extent (HOT: cold entries); the popped entry's index until refilled
        int nH = 1;                       // HOT: entries in the hot window (positions 0..nH-1)
        unsigned long long cb = ~0ull;    // HOT: hot keys <= cb < cold keys
        if (BIG) {
            if (GSCAN && lane == 0) { kset(0, 0ull); sjsm[0] = PK::make(0, PK::NONE, 0); }
            #pragma unroll 1
            for (int w_0 = 0; w_0 < (P.used_words); w_0 += 32) if (const int w = w_0 + lane; w < (P.used_words)) snap_used[w] = 0u;
        } else if (lane < 4) {
            snap_used[lane] = 0u;      // conservative snapshot-slot bitmap (alloc_snapshot_lazy)
        }
        __syncwarp();
        uint32_t work = 0, next_serial = 1, pops = 0, switches = 0;
        uint32_t bw = 0;                  // BREG: word `lane` of the working path's flat beta
        uint32_t c_fg = 0, c_bb = 0, c_ne = 0, c_sw = 0;     // CNT: executed work of this frame
        int work_pl = 0;
        // alpha memory content: stages s >= lev_mem hold the node (s, pos_mem >> s)
        // for the working path's beta (partial-spine reuse, reading R12)
        int pos_mem = 0, lev_mem = n;
        float r[6];                       // alpha stages 0..5 (Lambda <= 32): element i in lane i
#pragma unroll
        for (int t = 0; t < 6; t++) r[t] = 0.f;
        bool have_best = false;
        float best_pm = 0.f, out_pm = 0.f;
        int status = 0;
        bool from_best = false;
        const uint32_t pop_cap = (uint32_t)P.L * (uint32_t)(M + 1);

        #pragma unroll 1
        for (;;) {
            // (the watchdog cannot fire: cnt[j] <= L bounds the pops by L (M + 1);
            // the specialised kernels leave it out)
            if (nS == 0 || ((MODE == 0 || !POLAR_LEAN_WATCHDOG) && pops >= pop_cap)) {
                if (nS == 0) { from_best = true; out_pm = best_pm; status = 1; }   // reading R13
                else { status = 2; out_pm = -1.f; }        // watchdog: cannot happen (cnt[j] <= L)
                break;
            }
            // ---- select: min (PM, serial) (reading R7)
            uint32_t lpm = EMPTY, lser = EMPTY, ljsm = 0;
            int ls = 0;
            uint32_t ljsm_big = 0;
            if (HOT && nH == 0) {
                // refill the hot window from the cold store (nS > 0, so nA > 0).
                // Each lane keeps the two smallest keys of its strided share; with
                // t = the smallest of the lanes' second keys, every cold key <= t is
                // in those lists, so extracting the lists' minimum while it is <= t
                // yields the cold keys in ascending order, up to 32 of them
                unsigned long long k1 = ~0ull, k2 = ~0ull;
                int i1 = -1, i2 = -1;
                #pragma unroll 1
                for (int i0 = 0; i0 < nA; i0 += 128) {
                    unsigned long long k4[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const int i = i0 + 32 * q + lane;
                        k4[q] = (i < nA) ? __ldcg(skey + i) : ~0ull;
                    }
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const int i = i0 + 32 * q + lane;
                        if (k4[q] < k1) { k2 = k1; i2 = i1; k1 = k4[q]; i1 = i; }
                        else if (k4[q] < k2) { k2 = k4[q]; i2 = i; }
                    }
                }
                uint32_t th, tl;
                warp_min_key((uint32_t)(k2 >> 32), (uint32_t)k2, th, tl);
                const unsigned long long tk = ((unsigned long long)th << 32) | tl;
                uint32_t j1 = (i1 >= 0) ? __ldcg(sjsm + i1) : 0u, j2 = (i2 >= 0) ? __ldcg(sjsm + i2) : 0u;
                unsigned long long last = 0;
                #pragma unroll 1
                while (nH < 32) {
                    uint32_t mh, ml;
                    warp_min_key((uint32_t)(k1 >> 32), (uint32_t)k1, mh, ml);
                    const unsigned long long mk = ((unsigned long long)mh << 32) | ml;
                    if (mk == ~0ull || mk > tk) break;
                    const int ow = __ffs(__ballot_sync(FULL, k1 == mk)) - 1;
                    const uint32_t jj = __shfl_sync(FULL, j1, ow);
                    if (lane == nH) { s_pm[0] = mh; s_ser[0] = ml; s_jsm[0] = jj; }
                    if (lane == ow) {
                        skey[i1] = ~0ull;                          // taken: dropped by the compaction below
                        k1 = k2; i1 = i2; j1 = j2; k2 = ~0ull; i2 = -1;
                    }
                    last = mk;
                    nH++;
                }
                cb = last;
                __syncwarp();
                // compact the cold store (the working path's index follows its entry)
                int cntc = 0, nwidx = -1;
                #pragma unroll 1
                for (int i0 = 0; i0 < nA; i0 += 32) {
                    const int i = i0 + lane;
                    unsigned long long a = ~0ull;
                    uint32_t x = 0;
                    if (i < nA) { a = __ldcg(skey + i); x = __ldcg(sjsm + i); }
                    const bool keep = (a != ~0ull);
                    const uint32_t kb = __ballot_sync(FULL, keep);
                    const int o = cntc + __popc(kb & ((1u << lane) - 1u));
                    const uint32_t wbb = __ballot_sync(FULL, keep && i == widx);
                    if (wbb) nwidx = cntc + __popc(kb & ((1u << (__ffs(wbb) - 1)) - 1u));
                    __syncwarp();
                    if (keep) { skey[o] = a; sjsm[o] = x; }
                    cntc += __popc(kb);
                }
                widx = nwidx;
                nA = cntc;
                if (nA == 0) cb = ~0ull;
                __syncwarp();
            }
            if (GSCAN) {
                // window keys from shared memory, the rest from global memory with 4
                // independent loads in flight per lane per round
                unsigned long long lk = ~0ull;
                int lq = 0;
#pragma unroll
                for (int q = 0; q < 4; q++) {
                    const int i = 32 * q + lane;
                    const unsigned long long k = (i < nA) ? wkey[i] : ~0ull;
                    if (k < lk) { lk = k; lq = q; }
                }
                ls = 32 * lq + lane;
                #pragma unroll 1
                for (int i0 = KW; i0 < nA; i0 += 128) {
                    unsigned long long k4[4];
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const int i = i0 + 32 * q + lane;
                        k4[q] = (i < nA) ? __ldcg(skey + i) : ~0ull;
                    }
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if (k4[q] < lk) { lk = k4[q]; ls = i0 + 32 * q + lane; }
                }
                lpm = (uint32_t)(lk >> 32);
                lser = (uint32_t)lk;
                // speculative: every lane fetches the jsm word of its own best entry
                // while the warp reduction runs
                ljsm_big = (lk != ~0ull) ? __ldcg(sjsm + ls) : 0u;
            } else if (!SORTED) {
#pragma unroll
                for (int s = 0; s < SL; s++)
                    if (s_pm[s] < lpm || (s_pm[s] == lpm && s_ser[s] < lser)) { lpm = s_pm[s]; lser = s_ser[s]; ljsm = s_jsm[s]; ls = s; }
            }
            uint32_t mpm, mser;
            int owner = 0;
            if (SORTED) {
                // the sorted stack's head (lane 0) is the best path
                mpm = __shfl_sync(FULL, s_pm[0], 0);
                mser = NOSER ? 0u : __shfl_sync(FULL, s_ser[0], 0);
            } else {
                warp_min_key(lpm, lser, mpm, mser);
                owner = __ffs(__ballot_sync(FULL, lpm == mpm && lser == mser)) - 1;
            }
            uint32_t p_jsm;
            if (SORTED) {
                p_jsm = __shfl_sync(FULL, s_jsm[0], 0);
                if (lane == 0) { s_pm[0] = EMPTY; s_ser[0] = EMPTY; }
                if (HOT) nH--;
            } else if (BIG) {
                // remove entry `pi`: it becomes a hole that c1 of this pop refills
                const int pi = __shfl_sync(FULL, ls, owner);
                p_jsm = __shfl_sync(FULL, ljsm_big, owner);
                hole = pi;
                if (widx == pi) widx = -1;
            } else {
                p_jsm = __shfl_sync(FULL, ljsm, owner);
                if (lane == owner) {
#pragma unroll
                    for (int s = 0; s < SL; s++) if (s == ls) { s_pm[s] = EMPTY; s_ser[s] = EMPTY; }
                }
            }
            nS--;
            POLAR_DCHECK(nS >= 0 && nS < D);
            pops++;
            const float p_pm = __uint_as_float(mpm);
            const uint32_t p_ser = mser;
            const bool sw = NOSER ? ((p_jsm & WFLAG) == 0u) : (p_ser != work);   // p is not the working path
            // register beta: a switch restores p's fork snapshot; its load is issued
            // here, ahead of the counter, prune and record reads (the slot holds nw
            // words, so every lane's word is in bounds)
            uint32_t pre_nv = 0;
            if (BREG && POLAR_PREFETCH_SNAP && sw && lane < nw) {
                const uint32_t *ps_src = snap_slot((int)PK::snap(p_jsm));
                pre_nv = snap_sm ? ps_src[lane] : __ldcg(ps_src + lane);
            }
            const int j = (int)jsm_j(p_jsm);
#ifdef POLAR_TRACE_FRAME
            if (f == POLAR_TRACE_FRAME && lane == 0)
                printf("TRACE pop %u: pm %.9g (%#x) ser %u j %d work %u\n", pops, p_pm, mpm, p_ser, j, work);
#endif

            // ---- per-length counter and prune (readings R9, R10)
            const int c_j = (int)cnt[j] + 1;
            __syncwarp();
            if (lane == 0) cnt[j] = (uint16_t)c_j;
            if (c_j == P.L) {
                int cntv = 0;
                if (BIG) {
                    // in-place compaction of the entries with depth > j
                    int nwidx = -1;
                    #pragma unroll 1
                    for (int i0 = 0; i0 < nA; i0 += 32) {
                        const int i = i0 + lane;
                        unsigned long long a = 0;
                        uint32_t x = 0;
                        if (i < nA) { a = kget(i); x = __ldcg(sjsm + i); }
                        const bool keep = (i < nA) && i != hole && (int)PK::j(x) > j;
                        const uint32_t kb = __ballot_sync(FULL, keep);
                        const int o = cntv + __popc(kb & ((1u << lane) - 1u));
                        const uint32_t wbb = __ballot_sync(FULL, keep && i == widx);
                        if (wbb) nwidx = cntv + __popc(kb & ((1u << (__ffs(wbb) - 1)) - 1u));
                        __syncwarp();
                        if (keep) { kset(o, a); sjsm[o] = x; }
                        cntv += __popc(kb);
                    }
                    widx = nwidx;
                    nA = cntv;
                    hole = -1;
                    __syncwarp();
                }
                const int ncold = BIG ? cntv : 0;       // HOT: the cold survivors
                if (GSCAN) {
                } else if (SORTED && SL > 1) {
                    // survivors (depth > j) move to positions 1..cntv in order;
                    // position P takes survivor number P: word v holding it by the
                    // running counts, its bit by binary search on prefix counts
                    uint32_t kb[SL];
                    int cum[SL + 1];
                    cum[0] = 0;
#pragma unroll
                    for (int q = 0; q < SL; q++) {
                        kb[q] = __ballot_sync(FULL, (NOSER ? s_pm[q] : s_ser[q]) != EMPTY && (int)jsm_j(s_jsm[q]) > j);
                        cum[q + 1] = cum[q] + __popc(kb[q]);
                    }
                    cntv = cum[SL];
                    uint32_t npm[SL], nser[SL], njsm[SL];
#pragma unroll
                    for (int w = 0; w < SL; w++) {
                        const int k = 32 * w + lane - 1;             // survivor index (0-based)
                        const bool dst = (k >= 0 && k < cntv);
                        int v = 0, kk = k;
                        uint32_t wbits = kb[0];
#pragma unroll
                        for (int q = 1; q < SL; q++)
                            if (k >= cum[q]) { v = q; kk = k - cum[q]; wbits = kb[q]; }
                        int src = 0;
#pragma unroll
                        for (int st = 16; st >= 1; st >>= 1) {
                            const int hi = src + st - 1;
                            if (__popc(wbits & (hi >= 31 ? FULL : ((2u << hi) - 1u))) <= kk) src += st;
                        }
                        uint32_t gp = EMPTY, gs = EMPTY, gj = 0;
#pragma unroll
                        for (int q = 0; q < SL; q++) {
                            const uint32_t xp = __shfl_sync(FULL, s_pm[q], src);
                            const uint32_t xs = NOSER ? 0u : __shfl_sync(FULL, s_ser[q], src);
                            const uint32_t xj = __shfl_sync(FULL, s_jsm[q], src);
                            gp = (v == q) ? xp : gp; gs = (v == q) ? xs : gs; gj = (v == q) ? xj : gj;
                        }
                        npm[w] = dst ? gp : EMPTY;
                        nser[w] = dst ? gs : EMPTY;
                        njsm[w] = gj;
                    }
#pragma unroll
                    for (int w = 0; w < SL; w++) { s_pm[w] = npm[w]; s_ser[w] = nser[w]; s_jsm[w] = njsm[w]; }
                } else if (SORTED) {
                    // survivors (depth > j) move to lanes 1..cntv in order (a subset
                    // of a sorted list is sorted); lane 0 stays free
                    const uint32_t kb = __ballot_sync(FULL, (NOSER ? s_pm[0] : s_ser[0]) != EMPTY && (int)jsm_j(s_jsm[0]) > j);
                    cntv = __popc(kb);
                    const bool dst = (lane >= 1 && lane <= cntv);
                    // source lane = position of the lane-th set bit of kb (binary search on prefix counts)
                    int src = 0;
#pragma unroll
                    for (int st = 16; st >= 1; st >>= 1) {
                        const int hi = src + st - 1;                  // bits [0, hi] hold fewer than `lane` survivors?
                        if (__popc(kb & (hi >= 31 ? FULL : ((2u << hi) - 1u))) < lane) src += st;
                    }
                    const uint32_t npm = __shfl_sync(FULL, s_pm[0], src);
                    const uint32_t njsm = __shfl_sync(FULL, s_jsm[0], src);
                    s_pm[0] = dst ? npm : EMPTY;
                    if constexpr (!NOSER) {
                        const uint32_t nser = __shfl_sync(FULL, s_ser[0], src);
                        s_ser[0] = dst ? nser : EMPTY;
                    }
                    s_jsm[0] = njsm;
                } else {
#pragma unroll
                    for (int s = 0; s < SL; s++) {
                        if (s_ser[s] != EMPTY && (int)jsm_j(s_jsm[s]) <= j) { s_pm[s] = EMPTY; s_ser[s] = EMPTY; }
                        cntv += __popc(__ballot_sync(FULL, s_ser[s] != EMPTY));
                    }
                }
                if (HOT) {
                    nH = cntv;
                    cntv += ncold;
                    if (nA == 0) cb = ~0ull;
                }
                nS = cntv;
            }

            // the record of depth j: p's path length (= the start of node j,
            // PAPER.md:L784-791), node j, and the node j-1 that created p
            const uint4 ra = rec_at(j, 0), rb = rec_at(j, 1), rc = rec_at(j, 2), rd = rec_at(j, 3);
            const int pl = (int)ra.x;
            const int pkind = (int)rb.z, plam = (int)rd.z;

            // ---- path switch ---------------------
            int s_d = 0;
            if (sw) {
                switches++;
                // the path being left keeps its beta in a snapshot if it is still live
                if (BIG) {
                    const int wi = widx;
                    if (wi >= 0) {
                        const uint32_t wj = __ldcg(sjsm + wi);
                        if (PK::snap(wj) == PK::NONE) {
                            const int slot = alloc_snapshot_big(snap_used, uhint, sjsm, nA, D, hole, PK::snap(p_jsm), lane,
                                                                HOT, s_ser[0], s_jsm[0]);
                            uint32_t *dst = snap_slot(slot);
                            const int nwords = (work_pl + 31) >> 5;
                            if constexpr (CNT) c_sw += (uint32_t)nwords;
                            if (BREG) { if (lane < nwords) dst[lane] = bw; }
                            else {
                                #pragma unroll 1
                                for (int w_0 = 0; w_0 < (nwords); w_0 += 32) if (const int w = w_0 + lane; w < (nwords)) dst[w] = beta[w];
                            }
                            if (lane == 0) sjsm[wi] = PK::make(PK::j(wj), (uint32_t)slot, 0);
                            __syncwarp();
                        }
                    }
                }
                int wsl = -1;
#pragma unroll
                for (int s = 0; s < SL; s++)
                    if (!GSCAN && (NOSER ? (s_pm[s] != EMPTY && (s_jsm[s] & WFLAG) != 0u) : (s_ser[s] == work))) wsl = s;
                const uint32_t wb_ = __ballot_sync(FULL, wsl >= 0);
                if (!GSCAN && wb_) {
                    const int wl = __ffs(wb_) - 1;
                    uint32_t wj = 0;
#pragma unroll
                    for (int s = 0; s < SL; s++) if (s == wsl) wj = s_jsm[s];
                    wj = __shfl_sync(FULL, wj, wl);
                    const int wslot = __shfl_sync(FULL, wsl, wl);
                    if (PK::snap(wj) == PK::NONE) {
                        int slot;
                        if constexpr (HOT) slot = alloc_snapshot_big(snap_used, uhint, sjsm, nA, D, -1, PK::snap(p_jsm), lane,
                                                                     true, s_ser[0], s_jsm[0]);
                        else slot = alloc_snapshot_lazy<SL>(snap_used, NOSER ? s_pm : s_ser, s_jsm, D, -1, 0, jsm_snap(p_jsm), lane, nS);
                        uint32_t *dst = snap_slot(slot);
                        const int nwords = (work_pl + 31) >> 5;
                        if constexpr (CNT) c_sw += (uint32_t)nwords;
                        if (BREG) { if (lane < nwords) dst[lane] = bw; }
                        else {
                            #pragma unroll 1
                            for (int w_0 = 0; w_0 < (nwords); w_0 += 32) if (const int w = w_0 + lane; w < (nwords)) dst[w] = beta[w];
                        }
                        if (lane == wl) {
#pragma unroll
                            for (int s = 0; s < SL; s++)
                                if (s == wslot) s_jsm[s] = PK::make(PK::j(wj), (uint32_t)slot, 0);
                        }
                    }
                }
                if (NOSER) {                          // the path being left is no longer the working path
#pragma unroll
                    for (int s = 0; s < SL; s++) s_jsm[s] &= ~WFLAG;
                }
                // restore p's beta (fork snapshot), locating the first bit d where it
                // differs from the beta the alpha memory was computed from
                const uint32_t ps = PK::snap(p_jsm), rel = PK::mask(p_jsm);
                const uint32_t *src = snap_slot((int)ps);
                const int nwords = (pl + 31) >> 5;
                if constexpr (CNT) c_sw += (uint32_t)nwords;
                int d = 0x7FFFFFFF;
                if (BREG) {
                    uint32_t x = 0;
                    if (lane < nwords) {
                        const uint32_t nv = POLAR_PREFETCH_SNAP ? pre_nv : (snap_sm ? src[lane] : __ldcg(src + lane));
                        x = nv ^ bw;
                        if (lane == nwords - 1 && (pl & 31)) x &= (1u << (pl & 31)) - 1u;
                        bw = nv;
                    }
                    const uint32_t b = __ballot_sync(FULL, x != 0);
                    if (b) {
                        const int fl = __ffs(b) - 1;
                        d = 32 * fl + __ffs(__shfl_sync(FULL, x, fl)) - 1;
                    }
                }
                #pragma unroll 1
                for (int w0 = 0; !BREG && w0 < nwords; w0 += 32) {
                    const int w = w0 + lane;
                    uint32_t x = 0;
                    if (w < nwords) {
                        const uint32_t nv = snap_sm ? src[w] : __ldcg(src + w);
                        x = nv ^ beta[w];
                        if (w == nwords - 1 && (pl & 31)) x &= (1u << (pl & 31)) - 1u;
                        beta[w] = nv;
                    }
                    const uint32_t b = __ballot_sync(FULL, x != 0);
                    if (b && d == 0x7FFFFFFF) {
                        const int fl = __ffs(b) - 1;
                        const uint32_t xv = __shfl_sync(FULL, x, fl);
                        d = 32 * (w0 + fl) + __ffs(xv) - 1;
                    }
                }
                if (pl > d) s_d = bitlen((uint32_t)pl ^ (uint32_t)d);
                __syncwarp();
                if (rel != 0u) {
                    const int Lam = 1 << plam, seg = pl - Lam;      // node j-1
                    if (BREG) {
                        uint32_t fm = 0;          // this lane's word of the flip pattern
                        if (pkind == OP_REP) {
                            if (Lam >= 32) fm = (lane >= (seg >> 5) && lane < (seg >> 5) + (Lam >> 5)) ? FULL : 0u;
                            else if (lane == (seg >> 5)) fm = ((1u << Lam) - 1u) << (seg & 31);
                        } else {
                            const uint2 hh = *hdr_at((int)ps);
                            const uint32_t m[4] = {hh.x & 0xFFFFu, hh.x >> 16, hh.y & 0xFFFFu, hh.y >> 16};
#pragma unroll
                            for (int q = 0; q < 4; q++) {
                                const int pos = seg + (int)m[q];
                                if (((rel >> q) & 1u) && lane == (pos >> 5)) fm ^= 1u << (pos & 31);
                            }
                        }
                        bw ^= fm;
                    } else if (pkind == OP_REP) {
                        if (Lam >= 32) {
                            #pragma unroll 1
                            for (int t_0 = 0; t_0 < ((Lam >> 5)); t_0 += 32) if (const int t = t_0 + lane; t < ((Lam >> 5))) beta[(seg >> 5) + t] ^= FULL;
                        } else if (lane == 0) {
                            beta[seg >> 5] ^= ((1u << Lam) - 1u) << (seg & 31);
                        }
                    } else if (lane == 0) {
                        const uint2 hh = *hdr_at((int)ps);
                        const uint32_t h0 = hh.x, h1 = hh.y;
                        const uint32_t m[4] = {h0 & 0xFFFFu, h0 >> 16, h1 & 0xFFFFu, h1 >> 16};
#pragma unroll
                        for (int q = 0; q < 4; q++)
                            if ((rel >> q) & 1u) {
                                const int pos = seg + (int)m[q];
                                beta[pos >> 5] ^= 1u << (pos & 31);
                            }
                    }
                    __syncwarp();
                }
                work = p_ser;
                widx = -1;                      // the new working path is not on the stack
            }
            work_pl = pl;

            // ---- pending BETA ops of p: climb from its
            // last node while it is a right child.  The levels with 2 Lambda <= 32
            // act inside one word: one RMW with the record's masks, each level
            // x ^= (x >> Lambda) & mask; the rest word by word.
            const int l = (int)rb.w;                 // level where the climb ends
            if (rc.x != 0xFFFFFFFFu) {
                uint32_t x = BREG ? bw : beta[rc.x];
                x ^= (x >> 1) & rc.y;
                x ^= (x >> 2) & rc.z;
                x ^= (x >> 4) & rc.w;
                x ^= (x >> 8) & rd.x;
                x ^= (x >> 16) & rd.y;
                if (BREG) { if (lane == (int)rc.x) bw = x; }
                else if (lane == 0) beta[rc.x] = x;
                __syncwarp();
                if constexpr (CNT) c_bb += (uint32_t)(__popc(rc.y) + __popc(rc.z) + __popc(rc.w) + __popc(rd.x) + __popc(rd.y));
            }
            {
                int ph = (int)rb.y;
                #pragma unroll 1
                for (int lw = (int)rb.x; ph & 1; ph >>= 1, lw++) {
                    if (BREG) beta_op_reg(bw, lw, ph, lane);
                    else beta_op(beta, lw, ph, lane);
                    if constexpr (CNT) c_bb += 1u << lw;
                }
            }

            if (j == M) {
                // ---- complete path: CRC on the systematic bits
                if (BREG) {                      // the register beta lands in beta[] (CRC, copy, output)
                    if (lane < nw) beta[lane] = bw;
                    __syncwarp();
                }
                bool ok = true;
                if (MODE < 2 && P.c > 0) {
                    // syndrome = XOR of the contributions of the set systematic bits,
                    // looked up per beta byte (tables hold information positions only)
                    const uint32_t *cw = beta;
                    if (MODE == 0 && P.nonsys) {
                        #pragma unroll 1
                        for (int w_0 = 0; w_0 < (nw); w_0 += 32) if (const int w = w_0 + lane; w < (nw)) uhat[w] = beta[w];
                        __syncwarp();
                        xform_words(uhat, N, nw, lane);
                        cw = uhat;
                    }
                    uint32_t syn = 0;
                    #pragma unroll 1
                    for (int w_0 = 0; w_0 < (nw); w_0 += 32) if (const int w = w_0 + lane; w < (nw)) {
                        const uint32_t x = cw[w];
                        const uint32_t *tw = P.crc_bytes + (size_t)w * 1024;
                        syn ^= __ldg(tw + (x & 255u)) ^ __ldg(tw + 256 + ((x >> 8) & 255u)) ^
                               __ldg(tw + 512 + ((x >> 16) & 255u)) ^ __ldg(tw + 768 + (x >> 24));
                    }
                    syn = __reduce_xor_sync(FULL, syn);
                    ok = (syn == 0);
                }
                // best effort (reading R13): the first complete path popped.  Its
                // copy is taken before the exit test (stores on the path after a
                // data-dependent loop exit made ptxas treat the loop as divergent)
                if (!have_best) {
                    #pragma unroll 1
                    for (int w_0 = 0; w_0 < (nw); w_0 += 32) if (const int w = w_0 + lane; w < (nw)) best[w] = beta[w];
                    __syncwarp();
                }
                if (BIG && hole >= 0) {
                    // no candidate refills the hole: the last entry moves into it
                    // (before the exit test too, for the same reason as the copy)
                    if (hole != nA - 1) {
                        const unsigned long long k = kget(nA - 1);
                        const uint32_t x = __ldcg(sjsm + nA - 1);
                        __syncwarp();
                        if (lane == 0) { kset(hole, k); sjsm[hole] = x; }
                        if (widx == nA - 1) widx = hole;
                    }
                    __syncwarp();
                    nA--;
                    hole = -1;
                }
                if (SORTED) {
                    // nothing is inserted: the entries at positions 1..nS move to
                    // 0..nS-1 (before the exit test too, for the same reason as the copy)
#pragma unroll
                    for (int q = 0; q < SL; q++) {
                        const uint32_t dp = __shfl_down_sync(FULL, s_pm[q], 1);
                        const uint32_t ds = NOSER ? 0u : __shfl_down_sync(FULL, s_ser[q], 1);
                        const uint32_t dj = __shfl_down_sync(FULL, s_jsm[q], 1);
                        uint32_t up = EMPTY, us = EMPTY, uj = 0;
                        if (q + 1 < SL) {
                            up = __shfl_sync(FULL, s_pm[q + 1 < SL ? q + 1 : q], 0);
                            us = NOSER ? 0u : __shfl_sync(FULL, s_ser[q + 1 < SL ? q + 1 : q], 0);
                            uj = __shfl_sync(FULL, s_jsm[q + 1 < SL ? q + 1 : q], 0);
                        }
                        s_pm[q] = (lane == 31) ? up : dp;
                        s_ser[q] = (lane == 31) ? us : ds;
                        s_jsm[q] = (lane == 31) ? uj : dj;
                    }
                }
                if (ok) { out_pm = p_pm; status = 0; break; }
                // the climb above combined blocks that the alpha memory was
                // computed from, so beta no longer tells the next switch which
                // stages are stale: recompute the next spine from the channel
                lev_mem = n;
                if (!have_best) {
                    have_best = true;
                    best_pm = p_pm;
                }
                continue;
            }

            // ---- ALPHA ops down to node j (Eq. 4, Alg. 1 / Alg. 4): stage s
            // holds node (s, pl >> s); stages >= s_min are still valid
            const int kind = (int)ra.w, lam = (int)ra.z;
            float xr = 0.f;                    // node alpha element of this lane (Lambda <= 32)
            {
                int s_min = max(max(lev_mem, bitlen((uint32_t)(pos_mem ^ pl))), max(s_d, l + 1));
                s_min = min(s_min, n);
                const int s_hi = s_min - 1;
                // register stages (Lambda <= 32): lo = element i, hi = element i + Lambda
                // by shuffle; enter the cascade at the first stage to compute, leave
                // after the node's own stage (its value is the node input xr)
#define POLAR_RSTAGE(T)                                                                    \
    {                                                                                      \
        const int Lt = 1 << (T);                                                           \
        float lo, hi;                                                                      \
        if ((T) + 1 == n) {                                                                \
            lo = ld1<CHAN_SMEM>(chan + (lane & (Lt - 1)), true);                            \
            hi = ld1<CHAN_SMEM>(chan + Lt + (lane & (Lt - 1)), true);                       \
        } else if ((T) == 5) {                                                             \
            lo = SP(6)[lane];                                                              \
            hi = SP(6)[32 + lane];                                                         \
        } else {                                                                           \
            lo = r[((T) + 1) % 6];                                                         \
            hi = __shfl_down_sync(FULL, r[((T) + 1) % 6], Lt);                              \
        }                                                                                  \
        const int psi = pl >> (T);                                                         \
        if (psi & 1) {                                                                     \
            const int boff = (psi - 1) << (T);                                             \
            uint32_t bwd;                                                                  \
            if (BREG) bwd = ((T) == 5 || !POLAR_BWPL) ? __shfl_sync(FULL, bw, boff >> 5) : bw_pl; \
            else bwd = beta[boff >> 5];                                                    \
            const uint32_t bit = (bwd >> (((boff & 31) + lane) & 31)) & 1u;                \
            r[T] = g_exact(lo, hi, bit);                                                   \
        } else {                                                                           \
            r[T] = f_minsum(lo, hi);                                                       \
        }                                                                                  \
        xr = r[T];                                                                         \
        if constexpr (CNT) c_fg += Lt;                                                     \
        if (lam == (T)) break;                                                             \
    }
                // register beta: the left siblings of the stages below 5 lie in node
                // j's own word (psi odd puts bit T of pl, T <= 4, inside it)
                const uint32_t bw_pl = (BREG && POLAR_BWPL && lam <= 5) ? __shfl_sync(FULL, bw, pl >> 5) : 0u;
                if constexpr (NL > 0) {
                    // shared-memory stages with compile-time sizes, then the register
                    // stages, in one cascade entered at s_hi
#define POLAR_SSTAGE(T)                                                                       \
    if constexpr ((T) < NL && (T) >= 6) {                                                     \
        if ((T) < lam) break;                                                                 \
        if constexpr (CNT) c_fg += 1u << (T);                                                 \
        alpha_stage<CHAN_SMEM, ((NL == 10 && SLOTS == 1) || (NL == 11 && POLAR_UNR_BIG)), BREG>((T) + 1 == n ? chan : SP((T) + 1), SP(T), beta, bw, n, (T), pl >> (T), lane); \
    }
                    switch (s_hi) {
                    case 12: POLAR_SSTAGE(12)
                    case 11: POLAR_SSTAGE(11)
                    case 10: POLAR_SSTAGE(10)
                    case 9: POLAR_SSTAGE(9)
                    case 8: POLAR_SSTAGE(8)
                    case 7: POLAR_SSTAGE(7)
                    case 6: POLAR_SSTAGE(6)
                        if (lam > 5) break;
                    case 5: POLAR_RSTAGE(5)
                    case 4: POLAR_RSTAGE(4)
                    case 3: POLAR_RSTAGE(3)
                    case 2: POLAR_RSTAGE(2)
                    case 1: POLAR_RSTAGE(1)
                    case 0: POLAR_RSTAGE(0)
                    default: break;
                    }
#undef POLAR_SSTAGE
                } else {
                    #pragma unroll 1
                    for (int s = s_hi; s >= max(lam, 6); s--) {
                        if constexpr (CNT) c_fg += 1u << s;
                        alpha_stage<CHAN_SMEM>(s + 1 == n ? chan : SP(s + 1), SP(s), beta, 0u, n, s, pl >> s, lane);
                    }
                    if (lam <= 5) {
                        switch (min(s_hi, 5)) {
                        case 5: POLAR_RSTAGE(5)
                        case 4: POLAR_RSTAGE(4)
                        case 3: POLAR_RSTAGE(3)
                        case 2: POLAR_RSTAGE(2)
                        case 1: POLAR_RSTAGE(1)
                        case 0: POLAR_RSTAGE(0)
                        default: break;
                        }
                    }
                }
#undef POLAR_RSTAGE
#ifdef POLAR_TRACE_FRAME
                if (f == POLAR_TRACE_FRAME) {
                    float v[8];
#pragma unroll
                    for (int q = 0; q < 8; q++) v[q] = __shfl_sync(FULL, xr, q);
                    if (lane == 0)
                        printf("TRACE   node kind %d lam %d phi %d pl %d s_min %d (lev_mem %d pos_mem %d s_d %d l %d) alpha %.9g %.9g %.9g %.9g %.9g %.9g %.9g %.9g\n",
                               kind, lam, pl >> lam, pl, s_min, lev_mem, pos_mem, s_d, l, v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]);
                }
#endif
                pos_mem = pl;
                lev_mem = lam + 1;
            }

            // ---- decision node ----------
            const int Lam = 1 << lam;
            if constexpr (CNT) c_ne += (uint32_t)Lam;
            const int seg = pl;
            float *a = SP(lam);               // node alpha (Lambda > 32)
            if (Lam <= 32) {
                if (MODE == 0 && lam == n) xr = ld1<CHAN_SMEM>(chan + (lane & (Lam - 1)), true);
                if (lane >= Lam) xr = 0.f;
            } else if (MODE == 0 && lam == n) {
                // whole code is one node: copy the channel so the sums can work in place
                #pragma unroll 1
                for (int i_0 = 0; i_0 < (N); i_0 += 32) if (const int i = i_0 + lane; i < (N)) alpha[i] = ld1<CHAN_SMEM>(chan + i, true);
                __syncwarp();
                a = alpha;
            }
            // Candidates in (dPM, mask) order (reading R7).  With
            // A0 <= A1 <= A2 <= A3 the order is fixed up to one comparison, because
            // round-to-nearest addition of non-negative values is monotone:
            //   R1:          masks 0, 1, 2, 3          (0, A0, A1, A0+A1)
            //   SPC, even:   0, 3, 5, 6|9, 9|6, 10, 12, 15  (6 = A1+A2, 9 = A0+A3)
            //   SPC, odd:    1, 2, 4, 7|8, 8|7, 11, 13, 14  (7 = A0+A1+A2, 8 = A3)
            // clist holds the masks in that order, 4 bits each.
            uint32_t clist = 0;
            int nc = 1;
            float vn = 0.f, vp = 0.f;
            float A[4] = {0.f, 0.f, 0.f, 0.f};
            uint32_t mi[4] = {0, 0, 0, 0};
            uint32_t hdw_node = 0;             // HD word of a Lambda <= 32 R1/SPC node
            const bool sum_kind = (kind == OP_R0 || kind == OP_REP);

            if (sum_kind) {
                // tree-order sums T(neg(a)) and T(pos(a)) (reading R3)
                const bool rep = (kind == OP_REP);
                if (Lam > 32) {
                    const int R = Lam >> 5, H = R >> 1;
                    #pragma unroll 1
                    for (int t = 0; t < H; t++) {        // first level, in place, lane-private columns
                        const float x = a[32 * t + lane], y = a[32 * (t + H) + lane];
                        a[32 * t + lane] = negpart(x) + negpart(y);
                        a[32 * (t + H) + lane] = pospart(x) + pospart(y);
                    }
                    #pragma unroll 1
                    for (int h = H >> 1; h >= 1; h >>= 1)
                        #pragma unroll 1
                        for (int t = 0; t < h; t++) {
                            a[32 * t + lane] += a[32 * (t + h) + lane];
                            if (rep) a[32 * (H + t) + lane] += a[32 * (H + t + h) + lane];
                        }
                    vn = a[lane];
                    vp = a[32 * H + lane];
                    #pragma unroll 1
                    for (int h = 16; h >= 1; h >>= 1) {
                        vn += __shfl_down_sync(FULL, vn, h);
                        vp += __shfl_down_sync(FULL, vp, h);
                    }
                    __syncwarp();
                } else {
                    vn = negpart(xr);
                    vp = pospart(xr);
                    // lanes >= Lambda hold +0 and x + 0 = x exactly, so the full
                    // five-level tree equals the Lambda-element tree-order sum
                    if constexpr (SUMF) {
#pragma unroll
                        for (int h = 16; h >= 1; h >>= 1) {
                            vn += __shfl_down_sync(FULL, vn, h);
                            if (rep) vp += __shfl_down_sync(FULL, vp, h);
                        }
                    } else {
                        #pragma unroll 1
                        for (int h = Lam >> 1; h >= 1; h >>= 1) {
                            vn += __shfl_down_sync(FULL, vn, h);
                            if (rep) vp += __shfl_down_sync(FULL, vp, h);
                        }
                    }
                }
                vn = __shfl_sync(FULL, vn, 0);
                vp = __shfl_sync(FULL, vp, 0);
                if (rep) { nc = 2; clist = (vp < vn) ? 0x01u : 0x10u; }   // ties: zeros first
            } else {
                // R1 / SPC: hard-decision word, parity, least reliable positions
                const int need = (kind == OP_SPC) ? 4 : 2;
                uint32_t par = 0;
                if (Lam > 32) {
                    unsigned long long t0 = ~0ull, t1 = ~0ull, t2 = ~0ull, t3 = ~0ull;
                    const int R = Lam >> 5;
                    #pragma unroll 1
                    for (int t = 0; t < R; t++) {
                        const float x = a[32 * t + lane];
                        const uint32_t b = __ballot_sync(FULL, x < 0.f);
                        if (BREG) { if (lane == (seg >> 5) + t) bw = b; }
                        else if (lane == (t & 31)) beta[(seg >> 5) + t] = b;
                        par ^= (uint32_t)__popc(b);
                        top4_insert(((unsigned long long)__float_as_uint(fabsf(x)) << 32) | (uint32_t)(32 * t + lane),
                                    t0, t1, t2, t3);
                    }
#pragma unroll
                    for (int r = 0; r < 4; r++) {
                        if (r < need) {
                            uint32_t mh, ml;
                            warp_min_key((uint32_t)(t0 >> 32), (uint32_t)t0, mh, ml);
                            mi[r] = ml;
                            A[r] = __uint_as_float(mh);
                            if ((uint32_t)t0 == ml && (uint32_t)(t0 >> 32) == mh) { t0 = t1; t1 = t2; t2 = t3; t3 = ~0ull; }
                        }
                    }
                } else {
                    hdw_node = __ballot_sync(FULL, lane < Lam && xr < 0.f);   // written with c1's flips below
                    par = (uint32_t)__popc(hdw_node);
                    // least reliable: the lane is the index, so ties go to the lowest lane
                    uint32_t key = (lane < Lam) ? __float_as_uint(fabsf(xr)) : 0xFFFFFFFFu;
#define POLAR_LR_ROUND(R)                                                       \
    {                                                                           \
        const uint32_t mh = __reduce_min_sync(FULL, key);                       \
        const int ml = __ffs(__ballot_sync(FULL, key == mh)) - 1;               \
        mi[R] = (uint32_t)ml;                                                   \
        A[R] = __uint_as_float(mh);                                             \
        if (lane == ml) key = 0xFFFFFFFFu;                                      \
    }
                    POLAR_LR_ROUND(0)
                    if (Lam > 1) {
                        POLAR_LR_ROUND(1)
                        if (kind == OP_SPC) { POLAR_LR_ROUND(2) POLAR_LR_ROUND(3) }
                    }
#undef POLAR_LR_ROUND
                }
                par &= 1u;
                if (kind == OP_R1) {
                    nc = (Lam == 1) ? 2 : 4;                // Lambda = 1: HD and its flip (reading R6)
                    clist = 0x3210u;
                } else {
                    nc = 8;
                    if (par == 0) clist = ((A[0] + A[3]) < (A[1] + A[2])) ? 0xFCA69530u : 0xFCA96530u;
                    else          clist = (A[3] < (A[0] + A[1]) + A[2]) ? 0xEDB78421u : 0xEDB87421u;
                }
                __syncwarp();
            }
            // lane r computes candidate r's mask and dPM (R0/REP: tree sums; R1/SPC:
            // the flipped |alpha|s summed in order m1, m2, m3, m4)
            const uint32_t my_m = (clist >> (4 * (lane & 7))) & 15u;
            float my_d = 0.f;
            if (sum_kind) {
                my_d = my_m ? vp : vn;
            } else {
                // 0 + x = x and d + 0 = d exactly (all terms >= +0), so this equals the
                // ordered sum of the flipped terms
#pragma unroll
                for (int q = 0; q < 4; q++) my_d = my_d + (((my_m >> q) & 1u) ? A[q] : 0.f);
            }

            // ---- c1 continues in the working memory ------------------------
            const int m0 = (int)(clist & 15u);
            if (BREG) {
                // c1's segment into this lane's word: new bits nb under mask lm
                const int ws = seg >> 5, o = seg & 31;
                uint32_t nb = 0, lm = 0;
                if (sum_kind) {
                    const uint32_t fill = (kind == OP_REP && m0) ? FULL : 0u;
                    if (Lam >= 32) { lm = (lane >= ws && lane < ws + (Lam >> 5)) ? FULL : 0u; nb = fill; }
                    else { lm = (lane == ws) ? ((1u << Lam) - 1u) << o : 0u; nb = fill; }
                } else if (Lam <= 32) {
                    uint32_t wv = hdw_node;                // HD word with c1's flips
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if ((m0 >> q) & 1) wv ^= 1u << mi[q];
                    const uint32_t wm = (Lam == 32) ? FULL : (1u << Lam) - 1u;
                    lm = (lane == ws) ? wm << o : 0u;
                    nb = (wv & wm) << o;
                } else {
                    // the HD words are in place: flip c1's positions
#pragma unroll
                    for (int q = 0; q < 4; q++) {
                        const int pos = seg + (int)mi[q];
                        if (((m0 >> q) & 1) && lane == (pos >> 5)) bw ^= 1u << (pos & 31);
                    }
                }
                bw = (bw & ~lm) | (nb & lm);
            } else {
                if (sum_kind) {
                    const uint32_t fill = (kind == OP_REP && m0) ? FULL : 0u;
                    if (Lam >= 32) {
                        #pragma unroll 1
                        for (int t_0 = 0; t_0 < ((Lam >> 5)); t_0 += 32) if (const int t = t_0 + lane; t < ((Lam >> 5))) beta[(seg >> 5) + t] = fill;
                    } else if (lane == 0) {
                        const uint32_t lm = ((1u << Lam) - 1u) << (seg & 31);
                        beta[seg >> 5] = (beta[seg >> 5] & ~lm) | (fill & lm);
                    }
                } else if (Lam <= 32) {
                    if (lane == 0) {                      // HD word with c1's flips, one RMW
                        uint32_t wv = hdw_node;
#pragma unroll
                        for (int q = 0; q < 4; q++)
                            if ((m0 >> q) & 1) wv ^= 1u << mi[q];
                        const uint32_t lm = (Lam == 32) ? FULL : (1u << Lam) - 1u;
                        const int w = seg >> 5, o = seg & 31;
                        beta[w] = (beta[w] & ~(lm << o)) | ((wv & lm) << o);
                    }
                } else if (lane == 0 && m0) {
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if ((m0 >> q) & 1) {
                            const int pos = seg + (int)mi[q];
                            beta[pos >> 5] ^= 1u << (pos & 31);
                        }
                }
                __syncwarp();
            }
            const int jn = j + 1, npl = (int)ra.y;
            const uint32_t ser0 = next_serial;
            next_serial += (uint32_t)nc;

            // c1 and the siblings that fit take free entries, in rank order, in one
            // step (p's entry was freed, so c1 always fits: reading R8).  The
            // siblings share one fork snapshot: beta prefix [0, npl) with c1's
            // segment, plus m1..m4 for the flip descriptors.
            int fslot = -1;
            const int nfit = min(nc, D - nS);
            auto write_fork_snapshot = [&](int victim_lane, int victim_slot) {
                if (BIG) fslot = alloc_snapshot_big(snap_used, uhint, sjsm, nA, D, hole >= 0 ? hole : victim_slot, PK::NONE, lane,
                                                    HOT, s_ser[0], s_jsm[0]);
                else fslot = alloc_snapshot_lazy<SL>(snap_used, NOSER ? s_pm : s_ser, s_jsm, D, victim_lane, victim_slot, SNAP_NONE, lane, nS);
                uint32_t *dst = snap_slot(fslot);
                const int nwords = (npl + 31) >> 5;
                if constexpr (CNT) c_sw += (uint32_t)nwords;
                if (BREG) { if (lane < nwords) dst[lane] = bw; }
                else {
                    #pragma unroll 1
                    for (int w_0 = 0; w_0 < (nwords); w_0 += 32) if (const int w = w_0 + lane; w < (nwords)) dst[w] = beta[w];
                }
                if (lane == 0) *hdr_at(fslot) = make_uint2(mi[0] | (mi[1] << 16), mi[2] | (mi[3] << 16));
            };
            if (!SORTED && nfit > 1) write_fork_snapshot(-1, -1);
            int c1_lane = 0, c1_slot = 0;
            if (HOT) {
                // candidates (ascending keys) with key <= cb merge into the hot
                // window (the SLOTS = 1 merge), the rest are appended to the cold
                // store; window positions >= 32 spill to the cold store, and cb
                // drops below the first spilled key.  Then the largest keys beyond D
                // are dropped (cold first: every cold key exceeds every hot key),
                // which with the merge keeps the D smallest keys (reading R8).  The
                // siblings' fork snapshot is taken whenever there are siblings.
                if (nc > 1) write_fork_snapshot(-1, -1);
                const uint32_t cpm = (lane < nc) ? __float_as_uint(p_pm + my_d) : EMPTY;
                const unsigned long long ckey = ((unsigned long long)cpm << 32) | (ser0 + (uint32_t)lane);
                const int nch = __popc(__ballot_sync(FULL, lane < nc && ckey <= cb));   // a prefix of the candidates
                const uint32_t cph = (lane < nch) ? cpm : EMPTY;
                const int totH = nH + nch;                 // <= 31 + 8
                const uint32_t jb = PK::make(jn, fslot >= 0 ? (uint32_t)fslot : PK::NONE, 0);
                uint32_t xpm = EMPTY, xser = EMPTY, xjsm = 0;   // this lane's position 32 + lane (spill)
                const uint32_t e1 = __shfl_sync(FULL, s_pm[0], 1), clast = __shfl_sync(FULL, cph, (nch - 1) & 7);
                if (POLAR_MERGE_FAST_HOT && nch > 0 && totH <= 32 && clast < e1) {
                    // the window candidates all precede its entries: a shift (no spill)
                    const int sh = nch - 1;
                    const uint32_t upm = __shfl_up_sync(FULL, s_pm[0], sh), user = __shfl_up_sync(FULL, s_ser[0], sh);
                    const uint32_t ujsm = __shfl_up_sync(FULL, s_jsm[0], sh);
                    const bool live = lane < totH, isC = lane < nch;
                    s_pm[0] = !live ? EMPTY : (isC ? cph : upm);
                    s_ser[0] = !live ? EMPTY : (isC ? ser0 + (uint32_t)lane : user);
                    s_jsm[0] = (live && isC) ? (jb | ((my_m ^ (uint32_t)m0) << PK::MSH)) : ujsm;
                } else {
                const uint32_t epm = s_pm[0];
                int a = 0;
                if (__shfl_sync(FULL, cph, 3) < epm) a = 4;
                if (__shfl_sync(FULL, cph, a + 1) < epm) a += 2;
                if (__shfl_sync(FULL, cph, a) < epm) a += 1;
                if (__shfl_sync(FULL, cph, a) < epm) a += 1;
                const int epos = lane - 1 + a;
                const bool ekeep = lane >= 1 && lane <= nH;
                const uint32_t M0 = __reduce_or_sync(FULL, (ekeep && epos < 32) ? (1u << epos) : 0u);
                const uint32_t M1 = (totH > 32) ? __reduce_or_sync(FULL, (ekeep && epos >= 32) ? (1u << (epos & 31)) : 0u) : 0u;
                const uint32_t opm = s_pm[0], oser = s_ser[0], ojsm = s_jsm[0];
#pragma unroll
                for (int w = 0; w < 2; w++) {
                    if (w == 1 && totH <= 32) break;       // nothing spills (the common case)
                    const uint32_t Mw = w ? M1 : M0;
                    const int Pp = 32 * w + lane;
                    const int q = (w ? __popc(M0) : 0) + __popc(Mw & ((1u << lane) - 1u));
                    const bool isE = (Mw >> lane) & 1u;
                    const int t = (Pp - q) & 7;
                    const int sl = (q + 1) & 31;
                    const uint32_t gpm = __shfl_sync(FULL, opm, sl), gser = __shfl_sync(FULL, oser, sl);
                    const uint32_t gjsm = __shfl_sync(FULL, ojsm, sl);
                    const uint32_t ct = __shfl_sync(FULL, cph, t);
                    const bool live = Pp < totH;
                    const uint32_t mk = (clist >> (4 * t)) & 15u;
                    const uint32_t vpm = !live ? EMPTY : (isE ? gpm : ct);
                    const uint32_t vser = !live ? EMPTY : (isE ? gser : ser0 + (uint32_t)t);
                    const uint32_t vjsm = (live && !isE) ? (jb | ((mk ^ (uint32_t)m0) << PK::MSH)) : gjsm;
                    if (w == 0) { s_pm[0] = vpm; s_ser[0] = vser; s_jsm[0] = vjsm; }
                    else { xpm = vpm; xser = vser; xjsm = vjsm; }
                }
                }
                const int nsp = max(totH - 32, 0);         // spilled window entries (lanes 0..nsp-1 of x*)
                nH = totH - nsp;
                int nwidx = -1;
                if (nsp > 0) {
                    if (lane < nsp) {
                        skey[nA + lane] = ((unsigned long long)xpm << 32) | xser;
                        sjsm[nA + lane] = xjsm;
                    }
                    const uint32_t sp0 = __shfl_sync(FULL, xpm, 0), ss0 = __shfl_sync(FULL, xser, 0);
                    cb = (((unsigned long long)sp0 << 32) | ss0) - 1ull;
                    const uint32_t wbb = __ballot_sync(FULL, lane < nsp && xser == ser0);
                    if (wbb) nwidx = nA + __ffs(wbb) - 1;
                }
                // candidates above cb: appended after the spilled entries
                const int nco = nc - nch;
                if (nco > 0) {
                    const int t = nch + lane;
                    const uint32_t cpt = __shfl_sync(FULL, cpm, t & 7);
                    if (lane < nco) {
                        const uint32_t mk = (clist >> (4 * t)) & 15u;
                        skey[nA + nsp + lane] = ((unsigned long long)cpt << 32) | (ser0 + (uint32_t)t);
                        sjsm[nA + nsp + lane] = jb | ((mk ^ (uint32_t)m0) << PK::MSH);
                    }
                    if (nch == 0) nwidx = nA + nsp;        // c1 itself went to the cold store
                }
                nA += nsp + nco;
                widx = nwidx;                              // -1: c1 is in the hot window
                nS = nH + nA;
                __syncwarp();
                // the D limit: drop the largest keys, cold first.  One scan keeps
                // each lane's two largest cold keys; with t = the largest of the
                // lanes' second keys, every cold key >= t is in those lists, so the
                // lists' maximum is extracted while it is >= t (a full stack drops
                // up to nc - 1 keys per pop with one scan, rarely two)
                #pragma unroll 1
                while (nS > D && nA > 0) {
                    unsigned long long k1 = 0, k2 = 0;
                    int i1 = -1, i2 = -1;
                    #pragma unroll 1
                    for (int i0 = 0; i0 < nA; i0 += 128) {
                        unsigned long long k4[4];
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            const int i = i0 + 32 * q + lane;
                            k4[q] = (i < nA) ? __ldcg(skey + i) : 0ull;
                        }
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            const int i = i0 + 32 * q + lane;
                            if (i < nA) {
                                if (i1 < 0 || k4[q] > k1) { k2 = k1; i2 = i1; k1 = k4[q]; i1 = i; }
                                else if (i2 < 0 || k4[q] > k2) { k2 = k4[q]; i2 = i; }
                            }
                        }
                    }
                    // t: the largest second key (lanes without one do not bound it)
                    const uint32_t th = __reduce_max_sync(FULL, i2 >= 0 ? (uint32_t)(k2 >> 32) : 0u);
                    const uint32_t tl = __reduce_max_sync(FULL, (i2 >= 0 && (uint32_t)(k2 >> 32) == th) ? (uint32_t)k2 : 0u);
                    const bool any2 = __any_sync(FULL, i2 >= 0);
                    const unsigned long long tk = any2 ? (((unsigned long long)th << 32) | tl) : 0ull;
                    int ndead = 0;
                    #pragma unroll 1
                    while (nS > D) {
                        const bool v = (i1 >= 0);
                        if (!__any_sync(FULL, v)) break;
                        const uint32_t mh = __reduce_max_sync(FULL, v ? (uint32_t)(k1 >> 32) : 0u);
                        const uint32_t ml = __reduce_max_sync(FULL, (v && (uint32_t)(k1 >> 32) == mh) ? (uint32_t)k1 : 0u);
                        const unsigned long long mk = ((unsigned long long)mh << 32) | ml;
                        if (any2 && mk < tk) break;            // below the lists' guarantee: rescan
                        const int ow = __ffs(__ballot_sync(FULL, v && k1 == mk)) - 1;
                        if (lane == ow) {
                            skey[i1] = ~0ull;                  // dropped: removed by the compaction below
                            if (widx == i1) widx = -2;         // (the working path: not live any more)
                            k1 = k2; i1 = i2; i2 = -1;
                        }
                        widx = __shfl_sync(FULL, widx, ow);
                        ndead++;
                        nS--;
                    }
                    __syncwarp();
                    int cntc = 0, nwidx = -1;
                    #pragma unroll 1
                    for (int i0 = 0; i0 < nA; i0 += 32) {
                        const int i = i0 + lane;
                        unsigned long long a = ~0ull;
                        uint32_t x = 0;
                        if (i < nA) { a = __ldcg(skey + i); x = __ldcg(sjsm + i); }
                        const bool keep = (a != ~0ull);
                        const uint32_t kb = __ballot_sync(FULL, keep);
                        const int o = cntc + __popc(kb & ((1u << lane) - 1u));
                        const uint32_t wbb = __ballot_sync(FULL, keep && i == widx);
                        if (wbb) nwidx = cntc + __popc(kb & ((1u << (__ffs(wbb) - 1)) - 1u));
                        __syncwarp();
                        if (keep) { skey[o] = a; sjsm[o] = x; }
                        cntc += __popc(kb);
                    }
                    widx = nwidx;
                    nA = cntc;
                    __syncwarp();
                    (void)ndead;
                }
                #pragma unroll 1
                while (nS > D) {                           // no cold entries left: the window's tail
                    if (lane == nH - 1) { s_pm[0] = EMPTY; s_ser[0] = EMPTY; }
                    nH--;
                    nS--;
                }
                if (nA == 0) cb = ~0ull;
            } else if (R0F && kind == OP_R0) {
                // one candidate (an R0 node), no sibling, no fork snapshot: the entries
                // whose PM is not above the candidate's (a prefix 1..k of the sorted
                // positions; ties keep the entry first, its serial is smaller) move
                // down by one, the candidate takes position k, the rest stay.  nS < D
                // after the pop, so nothing is dropped.
                const uint32_t c = __float_as_uint(p_pm + vn);     // (vn is warp-uniform)
                int k = 0;
#pragma unroll
                for (int q = 0; q < SL; q++) k += __popc(__ballot_sync(FULL, s_pm[q] <= c));   // dead entries hold EMPTY
                const uint32_t cj = PK::make(jn, PK::NONE, 0) | (NOSER ? WFLAG : 0u);
#pragma unroll
                for (int q = 0; q < SL; q++) {
                    uint32_t np = __shfl_down_sync(FULL, s_pm[q], 1), nj = __shfl_down_sync(FULL, s_jsm[q], 1);
                    uint32_t ns = NOSER ? 0u : __shfl_down_sync(FULL, s_ser[q], 1);
                    if (q + 1 < SL) {
                        const int q1 = (q + 1 < SL) ? q + 1 : q;
                        const uint32_t up = __shfl_sync(FULL, s_pm[q1], 0), uj = __shfl_sync(FULL, s_jsm[q1], 0);
                        const uint32_t us = NOSER ? 0u : __shfl_sync(FULL, s_ser[q1], 0);
                        np = (lane == 31) ? up : np; nj = (lane == 31) ? uj : nj; ns = (lane == 31) ? us : ns;
                    }
                    const int Pp = 32 * q + lane;
                    s_pm[q] = (Pp < k) ? np : ((Pp == k) ? c : s_pm[q]);
                    s_jsm[q] = (Pp < k) ? nj : ((Pp == k) ? cj : s_jsm[q]);
                    if constexpr (!NOSER) s_ser[q] = (Pp < k) ? ns : ((Pp == k) ? ser0 : s_ser[q]);
                }
                nS++;
            } else if (REPF && kind == OP_REP) {
                // two warp-uniform candidates c0 <= c1 (a REP node: all zeros / all ones).
                // k0, k1 = the entries not above c0, c1 (prefixes of the sorted
                // positions 1..nS).  New position P takes: old P + 1 for P < k0, c0 at
                // k0, old P for k0 < P <= k1, c1 at k1 + 1, old P - 1 above; positions
                // >= min(D, nS + 2) are dropped (c1 survives iff k1 + 1 < D).
                const uint32_t m0u = clist & 15u;
                const uint32_t c0 = __float_as_uint(p_pm + (m0u ? vp : vn)), c1 = __float_as_uint(p_pm + (m0u ? vn : vp));
                int k0 = 0, k1 = 0;
#pragma unroll
                for (int q = 0; q < SL; q++) {
                    k0 += __popc(__ballot_sync(FULL, s_pm[q] <= c0));      // dead entries hold EMPTY
                    k1 += __popc(__ballot_sync(FULL, s_pm[q] <= c1));
                }
                const int total = min(D, nS + 2);
                if (k1 + 1 < D) write_fork_snapshot(-1, -1);
                const uint32_t jb = PK::make(jn, fslot >= 0 ? (uint32_t)fslot : PK::NONE, 0);
                const uint32_t cj0 = jb | (NOSER ? WFLAG : 0u), cj1 = jb | (1u << PK::MSH);   // c1's flip: mask 0 ^ 1
                uint32_t ppm = EMPTY, pjs = 0, pse = EMPTY;      // the previous slot's old words
#pragma unroll
                for (int q = 0; q < SL; q++) {
                    const uint32_t opm = s_pm[q], ojs = s_jsm[q], ose = s_ser[q];
                    uint32_t dp = __shfl_down_sync(FULL, opm, 1), dj = __shfl_down_sync(FULL, ojs, 1);
                    uint32_t up = __shfl_up_sync(FULL, opm, 1), uj = __shfl_up_sync(FULL, ojs, 1);
                    uint32_t ds = NOSER ? 0u : __shfl_down_sync(FULL, ose, 1), us = NOSER ? 0u : __shfl_up_sync(FULL, ose, 1);
                    if (q + 1 < SL) {
                        const int q1 = (q + 1 < SL) ? q + 1 : q;
                        const uint32_t xp = __shfl_sync(FULL, s_pm[q1], 0), xj = __shfl_sync(FULL, s_jsm[q1], 0);
                        const uint32_t xs = NOSER ? 0u : __shfl_sync(FULL, s_ser[q1], 0);
                        dp = (lane == 31) ? xp : dp; dj = (lane == 31) ? xj : dj; ds = (lane == 31) ? xs : ds;
                    }
                    if (q > 0) {
                        const uint32_t xp = __shfl_sync(FULL, ppm, 31), xj = __shfl_sync(FULL, pjs, 31);
                        const uint32_t xs = NOSER ? 0u : __shfl_sync(FULL, pse, 31);
                        up = (lane == 0) ? xp : up; uj = (lane == 0) ? xj : uj; us = (lane == 0) ? xs : us;
                    }
                    const int Pp = 32 * q + lane;
                    const bool lo = Pp < k0, at0 = Pp == k0, mid = Pp <= k1, at1 = Pp == k1 + 1;
                    const uint32_t vpm = lo ? dp : (at0 ? c0 : (mid ? opm : (at1 ? c1 : up)));
                    s_pm[q] = (Pp < total) ? vpm : EMPTY;
                    s_jsm[q] = lo ? dj : (at0 ? cj0 : (mid ? ojs : (at1 ? cj1 : uj)));
                    if constexpr (!NOSER) {
                        const uint32_t vs = lo ? ds : (at0 ? ser0 : (mid ? ose : (at1 ? ser0 + 1u : us)));
                        s_ser[q] = (Pp < total) ? vs : EMPTY;
                    }
                    ppm = opm; pjs = ojs; pse = ose;
                }
                nS = total;
            } else if (SORTED && SL > 1) {
                // the same merge over SL slots (position p = 32 s + lane): entry p
                // moves to p - 1 + a_p, which stays in slots s - 1 .. s + 1
                const uint32_t cpm = (lane < nc) ? __float_as_uint(p_pm + my_d) : EMPTY;
#if POLAR_MERGE_FAST
                const uint32_t e1 = __shfl_sync(FULL, s_pm[0], 1), clast = __shfl_sync(FULL, cpm, (nc - 1) & 7);
                if (clast < e1) {
                    // every candidate ahead of every entry: candidates at 0..nc-1, the
                    // entries shift up by nc - 1 (slots descending: slot q reads the
                    // old slots q and q - 1)
                    const int total = min(D, nS + nc);
                    if (min(nc, D) > 1) write_fork_snapshot(-1, -1);
                    const uint32_t jb = jsm_make(jn, fslot >= 0 ? (uint32_t)fslot : SNAP_NONE, 0);
                    const int sh = nc - 1;
#pragma unroll
                    for (int q = SL - 1; q >= 0; q--) {
                        uint32_t vp = __shfl_up_sync(FULL, s_pm[q], sh), vs = __shfl_up_sync(FULL, s_ser[q], sh);
                        uint32_t vj = __shfl_up_sync(FULL, s_jsm[q], sh);
                        if (q > 0) {
                            const int qq = q > 0 ? q - 1 : 0, sl = (lane + 32 - sh) & 31;
                            const uint32_t yp = __shfl_sync(FULL, s_pm[qq], sl), ys = __shfl_sync(FULL, s_ser[qq], sl);
                            const uint32_t yj = __shfl_sync(FULL, s_jsm[qq], sl);
                            vp = (lane < sh) ? yp : vp; vs = (lane < sh) ? ys : vs; vj = (lane < sh) ? yj : vj;
                        }
                        const int Pp = 32 * q + lane;
                        const bool live = Pp < total, isC = Pp < nc;
                        s_pm[q] = !live ? EMPTY : (isC ? cpm : vp);
                        s_ser[q] = !live ? EMPTY : (isC ? ser0 + (uint32_t)lane : vs);
                        s_jsm[q] = (live && isC) ? (jb | ((my_m ^ (uint32_t)m0) << 21)) : vj;
                    }
                    nS = total;
                } else
#endif
                {
                const uint32_t c3 = __shfl_sync(FULL, cpm, 3);
                uint32_t Mw[SL];
#pragma unroll
                for (int w = 0; w < SL; w++) Mw[w] = 0u;
#pragma unroll
                for (int q = 0; q < SL; q++) {
                    const uint32_t epm = s_pm[q];
                    int a = (c3 < epm) ? 4 : 0;
                    if (__shfl_sync(FULL, cpm, a + 1) < epm) a += 2;
                    if (__shfl_sync(FULL, cpm, a) < epm) a += 1;
                    if (__shfl_sync(FULL, cpm, a) < epm) a += 1;
                    const int pos = 32 * q + lane;
                    const int epos = pos - 1 + a;
                    const bool ekeep = pos >= 1 && pos <= nS && epos < D;
#pragma unroll
                    for (int w = (q > 0 ? q - 1 : 0); w <= q + 1 && w < SL; w++)
                        Mw[w] |= (ekeep && (epos >> 5) == w) ? (1u << (epos & 31)) : 0u;
                }
                int nE = 0;
#pragma unroll
                for (int w = 0; w < SL; w++) { Mw[w] = __reduce_or_sync(FULL, Mw[w]); nE += __popc(Mw[w]); }
                const int total = min(D, nS + nc);
                if (total - nE > 1) write_fork_snapshot(-1, -1);
                const uint32_t jb = jsm_make(jn, fslot >= 0 ? (uint32_t)fslot : SNAP_NONE, 0);
                // gather, ascending output slots; slot w - 1's old entries are kept
                uint32_t opm = EMPTY, oser = EMPTY, ojsm = 0;
                int qbase = 0;
#pragma unroll
                for (int w = 0; w < SL; w++) {
                    const int P = 32 * w + lane;
                    const int q = qbase + __popc(Mw[w] & ((1u << lane) - 1u));   // entries before position P
                    const bool isE = (Mw[w] >> lane) & 1u;
                    const int t = (P - q) & 7;                                   // candidate at position P
                    const int src = q + 1, sv = src >> 5, sl = src & 31;
                    uint32_t gpm = __shfl_sync(FULL, s_pm[w], sl), gser = NOSER ? 0u : __shfl_sync(FULL, s_ser[w], sl);
                    uint32_t gjsm = __shfl_sync(FULL, s_jsm[w], sl);
                    if (w > 0) {
                        const uint32_t xp = __shfl_sync(FULL, opm, sl), xs = NOSER ? 0u : __shfl_sync(FULL, oser, sl);
                        const uint32_t xj = __shfl_sync(FULL, ojsm, sl);
                        gpm = (sv == w - 1) ? xp : gpm; gser = (sv == w - 1) ? xs : gser; gjsm = (sv == w - 1) ? xj : gjsm;
                    }
                    if (w + 1 < SL) {
                        const int w1 = (w + 1 < SL) ? w + 1 : w;
                        const uint32_t xp = __shfl_sync(FULL, s_pm[w1], 0), xs = NOSER ? 0u : __shfl_sync(FULL, s_ser[w1], 0);
                        const uint32_t xj = __shfl_sync(FULL, s_jsm[w1], 0);
                        gpm = (sv == w + 1) ? xp : gpm; gser = (sv == w + 1) ? xs : gser; gjsm = (sv == w + 1) ? xj : gjsm;
                    }
                    qbase += __popc(Mw[w]);
                    const uint32_t ct = __shfl_sync(FULL, cpm, t);
                    const bool live = P < total;
                    const uint32_t mk = (clist >> (4 * t)) & 15u;
                    opm = s_pm[w]; oser = s_ser[w]; ojsm = s_jsm[w];
                    s_pm[w] = !live ? EMPTY : (isE ? gpm : ct);
                    if constexpr (!NOSER) s_ser[w] = !live ? EMPTY : (isE ? gser : ser0 + (uint32_t)t);
                    const bool isC = live && !isE;
                    s_jsm[w] = isC ? (jb | ((mk ^ (uint32_t)m0) << 21) | (NOSER ? ((uint32_t)(t - 1) & WFLAG) : 0u)) : gjsm;
                }
                nS = total;
                }
            } else if (SORTED) {
                // merge the candidates into the sorted stack, keeping the D smallest
                // keys.  Equivalent to c1 always + siblings while |S| < D + strict-PM
                // replacement of the worst (reading R8): candidate
                // serials exceed every live serial, so "PM < worst PM" is "key <
                // worst key", and the sequential rule keeps the D smallest keys.
                // Entries: lanes 1..nS (sorted); candidate t: lane t, key ascending in t.
                // candidate keys; lanes nc..7 hold EMPTY (above every live key)
                const uint32_t cpm = (lane < nc) ? __float_as_uint(p_pm + my_d) : EMPTY;
                const uint32_t epm = s_pm[0];
                // every candidate ahead of every entry (the search continues along
                // the best path: the common case): candidates take positions
                // 0..nc-1, the entries shift up by nc - 1
#if POLAR_MERGE_FAST
                const uint32_t e1 = __shfl_sync(FULL, epm, 1), clast = __shfl_sync(FULL, cpm, (nc - 1) & 7);
                if (clast < e1) {
                    const int total = min(D, nS + nc);
                    if (min(nc, D) > 1) write_fork_snapshot(-1, -1);
                    const uint32_t jb = jsm_make(jn, fslot >= 0 ? (uint32_t)fslot : SNAP_NONE, 0);
                    const int sh = nc - 1;
                    const uint32_t upm = __shfl_up_sync(FULL, epm, sh), user = __shfl_up_sync(FULL, s_ser[0], sh);
                    const uint32_t ujsm = __shfl_up_sync(FULL, s_jsm[0], sh);
                    const bool live = lane < total, isC = lane < nc;
                    s_pm[0] = !live ? EMPTY : (isC ? cpm : upm);
                    s_ser[0] = !live ? EMPTY : (isC ? ser0 + (uint32_t)lane : user);
                    s_jsm[0] = (live && isC) ? (jb | ((my_m ^ (uint32_t)m0) << 21)) : ujsm;
                    nS = total;
                } else
#endif
                {
                // a = #{t < nc : cpm_t < epm} (candidate keys ascend: binary search
                // over 8 slots, no branch on nc)
                int a = 0;
                if (__shfl_sync(FULL, cpm, 3) < epm) a = 4;
                if (__shfl_sync(FULL, cpm, a + 1) < epm) a += 2;
                if (__shfl_sync(FULL, cpm, a) < epm) a += 1;
                if (__shfl_sync(FULL, cpm, a) < epm) a += 1;          // a <= 7 before this step
                const int epos = lane - 1 + a;                      // merged position of entry lane
                const bool ekeep = lane >= 1 && lane <= nS && epos < D;
                const uint32_t Mp = __reduce_or_sync(FULL, ekeep ? (1u << epos) : 0u);
                const int total = min(D, nS + nc);
                // siblings that survive share one fork snapshot (taken before the
                // merge, like the unsorted stack: slots of entries the merge drops
                // count as used here, and at least D - nS slots are free)
                if (total - __popc(Mp) > 1) write_fork_snapshot(-1, -1);
                const uint32_t jb = jsm_make(jn, fslot >= 0 ? (uint32_t)fslot : SNAP_NONE, 0);
                const int q = __popc(Mp & ((1u << lane) - 1u));      // entries before position lane
                const bool isE = (Mp >> lane) & 1u;
                const int t = (lane - q) & 7;                       // candidate at position lane
                const uint32_t gpm = __shfl_sync(FULL, epm, q + 1);
                const uint32_t gser = NOSER ? 0u : __shfl_sync(FULL, s_ser[0], q + 1);
                const uint32_t gjsm = __shfl_sync(FULL, s_jsm[0], q + 1);
                const uint32_t ct = __shfl_sync(FULL, cpm, t);      // candidate t's PM bits
                const bool live = lane < total;
                const uint32_t mk = (clist >> (4 * t)) & 15u;
                s_pm[0] = !live ? EMPTY : (isE ? gpm : ct);
                if constexpr (!NOSER) s_ser[0] = !live ? EMPTY : (isE ? gser : ser0 + (uint32_t)t);
                const bool isC = live && !isE;
                // (NOSER: candidate 0 = c1 becomes the working path: t - 1 = all ones only for t = 0)
                s_jsm[0] = isC ? (jb | ((mk ^ (uint32_t)m0) << 21) | (NOSER ? ((uint32_t)(t - 1) & WFLAG) : 0u)) : gjsm;
                nS = total;
                }
            } else if (BIG) {
                const uint32_t jbase = PK::make(jn, (nfit == 1) ? PK::NONE : (uint32_t)fslot, 0);
                // c1 refills the hole left by p (if any), the siblings are appended
                const int pos0 = (hole >= 0) ? hole : nA;
                const int posk = (lane == 0) ? pos0 : (hole >= 0 ? nA + lane - 1 : nA + lane);
                if (lane < nfit) {
                    const uint32_t mk = (clist >> (4 * lane)) & 15u;
                    kset(posk, ((unsigned long long)__float_as_uint(p_pm + my_d) << 32) | (ser0 + (uint32_t)lane));
                    sjsm[posk] = jbase | ((mk ^ (uint32_t)m0) << PK::MSH);
                }
                POLAR_DCHECK(nA + nfit - (hole >= 0 ? 1 : 0) <= D);
                c1_slot = pos0;
                widx = pos0;
                __syncwarp();
                nA += nfit - (hole >= 0 ? 1 : 0);
                hole = -1;
                nS += nfit;
            } else {
                int base = 0;
                const uint32_t jbase = jsm_make(jn, (nfit == 1) ? SNAP_NONE : (uint32_t)fslot, 0);
                uint32_t fbs[SL];
#pragma unroll
                for (int s = 0; s < SL; s++) {
                    const bool fr = (s_ser[s] == EMPTY);
                    const uint32_t fb = __ballot_sync(FULL, fr);
                    const int k = base + __popc(fb & ((1u << lane) - 1u));    // rank among free entries
                    const float dk = __shfl_sync(FULL, my_d, k & 7);
                    if (fr && k < nfit) {
                        const uint32_t mk = (clist >> (4 * k)) & 15u;
                        s_pm[s] = __float_as_uint(p_pm + dk);
                        s_ser[s] = ser0 + (uint32_t)k;
                        s_jsm[s] = jbase | ((mk ^ (uint32_t)m0) << 21);
                    }
                    fbs[s] = fb;
                    base += __popc(fb);
                }
                // c1 took the first free entry in (slot, lane) order; found with
                // selects only (a flag set inside the unrolled loop made ptxas
                // treat the SLOTS = 4 decode loop as divergent)
#pragma unroll
                for (int s = SL - 1; s >= 0; s--) {
                    c1_lane = fbs[s] ? __ffs(fbs[s]) - 1 : c1_lane;
                    c1_slot = fbs[s] ? s : c1_slot;
                }
                nS += nfit;
            }
            work = ser0;
            work_pl = npl;

            // the rest (stack full): replace the least reliable iff strictly better
            // (PAPER.md:L599).  Ranks ascend, so the first one dropped ends the loop.
            #pragma unroll 1
            for (int r = nfit; !SORTED && r < nc; r++) {
                const int mt = (int)((clist >> (4 * r)) & 15u);
                const float dt = __shfl_sync(FULL, my_d, r);
                const uint32_t cpm = __float_as_uint(p_pm + dt);
                uint32_t xpm = 0, xser = 0;
                int xs = -1;
                if (BIG) {
                    unsigned long long xk = 0;
                    #pragma unroll 1
                    for (int i_0 = 0; i_0 < (nA); i_0 += 32) if (const int i = i_0 + lane; i < (nA)) {
                        const unsigned long long k = kget(i);
                        if (xs < 0 || k > xk) { xk = k; xs = i; }
                    }
                    xpm = (uint32_t)(xk >> 32);
                    xser = (uint32_t)xk;
                } else {
#pragma unroll
                    for (int s = 0; s < SL; s++)
                        if (s_ser[s] != EMPTY && (xs < 0 || s_pm[s] > xpm || (s_pm[s] == xpm && s_ser[s] > xser))) { xpm = s_pm[s]; xser = s_ser[s]; xs = s; }
                }
                const uint32_t Mpm = __reduce_max_sync(FULL, xpm);
                if (cpm >= Mpm) break;                      // dropped, and so are the rest
                const uint32_t Mser = __reduce_max_sync(FULL, (xs >= 0 && xpm == Mpm) ? xser : 0u);
                const int tl = __ffs(__ballot_sync(FULL, xs >= 0 && xpm == Mpm && xser == Mser)) - 1;
                const int ts = __shfl_sync(FULL, xs, tl);
                if (fslot < 0) write_fork_snapshot(tl, ts);
                if (BIG) {
                    if (lane == 0) {
                        kset(ts, ((unsigned long long)cpm << 32) | (ser0 + (uint32_t)r));
                        sjsm[ts] = PK::make(jn, (uint32_t)fslot, (uint32_t)(mt ^ m0));
                    }
                    __syncwarp();
                } else if (lane == tl) {
#pragma unroll
                    for (int s = 0; s < SL; s++)
                        if (s == ts) {
                            s_pm[s] = cpm; s_ser[s] = ser0 + (uint32_t)r;
                            s_jsm[s] = jsm_make(jn, (uint32_t)fslot, (uint32_t)(mt ^ m0));
                        }
                }
            }
            if (GSCAN) {
                if (fslot >= 0 && lane == 0) sjsm[c1_slot] = PK::make(jn, (uint32_t)fslot, 0);
                __syncwarp();
            } else if (!SORTED && fslot >= 0) {
                // selects, not a lane branch around the writes (that branch made
                // ptxas treat the SLOTS = 4 decode loop as divergent)
                const uint32_t c1j = jsm_make(jn, (uint32_t)fslot, 0);
#pragma unroll
                for (int s = 0; s < SL; s++) s_jsm[s] = (lane == c1_lane && s == c1_slot) ? c1j : s_jsm[s];
            }
        }

        // ---- output: x_hat (systematic) or u_hat = x_hat F
        // (non-systematic) restricted to A, ascending ---------
        {
            if (BREG && !from_best) {         // (a complete path staged it already; the watchdog exit did not)
                if (lane < nw) beta[lane] = bw;
                __syncwarp();
            }
            const uint32_t *bsrc = from_best ? best : beta;
            if (MODE == 0 && P.nonsys) {
                #pragma unroll 1
                for (int w_0 = 0; w_0 < (nw); w_0 += 32) if (const int w = w_0 + lane; w < (nw)) uhat[w] = bsrc[w];
                __syncwarp();
                xform_words(uhat, N, nw, lane);
                bsrc = uhat;
            }
            uint8_t *ob = P.out_bits + (size_t)f * K;
            #pragma unroll 1
            for (int q_0 = 0; q_0 < (K); q_0 += 32) if (const int q = q_0 + lane; q < (K)) {
                const int idx = P.info[q];
                ob[q] = (uint8_t)((bsrc[idx >> 5] >> (idx & 31)) & 1u);
            }
            if (lane == 0) {
                if (P.pm) P.pm[f] = out_pm;
                if (P.pops) P.pops[f] = pops;
                if (P.switches) P.switches[f] = switches;
                if (P.status) P.status[f] = (uint8_t)status;
                if constexpr (CNT) {
                    uint4 cw;
                    cw.x = c_fg; cw.y = c_bb; cw.z = c_ne; cw.w = c_sw;
                    reinterpret_cast<uint4 *>(P.counts)[f] = cw;
                }
            }
            __syncwarp();
        }
        f = fnext;
        fnext = __shfl_sync(FULL, fnext2, 0);
    }
}

template <int SLOTS, bool SM, bool CS, int NL = 0, bool GA = false, int MODE = 0, bool CNT = false>
static cudaError_t launch_t(const DecodeParams &p, int ctas, int smem, cudaStream_t st) {
    auto kern = fsscs_decode_kernel<SLOTS, SM, CS, NL, GA, MODE, CNT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<ctas, kDecodeWarps * 32, smem, st>>>(p);
    return cudaGetLastError();
}

template <bool SM, bool CS>
static cudaError_t launch_s(const DecodeParams &p, int slots, int ctas, int smem, cudaStream_t st) {
    if (slots == 0) return launch_t<0, SM, CS>(p, ctas, smem, st);
    if (slots == 1) return launch_t<1, SM, CS>(p, ctas, smem, st);
    if (slots == 2) return launch_t<2, SM, CS>(p, ctas, smem, st);
    return launch_t<4, SM, CS>(p, ctas, smem, st);
}

// code-length-specialised instantiations: the BASELINE configs in the
// placements create() picks for them (n = 12 with the top alpha stage(s) in a
// global arena when that raises the occupancy: GA)
int specialised_nl(int n, int slots, bool snap_smem, bool chan_smem, bool recs_smem) {
    if (POLAR_RECS_SMEM && !recs_smem && slots != 0) return 0;
    if (n == 7 && slots == 1 && snap_smem && chan_smem) return 7;
    if (n == 10 && slots == 1 && !snap_smem && !chan_smem) return 10;
    if (n == 11 && slots == 2 && !snap_smem && !chan_smem) return 11;
    if (n == 12 && slots == 4 && !snap_smem && !chan_smem) return 12;
    if (n == 10 && slots == 0 && !snap_smem && !chan_smem) return 100;   // the paper's workload, D > 128
    return 0;
}

cudaError_t launch_decode(const DecodeParams &p, int slots, bool snap_smem, bool chan_smem, int ctas, int smem,
                          cudaStream_t st) {
    switch (specialised_nl(p.n, slots, snap_smem, chan_smem, p.sched_words > 0)) {
    case 7:
        if (p.c == 0 && !p.nonsys && p.M > 1) return launch_t<1, true, true, 7, false, 2>(p, ctas, smem, st);
        return launch_t<1, true, true, 7>(p, ctas, smem, st);
    case 10:
        if (p.c == 0 && !p.nonsys && p.M > 1) return launch_t<1, false, false, 10, false, 2>(p, ctas, smem, st);
        if (!p.nonsys && p.M > 1) return launch_t<1, false, false, 10, false, 1>(p, ctas, smem, st);
        return launch_t<1, false, false, 10>(p, ctas, smem, st);
    case 11:
        if (!p.nonsys && p.M > 1) return launch_t<2, false, false, 11, true, 1>(p, ctas, smem, st);
        return launch_t<2, false, false, 11, true>(p, ctas, smem, st);
    case 12:
        if (!p.nonsys && p.M > 1) return launch_t<4, false, false, 12, true, 1>(p, ctas, smem, st);
        return launch_t<4, false, false, 12, true>(p, ctas, smem, st);
    case 100:
        if (!p.nonsys && p.M > 1) return launch_t<0, false, false, 10, false, 1>(p, ctas, smem, st);
        return launch_t<0, false, false, 10>(p, ctas, smem, st);
    default: break;
    }
    if (snap_smem) return chan_smem ? launch_s<true, true>(p, slots, ctas, smem, st) : launch_s<true, false>(p, slots, ctas, smem, st);
    return chan_smem ? launch_s<false, true>(p, slots, ctas, smem, st) : launch_s<false, false>(p, slots, ctas, smem, st);
}

// polar_scs_decode_counts: the generic instance with CNT (placement from the
// parameters, any layout the handle chose)
cudaError_t launch_decode_counts(const DecodeParams &p, int slots, int ctas, int smem, cudaStream_t st) {
    if (slots == 0) return launch_t<0, false, false, 0, false, 0, true>(p, ctas, smem, st);
    if (slots == 1) return launch_t<1, false, false, 0, false, 0, true>(p, ctas, smem, st);
    if (slots == 2) return launch_t<2, false, false, 0, false, 0, true>(p, ctas, smem, st);
    return launch_t<4, false, false, 0, false, 0, true>(p, ctas, smem, st);
}

template <int S, bool B, bool C, int NL = 0, bool GA = false, int MODE = 0>
static cudaError_t occ_t(int smem, int *blocks) {
    cudaError_t e = cudaFuncSetAttribute(fsscs_decode_kernel<S, B, C, NL, GA, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fsscs_decode_kernel<S, B, C, NL, GA, MODE>, kDecodeWarps * 32, smem);
}
template <bool B, bool C>
static cudaError_t occ_s(int slots, int smem, int *blocks) {
    if (slots == 0) return occ_t<0, B, C>(smem, blocks);
    if (slots == 1) return occ_t<1, B, C>(smem, blocks);
    if (slots == 2) return occ_t<2, B, C>(smem, blocks);
    return occ_t<4, B, C>(smem, blocks);
}

cudaError_t decode_occupancy(int n, int slots, bool snap_smem, bool chan_smem, int mode, bool recs_smem, int smem,
                             int *blocks_per_sm) {
    switch (specialised_nl(n, slots, snap_smem, chan_smem, recs_smem)) {
    case 7: return mode == 2 ? occ_t<1, true, true, 7, false, 2>(smem, blocks_per_sm) : occ_t<1, true, true, 7>(smem, blocks_per_sm);
    case 10: return mode == 2 ? occ_t<1, false, false, 10, false, 2>(smem, blocks_per_sm)
                  : mode == 1 ? occ_t<1, false, false, 10, false, 1>(smem, blocks_per_sm)
                              : occ_t<1, false, false, 10>(smem, blocks_per_sm);
    case 11: return mode >= 1 ? occ_t<2, false, false, 11, true, 1>(smem, blocks_per_sm)
                              : occ_t<2, false, false, 11, true>(smem, blocks_per_sm);
    case 12: return mode >= 1 ? occ_t<4, false, false, 12, true, 1>(smem, blocks_per_sm)
                              : occ_t<4, false, false, 12, true>(smem, blocks_per_sm);
    case 100: return mode >= 1 ? occ_t<0, false, false, 10, false, 1>(smem, blocks_per_sm)
                               : occ_t<0, false, false, 10>(smem, blocks_per_sm);
    default: break;
    }
    if (snap_smem) return chan_smem ? occ_s<true, true>(slots, smem, blocks_per_sm) : occ_s<true, false>(slots, smem, blocks_per_sm);
    return chan_smem ? occ_s<false, true>(slots, smem, blocks_per_sm) : occ_s<false, false>(slots, smem, blocks_per_sm);
}

}  // namespace polar

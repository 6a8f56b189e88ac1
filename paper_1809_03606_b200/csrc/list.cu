// list.cu — the FSSCL list decoder kernel for sm_100a (PAPER.md:L505-587,
// §2.2.3-2.2.4; memory per §3.2).
//
// One CTA decodes one frame at a time with L warps: warp w holds the path of
// rank w of the list.  All paths advance in lock-step through the FSSC
// schedule ("realized in the same manner as ... FSSC"); at every
// decision node (R0 included, reading R23) each path builds its node
// candidates (the FSSCL rules, L526-585, identical to the stack decoder's) and
// the CTA keeps the L smallest keys (PM, parent rank, candidate rank)
// (L507; reading R22), in key order, so rank r lands in warp r.
//
// Memory (LLR-domain lazy copy, L774-776): alpha stage s >= 6 has L buffers
// of 2^s floats in shared memory; a path owns "home" buffer w of every stage
// and inherits the buffers of stages above its next descent from its parent
// by reference (a 5-bit pointer per stage, packed in one u64 per path).  A
// descent rewrites every stage it touches into home buffers, and the stages it
// reads from are never written by anyone during that descent, so no alpha is
// ever copied.  Stages 0..5 (Lambda <= 32) live in registers (element i in
// lane i) and are handed to children through a 64-float shared-memory slot per
// path.  The flat N-bit beta is per path and double-buffered
// by node parity: a child copies its parent's prefix [0, PL) and applies its
// own flips.  Everything a child reads from its parent is double-buffered by
// node parity, so two __syncthreads per node suffice.
//
// Arithmetic and candidate order follow the oracle (O11) exactly: float32,
// -fmad=false, tree-order sums, (|alpha| bits, index) argmin keys.
#include <cuda_runtime.h>

#include "device_common.cuh"

namespace polar {

namespace {

// 5-bit buffer index of stage s (>= 6) in a path's pointer row
__device__ __forceinline__ int prow_get(unsigned long long row, int s) { return (int)((row >> (5 * (s - 6))) & 31ull); }
__device__ __forceinline__ unsigned long long prow_set(unsigned long long row, int s, int k) {
    const int sh = 5 * (s - 6);
    return (row & ~(31ull << sh)) | ((unsigned long long)k << sh);
}

// ALPHA(s, psi) for a shared-memory stage (Lambda = 2^s >= 64): dst from src
// (the parent stage s+1, or the channel row), f for even psi, g for odd psi
// with the left sibling's segment of the path's flat beta (Eq. 4).
__device__ __forceinline__ void list_alpha_stage(const float *src, bool src_global, float *dst, const uint32_t *beta,
                                                 int s, int psi, int lane) {
    const int Ls = 1 << s;
    const bool odd = (psi & 1) != 0;
    const int boff = (psi - 1) << s;
    #pragma unroll 1
    for (int i = lane * 2; i < Ls; i += 64) {
        float2 lo, hi;
        if (src_global) {
            lo = __ldg(reinterpret_cast<const float2 *>(src + i));
            hi = __ldg(reinterpret_cast<const float2 *>(src + Ls + i));
        } else {
            lo = *reinterpret_cast<const float2 *>(src + i);
            hi = *reinterpret_cast<const float2 *>(src + Ls + i);
        }
        float2 o;
        if (odd) {
            const uint32_t b = beta[(boff + i) >> 5] >> ((boff + i) & 31);
            o.x = g_exact(lo.x, hi.x, b & 1u);
            o.y = g_exact(lo.y, hi.y, (b >> 1) & 1u);
        } else {
            o.x = f_minsum(lo.x, hi.x);
            o.y = f_minsum(lo.y, hi.y);
        }
        *reinterpret_cast<float2 *>(dst + i) = o;
    }
    __syncwarp();
}

}  // namespace

// NL > 0: compile-time code length 2^NL (the BASELINE codes), else any N.
template <int LCAP, int NL = 0>
__global__ void __launch_bounds__(LCAP * 32) fsscl_decode_kernel(const ListParams P) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int tid = threadIdx.x;
    const int n = (NL > 0) ? NL : P.n, N = 1 << n, nw = (NL > 0) ? (NL >= 5 ? (1 << NL) / 32 : 1) : P.nw;
    const int L = P.L, M = P.M, K = P.K;

    uint32_t *nodes_s = smem;                                         // [M]
    float *abuf = reinterpret_cast<float *>(smem + P.o_alpha);         // stage s: L buffers of 2^s at L(2^s - 64)
    uint32_t *betaA = smem + P.o_beta;                                 // [2][L][nw]
    float *regst = reinterpret_cast<float *>(smem + P.o_reg);          // [2][L][64]: stage s at [2^s, 2^{s+1})
    uint32_t *clist_s = smem + P.o_clist;                              // [2][L]
    uint2 *mi_s = reinterpret_cast<uint2 *>(smem + P.o_mi);            // [2][L]
    unsigned long long *prow_s = reinterpret_cast<unsigned long long *>(smem + P.o_prow);  // [2][L]
    unsigned long long *cand_s = reinterpret_cast<unsigned long long *>(smem + P.o_cand);  // [8L]
    uint32_t *sel_s = smem + P.o_sel;                                  // [L]
    float *selpm_s = reinterpret_cast<float *>(smem + P.o_selpm);      // [L]
    uint32_t *ok_s = smem + P.o_ok;                                    // [L]
    unsigned long long *misc = reinterpret_cast<unsigned long long *>(smem + P.o_misc);  // [2] frame slots

    #pragma unroll 1
    for (int i = tid; i < M; i += blockDim.x) nodes_s[i] = P.nodes[i];
    auto stage_buf = [&](int s, int k) -> float * { return abuf + (size_t)L * ((1 << s) - 64) + (size_t)k * (1 << s); };
    auto beta_of = [&](int par, int k) -> uint32_t * { return betaA + (size_t)(par * L + k) * nw; };

    const unsigned long long nfr = (unsigned long long)P.n_frames;
    if (tid == 0) misc[0] = atomicAdd(P.queue, 1ull);
    __syncthreads();
    int slot = 0;
    unsigned long long f = misc[0];

    #pragma unroll 1
    while (f < nfr) {
        // claim the next frame (read after this frame's last barrier) and
        // prefetch its LLR row into L2
        if (w == 0) {
            unsigned long long fn = 0;
            if (lane == 0) { fn = atomicAdd(P.queue, 1ull); misc[slot ^ 1] = fn; }
            fn = __shfl_sync(FULL, fn, 0);
            if (fn < nfr) {
                const char *nr = reinterpret_cast<const char *>(P.llr + (size_t)fn * N);
                #pragma unroll 1
                for (int b = lane * 128; b < N * 4; b += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(nr + b));
            }
        }
        const float *chan = P.llr + (size_t)f * N;

        int nL = 1;                   // live paths (uniform)
        int par = 0;                  // node parity: selects the double-buffered areas
        float my_pm = 0.f;            // PM of this warp's path
        unsigned long long myrow = 0; // alpha buffer of every shared-memory stage
        int pos_mem = 0, lev_mem = n; // alpha stages >= lev_mem hold node (s, pos_mem >> s)
        float r[6];
#pragma unroll
        for (int t = 0; t < 6; t++) r[t] = 0.f;

        #pragma unroll 1
        for (int j = 0; j <= M; j++) {
            const bool live = (w < nL);
            uint32_t *beta = beta_of(par, w);
            // position after node j-1 and its pending BETA climb (L852)
            int pl = 0, l = n;
            if (j > 0) {
                const uint32_t pn = nodes_s[j - 1];
                const int plam = (int)op_lam(pn), pphi = (int)op_phi(pn);
                pl = (pphi + 1) << plam;
                int ph = pphi;
                l = plam;
                if (live && (ph & 1) && l < 5) {
                    const int wd = ((ph - 1) << l) >> 5;
                    uint32_t x = beta[wd];
                    #pragma unroll 1
                    while ((ph & 1) && l < 5) {
                        const int o = ((ph - 1) << l) & 31, Lm = 1 << l;
                        x ^= ((x >> (o + Lm)) & ((1u << Lm) - 1u)) << o;
                        ph >>= 1;
                        l++;
                    }
                    if (lane == 0) beta[wd] = x;
                    __syncwarp();
                }
                #pragma unroll 1
                while (ph & 1) {
                    if (live) beta_op(beta, l, ph, lane);
                    ph >>= 1;
                    l++;
                }
            }
            if (j == M) break;

            const uint32_t nd = nodes_s[j];
            const int kind = (int)op_kind(nd), lam = (int)op_lam(nd), phi = (int)op_phi(nd);
            const int Lam = 1 << lam;
            const int seg = phi << lam;
            const int nc = (kind == OP_R0) ? 1 : (kind == OP_REP ? 2 : (kind == OP_R1 ? (Lam == 1 ? 2 : 4) : 8));
            const int s_hi = min(max(max(lev_mem, bitlen((uint32_t)(pos_mem ^ pl))), l + 1), n) - 1;

            if (live) {
                // ---- ALPHA ops down to the node (Eq. 4, Alg. 1)
                float xr = 0.f;
                #pragma unroll 1
                for (int s = s_hi; s >= max(lam, 6); s--) {
                    const bool top = (s + 1 == n);
                    const float *src = top ? chan : stage_buf(s + 1, prow_get(myrow, s + 1));
                    list_alpha_stage(src, top, stage_buf(s, w), beta, s, pl >> s, lane);
                    myrow = prow_set(myrow, s, w);
                }
#define POLAR_LSTAGE(T)                                                                    \
    {                                                                                      \
        const int Lt = 1 << (T);                                                           \
        float lo, hi;                                                                      \
        if ((T) + 1 == n) {                                                                \
            lo = __ldg(chan + (lane & (Lt - 1)));                                          \
            hi = __ldg(chan + Lt + (lane & (Lt - 1)));                                     \
        } else if ((T) == 5) {                                                             \
            const float *s6 = stage_buf(6, prow_get(myrow, 6));                            \
            lo = s6[lane];                                                                 \
            hi = s6[32 + lane];                                                            \
        } else {                                                                           \
            lo = r[((T) + 1) % 6];                                                         \
            hi = __shfl_down_sync(FULL, r[((T) + 1) % 6], Lt);                              \
        }                                                                                  \
        const int psi = pl >> (T);                                                         \
        if (psi & 1) {                                                                     \
            const int boff = (psi - 1) << (T);                                             \
            const uint32_t bit = (beta[boff >> 5] >> (((boff & 31) + lane) & 31)) & 1u;     \
            r[T] = g_exact(lo, hi, bit);                                                   \
        } else {                                                                           \
            r[T] = f_minsum(lo, hi);                                                       \
        }                                                                                  \
        xr = r[T];                                                                         \
        if (lam == (T)) break;                                                             \
    }
                if (lam <= 5) {
                    switch (min(s_hi, 5)) {
                    case 5: POLAR_LSTAGE(5)
                    case 4: POLAR_LSTAGE(4)
                    case 3: POLAR_LSTAGE(3)
                    case 2: POLAR_LSTAGE(2)
                    case 1: POLAR_LSTAGE(1)
                    case 0: POLAR_LSTAGE(0)
                    default: break;
                    }
                }
#undef POLAR_LSTAGE

                // ---- node candidates, in (dPM, mask) order
                float *a = (lam < n && lam >= 6) ? stage_buf(lam, w) : nullptr;
                if (Lam <= 32) {
                    if (lam == n) xr = __ldg(chan + (lane & (Lam - 1)));
                    if (lane >= Lam) xr = 0.f;
                } else if (lam == n) {
                    // the whole code is one node: private scratch of N floats
                    a = abuf + (size_t)w * N;
                    #pragma unroll 1
                    for (int i = lane; i < N; i += 32) a[i] = __ldg(chan + i);
                    __syncwarp();
                }
                uint32_t clist = 0;
                float vn = 0.f, vp = 0.f;
                float A[4] = {0.f, 0.f, 0.f, 0.f};
                uint32_t mi[4] = {0, 0, 0, 0};
                uint32_t hdw_node = 0;
                const bool sum_kind = (kind == OP_R0 || kind == OP_REP);
                if (sum_kind) {
                    const bool rep = (kind == OP_REP);
                    if (Lam > 32) {
                        const int R = Lam >> 5, H = R >> 1;
                        #pragma unroll 1
                        for (int t = 0; t < H; t++) {
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
                        #pragma unroll 1
                        for (int h = Lam >> 1; h >= 1; h >>= 1) {
                            vn += __shfl_down_sync(FULL, vn, h);
                            if (rep) vp += __shfl_down_sync(FULL, vp, h);
                        }
                    }
                    vn = __shfl_sync(FULL, vn, 0);
                    vp = __shfl_sync(FULL, vp, 0);
                    if (rep) clist = (vp < vn) ? 0x01u : 0x10u;     // ties: zeros first
                } else {
                    const int need = (kind == OP_SPC) ? 4 : 2;
                    uint32_t parity = 0;
                    if (Lam > 32) {
                        unsigned long long t0 = ~0ull, t1 = ~0ull, t2 = ~0ull, t3 = ~0ull;
                        const int R = Lam >> 5;
                        #pragma unroll 1
                        for (int t = 0; t < R; t++) {
                            const float x = a[32 * t + lane];
                            const uint32_t b = __ballot_sync(FULL, x < 0.f);
                            if (lane == (t & 31)) beta[(seg >> 5) + t] = b;
                            parity ^= (uint32_t)__popc(b);
                            top4_insert(((unsigned long long)__float_as_uint(fabsf(x)) << 32) | (uint32_t)(32 * t + lane),
                                        t0, t1, t2, t3);
                        }
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < need) {
                                uint32_t mh, ml;
                                warp_min_key((uint32_t)(t0 >> 32), (uint32_t)t0, mh, ml);
                                mi[q] = ml;
                                A[q] = __uint_as_float(mh);
                                if ((uint32_t)t0 == ml && (uint32_t)(t0 >> 32) == mh) { t0 = t1; t1 = t2; t2 = t3; t3 = ~0ull; }
                            }
                        }
                    } else {
                        hdw_node = __ballot_sync(FULL, lane < Lam && xr < 0.f);
                        parity = (uint32_t)__popc(hdw_node);
                        uint32_t key = (lane < Lam) ? __float_as_uint(fabsf(xr)) : 0xFFFFFFFFu;
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < need && q < Lam) {
                                const uint32_t mh = __reduce_min_sync(FULL, key);
                                const int ml = __ffs(__ballot_sync(FULL, key == mh)) - 1;
                                mi[q] = (uint32_t)ml;
                                A[q] = __uint_as_float(mh);
                                if (lane == ml) key = 0xFFFFFFFFu;
                            }
                        }
                    }
                    parity &= 1u;
                    if (kind == OP_R1) {
                        clist = 0x3210u;
                    } else {
                        if (parity == 0) clist = ((A[0] + A[3]) < (A[1] + A[2])) ? 0xFCA69530u : 0xFCA96530u;
                        else             clist = (A[3] < (A[0] + A[1]) + A[2]) ? 0xEDB78421u : 0xEDB87421u;
                    }
                    __syncwarp();
                }
                // lane r: candidate r's mask and dPM
                const uint32_t my_m = (clist >> (4 * (lane & 7))) & 15u;
                float my_d = 0.f;
                if (sum_kind) {
                    my_d = my_m ? vp : vn;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; q++) my_d = my_d + (((my_m >> q) & 1u) ? A[q] : 0.f);
                }
                // the segment with c1's bits in this path's beta (children flip from it)
                const int m0 = (int)(clist & 15u);
                if (sum_kind) {
                    const uint32_t fill = (kind == OP_REP && m0) ? FULL : 0u;
                    if (Lam >= 32) {
                        #pragma unroll 1
                        for (int t = lane; t < (Lam >> 5); t += 32) beta[(seg >> 5) + t] = fill;
                    } else if (lane == 0) {
                        const uint32_t lm = ((1u << Lam) - 1u) << (seg & 31);
                        beta[seg >> 5] = (beta[seg >> 5] & ~lm) | (fill & lm);
                    }
                } else if (Lam <= 32) {
                    if (lane == 0) {
                        uint32_t wv = hdw_node;
#pragma unroll
                        for (int q = 0; q < 4; q++)
                            if ((m0 >> q) & 1) wv ^= 1u << mi[q];
                        const uint32_t lm = (Lam == 32) ? FULL : (1u << Lam) - 1u;
                        const int wd = seg >> 5, o = seg & 31;
                        beta[wd] = (beta[wd] & ~(lm << o)) | ((wv & lm) << o);
                    }
                } else if (lane == 0 && m0) {
#pragma unroll
                    for (int q = 0; q < 4; q++)
                        if ((m0 >> q) & 1) {
                            const int pos = seg + (int)mi[q];
                            beta[pos >> 5] ^= 1u << (pos & 31);
                        }
                }
                // ---- publish: candidate keys (PM, parent rank, candidate rank),
                // the flip descriptor, the alpha pointer row and register stages
                if (lane < nc)
                    cand_s[w * nc + lane] = ((unsigned long long)__float_as_uint(my_pm + my_d) << 32) |
                                            (uint32_t)((w << 3) | lane);
                if (lane == 0) {
                    clist_s[par * L + w] = clist;
                    mi_s[par * L + w] = make_uint2(mi[0] | (mi[1] << 16), mi[2] | (mi[3] << 16));
                    prow_s[par * L + w] = myrow;
                }
                float *rs = regst + (size_t)(par * L + w) * 64;
#pragma unroll
                for (int t = 0; t < 6; t++)
                    if (lane < (1 << t)) rs[(1 << t) + lane] = r[t];
            }
            pos_mem = pl;
            lev_mem = lam + 1;
            __syncthreads();

            // ---- prune to the L best keys (reading R22): rank by
            // counting (every thread reads the same key at a time: smem broadcast)
            const int total = nL * nc;
            if (tid < total) {
                const unsigned long long key = cand_s[tid];
                int rank = 0;
                #pragma unroll 4
                for (int u = 0; u < total; u++) rank += (cand_s[u] < key) ? 1 : 0;
                if (rank < L) {
                    sel_s[rank] = (uint32_t)key;
                    selpm_s[rank] = __uint_as_float((uint32_t)(key >> 32));
                }
            }
            __syncthreads();

            // ---- rank w takes its parent's state (lazy copy: beta prefix, pointers)
            const int nL2 = min(total, L);
            const int npar = par ^ 1;
            if (w < nL2) {
                const uint32_t sv = sel_s[w];
                const int p = (int)(sv >> 3), rk = (int)(sv & 7u);
                my_pm = selpm_s[w];
                const uint32_t *src = beta_of(par, p);
                uint32_t *dst = beta_of(npar, w);
                const int npl = (phi + 1) << lam;
                #pragma unroll 1
                for (int q = lane; q < ((npl + 31) >> 5); q += 32) dst[q] = src[q];
                __syncwarp();
                const uint32_t cl = clist_s[par * L + p];
                const uint32_t rel = ((cl >> (4 * rk)) & 15u) ^ (cl & 15u);
                if (rel) {
                    if (kind == OP_REP) {
                        if (Lam >= 32) {
                            #pragma unroll 1
                            for (int t = lane; t < (Lam >> 5); t += 32) dst[(seg >> 5) + t] ^= FULL;
                        } else if (lane == 0) {
                            dst[seg >> 5] ^= ((1u << Lam) - 1u) << (seg & 31);
                        }
                    } else if (lane == 0) {
                        const uint2 hh = mi_s[par * L + p];
                        const uint32_t m4[4] = {hh.x & 0xFFFFu, hh.x >> 16, hh.y & 0xFFFFu, hh.y >> 16};
#pragma unroll
                        for (int q = 0; q < 4; q++)
                            if ((rel >> q) & 1u) {
                                const int pos = seg + (int)m4[q];
                                dst[pos >> 5] ^= 1u << (pos & 31);
                            }
                    }
                }
                myrow = prow_s[par * L + p];
                const float *rs = regst + (size_t)(par * L + p) * 64;
#pragma unroll
                for (int t = 0; t < 6; t++) r[t] = (lane < (1 << t)) ? rs[(1 << t) + lane] : 0.f;
                __syncwarp();
            }
            par = npar;
            nL = nL2;
        }

        // ---- final selection (reading R24): CRC of every path
        const bool live = (w < nL);
        uint32_t *beta = beta_of(par, w);
        uint32_t *scratch = beta_of(par ^ 1, w);       // free at this point
        const uint32_t *cw = beta;
        if (live && (P.nonsys)) {
            #pragma unroll 1
            for (int q = lane; q < nw; q += 32) scratch[q] = beta[q];
            __syncwarp();
            xform_words(scratch, N, nw, lane);
            cw = scratch;
        }
        if (live) {
            bool ok = true;
            if (P.c > 0) {
                uint32_t syn = 0;
                #pragma unroll 1
                for (int q = lane; q < nw; q += 32) {
                    const uint32_t x = cw[q];
                    const uint32_t *tw = P.crc_bytes + (size_t)q * 1024;
                    syn ^= __ldg(tw + (x & 255u)) ^ __ldg(tw + 256 + ((x >> 8) & 255u)) ^
                           __ldg(tw + 512 + ((x >> 16) & 255u)) ^ __ldg(tw + 768 + (x >> 24));
                }
                syn = __reduce_xor_sync(FULL, syn);
                ok = (syn == 0);
            }
            if (lane == 0) ok_s[w] = ok ? 1u : 0u;
        }
        __syncthreads();
        int pick = 0, status = 1;
        for (int q = 0; q < nL; q++)
            if (ok_s[q]) { pick = q; status = 0; break; }
        if (w == pick) {
            uint8_t *ob = P.out_bits + (size_t)f * K;
            #pragma unroll 1
            for (int q = lane; q < K; q += 32) {
                const int idx = P.info[q];
                ob[q] = (uint8_t)((cw[idx >> 5] >> (idx & 31)) & 1u);
            }
            if (lane == 0) {
                if (P.pm) P.pm[f] = my_pm;
                if (P.status) P.status[f] = (uint8_t)status;
            }
        }
        __syncthreads();          // misc[slot ^ 1] is visible; every read of this frame's state is done
        slot ^= 1;
        f = misc[slot];
    }
}

template <int LCAP, int NL = 0>
static cudaError_t launch_list_t(const ListParams &p, int ctas, int smem, cudaStream_t st) {
    auto kern = fsscl_decode_kernel<LCAP, NL>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<ctas, p.L * 32, smem, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_list(const ListParams &p, int lcap, int ctas, int smem, cudaStream_t st) {
    if (lcap == 8 && p.n == 10) return launch_list_t<8, 10>(p, ctas, smem, st);
    if (lcap == 8 && p.n == 7) return launch_list_t<8, 7>(p, ctas, smem, st);
    if (lcap == 16 && p.n == 11) return launch_list_t<16, 11>(p, ctas, smem, st);
    switch (lcap) {
    case 8: return launch_list_t<8>(p, ctas, smem, st);
    case 16: return launch_list_t<16>(p, ctas, smem, st);
    default: return launch_list_t<32>(p, ctas, smem, st);
    }
}

template <int LCAP, int NL = 0>
static cudaError_t list_occ_t(int L, int smem, int *blocks) {
    cudaError_t e = cudaFuncSetAttribute(fsscl_decode_kernel<LCAP, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fsscl_decode_kernel<LCAP, NL>, L * 32, smem);
}

cudaError_t list_occupancy(int lcap, int n, int L, int smem, int *blocks_per_sm) {
    if (lcap == 8 && n == 10) return list_occ_t<8, 10>(L, smem, blocks_per_sm);
    if (lcap == 8 && n == 7) return list_occ_t<8, 7>(L, smem, blocks_per_sm);
    if (lcap == 16 && n == 11) return list_occ_t<16, 11>(L, smem, blocks_per_sm);
    switch (lcap) {
    case 8: return list_occ_t<8>(L, smem, blocks_per_sm);
    case 16: return list_occ_t<16>(L, smem, blocks_per_sm);
    default: return list_occ_t<32>(L, smem, blocks_per_sm);
    }
}

}  // namespace polar

// list_packed.cu — the FSSCL list decoder with one WARP per frame: all L
// paths of the list live in one warp (§2.2.3-2.2.4; list
// memory with lazy copy, §3.2).
//
// A kernel with one warp per path (round 1's list.cu, removed) idles: most decision nodes
// of a fast-simplified schedule are small (Lambda <= 4 for most of them), so
// such warps idle on 28+ lanes and pay two CTA barriers per node.  Here the
// lanes are spread over (path, element) pairs instead: a stage or node of
// size Lambda <= 32 processes 32 / Lambda paths per warp instruction (node
// reductions become segmented shuffles inside lane groups of Lambda lanes),
// larger ones loop over the paths, and the prune, the beta copies and the
// pointer hand-over run inside the warp with __syncwarp only.
//
// Memory per warp (shared): alpha stage s (all s < n) has L buffers of 2^s
// floats; a path writes the stages of its descent into its own buffer and
// reads the first stage above from the buffer its 5-bit pointer names (LLR-
// domain lazy copy: no alpha is ever copied); flat beta per path (PAPER.md:
// L852), double-buffered by node parity; PMs, pointer rows, flip descriptors
// and the candidate keys of the current node.
//
// Arithmetic and order are the oracle's (O11): float32, -fmad=false, tree-order
// sums, (|alpha| bits, index) argmin keys, candidates in (dPM, mask) order,
// prune keys (PM, parent rank, candidate rank) (reading R22).
#include <cuda_runtime.h>

#include "device_common.cuh"

namespace polar {

namespace {

__device__ __forceinline__ int prow5(unsigned long long row, int s) { return (int)((row >> (5 * s)) & 31ull); }

// closed-form candidate order of an R1 / SPC node from the ordered least
// reliable magnitudes A0 <= A1 <= A2 <= A3 (see decode.cu, reading R7)
__device__ __forceinline__ uint32_t cand_order(int kind, uint32_t parity, const float (&A)[4]) {
    if (kind == OP_R1) return 0x3210u;
    if (parity == 0) return ((A[0] + A[3]) < (A[1] + A[2])) ? 0xFCA69530u : 0xFCA96530u;
    return (A[3] < (A[0] + A[1]) + A[2]) ? 0xEDB78421u : 0xEDB87421u;
}

// dPM of the candidate with flip mask m: the flipped |alpha|s summed in order
// m1..m4 (0 + x = x and d + 0 = d exactly, all terms >= +0)
__device__ __forceinline__ float flip_dpm(uint32_t m, const float (&A)[4]) {
    float d = 0.f;
#pragma unroll
    for (int q = 0; q < 4; q++) d = d + (((m >> q) & 1u) ? A[q] : 0.f);
    return d;
}

}  // namespace

// PLAIN: compile-time "no CRC, systematic, more than one node" (the final
// CRC / re-encoding selection and the whole-code-node path left out)
// GB: the path betas live in the global arena P.gbeta (a separate instance, so
// the shared-memory instance keeps shared-memory addressing)
template <int NL, bool PLAIN = false, bool GB = false>
__global__ void __launch_bounds__(kListPackedWarps * 32, 8) fsscl_packed_kernel(const ListParams P) {
    extern __shared__ __align__(16) uint32_t smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int n = (NL > 0) ? NL : P.n, N = 1 << n;
    const int nw = (NL > 0) ? (NL >= 5 ? (1 << NL) / 32 : 1) : P.nw;
    const int L = P.L, M = P.M, K = P.K;

    uint32_t *nodes_s = smem;
    #pragma unroll 1
    for (int i = threadIdx.x; i < M; i += blockDim.x) nodes_s[i] = P.nodes[i];
    __syncthreads();
    uint32_t *wb = smem + P.o_warp0 + warp * P.words;
    float *abuf = reinterpret_cast<float *>(wb + P.o_alpha);           // stage s: L buffers at L(2^s - 1)
    // [2][L][nw]: shared memory, or this warp's block of the global arena
    uint32_t *betaA = GB ? P.gbeta + (size_t)(blockIdx.x * P.pwarps + warp) * (size_t)(2 * L * nw) : wb + P.o_beta;
    uint32_t *clist_s = wb + P.o_clist;                                // [L]
    uint2 *mi_s = reinterpret_cast<uint2 *>(wb + P.o_mi);              // [L]
    unsigned long long *prow_s = reinterpret_cast<unsigned long long *>(wb + P.o_prow);  // [2][L]
    unsigned long long *cand_s = reinterpret_cast<unsigned long long *>(wb + P.o_cand);  // [8L]
    uint32_t *sel_s = wb + P.o_sel;                                    // [L]
    float *pm_s = reinterpret_cast<float *>(wb + P.o_selpm);           // [2][L]
    uint32_t *ok_s = wb + P.o_ok;                                      // [L]
    // stages >= sg live in a per-warp global arena (L2), the rest in shared memory
    const int sg = P.sg;
    float *garena = P.galpha ? P.galpha + (size_t)(blockIdx.x * P.pwarps + warp) * P.gstride : nullptr;
    // shared stage s starts at L (2^s - 1) plus padding that keeps stages >= 2
    // 16-byte aligned (stage 0 takes round4(L), stage 1 round4(2L) floats)
    const int pad1 = ((L + 3) & ~3) - L, pad2 = pad1 + ((2 * L + 3) & ~3) - 2 * L;
    auto stage_buf = [&](int s, int k) -> float * {
        if (s >= sg) return garena + (size_t)L * ((1 << s) - (1 << sg)) + (size_t)k * (1 << s);
        return abuf + (size_t)L * ((1 << s) - 1) + (s >= 2 ? pad2 : (s == 1 ? pad1 : 0)) + (size_t)k * (1 << s);
    };
    auto beta_of = [&](int par, int k) -> uint32_t * { return betaA + (size_t)(par * L + k) * nw; };

    const unsigned long long nfr = (unsigned long long)P.n_frames;
    unsigned long long f = 0, fnext = 0;
    if (lane == 0) { f = atomicAdd(P.queue, 1ull); fnext = atomicAdd(P.queue, 1ull); }
    f = __shfl_sync(FULL, f, 0);
    fnext = __shfl_sync(FULL, fnext, 0);

    #pragma unroll 1
    while (f < nfr) {
        if (fnext < nfr) {
            const char *nr = reinterpret_cast<const char *>(P.llr + (size_t)fnext * N);
            #pragma unroll 1
            for (int b = lane * 128; b < N * 4; b += 32 * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(nr + b));
        }
        unsigned long long fnext2 = 0;
        if (lane == 0) fnext2 = atomicAdd(P.queue, 1ull);
        const float *chan = P.llr + (size_t)f * N;

        int nL = 1, par = 0;
        int pos_mem = 0, lev_mem = n;
        if (lane == 0) { pm_s[0] = 0.f; prow_s[0] = 0ull; }
        __syncwarp();

        #pragma unroll 1
        for (int j = 0; j <= M; j++) {
            // ---- pending BETA ops of every path after node j-1
            int pl = 0, l = n;
            if (j > 0) {
                const uint32_t pn = nodes_s[j - 1];
                const int plam = (int)op_lam(pn), pphi = (int)op_phi(pn);
                pl = (pphi + 1) << plam;
                int ph = pphi;
                l = plam;
                if ((ph & 1) && l < 5) {
                    // levels with 2 Lambda <= 32 act inside one word: lane k, path k
                    const int wd = ((ph - 1) << l) >> 5;
                    uint32_t x = 0;
                    if (lane < nL) x = beta_of(par, lane)[wd];
                    #pragma unroll 1
                    while ((ph & 1) && l < 5) {
                        const int o = ((ph - 1) << l) & 31, Lm = 1 << l;
                        x ^= ((x >> (o + Lm)) & ((1u << Lm) - 1u)) << o;
                        ph >>= 1;
                        l++;
                    }
                    if (lane < nL) beta_of(par, lane)[wd] = x;
                    __syncwarp();
                }
                #pragma unroll 1
                while (ph & 1) {
                    // BETA(l, ph), Lambda >= 32: lanes over (path, word)
                    const int nwd = 1 << (l - 5);
                    const int wd = ((ph - 1) << l) >> 5, ws = (ph << l) >> 5;
                    const int tot = nL << (l - 5);
                    #pragma unroll 1
                    for (int idx = lane; idx < tot; idx += 32) {
                        const int k = idx >> (l - 5), t = idx & (nwd - 1);
                        uint32_t *bk = beta_of(par, k);
                        bk[wd + t] ^= bk[ws + t];
                    }
                    __syncwarp();
                    ph >>= 1;
                    l++;
                }
            }
            if (j == M) break;

            const uint32_t nd = nodes_s[j];
            const int kind = (int)op_kind(nd), lam = (int)op_lam(nd), phi = (int)op_phi(nd);
            const int Lam = 1 << lam, seg = phi << lam;
            const int nc = (kind == OP_R0) ? 1 : (kind == OP_REP ? 2 : (kind == OP_R1 ? (Lam == 1 ? 2 : 4) : 8));
            const int s_hi = min(max(max(lev_mem, bitlen((uint32_t)(pos_mem ^ pl))), l + 1), n) - 1;

            // ---- ALPHA ops s_hi .. lam for every path (Eq. 4, Alg. 1): lanes over
            // (path, element); the top stage reads the inherited buffer
            #pragma unroll 1
            for (int s = s_hi; s >= lam; s--) {
                const int Ls = 1 << s;
                const int psi = pl >> s;
                const bool odd = (psi & 1) != 0;
                const int boff = (psi - 1) << s;
                const bool top = (s + 1 == n), first = (s == s_hi);
                const int tot = nL << s;
                // buffers of one stage are contiguous: path k's element i of stage s
                // is dst[(k << s) + i] = dst[idx]
                float *dst = stage_buf(s, 0);
                const float *sb = top ? chan : stage_buf(s + 1, 0);
                const uint32_t *bpar = betaA + (size_t)par * L * nw;
                if (Ls >= 4) {
                    // four consecutive elements of one path per lane (float4; the
                    // beta bits of a g sit in one word)
                    #pragma unroll 1
                    for (int idx = lane * 4; idx < tot; idx += 128) {
                        const int k = idx >> s, i = idx & (Ls - 1);
                        float4 lo, hi;
                        if (top) {
                            lo = __ldg(reinterpret_cast<const float4 *>(chan + i));
                            hi = __ldg(reinterpret_cast<const float4 *>(chan + Ls + i));
                        } else {
                            const int kb = first ? prow5(prow_s[par * L + k], s + 1) : k;
                            POLAR_DCHECK(kb < L && k < nL);
                            const float *src = sb + (kb << (s + 1)) + i;
                            lo = *reinterpret_cast<const float4 *>(src);
                            hi = *reinterpret_cast<const float4 *>(src + Ls);
                        }
                        float4 v;
                        if (odd) {
                            const int bp = boff + i;
                            const uint32_t b = bpar[k * nw + (bp >> 5)] >> (bp & 31);
                            v.x = g_exact(lo.x, hi.x, b & 1u); v.y = g_exact(lo.y, hi.y, (b >> 1) & 1u);
                            v.z = g_exact(lo.z, hi.z, (b >> 2) & 1u); v.w = g_exact(lo.w, hi.w, (b >> 3) & 1u);
                        } else {
                            v.x = f_minsum(lo.x, hi.x); v.y = f_minsum(lo.y, hi.y);
                            v.z = f_minsum(lo.z, hi.z); v.w = f_minsum(lo.w, hi.w);
                        }
                        *reinterpret_cast<float4 *>(dst + idx) = v;
                    }
                    __syncwarp();
                    continue;
                }
                #pragma unroll 1
                for (int idx = lane; idx < tot; idx += 32) {
                    const int k = idx >> s, i = idx & (Ls - 1);
                    float lo, hi;
                    if (top) {
                        lo = __ldg(chan + i);
                        hi = __ldg(chan + Ls + i);
                    } else {
                        const int kb = first ? prow5(prow_s[par * L + k], s + 1) : k;
                        const float *src = sb + (kb << (s + 1)) + i;
                        lo = src[0];
                        hi = src[Ls];
                    }
                    float v;
                    if (odd) {
                        const int bp = boff + i;
                        v = g_exact(lo, hi, (bpar[k * nw + (bp >> 5)] >> (bp & 31)) & 1u);
                    } else {
                        v = f_minsum(lo, hi);
                    }
                    dst[idx] = v;
                }
                __syncwarp();
            }
            if (lane < nL && s_hi >= lam) {
                // stages lam .. s_hi of path k now live in its own buffers
                unsigned long long row = prow_s[par * L + lane];
                #pragma unroll 1
                for (int s = lam; s <= s_hi; s++)
                    row = (row & ~(31ull << (5 * s))) | ((unsigned long long)lane << (5 * s));
                prow_s[par * L + lane] = row;
            }
            pos_mem = pl;
            lev_mem = lam + 1;

            // ---- node candidates of every path
            const bool sum_kind = (kind == OP_R0 || kind == OP_REP);
            if (Lam <= 32) {
                // lane groups of Lambda lanes, one path per group
                const int G = 32 >> lam;
                const int i = lane & (Lam - 1);
                const float *nb = (lam == n) ? chan : stage_buf(lam, 0);   // path k at nb[(k << lam) + i]
                #pragma unroll 1
                for (int k0 = 0; k0 < nL; k0 += G) {
                    const int k = k0 + (lane >> lam);
                    const bool valid = k < nL;
                    float xr = 0.f;
                    if (valid) xr = (!PLAIN && lam == n) ? __ldg(chan + i) : nb[(k << lam) + i];
                    const bool leader = valid && i == 0;
                    if (sum_kind) {
                        float vn = negpart(xr), vp = pospart(xr);
                        #pragma unroll 1
                        for (int h = Lam >> 1; h >= 1; h >>= 1) {
                            vn += __shfl_down_sync(FULL, vn, h);
                            vp += __shfl_down_sync(FULL, vp, h);
                        }
                        // the group leader holds the sums
                        vn = __shfl_sync(FULL, vn, lane & ~(Lam - 1));
                        vp = __shfl_sync(FULL, vp, lane & ~(Lam - 1));
                        const bool rep = (kind == OP_REP);
                        const uint32_t clist = rep ? ((vp < vn) ? 0x01u : 0x10u) : 0u;
                        if (valid) {
                            const float pm = pm_s[par * L + k];
                            #pragma unroll 1
                            for (int t = i; t < nc; t += Lam) {
                                const float d = ((clist >> (4 * t)) & 15u) ? vp : vn;
                                cand_s[k * nc + t] = ((unsigned long long)__float_as_uint(pm + d) << 32) | (uint32_t)((k << 3) | t);
                            }
                        }
                        if (leader) {
                            clist_s[k] = clist;
                            const uint32_t fill = (rep && (clist & 15u)) ? FULL : 0u;
                            const uint32_t lm = ((Lam == 32) ? FULL : ((1u << Lam) - 1u)) << (seg & 31);
                            uint32_t *bk = beta_of(par, k);
                            bk[seg >> 5] = (bk[seg >> 5] & ~lm) | (fill & lm);
                        }
                    } else {
                        const uint32_t b = __ballot_sync(FULL, valid && xr < 0.f);
                        const uint32_t lm = (Lam == 32) ? FULL : ((1u << Lam) - 1u);
                        const uint32_t gbits = (b >> (lane & ~(Lam - 1) & 31)) & lm;
                        const uint32_t parity = (uint32_t)__popc(gbits) & 1u;
                        uint32_t key = valid ? __float_as_uint(fabsf(xr)) : 0xFFFFFFFFu;
                        const int need = (kind == OP_SPC) ? 4 : (Lam == 1 ? 1 : 2);
                        float A[4] = {0.f, 0.f, 0.f, 0.f};
                        uint32_t m[4] = {0, 0, 0, 0};
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < need) {
                                // segmented argmin of (|alpha| bits, index) in the group:
                                // the group minimum by shuffles, the lowest lane holding it
                                // by one ballot (lowest index wins ties, reading R4)
                                uint32_t mk = key;
                                #pragma unroll 1
                                for (int off = 1; off < Lam; off <<= 1) mk = min(mk, __shfl_xor_sync(FULL, mk, off));
                                const uint32_t eqb = (__ballot_sync(FULL, key == mk) >> (lane & ~(Lam - 1) & 31)) & lm;
                                const uint32_t mx = (uint32_t)(__ffs(eqb) - 1);
                                m[q] = mx;
                                A[q] = __uint_as_float(mk);
                                if ((uint32_t)i == mx) key = 0xFFFFFFFFu;
                            }
                        }
                        const uint32_t clist = cand_order(kind, parity, A);
                        if (valid) {
                            const float pm = pm_s[par * L + k];
                            #pragma unroll 1
                            for (int t = i; t < nc; t += Lam) {
                                const float d = flip_dpm((clist >> (4 * t)) & 15u, A);
                                cand_s[k * nc + t] = ((unsigned long long)__float_as_uint(pm + d) << 32) | (uint32_t)((k << 3) | t);
                            }
                        }
                        if (leader) {
                            clist_s[k] = clist;
                            mi_s[k] = make_uint2(m[0] | (m[1] << 16), m[2] | (m[3] << 16));
                            // the HD word with c1's flips in path k's beta
                            uint32_t wv = gbits;
                            const uint32_t m0 = clist & 15u;
#pragma unroll
                            for (int q = 0; q < 4; q++)
                                if ((m0 >> q) & 1u) wv ^= 1u << m[q];
                            uint32_t *bk = beta_of(par, k);
                            const int wd = seg >> 5, o = seg & 31;
                            bk[wd] = (bk[wd] & ~(lm << o)) | ((wv & lm) << o);
                        }
                    }
                }
            } else {
                // Lambda > 32: one path at a time, warp-wide (as the stack decoder)
                #pragma unroll 1
                for (int k = 0; k < nL; k++) {
                    float *a = (!PLAIN && lam == n) ? abuf : stage_buf(lam, k);
                    if (!PLAIN && lam == n) {
                        #pragma unroll 1
                        for (int q = lane; q < N; q += 32) a[q] = __ldg(chan + q);
                        __syncwarp();
                    }
                    uint32_t *bk = beta_of(par, k);
                    const float pm = pm_s[par * L + k];
                    uint32_t clist = 0;
                    if (sum_kind) {
                        const bool rep = (kind == OP_REP);
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
                        float vn = a[lane], vp = a[32 * H + lane];
                        #pragma unroll 1
                        for (int h = 16; h >= 1; h >>= 1) {
                            vn += __shfl_down_sync(FULL, vn, h);
                            vp += __shfl_down_sync(FULL, vp, h);
                        }
                        vn = __shfl_sync(FULL, vn, 0);
                        vp = __shfl_sync(FULL, vp, 0);
                        __syncwarp();
                        if (rep) clist = (vp < vn) ? 0x01u : 0x10u;
                        if (lane < nc) {
                            const float d = ((clist >> (4 * lane)) & 15u) ? vp : vn;
                            cand_s[k * nc + lane] = ((unsigned long long)__float_as_uint(pm + d) << 32) | (uint32_t)((k << 3) | lane);
                        }
                        const uint32_t fill = (rep && (clist & 15u)) ? FULL : 0u;
                        #pragma unroll 1
                        for (int t = lane; t < R; t += 32) bk[(seg >> 5) + t] = fill;
                    } else {
                        const int need = (kind == OP_SPC) ? 4 : 2;
                        uint32_t parity = 0;
                        unsigned long long t0 = ~0ull, t1 = ~0ull, t2 = ~0ull, t3 = ~0ull;
                        const int R = Lam >> 5;
                        #pragma unroll 1
                        for (int t = 0; t < R; t++) {
                            const float x = a[32 * t + lane];
                            const uint32_t b = __ballot_sync(FULL, x < 0.f);
                            if (lane == (t & 31)) bk[(seg >> 5) + t] = b;
                            parity ^= (uint32_t)__popc(b);
                            top4_insert(((unsigned long long)__float_as_uint(fabsf(x)) << 32) | (uint32_t)(32 * t + lane),
                                        t0, t1, t2, t3);
                        }
                        float A[4] = {0.f, 0.f, 0.f, 0.f};
                        uint32_t m[4] = {0, 0, 0, 0};
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            if (q < need) {
                                uint32_t mh, ml;
                                warp_min_key((uint32_t)(t0 >> 32), (uint32_t)t0, mh, ml);
                                m[q] = ml;
                                A[q] = __uint_as_float(mh);
                                if ((uint32_t)t0 == ml && (uint32_t)(t0 >> 32) == mh) { t0 = t1; t1 = t2; t2 = t3; t3 = ~0ull; }
                            }
                        }
                        clist = cand_order(kind, parity & 1u, A);
                        if (lane < nc) {
                            const float d = flip_dpm((clist >> (4 * lane)) & 15u, A);
                            cand_s[k * nc + lane] = ((unsigned long long)__float_as_uint(pm + d) << 32) | (uint32_t)((k << 3) | lane);
                        }
                        __syncwarp();
                        if (lane == 0) {
                            mi_s[k] = make_uint2(m[0] | (m[1] << 16), m[2] | (m[3] << 16));
                            const uint32_t m0 = clist & 15u;
#pragma unroll
                            for (int q = 0; q < 4; q++)
                                if ((m0 >> q) & 1u) {
                                    const int pos = seg + (int)m[q];
                                    bk[pos >> 5] ^= 1u << (pos & 31);
                                }
                        }
                    }
                    if (lane == 0) clist_s[k] = clist;
                    __syncwarp();
                }
            }
            __syncwarp();

            // ---- prune to the L best keys (reading R22).  Each
            // path's nc keys ascend (dPM, then candidate rank), so the survivors
            // come out of a tournament over the paths' list heads: lane k holds
            // path k's head, L rounds of a warp minimum, the winner advances.
            const int total = nL * nc;
            const int npar = par ^ 1;
            const int nL2 = min(total, L);
            {
                int h = 0;
                unsigned long long head = (lane < nL) ? cand_s[lane * nc] : ~0ull;
                #pragma unroll 1
                for (int r = 0; r < nL2; r++) {
                    uint32_t mh, ml;
                    warp_min_key((uint32_t)(head >> 32), (uint32_t)head, mh, ml);
                    const unsigned long long mk = ((unsigned long long)mh << 32) | ml;
                    if (head == mk) {            // keys are unique: one winner
                        sel_s[r] = ml;
                        pm_s[npar * L + r] = __uint_as_float(mh);
                        h++;
                        head = (h < nc) ? cand_s[lane * nc + h] : ~0ull;
                    }
                }
            }
            __syncwarp();

            // ---- rank r takes its parent's beta prefix, flips and pointer row
            const int npl = (phi + 1) << lam;
            const int nwp = (npl + 31) >> 5;
            const uint32_t magic = (uint32_t)((0x100000000ull + (uint64_t)nwp - 1) / (uint64_t)nwp);
            #pragma unroll 1
            for (int idx = lane; idx < nL2 * nwp; idx += 32) {
                // idx / nwp by a reciprocal multiply (exact for idx <= 4096, nwp <= 128;
                // nwp = 1 has no 32-bit reciprocal)
                const int r = (nwp == 1) ? idx : (int)__umulhi((uint32_t)idx, magic), q = idx - r * nwp;
                beta_of(npar, r)[q] = beta_of(par, (int)(sel_s[r] >> 3))[q];
            }
            __syncwarp();
            if (lane < nL2) {
                const int r = lane;
                const int p = (int)(sel_s[r] >> 3), rk = (int)(sel_s[r] & 7u);
                POLAR_DCHECK(p < nL && rk < nc);
                const uint32_t cl = clist_s[p];
                const uint32_t rel = ((cl >> (4 * rk)) & 15u) ^ (cl & 15u);
                uint32_t *dst = beta_of(npar, r);
                if (rel) {
                    if (kind == OP_REP) {
                        if (Lam >= 32) {
                            #pragma unroll 1
                            for (int t = 0; t < (Lam >> 5); t++) dst[(seg >> 5) + t] ^= FULL;
                        } else {
                            dst[seg >> 5] ^= ((1u << Lam) - 1u) << (seg & 31);
                        }
                    } else {
                        const uint2 hh = mi_s[p];
                        const uint32_t m4[4] = {hh.x & 0xFFFFu, hh.x >> 16, hh.y & 0xFFFFu, hh.y >> 16};
#pragma unroll
                        for (int q = 0; q < 4; q++)
                            if ((rel >> q) & 1u) {
                                const int pos = seg + (int)m4[q];
                                dst[pos >> 5] ^= 1u << (pos & 31);
                            }
                    }
                }
                prow_s[npar * L + r] = prow_s[par * L + p];
            }
            __syncwarp();
            par = npar;
            nL = nL2;
        }

        // ---- final selection (reading R24): first path in rank
        // order whose block passes the CRC
        int pick = 0, status = 0;
        const uint32_t *pick_cw = beta_of(par, 0);
        if (!PLAIN && (P.c > 0 || P.nonsys)) {
            status = 1;
            #pragma unroll 1
            for (int k = 0; k < nL; k++) {
                const uint32_t *cw = beta_of(par, k);
                if (P.nonsys) {
                    uint32_t *scratch = beta_of(par ^ 1, k);
                    #pragma unroll 1
                    for (int q = lane; q < nw; q += 32) scratch[q] = cw[q];
                    __syncwarp();
                    xform_words(scratch, N, nw, lane);
                    cw = scratch;
                }
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
                    ok = (__reduce_xor_sync(FULL, syn) == 0);
                }
                if (ok) { pick = k; status = 0; pick_cw = cw; break; }
            }
            if (status == 1 && P.nonsys) pick_cw = beta_of(par ^ 1, 0);   // path 0, already transformed
            if (status == 1 && !P.nonsys) pick_cw = beta_of(par, 0);
        }
        uint8_t *ob = P.out_bits + (size_t)f * K;
        #pragma unroll 1
        for (int q = lane; q < K; q += 32) {
            const int idx = P.info[q];
            ob[q] = (uint8_t)((pick_cw[idx >> 5] >> (idx & 31)) & 1u);
        }
        if (lane == 0) {
            if (P.pm) P.pm[f] = pm_s[par * L + pick];
            if (P.status) P.status[f] = (uint8_t)status;
        }
        __syncwarp();
        f = fnext;
        fnext = __shfl_sync(FULL, fnext2, 0);
    }
}

template <int NL, bool PLAIN = false, bool GB = false>
static cudaError_t launch_packed_t(const ListParams &p, int ctas, int smem, cudaStream_t st) {
    auto kern = fsscl_packed_kernel<NL, PLAIN, GB>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    kern<<<ctas, p.pwarps * 32, smem, st>>>(p);
    return cudaGetLastError();
}

cudaError_t launch_list_packed(const ListParams &p, int ctas, int smem, cudaStream_t st) {
    if (p.gbeta) return launch_packed_t<0, false, true>(p, ctas, smem, st);
    if (p.n == 7) return launch_packed_t<7>(p, ctas, smem, st);
    if (p.n == 10) return (p.c == 0 && !p.nonsys && p.M > 1) ? launch_packed_t<10, true>(p, ctas, smem, st)
                                                               : launch_packed_t<10>(p, ctas, smem, st);
    return launch_packed_t<0>(p, ctas, smem, st);
}

template <int NL, bool GB = false>
static cudaError_t packed_occ_t(int pwarps, int smem, int *blocks) {
    cudaError_t e = cudaFuncSetAttribute(fsscl_packed_kernel<NL, false, GB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(blocks, fsscl_packed_kernel<NL, false, GB>, pwarps * 32, smem);
}

cudaError_t list_packed_occupancy(int n, int pwarps, int smem, int *blocks_per_sm, bool gbeta) {
    if (gbeta) return packed_occ_t<0, true>(pwarps, smem, blocks_per_sm);
    if (n == 7) return packed_occ_t<7>(pwarps, smem, blocks_per_sm);
    if (n == 10) return packed_occ_t<10>(pwarps, smem, blocks_per_sm);
    return packed_occ_t<0>(pwarps, smem, blocks_per_sm);
}

}  // namespace polar

// capi.cu — the extern "C" boundary of libpolarscs (include/polar_scs.h):
// argument validation, handle lifetime, launch configuration and the
// host-buffer pipeline.  Every computation runs in the kernels of decode.cu
// and codec.cu; this file only moves pointers, sizes and tables.
#include <cuda.h>   // driver types of the stream memory operation only (entry point resolved at run time)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <new>

#include "internal.h"

namespace polar {
cudaError_t launch_decode(const DecodeParams &p, int slots, bool snap_smem, bool chan_smem, int ctas, int smem,
                          cudaStream_t st);
int specialised_nl(int n, int slots, bool snap_smem, bool chan_smem, bool recs_smem);
cudaError_t decode_occupancy(int n, int slots, bool snap_smem, bool chan_smem, int mode, bool recs_smem, int smem,
                             int *blocks_per_sm);
cudaError_t launch_decode_counts(const DecodeParams &p, int slots, int ctas, int smem, cudaStream_t st);
cudaError_t launch_list_packed(const ListParams &p, int ctas, int smem, cudaStream_t st);
cudaError_t list_packed_occupancy(int n, int pwarps, int smem, int *blocks_per_sm, bool gbeta);
cudaError_t launch_crc_attach(const CodecParams &p, cudaStream_t st);
cudaError_t launch_encode(const CodecParams &p, cudaStream_t st);
cudaError_t launch_modulate(const CodecParams &p, cudaStream_t st);
cudaError_t launch_generate(const CodecParams &p, cudaStream_t st);
}  // namespace polar

using namespace polar;

namespace {

template <class T>
cudaError_t upload(T **dst, const std::vector<T> &src) {
    const size_t bytes = std::max<size_t>(1, src.size()) * sizeof(T);
    cudaError_t e = cudaMalloc(reinterpret_cast<void **>(dst), bytes);
    if (e != cudaSuccess) return e;
    if (!src.empty()) e = cudaMemcpy(*dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice);
    return e;
}

int slots_for(int D) { return D <= 32 ? 1 : (D <= 64 ? 2 : (D <= 128 ? 4 : 0)); }   // 0: global stack
int round4(int w) { return (w + 3) & ~3; }

void free_handle(polar_scs_t h) {
    if (!h) return;
    cudaFree(h->t.nodes); cudaFree(h->t.recs); cudaFree(h->t.info); cudaFree(h->t.crc_tab); cudaFree(h->t.crc_bytes); cudaFree(h->t.info_words);
    cudaFree(h->d_queue); cudaFree(h->d_snap); cudaFree(h->d_keys); cudaFree(h->d_jsm); cudaFree(h->d_hdr); cudaFree(h->d_galpha); cudaFree(h->d_gbeta); cudaFree(h->d_salpha);
    for (int b = 0; b < polar_scs_s::kStageBufs; b++) {
        cudaFree(h->d_stage_llr[b]); cudaFree(h->d_stage_bits[b]);
        if (h->ev_h2d[b]) cudaEventDestroy(h->ev_h2d[b]);
        if (h->ev_dec[b]) cudaEventDestroy(h->ev_dec[b]);
        if (h->ev_d2h[b]) cudaEventDestroy(h->ev_d2h[b]);
    }
    cudaFree(h->d_sllr); cudaFree(h->d_ready);
    if (h->ev_sreset) cudaEventDestroy(h->ev_sreset);
    if (h->ev_sdone) cudaEventDestroy(h->ev_sdone);
    if (h->s_h2d) cudaStreamDestroy(h->s_h2d);
    for (int b = 0; b < 2; b++)
        if (h->s_comp[b]) cudaStreamDestroy(h->s_comp[b]);
    if (h->s_d2h) cudaStreamDestroy(h->s_d2h);
    delete h;
}

double sigma2_of(double ebno_db, double rate) { return 1.0 / (2.0 * rate * std::pow(10.0, ebno_db / 10.0)); }

CodecParams codec_params(polar_scs_t h, int64_t n) {
    CodecParams p{};
    p.n_frames = n;
    p.N = h->t.N; p.n = h->t.n; p.K = h->t.K; p.c = h->t.c;
    p.nw = std::max(1, h->t.N / 32);
    p.info = h->t.info; p.crc_tab = h->t.crc_tab; p.info_words = h->t.info_words;
    p.nonsys = (h->flags & POLAR_FLAG_NONSYSTEMATIC) ? 1 : 0;
    return p;
}

int cuda_status(cudaError_t e) { return e == cudaSuccess ? POLAR_OK : (e == cudaErrorMemoryAllocation ? POLAR_ENOMEM : POLAR_ECUDA); }

// Every entry point that touches device memory runs on the handle's device:
// switch to it on entry, restore the caller's device on return.
struct DeviceGuard {
    int prev = -1;
    bool ok = true;
    explicit DeviceGuard(polar_scs_t h) {
        if (!h) return;
        int cur = 0;
        if (cudaGetDevice(&cur) != cudaSuccess) { ok = false; return; }
        if (cur == h->device) return;
        if (cudaSetDevice(h->device) != cudaSuccess) { ok = false; return; }
        prev = cur;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

// slot: which frame-queue counter / snapshot arena the launch uses; two slots
// let the host pipeline overlap one chunk's decode with the next one's
// streaming host pipeline: per-chunk ready flags, error word, log2 frames per chunk
struct StreamArgs {
    const uint32_t *ready;
    uint32_t *err;
    int shift;
};

int decode_impl(polar_scs_t h, const float *llr, int64_t n, uint8_t *bits, float *pm, uint32_t *pops,
                uint32_t *sw, uint8_t *status, cudaStream_t st, int slot = 0, const StreamArgs *sa = nullptr,
                uint32_t *counts = nullptr) {
    DecodeParams p = h->base;
    if (sa) { p.ready = sa->ready; p.err = sa->err; p.chunk_shift = sa->shift; }
    p.llr = llr; p.n_frames = n; p.out_bits = bits;
    p.pm = pm; p.pops = pops; p.switches = sw; p.status = status;
    p.queue = h->d_queue + slot;
    if (h->d_snap) p.snap_global = h->d_snap + (h->snap_bytes / 4) * (size_t)slot;
    if (h->d_salpha) p.galpha = h->d_salpha + h->salpha_floats * (size_t)slot;
    if (h->d_keys) { p.stack_keys = h->d_keys + h->stack_count * (size_t)slot; p.stack_jsm = h->d_jsm + h->stack_count * (size_t)slot; }
    if (h->d_hdr) p.hdr_global = h->d_hdr + h->hdr_count * (size_t)slot;
    cudaError_t e = cudaMemsetAsync(p.queue, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return cuda_status(e);
    if (counts) {
        p.counts = counts;
        p.chan_in_smem = h->chan_in_smem;
        p.snap_in_smem = h->snap_in_smem;
        return cuda_status(launch_decode_counts(p, slots_for(h->D), h->ctas, h->smem_per_cta, st));
    }
    return cuda_status(launch_decode(p, slots_for(h->D), h->snap_in_smem != 0, h->chan_in_smem != 0, h->ctas,
                                     h->smem_per_cta, st));
}

int list_impl(polar_scs_t h, const float *llr, int64_t n, uint8_t *bits, float *pm, uint8_t *status, cudaStream_t st,
              int slot = 0) {
    ListParams p = h->list;
    p.llr = llr; p.n_frames = n; p.out_bits = bits; p.pm = pm; p.status = status;
    p.queue = h->d_queue + slot;
    if (p.galpha) p.galpha += (size_t)h->list_ctas * p.pwarps * p.gstride * (size_t)slot;
    if (p.gbeta) p.gbeta += (size_t)h->list_ctas * p.pwarps * (size_t)(2 * p.L * p.nw) * (size_t)slot;
    cudaError_t e = cudaMemsetAsync(p.queue, 0, sizeof(unsigned long long), st);
    if (e != cudaSuccess) return cuda_status(e);
    const int ctas = (int)std::min<int64_t>(h->list_ctas, (n + p.pwarps - 1) / p.pwarps);
    return cuda_status(launch_list_packed(p, ctas, h->list_smem, st));
}

// packed FSSCL layout (list_packed.cu): node table, then one block per warp
// with the offsets below (words, 16-byte aligned areas).  Returns the words
// of one CTA.
int list_packed_layout(ListParams &p) {
    const int L = p.L, N = p.N;
    p.o_warp0 = round4(p.M);
    int o = 0;
    if (p.M == 1) p.sg = p.n;                 // the root node uses the alpha area as scratch
    p.o_alpha = o; o += round4(std::max(L * ((1 << p.sg) - 1) + 6, p.M == 1 ? N : 0));   // + stage padding
    p.gstride = (size_t)L * (size_t)(N - (1 << p.sg));
    p.o_beta = o;  if (!p.beta_global) o += round4(2 * L * p.nw);
    p.o_clist = o; o += round4(L);
    p.o_mi = o;    o += round4(2 * L);
    p.o_prow = o;  o += round4(4 * L);
    p.o_cand = o;  o += round4(16 * L);
    p.o_sel = o;   o += round4(L);
    p.o_selpm = o; o += round4(2 * L);
    p.o_ok = o;    o += round4(L);
    p.o_reg = p.o_misc = 0;
    p.words = o;
    return p.o_warp0 + p.pwarps * o;
}

}  // namespace

extern "C" {

const char *polar_scs_strerror(int status) {
    switch (status) {
    case POLAR_OK: return "ok";
    case POLAR_EINVAL: return "invalid argument";
    case POLAR_ENOMEM: return "out of memory";
    case POLAR_ECUDA: return "CUDA error";
    case POLAR_ENOTSYS: return "not supported for this code";
    default: return "unknown status";
    }
}

int polar_scs_create_ex(polar_scs_t *out, int32_t N, int32_t K, const uint8_t *frozen_mask, int32_t D, int32_t L,
                        uint32_t crc_poly, uint32_t flags) {
    if (!out) return POLAR_EINVAL;
    *out = nullptr;
    const uint32_t known = POLAR_FLAG_BIT_LEVEL | POLAR_FLAG_SNAP_GLOBAL | POLAR_FLAG_CHAN_GLOBAL |
                           POLAR_FLAG_SNAP_SMEM | POLAR_FLAG_CHAN_SMEM | POLAR_FLAG_NONSYSTEMATIC |
                           POLAR_FLAG_LIST_CTA | POLAR_FLAG_LIST_PACKED;
    if (flags & POLAR_FLAG_LIST_CTA) return POLAR_EINVAL;     // the CTA list kernel was removed (slower everywhere)
    if (D < 1 || D > kMaxD || L < 1 || L > 65536 || (flags & ~known)) return POLAR_EINVAL;
    if ((flags & POLAR_FLAG_SNAP_GLOBAL) && (flags & POLAR_FLAG_SNAP_SMEM)) return POLAR_EINVAL;
    if ((flags & POLAR_FLAG_CHAN_GLOBAL) && (flags & POLAR_FLAG_CHAN_SMEM)) return POLAR_EINVAL;
    HostCode hc;
    int rc = build_host_code(N, K, frozen_mask, crc_poly, (flags & POLAR_FLAG_BIT_LEVEL) != 0, hc);
    if (rc != POLAR_OK) return rc;

    polar_scs_t h = new (std::nothrow) polar_scs_s();
    if (!h) return POLAR_ENOMEM;
    h->flags = flags;
    h->D = D;
    // 16-bit per-depth counters are exact up to L = 65536: the L-th pop at a
    // depth prunes every entry of that depth or less, so no later pop has it
    h->L = L;
    cudaError_t e = cudaGetDevice(&h->device);
    CodeTables &t = h->t;
    t.N = hc.N; t.n = hc.n; t.K = hc.K; t.c = hc.c; t.M = hc.M; t.crc_poly = crc_poly;
    t.systematic_ok = hc.systematic_ok;
    t.nops = (int)hc.ops.size();
    if (e == cudaSuccess) e = upload(&t.nodes, hc.nodes);
    if (e == cudaSuccess) e = upload(&t.recs, hc.recs);
    if (e == cudaSuccess) e = upload(&t.info, hc.info);
    if (e == cudaSuccess) e = upload(&t.crc_tab, hc.crc_tab);
    if (e == cudaSuccess) e = upload(&t.crc_bytes, hc.crc_bytes);
    if (e == cudaSuccess) e = upload(&t.info_words, hc.info_words);
    if (e == cudaSuccess) e = cudaMalloc(&h->d_queue, 2 * sizeof(unsigned long long));
    if (e != cudaSuccess) { free_handle(h); return cuda_status(e); }

    // ---- decode launch layout (per-warp shared memory)
    int sms = 148, optin = 227 * 1024;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, h->device);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, h->device);
    const int nw = std::max(1, N / 32);
    const int cnt_words = (((t.M + 1) * 2 + 3) / 4 + 1) & ~1;   // even: the fork headers that follow are uint2
    const int sstride = nw;                       // snapshot slot: beta words (headers live in smem)
    const int slots = slots_for(D);
    // per-depth records in shared memory when they fit (not for the global
    // stack, whose occupancy is shared-memory bound: it reads them through L1)
    const int sched_words = (POLAR_RECS_SMEM && slots != 0 && (t.M + 1) * 64 <= 16384) ? 16 * (t.M + 1) : 0;

    DecodeParams &p = h->base;
    p.nodes = t.nodes; p.recs = reinterpret_cast<const uint4 *>(t.recs); p.info = t.info; p.crc_tab = t.crc_tab; p.crc_bytes = t.crc_bytes; p.queue = h->d_queue;
    p.N = N; p.n = t.n; p.K = K; p.c = t.c; p.D = D; p.L = h->L; p.M = t.M;
    p.nw = nw; p.snap_stride = sstride; p.sched_words = sched_words; p.cnt_words = cnt_words;
    p.nonsys = (flags & POLAR_FLAG_NONSYSTEMATIC) ? 1 : 0;
    p.hdr_words = slots ? 2 * D : 0;
    p.used_words = slots ? 4 : round4((D + 31) / 32);
    p.win_words = (slots || POLAR_BIG_HOT) ? 0 : 256;
    p.uhat_words = p.nonsys ? nw : 0;

    // Layout choice: per warp, alpha stages >= 6 (N floats incl. scratch), flat
    // beta, best-effort beta and counters always live in shared memory; the
    // channel row and the snapshot arena go to shared memory or L1/L2.  Among
    // the allowed placements take the one with the most resident warps per SM;
    // ties prefer shared memory.
    int best_occ = -1, best_smem = 0, best_ww = 0, best_gst = 0;
    // compile-time modes of the specialised kernels (decode.cu): 1 systematic
    // with more than one node, 2 also without CRC
    const int mode = (p.nonsys || t.M == 1) ? 0 : (t.c == 0 ? 2 : 1);
    bool best_snap = false, best_chan = false;
    // alpha stages >= n - gst may move to a global (L2) arena; the fewest such
    // stages that reach the best occupancy win (the root-node code keeps its
    // shared scratch)
    // (only the specialised N = 2048 / 4096 kernels are built with the arena:
    // measured +10% on C4, +12% on C5; a run-time arena cost C2 5%)
    // (and only when that kernel is the one launched: a code whose per-depth
    // records do not fit shared memory runs the general kernel, which has no arena —
    // choosing arena stages for it overran the shared alpha area: found by the
    // randomised sweep on N = 2048 random information sets with ~1000 nodes)
    const int snl = specialised_nl(t.n, slots, false, false, sched_words > 0);
    const int gst_max = (t.M == 1 || !(snl == 11 || snl == 12)) ? 0 : 2;
    for (int gst = 0; gst <= gst_max; gst++)
    for (int ci = 0; ci < 2; ci++) {
        const bool chan_smem = (ci == 0);
        if (chan_smem && (flags & POLAR_FLAG_CHAN_GLOBAL)) continue;
        if (!chan_smem && (flags & POLAR_FLAG_CHAN_SMEM)) continue;
        for (int si = 0; si < 2; si++) {
            const bool snap_smem = (si == 0);
            if (snap_smem && (flags & POLAR_FLAG_SNAP_GLOBAL)) continue;
            if (snap_smem && slots == 0) continue;          // D > 128: the arena is global
            if (!snap_smem && (flags & POLAR_FLAG_SNAP_SMEM)) continue;
            if (gst > 0 && (snap_smem || chan_smem)) continue;  // only the GA kernel has the arena
            const int aw = gst ? (1 << (t.n - gst)) : N;
            const int ww = round4(p.win_words + (chan_smem ? N : 0) + aw + 2 * nw + cnt_words + p.hdr_words + p.used_words +
                                  p.uhat_words +
                                  (snap_smem ? D * sstride : 0));
            const int smem = 4 * (sched_words + kDecodeWarps * ww);
            if (smem > optin) continue;
            int occ = 0;
            if (decode_occupancy(t.n, slots, snap_smem, chan_smem, mode, sched_words > 0, smem, &occ) != cudaSuccess ||
                occ < 1)
                continue;
            if (occ > best_occ) {
                best_occ = occ; best_smem = smem; best_ww = ww; best_snap = snap_smem; best_chan = chan_smem;
                best_gst = gst;
            }
        }
    }
    cudaGetLastError();
    if (best_occ < 1) { free_handle(h); return POLAR_EINVAL; }
    const int occ = best_occ;
    const bool use_smem = best_snap;
    p.warp_words = best_ww;
    p.sg = t.n - best_gst;
    p.alpha_words = best_gst ? (1 << p.sg) : N;
    h->smem_per_cta = best_smem;
    h->chan_in_smem = best_chan ? 1 : 0;
    cudaGetLastError();
    h->snap_in_smem = use_smem ? 1 : 0;
    h->warps_per_cta = kDecodeWarps;
    h->ctas = occ * sms;
    if (!use_smem) {
        h->snap_bytes = (size_t)h->ctas * kDecodeWarps * (size_t)D * sstride * 4;
        e = cudaMalloc(&h->d_snap, 2 * h->snap_bytes);
        if (e != cudaSuccess) { free_handle(h); return cuda_status(e); }
        p.snap_global = h->d_snap;
    }
    if (best_gst > 0) {
        h->salpha_floats = (size_t)h->ctas * kDecodeWarps * (size_t)N;
        e = cudaMalloc(&h->d_salpha, 2 * h->salpha_floats * sizeof(float));
        if (e != cudaSuccess) { free_handle(h); return cuda_status(e); }
        p.galpha = h->d_salpha;
    }
    if (slots == 0) {
        const size_t warps = (size_t)h->ctas * kDecodeWarps;
        h->stack_count = warps * (size_t)(D + kColdPad);
        h->hdr_count = warps * (size_t)D;
        e = cudaMalloc(&h->d_keys, 2 * h->stack_count * sizeof(unsigned long long));
        if (e == cudaSuccess) e = cudaMalloc(&h->d_jsm, 2 * h->stack_count * sizeof(uint32_t));
        if (e == cudaSuccess) e = cudaMalloc(&h->d_hdr, 2 * h->hdr_count * sizeof(uint2));
        if (e != cudaSuccess) { free_handle(h); return cuda_status(e); }
        p.stack_keys = h->d_keys;
        p.stack_jsm = h->d_jsm;
        p.hdr_global = h->d_hdr;
    }
    // ---- FSSCL launch (polar_scl_decode): one warp per frame with the paths
    // packed across its lanes (list_packed.cu)
    if (h->L <= 32) {
        ListParams base{};
        base.nodes = t.nodes; base.info = t.info; base.crc_bytes = t.crc_bytes; base.queue = h->d_queue;
        base.N = N; base.n = t.n; base.K = K; base.c = t.c; base.L = h->L; base.M = t.M; base.nw = nw;
        base.nonsys = p.nonsys;
        ListParams lpk = base;
        int occ_p = 0;
        // packed: 4, 2 or 1 warps per CTA, whichever keeps the most warps resident
        int smem_p = 0, pw_best = 0;
        // the top alpha stages move to a global (L2-resident) arena while that
        // raises the resident warps (frames) per SM: take the fewest global
        // stages that reach the best occupancy
        // the path betas (2 L N/32 words per frame) may move to a global arena
        // too; that placement is taken only when it at least doubles the
        // resident warps (measured: C5, L = 32: 6 -> 32 warps/SM, 624 -> 1307
        // Mbps; C4, L = 16: 20 -> 32 warps/SM, 2271 -> 2250)
        int occ_b[2] = {0, 0}, pw_b[2] = {0, 0}, smem_b[2] = {0, 0};
        ListParams lp_b[2] = {base, base};
        for (int bg = 0; bg <= 1; bg++)
        for (int gst = 0; gst <= t.n; gst++) {
            for (int pw = kListPackedWarps; pw >= 1; pw >>= 1) {
                ListParams tp = base;
                tp.pwarps = pw;
                tp.sg = t.n - gst;
                tp.beta_global = bg;
                const int sm = 4 * list_packed_layout(tp);
                int oc = 0;
                if (sm > optin || list_packed_occupancy(t.n, pw, sm, &oc, bg != 0) != cudaSuccess) oc = 0;
                cudaGetLastError();
                if (oc * pw > occ_b[bg] * pw_b[bg]) { occ_b[bg] = oc; pw_b[bg] = pw; smem_b[bg] = sm; lp_b[bg] = tp; }
            }
        }
        const int bsel = (occ_b[1] * pw_b[1] >= 2 * occ_b[0] * pw_b[0] && occ_b[1] > 0) ? 1 : 0;
        occ_p = occ_b[bsel]; pw_best = pw_b[bsel]; smem_p = smem_b[bsel]; lpk = lp_b[bsel];
        if (occ_p >= 1) {
            h->list = lpk; h->list_packed = 1; h->list_ctas = occ_p * sms; h->list_smem = smem_p;
            if (lpk.gstride > 0) {
                const size_t per = (size_t)h->list_ctas * lpk.pwarps * lpk.gstride;
                e = cudaMalloc(&h->d_galpha, 2 * per * sizeof(float));
                if (e != cudaSuccess) { free_handle(h); return cuda_status(e); }
                h->list.galpha = h->d_galpha;
            }
            if (lpk.beta_global) {
                const size_t per = (size_t)h->list_ctas * lpk.pwarps * (size_t)(2 * lpk.L * lpk.nw);
                e = cudaMalloc(&h->d_gbeta, 2 * per * sizeof(uint32_t));
                if (e != cudaSuccess) { free_handle(h); return cuda_status(e); }
                h->list.gbeta = h->d_gbeta;
            }
        }
    }
    *out = h;
    return POLAR_OK;
}

int polar_scs_create(polar_scs_t *out, int32_t N, int32_t K, const uint8_t *frozen_mask, int32_t D, int32_t L,
                     uint32_t crc_poly) {
    return polar_scs_create_ex(out, N, K, frozen_mask, D, L, crc_poly, 0u);
}

void polar_scs_destroy(polar_scs_t h) {
    if (!h) return;
    DeviceGuard g(h);
    cudaDeviceSynchronize();
    free_handle(h);
}

int polar_scs_get_info(polar_scs_t h, polar_scs_info_t *o) {
    if (!h || !o) return POLAR_EINVAL;
    o->N = h->t.N; o->n = h->t.n; o->K = h->t.K; o->crc_bits = h->t.c; o->D = h->D; o->L = h->L;
    o->num_ops = h->t.nops; o->num_nodes = h->t.M;
    o->warps_per_cta = h->warps_per_cta; o->ctas = h->ctas; o->smem_per_cta = h->smem_per_cta;
    o->snap_in_smem = h->snap_in_smem; o->chan_in_smem = h->chan_in_smem; o->systematic_ok = h->t.systematic_ok ? 1 : 0; o->flags = h->flags;
    o->list_ctas = h->list_ctas; o->list_smem_per_cta = h->list_smem; o->list_packed = h->list_packed;
    o->list_warps_per_cta = h->list_packed ? h->list.pwarps : h->L;
    return POLAR_OK;
}

int polar_scs_decode_stats(polar_scs_t h, const float *llr, int64_t n, uint8_t *bits, float *pm, uint32_t *pops,
                           uint32_t *sw, uint8_t *status, void *stream) {
    if (!h || n < 0) return POLAR_EINVAL;
    if (n == 0) return POLAR_OK;
    DeviceGuard g(h);
    if (!g.ok) return POLAR_ECUDA;
    if (!llr || !bits) return POLAR_EINVAL;
    if (h->t.N >= 4 && (reinterpret_cast<uintptr_t>(llr) & 15u)) return POLAR_EINVAL;
    return decode_impl(h, llr, n, bits, pm, pops, sw, status, static_cast<cudaStream_t>(stream));
}

int polar_scs_decode(polar_scs_t h, const float *llr, int64_t n, uint8_t *bits, void *stream) {
    return polar_scs_decode_stats(h, llr, n, bits, nullptr, nullptr, nullptr, nullptr, stream);
}

int polar_scs_decode_counts(polar_scs_t h, const float *llr, int64_t n, uint8_t *bits, uint32_t *counts,
                            void *stream) {
    if (!h || n < 0) return POLAR_EINVAL;
    if (n == 0) return POLAR_OK;
    DeviceGuard g(h);
    if (!g.ok) return POLAR_ECUDA;
    if (!llr || !bits || !counts) return POLAR_EINVAL;
    if (h->t.N >= 4 && (reinterpret_cast<uintptr_t>(llr) & 15u)) return POLAR_EINVAL;
    if (reinterpret_cast<uintptr_t>(counts) & 15u) return POLAR_EINVAL;
    return decode_impl(h, llr, n, bits, nullptr, nullptr, nullptr, nullptr, static_cast<cudaStream_t>(stream), 0,
                       nullptr, counts);
}

int polar_scl_decode(polar_scs_t h, const float *llr, int64_t n, uint8_t *bits, float *pm, uint8_t *status,
                     void *stream) {
    if (!h || n < 0) return POLAR_EINVAL;
    if (h->list_ctas == 0) return POLAR_ENOTSYS;
    if (n == 0) return POLAR_OK;
    DeviceGuard g(h);
    if (!g.ok) return POLAR_ECUDA;
    if (!llr || !bits) return POLAR_EINVAL;
    if (h->t.N >= 4 && (reinterpret_cast<uintptr_t>(llr) & 15u)) return POLAR_EINVAL;
    return list_impl(h, llr, n, bits, pm, status, static_cast<cudaStream_t>(stream));
}

typedef CUresult (*WriteValue32Fn)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);

// cuStreamWriteValue32 (a stream-ordered 32-bit store done by the GPU front
// end), resolved once through the runtime; null when unavailable
static WriteValue32Fn write_value32() {
    static WriteValue32Fn fn = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *ptr = nullptr;
        cudaDriverEntryPointQueryResult q = cudaDriverEntryPointSymbolNotFound;
        if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &ptr, 12000, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<WriteValue32Fn>(ptr);
    }
    return fn;
}

// Streaming host pipeline: ONE decode launch per batch of up to
// kStreamChunks chunks, started before its LLRs arrive; the copy stream lands
// the chunks in order and sets each chunk's ready flag with a stream memory
// operation right after its copy, and a warp whose frame lies in a chunk not
// yet landed waits on that flag.  The decoded bits are written by the kernel
// straight into the caller's pinned output buffer (bits_dev is its device
// alias).  No launch boundaries and no per-chunk tail: the copy and the decode
// overlap at their own rates.  Returns 1 when streaming is unavailable (no
// stream memory operations), so the caller uses the chunked pipeline.
static int decode_host_stream(polar_scs_t h, const float *llr_host, int64_t n, uint8_t *bits_dev,
                              cudaStream_t stream) {
    WriteValue32Fn wv = write_value32();
    if (!wv) return 1;
    // the launch waits for copies queued after it: with blocking launches
    // (CUDA_LAUNCH_BLOCKING=1) they would only be issued once it returned
    static const bool blocking = [] {
        const char *v = std::getenv("CUDA_LAUNCH_BLOCKING");
        return v && v[0] && v[0] != '0';
    }();
    if (blocking) return 1;
    const int N = h->t.N, K = h->t.K;
    cudaError_t e = cudaSuccess;
    if (!h->d_ready) {
        // one probe of the memory operation on this device before relying on it
        e = cudaMalloc(&h->d_ready, (polar_scs_s::kStreamChunks + 1) * sizeof(uint32_t));
        if (e != cudaSuccess) return cuda_status(e);
        uint32_t v = 0;
        e = cudaMemsetAsync(h->d_ready, 0, sizeof(uint32_t), h->s_h2d);
        if (e == cudaSuccess && wv(reinterpret_cast<CUstream>(h->s_h2d), reinterpret_cast<CUdeviceptr>(h->d_ready), 7u, 0) != CUDA_SUCCESS)
            e = cudaErrorNotSupported;
        if (e == cudaSuccess) e = cudaStreamSynchronize(h->s_h2d);
        if (e == cudaSuccess) e = cudaMemcpy(&v, h->d_ready, sizeof(v), cudaMemcpyDeviceToHost);
        h->stream_ok = (e == cudaSuccess && v == 7u) ? 1 : -1;
        cudaGetLastError();
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_sreset, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&h->ev_sdone, cudaEventDisableTiming);
        if (e != cudaSuccess) h->stream_ok = -1;
    }
    if (h->stream_ok != 1) return 1;
    // chunks of 2^shift frames: 8 MiB of LLRs, halved while a batch would have
    // fewer than 16 chunks (down to 256 KiB), so small batches still overlap
    const int64_t fbytes = 4ll * N;
    int shift = 0;
    while (((int64_t)2 << shift) * fbytes <= (8ll << 20)) shift++;
    while (shift > 0 && (((int64_t)1 << shift) * 16 > n) && ((int64_t)1 << shift) * fbytes > (256ll << 10)) shift--;
    const int64_t cf = (int64_t)1 << shift;
    const int64_t batch = std::min<int64_t>(n, cf * polar_scs_s::kStreamChunks);
    if (h->stream_cap < batch) {
        cudaFree(h->d_sllr);
        h->d_sllr = nullptr;
        h->stream_cap = 0;
        e = cudaMalloc(&h->d_sllr, (size_t)batch * N * 4);
        if (e != cudaSuccess) return cuda_status(e);
        h->stream_cap = batch;
    }
    uint32_t *ready = h->d_ready, *err = h->d_ready + polar_scs_s::kStreamChunks;
    const StreamArgs sa{ready, err, shift};
    cudaEvent_t start;
    e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_status(e);
    cudaEventRecord(start, stream);
    cudaStreamWaitEvent(h->s_h2d, start, 0);
    cudaStreamWaitEvent(h->s_comp[0], start, 0);
    int rc = POLAR_OK;
    bool launched = false;
    e = cudaMemsetAsync(err, 0, sizeof(uint32_t), h->s_h2d);
    for (int64_t off = 0; off < n && rc == POLAR_OK && e == cudaSuccess; off += batch) {
        const int64_t m = std::min<int64_t>(batch, n - off);
        const int64_t nch = (m + cf - 1) / cf;
        if (off > 0) cudaStreamWaitEvent(h->s_h2d, h->ev_sdone, 0);   // the previous launch has read the staging
        e = cudaMemsetAsync(ready, 0, (size_t)nch * sizeof(uint32_t), h->s_h2d);
        if (e != cudaSuccess) break;
        cudaEventRecord(h->ev_sreset, h->s_h2d);
        // chunk i: H2D copy, then its ready flag (a stream memory operation)
        auto land = [&](int64_t i) {
            const int64_t cnt = std::min<int64_t>(cf, m - i * cf);
            e = cudaMemcpyAsync(h->d_sllr + (size_t)(i * cf) * N, llr_host + (size_t)(off + i * cf) * N, (size_t)cnt * N * 4,
                                cudaMemcpyHostToDevice, h->s_h2d);
            if (e == cudaSuccess && wv(reinterpret_cast<CUstream>(h->s_h2d), reinterpret_cast<CUdeviceptr>(ready + i), 1u, 0) != CUDA_SUCCESS)
                e = cudaErrorUnknown;
        };
        land(0);                          // the first chunk is queued before the launch that waits for it
        if (e != cudaSuccess) break;
        cudaStreamWaitEvent(h->s_comp[0], h->ev_sreset, 0);
        rc = decode_impl(h, h->d_sllr, m, bits_dev + off * K, nullptr, nullptr, nullptr, nullptr, h->s_comp[0], 0, &sa);
        if (rc != POLAR_OK) break;
        launched = true;
        cudaEventRecord(h->ev_sdone, h->s_comp[0]);
        for (int64_t i = 1; i < nch && e == cudaSuccess; i++) land(i);
    }
    if (rc == POLAR_OK && e != cudaSuccess) rc = cuda_status(e);
    if (e != cudaSuccess && launched) {
        // a launch may be waiting for flags that will not come: release it by
        // setting the error word with a stream memory operation (done by the
        // GPU front end, so it needs no free SM); every wait of the launch then
        // returns at once and the host reports the failure below
        wv(reinterpret_cast<CUstream>(h->s_h2d), reinterpret_cast<CUdeviceptr>(err), 1u, 0);
    }
    cudaError_t e2 = cudaStreamSynchronize(h->s_h2d);
    const cudaError_t e3 = cudaStreamSynchronize(h->s_comp[0]);
    if (e2 == cudaSuccess) e2 = e3;
    if (rc == POLAR_OK && e2 != cudaSuccess) rc = cuda_status(e2);
    if (rc == POLAR_OK) {
        uint32_t ev = 0;
        e2 = cudaMemcpy(&ev, err, sizeof(ev), cudaMemcpyDeviceToHost);
        if (e2 != cudaSuccess || ev != 0) rc = POLAR_ECUDA;
    }
    cudaEventDestroy(start);
    return rc;
}

static int decode_host_impl(polar_scs_t h, bool list, const float *llr_host, int64_t n, uint8_t *bits_host,
                            void *stream) {
    if (!h || n < 0) return POLAR_EINVAL;
    if (list && h->list_ctas == 0) return POLAR_ENOTSYS;
    if (n == 0) return POLAR_OK;
    DeviceGuard g(h);
    if (!g.ok) return POLAR_ECUDA;
    if (!llr_host || !bits_host) return POLAR_EINVAL;
    const int N = h->t.N, K = h->t.K;
    cudaError_t e = cudaSuccess;
    if (!h->s_comp[0]) {
        // chunks of up to 256 MiB of LLRs in a ring of up to kStageBufs device
        // buffers, so the copy engine can run several chunks ahead while the
        // decode is slow (low-SNR frames) and the decode catches up on fast
        // stretches; consecutive chunks decode on two streams with separate
        // queue/arena slots, so the next chunk's CTAs fill the SMs while the
        // previous chunk's last frames finish
        h->stage_frames = std::max<int64_t>(1, (int64_t)(256ll << 20) / (4ll * N));
        e = cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking);
        for (int b = 0; b < 2 && e == cudaSuccess; b++) e = cudaStreamCreateWithFlags(&h->s_comp[b], cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking);
        if (e != cudaSuccess) return cuda_status(e);
    }
    static const bool no_stream = std::getenv("POLAR_NO_STREAMING") != nullptr;   // A/B knob: chunked pipeline only
    // Stack decoder only: below 32 MiB of LLRs the fixed costs of the streaming
    // set-up outweigh it, and the list kernel measured slower streaming
    // (C2 e2e 4630 -> 4507 Mbps) while its chunked pipeline already reaches
    // 93% of the device-resident rate
    if (!list && !no_stream && n * 4ll * N >= (32ll << 20)) {
        // streaming when the output buffer is pinned (the kernel writes the bits
        // straight into it) and the GPU front end does stream memory operations
        cudaPointerAttributes pa{};
        if (cudaPointerGetAttributes(&pa, bits_host) == cudaSuccess && pa.type == cudaMemoryTypeHost && pa.devicePointer) {
            const int rs = decode_host_stream(h, llr_host, n, static_cast<uint8_t *>(pa.devicePointer),
                                              static_cast<cudaStream_t>(stream));
            if (rs != 1) return rs;
        }
        cudaGetLastError();
    }
    cudaEvent_t start;
    e = cudaEventCreateWithFlags(&start, cudaEventDisableTiming);
    if (e != cudaSuccess) return cuda_status(e);
    cudaEventRecord(start, static_cast<cudaStream_t>(stream));
    cudaStreamWaitEvent(h->s_h2d, start, 0);
    cudaStreamWaitEvent(h->s_comp[0], start, 0);
    cudaStreamWaitEvent(h->s_comp[1], start, 0);
    int rc = POLAR_OK;
    int64_t i = 0;
    // chunk sizes ramp up geometrically from ~16 MiB, so the first decode
    // starts after a short copy, to the staging size
    // (a batch under 32 MiB starts with half of it, so its two copies overlap
    // the first half's decode)
    int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(h->stage_frames, (int64_t)(16ll << 20) / (4ll * N)));
    if (n * 4ll * N < (32ll << 20)) chunk = std::max<int64_t>(1, std::min<int64_t>(chunk, (n + 1) / 2));
    for (int64_t off = 0; off < n && rc == POLAR_OK; off += chunk, chunk = std::min<int64_t>(2 * chunk, h->stage_frames), i++) {
        const int b = (int)(i % polar_scs_s::kStageBufs), c = (int)(i & 1);
        const int64_t cnt = std::min<int64_t>(chunk, n - off);
        if (!h->d_stage_llr[b]) {
            e = cudaMalloc(&h->d_stage_llr[b], (size_t)h->stage_frames * N * 4);
            if (e == cudaSuccess) e = cudaMalloc(&h->d_stage_bits[b], (size_t)h->stage_frames * K);
            if (e == cudaSuccess && !h->ev_h2d[b]) e = cudaEventCreateWithFlags(&h->ev_h2d[b], cudaEventDisableTiming);
            if (e == cudaSuccess && !h->ev_dec[b]) e = cudaEventCreateWithFlags(&h->ev_dec[b], cudaEventDisableTiming);
            if (e == cudaSuccess && !h->ev_d2h[b]) e = cudaEventCreateWithFlags(&h->ev_d2h[b], cudaEventDisableTiming);
            if (e != cudaSuccess) {
                cudaFree(h->d_stage_llr[b]); cudaFree(h->d_stage_bits[b]);
                h->d_stage_llr[b] = nullptr; h->d_stage_bits[b] = nullptr;
                rc = cuda_status(e);
                break;
            }
        }
        cudaStreamWaitEvent(h->s_h2d, h->ev_dec[b], 0);   // buffer b's previous decode has read it
        e = cudaMemcpyAsync(h->d_stage_llr[b], llr_host + off * N, (size_t)cnt * N * 4, cudaMemcpyHostToDevice, h->s_h2d);
        if (e != cudaSuccess) { rc = cuda_status(e); break; }
        cudaEventRecord(h->ev_h2d[b], h->s_h2d);
        cudaStreamWaitEvent(h->s_comp[c], h->ev_h2d[b], 0);
        cudaStreamWaitEvent(h->s_comp[c], h->ev_d2h[b], 0);   // bits buffer b has been copied out
        rc = list ? list_impl(h, h->d_stage_llr[b], cnt, h->d_stage_bits[b], nullptr, nullptr, h->s_comp[c], c)
                  : decode_impl(h, h->d_stage_llr[b], cnt, h->d_stage_bits[b], nullptr, nullptr, nullptr, nullptr,
                                h->s_comp[c], c);
        cudaEventRecord(h->ev_dec[b], h->s_comp[c]);
        cudaStreamWaitEvent(h->s_d2h, h->ev_dec[b], 0);
        e = cudaMemcpyAsync(bits_host + off * K, h->d_stage_bits[b], (size_t)cnt * K, cudaMemcpyDeviceToHost, h->s_d2h);
        if (e != cudaSuccess) { rc = cuda_status(e); break; }
        cudaEventRecord(h->ev_d2h[b], h->s_d2h);
    }
    e = cudaStreamSynchronize(h->s_d2h);
    if (rc == POLAR_OK && e != cudaSuccess) rc = cuda_status(e);
    for (int b = 0; b < 2; b++) {
        const cudaError_t e2 = cudaStreamSynchronize(h->s_comp[b]);
        if (e == cudaSuccess) e = e2;
    }
    if (rc == POLAR_OK && e != cudaSuccess) rc = cuda_status(e);
    cudaEventDestroy(start);
    return rc;
}

int polar_scs_decode_host(polar_scs_t h, const float *llr_host, int64_t n, uint8_t *bits_host, void *stream) {
    return decode_host_impl(h, false, llr_host, n, bits_host, stream);
}

int polar_scl_decode_host(polar_scs_t h, const float *llr_host, int64_t n, uint8_t *bits_host, void *stream) {
    return decode_host_impl(h, true, llr_host, n, bits_host, stream);
}

int polar_crc_attach_batch(polar_scs_t h, const uint8_t *payload, int64_t n, uint8_t *block, void *stream) {
    if (!h || n < 0) return POLAR_EINVAL;
    if (n == 0) return POLAR_OK;
    DeviceGuard g(h);
    if (!g.ok) return POLAR_ECUDA;
    if (!payload || !block) return POLAR_EINVAL;
    CodecParams p = codec_params(h, n);
    p.payload = payload; p.block_out = block;
    return cuda_status(launch_crc_attach(p, static_cast<cudaStream_t>(stream)));
}

int polar_encode_batch(polar_scs_t h, const uint8_t *block, int64_t n, uint8_t *codeword, void *stream) {
    if (!h || n < 0) return POLAR_EINVAL;
    if (!h->t.systematic_ok && !(h->flags & POLAR_FLAG_NONSYSTEMATIC)) return POLAR_ENOTSYS;
    if (n == 0) return POLAR_OK;
    DeviceGuard g(h);
    if (!g.ok) return POLAR_ECUDA;
    if (!block || !codeword) return POLAR_EINVAL;
    CodecParams p = codec_params(h, n);
    p.block_in = block; p.codeword = codeword;
    return cuda_status(launch_encode(p, static_cast<cudaStream_t>(stream)));
}

int polar_modulate_batch(polar_scs_t h, const uint8_t *codeword, const float *noise, int64_t n, double ebno_db,
                         float *llr, void *stream) {
    if (!h || n < 0) return POLAR_EINVAL;
    if (n == 0) return POLAR_OK;
    DeviceGuard g(h);
    if (!g.ok) return POLAR_ECUDA;
    if (!codeword || !noise || !llr) return POLAR_EINVAL;
    CodecParams p = codec_params(h, n);
    const double var = sigma2_of(ebno_db, (double)h->t.K / (double)h->t.N);
    p.sigma_f = (float)std::sqrt(var);
    p.scale_f = (float)(2.0 / var);
    p.codeword = const_cast<uint8_t *>(codeword); p.noise = noise; p.llr = llr;
    return cuda_status(launch_modulate(p, static_cast<cudaStream_t>(stream)));
}

int polar_generate_batch(polar_scs_t h, uint64_t seed, double ebno_db, int64_t first_frame, int64_t n,
                         uint8_t *block, float *llr, void *stream) {
    if (!h || n < 0 || first_frame < 0) return POLAR_EINVAL;
    if (!h->t.systematic_ok && !(h->flags & POLAR_FLAG_NONSYSTEMATIC)) return POLAR_ENOTSYS;
    if (n == 0) return POLAR_OK;
    DeviceGuard g(h);
    if (!g.ok) return POLAR_ECUDA;
    if (!llr) return POLAR_EINVAL;
    if (h->t.N >= 4 && (reinterpret_cast<uintptr_t>(llr) & 15u)) return POLAR_EINVAL;
    CodecParams p = codec_params(h, n);
    const double var = sigma2_of(ebno_db, (double)h->t.K / (double)h->t.N);
    p.sigma_f = (float)std::sqrt(var);
    p.scale_f = (float)(2.0 / var);
    p.seed = seed; p.first_frame = first_frame; p.block_out = block; p.llr = llr;
    return cuda_status(launch_generate(p, static_cast<cudaStream_t>(stream)));
}

}  // extern "C"

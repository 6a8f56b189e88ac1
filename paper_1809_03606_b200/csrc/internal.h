// internal.h — product-internal definitions of libpolarscs (not part of the ABI).
// The public boundary is include/polar_scs.h.
#pragma once
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/polar_scs.h"

namespace polar {

// Schedule op word: kind | lambda << 3 | phi << 8   (Fig. 5)
enum OpKind : uint32_t { OP_ALPHA = 0, OP_BETA = 1, OP_R0 = 2, OP_R1 = 3, OP_REP = 4, OP_SPC = 5 };
__host__ __device__ inline uint32_t op_make(uint32_t kind, uint32_t lam, uint32_t phi) {
    return kind | (lam << 3) | (phi << 8);
}
__host__ __device__ inline uint32_t op_kind(uint32_t op) { return op & 7u; }
__host__ __device__ inline uint32_t op_lam(uint32_t op) { return (op >> 3) & 31u; }
__host__ __device__ inline uint32_t op_phi(uint32_t op) { return op >> 8; }

constexpr int kMaxN = 4096;
constexpr int kMaxD = 8192;     // D > 128: global-memory stack (the paper's D = NL)
constexpr int kDecodeWarps = 4;      // warps (frames in flight) per decode CTA
// D > 128: the stack is a sorted 32-entry register window (hot) over an
// unsorted global store (cold); 0 builds the scan-every-pop global stack (A/B)
#ifndef POLAR_BIG_HOT
#define POLAR_BIG_HOT 1
#endif
#ifndef POLAR_RECS_SMEM
#define POLAR_RECS_SMEM 1      // per-depth records staged in shared memory (register-stack kernels); 0: read through L1
#endif
constexpr int kColdPad = 8;          // cold entries beyond D before the D-limit drop (one node's candidates)
constexpr int kDecodeMinBlocks = 8;  // launch bound: 32 resident warps/SM => <= 64 registers
constexpr int kCodecWarps = 4;       // warps per CTA of the generator/encoder kernels
constexpr int kListPackedWarps = 4;  // max warps (frames in flight) per CTA of the packed FSSCL kernel

// Host-side compiled code description (host.cpp)
struct CodeTables {
    int N = 0, n = 0, K = 0, c = 0, M = 0;
    uint32_t crc_poly = 0;
    bool systematic_ok = false;
    uint32_t *nodes = nullptr;  int nops = 0;   // decision nodes (kind, lambda, phi) in schedule order
    uint32_t *recs = nullptr;                   // [M+1][16] per-depth records (host.cpp)
    uint16_t *info = nullptr;                   // A ascending, [K]
    uint32_t *crc_tab = nullptr;                // [K] syndrome contribution of block bit k
    uint32_t *crc_bytes = nullptr;              // [nw][4][256] per beta byte (CRC codes)
    uint32_t *info_words = nullptr;             // [max(1,N/32)] bit i set iff i in A
};

// Kernel parameter block of the decoder
struct DecodeParams {
    const float *llr;
    int64_t n_frames;
    uint8_t *out_bits;
    float *pm;
    uint32_t *pops, *switches;
    uint8_t *status;
    const uint32_t *nodes;      // [M] node records; the BETA/ALPHA walk between them is implied
    const uint4 *recs;          // [M+1][4] per-depth records (host.cpp build_host_code)
    const uint16_t *info;
    const uint32_t *crc_tab;
    const uint32_t *crc_bytes;  // [nw][4][256] syndrome contribution of each beta byte (CRC codes)
    unsigned long long *queue;
    uint32_t *snap_global;      // arena when snapshots live in global memory
    unsigned long long *stack_keys;   // D > 128: per warp [D + kColdPad] (PM bits << 32 | serial)
    uint32_t *stack_jsm;        // D > 128: per warp [D + kColdPad] (depth | snapshot | flips)
    uint2 *hdr_global;          // D > 128: per warp [D] fork headers m1..m4
    int N, n, K, c, D, L, M;
    int nw;                     // beta words = max(1, N/32)
    int snap_stride;            // words per snapshot slot = nw (headers m1..m4 in shared memory)
    int sched_words;            // per-depth record words staged in shared memory (0 = read global)
    int warp_words;             // shared-memory words per warp
    int cnt_words;              // words of the per-length counters (u16 each)
    int hdr_words;              // shared-memory fork headers: 2 D (register stacks) or 0
    int used_words;             // snapshot-slot bitmap words: 4, or ceil(D/32) rounded (D > 128)
    int uhat_words;             // nw when non-systematic (u_hat scratch), else 0
    int win_words;              // D > 128, scan stack: shared-memory window of the first 128 keys (256 words); 0 with the hot window
    int alpha_words;            // shared alpha memory (floats): N, or 2^sg when stages >= sg are global
    int sg;                     // first alpha stage kept in the global arena (n: none)
    float *galpha;              // global alpha arena, N floats per resident warp (or null)
    int nonsys;                 // 1: read u_hat = x_hat F restricted to A (non-systematic)
    const uint32_t *ready;      // streaming host pipeline: per-chunk "LLRs landed" flags (null: all resident)
    uint32_t *err;              // streaming: set when a flag wait timed out
    int chunk_shift;            // streaming: log2 frames per chunk
    uint32_t *counts;           // polar_scs_decode_counts: [n_frames] x 4 executed-work counters
    int chan_in_smem, snap_in_smem;   // placement (read by the counting instance only)
};

// Kernel parameter block of the FSSCL list decoder (list_packed.cu).  One warp
// per frame; the shared-memory offsets (in 32-bit words) are computed
// by the host (capi.cu, list_layout).
struct ListParams {
    const float *llr;
    int64_t n_frames;
    uint8_t *out_bits;
    float *pm;
    uint8_t *status;
    const uint32_t *nodes;
    const uint16_t *info;
    const uint32_t *crc_bytes;
    unsigned long long *queue;
    int N, n, K, c, L, M, nw, nonsys;
    int o_alpha, o_beta, o_reg, o_clist, o_mi, o_prow, o_cand, o_sel, o_selpm, o_ok, o_misc, words;
    int o_warp0;                // packed kernel: words before the per-warp blocks (node table)
    int pwarps;                 // packed kernel: warps (frames) per CTA
    int sg;                     // packed kernel: first alpha stage kept in the global arena (n: none)
    float *galpha;              // packed kernel: global alpha arena (stages >= sg), gstride floats per warp
    uint32_t *gbeta;            // packed kernel: the double-buffered path betas in a global arena
                                // (2 L nw words per warp) instead of shared memory (or null)
    int beta_global;            // layout: 1 when gbeta holds the betas
    size_t gstride;
};

struct CodecParams {
    const uint8_t *payload;     // crc attach input
    const uint8_t *block_in;    // encode input
    uint8_t *block_out;
    uint8_t *codeword;
    const float *noise;
    float *llr;
    int64_t n_frames, first_frame;
    uint64_t seed;
    float sigma_f, scale_f;
    int N, n, K, c, nw;
    int nonsys;                 // 1: non-systematic encoding c = u F
    const uint16_t *info;
    const uint32_t *crc_tab;
    const uint32_t *info_words;
};

}  // namespace polar

struct polar_scs_s {
    int device = 0;
    uint32_t flags = 0;
    int D = 0, L = 0;
    polar::CodeTables t;            // device pointers
    unsigned long long *d_queue = nullptr;  // [2] frame-queue counters (slot 0: decode API; 0/1: host pipeline)
    uint32_t *d_snap = nullptr;     // global snapshot arena, 2 slots (or null)
    unsigned long long *d_keys = nullptr;   // global stacks (D > 128), 2 slots
    uint32_t *d_jsm = nullptr;
    uint2 *d_hdr = nullptr;         // global fork headers (D > 128), 2 slots
    float *d_salpha = nullptr;      // global alpha arena of the top stages (stack decoder), 2 slots
    size_t salpha_floats = 0;       // per slot
    size_t stack_count = 0, hdr_count = 0;   // entries per slot
    size_t snap_bytes = 0;          // bytes per slot
    int snap_in_smem = 0;
    int chan_in_smem = 0;
    int warps_per_cta = 0, ctas = 0, smem_per_cta = 0;
    polar::DecodeParams base{};     // prefilled params
    int list_ctas = 0, list_smem = 0, list_lcap = 0;   // FSSCL launch (0 = list decode unsupported)
    int list_packed = 0;            // 1: the warp-per-frame packed FSSCL kernel (list_packed.cu)
    float *d_galpha = nullptr;      // packed FSSCL: global arena of the top alpha stages, 2 slots
    uint32_t *d_gbeta = nullptr;    // packed FSSCL: global arena of the path betas, 2 slots
    polar::ListParams list{};       // prefilled FSSCL params
    // host-staging for polar_scs_decode_host (lazily allocated)
    cudaStream_t s_h2d = nullptr, s_comp[2] = {nullptr, nullptr}, s_d2h = nullptr;
    // host pipeline staging ring (allocated on first use, buffer by buffer)
    static constexpr int kStageBufs = 8;
    float *d_stage_llr[kStageBufs] = {};
    uint8_t *d_stage_bits[kStageBufs] = {};
    cudaEvent_t ev_h2d[kStageBufs] = {}, ev_dec[kStageBufs] = {}, ev_d2h[kStageBufs] = {};
    int64_t stage_frames = 0;
    // streaming host pipeline (capi.cu, decode_host_stream)
    static constexpr int kStreamChunks = 512;   // ready flags per launch (+1 error word)
    uint32_t *d_ready = nullptr;
    float *d_sllr = nullptr;                    // staging of one launch's LLRs
    int64_t stream_cap = 0;                     // frames d_sllr holds
    int stream_ok = 0;                          // 1: memory operations work, -1: not available
    cudaEvent_t ev_sreset = nullptr, ev_sdone = nullptr;
};

// host.cpp — code compilation on the host (validation, schedule, tables)
namespace polar {
struct HostCode {
    int N = 0, n = 0, K = 0, c = 0, M = 0;
    uint32_t crc_poly = 0;
    bool systematic_ok = false;
    std::vector<uint32_t> ops;      // full FSSC schedule (ALPHA/BETA/nodes), Fig. 5
    std::vector<uint32_t> nodes;    // its decision nodes only
    std::vector<uint32_t> recs;     // [M+1][16] per-depth records of the stack decoder
    std::vector<uint16_t> info;
    std::vector<uint32_t> crc_tab;
    std::vector<uint32_t> crc_bytes;
    std::vector<uint32_t> info_words;
};
int build_host_code(int N, int K, const uint8_t *frozen, uint32_t crc_poly, bool bit_level, HostCode &hc);
int crc_degree(uint32_t poly_full);
}  // namespace polar

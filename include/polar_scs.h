/*
 * polar_scs.h — C ABI of the B200-native batched fast-simplified successive
 * cancellation stack (FSSCS-RM) polar decoder.
 *
 * Method: H. Aurora, W. Gross, "Towards Practical Software Stack Decoding of
 * Polar Codes", arXiv:1809.03606.  Citations below are
 * PAPER.md:L<line> (section / equation / algorithm / figure).  Where the paper
 * is silent or garbled the reading adopted is listed in DESIGN.md §Readings
 * (R1..R19); the same readings define the CPU oracle the tests compare with.
 *
 * Conventions (all entry points):
 *   - Return value: POLAR_OK (0) or a negative POLAR_E* code; no exception or
 *     abort crosses the ABI.  polar_scs_strerror() names the code.
 *   - "device" pointers are CUDA device (or managed) memory on the handle's
 *     device; "host" pointers are CPU memory (pinned for full copy speed).
 *     The caller owns every I/O buffer; the handle owns its tables and
 *     workspace, all allocated in polar_scs_create (decode calls allocate
 *     nothing, except the host-staging buffers of polar_scs_decode_host,
 *     allocated once on first use).
 *   - Layouts are row-major per frame: llr [n_frames][N] float32, bits and
 *     codewords [n_frames][K] / [n_frames][N] uint8 holding 0/1.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *     stream).  Device-pointer calls are asynchronous: results are valid once
 *     the stream is synchronised.  A handle serves ONE in-flight call at a
 *     time (its frame queue and snapshot arena are per handle).
 *   - n_frames == 0 is a no-op returning POLAR_OK.
 *   - Input contract: LLRs are finite (NaN/Inf is undefined behaviour).
 */
#ifndef POLAR_SCS_H
#define POLAR_SCS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POLAR_OK        0
#define POLAR_EINVAL   (-1)   /* bad argument (sizes, mask weight, NULL pointer) */
#define POLAR_ENOMEM   (-2)   /* device or host allocation failed                */
#define POLAR_ECUDA    (-3)   /* a CUDA runtime call or kernel launch failed     */
#define POLAR_ENOTSYS  (-4)   /* unsupported for this code (e.g. not systematic) */

/* create() flags */
#define POLAR_FLAG_BIT_LEVEL    0x1u  /* leaf-only schedule: bit-level SCS-RM
                                          */
#define POLAR_FLAG_SNAP_GLOBAL  0x2u  /* force the path-snapshot arena into
                                         global memory (L2) instead of shared */
#define POLAR_FLAG_CHAN_GLOBAL  0x4u  /* read the channel LLR row through L1/L2
                                         instead of staging it in shared memory */
#define POLAR_FLAG_SNAP_SMEM    0x8u  /* force snapshots into shared memory */
#define POLAR_FLAG_CHAN_SMEM    0x10u /* force channel staging in shared memory */
#define POLAR_FLAG_NONSYSTEMATIC 0x40u /* non-systematic code: encoders emit c = u F,
                                          decoders read u_hat = x_hat F restricted to A
                                          (PAPER.md:L503); any mask is allowed */
#define POLAR_FLAG_LIST_CTA     0x80u /* reserved: the CTA-per-frame list kernel was removed
                                         (slower than the packed kernel on every config);
                                         create returns POLAR_EINVAL */
#define POLAR_FLAG_LIST_PACKED  0x100u /* polar_scl_decode: one warp per frame with the L
                                          paths packed across its lanes (the only list
                                          kernel; accepted for compatibility) */

typedef struct polar_scs_s *polar_scs_t;

/* Read-only description of a handle (for benches and tests). */
typedef struct {
    int32_t N, n, K, crc_bits, D, L;
    int32_t num_ops;          /* FSSC schedule length |S|        */
    int32_t num_nodes;        /* M = decision nodes in the schedule               */
    int32_t warps_per_cta, ctas, smem_per_cta;  /* decode launch configuration   */
    int32_t snap_in_smem;     /* 1: path snapshots in shared memory, 0: global    */
    int32_t chan_in_smem;     /* 1: channel row staged in shared memory           */
    int32_t systematic_ok;    /* 1 if the mask is systematic-encodable            */
    uint32_t flags;
    int32_t list_ctas, list_smem_per_cta;  /* polar_scl_decode launch (0: unsupported) */
    int32_t list_packed;      /* 1: warp-per-frame packed FSSCL kernel, 0: CTA of L warps */
    int32_t list_warps_per_cta;
} polar_scs_info_t;

/*
 * Bhattacharyya-parameter code construction (host only, no device work).
 * z0 = exp(-(K/N) 10^(EbN0/10)); the bits of index i, MSB first, map
 * 1 -> z^2 and 0 -> 2z - z^2 (BEC bound), in the log domain; the K indices
 * of smallest z carry information (ties: higher index).
 * (information set A); reading R16.
 *   N: power of two in [1, 65536]; 0 <= K <= N; frozen_mask: host [N],
 *   written 1 = frozen, 0 = information.  Returns POLAR_EINVAL on bad sizes.
 */
int polar_construct_bhattacharyya(int32_t N, int32_t K, double design_ebno_db, uint8_t *frozen_mask);

/*
 * Information set from a user-supplied reliability sequence listed LEAST
 * reliable first (SPEC.md:L42-44 format; e.g. the 3GPP TS 38.212 sequence the
 * paper uses, PAPER.md:L966 — not shipped): the K most reliable entries below N
 * carry information.  seq: host [len], a permutation of [0, len) with len >= N;
 * frozen_mask: host [N] output.  POLAR_EINVAL on a bad sequence or sizes.
 */
int polar_construct_from_sequence(int32_t N, int32_t K, const int32_t *seq, int32_t len, uint8_t *frozen_mask);

/*
 * Create a decoder for PC(N, K) with a stack of depth D and
 * per-length visit limit L and an optional CRC selecting
 * among complete paths.  Compiles the FSSC schedule
 * (Fig. 5; node precedence R0 > R1 > REP > SPC, reading R5),
 * uploads it with the information-set and CRC tables, and sizes the
 * persistent decode launch and its workspace.  Host only + cudaMalloc/copies.
 *   N: power of two in [2, 4096]; K = number of information bits INCLUDING
 *   the crc bits (reading R14), 1 <= K <= N; frozen_mask: host [N], 1 =
 *   frozen, must have exactly N-K ones; D in [1, 8192] (D <= 128: the stack
 *   lives in registers; D > 128, up to the paper's D = NL = 8192 (PAPER.md:
 *   L599, L966): a per-warp stack in global memory, L2-resident in practice,
 *   with its snapshot arena of D x N/8 bytes per resident warp); L in
 *   [1, 65536] (16-bit per-depth counters; exact over the whole range since
 *   the L-th pop at a depth prunes that depth for good); crc_poly: 0 = none, else the full
 *   generator including the x^c term (0x11021 = CRC-16 0x1021, 0x107 = CRC-8
 *   0x07), degree c in [1, 31] and c < K; flags: POLAR_FLAG_*.
 *   On success *out receives the handle (owned by the caller; release with
 *   polar_scs_destroy).  Errors: POLAR_EINVAL, POLAR_ENOMEM, POLAR_ECUDA.
 */
int polar_scs_create(polar_scs_t *out, int32_t N, int32_t K, const uint8_t *frozen_mask,
                     int32_t stack_depth_D, int32_t visit_limit_L, uint32_t crc_poly);
int polar_scs_create_ex(polar_scs_t *out, int32_t N, int32_t K, const uint8_t *frozen_mask,
                        int32_t stack_depth_D, int32_t visit_limit_L, uint32_t crc_poly,
                        uint32_t flags);

void polar_scs_destroy(polar_scs_t h);                 /* NULL is a no-op */
int  polar_scs_get_info(polar_scs_t h, polar_scs_info_t *out);
const char *polar_scs_strerror(int status);

/*
 * Decode n_frames independent frames with the FSSCS-RM stack decoder
 * (PAPER.md:L589-599 SCS; L797-799 reduced memory; L815-842 Alg. 4 alpha
 * recompute on a path switch; L846-854 fast-simplified nodes, schedule
 * progress and flat beta).  One warp per frame, persistent kernel with a
 * frame queue.
 *   llr: device [n_frames][N] float32 channel LLRs (positive favours 0),
 *   rows 16-byte aligned when N >= 4.
 *   out_bits: device [n_frames][K] uint8 — the decoded K-bit block (payload ||
 *   CRC), read from the systematic codeword estimate x_hat at the ascending
 *   information indices (reading R15).
 * polar_scs_decode_stats additionally writes, per frame (any may be NULL):
 *   pm: final path metric (float32, PAPER.md:L511-517 Eq. PMupd summed over
 *   nodes), pops: stack pops (selections), switches: path switches (pops of
 *   a path other than the one just extended), status: 0 = a complete path
 *   passed the CRC (or no CRC), 1 = every complete path failed the CRC and
 *   the first complete path popped is returned (reading R13).
 */
int polar_scs_decode(polar_scs_t h, const float *llr, int64_t n_frames, uint8_t *out_bits,
                     void *stream);
int polar_scs_decode_stats(polar_scs_t h, const float *llr, int64_t n_frames, uint8_t *out_bits,
                           float *pm, uint32_t *pops, uint32_t *switches, uint8_t *status,
                           void *stream);

/*
 * Instrumented decode for roofline accounting: the same decode as
 * polar_scs_decode (identical out_bits) by an instance of the kernel that
 * also counts, per frame, the work it executed:
 *   counts: device [n_frames][4] uint32, 16-byte aligned:
 *     [0] f/g evaluations (Eq. 4; Alg. 4 spines after a switch start at the
 *         first alpha stage whose node or beta prefix changed, reading R12),
 *     [1] bits XOR-ed by BETA ops,
 *     [2] node elements (sum of Lambda over decision-node visits, L846),
 *     [3] 32-bit words moved into or out of beta snapshots (L854).
 * Slower than polar_scs_decode (a generic, unspecialised instance): for
 * measurement, not for throughput.  Errors as polar_scs_decode.
 */
int polar_scs_decode_counts(polar_scs_t h, const float *llr, int64_t n_frames, uint8_t *out_bits,
                            uint32_t *counts, void *stream);

/*
 * Decode n_frames independent frames with the FSSCL LIST decoder (PAPER.md:
 * L505-519 SCL; L521-587 fast-simplified node path creation; L772-780 list
 * memory with lazy copy), list size = the handle's L (the visit limit that
 * gives the stack decoder "the same search space as SCL").
 * With POLAR_FLAG_BIT_LEVEL the handle's leaf-only schedule gives plain SCL.
 * At every decision node each of the <= L paths creates its node candidates
 * and the L smallest keys (PM, parent rank, candidate rank) survive (reading
 * R22); the output is the first path of the final list, in rank order, whose
 * block passes the CRC (the first path without a CRC); if none passes, the
 * first path with status 1 (reading R24).  One CTA of L warps per frame,
 * persistent kernel with a frame queue; D is not used.
 *   llr, out_bits: as polar_scs_decode.  pm: device [n] float32 final PM of the
 *   output path (may be NULL); status: device [n] uint8 (may be NULL).
 *   POLAR_ENOTSYS if L > 32 or the per-frame list memory (about 4 L N bytes
 *   of alpha plus 8 L N/32 bytes of beta) does not fit in shared memory; the
 *   handle's D limits do not apply.  Shares the handle's frame queue: one
 *   in-flight call per handle, as for the stack decoder.
 */
int polar_scl_decode(polar_scs_t h, const float *llr, int64_t n_frames, uint8_t *out_bits,
                     float *pm, uint8_t *status, void *stream);

/*
 * End-to-end decode from HOST buffers: llr_host ([n][N] float32) in,
 * out_bits_host ([n][K] uint8) out.  Two internal pipelines:
 *   - streaming (stack decoder, out_bits_host pinned / device-accessible, at
 *     least 32 MiB of LLRs, stream memory operations available): one decode
 *     launch per batch of up to 512 chunks (chunks of 256 KiB .. 8 MiB of
 *     LLRs), started before the LLRs arrive; each chunk's H2D copy is followed
 *     by a stream-ordered flag write that releases its frames to the kernel,
 *     which writes the bits straight into out_bits_host.  Staging: one device
 *     buffer of up to 4 GiB of LLRs, kept by the handle.
 *   - chunked (otherwise, and for polar_scl_decode_host): chunks of 16 MiB
 *     ramping to 256 MiB of LLRs in a ring of up to 8 device buffers, each
 *     chunk copied in, decoded (two decode slots) and its bits copied out on
 *     internal streams, later copies overlapping earlier decodes.
 * Staging is allocated on first use (POLAR_ENOMEM if that fails; the call
 * then returns without completing the batch).  POLAR_ECUDA if a streaming
 * chunk's flag never arrives (the kernel gives up after > 17 s).  Blocking:
 * returns when out_bits_host is complete.  Pinned host memory gives full
 * PCIe/C2C speed.  `stream` orders the call after prior work on it.
 * The environment variable POLAR_NO_STREAMING forces the chunked pipeline.
 */
int polar_scs_decode_host(polar_scs_t h, const float *llr_host, int64_t n_frames,
                          uint8_t *out_bits_host, void *stream);
/* The same host-buffer pipeline around the FSSCL list decoder (polar_scl_decode). */
int polar_scl_decode_host(polar_scs_t h, const float *llr_host, int64_t n_frames,
                          uint8_t *out_bits_host, void *stream);

/*
 * CRC attach: block = payload || crc(payload), CRC computed MSB first with zero
 * init, no reflection, no output XOR.
 *   payload: device [n][K-c] uint8; block: device [n][K] uint8.
 *   Without a CRC the payload is copied.
 */
int polar_crc_attach_batch(polar_scs_t h, const uint8_t *payload, int64_t n_frames,
                           uint8_t *block, void *stream);

/*
 * Systematic encoding (PAPER.md:L30-36 c = u F^{(x)n}; L503, L854): u[A] =
 * block, u[A^c] = 0, x = u F^{(x)n}, zero x on A^c, codeword = x F^{(x)n};
 * then codeword restricted to A (ascending) equals block.
 *   block: device [n][K] uint8; codeword: device [n][N] uint8.
 *   POLAR_ENOTSYS if the mask is not systematic-encodable.
 */
int polar_encode_batch(polar_scs_t h, const uint8_t *block, int64_t n_frames,
                       uint8_t *codeword, void *stream);

/*
 * BPSK over AWGN with caller-supplied unit normals (formula
 * SURVEY §8(c) O4): sigma^2 = 1/(2 (K/N) 10^(EbN0/10)), sigma_f = (float)sigma,
 * scale_f = (float)(2/sigma^2) computed in double on the host, then per bit
 * llr = scale_f * ((1 - 2 x) + sigma_f * noise), two float32 roundings, no FMA.
 *   codeword: device [n][N] uint8; noise: device [n][N] float32; llr: device
 *   [n][N] float32.
 */
int polar_modulate_batch(polar_scs_t h, const uint8_t *codeword, const float *noise,
                         int64_t n_frames, double ebno_db, float *llr, void *stream);

/*
 * Seeded device-side workload generator (one fused kernel): Philox4x32-10
 * payload bits (stream 0) -> CRC attach -> systematic encode -> Philox unit
 * normals (stream 1, Box-Muller in double) -> BPSK/AWGN LLRs as in
 * polar_modulate_batch.  Counter layout: DESIGN.md §Input recipe; frame f of
 * the batch is global frame first_frame + f, so any frame range is
 * reproducible independently.
 *   block: device [n][K] uint8 (may be NULL); llr: device [n][N] float32.
 */
int polar_generate_batch(polar_scs_t h, uint64_t seed, double ebno_db, int64_t first_frame,
                         int64_t n_frames, uint8_t *block, float *llr, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* POLAR_SCS_H */

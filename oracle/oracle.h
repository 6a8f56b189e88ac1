/*
 * oracle.h — CPU ORACLE for the FSSCS-RM polar decoder.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference leg may load this library.  The product path
 * (paper_1809_03606_b200/) never imports, links or executes it, and this file
 * shares no code, header, table or constant generator with the product.
 *
 * Every function follows a passage of PAPER.md ("Towards Practical Software
 * Stack Decoding of Polar Codes", Aurora & Gross, arXiv:1809.03606); the
 * citation is PAPER.md:L<line> (section / equation / algorithm / figure).
 * Where the paper is silent or garbled the reading is the one listed in
 * SURVEY.md §8(c) and DESIGN.md "Readings" (R1..R26).  Parity unpinned (see
 * oracle.c): Bhattacharyya sets for N > 16 beyond closure; search counts for
 * N > 64.
 *
 * Arithmetic: alpha values and path metrics are IEEE float32 (PAPER.md:L968,
 * "alpha ... implemented using 32-bit floating point numbers"); the library is
 * built with -O2 -ffp-contract=off and without fast-math so every float op is
 * a single correctly-rounded IEEE operation in the order written.
 */
#ifndef POLAR_ORACLE_H
#define POLAR_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* schedule op kinds (Fig. 5) */
enum { ORC_ALPHA = 0, ORC_BETA = 1, ORC_R0 = 2, ORC_R1 = 3, ORC_REP = 4, ORC_SPC = 5 };

/* O1 — Bhattacharyya construction (BASELINE.json configs; reading R16). */
int orc_bhattacharyya_mask(int N, int K, double design_ebno_db, uint8_t *frozen /* [N], 1=frozen */);

/* O1b — information set from a reliability sequence (least reliable first):
 * A = the K most reliable entries < N (the paper's 3GPP
 * sequence, is user-supplied).  -1 if seq is not a permutation
 * of [0, len) or has fewer than N entries < N. */
int orc_mask_from_sequence(int N, int K, const int32_t *seq, int len, uint8_t *frozen);

/* O2 — x <- x F^{(x)n} in place, n butterfly stages (Fig. 1). */
void orc_polar_transform(int N, uint8_t *x);
/* O2 — systematic encoding: u[A]=block, u[A^c]=0, encode, zero A^c, encode
 * (SPEC.md:L67).  Returns 0, or -1 if N invalid. */
int orc_encode_systematic(int N, const uint8_t *frozen, const uint8_t *block /* [K] */, uint8_t *codeword /* [N] */);
/* O2 — non-systematic encoding: u[A] = block, u[A^c] = 0, c = u F^{(x)n} */
int orc_encode_nonsystematic(int N, const uint8_t *frozen, const uint8_t *block, uint8_t *codeword);

/* O3 — CRC remainder of bits * x^c mod poly (MSB first, zero init, no
 * reflection, no xorout).  poly_full includes the
 * x^c term (0x11021 = CRC-16 0x1021, 0x107 = CRC-8 0x07).  Writes c bits
 * (MSB first) and returns c, or -1 for poly_full < 2. */
int orc_crc_bits(const uint8_t *bits, int nbits, uint32_t poly_full, uint8_t *crc_out);
/* degree c of a full generator polynomial (0 if poly_full == 0) */
int orc_crc_degree(uint32_t poly_full);

/* O4 — channel: sigma^2 = 1/(2 R 10^(EbN0/10)); sigma_f = (float)sigma,
 * scale_f = (float)(2/sigma^2). */
void orc_sigma(double ebno_db, double rate, float *sigma_f, float *scale_f);
/* LLR_i = scale_f * ((1 - 2 x_i) + sigma_f * n_i), two float32 ops, no FMA */
void orc_awgn_llr(int N, const uint8_t *codeword, const float *noise, float sigma_f, float scale_f, float *llr);

/* O5 — FSSC schedule (Fig. 5).  bit_level=1 emits only
 * leaf (Lambda=1) nodes.  ops[k] = kind | lambda<<8 | phi<<16.  Returns the
 * number of ops, or -(needed) if cap is too small. */
int orc_build_schedule(int N, const uint8_t *frozen, int bit_level, int32_t *ops, int cap);

/* primitives (Eq. 1-3; g corrected per reading R1) */
float orc_f(float a, float b);
float orc_g(float a_lo, float a_hi, int beta);
int   orc_hd(float x);

/* node candidates (test hook): sorted by (dPM, mask); returns their count */
int orc_node_candidates(int kind, const float *a, int Lam, float *dpm, int *mask, uint8_t *segs);

/* O6 — textbook recursive SC (Alg. 1-2 structure) */
void orc_sc_decode(int N, const uint8_t *frozen, const float *llr, uint8_t *u_hat /* [N] */, uint8_t *x_hat /* [N] */);

/* O7 — the FSSCS-RM engine */
typedef struct orc_scs_s orc_scs_t;
/* counters (O10) accumulated per decoded frame */
typedef struct {
    uint64_t pops, switches;
    uint64_t f_ops, g_ops;          /* f/g evaluations (clean pass + spines) */
    uint64_t spine_elems;           /* f/g evaluated inside spine recomputes */
    uint64_t beta_xor_bits;         /* bits XOR-ed by BETA ops */
    uint64_t node_elems;            /* alpha elements read by node ops */
    uint64_t node_visits;           /* node ops executed */
    uint64_t cand_created, cand_inserted, cand_replaced, cand_dropped;
    uint64_t pruned;                /* entries removed by the per-length rule */
    uint64_t crc_checks;
    uint64_t sel_compares;
    uint64_t stack_peak;            /* stack decoder: max live entries seen (a max, not a sum) */
    uint64_t key_compares;          /* stack decoder: entries examined by the linear searches
                                       (selection, L793, and worst-entry search, L599) */
    uint64_t fg_reuse;              /* stack decoder: f/g of the stage-reuse model (alpha_op in
                                       oracle.c): a lower bound on what a decoder that keeps the
                                       alpha stages must evaluate; f_ops + g_ops (Alg. 4 spines)
                                       is the upper bound */
} orc_counters_t;

orc_scs_t *orc_scs_create(int N, const uint8_t *frozen, int D, int L, uint32_t crc_poly, int bit_level);
/* nonsystematic = 1: the block (and the CRC check) is u_hat restricted to A,
 * u_hat = x_hat F^{(x)n} — re-encoding the root beta */
orc_scs_t *orc_scs_create_ex(int N, const uint8_t *frozen, int D, int L, uint32_t crc_poly, int bit_level,
                             int nonsystematic);
void orc_scs_destroy(orc_scs_t *h);
int  orc_scs_num_ops(const orc_scs_t *h);
int  orc_scs_num_nodes(const orc_scs_t *h);
int  orc_scs_K(const orc_scs_t *h);
/* Decode n_frames rows of llr ([n][N] float32).  Any of the outputs may be NULL.
 * block: [n][K] u8; xhat: [n][N] u8; status: 0 ok, 1 CRC failed (best effort).
 * Returns 0 or -1 (allocation failure). */
int orc_scs_decode(const orc_scs_t *h, const float *llr, int64_t n_frames,
                   uint8_t *block, uint8_t *xhat, float *pm, uint32_t *pops,
                   uint32_t *switches, uint8_t *status, orc_counters_t *counters);

/* O11 — the FSSCL list decoder (readings R22-R24).
 * L = list size.  bit_level = 1 gives plain SCL (leaf nodes only).  Outputs as
 * orc_scs_decode; crc_checks[f] = complete paths CRC-checked before the pick. */
typedef struct orc_scl_s orc_scl_t;
orc_scl_t *orc_scl_create(int N, const uint8_t *frozen, int L, uint32_t crc_poly, int bit_level, int nonsystematic);
void orc_scl_destroy(orc_scl_t *h);
int  orc_scl_K(const orc_scl_t *h);
int  orc_scl_num_nodes(const orc_scl_t *h);
int  orc_scl_decode(const orc_scl_t *h, const float *llr, int64_t n_frames, uint8_t *block, uint8_t *xhat,
                    float *pm, uint8_t *status, uint32_t *crc_checks, orc_counters_t *counters);

#ifdef __cplusplus
}
#endif
#endif

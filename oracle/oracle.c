/*
 * oracle.c — plain, slow, obviously-correct CPU ORACLE of the FSSCS-RM polar
 * decoder.  TEST INFRASTRUCTURE ONLY (see oracle.h): only tests/, smoke() and
 * bench.py's CPU-baseline / reference leg may load it; it shares no code with
 * the CUDA product path and neither side includes the other.
 *
 * It follows PAPER.md step by step, in the paper's order and notation
 * (lambda = stage, phi = branch, Lambda = 2^lambda, alpha = LLR memory,
 * beta = bit estimates).  Readings of silent/garbled passages: DESIGN.md
 * "Readings" R1..R26 (R1..R19 = SURVEY.md §8(c)).
 *
 * Pins (tests/test_oracle*.py): every part is checked against the paper's
 * worked examples, closed forms, textbook SC, brute-force ML, the DFS optimum
 * of the candidate tree, and (search counts, PM, bits) an independent plain
 * SCS / SCL written in Python.  Parity unpinned: the Bhattacharyya set for
 * N > 16 beyond its partial-order closure (an input both sides share), and
 * the stack search counts for N > 64 (the pinned engine is the same code).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fPIC -shared.
 */
#include "oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

static int ilog2(int N)
{
    int n = 0;
    while ((1 << n) < N) n++;
    return ((1 << n) == N) ? n : -1;
}

/* ------------------------------------------------------------------------ */
/* O1  Bhattacharyya construction (reading R16).  z0 = exp(-R*10^(EbN0/10)),
 * R = K/N.  The bits of the channel index are walked MSB -> LSB because the
 * root-level transform is the first split of the natural-order SC tree
 * (Eq. 4): bit 1 (right child, g) -> z^2; bit 0 (left
 * child, f) -> 2z - z^2 (BEC bound).  Log domain, double precision.  A =
 * the K indices of smallest ln z; ties -> higher index first.               */
int orc_bhattacharyya_mask(int N, int K, double design_ebno_db, uint8_t *frozen)
{
    int n = ilog2(N);
    if (n < 0 || K < 0 || K > N) return -1;
    double R = (double)K / (double)N;
    double lz0 = -R * pow(10.0, design_ebno_db / 10.0);
    double *lz = (double *)malloc(sizeof(double) * (size_t)N);
    int *idx = (int *)malloc(sizeof(int) * (size_t)N);
    if (!lz || !idx) { free(lz); free(idx); return -1; }
    for (int i = 0; i < N; i++) {
        double l = lz0;
        for (int b = n - 1; b >= 0; b--) {
            if ((i >> b) & 1) l = 2.0 * l;                 /* z+ = z^2       */
            else              l = l + log(2.0 - exp(l));   /* z- = 2z - z^2  */
        }
        lz[i] = l;
        idx[i] = i;
    }
    /* plain insertion sort by (ln z ascending, index descending) */
    for (int a = 1; a < N; a++) {
        int v = idx[a];
        int b = a - 1;
        while (b >= 0 && (lz[idx[b]] > lz[v] || (lz[idx[b]] == lz[v] && idx[b] < v))) {
            idx[b + 1] = idx[b];
            b--;
        }
        idx[b + 1] = v;
    }
    for (int i = 0; i < N; i++) frozen[i] = 1;
    for (int r = 0; r < K; r++) frozen[idx[r]] = 0;
    free(lz);
    free(idx);
    return 0;
}

/* O1b  information set from a reliability sequence, least reliable first
 * (SPEC.md:L42-44): keep the entries < N in order; the last K are A.       */
int orc_mask_from_sequence(int N, int K, const int32_t *seq, int len, uint8_t *frozen)
{
    if (ilog2(N) < 0 || K < 0 || K > N || len < N || !seq) return -1;
    uint8_t *seen = (uint8_t *)calloc((size_t)len, 1);
    int *sub = (int *)malloc(sizeof(int) * (size_t)N);
    int ok = seen && sub, m = 0;
    for (int i = 0; ok && i < len; i++) {
        if (seq[i] < 0 || seq[i] >= len || seen[seq[i]]) ok = 0;
        else { seen[seq[i]] = 1; if (seq[i] < N) sub[m++] = seq[i]; }
    }
    if (ok && m != N) ok = 0;
    if (ok) {
        for (int i = 0; i < N; i++) frozen[i] = 1;
        for (int r = N - K; r < N; r++) frozen[sub[r]] = 0;
    }
    free(seen); free(sub);
    return ok ? 0 : -1;
}

/* ------------------------------------------------------------------------ */
/* O2  c = u F^{(x)n}, F = [[1,0],[1,1]]: the n-stage XOR tree of Fig. 1
 * (PAPER.md:L30-36).  Stage with span h: x[i] ^= x[i+h] for (i & h) == 0.  */
void orc_polar_transform(int N, uint8_t *x)
{
    for (int h = 1; h < N; h *= 2)
        for (int i = 0; i < N; i++)
            if ((i & h) == 0) x[i] ^= x[i + h];
}

/* systematic encoding ("with systematic encoding ... u
 * directly available in beta_(n,0)"; construction SPEC.md:L67).          */
int orc_encode_systematic(int N, const uint8_t *frozen, const uint8_t *block, uint8_t *codeword)
{
    if (ilog2(N) < 0) return -1;
    int k = 0;
    for (int i = 0; i < N; i++) codeword[i] = frozen[i] ? 0 : (uint8_t)(block[k++] & 1);
    orc_polar_transform(N, codeword);
    for (int i = 0; i < N; i++) if (frozen[i]) codeword[i] = 0;
    orc_polar_transform(N, codeword);
    return 0;
}

int orc_encode_nonsystematic(int N, const uint8_t *frozen, const uint8_t *block, uint8_t *codeword)
{
    if (ilog2(N) < 0) return -1;
    int k = 0;
    for (int i = 0; i < N; i++) codeword[i] = frozen[i] ? 0 : (uint8_t)(block[k++] & 1);
    orc_polar_transform(N, codeword);
    return 0;
}

/* ------------------------------------------------------------------------ */
/* O3  CRC by bitwise polynomial long division.       */
int orc_crc_degree(uint32_t poly_full)
{
    int c = 0;
    if (poly_full == 0) return 0;
    while ((poly_full >> (c + 1)) != 0) c++;
    return c;
}

int orc_crc_bits(const uint8_t *bits, int nbits, uint32_t poly_full, uint8_t *crc_out)
{
    if (poly_full < 2) return -1;
    int c = orc_crc_degree(poly_full);
    /* dividend = bits followed by c zeros; long division bit by bit */
    int total = nbits + c;
    uint8_t *r = (uint8_t *)calloc((size_t)total, 1);
    if (!r) return -1;
    for (int i = 0; i < nbits; i++) r[i] = bits[i] & 1;
    for (int i = 0; i < nbits; i++) {
        if (r[i]) {
            for (int d = 0; d <= c; d++)            /* subtract poly * x^(...) */
                r[i + d] ^= (uint8_t)((poly_full >> (c - d)) & 1);
        }
    }
    for (int d = 0; d < c; d++) crc_out[d] = r[nbits + d];
    free(r);
    return c;
}

/* ------------------------------------------------------------------------ */
/* O4  BPSK over AWGN (PAPER.md:L966-968 gives no formula).   */
void orc_sigma(double ebno_db, double rate, float *sigma_f, float *scale_f)
{
    double var = 1.0 / (2.0 * rate * pow(10.0, ebno_db / 10.0));
    *sigma_f = (float)sqrt(var);
    *scale_f = (float)(2.0 / var);
}

void orc_awgn_llr(int N, const uint8_t *codeword, const float *noise, float sigma_f, float scale_f, float *llr)
{
    for (int i = 0; i < N; i++) {
        float s = codeword[i] ? -1.0f : 1.0f;    /* BPSK 0 -> +1, 1 -> -1 */
        float y = s + sigma_f * noise[i];          /* two roundings (no FMA) */
        llr[i] = scale_f * y;
    }
}

/* ------------------------------------------------------------------------ */
/* primitives.  Eq. (1) PAPER.md:L288 min-sum f; Eq. (2) PAPER.md:L289 g,
 * CORRECTED per reading R1: the paper's alpha0 + (-1)^beta alpha1 is
 * transposed w.r.t. its own F (L28) and beta rule (L451-452); the right-child
 * LLR is alpha_p[i+Lambda] + (1-2 beta) alpha_p[i].  HD per Eq. (3), R2.    */
int orc_hd(float x) { return x < 0.0f ? 1 : 0; }

float orc_f(float a, float b)
{
    float m = fminf(fabsf(a), fabsf(b));
    return ((a < 0.0f) != (b < 0.0f)) ? -m : m;
}

float orc_g(float a_lo, float a_hi, int beta) { return beta ? (a_hi - a_lo) : (a_hi + a_lo); }

/* ------------------------------------------------------------------------ */
/* O5  FSSC schedule ("created and stored as the decoder is
 * instantiated", Fig. 5).  Node classes with precedence
 * R0 > R1 > REP > SPC at every size (reading R5).                           */
typedef struct { int32_t *ops; int len, cap; } sched_buf;

static void emit(sched_buf *s, int kind, int lam, int phi)
{
    if (s->len < s->cap) s->ops[s->len] = kind | (lam << 8) | (phi << 16);
    s->len++;
}

static int classify(const uint8_t *frozen, int lam, int phi, int bit_level)
{
    int Lam = 1 << lam, base = phi * Lam, nf = 0;
    for (int i = 0; i < Lam; i++) nf += frozen[base + i] ? 1 : 0;
    if (bit_level && lam > 0) return -1;
    if (nf == Lam) return ORC_R0;                        /* all frozen        */
    if (nf == 0) return ORC_R1;                          /* all information   */
    if (nf == Lam - 1 && !frozen[base + Lam - 1]) return ORC_REP; /* only last info */
    if (nf == 1 && frozen[base]) return ORC_SPC;         /* only first frozen */
    return -1;
}

static void rec(sched_buf *s, const uint8_t *frozen, int lam, int phi, int bit_level)
{
    int kind = classify(frozen, lam, phi, bit_level);
    if (kind >= 0) { emit(s, kind, lam, phi); return; }
    for (int c = 2 * phi; c <= 2 * phi + 1; c++) {
        emit(s, ORC_ALPHA, lam - 1, c);                  /* Eq. (4)           */
        rec(s, frozen, lam - 1, c, bit_level);
    }
    emit(s, ORC_BETA, lam - 1, 2 * phi + 1);             /* Eq. bitcalc       */
}

int orc_build_schedule(int N, const uint8_t *frozen, int bit_level, int32_t *ops, int cap)
{
    int n = ilog2(N);
    if (n < 0) return 0;
    sched_buf s = { ops, 0, cap };
    rec(&s, frozen, n, 0, bit_level);
    return (s.len <= cap) ? s.len : -s.len;
}

/* ------------------------------------------------------------------------ */
/* O6  Textbook SC decoding: recursive f to the left
 * child, decide it, g to the right child with its beta, then combine
 * beta_v[i] = beta_l[i] ^ beta_r[i], beta_v[i+Lambda/2] = beta_r[i]
 * (Eq. bitcalc).  Leaves follow Eq. (3).                 */
static void sc_rec(int lam, int phi, const float *a, const uint8_t *frozen, uint8_t *u_hat, uint8_t *beta)
{
    if (lam == 0) {
        beta[0] = frozen[phi] ? 0 : (uint8_t)orc_hd(a[0]);
        u_hat[phi] = beta[0];
        return;
    }
    int h = 1 << (lam - 1);
    float *child = (float *)calloc((size_t)h, sizeof(float));
    uint8_t *bl = (uint8_t *)malloc((size_t)h), *br = (uint8_t *)malloc((size_t)h);
    for (int i = 0; i < h; i++) child[i] = orc_f(a[i], a[i + h]);
    sc_rec(lam - 1, 2 * phi, child, frozen, u_hat, bl);
    for (int i = 0; i < h; i++) child[i] = orc_g(a[i], a[i + h], bl[i]);
    sc_rec(lam - 1, 2 * phi + 1, child, frozen, u_hat, br);
    for (int i = 0; i < h; i++) { beta[i] = bl[i] ^ br[i]; beta[i + h] = br[i]; }
    free(child); free(bl); free(br);
}

void orc_sc_decode(int N, const uint8_t *frozen, const float *llr, uint8_t *u_hat, uint8_t *x_hat)
{
    int n = ilog2(N);
    uint8_t *beta = (uint8_t *)malloc((size_t)N);
    sc_rec(n, 0, llr, frozen, u_hat, beta);
    if (x_hat) memcpy(x_hat, beta, (size_t)N);
    free(beta);
}

/* ------------------------------------------------------------------------ */
/* Node candidate rules (FSSCL path creation, applied to
 * the stack per L846).  A candidate = (segment bits, dPM, mask).  Sums use
 * the butterfly tree order T (reading R3); argmin keys are (|alpha| bits,
 * index) (reading R4); candidates are sorted by (dPM, mask) (reading R7).   */
typedef struct { float dpm; int mask; } cand_t;

/* T(v): for h = Lambda/2 .. 1: v[i] = v[i] + v[i+h], i < h.  Destroys v.   */
static float tree_sum(float *v, int Lam)
{
    for (int h = Lam / 2; h >= 1; h /= 2)
        for (int i = 0; i < h; i++) v[i] = v[i] + v[i + h];
    return v[0];
}

static uint32_t fbits(float x) { uint32_t u; memcpy(&u, &x, 4); return u; }

/* the `cnt` smallest (|a| bits, index) keys, ascending; plain selection.   */
static void least_reliable(const float *a, int Lam, int cnt, int *m)
{
    for (int r = 0; r < cnt; r++) {
        int best = -1;
        for (int i = 0; i < Lam; i++) {
            int used = 0;
            for (int q = 0; q < r; q++) used |= (m[q] == i);
            if (used) continue;
            if (best < 0 || fbits(fabsf(a[i])) < fbits(fabsf(a[best]))) best = i;
            /* equal keys keep the lower index: scan is ascending */
        }
        m[r] = best;
    }
}

static int popcount4(int x) { return (x & 1) + ((x >> 1) & 1) + ((x >> 2) & 1) + ((x >> 3) & 1); }

/* Build the candidates of node `kind` over a[0..Lam).  seg_base receives the
 * c-independent base word (HD word, or zeros); a candidate's segment is the
 * base with its flip set applied (flip set = mask over m[], or, for REP, the
 * whole segment when mask == 1).  Returns the number of candidates, sorted. */
static int node_candidates(int kind, const float *a, int Lam, uint8_t *seg_base, int *m, cand_t *c, float *tmp)
{
    int nc = 0;
    switch (kind) {
    case ORC_R0:   /* beta = 0; dPM = sum HD(a)|a| */
        for (int i = 0; i < Lam; i++) { seg_base[i] = 0; tmp[i] = a[i] < 0.0f ? -a[i] : 0.0f; }
        c[0].dpm = tree_sum(tmp, Lam); c[0].mask = 0; nc = 1;
        break;
    case ORC_REP: { /* all-0 / all-1 with complementary dPM */
        for (int i = 0; i < Lam; i++) { seg_base[i] = 0; tmp[i] = a[i] < 0.0f ? -a[i] : 0.0f; }
        c[0].dpm = tree_sum(tmp, Lam); c[0].mask = 0;
        for (int i = 0; i < Lam; i++) tmp[i] = a[i] < 0.0f ? 0.0f : a[i];
        c[1].dpm = tree_sum(tmp, Lam); c[1].mask = 1;
        nc = 2;
        break; }
    case ORC_R1:   /* HD word; Chase-II over the two least reliable (L551-581) */
        for (int i = 0; i < Lam; i++) seg_base[i] = (uint8_t)orc_hd(a[i]);
        if (Lam == 1) {
            m[0] = 0;
            c[0].dpm = 0.0f; c[0].mask = 0;
            c[1].dpm = fabsf(a[0]); c[1].mask = 1;
            nc = 2;
        } else {
            least_reliable(a, Lam, 2, m);
            for (int s = 0; s < 4; s++) {
                float d = 0.0f; int first = 1;
                for (int k = 0; k < 2; k++)
                    if ((s >> k) & 1) { d = first ? fabsf(a[m[k]]) : d + fabsf(a[m[k]]); first = 0; }
                c[nc].dpm = d; c[nc].mask = s; nc++;
            }
        }
        break;
    case ORC_SPC: { /* HD word; 8 parity-satisfying flips of m1..m4 (L583-585) */
        int p = 0;
        for (int i = 0; i < Lam; i++) { seg_base[i] = (uint8_t)orc_hd(a[i]); p ^= seg_base[i]; }
        least_reliable(a, Lam, 4, m);
        for (int s = 0; s < 16; s++) {
            if ((popcount4(s) & 1) != p) continue;
            float d = 0.0f; int first = 1;
            for (int k = 0; k < 4; k++)
                if ((s >> k) & 1) { d = first ? fabsf(a[m[k]]) : d + fabsf(a[m[k]]); first = 0; }
            c[nc].dpm = d; c[nc].mask = s; nc++;
        }
        break; }
    }
    /* insertion sort by (dPM, mask) */
    for (int x = 1; x < nc; x++) {
        cand_t v = c[x];
        int y = x - 1;
        while (y >= 0 && (c[y].dpm > v.dpm || (c[y].dpm == v.dpm && c[y].mask > v.mask))) { c[y + 1] = c[y]; y--; }
        c[y + 1] = v;
    }
    return nc;
}

static void apply_candidate(int kind, int Lam, const uint8_t *seg_base, const int *m, int mask, uint8_t *seg_out)
{
    for (int i = 0; i < Lam; i++) seg_out[i] = seg_base[i];
    if (kind == ORC_REP) {
        if (mask) for (int i = 0; i < Lam; i++) seg_out[i] ^= 1;
    } else if (kind == ORC_R1 || kind == ORC_SPC) {
        for (int k = 0; k < 4; k++) if ((mask >> k) & 1) seg_out[m[k]] ^= 1;
    }
}

/* ------------------------------------------------------------------------ */
/* O7  the stack engine (FSSCS-RM).  State: one alpha memory (stage lambda
 * holds Lambda floats), one working flat beta of N bits
 * (PAPER.md:L850-852), a stack S of <= D entries {PM, serial, k = schedule
 * progress (L848), j = depth = decision-node ordinal, PL, beta copy (L854)},
 * and the per-length counters cnt[0..M] (L595).                              */
struct orc_scs_s {
    int N, n, K, D, L, c, M, nops, bit_level, nonsys;
    uint32_t crc_poly;
    uint8_t *frozen;
    int *info;       /* A ascending */
    int32_t *ops;
    int *node_ordinal; /* j of the node at schedule index k (or -1) */
};

typedef struct {
    float pm;
    uint32_t serial;
    int k, j, pl;
    uint8_t *beta;   /* N bytes, owned */
} entry_t;

orc_scs_t *orc_scs_create(int N, const uint8_t *frozen, int D, int L, uint32_t crc_poly, int bit_level)
{
    return orc_scs_create_ex(N, frozen, D, L, crc_poly, bit_level, 0);
}

orc_scs_t *orc_scs_create_ex(int N, const uint8_t *frozen, int D, int L, uint32_t crc_poly, int bit_level,
                             int nonsystematic)
{
    int n = ilog2(N);
    if (n < 0 || D < 1 || L < 1) return NULL;
    orc_scs_t *h = (orc_scs_t *)calloc(1, sizeof(*h));
    h->N = N; h->n = n; h->D = D; h->L = L; h->crc_poly = crc_poly; h->bit_level = bit_level;
    h->nonsys = nonsystematic ? 1 : 0;
    h->c = orc_crc_degree(crc_poly);
    h->frozen = (uint8_t *)malloc((size_t)N);
    memcpy(h->frozen, frozen, (size_t)N);
    h->info = (int *)malloc(sizeof(int) * (size_t)N);
    for (int i = 0; i < N; i++) if (!frozen[i]) h->info[h->K++] = i;
    if (h->c >= h->K && h->c > 0) { orc_scs_destroy(h); return NULL; }
    int need = -orc_build_schedule(N, frozen, bit_level, NULL, 0);
    h->ops = (int32_t *)malloc(sizeof(int32_t) * (size_t)(need > 0 ? need : 1));
    h->nops = orc_build_schedule(N, frozen, bit_level, h->ops, need);
    h->node_ordinal = (int *)malloc(sizeof(int) * (size_t)h->nops);
    for (int k = 0; k < h->nops; k++) {
        int kind = h->ops[k] & 0xff;
        h->node_ordinal[k] = (kind >= ORC_R0) ? h->M++ : -1;
    }
    return h;
}

void orc_scs_destroy(orc_scs_t *h)
{
    if (!h) return;
    free(h->frozen); free(h->info); free(h->ops); free(h->node_ordinal);
    free(h);
}

int orc_scs_num_ops(const orc_scs_t *h) { return h->nops; }
int orc_scs_num_nodes(const orc_scs_t *h) { return h->M; }
int orc_scs_K(const orc_scs_t *h) { return h->K; }

/* (PM, serial) order: lower PM wins, then lower serial (reading R7) */
static int key_less(const entry_t *a, const entry_t *b)
{
    return (a->pm < b->pm) || (a->pm == b->pm && a->serial < b->serial);
}

/* Reuse model (O10, counter fg_reuse only; no effect on any result): the f/g
 * a decoder must evaluate if it keeps every alpha stage and recomputes a stage
 * only when its inputs changed.  ALPHA(lam, phi) reads alpha_{lam+1} (node
 * (lam+1, phi>>1)) and, for odd phi, the beta segment of its left sibling
 * (Eq. 4); its result is identical to the stage's current
 * content when the stage holds the same node, computed from the same version
 * of stage lam+1 and the same beta segment.  Each stage is tagged with the
 * node it holds, the version of its parent it was computed from, that beta
 * segment and its own version (bumped on every evaluation).  Stage n (the
 * channel) never changes.  A lower bound on the f/g of any stage-reusing
 * decoder; Alg. 4's whole-spine recompute (f_ops + g_ops) is the upper one. */
typedef struct {
    int *node;          /* [n] phi held by stage s, -1 = none */
    uint64_t *pver;     /* [n] version of stage s+1 it was computed from */
    uint64_t *ver;      /* [n+1] current version of stage s (ver[n] = 0) */
    uint8_t **bseg;     /* [n] beta segment used (odd phi) */
    uint64_t next;
} reuse_t;

static void reuse_reset(reuse_t *rm, int n)
{
    for (int s = 0; s < n; s++) { rm->node[s] = -1; rm->pver[s] = 0; rm->ver[s] = 0; }
    rm->ver[n] = 0;
    rm->next = 1;
}

/* ALPHA(lam, phi) from stage lam+1 (Eq. 4, Alg. 1): f for even phi, g for odd
 * phi with beta_u = left-sibling segment of the flat beta.  */
static void alpha_op(const orc_scs_t *h, float **alpha, const float *chan, const uint8_t *beta,
                     int lam, int phi, orc_counters_t *ct, int spine, reuse_t *rm)
{
    int Lam = 1 << lam;
    const float *p = (lam + 1 == h->n) ? chan : alpha[lam + 1];
    float *v = alpha[lam];
    for (int i = 0; i < Lam; i++) {
        if ((phi & 1) == 0) v[i] = orc_f(p[i], p[i + Lam]);
        else                v[i] = orc_g(p[i], p[i + Lam], beta[(phi - 1) * Lam + i]);
    }
    if (ct) {
        if (phi & 1) ct->g_ops += (uint64_t)Lam; else ct->f_ops += (uint64_t)Lam;
        if (spine) ct->spine_elems += (uint64_t)Lam;
    }
    if (rm) {
        const uint8_t *b = beta + (size_t)(phi - 1) * (size_t)Lam;
        int same = rm->node[lam] == phi && rm->pver[lam] == rm->ver[lam + 1] &&
                   (!(phi & 1) || memcmp(rm->bseg[lam], b, (size_t)Lam) == 0);
        if (!same) {
            if (ct) ct->fg_reuse += (uint64_t)Lam;
            rm->node[lam] = phi;
            rm->pver[lam] = rm->ver[lam + 1];
            rm->ver[lam] = rm->next++;
            if (phi & 1) memcpy(rm->bseg[lam], b, (size_t)Lam);
        }
    }
}

/* the K-bit block of a complete path: x_hat restricted to A (systematic,
 * PAPER.md:L854), or u_hat = x_hat F^{(x)n} restricted to A */
static void read_block(const orc_scs_t *h, const uint8_t *xhat, uint8_t *tmp, uint8_t *block)
{
    const uint8_t *src = xhat;
    if (h->nonsys) {
        memcpy(tmp, xhat, (size_t)h->N);
        orc_polar_transform(h->N, tmp);
        src = tmp;
    }
    for (int q = 0; q < h->K; q++) block[q] = src[h->info[q]];
}

static int decode_one(const orc_scs_t *h, const float *chan, uint8_t *block, uint8_t *xhat,
                      float *pm_out, uint32_t *pops_out, uint32_t *sw_out, uint8_t *st_out,
                      orc_counters_t *ct, float **alpha, entry_t *S, uint8_t *beta_work,
                      uint8_t *best_beta, int *cnt, float *tmp, uint8_t *seg_base, uint8_t *seg, reuse_t *rm)
{
    const int N = h->N, D = h->D;
    int nS = 0;
    uint32_t work = 0, next_serial = 1, pops = 0, switches = 0;
    int have_best = 0;
    float best_pm = 0.0f;
    for (int j = 0; j <= h->M; j++) cnt[j] = 0;
    if (rm) reuse_reset(rm, h->n);

    /* Init: the root path (PM 0, serial 0, k 0, j 0, PL 0) */
    S[0].pm = 0.0f; S[0].serial = 0; S[0].k = 0; S[0].j = 0; S[0].pl = 0;
    memset(S[0].beta, 0, (size_t)N);
    memset(beta_work, 0, (size_t)N);
    nS = 1;

    for (;;) {
        if (nS == 0) {
            /* every complete path failed the CRC: best effort (reading R13) */
            if (block) read_block(h, best_beta, seg_base, block);
            if (xhat) memcpy(xhat, best_beta, (size_t)N);
            if (pm_out) *pm_out = best_pm;
            if (pops_out) *pops_out = pops;
            if (sw_out) *sw_out = switches;
            if (st_out) *st_out = 1;
            return 0;
        }
        /* select: linear search for the winning (PM, serial) */
        int w = 0;
        for (int e = 1; e < nS; e++) if (key_less(&S[e], &S[w])) w = e;
        if (ct) ct->key_compares += (uint64_t)nS;
        entry_t p = S[w];
        S[w] = S[nS - 1];           /* remove it; its beta buffer moves to the tail */
        S[nS - 1] = p;
        nS--;
        pops++;
        if (ct) ct->pops++;
        /* per-length prune (readings R9, R10) */
        cnt[p.j]++;
        if (cnt[p.j] == h->L) {
            int keep = 0;
            for (int e = 0; e < nS; e++) {
                if (S[e].j <= p.j) { if (ct) ct->pruned++; continue; }
                entry_t t = S[keep]; S[keep] = S[e]; S[e] = t;
                keep++;
            }
            nS = keep;   /* entries at index >= nS (pruned, popped) are free buffers */
        }
        int spine_dirty = 0;
        if (p.serial != work) {
            /* path switch (SCS-RM): load the winner's beta
             * (no repopulation) and recompute alpha from the root */
            switches++;
            if (ct) ct->switches++;
            memcpy(beta_work, p.beta, (size_t)N);
            work = p.serial;
            spine_dirty = 1;
        }
        /* continue the schedule from the stored progress */
        int k = p.k;
        while (k < h->nops && (h->ops[k] & 0xff) < ORC_R0) {
            int kind = h->ops[k] & 0xff, lam = (h->ops[k] >> 8) & 0xff, phi = h->ops[k] >> 16;
            int Lam = 1 << lam;
            if (kind == ORC_BETA) {
                /* in-place XOR of the right segment into the left (Fig. 7d) */
                for (int i = 0; i < Lam; i++) beta_work[(phi - 1) * Lam + i] ^= beta_work[phi * Lam + i];
                if (ct) ct->beta_xor_bits += (uint64_t)Lam;
            } else {
                if (spine_dirty) {
                    /* Alg. 4 (typos per R12): recompute the
                     * ancestors of (lam, phi) from the channel downwards */
                    for (int s = h->n - 1; s > lam; s--)
                        alpha_op(h, alpha, chan, beta_work, s, phi >> (s - lam), ct, 1, rm);
                    spine_dirty = 0;
                    alpha_op(h, alpha, chan, beta_work, lam, phi, ct, 1, rm);
                } else {
                    alpha_op(h, alpha, chan, beta_work, lam, phi, ct, 0, rm);
                }
            }
            k++;
        }
        if (k == h->nops) {
            /* complete path: CRC on the systematic bits */
            int ok = 1;
            if (h->c > 0) {
                if (ct) ct->crc_checks++;
                read_block(h, beta_work, seg_base, seg);
                uint8_t rem[32];
                orc_crc_bits(seg, h->K - h->c, h->crc_poly, rem);
                for (int d = 0; d < h->c; d++) ok &= (rem[d] == seg[h->K - h->c + d]);
            }
            if (ok) {
                if (block) read_block(h, beta_work, seg_base, block);
                if (xhat) memcpy(xhat, beta_work, (size_t)N);
                if (pm_out) *pm_out = p.pm;
                if (pops_out) *pops_out = pops;
                if (sw_out) *sw_out = switches;
                if (st_out) *st_out = 0;
                return 0;
            }
            if (!have_best) { have_best = 1; best_pm = p.pm; memcpy(best_beta, beta_work, (size_t)N); }
            continue;
        }
        /* decision node at (lam, phi): candidates */
        int kind = h->ops[k] & 0xff, lam = (h->ops[k] >> 8) & 0xff, phi = h->ops[k] >> 16;
        int Lam = 1 << lam;
        const float *a = (lam == h->n) ? chan : alpha[lam];
        int m[4] = { 0, 0, 0, 0 };
        cand_t c[8] = { { 0.0f, 0 } };
        int nc = node_candidates(kind, a, Lam, seg_base, m, c, tmp);
        if (ct) { ct->node_visits++; ct->node_elems += (uint64_t)Lam; ct->cand_created += (uint64_t)nc; }
        int kn = k + 1, jn = p.j + 1, pl = (phi + 1) * Lam;
        float parent_pm = p.pm;
        uint32_t ser0 = next_serial;
        next_serial += (uint32_t)nc;
        /* c1 continues in the working memory */
        apply_candidate(kind, Lam, seg_base, m, c[0].mask, seg);
        memcpy(beta_work + phi * Lam, seg, (size_t)Lam);
        /* p's slot was freed, so c1 always fits (reading R8) */
        {
            entry_t *e = &S[nS];
            e->pm = parent_pm + c[0].dpm; e->serial = ser0; e->k = kn; e->j = jn; e->pl = pl;
            memcpy(e->beta, beta_work, (size_t)N);
            nS++;
            if (ct) ct->cand_inserted++;
        }
        work = ser0;
        for (int t = 1; t < nc; t++) {
            float cpm = parent_pm + c[t].dpm;
            entry_t *dst = NULL;
            if (nS < D) {
                dst = &S[nS]; nS++;
                if (ct) ct->cand_inserted++;
            } else {
                /* full stack: replace the least reliable iff strictly better */
                int worst = 0;
                for (int e = 1; e < nS; e++) if (key_less(&S[worst], &S[e])) worst = e;
                if (ct) ct->key_compares += (uint64_t)nS;
                if (cpm < S[worst].pm) { dst = &S[worst]; if (ct) ct->cand_replaced++; }
                else if (ct) ct->cand_dropped++;
            }
            if (!dst) continue;
            dst->pm = cpm; dst->serial = ser0 + (uint32_t)t; dst->k = kn; dst->j = jn; dst->pl = pl;
            memcpy(dst->beta, beta_work, (size_t)N);
            apply_candidate(kind, Lam, seg_base, m, c[t].mask, dst->beta + phi * Lam);
        }
        if (ct && (uint64_t)nS > ct->stack_peak) ct->stack_peak = (uint64_t)nS;
    }
}

int orc_scs_decode(const orc_scs_t *h, const float *llr, int64_t n_frames,
                   uint8_t *block, uint8_t *xhat, float *pm, uint32_t *pops,
                   uint32_t *switches, uint8_t *status, orc_counters_t *counters)
{
    const int N = h->N, D = h->D;
    int rc = 0;
    float **alpha = (float **)calloc((size_t)h->n + 1, sizeof(float *));
    entry_t *S = (entry_t *)calloc((size_t)D + 1, sizeof(entry_t));
    uint8_t *beta_work = (uint8_t *)malloc((size_t)N);
    uint8_t *best_beta = (uint8_t *)malloc((size_t)N);
    int *cnt = (int *)malloc(sizeof(int) * (size_t)(h->M + 1));
    float *tmp = (float *)malloc(sizeof(float) * (size_t)N);
    uint8_t *seg_base = (uint8_t *)malloc((size_t)N);
    uint8_t *seg = (uint8_t *)malloc((size_t)N);
    reuse_t rm = { 0 }, *rmp = NULL;
    int ok = alpha && S && beta_work && best_beta && cnt && tmp && seg_base && seg;
    for (int l = 0; ok && l < h->n; l++) ok = (alpha[l] = (float *)malloc(sizeof(float) * ((size_t)1 << l))) != NULL;
    if (ok && counters) {
        rm.node = (int *)calloc((size_t)h->n + 1, sizeof(int));
        rm.pver = (uint64_t *)calloc((size_t)h->n + 1, sizeof(uint64_t));
        rm.ver = (uint64_t *)calloc((size_t)h->n + 1, sizeof(uint64_t));
        rm.bseg = (uint8_t **)calloc((size_t)h->n + 1, sizeof(uint8_t *));
        ok = rm.node && rm.pver && rm.ver && rm.bseg;
        for (int l = 0; ok && l < h->n; l++) ok = (rm.bseg[l] = (uint8_t *)malloc((size_t)1 << l)) != NULL;
        rmp = &rm;
    }
    for (int e = 0; ok && e < D + 1; e++) ok = (S[e].beta = (uint8_t *)malloc((size_t)N)) != NULL;
    if (!ok) rc = -1;
    for (int64_t f = 0; ok && f < n_frames; f++) {
        decode_one(h, llr + f * N, block ? block + f * h->K : NULL, xhat ? xhat + f * N : NULL,
                   pm ? pm + f : NULL, pops ? pops + f : NULL, switches ? switches + f : NULL,
                   status ? status + f : NULL, counters, alpha, S, beta_work, best_beta, cnt, tmp,
                   seg_base, seg, rmp);
    }
    if (rm.bseg) for (int l = 0; l < h->n; l++) free(rm.bseg[l]);
    free(rm.node); free(rm.pver); free(rm.ver); free(rm.bseg);
    if (alpha) for (int l = 0; l < h->n; l++) free(alpha[l]);
    if (S) for (int e = 0; e < D + 1; e++) free(S[e].beta);
    free(alpha); free(S); free(beta_work); free(best_beta); free(cnt); free(tmp); free(seg_base); free(seg);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* O11  the FSSCL list decoder (§2.2.3-2.2.4; memory per
 * L772-780).  L paths advance in lock-step through the FSSC schedule; at every
 * decision node (R0 included, reading R23) each path creates its node
 * candidates (the same rules as O7, L526-585) and the union is pruned back to
 * the L best (L507).  Written with a naive full copy of alpha and beta per
 * path: the lazy copy of L774-776 is a memory optimisation that must not
 * change any result.
 *
 * Readings: R22 the list is kept in rank order; a candidate's key
 * is (PM, parent rank, candidate rank in (dPM, mask) order) and the L smallest
 * keys survive, in key order ("ties broken by lower parent path
 * id, then lower candidate ordinal").  R24 final selection (L519): the first
 * path in rank order whose block passes the CRC (the first path when there is
 * no CRC); if none passes, the first path with status 1.     */
struct orc_scl_s {
    int N, n, K, L, c, M, nops, nonsys;
    uint32_t crc_poly;
    uint8_t *frozen;
    int *info;
    int32_t *ops;
};

typedef struct {
    float pm;
    float **alpha;   /* stages 0..n-1, own copy */
    uint8_t *beta;   /* N bytes */
} lpath_t;

typedef struct { float pm; int parent, rank, mask; } lcand_t;

/* (PM, parent rank, candidate rank) order (reading R22) */
static int lcand_less(const lcand_t *a, const lcand_t *b)
{
    if (a->pm != b->pm) return a->pm < b->pm;
    if (a->parent != b->parent) return a->parent < b->parent;
    return a->rank < b->rank;
}

orc_scl_t *orc_scl_create(int N, const uint8_t *frozen, int L, uint32_t crc_poly, int bit_level, int nonsystematic)
{
    int n = ilog2(N);
    if (n < 0 || L < 1) return NULL;
    orc_scl_t *h = (orc_scl_t *)calloc(1, sizeof(*h));
    h->N = N; h->n = n; h->L = L; h->crc_poly = crc_poly; h->nonsys = nonsystematic ? 1 : 0;
    h->c = orc_crc_degree(crc_poly);
    h->frozen = (uint8_t *)malloc((size_t)N);
    memcpy(h->frozen, frozen, (size_t)N);
    h->info = (int *)malloc(sizeof(int) * (size_t)N);
    for (int i = 0; i < N; i++) if (!frozen[i]) h->info[h->K++] = i;
    if (h->c >= h->K && h->c > 0) { orc_scl_destroy(h); return NULL; }
    int need = -orc_build_schedule(N, frozen, bit_level, NULL, 0);
    h->ops = (int32_t *)malloc(sizeof(int32_t) * (size_t)(need > 0 ? need : 1));
    h->nops = orc_build_schedule(N, frozen, bit_level, h->ops, need);
    for (int k = 0; k < h->nops; k++) if ((h->ops[k] & 0xff) >= ORC_R0) h->M++;
    return h;
}

void orc_scl_destroy(orc_scl_t *h)
{
    if (!h) return;
    free(h->frozen); free(h->info); free(h->ops);
    free(h);
}

int orc_scl_K(const orc_scl_t *h) { return h->K; }
int orc_scl_num_nodes(const orc_scl_t *h) { return h->M; }

/* the CRC check of a complete path's block */
static int scl_crc_ok(const orc_scl_t *h, const uint8_t *xhat, uint8_t *tmp, uint8_t *blk)
{
    if (h->c == 0) return 1;
    const uint8_t *src = xhat;
    if (h->nonsys) { memcpy(tmp, xhat, (size_t)h->N); orc_polar_transform(h->N, tmp); src = tmp; }
    for (int q = 0; q < h->K; q++) blk[q] = src[h->info[q]];
    uint8_t rem[32];
    orc_crc_bits(blk, h->K - h->c, h->crc_poly, rem);
    int ok = 1;
    for (int d = 0; d < h->c; d++) ok &= (rem[d] == blk[h->K - h->c + d]);
    return ok;
}

static void scl_copy_path(const orc_scl_t *h, lpath_t *dst, const lpath_t *src)
{
    dst->pm = src->pm;
    for (int l = 0; l < h->n; l++) memcpy(dst->alpha[l], src->alpha[l], sizeof(float) * ((size_t)1 << l));
    memcpy(dst->beta, src->beta, (size_t)h->N);
}

int orc_scl_decode(const orc_scl_t *h, const float *llr, int64_t n_frames, uint8_t *block, uint8_t *xhat,
                   float *pm_out, uint8_t *status, uint32_t *crc_checks, orc_counters_t *ct)
{
    const int N = h->N, L = h->L, n = h->n;
    lpath_t *cur = (lpath_t *)calloc((size_t)L, sizeof(lpath_t));
    lpath_t *nxt = (lpath_t *)calloc((size_t)L, sizeof(lpath_t));
    lcand_t *cand = (lcand_t *)malloc(sizeof(lcand_t) * (size_t)L * 8);
    int (*mm)[4] = (int (*)[4])malloc(sizeof(int[4]) * (size_t)L);
    uint8_t *base = (uint8_t *)malloc((size_t)L * (size_t)N);
    float *tmp = (float *)malloc(sizeof(float) * (size_t)N);
    uint8_t *t1 = (uint8_t *)malloc((size_t)N), *t2 = (uint8_t *)malloc((size_t)N);
    int ok = cur && nxt && cand && mm && base && tmp && t1 && t2;
    for (int l = 0; ok && l < L; l++) {
        lpath_t *ps[2] = { &cur[l], &nxt[l] };
        for (int q = 0; q < 2 && ok; q++) {
            ps[q]->alpha = (float **)calloc((size_t)n + 1, sizeof(float *));
            ps[q]->beta = (uint8_t *)malloc((size_t)N);
            ok = ps[q]->alpha && ps[q]->beta;
            for (int s = 0; ok && s < n; s++) ok = (ps[q]->alpha[s] = (float *)malloc(sizeof(float) * ((size_t)1 << s))) != NULL;
        }
    }
    for (int64_t f = 0; ok && f < n_frames; f++) {
        const float *chan = llr + f * N;
        int nL = 1;
        cur[0].pm = 0.0f;
        memset(cur[0].beta, 0, (size_t)N);
        uint32_t checks = 0;
        for (int k = 0; k < h->nops; k++) {
            int kind = h->ops[k] & 0xff, lam = (h->ops[k] >> 8) & 0xff, phi = h->ops[k] >> 16;
            int Lam = 1 << lam;
            if (kind == ORC_BETA) {          /* in-place XOR, every path */
                for (int l = 0; l < nL; l++)
                    for (int i = 0; i < Lam; i++) cur[l].beta[(phi - 1) * Lam + i] ^= cur[l].beta[phi * Lam + i];
                if (ct) ct->beta_xor_bits += (uint64_t)Lam * (uint64_t)nL;
                continue;
            }
            if (kind == ORC_ALPHA) {         /* Eq. (4), every path on its own memory */
                for (int l = 0; l < nL; l++) {
                    const float *p = (lam + 1 == n) ? chan : cur[l].alpha[lam + 1];
                    float *v = cur[l].alpha[lam];
                    for (int i = 0; i < Lam; i++)
                        v[i] = (phi & 1) ? orc_g(p[i], p[i + Lam], cur[l].beta[(phi - 1) * Lam + i])
                                         : orc_f(p[i], p[i + Lam]);
                }
                if (ct) { if (phi & 1) ct->g_ops += (uint64_t)Lam * (uint64_t)nL; else ct->f_ops += (uint64_t)Lam * (uint64_t)nL; }
                continue;
            }
            /* decision node: candidates of every path */
            int nc_all = 0;
            for (int l = 0; l < nL; l++) {
                const float *a = (lam == n) ? chan : cur[l].alpha[lam];
                cand_t c[8];
                int nc = node_candidates(kind, a, Lam, base + (size_t)l * N, mm[l], c, tmp);
                for (int t = 0; t < nc; t++) {
                    cand[nc_all].pm = cur[l].pm + c[t].dpm;
                    cand[nc_all].parent = l; cand[nc_all].rank = t; cand[nc_all].mask = c[t].mask;
                    nc_all++;
                }
            }
            if (ct) {
                ct->node_visits += (uint64_t)nL; ct->node_elems += (uint64_t)Lam * (uint64_t)nL;
                ct->cand_created += (uint64_t)nc_all; { int lg = 0; while ((1 << lg) < nc_all) lg++; ct->sel_compares += (uint64_t)nc_all * (uint64_t)lg; }
                ct->pruned += (uint64_t)(nc_all > L ? nc_all - L : 0);
            }
            /* prune to the L best (reading R22): insertion sort */
            for (int x = 1; x < nc_all; x++) {
                lcand_t v = cand[x];
                int y = x - 1;
                while (y >= 0 && lcand_less(&v, &cand[y])) { cand[y + 1] = cand[y]; y--; }
                cand[y + 1] = v;
            }
            int nL2 = nc_all < L ? nc_all : L;
            for (int r = 0; r < nL2; r++) {
                const lcand_t *cd = &cand[r];
                scl_copy_path(h, &nxt[r], &cur[cd->parent]);
                nxt[r].pm = cd->pm;
                apply_candidate(kind, Lam, base + (size_t)cd->parent * N, mm[cd->parent], cd->mask,
                                nxt[r].beta + phi * Lam);
            }
            lpath_t *sw = cur; cur = nxt; nxt = sw;
            nL = nL2;
        }
        /* final selection (reading R24) */
        int sel = -1;
        for (int r = 0; r < nL && sel < 0; r++) {
            if (h->c > 0) checks++;
            if (scl_crc_ok(h, cur[r].beta, t1, t2)) sel = r;
        }
        int st = 0;
        if (sel < 0) { sel = 0; st = 1; }
        if (block) {
            const uint8_t *src = cur[sel].beta;
            if (h->nonsys) { memcpy(t1, cur[sel].beta, (size_t)N); orc_polar_transform(N, t1); src = t1; }
            for (int q = 0; q < h->K; q++) block[f * h->K + q] = src[h->info[q]];
        }
        if (xhat) memcpy(xhat + f * N, cur[sel].beta, (size_t)N);
        if (pm_out) pm_out[f] = cur[sel].pm;
        if (status) status[f] = (uint8_t)st;
        if (crc_checks) crc_checks[f] = checks;
        if (ct) ct->crc_checks += checks;
    }
    for (int l = 0; l < L; l++) {
        lpath_t *ps[2] = { cur ? &cur[l] : NULL, nxt ? &nxt[l] : NULL };
        for (int q = 0; q < 2; q++) {
            if (!ps[q]) continue;
            if (ps[q]->alpha) for (int s = 0; s < n; s++) free(ps[q]->alpha[s]);
            free(ps[q]->alpha); free(ps[q]->beta);
        }
    }
    free(cur); free(nxt); free(cand); free(mm); free(base); free(tmp); free(t1); free(t2);
    return ok ? 0 : -1;
}

/* test hook: the sorted candidates of one node over a[0..Lam) — segments
 * written to segs[t*Lam .. (t+1)*Lam), dPM to dpm[t], mask to mask[t].     */
int orc_node_candidates(int kind, const float *a, int Lam, float *dpm, int *mask, uint8_t *segs)
{
    float *tmp = (float *)malloc(sizeof(float) * (size_t)Lam);
    uint8_t *base = (uint8_t *)malloc((size_t)Lam);
    int m[4] = { 0, 0, 0, 0 };
    cand_t c[8] = { { 0.0f, 0 } };
    int nc = node_candidates(kind, a, Lam, base, m, c, tmp);
    for (int t = 0; t < nc; t++) {
        dpm[t] = c[t].dpm;
        mask[t] = c[t].mask;
        apply_candidate(kind, Lam, base, m, c[t].mask, segs + (size_t)t * (size_t)Lam);
    }
    free(tmp); free(base);
    return nc;
}

// host.cpp — host-side code preparation of libpolarscs: Bhattacharyya
// construction, mask validation, FSSC schedule compilation and the
// information-set / CRC tables uploaded at polar_scs_create.
//
// Independent of oracle/ (test infrastructure): nothing here includes,
// links or calls it.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>

#include "internal.h"

namespace polar {

static int ilog2_exact(int N) {
    if (N < 1) return -1;
    int n = 0;
    while ((1 << n) < N) n++;
    return (1 << n) == N ? n : -1;
}

int crc_degree(uint32_t poly_full) {
    if (poly_full < 2) return 0;
    return 31 - __builtin_clz(poly_full);
}

// Word-parallel x <- x F^{(x)n}: stage span h moves bit i+h
// onto bit i for every i with (i & h) == 0.
static void transform_words(std::vector<uint64_t> &w, int N) {
    static const uint64_t kMask[6] = {0x5555555555555555ull, 0x3333333333333333ull, 0x0F0F0F0F0F0F0F0Full,
                                      0x00FF00FF00FF00FFull, 0x0000FFFF0000FFFFull, 0x00000000FFFFFFFFull};
    const int nw = (int)w.size();
    for (int s = 0; (1 << s) < N && s < 6; s++)
        for (int j = 0; j < nw; j++) w[j] ^= (w[j] >> (1 << s)) & kMask[s];
    for (int H = 1; H < nw; H <<= 1)
        for (int j = 0; j < nw; j++)
            if ((j & H) == 0) w[j] ^= w[j + H];
}

// Systematic encodability: the double transform with frozen re-zeroing must
// reproduce every unit message on A.
static bool check_systematic(int N, const std::vector<int> &info, const std::vector<uint64_t> &info_mask) {
    const int nw = (N + 63) / 64;
    std::vector<uint64_t> w(nw);
    for (size_t k = 0; k < info.size(); k++) {
        std::fill(w.begin(), w.end(), 0);
        w[info[k] >> 6] |= 1ull << (info[k] & 63);
        transform_words(w, N);
        for (int j = 0; j < nw; j++) w[j] &= info_mask[j];
        transform_words(w, N);
        for (int j = 0; j < nw; j++) {
            uint64_t expect = (j == (info[k] >> 6)) ? (1ull << (info[k] & 63)) : 0;
            if ((w[j] & info_mask[j]) != expect) return false;
        }
    }
    return true;
}

int build_host_code(int N, int K, const uint8_t *frozen, uint32_t crc_poly, bool bit_level, HostCode &hc) {
    const int n = ilog2_exact(N);
    if (n < 1 || N > kMaxN || K < 1 || K > N || !frozen) return POLAR_EINVAL;
    int nfrozen = 0;
    for (int i = 0; i < N; i++) {
        if (frozen[i] > 1) return POLAR_EINVAL;
        nfrozen += frozen[i];
    }
    if (nfrozen != N - K) return POLAR_EINVAL;
    const int c = crc_degree(crc_poly);
    if (crc_poly == 1 || c > 31 || c >= K) return POLAR_EINVAL;

    hc = HostCode{};
    hc.N = N; hc.n = n; hc.K = K; hc.c = c; hc.crc_poly = crc_poly;

    // information set, ascending
    std::vector<int> info;
    for (int i = 0; i < N; i++) if (!frozen[i]) info.push_back(i);
    hc.info.assign(info.begin(), info.end());
    const int nw32 = std::max(1, N / 32);
    hc.info_words.assign(nw32, 0);
    std::vector<uint64_t> info_mask((N + 63) / 64, 0);
    for (int i : info) {
        hc.info_words[i >> 5] |= 1u << (i & 31);
        info_mask[i >> 6] |= 1ull << (i & 63);
    }
    hc.systematic_ok = check_systematic(N, info, info_mask);

    // FSSC schedule (Fig. 5): classify each subtree from prefix
    // counts of frozen leaves — R0 (all frozen) > R1 (none) > REP (only the last
    // leaf informative) > SPC (only the first leaf frozen,
    // PAPER.md:L487-499); otherwise ALPHA + recurse per child, BETA after the
    // right child (Eq. 4 / Eq. bitcalc).
    std::vector<int> pre(N + 1, 0);
    for (int i = 0; i < N; i++) pre[i + 1] = pre[i] + frozen[i];
    auto node_kind = [&](int lam, int phi) -> int {
        if (bit_level && lam > 0) return -1;
        const int a = phi << lam, b = (phi + 1) << lam, L = 1 << lam;
        const int nf = pre[b] - pre[a];
        if (nf == L) return OP_R0;
        if (nf == 0) return OP_R1;
        if (nf == L - 1 && !frozen[b - 1]) return OP_REP;
        if (nf == 1 && frozen[a]) return OP_SPC;
        return -1;
    };
    struct Rec {
        HostCode &h;
        decltype(node_kind) &kind;
        void operator()(int lam, int phi) {
            int k = kind(lam, phi);
            if (k >= 0) { h.ops.push_back(op_make(k, lam, phi)); h.M++; return; }
            h.ops.push_back(op_make(OP_ALPHA, lam - 1, 2 * phi));
            (*this)(lam - 1, 2 * phi);
            h.ops.push_back(op_make(OP_ALPHA, lam - 1, 2 * phi + 1));
            (*this)(lam - 1, 2 * phi + 1);
            h.ops.push_back(op_make(OP_BETA, lam - 1, 2 * phi + 1));
        }
    } rec{hc, node_kind};
    rec(n, 0);
    if (hc.ops.size() > 65535 || hc.M > 8191) return POLAR_EINVAL;
    for (uint32_t op : hc.ops)
        if (op_kind(op) >= OP_R0) hc.nodes.push_back(op);
    // per-depth records of the stack decoder (decode.cu), 16 words each: a path
    // of depth j (j nodes decided) resumes at node j after the BETA climb that
    // finishes node j-1; everything the pop needs about
    // both nodes and that climb, unpacked:
    //   [0] start of node j (= p's path length; N at j = M), [1] end of node j,
    //   [2] lambda_j, [3] kind_j,
    //   [4] level lw where the word-level part of the climb starts, [5] its phi,
    //   [6] kind_{j-1}, [7] level where the climb ends,
    //   [8] word of the in-word part (levels < 5, 2 Lambda <= 32; ~0u: none),
    //   [9..13] its masks: level l XORs (x >> 2^l) & mask_l into x (0: level
    //   not climbed), [14] lambda_{j-1}, [15] 0
    hc.recs.assign(16 * (size_t)(hc.M + 1), 0u);
    for (int j = 0; j <= hc.M; j++) {
        uint32_t *r = &hc.recs[16 * (size_t)j];
        if (j < hc.M) {
            const uint32_t nd = hc.nodes[j], lam = op_lam(nd), phi = op_phi(nd);
            r[0] = phi << lam; r[1] = (phi + 1) << lam; r[2] = lam; r[3] = op_kind(nd);
        } else {
            r[0] = r[1] = (uint32_t)N;
        }
        r[8] = ~0u;
        if (j == 0) {
            r[4] = (uint32_t)n; r[5] = 0; r[7] = (uint32_t)n; r[14] = (uint32_t)n;
            continue;
        }
        const uint32_t pn = hc.nodes[j - 1];
        int l = (int)op_lam(pn);
        uint32_t ph = op_phi(pn);
        r[6] = op_kind(pn);
        r[14] = (uint32_t)l;
        if ((ph & 1) && l < 5) {
            r[8] = ((ph - 1) << l) >> 5;
            while ((ph & 1) && l < 5) {
                const uint32_t o = ((ph - 1) << l) & 31, Lm = 1u << l;
                r[9 + l] = ((1u << Lm) - 1u) << o;    // left segment [o, o + Lm) ^= right [o + Lm, o + 2 Lm)
                ph >>= 1;
                l++;
            }
        }
        r[4] = (uint32_t)l; r[5] = ph;
        while (ph & 1) { ph >>= 1; l++; }
        r[7] = (uint32_t)l;
    }
    // CRC syndrome table: block bit k < P = K-c is the
    // payload coefficient of x^(P-1-k); its contribution to the remainder of
    // payload * x^c is x^(P-1-k+c) mod g.  A received CRC bit k >= P weighs
    // x^(K-1-k).  syndrome = XOR over set block bits == 0  <=>  CRC holds.
    hc.crc_tab.assign(K, 0);
    if (c > 0) {
        const int P = K - c;
        const uint32_t low = crc_poly ^ (1u << c);     // x^c mod g
        const uint32_t topbit = 1u << (c - 1);
        const uint32_t cmask = (c == 32) ? 0xFFFFFFFFu : ((1u << c) - 1);
        uint32_t r = low;                              // x^c mod g
        for (int e = c; e <= P - 1 + c; e++) {
            const int k = P - 1 - (e - c);
            hc.crc_tab[k] = r;
            // r <- x * r mod g
            const bool carry = (r & topbit) != 0;
            r = (r << 1) & cmask;
            if (carry) r ^= low;
        }
        for (int k = P; k < K; k++) hc.crc_tab[k] = 1u << (K - 1 - k);
        // per beta byte (word w, byte b, value v): XOR of the contributions of
        // the information positions among the set bits of v
        std::vector<int> rank(N, -1);
        for (int k = 0; k < K; k++) rank[info[k]] = k;
        hc.crc_bytes.assign((size_t)nw32 * 1024, 0);
        for (int w = 0; w < nw32; w++)
            for (int b = 0; b < 4; b++)
                for (int v = 0; v < 256; v++) {
                    uint32_t acc = 0;
                    for (int bit = 0; bit < 8; bit++) {
                        const int pos = 32 * w + 8 * b + bit;
                        if (((v >> bit) & 1) && pos < N && rank[pos] >= 0) acc ^= hc.crc_tab[rank[pos]];
                    }
                    hc.crc_bytes[(size_t)w * 1024 + 256 * b + v] = acc;
                }
    }
    return POLAR_OK;
}

}  // namespace polar

// Information set from a reliability sequence listed least reliable first
// (e.g. the 3GPP TS 38.212 sequence of PAPER.md:L966, which the
// user supplies): the K most reliable entries below N carry information.
extern "C" int polar_construct_from_sequence(int32_t N, int32_t K, const int32_t *seq, int32_t len,
                                             uint8_t *frozen_mask) {
    if (N < 1 || N > 65536 || (N & (N - 1)) != 0 || K < 0 || K > N || !seq || !frozen_mask || len < N)
        return POLAR_EINVAL;
    std::vector<char> seen((size_t)len, 0);
    std::vector<int> below;
    below.reserve(N);
    for (int32_t i = 0; i < len; i++) {
        const int32_t v = seq[i];
        if (v < 0 || v >= len || seen[v]) return POLAR_EINVAL;
        seen[v] = 1;
        if (v < N) below.push_back(v);
    }
    if ((int)below.size() != N) return POLAR_EINVAL;
    std::memset(frozen_mask, 1, (size_t)N);
    for (int r = N - K; r < N; r++) frozen_mask[below[r]] = 0;
    return POLAR_OK;
}

// Bhattacharyya construction, level-by-level doubling in the log domain: at
// each level every parameter z spawns 2z - z^2 (appended bit 0) and z^2
// (appended bit 1); the first appended bit is the index MSB.
extern "C" int polar_construct_bhattacharyya(int32_t N, int32_t K, double design_ebno_db, uint8_t *frozen_mask) {
    if (N < 1 || N > 65536 || (N & (N - 1)) != 0 || K < 0 || K > N || !frozen_mask) return POLAR_EINVAL;
    std::vector<double> lz(1, -((double)K / (double)N) * std::pow(10.0, design_ebno_db / 10.0));
    while ((int)lz.size() < N) {
        std::vector<double> nxt(lz.size() * 2);
        for (size_t i = 0; i < lz.size(); i++) {
            const double l = lz[i];
            nxt[2 * i] = l + std::log(2.0 - std::exp(l));
            nxt[2 * i + 1] = 2.0 * l;
        }
        lz.swap(nxt);
    }
    std::vector<int> idx(N);
    std::iota(idx.begin(), idx.end(), 0);
    std::sort(idx.begin(), idx.end(), [&](int a, int b) { return lz[a] < lz[b] || (lz[a] == lz[b] && a > b); });
    std::memset(frozen_mask, 1, (size_t)N);
    for (int r = 0; r < K; r++) frozen_mask[idx[r]] = 0;
    return POLAR_OK;
}

// ASan/UBSan driver for the product's host code (host.cpp): construction,
// schedule compile, node table, CRC tables, systematic check, for many codes.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <numeric>
#include <random>
#include <algorithm>
#include "../paper_1809_03606_b200/csrc/internal.h"
extern "C" int polar_construct_bhattacharyya(int32_t N, int32_t K, double db, uint8_t *frozen);
extern "C" int polar_construct_from_sequence(int32_t N, int32_t K, const int32_t *seq, int32_t len, uint8_t *frozen);
int main() {
    std::mt19937 rng(1);
    const uint32_t polys[4] = {0, 0x107, 0x11021, 0x1B2B117};
    int count = 0;
    for (int n = 1; n <= 12; n++) {
        const int N = 1 << n;
        for (int rep = 0; rep < 12; rep++) {
            const int K = 1 + (int)(rng() % N);
            std::vector<uint8_t> fr(N);
            if (rep % 2) {
                if (polar_construct_bhattacharyya(N, K, (rng() % 40) / 10.0, fr.data()) != 0) return 1;
            } else {
                std::vector<int32_t> seq(N);
                std::iota(seq.begin(), seq.end(), 0);
                std::shuffle(seq.begin(), seq.end(), rng);
                if (polar_construct_from_sequence(N, K, seq.data(), N, fr.data()) != 0) return 2;
            }
            for (int bit = 0; bit < 2; bit++)
                for (uint32_t poly : polys) {
                    polar::HostCode hc;
                    const int rc = polar::build_host_code(N, K, fr.data(), poly, bit != 0, hc);
                    count += (rc == 0);
                }
        }
    }
    // invalid arguments must be rejected without touching memory
    std::vector<uint8_t> fr(8, 1);
    polar::HostCode hc;
    if (polar::build_host_code(8, 4, fr.data(), 0, false, hc) == 0) return 3;     // weight mismatch
    if (polar_construct_bhattacharyya(6, 3, 2.0, fr.data()) == 0) return 4;      // N not a power of two
    printf("host code built for %d (code, CRC, schedule) cases\n", count);
    return 0;
}

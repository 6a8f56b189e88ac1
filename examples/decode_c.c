/*
 * Plain-C use of the libpolarscs ABI (include/polar_scs.h): build a
 * PC(1024,512) code by Bhattacharyya construction, generate 100,000 noisy
 * frames on the device, decode them with the FSSCS-RM stack decoder and the
 * FSSCL list decoder, and count frame errors.  No Python, no torch.
 *
 *   nvcc -O2 -o decode_c examples/decode_c.c -Iinclude \
 *        -Lpaper_1809_03606_b200 -lpolarscs -Xlinker -rpath=$PWD/paper_1809_03606_b200
 *   ./decode_c [ebno_db]
 */
#include <stdio.h>
#include <stdlib.h>
#include <cuda_runtime.h>

#include "polar_scs.h"

#define CHECK(x) do { int rc_ = (x); if (rc_ != POLAR_OK) { \
    fprintf(stderr, "%s failed: %s (%d)\n", #x, polar_scs_strerror(rc_), rc_); return 1; } } while (0)

int main(int argc, char **argv) {
    const int N = 1024, K = 512, D = 32, L = 8;
    const int64_t n = 100000;
    const double ebno = argc > 1 ? atof(argv[1]) : 2.0;
    uint8_t frozen[1024];
    CHECK(polar_construct_bhattacharyya(N, K, 2.0, frozen));
    polar_scs_t h;
    CHECK(polar_scs_create(&h, N, K, frozen, D, L, 0));

    float *llr; uint8_t *blk, *bits;
    cudaMalloc((void **)&llr, (size_t)n * N * sizeof(float));
    cudaMalloc((void **)&blk, (size_t)n * K);
    cudaMalloc((void **)&bits, (size_t)n * K);
    CHECK(polar_generate_batch(h, 1, ebno, 0, n, blk, llr, NULL));

    uint8_t *hb = (uint8_t *)malloc((size_t)n * K), *hr = (uint8_t *)malloc((size_t)n * K);
    cudaMemcpy(hb, blk, (size_t)n * K, cudaMemcpyDeviceToHost);
    const char *names[2] = {"FSSCS-RM (stack, D=32, L=8)", "FSSCL (list, L=8)"};
    for (int dec = 0; dec < 2; dec++) {
        cudaEvent_t a, b;
        cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a, 0);
        if (dec == 0) CHECK(polar_scs_decode(h, llr, n, bits, NULL));
        else CHECK(polar_scl_decode(h, llr, n, bits, NULL, NULL, NULL));
        cudaEventRecord(b, 0);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        cudaMemcpy(hr, bits, (size_t)n * K, cudaMemcpyDeviceToHost);
        int64_t errs = 0;
        for (int64_t f = 0; f < n; f++) {
            for (int k = 0; k < K; k++)
                if (hr[f * K + k] != hb[f * K + k]) { errs++; break; }
        }
        printf("%-30s Eb/N0 %.1f dB: %lld frames in %.2f ms = %.0f Mbps, FER %.3e\n", names[dec], ebno,
               (long long)n, ms, (double)n * K / (ms * 1e3), (double)errs / (double)n);
    }
    polar_scs_destroy(h);
    cudaFree(llr); cudaFree(blk); cudaFree(bits);
    free(hb); free(hr);
    return 0;
}

// codec.cu — workload-side kernels of libpolarscs: CRC attach, systematic
// polar encoding, BPSK/AWGN modulation and the fused seeded generator.
// One warp per frame (grid-stride over frames); the frame's bits live
// bit-packed in shared memory so the n-stage XOR tree of Fig. 1 runs as
// word-wide shifts/XORs.
#include <cuda_runtime.h>

#include <algorithm>

#include "internal.h"

namespace polar {

constexpr uint32_t kFull = 0xFFFFFFFFu;

// ---------------------------------------------------------------- Philox4x32-10
struct U4 { uint32_t x, y, z, w; };

__device__ __forceinline__ U4 philox(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        const uint32_t lo0 = 0xD2511F53u * c.x, hi0 = __umulhi(0xD2511F53u, c.x);
        const uint32_t lo1 = 0xCD9E8D57u * c.z, hi1 = __umulhi(0xCD9E8D57u, c.z);
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

// ---------------------------------------------------------------- helpers
// x <- x F^{(x)n} on nw bit-packed words in shared memory
__device__ void transform_smem(uint32_t *w, int N, int nw, int lane) {
    const uint32_t masks[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};
    for (int j = lane; j < nw; j += 32) {
        uint32_t x = w[j];
#pragma unroll
        for (int s = 0; s < 5; s++)
            if ((1 << s) < N) x ^= (x >> (1 << s)) & masks[s];
        w[j] = x;
    }
    __syncwarp();
    for (int H = 1; H < nw; H <<= 1) {
        for (int j = lane; j < nw; j += 32)
            if ((j & H) == 0) w[j] ^= w[j + H];
        __syncwarp();
    }
}

// block bits (K) -> systematic codeword bits in w
__device__ void systematic_encode_smem(uint32_t *w, const CodecParams &P, int lane) {
    transform_smem(w, P.N, P.nw, lane);
    if (P.nonsys) return;                                 // non-systematic: c = u F
    for (int j = lane; j < P.nw; j += 32) w[j] &= P.info_words[j];
    __syncwarp();
    transform_smem(w, P.N, P.nw, lane);
}

// CRC remainder of the payload held as bytes (table-driven, linear over GF(2))
__device__ uint32_t crc_remainder_bytes(const uint8_t *payload, const CodecParams &P, int lane) {
    uint32_t syn = 0;
    const int Pl = P.K - P.c;
    for (int q = lane; q < Pl; q += 32)
        if (payload[q]) syn ^= P.crc_tab[q];
    return __reduce_xor_sync(kFull, syn);
}

// ---------------------------------------------------------------- kernels
__global__ void __launch_bounds__(kCodecWarps * 32) crc_attach_kernel(CodecParams P) {
    const int lane = threadIdx.x & 31;
    const int64_t wid = (int64_t)blockIdx.x * kCodecWarps + (threadIdx.x >> 5);
    const int64_t nwarps = (int64_t)gridDim.x * kCodecWarps;
    const int Pl = P.K - P.c;
    for (int64_t f = wid; f < P.n_frames; f += nwarps) {
        const uint8_t *pay = P.payload + f * Pl;
        uint8_t *blk = P.block_out + f * P.K;
        const uint32_t rem = P.c ? crc_remainder_bytes(pay, P, lane) : 0u;
        for (int q = lane; q < Pl; q += 32) blk[q] = pay[q];
        for (int d = lane; d < P.c; d += 32) blk[Pl + d] = (uint8_t)((rem >> (P.c - 1 - d)) & 1u);
    }
}

__global__ void __launch_bounds__(kCodecWarps * 32) encode_kernel(CodecParams P) {
    extern __shared__ uint32_t sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t *w = sm + warp * P.nw;
    const int64_t wid = (int64_t)blockIdx.x * kCodecWarps + warp;
    const int64_t nwarps = (int64_t)gridDim.x * kCodecWarps;
    for (int64_t f = wid; f < P.n_frames; f += nwarps) {
        for (int j = lane; j < P.nw; j += 32) w[j] = 0;
        __syncwarp();
        const uint8_t *blk = P.block_in + f * P.K;
        for (int q = lane; q < P.K; q += 32) {
            const int idx = P.info[q];
            if (blk[q] & 1) atomicOr(&w[idx >> 5], 1u << (idx & 31));
        }
        __syncwarp();
        systematic_encode_smem(w, P, lane);
        uint8_t *cw = P.codeword + f * P.N;
        for (int i = lane; i < P.N; i += 32) cw[i] = (uint8_t)((w[i >> 5] >> (i & 31)) & 1u);
        __syncwarp();
    }
}

// llr = scale * ((1 - 2x) + sigma * noise): two float32 roundings, no FMA
__global__ void modulate_kernel(CodecParams P) {
    const int64_t total = P.n_frames * P.N;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const float s = P.codeword[i] ? -1.0f : 1.0f;
        P.llr[i] = __fmul_rn(P.scale_f, __fadd_rn(s, __fmul_rn(P.sigma_f, P.noise[i])));
    }
}

// Fused generator: Philox payload (stream 0) -> CRC -> systematic encode ->
// Philox normals (stream 1, Box-Muller in double) -> LLR.
__global__ void __launch_bounds__(kCodecWarps * 32) generate_kernel(CodecParams P) {
    extern __shared__ uint32_t sm[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int pw = (P.K + 127) / 128 * 4;          // payload words (whole Philox counters)
    uint32_t *w = sm + warp * (P.nw + pw);
    uint32_t *pay = w + P.nw;
    const int64_t wid = (int64_t)blockIdx.x * kCodecWarps + warp;
    const int64_t nwarps = (int64_t)gridDim.x * kCodecWarps;
    const uint32_t k0 = (uint32_t)P.seed, k1 = (uint32_t)(P.seed >> 32);
    const int Pl = P.K - P.c;
    for (int64_t fl = wid; fl < P.n_frames; fl += nwarps) {
        const uint64_t fg = (uint64_t)(P.first_frame + fl);
        const uint32_t flo = (uint32_t)fg, fhi = (uint32_t)(fg >> 32);
        // payload bits: counter (q, frame_lo, frame_hi, 0) -> 128 bits
        for (int q = lane; q < pw / 4; q += 32) {
            const U4 r = philox(U4{(uint32_t)q, flo, fhi, 0u}, k0, k1);
            pay[4 * q] = r.x; pay[4 * q + 1] = r.y; pay[4 * q + 2] = r.z; pay[4 * q + 3] = r.w;
        }
        for (int j = lane; j < P.nw; j += 32) w[j] = 0;
        __syncwarp();
        // CRC over the payload, block = payload || crc, placed on A
        uint32_t syn = 0;
        for (int q = lane; q < Pl; q += 32)
            if ((pay[q >> 5] >> (q & 31)) & 1u) syn ^= P.crc_tab[q];
        const uint32_t rem = P.c ? __reduce_xor_sync(kFull, syn) : 0u;
        uint8_t *blk = P.block_out ? P.block_out + fl * P.K : nullptr;
        for (int q = lane; q < P.K; q += 32) {
            const uint32_t bit = (q < Pl) ? ((pay[q >> 5] >> (q & 31)) & 1u) : ((rem >> (P.c - 1 - (q - Pl))) & 1u);
            if (bit) {
                const int idx = P.info[q];
                atomicOr(&w[idx >> 5], 1u << (idx & 31));
            }
            if (blk) blk[q] = (uint8_t)bit;
        }
        __syncwarp();
        systematic_encode_smem(w, P, lane);
        // noise: counter (q, frame_lo, frame_hi, 1) -> 4 normals
        float *out = P.llr + fl * P.N;
        for (int q = lane; q < (P.N + 3) / 4; q += 32) {
            const U4 r = philox(U4{(uint32_t)q, flo, fhi, 1u}, k0, k1);
            const double u0 = ((double)r.x + 0.5) * (1.0 / 4294967296.0);
            const double u1 = ((double)r.y + 0.5) * (1.0 / 4294967296.0);
            const double u2 = ((double)r.z + 0.5) * (1.0 / 4294967296.0);
            const double u3 = ((double)r.w + 0.5) * (1.0 / 4294967296.0);
            const double r0 = sqrt(-2.0 * log(u0)), r1 = sqrt(-2.0 * log(u2));
            const double t0 = 2.0 * 3.141592653589793 * u1, t1 = 2.0 * 3.141592653589793 * u3;
            const float z[4] = {(float)(r0 * cos(t0)), (float)(r0 * sin(t0)), (float)(r1 * cos(t1)), (float)(r1 * sin(t1))};
            float o[4];
#pragma unroll
            for (int e = 0; e < 4; e++) {
                const int i = 4 * q + e;
                const float s = (i < P.N && ((w[i >> 5] >> (i & 31)) & 1u)) ? -1.0f : 1.0f;
                o[e] = __fmul_rn(P.scale_f, __fadd_rn(s, __fmul_rn(P.sigma_f, z[e])));
            }
            if (P.N >= 4) {
                *reinterpret_cast<float4 *>(out + 4 * q) = make_float4(o[0], o[1], o[2], o[3]);
            } else {
                for (int e = 0; e < 4 && 4 * q + e < P.N; e++) out[4 * q + e] = o[e];
            }
        }
        __syncwarp();
    }
}

static int codec_grid(int64_t n_frames) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n_frames + kCodecWarps - 1) / kCodecWarps;
    return (int)std::min<int64_t>(want, (int64_t)sms * 16);
}

cudaError_t launch_crc_attach(const CodecParams &p, cudaStream_t st) {
    crc_attach_kernel<<<codec_grid(p.n_frames), kCodecWarps * 32, 0, st>>>(p);
    return cudaGetLastError();
}
cudaError_t launch_encode(const CodecParams &p, cudaStream_t st) {
    encode_kernel<<<codec_grid(p.n_frames), kCodecWarps * 32, kCodecWarps * p.nw * 4, st>>>(p);
    return cudaGetLastError();
}
cudaError_t launch_modulate(const CodecParams &p, cudaStream_t st) {
    const int64_t total = p.n_frames * p.N;
    const int grid = (int)std::min<int64_t>((total + 255) / 256, 148 * 32);
    modulate_kernel<<<grid, 256, 0, st>>>(p);
    return cudaGetLastError();
}
cudaError_t launch_generate(const CodecParams &p, cudaStream_t st) {
    const int pw = (p.K + 127) / 128 * 4;
    generate_kernel<<<codec_grid(p.n_frames), kCodecWarps * 32, kCodecWarps * (p.nw + pw) * 4, st>>>(p);
    return cudaGetLastError();
}

}  // namespace polar

// Device Gaussian sinogram noise: the reference's documented recipe
// (simulate.gaussian_field, simulate.py:113-133) on the GPU.
//
// Stream: numpy's Philox4x64-10 bit generator keyed (master_seed mod 2^64,
// gate_index) with a zero counter.  Output word i of the stream is lane i % 4 of
// the block computed at counter (i / 4 + 1, 0, 0, 0) (numpy increments the
// counter before producing each block); Generator.random() maps a word w to
// (w >> 11) * 2^-53.  gaussian_field draws `pairs = ceil(count/2)` uniforms u1,
// then `pairs` uniforms u2, and writes sample 2k = r cos(phi), 2k+1 = r sin(phi)
// with r = sqrt(-2 log1p(-u1[k])), phi = 2 pi u2[k].
//
// The uniforms are bit-identical to numpy's.  sqrt is correctly rounded on both
// sides; log1p / sin / cos are CUDA's fp64 functions (<= 2 ulp vs the host libm),
// so a sample agrees with the host recipe to a few ulp (tests pin 1e-14).
#include "mct_internal.cuh"

namespace {

struct U64x4 {
    unsigned long long v[4];
};

__device__ __forceinline__ U64x4 philox4x64_10(unsigned long long blk, unsigned long long k0,
                                               unsigned long long k1) {
    const unsigned long long M0 = 0xD2E7470EE14C6C93ull, M1 = 0xCA5A826395121157ull;
    const unsigned long long W0 = 0x9E3779B97F4A7C15ull, W1 = 0xBB67AE8584CAA73Bull;
    unsigned long long c0 = blk, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r > 0) {
            k0 += W0;
            k1 += W1;
        }
        const unsigned long long hi0 = __umul64hi(M0, c0), lo0 = M0 * c0;
        const unsigned long long hi1 = __umul64hi(M1, c2), lo1 = M1 * c2;
        const unsigned long long n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0;
        c1 = lo1;
        c2 = n2;
        c3 = lo0;
    }
    U64x4 o;
    o.v[0] = c0;
    o.v[1] = c1;
    o.v[2] = c2;
    o.v[3] = c3;
    return o;
}

__device__ __forceinline__ double u01(unsigned long long w) {
    return (double)(w >> 11) * (1.0 / 9007199254740992.0);
}

__device__ __forceinline__ unsigned long long lane_of(const U64x4& b, int lane) {
    return lane == 0 ? b.v[0] : lane == 1 ? b.v[1] : lane == 2 ? b.v[2] : b.v[3];
}

// One thread per 4 consecutive sample pairs (one Philox block of u1 words).
__global__ void gaussian_field_kernel(unsigned long long k0, unsigned long long k1,
                                      long long count, double scale, const float* __restrict__ base,
                                      void* out, int out_f64) {
    const long long pairs = (count + 1) / 2;
    const long long g = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long k_beg = 4 * g;
    if (k_beg >= pairs) return;
    const U64x4 w1 = philox4x64_10((unsigned long long)g + 1, k0, k1);
    // u2 words pairs + k_beg .. +3 lie in (at most) two consecutive blocks
    const unsigned long long i2 = (unsigned long long)(pairs + k_beg);
    const U64x4 w2a = philox4x64_10(i2 / 4 + 1, k0, k1);
    const U64x4 w2b = philox4x64_10(i2 / 4 + 2, k0, k1);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const long long k = k_beg + j;
        if (k >= pairs) break;
        const double a1 = u01(w1.v[j]);
        const int l2 = (int)(i2 & 3) + j;  // lane of word pairs + k, across the two blocks
        const double a2 = u01(l2 < 4 ? lane_of(w2a, l2) : lane_of(w2b, l2 - 4));
        const double radius = sqrt(-2.0 * log1p(-a1));
        const double angle = (2.0 * 3.141592653589793) * a2;
        double sn, cs;
        sincos(angle, &sn, &cs);
        const double z[2] = {radius * cs, radius * sn};
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const long long e = 2 * k + h;
            if (e >= count) break;
            // numpy order: base + (scale * z), two roundings (no FMA contraction)
            const double v = __dadd_rn(base ? (double)base[e] : 0.0, __dmul_rn(scale, z[h]));
            if (out_f64)
                static_cast<double*>(out)[e] = v;
            else
                static_cast<float*>(out)[e] = (float)v;
        }
    }
}

}  // namespace

cudaError_t launch_gaussian_field(unsigned long long k0, unsigned long long k1, long long count,
                                  double scale, const float* base, void* out, int out_f64,
                                  cudaStream_t st) {
    const long long pairs = (count + 1) / 2;
    const long long threads = (pairs + 3) / 4;
    if (threads == 0) return cudaSuccess;
    const int block = 256;
    gaussian_field_kernel<<<(unsigned)((threads + block - 1) / block), block, 0, st>>>(
        k0, k1, count, scale, base, out, out_f64);
    return cudaGetLastError();
}

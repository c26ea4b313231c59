// Microbenchmark (tuning aid, not product): L1-resident gathers in K2's access
// pattern (32 lanes at element stride P along a row, rows advance) with 8-, 16-
// and 32-byte elements.  Reports gate-samples/s per element width (W gates per
// element: 8 B = 1, 16 B = 2, 32 B = 4).
#include <cstdio>
#include <cuda_runtime.h>

template <int W>
__global__ void __launch_bounds__(128) gather(const float* __restrict__ img, int rowlen, int rows,
                                              float P, int iters, float* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // each warp: one "ray bundle" starting at a block-dependent column
    const float c0 = (float)((blockIdx.x * 37 + warp * 11) % 64) + lane * P;
    float acc = 0.f;
    for (int it = 0; it < iters; ++it) {
        for (int r = 0; r < rows; r += 1) {
            const int c = (int)(c0 + r * 0.37f) + r * rowlen;
            const float* p = img + (size_t)c * (2 * W);
            if (W == 1) {
                float2 v = __ldg(reinterpret_cast<const float2*>(p));
                acc += v.x + v.y;
            } else if (W == 2) {
                float4 v = __ldg(reinterpret_cast<const float4*>(p));
                acc += v.x + v.y + v.z + v.w;
            } else {
                float a0, a1, a2, a3, a4, a5, a6, a7;
                asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                             : "=f"(a0), "=f"(a1), "=f"(a2), "=f"(a3), "=f"(a4), "=f"(a5), "=f"(a6),
                               "=f"(a7)
                             : "l"(p));
                acc += ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
            }
        }
    }
    if (acc == 12345.f) out[0] = acc;
}

int main() {
    const int rowlen = 160, rows = 64;  // 160 elements x 64 rows, x 32 B = 320 KB max (L2), per-block window small
    float* img;
    cudaMalloc(&img, (size_t)rowlen * (rows + 2) * 8 * sizeof(float) * 2);
    cudaMemset(img, 0, (size_t)rowlen * (rows + 2) * 8 * sizeof(float) * 2);
    float* out;
    cudaMalloc(&out, 4);
    const int blocks = 148 * 12, iters = 64;
    for (float P : {1.0f, 1.2f, 1.414f}) {
        for (int w = 1; w <= 4; w *= 2) {
            cudaEvent_t a, b;
            cudaEventCreate(&a);
            cudaEventCreate(&b);
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(a);
                if (w == 1) gather<1><<<blocks, 128>>>(img, rowlen, rows, P, iters, out);
                if (w == 2) gather<2><<<blocks, 128>>>(img, rowlen, rows, P, iters, out);
                if (w == 4) gather<4><<<blocks, 128>>>(img, rowlen, rows, P, iters, out);
                cudaEventRecord(b);
                cudaEventSynchronize(b);
            }
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            const double loads = (double)blocks * 4 * 32 * iters * rows;
            printf("P=%.3f W=%d  %.3f ms  lane-loads/s %.3e  gate-samples/s %.3e  B/s %.3e\n", P, w, ms,
                   loads / ms * 1e3, loads * w / ms * 1e3, loads * 8 * w / ms * 1e3);
        }
    }
    return 0;
}

// Microbenchmark (measurement aid, not product): the L1 data-pipe ceiling that
// K2 / K3 are bound by.  Every warp issues 16-byte __ldg loads from an
// L1-resident window; lane l of a request reads element base + l*P (P = element
// spacing: 1 = one contiguous 512-byte request = the 4-wavefront floor; K3's
// requests sit there, K2's 32 bins spread over P in [1, 1.41] columns).  Sixteen
// independent loads in flight per thread, 8 warps per block, 4 blocks per SM (one wave).
//
// Output (JSON on stdout): per P the delivered bytes/s (32 lanes x 16 B per
// request), requests/s, and the ratio to 128 B/clk/SM x SMs x the SM clock read
// with clock64 over the run (the data-pipe peak of one wavefront per cycle).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 4) gather16(const float4* __restrict__ buf, int mask,
                                                float P, int iters, unsigned* out,
                                                long long* span) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long t0 = clock64();
    unsigned acc = 0;
    int base = (blockIdx.x * 97 + warp * 13) & mask;
    const int off = (int)(lane * P);
    for (int it = 0; it < iters; ++it) {
        float4 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldg(buf + ((base + u * 64 + off) & mask));
#pragma unroll
        for (int u = 0; u < 16; ++u)
            acc ^= __float_as_uint(v[u].x) ^ __float_as_uint(v[u].y) ^ __float_as_uint(v[u].z) ^
                   __float_as_uint(v[u].w);
        base = (base + 1031) & mask;
    }
    if (acc == 0x12345u) out[0] = acc;
    if (threadIdx.x == 0) {  // per-block [start, end] in SM clocks
        span[2 * blockIdx.x] = t0;
        span[2 * blockIdx.x + 1] = clock64();
    }
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int window = 4096;  // 64 KB of float4: L1-resident on every SM
    float4* buf;
    cudaMalloc(&buf, (size_t)window * sizeof(float4));
    cudaMemset(buf, 0, (size_t)window * sizeof(float4));
    unsigned* out;
    long long* span;
    const int blocks = sms * 4, threads = 256, iters = 4096;  // one wave: 4 blocks per SM
    cudaMalloc(&out, 4);
    cudaMalloc(&span, 16 * (size_t)blocks);
    long long* hs = new long long[2 * blocks];
    printf("{\"sms\": %d, \"runs\": [", sms);
    bool first = true;
    for (float P : {1.0f, 1.2f, 1.414f}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float ms = 0.f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            gather16<<<blocks, threads>>>(buf, window - 1, P, iters, out, span);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        cudaMemcpy(hs, span, 16 * (size_t)blocks, cudaMemcpyDeviceToHost);
        // SM clock: the mean block lifetime (clock64 cycles) over the mean block
        // lifetime in ns is unknown per block; use the longest block's cycles over the
        // event time as a lower bound of the clock (blocks run the whole kernel)
        long long cmax = 0;
        for (int i = 0; i < blocks; ++i) cmax = hs[2 * i + 1] - hs[2 * i] > cmax ? hs[2 * i + 1] - hs[2 * i] : cmax;
        const double requests = (double)blocks * (threads / 32) * iters * 16;
        const double bytes = requests * 512.0;
        const double clk_hz = (double)cmax / (ms * 1e-3);
        const double peak = 128.0 * sms * clk_hz;
        printf("%s{\"P\": %.3f, \"ms\": %.4f, \"requests_per_s\": %.4e, \"delivered_GBps\": %.1f, "
               "\"sm_clock_mhz_est\": %.0f, \"pipe_peak_GBps\": %.1f, \"frac_of_pipe_peak\": %.4f, "
               "\"bytes_per_clk_per_sm\": %.1f}",
               first ? "" : ", ", P, ms, requests / (ms * 1e-3), bytes / (ms * 1e-3) / 1e9,
               clk_hz / 1e6, peak / 1e9, bytes / (ms * 1e-3) / peak,
               bytes / (ms * 1e-3) / sms / clk_hz);
        first = false;
    }
    printf("]}\n");
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

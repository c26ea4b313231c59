// Microbenchmark (measurement aid, not product): the L1 data-pipe ceiling that
// K2 / K3 are bound by.  Every warp issues 16-byte __ldg loads from an
// L1-resident window; lane l of a request reads element base + l*P (P = element
// spacing: 1 = one contiguous 512-byte request = the 4-wavefront floor; K3's
// requests sit there, K2's 32 bins spread over P in [1, 1.41] columns).  Eight
// independent loads in flight per thread, 8 warps per block, 8 blocks per SM.
//
// Output (JSON on stdout): per P the delivered bytes/s (32 lanes x 16 B per
// request), requests/s, and the ratio to 128 B/clk/SM x SMs x the SM clock read
// with clock64 over the run (the data-pipe peak of one wavefront per cycle).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256) gather16(const float4* __restrict__ buf, int window,
                                                float P, int iters, float* out,
                                                long long* cycles) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long t0 = clock64();
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    int base = (blockIdx.x * 97 + warp * 13) % (window / 2);
    const int off = (int)(lane * P);
    for (int it = 0; it < iters; ++it) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldg(buf + ((base + u * 48 + off) % window));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            acc.x += v[u].x;
            acc.y += v[u].y;
            acc.z += v[u].z;
            acc.w += v[u].w;
        }
        base = (base + 7) % (window / 2);
    }
    if (acc.x + acc.y + acc.z + acc.w == 12345.f) out[0] = acc.x;
    if (threadIdx.x == 0 && blockIdx.x == 0) *cycles = clock64() - t0;
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int window = 4096;  // 64 KB of float4: L1-resident per SM
    float4* buf;
    cudaMalloc(&buf, (size_t)window * sizeof(float4) + 4096);
    cudaMemset(buf, 0, (size_t)window * sizeof(float4) + 4096);
    float* out;
    long long* cyc;
    cudaMalloc(&out, 4);
    cudaMalloc(&cyc, 8);
    const int blocks = sms * 8, threads = 256, iters = 4096;
    printf("{\"sms\": %d, \"runs\": [", sms);
    bool first = true;
    for (float P : {1.0f, 1.2f, 1.414f}) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float ms = 0.f;
        for (int rep = 0; rep < 3; ++rep) {
            cudaEventRecord(a);
            gather16<<<blocks, threads>>>(buf, window, P, iters, out, cyc);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            cudaEventElapsedTime(&ms, a, b);
        }
        long long c = 0;
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        const double requests = (double)blocks * (threads / 32) * iters * 8;
        const double bytes = requests * 512.0;
        const double clk_hz = (double)c / (ms * 1e-3);  // block 0 spans ~the whole run
        const double peak = 128.0 * sms * clk_hz;
        printf("%s{\"P\": %.3f, \"ms\": %.4f, \"requests_per_s\": %.4e, \"delivered_GBps\": %.1f, "
               "\"sm_clock_mhz_est\": %.0f, \"pipe_peak_GBps\": %.1f, \"frac_of_pipe_peak\": %.4f}",
               first ? "" : ", ", P, ms, requests / (ms * 1e-3), bytes / (ms * 1e-3) / 1e9,
               clk_hz / 1e6, peak / 1e9, bytes / (ms * 1e-3) / peak);
        first = false;
    }
    printf("]}\n");
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

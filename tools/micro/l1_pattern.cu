// Microbenchmark (measurement aid, not product): L1 data-pipe cost of a warp-wide
// 16-byte gather as a function of the lane spacing P (lane l reads element
// floor(phase + l*P) of an L1-resident window), i.e. the access patterns of
// K2 (32 bins of one angle: P = sp/|cos| in [1, 1.41] columns) and K3 (32 columns
// of one row: P = |cos|/sp in [0, 1] bins).  For each P: SM cycles per warp request
// (one wave, 16 independent loads in flight per thread, phases averaged over 8
// fractional offsets).  The kernels' own cost per request is then compared with
// the pattern's cost averaged over their angle distribution (tools/micro/README).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void __launch_bounds__(256, 4) gather(const float4* __restrict__ buf, int mask, float P,
                                                 float phase, int iters, unsigned* out,
                                                 long long* span) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const long long t0 = clock64();
    unsigned acc = 0;
    int base = ((blockIdx.x * 97 + warp * 13) * 8) & mask;
    const int off = (int)(phase + lane * P);
    for (int it = 0; it < iters; ++it) {
        float4 v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) v[u] = __ldg(buf + ((base + u * 72 + off) & mask));
#pragma unroll
        for (int u = 0; u < 16; ++u)
            acc ^= __float_as_uint(v[u].x) ^ __float_as_uint(v[u].y) ^ __float_as_uint(v[u].z) ^
                   __float_as_uint(v[u].w);
        base = (base + 1031) & mask;
    }
    if (acc == 0x12345u) out[0] = acc;
    if (threadIdx.x == 0) {
        span[2 * blockIdx.x] = t0;
        span[2 * blockIdx.x + 1] = clock64();
    }
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int window = 4096;
    float4* buf;
    cudaMalloc(&buf, (size_t)window * sizeof(float4));
    cudaMemset(buf, 0, (size_t)window * sizeof(float4));
    unsigned* out;
    long long* span;
    const int blocks = sms * 4, threads = 256, iters = 1024;
    cudaMalloc(&out, 4);
    cudaMalloc(&span, 16 * (size_t)blocks);
    long long* hs = new long long[2 * blocks];
    printf("{\"sms\": %d, \"unit\": \"SM cycles per 32-lane 16-byte request\", \"runs\": [", sms);
    bool first = true;
    const float Ps[] = {0.0f, 0.125f, 0.25f, 0.375f, 0.5f, 0.625f, 0.75f, 0.875f, 1.0f,
                        1.05f, 1.1f, 1.15f, 1.2f, 1.25f, 1.3f, 1.35f, 1.414f, 1.5f, 2.0f};
    for (float P : Ps) {
        double cyc_sum = 0.0;
        for (int ph = 0; ph < 8; ++ph) {
            const float phase = ph / 8.0f;
            for (int rep = 0; rep < 2; ++rep)
                gather<<<blocks, threads>>>(buf, window - 1, P, phase, iters, out, span);
            cudaDeviceSynchronize();
            cudaMemcpy(hs, span, 16 * (size_t)blocks, cudaMemcpyDeviceToHost);
            long long cmax = 0;
            for (int i = 0; i < blocks; ++i)
                cmax = hs[2 * i + 1] - hs[2 * i] > cmax ? hs[2 * i + 1] - hs[2 * i] : cmax;
            const double req_per_sm = 4.0 * (threads / 32) * iters * 16;
            cyc_sum += (double)cmax / req_per_sm;
        }
        printf("%s{\"P\": %.3f, \"cycles_per_request\": %.3f}", first ? "" : ", ", P, cyc_sum / 8);
        first = false;
    }
    printf("]}\n");
    return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

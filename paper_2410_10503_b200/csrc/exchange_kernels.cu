// Fused cross-GPU exchange of gate-sharded PDHG over NVLink peer memory
// (one image-sized sum per iteration).
//
// Every rank's K4 (mct_iter_adjoint_update, mode 2) writes its partial
// dz_r = sum_{i in gates(r)} D_i^* A_i^* dy_i straight into its own half of a
// peer-visible (symmetric) buffer, double-buffered by iteration parity.  Then:
//   post   — one thread per peer q stores `epoch` into slot r of q's signal pad
//            with a system-scope release (after a system fence, so dz_r is
//            visible to q before the flag is);
//   update — every block acquires all W slots of its own pad (>= epoch), then
//            each element sums the W partials in rank order over NVLink loads
//            (identical arithmetic, hence identical z on every rank) and applies
//            z += dz, zbar = z + theta*dz  (the reference's z / z-bar update,
//            solvers.py:356-366, with p_i = 1).
// No collective library, no host round trip: the transfer is the update's own
// loads.  Parity double-buffering makes one flag per iteration sufficient: a
// rank overwrites its buffer of parity e only in iteration e+2, after it has
// seen every peer's post of e+1, which each peer issues only after its update
// of e (the last reader of that buffer) completed in stream order.
// The wait is bounded (~seconds): on expiry a device flag is raised and the host
// reports an error instead of hanging the GPU.
#include "mct_internal.cuh"

namespace {

#define XCH_SPIN_LIMIT (1ll << 24)

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__global__ void exchange_post_kernel(unsigned long long* const* pads, int world, int rank,
                                     unsigned long long epoch) {
    const int q = threadIdx.x;
    if (q >= world) return;
    __threadfence_system();
    st_release_sys(pads[q] + rank, epoch);
}

__global__ void __launch_bounds__(256) exchange_update_kernel(
    const float* const* parts, const unsigned long long* my_pad, int world,
    unsigned long long epoch, long long n, float* z, float* zbar, float theta,
    unsigned int* failed) {
    __shared__ int s_ok;
    if (threadIdx.x == 0) {
        int ok = 1;
        for (int q = 0; q < world && ok; ++q) {
            long long spins = 0;
            while (ld_acquire_sys(my_pad + q) < epoch) {
                if (++spins > XCH_SPIN_LIMIT) {
                    ok = 0;
                    break;
                }
                __nanosleep(64);
            }
        }
        if (!ok) atomicExch(failed, 1u);
        s_ok = ok;
    }
    __syncthreads();
    if (!s_ok) return;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        // volatile loads (ld.global.cv): a buffer is reused every other
        // iteration, so no cached copy of a peer's line may be trusted
        float s = __ldcv(parts[0] + i);
        for (int q = 1; q < world; ++q) s += __ldcv(parts[q] + i);  // rank order
        const float zq = z[i] + s;
        z[i] = zq;
        zbar[i] = fmaf(theta, s, zq);
    }
}

}  // namespace

cudaError_t launch_exchange_post(unsigned long long* const* pads, int world, int rank,
                                 unsigned long long epoch, cudaStream_t st) {
    exchange_post_kernel<<<1, ((world + 31) / 32) * 32, 0, st>>>(pads, world, rank, epoch);
    return cudaGetLastError();
}

cudaError_t launch_exchange_update(const float* const* parts, const unsigned long long* my_pad,
                                   int world, unsigned long long epoch, long long n, float* z,
                                   float* zbar, float theta, unsigned int* failed,
                                   cudaStream_t st) {
    int dev = 0, sms = 148;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    long long blocks = (n + 255) / 256;
    const long long cap = (long long)sms * 4;  // all blocks resident: one wait each
    blocks = blocks < cap ? blocks : cap;
    if (blocks < 1) blocks = 1;
    exchange_update_kernel<<<(unsigned)blocks, 256, 0, st>>>(parts, my_pad, world, epoch, n, z,
                                                             zbar, theta, failed);
    return cudaGetLastError();
}

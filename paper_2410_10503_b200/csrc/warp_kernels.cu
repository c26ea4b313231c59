// sm_100a kernels: warp adjoint fused with the z / zbar / x update (K4), the
// standalone warp forward, the dense-field transpose build, reductions.
//
// Reference: motion.py:178-194 (D, D^*), solvers.py:358-363 (z, zbar, x updates),
// linops.py:262-263 / functionals.py:71-82 (inner products).
#include "mct_internal.cuh"
#include "warp_math.cuh"

#include <cub/cub.cuh>

namespace {

#ifndef K4_LANES
#define K4_LANES 4
#endif
#ifndef K4_BLOCK1
#define K4_BLOCK1 256  // threads per block of single-lane (single-gate) launches
#endif
#ifndef K4_MINB1
#define K4_MINB1 0  // single-lane (single-gate) launches: compiler default
#endif
#ifndef K4_MINB
// gate-lane launches (blocks of 32 x K4_LANES threads): K4_MINB resident blocks of
// that size, i.e. 12 x 128 = 1536 threads per SM -> a 40-register cap (the
// allocation granularity rounds 65536 / 1536 down): more resident warps for the
// CSR gathers (C3 PDHG K4 94 -> 86 us)
#define K4_MINB 12
#endif
// K4 — one thread per pixel q of one slice (blockIdx.y): sums D_g^* img_k over
// the slice's items in a fixed order (deterministic), then
//   mode 0: out = sum                       (standalone D^* / gated adjoint)
//   mode 1: z += sum; zbar = z + sum_k (theta/p_k) D^*img_k; x = x_next
//   mode 2: dz = sum; x = x_next            (gate-sharded PDHG partial)
// LANES > 1 (multi-gate launches): a block is 32 pixels x LANES gate lanes;
// lane l sums gates l, l+LANES, ... in order, then lane 0 adds the LANES partial
// sums in lane order (fixed association: deterministic), so the per-pixel gate
// chains run LANES-wide in parallel instead of one after the other.
template <int MODE, int LANES>
__global__ void __launch_bounds__(LANES > 1 ? 32 * LANES : K4_BLOCK1, LANES > 1 ? K4_MINB : K4_MINB1)
update_kernel(UpdArgs p) {
    const int slice = blockIdx.y;
    const long long n = (long long)p.rows * p.cols;
    const int lane = LANES > 1 ? (int)threadIdx.y : 0;
    const long long q = (long long)blockIdx.x * (LANES > 1 ? 32 : blockDim.x) + threadIdx.x;
    if (LANES == 1 && q >= n) return;
    const bool valid = q < n;
    const long long qv = valid ? q : n - 1;
    const int qr = (int)(qv / p.cols), qc = (int)(qv - (long long)qr * p.cols);
    const long long o = (long long)slice * n + qv;
    // state loads issued ahead of the gather's dependent chain
    const float z0 = MODE == 1 && lane == 0 ? p.z[o] : 0.0f;
    const float xn = MODE != 0 && lane == 0 ? __ldg(p.x_next + o) : 0.0f;
    float sum = 0.0f, wsum = 0.0f;
    // paired items of the K3 launch whose partial images this gathers
    const int np = mct_pair_items(p.sel.ips * p.sel.num_slices, p.sel.last_part);
    for (int k = lane; k < p.sel.ips; k += LANES) {
        const int item = slice * p.sel.ips + k;
        int gate, iter;
        resolve_slice_item(p.sel, slice, k, gate, iter);
        const char* img = p.img_override
                              ? reinterpret_cast<const char*>(p.img_override)
                              : p.ws + mct_img_off(item, np, p.asplit, p.img_slot_bytes, p.wsg) +
                                    p.off_img;
        const int asplit = p.asplit;
        const size_t slot = p.img_slot_bytes;
        // sum of the adjoint's partial-image slots, fixed order (loads four at a time)
        auto fetch = [&](long long e) -> float {
            float v = __ldg(reinterpret_cast<const float*>(img) + e);
            for (int s = 1; s < asplit; s += 4) {
                float t[4];
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    t[j] = s + j < asplit
                               ? __ldg(reinterpret_cast<const float*>(img + (s + j) * slot) + e)
                               : 0.0f;
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    if (s + j < asplit) v += t[j];
            }
            return v;
        };
        float v;
        if (p.warps == nullptr) {
            v = fetch(q);
        } else {
            const WarpT wd = load_warp_t(p.warps + (p.sel.gates ? (long long)slice * p.N + gate : 0));
            v = warp_adjoint_at(wd, fetch, qr, qc);
        }
        sum += v;
        if (MODE == 1) wsum = fmaf(p.gp[gate].theta_over_p, v, wsum);
    }
    if (LANES > 1) {
        __shared__ float s_sum[LANES][32], s_w[LANES][32];
        s_sum[lane][threadIdx.x] = sum;
        s_w[lane][threadIdx.x] = wsum;
        __syncthreads();
        if (lane != 0 || !valid) return;
#pragma unroll
        for (int l = 1; l < LANES; ++l) {
            sum += s_sum[l][threadIdx.x];
            wsum += s_w[l][threadIdx.x];
        }
    }
    if (MODE == 0) {
        p.out[o] = sum;
    } else if (MODE == 1) {
        const float zq = z0 + sum;
        p.z[o] = zq;
        p.zbar[o] = zq + wsum;
        p.x[o] = xn;
    } else {
        p.dz[o] = sum;
        p.x[o] = xn;
    }
}

__global__ void z_update_kernel(long long n, const float* __restrict__ dz, float* z, float* zbar,
                                float theta) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const float d = dz[i];
        const float zq = z[i] + d;
        z[i] = zq;
        zbar[i] = fmaf(theta, d, zq);
    }
}

__global__ void epoch_advance_kernel(int* ctr, int inc) { *ctr += inc; }

__global__ void warp_fwd_plain_kernel(const WarpDesc* __restrict__ desc, const float* __restrict__ x,
                                      float* out, int rows, int cols) {
    const long long n = (long long)rows * cols;
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const WarpDesc wd = *desc;
    const int r = (int)(q / cols), c = (int)(q - (long long)r * cols);
    if (wd.kind == MCT_WARP_IDENTITY) {
        out[q] = x[q];
        return;
    }
    out[q] = warp_apply_at(wd, r, c,
                           [&](int rr, int cc) { return __ldg(x + (long long)rr * cols + cc); });
}

// ------------------------------------------------- dense transpose build --
__global__ void dense_count_kernel(WarpDesc wd, int* cnt) {
    const long long n = (long long)wd.rows * wd.cols;
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int r = (int)(p / wd.cols), c = (int)(p - (long long)r * wd.cols);
    TapSet t = warp_taps(wd, r, c);
    for (int dr = 0; dr < 2; ++dr)
        for (int dc = 0; dc < 2; ++dc) {
            int rr = t.r0 + dr, cc = t.c0 + dc;
            if (rr >= 0 && rr < wd.rows && cc >= 0 && cc < wd.cols && tap_weight(t, dr, dc) != 0.0f)
                atomicAdd(cnt + (long long)rr * wd.cols + cc, 1);
        }
}

__global__ void dense_fill_kernel(WarpDesc wd, int* cursor, int* tidx, float* tw) {
    const long long n = (long long)wd.rows * wd.cols;
    const long long p = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= n) return;
    const int r = (int)(p / wd.cols), c = (int)(p - (long long)r * wd.cols);
    TapSet t = warp_taps(wd, r, c);
    for (int dr = 0; dr < 2; ++dr)
        for (int dc = 0; dc < 2; ++dc) {
            int rr = t.r0 + dr, cc = t.c0 + dc;
            float w = tap_weight(t, dr, dc);
            if (rr >= 0 && rr < wd.rows && cc >= 0 && cc < wd.cols && w != 0.0f) {
                int pos = atomicAdd(cursor + (long long)rr * wd.cols + cc, 1);
                tidx[pos] = (int)p;
                tw[pos] = w;
            }
        }
}

// Sort each (short) segment by source pixel so the gather order — and hence the
// fp32 sum — is independent of atomic arrival order.
__global__ void dense_sort_kernel(long long n, const int* tptr, int* tidx, float* tw) {
    const long long q = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= n) return;
    const int e0 = tptr[q], e1 = tptr[q + 1];
    for (int i = e0 + 1; i < e1; ++i) {
        int key = tidx[i];
        float w = tw[i];
        int k = i - 1;
        while (k >= e0 && tidx[k] > key) {
            tidx[k + 1] = tidx[k];
            tw[k + 1] = tw[k];
            --k;
        }
        tidx[k + 1] = key;
        tw[k + 1] = w;
    }
}

// ------------------------------------------------------------ reductions --
// Fixed thread->element map and fixed trees: the fp64 result is bitwise
// reproducible run to run.  Pass 1: `parts` blocks per segment, each a
// contiguous chunk; pass 2 (parts > 1): one block sums the partials in order.
template <typename T>
__device__ __forceinline__ double block_sum(double acc, T* sh) {
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
        __syncthreads();
    }
    return sh[0];
}

__global__ void __launch_bounds__(256) reduce_kernel(const float* __restrict__ a,
                                                     const float* __restrict__ b, long long len,
                                                     long long stride, int mode, int parts,
                                                     double* out) {
    __shared__ double sh[256];
    const int s = blockIdx.y, part = blockIdx.x;
    const long long chunk = (len + parts - 1) / parts;
    const long long lo = part * chunk, hi = min(len, lo + chunk);
    const float* as = a + (long long)s * stride;
    const float* bs = b ? b + (long long)s * stride : nullptr;
    double acc = 0.0;
#pragma unroll 4
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) {
        const double x = (double)__ldg(as + i);
        if (mode == MCT_REDUCE_DOT) {
            acc += x * (double)(bs ? __ldg(bs + i) : 1.0f);
        } else {
            const double d = bs ? x - (double)__ldg(bs + i) : x;
            acc += d * d;
        }
    }
    const double r = block_sum(acc, sh);
    if (threadIdx.x == 0) out[(long long)s * parts + part] = r;
}

__global__ void __launch_bounds__(256) dot_f64_kernel(const double* __restrict__ a,
                                                      const double* __restrict__ b, long long len,
                                                      int parts, double* out) {
    __shared__ double sh[256];
    const int part = blockIdx.x;
    const long long chunk = (len + parts - 1) / parts;
    const long long lo = part * chunk, hi = min(len, lo + chunk);
    double acc = 0.0;
    for (long long i = lo + threadIdx.x; i < hi; i += blockDim.x) acc += a[i] * (b ? b[i] : 1.0);
    const double r = block_sum(acc, sh);
    if (threadIdx.x == 0) out[part] = r;
}

// sum `parts` consecutive partials of each segment, in order
__global__ void __launch_bounds__(256) partials_kernel(const double* __restrict__ part_in,
                                                       int parts, double* out) {
    __shared__ double sh[256];
    const int s = blockIdx.x;
    double acc = 0.0;
    for (int i = threadIdx.x; i < parts; i += blockDim.x) acc += part_in[(long long)s * parts + i];
    const double r = block_sum(acc, sh);
    if (threadIdx.x == 0) out[s] = r;
}

__global__ void axpby_kernel(long long n, float alpha, const float* __restrict__ x, float beta,
                             float* y) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        y[i] = fmaf(alpha, x[i], beta * y[i]);
}

__global__ void axpby_mixed_kernel(long long n, double alpha, const void* __restrict__ x, int xf64,
                                   double beta, void* y, int yf64) {
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double xv = xf64 ? static_cast<const double*>(x)[i] : (double)static_cast<const float*>(x)[i];
        if (yf64) {
            double* yp = static_cast<double*>(y);
            yp[i] = alpha * xv + (beta == 0.0 ? 0.0 : beta * yp[i]);
        } else {
            float* yp = static_cast<float*>(y);
            yp[i] = (float)(alpha * xv + (beta == 0.0 ? 0.0 : beta * (double)yp[i]));
        }
    }
}

// max |x| over the grid: block maxima combined with an integer atomicMax on the
// bit patterns (order-preserving for non-negative floats; max is order-free, so
// the result is deterministic).  *out must be zeroed first.
__global__ void absmax_kernel(const float* __restrict__ x, long long n, float* out) {
    __shared__ float sh[256];
    float m = 0.0f;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x)
        m = fmaxf(m, fabsf(x[i]));
    sh[threadIdx.x] = m;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) sh[threadIdx.x] = fmaxf(sh[threadIdx.x], sh[threadIdx.x + w]);
        __syncthreads();
    }
    if (threadIdx.x == 0) atomicMax(reinterpret_cast<int*>(out), __float_as_int(sh[0]));
}

inline int grid_for(long long n, int block) {
    long long g = (n + block - 1) / block;
    if (g > 148LL * 32) g = 148LL * 32;
    return (int)(g < 1 ? 1 : g);
}

}  // namespace

cudaError_t launch_update(const UpdArgs& a, int mode, int slices, cudaStream_t st) {
    const long long n = (long long)a.rows * a.cols;
    if (a.sel.ips >= K4_LANES && K4_LANES > 1) {  // several gates per slice: gate lanes
        dim3 block(32, K4_LANES), grid((unsigned)((n + 31) / 32), slices);
        switch (mode) {
            case 0: update_kernel<0, K4_LANES><<<grid, block, 0, st>>>(a); break;
            case 1: update_kernel<1, K4_LANES><<<grid, block, 0, st>>>(a); break;
            case 2: update_kernel<2, K4_LANES><<<grid, block, 0, st>>>(a); break;
            default: return cudaErrorInvalidValue;
        }
        return cudaGetLastError();
    }
    dim3 block(K4_BLOCK1), grid((unsigned)((n + K4_BLOCK1 - 1) / K4_BLOCK1), slices);
    switch (mode) {
        case 0: update_kernel<0, 1><<<grid, block, 0, st>>>(a); break;
        case 1: update_kernel<1, 1><<<grid, block, 0, st>>>(a); break;
        case 2: update_kernel<2, 1><<<grid, block, 0, st>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

cudaError_t launch_z_update(long long n, const float* dz, float* z, float* zbar, float theta,
                            cudaStream_t st) {
    z_update_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, dz, z, zbar, theta);
    return cudaGetLastError();
}

cudaError_t launch_epoch_advance(int* ctr, int inc, cudaStream_t st) {
    epoch_advance_kernel<<<1, 1, 0, st>>>(ctr, inc);
    return cudaGetLastError();
}

cudaError_t launch_warp_fwd_plain(const WarpDesc* d_desc, const float* x, float* out, int rows,
                                  int cols, cudaStream_t st) {
    const long long n = (long long)rows * cols;
    warp_fwd_plain_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(d_desc, x, out, rows, cols);
    return cudaGetLastError();
}

static int reduce_parts(long long len) {
    long long p = (len + 2047) / 2048;  // >= 2K elements per block
    return (int)(p < 1 ? 1 : (p > MCT_REDUCE_PARTS ? MCT_REDUCE_PARTS : p));
}

cudaError_t launch_reduce(const float* a, const float* b, long long len, int segs, long long stride,
                          int mode, double* out, double* scratch, cudaStream_t st) {
    const int parts = scratch ? reduce_parts(len) : 1;
    if (parts == 1) {
        reduce_kernel<<<dim3(1, segs), 256, 0, st>>>(a, b, len, stride, mode, 1, out);
        return cudaGetLastError();
    }
    reduce_kernel<<<dim3(parts, segs), 256, 0, st>>>(a, b, len, stride, mode, parts, scratch);
    partials_kernel<<<segs, 256, 0, st>>>(scratch, parts, out);
    return cudaGetLastError();
}

cudaError_t launch_axpby(long long n, float alpha, const float* x, float beta, float* y,
                         cudaStream_t st) {
    axpby_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, alpha, x, beta, y);
    return cudaGetLastError();
}

cudaError_t launch_axpby_mixed(long long n, double alpha, const void* x, int xf64, double beta,
                               void* y, int yf64, cudaStream_t st) {
    axpby_mixed_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, alpha, x, xf64, beta, y, yf64);
    return cudaGetLastError();
}

cudaError_t launch_dot_f64(const double* a, const double* b, long long n, double* out,
                           double* scratch, cudaStream_t st) {
    const int parts = scratch ? reduce_parts(n) : 1;
    if (parts == 1) {
        dot_f64_kernel<<<1, 256, 0, st>>>(a, b, n, 1, out);
        return cudaGetLastError();
    }
    dot_f64_kernel<<<parts, 256, 0, st>>>(a, b, n, parts, scratch);
    partials_kernel<<<1, 256, 0, st>>>(scratch, parts, out);
    return cudaGetLastError();
}

cudaError_t launch_absmax(const float* x, long long n, float* out, cudaStream_t st) {
    cudaError_t e = cudaMemsetAsync(out, 0, sizeof(float), st);
    if (e != cudaSuccess) return e;
    absmax_kernel<<<grid_for(n, 256), 256, 0, st>>>(x, n, out);
    return cudaGetLastError();
}

// Synchronous (plan construction only).
cudaError_t build_dense_transpose(const WarpDesc& desc, int** tptr_out, int** tidx_out,
                                  float** tw_out, long long* nnz_out, cudaStream_t st) {
    const long long n = (long long)desc.rows * desc.cols;
    int *cnt = nullptr, *tptr = nullptr, *tidx = nullptr;
    float* tw = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    int total = 0;
    cudaError_t e;
    const unsigned nb = (unsigned)((n + 255) / 256);
#define CK(x)              \
    do {                   \
        e = (x);           \
        if (e != cudaSuccess) goto fail; \
    } while (0)
    CK(cudaMalloc(&cnt, (n + 1) * sizeof(int)));
    CK(cudaMalloc(&tptr, (n + 1) * sizeof(int)));
    CK(cudaMemsetAsync(cnt, 0, (n + 1) * sizeof(int), st));
    dense_count_kernel<<<nb, 256, 0, st>>>(desc, cnt);
    CK(cudaGetLastError());
    CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, cnt, tptr, (int)(n + 1), st));
    CK(cudaMalloc(&tmp, tmp_bytes));
    CK(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, tptr, (int)(n + 1), st));
    CK(cudaMemcpyAsync(&total, tptr + n, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaMalloc(&tidx, (size_t)(total > 0 ? total : 1) * sizeof(int)));
    CK(cudaMalloc(&tw, (size_t)(total > 0 ? total : 1) * sizeof(float)));
    CK(cudaMemcpyAsync(cnt, tptr, n * sizeof(int), cudaMemcpyDeviceToDevice, st));
    dense_fill_kernel<<<nb, 256, 0, st>>>(desc, cnt, tidx, tw);
    CK(cudaGetLastError());
    dense_sort_kernel<<<nb, 256, 0, st>>>(n, tptr, tidx, tw);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    cudaFree(cnt);
    cudaFree(tmp);
    *tptr_out = tptr;
    *tidx_out = tidx;
    *tw_out = tw;
    *nnz_out = total;
    return cudaSuccess;
fail:
    cudaFree(cnt);
    cudaFree(tmp);
    cudaFree(tptr);
    cudaFree(tidx);
    cudaFree(tw);
    return e;
#undef CK
}

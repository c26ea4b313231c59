// sm_100a kernels of the hot path: fused prox+warp+pack, Joseph forward with
// fused dual prox, pixel-driven transpose-gather adjoint.
//
// Reference: projector.py:126-217 (Joseph traversal tables, gather/scatter),
// motion.py:132-183 (warp), functionals.py:40-68 (proxes), solvers.py:316-366.
#include "mct_internal.cuh"
#include "warp_math.cuh"

#include <math.h>

namespace {

// ---------------------------------------------------------------------------
// K1 / pack: W = D_g(x_new), x_new = prox_g(x - tau*zbar) (or x_new = x), written
// into the padded row-major X and padded transposed XT of the item workspace.
// Tile 32x32, block 32x8, transposed store staged through shared memory.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) pack_kernel(PackArgs p) {
    __shared__ float tile[32][33];
    const int item = blockIdx.z;
    int slice, gate, iter;
    resolve_item(p.sel, item, slice, gate, iter);
    const int k_in_slice = item - slice * p.sel.ips;
    const float* __restrict__ x = p.x + (long long)slice * p.x_slice_stride;
    const float* __restrict__ zb = p.zbar ? p.zbar + (long long)slice * p.x_slice_stride : nullptr;
    const bool prox = (zb != nullptr);
    const float tau = p.tau, cp = p.cprox;
    const int rows = p.rows, cols = p.cols;

    WarpDesc wd;
    bool ident = (p.warps == nullptr);
    if (!ident) {
        wd = p.warps[p.sel.gates ? (long long)slice * p.N + gate : 0];
        ident = (wd.kind == MCT_WARP_IDENTITY);
    }

    auto xnew = [&](int rr, int cc) -> float {
        long long o = (long long)rr * cols + cc;
        float v = __ldg(x + o);
        if (prox) v = (v - tau * __ldg(zb + o)) * cp;
        return v;
    };

    char* base = p.ws + (size_t)item * p.item_bytes;
    float* X = reinterpret_cast<float*>(base + p.off_x);
    float* XT = reinterpret_cast<float*>(base + p.off_xt);

    const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
    const int tx = threadIdx.x, ty = threadIdx.y;
    const bool writer = prox && k_in_slice == 0 && p.x_next != nullptr;
    bool bad = false;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int r = r0 + ty + 8 * k, c = c0 + tx;
        float w = 0.0f;
        if (r < rows && c < cols) {
            if (ident) {
                w = xnew(r, c);
            } else {
                w = warp_apply_at(wd, r, c, xnew);
            }
            X[(long long)r * p.wx + MCT_PADX + c] = w;
            if (writer) {
                float xn = xnew(r, c);
                p.x_next[(long long)slice * p.x_slice_stride + (long long)r * cols + c] = xn;
                bad |= !isfinite(xn);
            }
        }
        tile[ty + 8 * k][tx] = w;
    }
    if (writer && p.status && __any_sync(0xffffffffu, bad)) {
        if ((threadIdx.x & 31) == 0) atomicMin(p.status, (unsigned long long)iter);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        int c = c0 + ty + 8 * k, r = r0 + tx;
        if (r < rows && c < cols) XT[(long long)c * p.wxt + MCT_PADX + r] = tile[tx][ty + 8 * k];
    }
}

// Copy a plain (A, B) sinogram into the padded DY layout of each item.
__global__ void pad_sino_kernel(const float* __restrict__ sino, char* ws, size_t item_bytes,
                                size_t off_dy, int A, int B, int wy, int pb) {
    const int item = blockIdx.z;
    const int a = blockIdx.y;
    float* DY = reinterpret_cast<float*>(ws + (size_t)item * item_bytes + off_dy);
    const float* s = sino + ((long long)item * A + a) * B;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < B; j += gridDim.x * blockDim.x)
        DY[(long long)a * wy + pb + j] = s[j];
}

// ---------------------------------------------------------------------------
// K2: Joseph forward A (projector.py:201-207 with the weights of :160-183).
// Block = 8 warps = 8 consecutive angles x 32 consecutive bins: the warps walk
// nearly the same image lines so most of the 2 taps per sample hit L1.
// Along the dominant axis the continuous minor index advances by a constant
// slope; it is carried in 32.32 fixed point (integer part = tap index, fraction
// = interpolation weight), anchored on a per-ray fp64 start, so no float
// conversions sit in the inner loop.  Rows that cannot contribute are skipped
// analytically; the padded layout keeps the loop branch-free.
// MODE 0: plain store.  MODE 1: fused dual prox (functionals.py:53-68,
// solvers.py:341-357) writing y, dy (padded, for K3) and optionally proj.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float frac_from_fx(unsigned lo) {
    return __uint_as_float(0x3f800000u | (lo >> 9)) - 1.0f;
}

template <int MODE>
__global__ void __launch_bounds__(256) fwd_kernel(FwdArgs p) {
    const int item = blockIdx.z;
    const int a = blockIdx.y * 8 + threadIdx.y;
    const int j = blockIdx.x * 32 + threadIdx.x;
    if (a >= p.A) return;  // warp-uniform (one angle per warp)
    const bool active = j < p.B;
    const RayAngle ra = p.ang[a];
    const char* base = p.ws + (size_t)item * p.item_bytes;
    const int cd = ra.cols_dom;
    const float* __restrict__ X =
        reinterpret_cast<const float*>(base + (cd ? p.off_xt : p.off_x)) + MCT_PADX;
    const int stride = cd ? p.wxt : p.wx;
    const int nmaj = cd ? p.cols : p.rows;
    const int lim = cd ? p.rows : p.cols;

    // per-ray range of dominant-axis samples with a tap inside the grid
    double c0 = 0.0;
    int lo = nmaj, hi = -1;
    if (active) {
        const double sj = ((double)j - p.jmid) * p.sp;
        c0 = ra.P * sj + ra.Q;
        if (ra.slope == 0.0) {
            if (c0 > -1.0 && c0 < (double)lim) { lo = 0; hi = nmaj - 1; }
        } else {
            const double ka = (-1.0 - c0) / ra.slope, kb = ((double)lim - c0) / ra.slope;
            const double top = (double)nmaj + 2.0;
            const double kmin = fmin(fmax(fmin(ka, kb), -2.0), top);
            const double kmax = fmin(fmax(fmax(ka, kb), -2.0), top);
            lo = max(0, (int)floor(kmin));
            hi = min(nmaj - 1, (int)ceil(kmax));
        }
    }
    // the warp walks the union of its rays' ranges in lock-step so every load
    // instruction reads one contiguous segment of one image row (coalesced);
    // samples whose taps fall outside the grid are predicated off.
    const int wlo = __reduce_min_sync(0xffffffffu, lo);
    const int whi = __reduce_max_sync(0xffffffffu, hi);
    float acc = 0.0f;
    if (wlo <= whi) {
        const unsigned lim1 = active ? (unsigned)(lim + 1) : 0u;
        long long fx = __double2ll_rn((c0 + (double)wlo * ra.slope) * 4294967296.0);
        const long long sfx = ra.slope_fx;
        const float* row = X + (long long)wlo * stride;
        float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
        int k = wlo;
#define MCT_FWD_SAMPLE(ACC, FX, ROW)                                           \
        {                                                                      \
            const int i0 = (int)((FX) >> 32);                                  \
            float v0 = 0.f, v1 = 0.f;                                          \
            if ((unsigned)(i0 + 1) < lim1) {                                   \
                v0 = __ldg((ROW) + i0);                                        \
                v1 = __ldg((ROW) + i0 + 1);                                    \
            }                                                                  \
            ACC += fmaf(frac_from_fx((unsigned)(FX)), v1 - v0, v0);            \
        }
        for (; k + 3 <= whi; k += 4) {
            const long long f1 = fx + sfx, f2 = f1 + sfx, f3 = f2 + sfx;
            MCT_FWD_SAMPLE(a0, fx, row)
            MCT_FWD_SAMPLE(a1, f1, row + stride)
            MCT_FWD_SAMPLE(a2, f2, row + 2 * stride)
            MCT_FWD_SAMPLE(a3, f3, row + 3 * stride)
            fx = f3 + sfx;
            row += 4 * stride;
        }
        for (; k <= whi; ++k) {
            MCT_FWD_SAMPLE(a0, fx, row)
            fx += sfx;
            row += stride;
        }
#undef MCT_FWD_SAMPLE
        acc = (a0 + a1) + (a2 + a3);
    }
    const float proj = acc * ra.step;
    if (!active) return;
    if (MODE == 0) {
        p.out[(long long)item * p.out_item_stride + (long long)a * p.B + j] = proj;
    } else {
        int slice, gate, iter;
        resolve_item(p.sel, item, slice, gate, iter);
        const long long off = (((long long)slice * p.N + gate) * p.A + a) * p.B + j;
        const GateParam gp = p.gp[gate];
        const float yv = p.y[off];
        const float dv = __ldg(p.d + off);
        const float yn = (fmaf(gp.sigma, proj, yv) - gp.sigma * dv) * gp.dual_inv;
        p.y[off] = yn;
        float* DY = reinterpret_cast<float*>(const_cast<char*>(base) + p.off_dy);
        DY[(long long)a * p.wy + p.pb + j] = yn - yv;
        if (p.proj) p.proj[off] = proj;
        if (!isfinite(yn) && p.status)
            atomicMin(p.status + 1, ((unsigned long long)iter << 20) | (unsigned long long)gate);
    }
}

// ---------------------------------------------------------------------------
// K3: A^* as a deterministic transpose-gather (no atomics).  Pixel (r, c) at
// angle a receives  step * max(0, 1 - |j - jc|*g) * dy[a, j]  from the bins j
// around its detector coordinate jc — exactly the Joseph weight of
// projector.py:161-166 seen from the pixel (the tent identity pinned by
// test_projector.py:78-93).  jc is anchored per 16x16 tile and angle in fp64
// (integer bin + fp32 fraction) and offset per pixel in fp32, which keeps the
// coordinate error ~1e-6 bins at 1024^2.
// ---------------------------------------------------------------------------
#define ADJ_TW 32      // tile width (columns) = one warp
#define ADJ_TH 16      // tile height (rows)
#define ADJ_PPT 4      // pixels per thread (rows ty, ty+4, ty+8, ty+12)
#define ADJ_THREADS (ADJ_TW * ADJ_TH / ADJ_PPT)
#define ADJ_CH ADJ_THREADS
#define MAGIC_F 12582912.0f  // 1.5 * 2^23
#define MAGIC_I 0x4B400000

// Each thread owns ADJ_PPT pixels of one tile column so the per-angle constants
// (two shared-memory broadcasts) are amortised over several pixels; a warp
// covers 32 consecutive columns of a row, so its bin reads are one contiguous
// run of the sinogram row (coalesced, L1-resident).
template <int K>
__global__ void __launch_bounds__(ADJ_THREADS) adj_kernel(AdjArgs p, float* out,
                                                          long long out_stride) {
    __shared__ float4 s_a[ADJ_CH];  // f0 - 0.5, cos/sp, sin/sp, step*g
    __shared__ float2 s_b[ADJ_CH];  // step - step*g/2, row offset (int bits)
    __shared__ float s_c[ADJ_CH];   // step (general footprint path)
    const int item = blockIdx.z;
    const int tid = threadIdx.y * ADJ_TW + threadIdx.x;
    const int r0 = blockIdx.y * ADJ_TH, c0 = blockIdx.x * ADJ_TW;
    const int c = c0 + threadIdx.x;
    const double u0 = (double)r0 + 0.5 * (ADJ_TH - 1) - 0.5 * (double)(p.rows - 1);
    const double v0 = (double)c0 + 0.5 * (ADJ_TW - 1) - 0.5 * (double)(p.cols - 1);
    const float dv = (float)threadIdx.x - 0.5f * (ADJ_TW - 1);
    float du[ADJ_PPT];
    bool inside[ADJ_PPT];
#pragma unroll
    for (int m = 0; m < ADJ_PPT; ++m) {
        const int rr = threadIdx.y + (ADJ_TH / ADJ_PPT) * m;
        inside[m] = (r0 + rr < p.rows) && (c < p.cols);
        // rows below the image reuse the thread's first row (result discarded) so
        // every bin read stays inside the padded sinogram
        du[m] = (float)(inside[m] ? rr : threadIdx.y) - 0.5f * (ADJ_TH - 1);
    }
    const char* base = p.ws + (size_t)item * p.item_bytes;
    const float* __restrict__ DY = reinterpret_cast<const float*>(base + p.off_dy);

    float acc[ADJ_PPT];
#pragma unroll
    for (int m = 0; m < ADJ_PPT; ++m) acc[m] = 0.0f;
    const bool any_inside = inside[0];
    for (int a0 = 0; a0 < p.A; a0 += ADJ_CH) {
        const int cnt = min(ADJ_CH, p.A - a0);
        __syncthreads();
        if (tid < cnt) {
            const AdjAngle aa = p.ang[a0 + tid];
            const double jc = v0 * aa.cs - u0 * aa.sn + p.jmid;
            const double J = floor(jc);
            const float gs = aa.step * aa.g;
            s_a[tid] = make_float4((float)(jc - J) - 0.5f, (float)aa.cs, (float)aa.sn, gs);
            s_b[tid] = make_float2(aa.step - 0.5f * gs,
                                   __int_as_float((a0 + tid) * p.wy + p.pb + (int)J));
            s_c[tid] = aa.step;
        }
        __syncthreads();
        if (!any_inside) continue;
#pragma unroll 2
        for (int t = 0; t < cnt; ++t) {
            const float4 A4 = s_a[t];
            const float2 B2 = s_b[t];
            const float tv = fmaf(dv, A4.y, A4.x);  // anchor fraction - 0.5 + dv*cos/sp
            const float* q = DY + __float_as_int(B2.y);
#pragma unroll
            for (int m = 0; m < ADJ_PPT; ++m) {
                const float tm = fmaf(-du[m], A4.z, tv);        // jc - J - 0.5
                const float tb = tm + MAGIC_F;
                const int kf = __float_as_int(tb) - MAGIC_I;     // ~floor(jc - J)
                const float e = tm - (tb - MAGIC_F);             // jc - J - kf - 0.5
                const float* qq = q + kf;
                if (K == 0) {
                    // bins kf, kf+1 at distances 0.5+e, 0.5-e
                    const float w0 = fmaxf(0.0f, fmaf(-e, A4.w, B2.x));
                    const float w1 = fmaxf(0.0f, fmaf(e, A4.w, B2.x));
                    acc[m] = fmaf(w0, __ldg(qq), acc[m]);
                    acc[m] = fmaf(w1, __ldg(qq + 1), acc[m]);
                } else {
                    const float step = s_c[t];
                    const float d = e + 0.5f;
#pragma unroll
                    for (int mm = -K; mm <= K + 1; ++mm) {
                        const float dist = fabsf((float)mm - d);
                        const float w = fmaxf(0.0f, fmaf(-dist, A4.w, step));
                        acc[m] = fmaf(w, __ldg(qq + mm), acc[m]);
                    }
                }
            }
        }
    }
#pragma unroll
    for (int m = 0; m < ADJ_PPT; ++m) {
        if (!inside[m]) continue;
        const int r = r0 + threadIdx.y + (ADJ_TH / ADJ_PPT) * m;
        if (out) {
            out[(long long)item * out_stride + (long long)r * p.cols + c] = acc[m];
        } else {
            float* IMG = reinterpret_cast<float*>(const_cast<char*>(base) + p.off_img);
            IMG[(long long)r * p.cols + c] = acc[m];
        }
    }
}

}  // namespace

cudaError_t launch_pack(const PackArgs& a, int items, cudaStream_t st) {
    dim3 block(32, 8), grid((a.cols + 31) / 32, (a.rows + 31) / 32, items);
    pack_kernel<<<grid, block, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_pad_sino(const float* sino, char* ws, size_t item_bytes, size_t off_dy, int A,
                            int B, int wy, int pb, int items, cudaStream_t st) {
    dim3 block(256), grid((B + 255) / 256, A, items);
    pad_sino_kernel<<<grid, block, 0, st>>>(sino, ws, item_bytes, off_dy, A, B, wy, pb);
    return cudaGetLastError();
}

cudaError_t launch_fwd(const FwdArgs& a, int mode, int items, cudaStream_t st) {
    dim3 block(32, 8), grid((a.B + 31) / 32, (a.A + 7) / 8, items);
    if (mode == 0)
        fwd_kernel<0><<<grid, block, 0, st>>>(a);
    else
        fwd_kernel<1><<<grid, block, 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_adj(const AdjArgs& a, int kfoot, int items, float* out,
                       long long out_item_stride, cudaStream_t st) {
    dim3 block(ADJ_TW, ADJ_TH / ADJ_PPT),
        grid((a.cols + ADJ_TW - 1) / ADJ_TW, (a.rows + ADJ_TH - 1) / ADJ_TH, items);
    switch (kfoot) {
        case 0: adj_kernel<0><<<grid, block, 0, st>>>(a, out, out_item_stride); break;
        case 1: adj_kernel<1><<<grid, block, 0, st>>>(a, out, out_item_stride); break;
        case 2: adj_kernel<2><<<grid, block, 0, st>>>(a, out, out_item_stride); break;
        case 3: adj_kernel<3><<<grid, block, 0, st>>>(a, out, out_item_stride); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

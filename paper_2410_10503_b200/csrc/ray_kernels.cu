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
        double dacc = 0.0;
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
        // fp32 partial sums over chunks of <= 64 samples, chunk totals in fp64:
        // the accumulation error stays ~1e-7 relative at n = 1024
        for (int kc = wlo; kc <= whi; kc += 64) {
            const int kend = min(whi, kc + 63);
            float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
            int k = kc;
            for (; k + 3 <= kend; k += 4) {
                const long long f1 = fx + sfx, f2 = f1 + sfx, f3 = f2 + sfx;
                MCT_FWD_SAMPLE(a0, fx, row)
                MCT_FWD_SAMPLE(a1, f1, row + stride)
                MCT_FWD_SAMPLE(a2, f2, row + 2 * stride)
                MCT_FWD_SAMPLE(a3, f3, row + 3 * stride)
                fx = f3 + sfx;
                row += 4 * stride;
            }
            for (; k <= kend; ++k) {
                MCT_FWD_SAMPLE(a0, fx, row)
                fx += sfx;
                row += stride;
            }
            dacc += (double)((a0 + a1) + (a2 + a3));
        }
#undef MCT_FWD_SAMPLE
        acc = (float)dacc;
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
#define ADJ_TH 32      // tile height (rows)
#define ADJ_PPT 8      // consecutive rows per thread
#define ADJ_THREADS (ADJ_TW * ADJ_TH / ADJ_PPT)
#define ADJ_CH ADJ_THREADS

// K3: A^* as a deterministic transpose-gather (no atomics).  Pixel (r, c) at
// angle a receives  step * max(0, 1 - |j - jc|*g) * dy[a, j]  from the bins j
// around its detector coordinate jc = (v cos - u sin)/sp + (B-1)/2: exactly the
// Joseph weight of projector.py:161-166 seen from the pixel (the tent identity
// pinned by test_projector.py:78-93).
// jc is carried in 32.32 fixed point: an fp64 anchor per (tile, angle) plus
// exact integer steps cos/sp, sin/sp per column / row, so the bin index and the
// interpolation fraction are exact to ~1e-9 bins at any image size.
// Each thread owns 8 consecutive rows of one column: the two shared-memory
// broadcasts of the per-angle constants are amortised over 8 pixels, and a warp
// reads one contiguous run of a sinogram row per pixel row (coalesced, L1).
// The angle loop may be split over blockIdx.z (partial image slots, summed in a
// fixed order by K4).  fp32 partial sums per chunk of 128 angles, fp64 totals.
template <int K>
__global__ void __launch_bounds__(ADJ_THREADS) adj_kernel(AdjArgs p) {
    __shared__ longlong2 s_t[ADJ_CH];  // anchor (with sinogram row base), cos/sp
    __shared__ int4 s_u[ADJ_CH];       // sin/sp (lo, hi), step, step*g
    const int item = blockIdx.z / p.asplit;
    const int split = blockIdx.z - item * p.asplit;
    const int a_beg = (int)((long long)p.A * split / p.asplit);
    const int a_end = (int)((long long)p.A * (split + 1) / p.asplit);
    const int tid = threadIdx.y * ADJ_TW + threadIdx.x;
    const int r0 = blockIdx.y * ADJ_TH, c0 = blockIdx.x * ADJ_TW;
    const int c = c0 + threadIdx.x;
    const int rt = r0 + threadIdx.y * ADJ_PPT;
    const int nrows = min(ADJ_PPT, p.rows - rt);         // warp-uniform
    const int txc = min((int)threadIdx.x, p.cols - 1 - c0);  // clamp lanes past the image
    const double u0 = (double)r0 - 0.5 * (double)(p.rows - 1);
    const double v0 = (double)c0 - 0.5 * (double)(p.cols - 1);
    const char* base = p.ws + (size_t)item * p.item_bytes;
    const float* __restrict__ DY = reinterpret_cast<const float*>(base + p.off_dy);
    const long long row_off = (long long)(threadIdx.y * ADJ_PPT);

    double tot[ADJ_PPT];
#pragma unroll
    for (int m = 0; m < ADJ_PPT; ++m) tot[m] = 0.0;
    for (int a0 = a_beg; a0 < a_end; a0 += ADJ_CH) {
        const int cnt = min(ADJ_CH, a_end - a0);
        __syncthreads();
        if (tid < cnt) {
            const AdjAngle aa = p.ang[a0 + tid];
            const double jcA = v0 * aa.cs - u0 * aa.sn + p.jmid;
            const long long TA = __double2ll_rn(jcA * 4294967296.0) +
                                 ((long long)((a0 + tid) * p.wy + p.pb) << 32);
            s_t[tid] = make_longlong2(TA, aa.csx);
            s_u[tid] = make_int4((int)(unsigned)aa.snx, (int)(aa.snx >> 32),
                                 __float_as_int(aa.step), __float_as_int(aa.step * aa.g));
        }
        __syncthreads();
        if (nrows <= 0) continue;
        float acc[ADJ_PPT];
#pragma unroll
        for (int m = 0; m < ADJ_PPT; ++m) acc[m] = 0.0f;
#pragma unroll 2
        for (int t = 0; t < cnt; ++t) {
            const longlong2 T2 = s_t[t];
            const int4 U = s_u[t];
            const long long snx = ((long long)U.y << 32) | (unsigned)U.x;
            const float step = __int_as_float(U.z), gs = __int_as_float(U.w);
            const float h = step - gs;
            long long T = T2.x + (long long)txc * T2.y - row_off * snx;
#pragma unroll
            for (int m = 0; m < ADJ_PPT; ++m) {
                if (m < nrows) {
                    const int kf = (int)(T >> 32);                // bin index (incl. row base)
                    const float d = frac_from_fx((unsigned)T);     // jc - floor(jc) in [0,1)
                    const float* qq = DY + kf;
                    if (K == 0) {
                        const float w0 = fmaxf(0.0f, fmaf(-d, gs, step));  // bin floor(jc)
                        const float w1 = fmaxf(0.0f, fmaf(d, gs, h));      // bin floor(jc)+1
                        acc[m] = fmaf(w0, __ldg(qq), acc[m]);
                        acc[m] = fmaf(w1, __ldg(qq + 1), acc[m]);
                    } else {
#pragma unroll
                        for (int mm = -K; mm <= K + 1; ++mm) {
                            const float dist = fabsf((float)mm - d);
                            const float w = fmaxf(0.0f, fmaf(-dist, gs, step));
                            acc[m] = fmaf(w, __ldg(qq + mm), acc[m]);
                        }
                    }
                }
                T -= snx;
            }
        }
#pragma unroll
        for (int m = 0; m < ADJ_PPT; ++m) tot[m] += (double)acc[m];
    }
    if (c >= p.cols) return;
    float* IMG = reinterpret_cast<float*>(const_cast<char*>(base) + p.off_img +
                                          (size_t)split * p.img_slot_bytes);
#pragma unroll
    for (int m = 0; m < ADJ_PPT; ++m)
        if (m < nrows) IMG[(long long)(rt + m) * p.cols + c] = (float)tot[m];
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

int choose_asplit(const mct_ray_plan* rp, int items) {
    const long long tiles = (long long)((rp->cols + ADJ_TW - 1) / ADJ_TW) *
                            ((rp->rows + ADJ_TH - 1) / ADJ_TH) * (items > 0 ? items : 1);
    const long long target = 148LL * 8;  // >= 8 resident blocks per SM
    long long s = (target + tiles - 1) / tiles;
    s = s < 1 ? 1 : s;
    s = s > MCT_MAX_ASPLIT ? MCT_MAX_ASPLIT : s;
    const long long by_angles = rp->A / 16 > 0 ? rp->A / 16 : 1;  // >= 16 angles per split
    return (int)(s < by_angles ? s : by_angles);
}

cudaError_t launch_adj(const AdjArgs& a, int kfoot, int items, cudaStream_t st) {
    dim3 block(ADJ_TW, ADJ_TH / ADJ_PPT),
        grid((a.cols + ADJ_TW - 1) / ADJ_TW, (a.rows + ADJ_TH - 1) / ADJ_TH, items * a.asplit);
    switch (kfoot) {
        case 0: adj_kernel<0><<<grid, block, 0, st>>>(a); break;
        case 1: adj_kernel<1><<<grid, block, 0, st>>>(a); break;
        case 2: adj_kernel<2><<<grid, block, 0, st>>>(a); break;
        case 3: adj_kernel<3><<<grid, block, 0, st>>>(a); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// sm_100a kernels of the hot path: fused prox+warp+pack (K1), Joseph forward with
// fused dual prox (K2), pixel-driven transpose-gather adjoint (K3).
//
// Reference: projector.py:126-217 (Joseph traversal tables, gather/scatter),
// motion.py:132-183 (warp), functionals.py:40-68 (proxes), solvers.py:316-366.
#include "mct_internal.cuh"
#include "warp_math.cuh"

#include <math.h>

#include <map>
#include <mutex>
#include <type_traits>
#include <utility>

namespace {

// Angle slots of a single-item (mirror) launch: slot s < nsingle is a
// self-paired angle (0, and A/2 for even A), slot s >= nsingle the mirror pair
// (q, A-q), q = s - nsingle + 1.  Sinogram row / float2 slot of angle a in the
// mirror DY layout: pairs (q, h), self-paired angles (0, s).
__host__ __device__ __forceinline__ int mir_nsingle(int A) { return (A % 2 == 0) ? 2 : 1; }
__host__ __device__ __forceinline__ int mir_slots(int A) { return mir_nsingle(A) + (A - 1) / 2; }
__device__ __forceinline__ void mir_row_slot(int a, int A, int& row, int& slot) {
    const int np = (A - 1) / 2;
    if (a == 0) { row = 0; slot = 0; }
    else if (a <= np) { row = a; slot = 0; }
    else if (2 * a == A) { row = 0; slot = 1; }
    else { row = A - a; slot = 1; }
}

// ---------------------------------------------------------------------------
// K1 / pack: W = D_g(x_new), x_new = prox_g(x - tau*zbar) (or x_new = x), written
// into the padded row-major X2 and transposed XT2 of the item workspace in the
// "value + forward difference" pair layout: X2[r][c] = (W[r][c], W[r][c+1] -
// W[r][c]) (zero outside the image), so a Joseph sample is one 8-byte load and
// one FMA, v.x + frac * v.y.  A TxT tile plus a one-pixel halo of W is built in
// shared memory, then both layouts are stored coalesced.  Multi-gate launches
// use 32x32 tiles (4 elements per thread); single-gate launches 16x16 tiles with
// one halo element per thread, so the warp's dependent load chain is paid once
// per thread on a small grid.  Same per-element arithmetic (bitwise equal).
// ---------------------------------------------------------------------------
template <int T, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) pack_kernel(PackArgs p) {
    constexpr int HR = T + 1, HC = T + 2;  // rows r0 .. r0+T, cols c0-1 .. c0+T
    __shared__ float tile[HR][HC + 1];
    const int item = p.sel.first + blockIdx.z;
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

    // Both layouts hold float4 elements = two float2 slots (value, forward
    // difference).  Pair mode: slot (item & 1) of the pair region holds this
    // item.  Single-item (mirror) mode: slot 0 holds W, slot 1 the column mirror
    // Wm[r][c] = W[r][cols-1-c] (X) / XT[cols-1-c] (XT) of the item's own region.
    const bool paired = item < p.pair_items;
    char* base = paired ? p.ws + mct_pair_off(item >> 1, p.wsg)
                        : p.ws + mct_item_off(item, p.pair_items, p.wsg);
    const int s0 = paired ? (item & 1) : 0;
    float2* X = reinterpret_cast<float2*>(base + (paired ? p.off_px : p.off_x)) + 2 * MCT_PADX;
    float2* XT = reinterpret_cast<float2*>(base + (paired ? p.off_pxt : p.off_xt)) + 2 * MCT_PADX;

    const int c0 = blockIdx.x * T, r0 = blockIdx.y * T;
    const int tid = threadIdx.x;
    const bool writer = prox && k_in_slice == 0 && p.x_next != nullptr;
    bool bad = false;
    for (int idx = tid; idx < HR * HC; idx += THREADS) {
        const int i = idx / HC, jj = idx - i * HC;
        const int r = r0 + i, c = c0 - 1 + jj;
        float w = 0.0f;
        if (r < rows && c >= 0 && c < cols) {
            w = ident ? xnew(r, c) : warp_apply_at(wd, r, c, xnew);
            if (writer && i < T && jj >= 1 && jj <= T) {
                const float xn = xnew(r, c);
                p.x_next[(long long)slice * p.x_slice_stride + (long long)r * cols + c] = xn;
                bad |= !isfinite(xn);
            }
        }
        tile[i][jj] = w;
    }
    if (writer && p.status && __any_sync(0xffffffffu, bad)) {
        if ((threadIdx.x & 31) == 0) atomicMin(p.status, (unsigned long long)iter);
    }
    __syncthreads();
#pragma unroll
    for (int o = tid; o < T * T; o += THREADS) {
        const int i = o / T, tx = o - i * T;
        const int r = r0 + i, c = c0 + tx;
        if (r < rows && c < cols) {
            const float w = tile[i][tx + 1];
            const long long row = (long long)r * p.wx;
            X[2 * (row + c) + s0] = make_float2(w, tile[i][tx + 2] - w);
            if (c == 0) X[2 * (row - 1) + s0] = make_float2(0.0f, w);
            if (!paired) {  // mirror slot: element cols-1-c pairs W[c] with W[c-1]
                X[2 * (row + cols - 1 - c) + 1] = make_float2(w, tile[i][tx] - w);
                if (c == cols - 1) X[2 * (row - 1) + 1] = make_float2(0.0f, w);
            }
        }
        // transposed: element (c, r) pairs W[r][c] with W[r+1][c]
        const int ct = c0 + i, rt = r0 + tx;
        if (rt < rows && ct < cols) {
            const float w = tile[tx][i + 1];
            const float2 v = make_float2(w, tile[tx + 1][i + 1] - w);
            XT[2 * ((long long)ct * p.wxt + rt) + s0] = v;
            if (rt == 0) XT[2 * ((long long)ct * p.wxt - 1) + s0] = make_float2(0.0f, w);
            if (!paired) {  // mirror slot: row cols-1-ct of the transposed layout
                const long long rowm = (long long)(cols - 1 - ct) * p.wxt;
                XT[2 * (rowm + rt) + 1] = v;
                if (rt == 0) XT[2 * (rowm - 1) + 1] = make_float2(0.0f, w);
            }
        }
    }
}

// Copy a plain (A, B) sinogram into the padded float4 DY layout of each item,
// pre-scaled by the angle's step length (A^* then only needs the tent weights):
// paired items into their slot of the pair region (row a), single items into
// the mirror layout of their own region (row / slot of mir_row_slot).
__global__ void pad_sino_kernel(const float* __restrict__ sino, const AdjAngle* __restrict__ ang,
                                char* ws, WsGeom wsg, size_t off_dy1,
                                size_t off_dy2, int A, int B, int wy, int pb, int pair_items,
                                int first) {
    const int item = first + blockIdx.z;
    const bool paired = item < pair_items;
    const int a = blockIdx.y;
    const float step = ang[a].step;
    int row = a, slot = item & 1;
    if (!paired) mir_row_slot(a, A, row, slot);
    float* DY = reinterpret_cast<float*>(
                    ws + (paired ? mct_pair_off(item >> 1, wsg)
                                 : mct_item_off(item, pair_items, wsg)) +
                    (paired ? off_dy2 : off_dy1)) + slot;
    const float* s = sino + ((long long)item * A + a) * B;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < B; j += gridDim.x * blockDim.x) {
        const long long e = 4 * ((long long)row * wy + pb + j);
        const float v = s[j] * step;
        DY[e] = v;      // element j: (slot 0, slot 1) at bin j, then at bin j + 1
        DY[e - 2] = v;  // element j - 1, bin j
    }
}

// ---------------------------------------------------------------------------
// K2: Joseph forward A (projector.py:201-207 with the weights of :160-183).
// Block = FWD_ANGLES (4) warps = 4 consecutive angle slots x 32 consecutive bins:
// the warps walk nearly the same image lines, so most taps hit L1.
// Along the dominant axis the continuous minor index advances by a constant
// slope.  It is carried in 32.32 fixed point whose integer part also carries
// the row offset, so one 64-bit add advances both, the integer part is the
// pair-packed tap address and the low word is the interpolation fraction; the
// start is anchored per ray in fp64.  Each warp walks the union of its 32 rays'
// sample ranges in lock-step (every load = one contiguous row segment); the
// common core of the ranges runs without predicates, the ragged edges with.
// fp32 partial sums per 64-sample chunk, fp64 chunk totals.
// MODE 0: plain store.  MODE 1: fused dual prox (functionals.py:53-68,
// solvers.py:341-357) writing y, dy (pair-packed, for K3) and optionally proj.
// ---------------------------------------------------------------------------
#define FX_ONE 4294967296.0
#define INV_2_24 5.9604644775390625e-08f

// 32.32 fixed-point add / subtract on an explicit (lo, hi) register pair, so the
// integer part stays a plain 32-bit register usable as an unsigned index.
__device__ __forceinline__ void fx_add(unsigned& lo, unsigned& hi, unsigned ilo, unsigned ihi) {
    asm("add.cc.u32 %0, %0, %2;\n\taddc.u32 %1, %1, %3;" : "+r"(lo), "+r"(hi) : "r"(ilo), "r"(ihi));
}
__device__ __forceinline__ void fx_sub(unsigned& lo, unsigned& hi, unsigned ilo, unsigned ihi) {
    asm("sub.cc.u32 %0, %0, %2;\n\tsubc.u32 %1, %1, %3;" : "+r"(lo), "+r"(hi) : "r"(ilo), "r"(ihi));
}

#ifndef FWD_ACQREL
#define FWD_ACQREL 1
#endif
#define FWD_ANGLES MCT_FWD_ANGLES  // warps (= consecutive angles) per block; they share L1 lines
#ifndef FWD_MIN_BLOCKS2
#define FWD_MIN_BLOCKS2 16        // gate pairs: 16 x 2 warps resident, 64 registers
#endif
#ifndef FWD_LPT_NOSPLIT
#define FWD_LPT_NOSPLIT 0  // 1: longest-rays-first order for unsplit single-gate walks too
#endif
#ifndef FWD_LPT_SPLIT
#define FWD_LPT_SPLIT 1    // longest-rays-first order for split single-gate walks
#endif
#ifndef FWD_MIN_BLOCKS_M
#define FWD_MIN_BLOCKS_M 7        // single-item mirror walks (72 registers, no spills)
#endif

// (value, forward difference) of float2 slot h of a float4 element
__device__ __forceinline__ float tv(const float4& v, int h) { return h ? v.z : v.x; }
__device__ __forceinline__ float td(const float4& v, int h) { return h ? v.w : v.y; }
// DY (sinogram increments for A^*) element j: (slot 0, slot 1) at bin j in .xy and
// at bin j + 1 in .zw, so both slots' taps are float2 lanes (FFMA2 in K3)
__device__ __forceinline__ float dlo(const float4& v, int h) { return h ? v.y : v.x; }
__device__ __forceinline__ float dhi(const float4& v, int h) { return h ? v.w : v.z; }

// K2 walks two rays per warp lane at once, one 16-byte load per sample:
//   MIR = 0 (gate pairs): items 2p, 2p+1 at angle a (pair region);
//   MIR = 1 (single item): angles a and A-a of one item, the second through the
//     column-mirrored image (item region, slot 1) -- ray (A-a, j) of W is ray
//     (a, j) of Wm[r][c] = W[r][cols-1-c] (rows-dominant: cont' = cols-1-cont;
//     cols-dominant: the same samples in reverse column order), so one walk and
//     one set of fractions serve both angles.
// Every per-ray sum is accumulated as by the one-ray walk: 8 samples per trip,
// fp32 partial sums per 64 samples, fp64 totals.
template <int MODE, int LPT, int MIR>
__global__ void __launch_bounds__(32 * (MIR ? FWD_ANGLES : MCT_FWD_ANGLES_P),
                                  MIR ? FWD_MIN_BLOCKS_M : FWD_MIN_BLOCKS2)
    fwd_kernel(FwdArgs p) {
    using V = float4;
    constexpr int G = 2;
    const int ks = MIR ? p.ksplit : 1;  // gate pairs never split rays (launch_fwd)
    const int group = blockIdx.z / ks;  // item (MIR) or gate pair
    const int part = blockIdx.z - group * ks;
    // LPT (single-gate launches): grid (angle groups, bin tiles by distance rank, parts): every angle group's
    // central tiles (the longest rays) are dispatched before any edge tile, so the
    // last, partial wave holds the shortest blocks
    // (multi-gate launches keep bins fastest: better L2 locality across gates)
    const int btile = LPT ? [&] {
        const int ntile = gridDim.y, c = ntile / 2, k = blockIdx.y;
        if (k == 0) return c;
        const int jr = k - 1, below = c, above = ntile - 1 - c;
        const int pairs = below < above ? below : above;
        if (jr < 2 * pairs) return (jr & 1) ? c + 1 + (jr >> 1) : c - 1 - (jr >> 1);
        const int r = jr - 2 * pairs;
        return below > above ? c - 1 - pairs - r : c + 1 + pairs + r;
    }() : (int)blockIdx.x;
    // lane -> (bin, slot): IL consecutive lanes walk the same bin of IL consecutive angle
    // slots (nearly parallel rays), so 8 lanes of a request span 8 / IL bins: the L1
    // delivers a 16-byte request in 4 clocks while 8 consecutive lanes stay inside 128
    // bytes, 8 clocks once they spread further (tools/micro/l1_pattern.cu)
    constexpr int IL = MCT_FWD_IL, BW = 32 / IL;
    constexpr int NW = MIR ? FWD_ANGLES : MCT_FWD_ANGLES_P;  // warps per block
    const int s_raw = ((LPT ? blockIdx.x : blockIdx.y) * NW + threadIdx.y) * IL +
                      (int)threadIdx.x % IL;
    const int nslot = MIR ? mir_slots(p.A) : p.A;
    bool warp_on = s_raw < nslot;            // per lane; no early exit (block syncs below)
    if (MIR && p.sel.last_part && p.item0 + (int)blockIdx.z / ks == p.n_items - 1) {
        // a half item: slots of the first (part 1) or second (part 2) half of the angle pairs
        const int s_mid = mir_nsingle(p.A) + mct_half_q(p.A) - 1;
        warp_on = warp_on && (p.sel.last_part == 1 ? s_raw < s_mid : s_raw >= s_mid);
    }
    const int sl = warp_on ? s_raw : nslot - 1;
    const int nsingle = MIR ? mir_nsingle(p.A) : 0;
    // angle walked by this warp (slot 0); MIR: slot 1 is angle A - a
    const int a = !MIR ? sl : (sl < nsingle ? (sl == 0 ? 0 : p.A / 2) : sl - nsingle + 1);
    const bool pair1 = !MIR || sl >= nsingle;  // slot 1 holds a real ray
    const int j = btile * BW + (int)threadIdx.x / IL;
    const bool active = warp_on && j < p.B;
    const int jj = active ? j : p.B - 1;  // idle lanes shadow the last bin (no store)
    const RayAngle ra = p.ang[a];
    const int item0 = p.item0 + (MIR ? group : G * group);  // pairs: item0 is even
    const int np = mct_pair_items(p.n_items, p.sel.last_part);  // paired items of the call
    const char* base0 = p.ws + mct_item_off(item0, np, p.wsg);  // counters
    const char* tb = MIR ? base0 : p.ws + mct_pair_off(item0 >> 1, p.wsg);
    const int cd = ra.cols_dom;
    // tap index = hi(fx) >= 0: the row pad is folded into fx so the address is one
    // unsigned 32x64 multiply-add
    const V* __restrict__ X2 = reinterpret_cast<const V*>(
        tb + (MIR ? (cd ? p.off_xt : p.off_x) : (cd ? p.off_pxt : p.off_px)));
    const int stride = cd ? p.wxt : p.wx;
    const int nmaj = cd ? p.cols : p.rows;
    const int lim = cd ? p.rows : p.cols;

    // per-ray range of dominant-axis samples that can have a tap inside the grid
    const double sj = ((double)jj - p.jmid) * p.sp;
    const double c0 = ra.P * sj + ra.Q;
    int lo = nmaj, hi = -1;
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
    int wlo = __reduce_min_sync(0xffffffffu, lo);  // union of the warp's ranges
    int whi = __reduce_max_sync(0xffffffffu, hi);
    int clo = __reduce_max_sync(0xffffffffu, lo);        // common core
    int chi = __reduce_min_sync(0xffffffffu, hi);
    // this block's share of the walk: part `part` of ks equal pieces
    const int wlen = whi - wlo + 1;
    const int k_lo = wlo + (int)((long long)wlen * part / ks);
    const int k_hi = wlo + (int)((long long)wlen * (part + 1) / ks) - 1;
    wlo = k_lo;
    whi = k_hi;
    clo = max(clo, k_lo);
    chi = min(chi, k_hi);
    double tot[G];
#pragma unroll
    for (int h = 0; h < G; ++h) tot[h] = 0.0;
    if (warp_on && wlo <= whi) {
        if (clo > chi) { clo = whi + 1; chi = whi; }     // no common core: all edge
        const long long inc64 = ra.slope_fx + ((long long)stride << 32);
        const unsigned ilo = (unsigned)inc64, ihi = (unsigned)(inc64 >> 32);
        const long long fx0 = __double2ll_rn((c0 + (double)wlo * ra.slope) * FX_ONE) +
                              ((long long)(wlo * stride + MCT_PADX) << 32);
        unsigned flo = (unsigned)fx0, fhi = (unsigned)(fx0 >> 32);
        int rowoff = wlo * stride + MCT_PADX;
        const unsigned lim1 = (unsigned)(lim + 1);
        double dacc[G];
        float ea[G];  // ragged-edge samples (predicated on the tap range)
#pragma unroll
        for (int h = 0; h < G; ++h) { dacc[h] = 0.0; ea[h] = 0.0f; }
        // lanes of one warp may walk different angles (MCT_FWD_IL); with a non-square
        // image their dominant axes differ in length and the union walk steps past the
        // shorter one's last row: X / XT carry max(rows, cols) rows, zero beyond the
        // image, so those samples read zeros
        int k = wlo;
        for (; k < clo; ++k) {
            const int i0 = (int)fhi - rowoff;
            if ((unsigned)(i0 + 1) < lim1) {
                const V v = __ldg(X2 + fhi);
                const float f = (float)(flo >> 8) * INV_2_24;
#pragma unroll
                for (int h = 0; h < G; ++h) ea[h] += fmaf(f, td(v, h), tv(v, h));
            }
            fx_add(flo, fhi, ilo, ihi);
            rowoff += stride;
        }
        // core: every lane's taps are inside the padded row (pads read zero)
        for (int kc = k; kc <= chi; kc += 64) {
            const int kend = min(chi, kc + 63);
            float s[G][4], t[G][4];  // sums of v0 and of frac*2^24*(x[i+1] - x[i])
#pragma unroll
            for (int h = 0; h < G; ++h)
#pragma unroll
                for (int q = 0; q < 4; ++q) s[h][q] = t[h][q] = 0.0f;
            int kk = kc;
            // 8 samples per trip
            for (; kk + 7 <= kend; kk += 8) {
                unsigned lo8[8], hi8[8];
                lo8[0] = flo;
                hi8[0] = fhi;
#pragma unroll
                for (int u = 1; u < 8; ++u) {
                    lo8[u] = lo8[u - 1];
                    hi8[u] = hi8[u - 1];
                    fx_add(lo8[u], hi8[u], ilo, ihi);
                }
                V v[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) v[u] = __ldg(X2 + hi8[u]);
                flo = lo8[7];
                fhi = hi8[7];
                fx_add(flo, fhi, ilo, ihi);
#pragma unroll
                for (int hb = 0; hb < 2; ++hb) {
#pragma unroll
                    for (int h = 0; h < G; ++h)
#pragma unroll
                        for (int q = 0; q < 4; ++q) s[h][q] += tv(v[4 * hb + q], h);
#pragma unroll
                    for (int h = 0; h < G; ++h)
#pragma unroll
                        for (int q = 0; q < 4; ++q)
                            t[h][q] = fmaf((float)(lo8[4 * hb + q] >> 8), td(v[4 * hb + q], h), t[h][q]);
                }
            }
            for (; kk <= kend; ++kk) {
                const V v0 = __ldg(X2 + fhi);
                const float f = (float)(flo >> 8);
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    s[h][0] += tv(v0, h);
                    t[h][0] = fmaf(f, td(v0, h), t[h][0]);
                }
                fx_add(flo, fhi, ilo, ihi);
            }
#pragma unroll
            for (int h = 0; h < G; ++h)
                dacc[h] += (double)((s[h][0] + s[h][1]) + (s[h][2] + s[h][3])) +
                           (double)((t[h][0] + t[h][1]) + (t[h][2] + t[h][3])) * (double)INV_2_24;
            k = kend + 1;
        }
        rowoff = k * stride + MCT_PADX;
        for (; k <= whi; ++k) {
            const int i0 = (int)fhi - rowoff;
            if ((unsigned)(i0 + 1) < lim1) {
                const V v = __ldg(X2 + fhi);
                const float f = (float)(flo >> 8) * INV_2_24;
#pragma unroll
                for (int h = 0; h < G; ++h) ea[h] += fmaf(f, td(v, h), tv(v, h));
            }
            fx_add(flo, fhi, ilo, ihi);
            rowoff += stride;
        }
#pragma unroll
        for (int h = 0; h < G; ++h) tot[h] = dacc[h] + (double)ea[h];
    }
    // ray h of this lane: item and angle
    auto ray_item = [&](int h) { return MIR ? item0 : item0 + h; };
    auto ray_angle = [&](int h) { return (MIR && h) ? p.A - a : a; };
    double sum[G];
#pragma unroll
    for (int h = 0; h < G; ++h) sum[h] = tot[h];
    if (ks > 1) {
        // combine the parts: the last block of this tile to arrive sums them in order
        if (active) {
#pragma unroll
            for (int h = 0; h < G; ++h) {
                if (h == 0 || pair1) {
                    double* PART = reinterpret_cast<double*>(
                        const_cast<char*>(p.ws) +
                        mct_item_off(ray_item(h), np, p.wsg) + p.off_part);
                    PART[((long long)part * p.A + ray_angle(h)) * p.B + j] = tot[h];
                }
            }
        }
        __shared__ int s_last;
        __syncthreads();
        if (threadIdx.x == 0 && threadIdx.y == 0) {
            int* cnt = reinterpret_cast<int*>(const_cast<char*>(base0) + p.off_cnt) +
                       blockIdx.y * gridDim.x + blockIdx.x;
#if FWD_ACQREL
            // release: the block's PART stores (ordered before by the barrier);
            // acquire: the other parts' stores, for the last block to arrive
            int prev;
            asm volatile("atom.acq_rel.gpu.global.add.s32 %0, [%1], 1;"
                         : "=r"(prev) : "l"(cnt) : "memory");
#else
            __threadfence();
            const int prev = atomicAdd(cnt, 1);
#endif
            s_last = (prev == ks - 1);
            if (s_last) *cnt = 0;  // every part has arrived: re-arm for the next launch
        }
        __syncthreads();
        if (!s_last || !active) return;
#if !FWD_ACQREL
        __threadfence();
#endif
#pragma unroll
        for (int h = 0; h < G; ++h) {
            if (h == 0 || pair1) {
                const double* PART = reinterpret_cast<const double*>(
                    p.ws + mct_item_off(ray_item(h), np, p.wsg) + p.off_part);
                double acc = 0.0;
                for (int q = 0; q < ks; ++q)
                    acc += __ldcg(PART + ((long long)q * p.A + ray_angle(h)) * p.B + j);
                sum[h] = acc;
            }
        }
    } else if (!active) {
        return;
    }
#pragma unroll
    for (int h = 0; h < G; ++h) {
        if (h == 1 && !pair1) break;
        const int item = ray_item(h), ah = ray_angle(h);
        const float proj = (float)sum[h] * ra.step;
        if (MODE == 0) {
            p.out[(long long)item * p.out_item_stride + (long long)ah * p.B + j] = proj;
        } else {
            int slice, gate, iter;
            resolve_item(p.sel, item, slice, gate, iter);
            const long long off = (((long long)slice * p.N + gate) * p.A + ah) * p.B + j;
            const GateParam gp = p.gp[gate];
            const float yv = p.y[off];
            const float dv = __ldg(p.d + off);
            const float yn = (fmaf(gp.sigma, proj, yv) - gp.sigma * dv) * gp.dual_inv;
            p.y[off] = yn;
            // DY element (row, j), float2 slot: gate pairs (a, item & 1); mirror
            // layout (pair row q, h) or (0, self-paired slot)
            int row = ah, slot = h;
            if (MIR) {
                row = sl < nsingle ? 0 : a;
                slot = sl < nsingle ? sl : h;
            }
            float* DY = reinterpret_cast<float*>(const_cast<char*>(tb) +
                                                 (MIR ? p.off_dy : p.off_pdy)) + slot;
            const long long e = 4 * ((long long)row * p.wy + p.pb + j);
            const float dlt = (yn - yv) * ra.step;  // pre-scaled for A^* (see K3)
            DY[e] = dlt;      // element j (bin j of both slots, then bin j + 1)
            DY[e - 2] = dlt;  // element j - 1, bin j
            if (p.proj) p.proj[off] = proj;
            if (!isfinite(yn) && p.status)
                atomicMin(p.status + 1, ((unsigned long long)iter << 20) | (unsigned long long)gate);
        }
    }
}

// ---------------------------------------------------------------------------
// K3: A^* as a deterministic transpose-gather (no atomics).  Pixel (r, c) at
// angle a receives  step * max(0, 1 - |j - jc|*g) * dy[a, j]  from the bins j
// around its detector coordinate jc = (v cos - u sin)/sp + (B-1)/2: exactly the
// Joseph weight of projector.py:161-166 seen from the pixel (the tent identity
// pinned by test_projector.py:78-93).  The sinogram is pre-scaled by the step.
// jc is carried in 32.32 fixed point: an fp64 anchor per (tile, angle) plus
// exact integer steps cos/sp, sin/sp per column / row, so the bin index and the
// interpolation fraction are exact to ~1e-9 bins at any image size.
//
// Mirror pairing: angles theta_a and theta_{A-a} = pi - theta_a give the mirrored
// pixel (u, -v) the same detector coordinate as (u, v).  A thread therefore owns
// ADJ_PPT consecutive rows of a column c in the left half of the image *and* of
// its mirror column cm = cols-1-c; for every angle pair (a, A-a) it computes two
// sets of bin indices / tent weights (those of c and of cm at angle a) and uses
// each twice: jc_a(c) = jc_{A-a}(cm) and jc_a(cm) = jc_{A-a}(c).  Half the
// coordinate and weight arithmetic per pixel-angle; angles 0 and A/2
// (self-paired) are done per pixel.
// The angle pairs may be split over blockIdx.z (partial image slots, summed in
// a fixed order by K4).  fp32 partial sums per chunk, fp64 totals.
// ---------------------------------------------------------------------------
#define ADJ_TW 32      // tile width (left-half columns) = one warp
#ifndef ADJ_PPT
#define ADJ_PPT 4      // consecutive rows per thread
#endif
#ifndef ADJ_WARPS
#define ADJ_WARPS 4
#endif
#define ADJ_THREADS (ADJ_TW * ADJ_WARPS)
#ifndef ADJ_CH
#define ADJ_CH ADJ_THREADS
#endif
#ifndef ADJ_MIN_BLOCKS
#define ADJ_MIN_BLOCKS 7   // single-item A^* (72 registers; fewer, longer angle splits)
#endif
#ifndef ADJ_PATCH
#define ADJ_PATCH 0    // 1: 8 x 4 pixel patches per warp (see adj_kernel)
#endif
#ifndef ADJ_SPLIT_RULE
#define ADJ_SPLIT_RULE 1
#endif
#define INV_2_32 2.3283064365386963e-10f
#ifndef ADJ_TMA
#define ADJ_TMA 1      // K = 0 gate pairs: sinogram segments staged in shared memory by TMA
#endif
#ifndef ADJ_TMA1
#define ADJ_TMA1 1     // the same for single items (mirror layout)
#endif
#define ADJ_STAGED(K, G) ((K) == 0 && ((G) == 2 ? ADJ_TMA : ADJ_TMA1))
#ifndef ADJ_TC
#define ADJ_TC 4       // angle pairs per TMA stage (gate pairs)
#endif
#ifndef ADJ_TC1
#define ADJ_TC1 6      // angle pairs per TMA stage (single items: half the bytes per pair)
#endif
#define ADJ_TCG(G) ((G) == 2 ? ADJ_TC : ADJ_TC1)
#ifndef ADJ_STU2
#define ADJ_STU2 4     // unroll of the staged angle-pair loop (gate pairs: a whole stage)
#endif
#ifndef ADJ_STU1
#define ADJ_STU1 6     // ... (single items: a whole stage)
#endif
#ifndef ADJ_NST
#define ADJ_NST 2      // stage buffers (ring): one computed, NST - 1 in flight
#endif
#ifndef ADJ_STAGE_FULL
#define ADJ_STAGE_FULL 1  // guard-free row loop for full tiles in the staged kernel
#endif
#ifndef ADJ_FFMA2_1
#define ADJ_FFMA2_1 1  // single-item A^*: both angles of an element as one FFMA2
#endif
#ifndef ADJ_SEGW
#define ADJ_SEGW 40    // staged segment capacity (elements); larger plans take the unstaged path
#endif

// 1-D TMA (cp.async.bulk) global -> shared with mbarrier completion (sm_90+).
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, unsigned bytes,
                                            unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// One tent (bin index thi, fraction tlo/2^32) applied to two sinogram rows, the
// row of pixel p at angle a and the row of its mirror at A-a:
//   G = 1 (single item, mirror DY layout): both rows share the float4 element
//     (slot 0: angle a, slot 1: angle A-a) -- one 16-byte load;
//   G = 2 (gate pairs): rows a and a + delta of the pair region, each float4
//     holding the two items' pairs.
// The K = 0 tent on loaded elements: v = the row of angle a at the bin, vm = the
// row of angle A-a (G = 2; G = 1: both angles are the two slots of v).
template <int G>
__device__ __forceinline__ void adj_fma2(const float4& v, const float4& vm, unsigned tlo,
                                         float g32, float omg, float* acc_a, float* acc_b) {
    const float F = (float)tlo;
    const float w0 = __saturatef(fmaf(-F, g32, 1.0f));  // bin floor(jc)
    const float w1 = __saturatef(fmaf(F, g32, omg));    // bin floor(jc) + 1
    if (G == 1) {  // the element's two slots are angles a (-> acc_a) and A-a (-> acc_b)
#if ADJ_FFMA2_1
        float2 a = make_float2(acc_a[0], acc_b[0]);
        a = __ffma2_rn(make_float2(w0, w0), make_float2(v.x, v.y),
                       __ffma2_rn(make_float2(w1, w1), make_float2(v.z, v.w), a));
        acc_a[0] = a.x;
        acc_b[0] = a.y;
#else
        acc_a[0] = fmaf(w0, v.x, fmaf(w1, v.z, acc_a[0]));
        acc_b[0] = fmaf(w0, v.y, fmaf(w1, v.w, acc_b[0]));
#endif
    } else {
        // both items at once: per lane the same fmaf(w0, y_j, fmaf(w1, y_j+1, acc))
        float2 a = make_float2(acc_a[0], acc_a[1]), b = make_float2(acc_b[0], acc_b[1]);
        a = __ffma2_rn(make_float2(w0, w0), make_float2(v.x, v.y),
                       __ffma2_rn(make_float2(w1, w1), make_float2(v.z, v.w), a));
        b = __ffma2_rn(make_float2(w0, w0), make_float2(vm.x, vm.y),
                       __ffma2_rn(make_float2(w1, w1), make_float2(vm.z, vm.w), b));
        acc_a[0] = a.x; acc_a[1] = a.y;
        acc_b[0] = b.x; acc_b[1] = b.y;
    }
}

template <int K, int G>
__device__ __forceinline__ void adj_tap2(const float4* __restrict__ DY2, unsigned tlo, int thi,
                                         int delta, float g32, float omg, float* acc_a,
                                         float* acc_b, int kr) {
    const float F = (float)tlo;
    if (K == 0) {
        const float4 v = __ldg(DY2 + (unsigned)thi);
        const float4 vm = G == 1 ? v : __ldg(DY2 + (unsigned)(thi + delta));
        adj_fma2<G>(v, vm, tlo, g32, omg, acc_a, acc_b);
    } else {
        const float d = F * INV_2_32;
        const float g = g32 * 4294967296.0f;
#pragma unroll
        for (int mm = -(K >= 0 ? K : kr); mm <= (K >= 0 ? K : kr); mm += 2) {
            const float wa = __saturatef(fmaf(-fabsf((float)mm - d), g, 1.0f));
            const float wb = __saturatef(fmaf(-fabsf((float)(mm + 1) - d), g, 1.0f));
            if (G == 1) {
                const float4 v = __ldg(DY2 + (thi + mm));
                acc_a[0] = fmaf(wa, v.x, fmaf(wb, v.z, acc_a[0]));
                acc_b[0] = fmaf(wa, v.y, fmaf(wb, v.w, acc_b[0]));
            } else {
                const float4 v = __ldg(DY2 + (thi + mm));
                const float4 vm = __ldg(DY2 + (thi + delta + mm));
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    acc_a[h] = fmaf(wa, dlo(v, h), fmaf(wb, dhi(v, h), acc_a[h]));
                    acc_b[h] = fmaf(wa, dlo(vm, h), fmaf(wb, dhi(vm, h), acc_b[h]));
                }
            }
        }
    }
}

// One tent on one sinogram row: G = 1: float2 slot `slot` of the element; G = 2:
// both items' pairs.
template <int K, int G>
__device__ __forceinline__ void adj_tap1(const float4* __restrict__ DY2, unsigned tlo, int thi,
                                         int slot, float g32, float omg, float* acc, int kr) {
    const float F = (float)tlo;
    if (K == 0) {
        const float4 v = __ldg(DY2 + (unsigned)thi);
        const float w0 = __saturatef(fmaf(-F, g32, 1.0f));
        const float w1 = __saturatef(fmaf(F, g32, omg));
        if (G == 1)
            acc[0] = fmaf(w0, dlo(v, slot), fmaf(w1, dhi(v, slot), acc[0]));
        else
#pragma unroll
            for (int h = 0; h < G; ++h) acc[h] = fmaf(w0, dlo(v, h), fmaf(w1, dhi(v, h), acc[h]));
    } else {
        const float d = F * INV_2_32;
        const float g = g32 * 4294967296.0f;
#pragma unroll
        for (int mm = -(K >= 0 ? K : kr); mm <= (K >= 0 ? K : kr); mm += 2) {
            const float4 v = __ldg(DY2 + (thi + mm));
            const float wa = __saturatef(fmaf(-fabsf((float)mm - d), g, 1.0f));
            const float wb = __saturatef(fmaf(-fabsf((float)(mm + 1) - d), g, 1.0f));
            if (G == 1)
                acc[0] = fmaf(wa, dlo(v, slot), fmaf(wb, dhi(v, slot), acc[0]));
            else
#pragma unroll
                for (int h = 0; h < G; ++h) acc[h] = fmaf(wa, dlo(v, h), fmaf(wb, dhi(v, h), acc[h]));
        }
    }
}

#ifndef ADJ_PPT2
#define ADJ_PPT2 4     // rows per thread of the gate-pair kernel (= ADJ_PPT: same tiles, so a
                       // batch and a single item agree bitwise)
#endif
#ifndef ADJ_MIN_BLOCKS2
#define ADJ_MIN_BLOCKS2 5  // staged (TMA) gate-pair kernel: shared memory allows 5 blocks/SM anyway
#endif
template <int G> struct AdjShape;
#ifndef ADJ_TU2
#define ADJ_TU2 4      // unroll of the angle-pair loop (gate-pair kernel)
#endif
template <> struct AdjShape<1> { static constexpr int PPT = ADJ_PPT, MINB = ADJ_MIN_BLOCKS, TU = 2; };
template <> struct AdjShape<2> {
    static constexpr int PPT = ADJ_PPT2, MINB = ADJ_MIN_BLOCKS2, TU = ADJ_TU2;
};

// G = 2: a thread owns its pixels in the two items of a gate pair; the bins and
// tent weights are computed once and applied to both items' rows (one 16-byte
// load per pixel-angle).  Per-item arithmetic identical to G = 1.
template <int K, int G>
__global__ void __launch_bounds__(ADJ_THREADS, AdjShape<G>::MINB) adj_kernel(AdjArgs p) {
    using V = float4;
    constexpr int PPT = AdjShape<G>::PPT;
    constexpr int TH = PPT * ADJ_WARPS;
    __shared__ longlong2 s_t[ADJ_CH];  // anchor (with sinogram row base of a), cos/sp
    __shared__ int4 s_u[ADJ_CH];       // sin/sp (lo, hi), g*2^-32, 1 - g
    __shared__ int s_d[ADJ_CH];        // sinogram offset of row A-a relative to row a
    __shared__ double s_tot[G][2 * PPT][ADJ_THREADS];
    // TMA staging (K = 0): per angle pair the block's sinogram segments -- the bins
    // under the tile's primary columns and under its mirror columns, in row a (and
    // row A-a, G = 2) -- first element and length; two stage buffers of ADJ_TCG(G) pairs
    __shared__ int4 s_lo[ADJ_STAGED(K, G) ? ADJ_CH : 1];
    __shared__ unsigned long long s_full[ADJ_NST];
    extern __shared__ float4 s_stage[];
    const int group = blockIdx.z / p.asplit;
    const int split = blockIdx.z - group * p.asplit;
    const int A = p.A;
    const int npairs = (A - 1) / 2;  // pairs (a, A-a), a = 1 .. npairs
    // angle pairs [q_lo, q_hi) of this item (a half item: one half), split evenly
    int q_lo = 1, q_hi = npairs + 1;
    bool singles = true;
    const int part = (G == 1 && p.last_part && p.item0 + group == p.n_items - 1) ? p.last_part : 0;
    if (part == 1) q_hi = mct_half_q(A);
    if (part == 2) { q_lo = mct_half_q(A); singles = false; }
    const int q_beg = q_lo + (int)((long long)(q_hi - q_lo) * split / p.asplit);
    const int q_end = q_lo + (int)((long long)(q_hi - q_lo) * (split + 1) / p.asplit);
    const int tid = threadIdx.y * ADJ_TW + threadIdx.x;
    const int ncl = (p.cols + 1) >> 1;                      // left-half columns (incl. centre)
    const int r0 = blockIdx.y * TH, c0 = blockIdx.x * ADJ_TW;
    // lane -> pixels: ADJ_PATCH = 0: a warp is 32 columns, a thread PPT consecutive
    // rows; ADJ_PATCH = 1: a warp is 8 columns x 4 rows, a thread rows rb, rb+4, ...
    // (the same 32 x TH tile and per-pixel arithmetic either way)
    constexpr int RSTEP = ADJ_PATCH ? 4 : 1;
    const int lcol = ADJ_PATCH ? (int)threadIdx.y * 8 + ((int)threadIdx.x & 7) : (int)threadIdx.x;
    const int rbase = ADJ_PATCH ? ((int)threadIdx.x >> 3) : (int)threadIdx.y * PPT;
    const int c = c0 + lcol;                                 // primary column
    const int cm = p.cols - 1 - c;                           // mirror column
    const int rt = r0 + rbase;
    const int nrows = rt < p.rows ? min(PPT, (p.rows - rt + RSTEP - 1) / RSTEP) : 0;
    const int txc = min(lcol, ncl - 1 - c0);                 // clamp lanes past the half
    const int cmc = p.cols - 1 - (c0 + txc);                 // (clamped) mirror column
    const double u0 = (double)r0 - 0.5 * (double)(p.rows - 1);
    const double v0 = (double)c0 - 0.5 * (double)(p.cols - 1);
    const int item0 = p.item0 + G * group;  // G = 2: item0 is even
    const int np = mct_pair_items(p.n_items, p.last_part);  // paired items of the call
    const char* tb = G == 1 ? p.ws + mct_item_off(item0, np, p.wsg)
                            : p.ws + mct_pair_off(item0 >> 1, p.wsg);
    const V* __restrict__ DY2 = reinterpret_cast<const V*>(tb + (G == 1 ? p.off_dy : p.off_pdy));
    const long long row_off = (long long)rbase;

#pragma unroll
    for (int h = 0; h < G; ++h)
#pragma unroll
        for (int m = 0; m < 2 * PPT; ++m) s_tot[h][m][tid] = 0.0;
    constexpr bool STAGED = ADJ_STAGED(K, G);
    // stage ring: full[b] completes when the bytes of the stage in buffer b landed
    // (TMA transaction count); `uses` counts the stages run through the ring so far
    // (buffer = use % NST, parity = (use / NST) & 1)
    unsigned uses = 0;
    if (STAGED && tid == 0) {
        for (int b = 0; b < ADJ_NST; ++b) mbar_init(&s_full[b], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }

    // ---- self-paired angles 0 and A/2 (split 0 only), pixel by pixel
    if (split == 0 && singles) {
        const int nsingle = (A % 2 == 0 && A >= 2) ? 2 : 1;
        for (int si = 0; si < nsingle; ++si) {
            const int a = si == 0 ? 0 : A / 2;
            const int arow = G == 1 ? 0 : a;  // mirror layout: row 0, slot si
            const AdjAngle aa = p.ang[a];
            const double jcA = v0 * aa.cs - u0 * aa.sn + p.jmid;
            const long long TA =
                __double2ll_rn(jcA * FX_ONE) + ((long long)(arow * p.wy + p.pb) << 32);
            const float g32 = aa.g * INV_2_32, omg = 1.0f - aa.g;
            long long T = TA + (long long)txc * aa.csx - row_off * aa.snx;
            long long Tm = TA + (long long)(cmc - c0) * aa.csx - row_off * aa.snx;
            for (int m = 0; m < nrows; ++m) {
                float acc[G], accm[G];
#pragma unroll
                for (int h = 0; h < G; ++h) acc[h] = accm[h] = 0.0f;
                adj_tap1<K, G>(DY2, (unsigned)T, (int)(T >> 32), si, g32, omg, acc, p.kfoot);
                adj_tap1<K, G>(DY2, (unsigned)Tm, (int)(Tm >> 32), si, g32, omg, accm, p.kfoot);
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    s_tot[h][m][tid] += (double)acc[h];
                    s_tot[h][PPT + m][tid] += (double)accm[h];
                }
                T -= RSTEP * aa.snx;
                Tm -= RSTEP * aa.snx;
            }
        }
    }

    // ---- mirror pairs (a, A-a)
    for (int q0 = q_beg; q0 < q_end; q0 += ADJ_CH) {
        const int cnt = min(ADJ_CH, q_end - q0);
        __syncthreads();
        if (tid < cnt) {
            const int a = q0 + tid;
            const AdjAngle aa = p.ang[a];
            const double jcA = v0 * aa.cs - u0 * aa.sn + p.jmid;
            const long long TA =
                __double2ll_rn(jcA * FX_ONE) + ((long long)(a * p.wy + p.pb) << 32);
            s_t[tid] = make_longlong2(TA, aa.csx);
            s_u[tid] = make_int4((int)(unsigned)aa.snx, (int)(aa.snx >> 32),
                                 __float_as_int(aa.g * INV_2_32), __float_as_int(1.0f - aa.g));
            s_d[tid] = (A - 2 * a) * p.wy;
            if (STAGED) {
                // element range of the tile at this angle: T(x, r) = TA + x csx - r snx is
                // linear, so its integer part is extremal at the corners (x in [0, X1]
                // primary / mirrored, r in [0, R1])
                const int X1 = min(ADJ_TW - 1, ncl - 1 - c0);
                const int R1 = min(TH, p.rows - r0) - 1;
                const long long xm0 = (long long)(p.cols - 1 - 2 * c0);
                auto rng = [&](long long x0, long long x1, int& lo, int& n) {
                    const long long e[4] = {TA + x0 * aa.csx, TA + x1 * aa.csx,
                                            TA + x0 * aa.csx - R1 * aa.snx,
                                            TA + x1 * aa.csx - R1 * aa.snx};
                    int l = (int)(e[0] >> 32), h = l;
#pragma unroll
                    for (int k = 1; k < 4; ++k) {
                        l = min(l, (int)(e[k] >> 32));
                        h = max(h, (int)(e[k] >> 32));
                    }
                    lo = l;
                    n = min(h - l + 1, ADJ_SEGW);  // the host's bound (launch_adj_g) holds
                };
                int lc, nc, lm, nm;
                rng(0, X1, lc, nc);
                rng(xm0 - X1, xm0, lm, nm);
                s_lo[tid] = make_int4(lc, nc, lm, nm);
            }
        }
        __syncthreads();
        if constexpr (STAGED) {
            // stage ring of NST buffers: while the block computes stage s, stages
            // s + 1 .. s + NST - 1 are in flight; thread 0 refills the buffer of stage s
            // with stage s + NST once every warp left it (__syncthreads, then an
            // async-proxy fence before the TMA writes)
            constexpr int NSEG = G == 2 ? 4 : 2;
            constexpr int segw = ADJ_SEGW;
            const int nst = (cnt + ADJ_TCG(G) - 1) / ADJ_TCG(G);
            auto issue = [&](int st) {  // stage st of this chunk (ring use uses + st)
                const unsigned u = uses + (unsigned)st;
                const int b = (int)(u % ADJ_NST);
                fence_proxy_async();
                const int t0 = st * ADJ_TCG(G), t1 = min(cnt, t0 + ADJ_TCG(G));
                unsigned bytes = 0;
                for (int t = t0; t < t1; ++t) {
                    const int4 L = s_lo[t];
                    bytes += (unsigned)(L.y + L.w) * 16u * (G == 2 ? 2u : 1u);
                }
                mbar_expect_tx(&s_full[b], bytes);
                for (int t = t0; t < t1; ++t) {
                    const int4 L = s_lo[t];
                    float4* dst = s_stage + (size_t)(b * ADJ_TCG(G) + (t - t0)) * NSEG * segw;
                    tma_load_1d(dst, DY2 + L.x, L.y * 16u, &s_full[b]);
                    tma_load_1d(dst + segw, DY2 + L.z, L.w * 16u, &s_full[b]);
                    if (G == 2) {
                        const int dl = s_d[t];
                        tma_load_1d(dst + 2 * segw, DY2 + L.x + dl, L.y * 16u, &s_full[b]);
                        tma_load_1d(dst + 3 * segw, DY2 + L.z + dl, L.w * 16u, &s_full[b]);
                    }
                }
            };
            if (tid == 0)
                for (int st = 0; st < min(nst, ADJ_NST); ++st) issue(st);
            float acc[PPT][G], accm[PPT][G];
#pragma unroll
            for (int m = 0; m < PPT; ++m)
#pragma unroll
                for (int h = 0; h < G; ++h) acc[m][h] = accm[m][h] = 0.0f;
            for (int st = 0; st < nst; ++st) {
                const unsigned u = uses + (unsigned)st;
                const int b = (int)(u % ADJ_NST);
                mbar_wait(&s_full[b], (u / ADJ_NST) & 1u);
                const int t0 = st * ADJ_TCG(G), t1 = min(cnt, t0 + ADJ_TCG(G));
                // FULL: all PPT rows in the image (warp-uniform), no per-row guard
                auto stage = [&](auto full) {
                    constexpr bool FULL = decltype(full)::value;
                    constexpr int SU = G == 2 ? ADJ_STU2 : ADJ_STU1;
#pragma unroll (SU)
                    for (int t = t0; t < t1; ++t) {
                        const longlong2 T2 = s_t[t];
                        const int4 U = s_u[t];
                        const int4 L = s_lo[t];
                        const long long snx = ((long long)U.y << 32) | (unsigned)U.x;
                        const long long snr = RSTEP * snx;
                        const float g32 = __int_as_float(U.z), omg = __int_as_float(U.w);
                        const long long T = T2.x + (long long)txc * T2.y - row_off * snx;
                        const long long Tm = T2.x + (long long)(cmc - c0) * T2.y - row_off * snx;
                        unsigned tlo = (unsigned)T, thi = (unsigned)(T >> 32);
                        unsigned mlo = (unsigned)Tm, mhi = (unsigned)(Tm >> 32);
                        // segments: [primary, row a | mirror, row a | primary, row A-a |
                        // mirror, row A-a], each segw elements
                        const float4* sb = s_stage + (size_t)(b * ADJ_TCG(G) + (t - t0)) * NSEG * segw;
#pragma unroll
                        for (int m = 0; m < PPT; ++m) {
                            if (FULL || m < nrows) {
                                const int ic = (int)thi - L.x, im = segw + (int)mhi - L.z;
                                const float4 v = sb[ic];
                                const float4 vm = G == 2 ? sb[2 * segw + ic] : v;
                                adj_fma2<G>(v, vm, tlo, g32, omg, acc[m], accm[m]);
                                const float4 w = sb[im];
                                const float4 wm = G == 2 ? sb[2 * segw + im] : w;
                                adj_fma2<G>(w, wm, mlo, g32, omg, accm[m], acc[m]);
                            }
                            fx_sub(tlo, thi, (unsigned)snr, (unsigned)(snr >> 32));
                            fx_sub(mlo, mhi, (unsigned)snr, (unsigned)(snr >> 32));
                        }
                    }
                };
                if (ADJ_STAGE_FULL && nrows == PPT)
                    stage(std::true_type{});
                else if (nrows > 0)
                    stage(std::false_type{});
                __syncthreads();  // every warp is done with buffer b
                if (tid == 0 && st + ADJ_NST < nst) issue(st + ADJ_NST);
            }
            uses += (unsigned)nst;
#pragma unroll
            for (int m = 0; m < PPT; ++m)
#pragma unroll
                for (int h = 0; h < G; ++h) {
                    s_tot[h][m][tid] += (double)acc[m][h];
                    s_tot[h][PPT + m][tid] += (double)accm[m][h];
                }
            continue;
        }
        if (nrows <= 0) continue;
        float acc[PPT][G], accm[PPT][G];
#pragma unroll
        for (int m = 0; m < PPT; ++m)
#pragma unroll
            for (int h = 0; h < G; ++h) acc[m][h] = accm[m][h] = 0.0f;
#pragma unroll (AdjShape<G>::TU)
        for (int t = 0; t < cnt; ++t) {
            const longlong2 T2 = s_t[t];
            const int4 U = s_u[t];
            const int delta = s_d[t];
            const long long snx = ((long long)U.y << 32) | (unsigned)U.x;
            const long long snr = RSTEP * snx;  // per-row step of this thread's rows
            const float g32 = __int_as_float(U.z), omg = __int_as_float(U.w);
            // c at angle a == cm at angle A-a ; cm at angle a == c at angle A-a
            const long long T = T2.x + (long long)txc * T2.y - row_off * snx;
            const long long Tm = T2.x + (long long)(cmc - c0) * T2.y - row_off * snx;
            unsigned tlo = (unsigned)T, thi = (unsigned)(T >> 32);
            unsigned mlo = (unsigned)Tm, mhi = (unsigned)(Tm >> 32);
#pragma unroll
            for (int m = 0; m < PPT; ++m) {
                if (m < nrows) {
                    adj_tap2<K, G>(DY2, tlo, (int)thi, delta, g32, omg, acc[m], accm[m], p.kfoot);
                    adj_tap2<K, G>(DY2, mlo, (int)mhi, delta, g32, omg, accm[m], acc[m], p.kfoot);
                }
                fx_sub(tlo, thi, (unsigned)snr, (unsigned)(snr >> 32));
                fx_sub(mlo, mhi, (unsigned)snr, (unsigned)(snr >> 32));
            }
        }
#pragma unroll
        for (int m = 0; m < PPT; ++m)
#pragma unroll
            for (int h = 0; h < G; ++h) {
                s_tot[h][m][tid] += (double)acc[m][h];
                s_tot[h][PPT + m][tid] += (double)accm[m][h];
            }
    }
    if (c >= ncl) return;
#pragma unroll
    for (int h = 0; h < G; ++h) {
        float* IMG = reinterpret_cast<float*>(
            const_cast<char*>(p.ws) +
            mct_img_off(item0 + h, np, p.asplit, p.img_slot_bytes, p.wsg) + p.off_img +
            (size_t)split * p.img_slot_bytes);
        for (int m = 0; m < nrows; ++m) {
            const long long row = (long long)(rt + RSTEP * m) * p.cols;
            if (cm == c) {  // centre column of an odd width: the primary role already
                IMG[row + c] = (float)s_tot[h][m][tid];  // holds every angle (mirror = duplicate)
            } else {
                IMG[row + c] = (float)s_tot[h][m][tid];
                IMG[row + cm] = (float)s_tot[h][PPT + m][tid];
            }
        }
    }
}

}  // namespace

#ifndef PACK_SMALL_ITEMS
#define PACK_SMALL_ITEMS 1
#endif
#ifndef PACK16_MINB
#define PACK16_MINB 4
#endif
#ifndef PACK32_MINB
#define PACK32_MINB 6
#endif
#ifndef PACK32_THREADS
#define PACK32_THREADS 256
#endif
cudaError_t launch_pack(const PackArgs& a_in, int items, cudaStream_t st) {
    PackArgs a = a_in;
    a.pair_items = mct_pair_items(items, a.sel.last_part);
    const int n = a.sel.count ? a.sel.count : items - a.sel.first;  // this chunk
    if (items <= PACK_SMALL_ITEMS) {  // few gates: small tiles, one halo element per thread
        dim3 grid((a.cols + 15) / 16, (a.rows + 15) / 16, n);
        pack_kernel<16, 320, PACK16_MINB><<<grid, 320, 0, st>>>(a);
    } else {
        dim3 grid((a.cols + 31) / 32, (a.rows + 31) / 32, n);
        pack_kernel<32, PACK32_THREADS, PACK32_MINB><<<grid, PACK32_THREADS, 0, st>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_pad_sino(const float* sino, const mct_ray_plan* rp, char* ws,
                            const WsGeom& wsg, int items, int first, int count, cudaStream_t st) {
    dim3 block(256), grid((rp->B + 255) / 256, rp->A, count ? count : items - first);
    pad_sino_kernel<<<grid, block, 0, st>>>(sino, rp->d_adj, ws, wsg,
                                            rp->off_dy, rp->off_pdy, rp->A, rp->B, rp->wy, rp->pb,
                                            mct_pair_items(items), first);
    return cudaGetLastError();
}

// K2 ray split of single-item launches (a plan constant, see MCT_KSPLIT_MIN):
// enough parts to fill about one wave of resident blocks.
int choose_ksplit(int A, int B, int n) {
    static int slots = 0;  // resident fwd blocks per GPU (queried once)
    if (slots == 0) {
        int dev = 0, sms = 148, per_sm = FWD_MIN_BLOCKS2;
        if (cudaGetDevice(&dev) == cudaSuccess)
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fwd_kernel<1, 1, 1>,
                                                          32 * FWD_ANGLES, 0) != cudaSuccess ||
            per_sm < 1)
            per_sm = FWD_MIN_BLOCKS2;
        slots = sms * per_sm;
    }
    const long long blocks =
        (long long)mct_fwd_btiles(B) * mct_fwd_groups(mir_slots(A));
    long long k = (slots + blocks - 1) / blocks;
    const long long by_len = n / 16 > 1 ? n / 16 : 1;  // >= 16 samples per part
    k = k < by_len ? k : by_len;
    k = k > MCT_KSPLIT_MAX ? MCT_KSPLIT_MAX : k;
    k = k < MCT_KSPLIT_MIN ? MCT_KSPLIT_MIN : k;
    return (int)k;
}

// K2 lives on its L1 hit rate (the four angles of a block re-read the same lines
// while their warps drift apart by a few rows): ask for the smallest shared-memory
// carve-out that still fits the resident blocks, i.e. the largest L1.
static void fwd_prefer_l1() {
    static bool done = false;
    if (done) return;
    done = true;
#ifdef FWD_CARVEOUT_PCT
    const int pct = FWD_CARVEOUT_PCT;
#else
    const int pct = 7;  // >= 8 blocks x 1 KB reserved of 228 KB -> the 16 KB config
#endif
    cudaFuncSetAttribute(fwd_kernel<0, 0, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(fwd_kernel<1, 0, 0>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(fwd_kernel<0, 0, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(fwd_kernel<1, 0, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(fwd_kernel<0, 1, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
    cudaFuncSetAttribute(fwd_kernel<1, 1, 1>, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

// A launch with gate pairs and an odd last item runs the two (independent) grids
// concurrently: the odd item's on a side stream forked from and joined back to
// the caller's stream with events (graph-capture safe).  One side stream per
// (device, caller stream), so concurrent callers on different streams never share
// one; events are per call.
#ifndef MCT_SIDE_STREAM
#define MCT_SIDE_STREAM 1
#endif
static cudaStream_t side_stream_for(cudaStream_t st) {
    static std::mutex mu;
    static std::map<std::pair<int, cudaStream_t>, cudaStream_t> streams;
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(dev, st);
    auto it = streams.find(key);
    if (it != streams.end()) return it->second;
    // never create a stream while the caller's stream is being captured (a global-mode
    // capture would be invalidated): such a first call runs serially instead
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cap) != cudaSuccess || cap != cudaStreamCaptureStatusNone)
        return nullptr;
    cudaStream_t side = nullptr;
    if (cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    streams[key] = side;
    return side;
}

template <class MainF, class SideF>
static cudaError_t fork_join(cudaStream_t st, MainF main_launch, SideF side_launch) {
    cudaStream_t side = MCT_SIDE_STREAM ? side_stream_for(st) : nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
    if (side == nullptr || cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&join, cudaEventDisableTiming) != cudaSuccess) {
        if (fork) cudaEventDestroy(fork);
        main_launch(st);  // serial fallback on the caller's stream
        side_launch(st);
        return cudaGetLastError();
    }
    cudaError_t e = cudaEventRecord(fork, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(side, fork, 0);
    if (e == cudaSuccess) {
        side_launch(side);
        main_launch(st);
        e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaEventRecord(join, side);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, join, 0);
    cudaEventDestroy(fork);
    cudaEventDestroy(join);
    return e;
}

cudaError_t launch_fwd(const FwdArgs& a_in, int mode, int items, cudaStream_t st) {
    fwd_prefer_l1();
    const dim3 block(32, FWD_ANGLES), block_p(32, MCT_FWD_ANGLES_P);
    const unsigned ntile = mct_fwd_btiles(a_in.B);
    const int np = mct_pair_items(items, a_in.sel.last_part);
    // this chunk's paired items [p_lo, p_hi); the unpaired tail runs with the last chunk
    const int first = a_in.sel.first, end = a_in.sel.count ? first + a_in.sel.count : items;
    const int p_lo = first < np ? first : np, p_hi = end < np ? end : np;
    const bool tail = end == items && items > np;
    // gate pairs (bins fastest: L2 locality across pairs)
    auto pairs = [&](cudaStream_t s) {
        FwdArgs a = a_in;
        a.item0 = p_lo;
        a.n_items = items;
        a.ksplit = 1;  // >= 2 items fill the GPU without splitting rays (no partials)
        dim3 grid(ntile, mct_fwd_groups(a.A, MCT_FWD_ANGLES_P), ((p_hi - p_lo) / 2) * a.ksplit);
        if (mode == 0)
            fwd_kernel<0, 0, 0><<<grid, block_p, 0, s>>>(a);
        else
            fwd_kernel<1, 0, 0><<<grid, block_p, 0, s>>>(a);
    };
    // single items (mirror-angle walks; an odd last item after the pairs).  One
    // single-gate item: longest-rays-first dispatch order (LPT) shrinks the last
    // partial wave; with several items the item-major order keeps better L2
    // locality.  Same arithmetic either way (block order only).
    auto singles = [&](cudaStream_t s) {
        FwdArgs a = a_in;
        a.item0 = np;
        a.n_items = items;
        const int rest = items - np;
        const unsigned ngroup = mct_fwd_groups(mir_slots(a.A));
        const bool lpt = (a.ksplit > 1 ? FWD_LPT_SPLIT : FWD_LPT_NOSPLIT) && rest == 1;
        dim3 grid(lpt ? ngroup : ntile, lpt ? ntile : ngroup, rest * a.ksplit);
        if (lpt) {
            if (mode == 0)
                fwd_kernel<0, 1, 1><<<grid, block, 0, s>>>(a);
            else
                fwd_kernel<1, 1, 1><<<grid, block, 0, s>>>(a);
        } else if (mode == 0) {
            fwd_kernel<0, 0, 1><<<grid, block, 0, s>>>(a);
        } else {
            fwd_kernel<1, 0, 1><<<grid, block, 0, s>>>(a);
        }
    };
    if (p_hi > p_lo && tail) return fork_join(st, pairs, singles);
    if (p_hi > p_lo) pairs(st);
    if (tail) singles(st);
    return cudaGetLastError();
}

// Angle split of A^* for launches with fewer tiles than resident blocks
// (single-gate SPDHG): chosen by a wave-quantisation cost model (below); every
// split keeps >= MCT_ASPLIT_MIN_PAIRS angle pairs.
static inline int adj_tiles_x(int cols) { return ((cols + 1) / 2 + ADJ_TW - 1) / ADJ_TW; }

static int adj_split_for(long long tiles, long long slots, const mct_ray_plan* rp) {
    // >= MCT_ASPLIT_MIN_PAIRS angle pairs per split
    const long long by_angles =
        rp->A / (2 * MCT_ASPLIT_MIN_PAIRS) > 0 ? rp->A / (2 * MCT_ASPLIT_MIN_PAIRS) : 1;
    const long long smax = by_angles < MCT_MAX_ASPLIT ? by_angles : MCT_MAX_ASPLIT;
#if ADJ_SPLIT_RULE == 0
    long long s = tiles >= slots ? 1 : slots / tiles;  // fill at most one wave
    s = s < 1 ? 1 : s;
    return (int)(s < smax ? s : smax);
#else
    // launches of a wave or more already balance dynamically: no split (every
    // extra slot costs K4 one more partial-image read per gather)
    if (tiles >= slots) return 1;
    // fewer tiles than resident blocks: the split minimising (waves, rounded up)
    // x (angle pairs per block), e.g. C3 single gate: 11 splits in 1.9 waves
    // beat 5 splits in one 86 %-full wave
    const long long P = rp->A > 2 ? (rp->A - 1) / 2 : 1;
    long long best = 1, best_cost = -1;
    for (long long s = 1; s <= smax; ++s) {
        const long long waves = (tiles * s + slots - 1) / slots;
        const long long cost = waves * ((P + s - 1) / s);
        if (best_cost < 0 || cost * 100 < best_cost * 97) {  // >= 3 % better to split more
            best = s;
            best_cost = cost;
        }
    }
    return (int)best;
#endif
}

// Elements of one staged sinogram segment (see adj_kernel): the bins a tile's
// primary (or mirror) columns and rows reach at one angle, bounded over the plan's
// angles from the same fixed-point steps the kernel walks (+ 2 for the floors).
int adj_segw(const mct_ray_plan* rp) {
    constexpr int TH = ADJ_PPT * ADJ_WARPS;
    static_assert(ADJ_PPT == ADJ_PPT2, "one tile height for both A^* kernels");
    double w = 0.0;
    for (size_t a = 0; a < rp->h_acs.size(); ++a)
        w = std::max(w, (ADJ_TW - 1) * rp->h_acs[a] + (TH - 1) * rp->h_asn[a]);
    return (int)ceil(w) + 3;
}

// Dynamic shared memory of the staged K = 0 kernel; 0 when the plan's segments do
// not fit ADJ_SEGW (launch_adj_g then runs the unstaged runtime-footprint kernel).
size_t adj_stage_bytes(int G, int segw) {
    return ADJ_STAGED(0, G) && segw <= ADJ_SEGW
               ? (size_t)ADJ_NST * ADJ_TCG(G) * (G == 2 ? 4 : 2) * ADJ_SEGW * sizeof(float4)
               : 0;
}

static void adj_configure(int G, size_t dyn) {
    static std::mutex mu;
    static size_t done[3] = {0, 0, 0};
    std::lock_guard<std::mutex> lock(mu);
    if (done[G] >= dyn + 1) return;
    done[G] = dyn + 1;
    const void* f = G == 1 ? (const void*)adj_kernel<0, 1> : (const void*)adj_kernel<0, 2>;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
    if (ADJ_STAGED(0, G)) cudaFuncSetAttribute(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

static long long adj_slots(int G, size_t dyn) {
    // resident adj blocks per GPU, per (G, dynamic shared memory) (queried once)
    static std::mutex mu;
    static std::map<std::pair<int, size_t>, long long> slots;
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_pair(G, dyn);
    auto it = slots.find(key);
    if (it != slots.end()) return it->second;
    int dev = 0, sms = 148, per_sm = 8;
    if (cudaGetDevice(&dev) == cudaSuccess)
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const cudaError_t e =
        G == 1 ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adj_kernel<0, 1>, ADJ_THREADS, dyn)
               : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, adj_kernel<0, 2>, ADJ_THREADS, dyn);
    if (e != cudaSuccess || per_sm < 1) per_sm = 8;
    return slots[key] = (long long)sms * per_sm;
}
static long long adj_slots(int G, const mct_ray_plan* rp) {
    const size_t dyn = rp->kfoot == 0 ? adj_stage_bytes(G, rp->adj_segw) : 0;
    adj_configure(G, dyn);
    return adj_slots(G, dyn);
}

// A^* partial-image slots a plan's items hold: the single-item split, and at
// least MCT_MIN_ASLOTS so multi-gate launches with an odd last item (gate-sharded
// ranks) can split too.
#ifndef MCT_MIN_ASLOTS
#define MCT_MIN_ASLOTS 4
#endif
int adj_plan_slots(const mct_ray_plan* rp) {
    constexpr int TH1 = AdjShape<1>::PPT * ADJ_WARPS;
    const long long tiles1 = (long long)adj_tiles_x(rp->cols) * ((rp->rows + TH1 - 1) / TH1);
    const int s1 = adj_split_for(tiles1, adj_slots(1, rp), rp);
    const long long by_angles =
        rp->A / (2 * MCT_ASPLIT_MIN_PAIRS) > 0 ? rp->A / (2 * MCT_ASPLIT_MIN_PAIRS) : 1;
    const int lo = (int)(by_angles < MCT_MIN_ASLOTS ? by_angles : MCT_MIN_ASLOTS);
    return s1 > lo ? s1 : lo;
}

int choose_asplit(const mct_ray_plan* rp, int items, int last_part) {
    const int n = items > 0 ? items : 1;
    constexpr int TH1 = AdjShape<1>::PPT * ADJ_WARPS, TH2 = AdjShape<2>::PPT * ADJ_WARPS;
    const long long tiles1 = (long long)adj_tiles_x(rp->cols) * ((rp->rows + TH1 - 1) / TH1);
    const int s1 = adj_split_for(tiles1, adj_slots(1, rp), rp);  // single item: the plan's slot count
    const int np = mct_pair_items(n, last_part);
    if (np == 0) return n == 1 ? s1 : adj_split_for(tiles1 * n, adj_slots(1, rp), rp);
    // pair launch + (odd last item) single launch run one after the other: the split
    // minimising the sum of their (waves, rounded up) x (angle pairs per block),
    // e.g. C3 with 3 local gates (one rank of 8): 3 splits, each launch one full
    // wave, instead of two 0.3-wave launches; 10 local gates: 2.9 instead of 1.4
    // waves.  At most the plan's slot count.
    const long long tiles2 = (long long)adj_tiles_x(rp->cols) * ((rp->rows + TH2 - 1) / TH2);
    const long long b2 = tiles2 * (np / 2), b1 = tiles1 * (n - np);
    const long long sl2 = adj_slots(2, rp), sl1 = adj_slots(1, rp);
    const long long P = rp->A > 2 ? (rp->A - 1) / 2 : 1;
    const long long by_angles =
        rp->A / (2 * MCT_ASPLIT_MIN_PAIRS) > 0 ? rp->A / (2 * MCT_ASPLIT_MIN_PAIRS) : 1;
    long long smax = by_angles < MCT_MAX_ASPLIT ? by_angles : MCT_MAX_ASPLIT;
    const long long cap = adj_plan_slots(rp);
    smax = smax < cap ? smax : cap;
#ifdef MCT_PAIR_ASPLIT_MAX
    smax = smax < MCT_PAIR_ASPLIT_MAX ? smax : MCT_PAIR_ASPLIT_MAX;
#endif
    long long best = 1, best_cost = -1;
    for (long long sp = 1; sp <= smax; ++sp) {
        const long long waves = (b2 * sp + sl2 - 1) / sl2 + (b1 * sp + sl1 - 1) / sl1;
        const long long cost = waves * ((P + sp - 1) / sp);
        if (best_cost < 0 || cost * 100 < best_cost * 97) {  // >= 3 % better to split more
            best = sp;
            best_cost = cost;
        }
    }
    return (int)best;
}

template <int G>
static void launch_adj_g(const AdjArgs& a, int kfoot, int groups, cudaStream_t st) {
    // kfoot: by value, may switch to the runtime-footprint kernel below
    constexpr int TH = AdjShape<G>::PPT * ADJ_WARPS;
    dim3 block(ADJ_TW, ADJ_WARPS),
        grid(adj_tiles_x(a.cols), (a.rows + TH - 1) / TH, groups * a.asplit);
    const size_t dyn = kfoot == 0 ? adj_stage_bytes(G, a.segw) : 0;
    if (kfoot == 0 && ADJ_STAGED(0, G) && dyn == 0) kfoot = -1;  // segments too long to stage
    if (kfoot == 0) adj_configure(G, dyn);
    switch (kfoot) {
        case 0: adj_kernel<0, G><<<grid, block, dyn, st>>>(a); break;
        case 1: adj_kernel<1, G><<<grid, block, 0, st>>>(a); break;
        case 2: adj_kernel<2, G><<<grid, block, 0, st>>>(a); break;
        case 3: adj_kernel<3, G><<<grid, block, 0, st>>>(a); break;
        default: adj_kernel<-1, G><<<grid, block, 0, st>>>(a); break;  // runtime footprint
    }
}

// Pairs first, then an odd last item on its own; both launches use the caller's
// angle split (K4 sums the same number of partial slots for every item).
cudaError_t launch_adj(const AdjArgs& a_in, int kfoot, int items, cudaStream_t st) {
    if (kfoot < 0) return cudaErrorInvalidValue;
    const int np = mct_pair_items(items, a_in.last_part);
    const int first = a_in.first, end = a_in.count ? first + a_in.count : items;
    const int p_lo = first < np ? first : np, p_hi = end < np ? end : np;
    const bool tail = end == items && items > np;
    auto pairs = [&](cudaStream_t s) {
        AdjArgs a = a_in;
        a.item0 = p_lo;
        a.n_items = items;
        launch_adj_g<2>(a, kfoot, (p_hi - p_lo) / 2, s);
    };
    auto singles = [&](cudaStream_t s) {
        AdjArgs a = a_in;
        a.item0 = np;
        a.n_items = items;
        launch_adj_g<1>(a, kfoot, items - np, s);
    };
    if (p_hi > p_lo && tail) return fork_join(st, pairs, singles);  // concurrent
    if (p_hi > p_lo) pairs(st);
    if (tail) singles(st);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- workspace
// (layout: mct_internal.cuh)
int mct_chunk_items(const mct_ray_plan* rp, int items) {
    return items / 2 > rp->wsg.ring ? 2 * rp->wsg.ring : items;
}

size_t mct_ws_bytes(const mct_ray_plan* rp, int items) {
    const WsGeom& g = rp->wsg;
    if (items <= 1) return g.item_bytes;
    const int pairs = items / 2;
    size_t bytes = 2 * g.item_bytes + (size_t)(pairs < g.ring ? pairs : g.ring) * g.pair_block;
    if (pairs > g.ring) {
        // overflow IMG area: the most slots any launch of <= items items needs beyond
        // the blocks' own (its paired items past the ring x its angle split; a half
        // last item changes both)
        long long slots = 0;
        for (int n = 2 * g.ring + 2; n <= items; ++n)
            for (int part = 0; part <= 1; ++part) {
                const long long over = mct_pair_items(n, part) - 2 * g.ring;
                const long long s = over * choose_asplit(rp, n, part);
                slots = s > slots ? s : slots;
            }
        bytes += (size_t)slots * rp->img_slot_bytes;
    }
    return bytes;
}

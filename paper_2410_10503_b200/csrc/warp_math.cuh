// Bilinear inverse-mapping warp D (motion.py:132-183) and its transpose
// (motion.py:185-194), restated as per-pixel device functions.
//
// The forward computes the source position of output pixel p and its four
// bilinear taps; the adjoint enumerates the output pixels p whose taps contain
// q and re-evaluates *the same* function, so forward and adjoint weights are
// bit-identical (the pair is an exact transpose up to summation order).
#pragma once

#include "mct_internal.cuh"

struct TapSet {
    int r0, c0;
    float fr, fc;
};

// Source position of output pixel (r, c).
//  rigid      : motion.py:139-151 (snapped cos/sin supplied by the host),
//               du = u - t_r; dv = v - t_c; su = cos*du + sin*dv; sv = -sin*du + cos*dv
//  dilatation : motion.py:152-154, su = u/scale, sv = v/scale
//  dense      : src = (r + phi_r, c + phi_c); integer part taken from phi alone so
//               the index is exact in fp32
// The _rn intrinsics forbid FMA contraction so the rigid/dilatation source
// coordinates round exactly like numpy's separate multiply and add.
__device__ __forceinline__ TapSet warp_taps(const WarpDesc& w, int r, int c) {
    TapSet t;
    if (w.kind == MCT_WARP_DENSE) {
        const long long n = (long long)w.rows * w.cols;
        const long long p = (long long)r * w.cols + c;
        float pr = __ldg(w.phi + p);
        float pc = __ldg(w.phi + n + p);
        float flr = floorf(pr), flc = floorf(pc);
        t.r0 = r + (int)flr;
        t.c0 = c + (int)flc;
        t.fr = pr - flr;
        t.fc = pc - flc;
        return t;
    }
    double u = __dsub_rn((double)r, w.hr);
    double v = __dsub_rn((double)c, w.hc);
    double su, sv;
    if (w.kind == MCT_WARP_RIGID) {
        double du = __dsub_rn(u, w.tr);
        double dv = __dsub_rn(v, w.tc);
        su = __dadd_rn(__dmul_rn(w.cs, du), __dmul_rn(w.sn, dv));
        sv = __dadd_rn(__dmul_rn(-w.sn, du), __dmul_rn(w.cs, dv));
    } else {  // dilatation
        su = __ddiv_rn(u, w.scale);
        sv = __ddiv_rn(v, w.scale);
    }
    double sr = __dadd_rn(su, w.hr);
    double sc = __dadd_rn(sv, w.hc);
    double fr0 = floor(sr), fc0 = floor(sc);
    // clamp before int conversion (far out-of-frame translations)
    fr0 = fmin(fmax(fr0, -4.0), (double)w.rows + 4.0);
    fc0 = fmin(fmax(fc0, -4.0), (double)w.cols + 4.0);
    t.r0 = (int)fr0;
    t.c0 = (int)fc0;
    t.fr = (float)__dsub_rn(sr, floor(sr));
    t.fc = (float)__dsub_rn(sc, floor(sc));
    return t;
}

// Weight of tap (dr, dc) in {0,1}^2 — motion.py:157-161 ordering.
__device__ __forceinline__ float tap_weight(const TapSet& t, int dr, int dc) {
    float wr = dr ? t.fr : (1.0f - t.fr);
    float wc = dc ? t.fc : (1.0f - t.fc);
    return wr * wc;
}

// Forward warp value at output pixel (r, c) reading input through `fetch(tr, tc)`
// (only called for in-grid taps).
template <typename Fetch>
__device__ __forceinline__ float warp_apply_at(const WarpDesc& w, int r, int c, Fetch fetch) {
    TapSet t = warp_taps(w, r, c);
    float acc = 0.0f;
#pragma unroll
    for (int dr = 0; dr < 2; ++dr) {
#pragma unroll
        for (int dc = 0; dc < 2; ++dc) {
            int rr = t.r0 + dr, cc = t.c0 + dc;
            if (rr >= 0 && rr < w.rows && cc >= 0 && cc < w.cols) {
                acc = fmaf(tap_weight(t, dr, dc), fetch(rr, cc), acc);
            }
        }
    }
    return acc;
}

// Transpose at pixel q = (qr, qc): sum over output pixels p with q among taps(p)
// of w(p, q) * y[p], reading y through `fetch(flat_index)`.  The plan's
// transposed gather list (sorted by p, built from warp_taps itself) makes the
// weights bit-identical to the forward's and the order fixed (deterministic).
// The adjoint's view of a warp descriptor, held in registers (a WarpDesc in global
// memory would be re-read for every entry: the compiler cannot prove it unaliased).
struct WarpT {
    int kind, cols;
    const int* tptr;
    const int* tidx;
    const float* tw;
};
__device__ __forceinline__ WarpT load_warp_t(const WarpDesc* d) {
    WarpT w;
    w.kind = __ldg(&d->kind);
    w.cols = __ldg(&d->cols);
    w.tptr = reinterpret_cast<const int*>(
        __ldg(reinterpret_cast<const unsigned long long*>(&d->tptr)));
    w.tidx = reinterpret_cast<const int*>(
        __ldg(reinterpret_cast<const unsigned long long*>(&d->tidx)));
    w.tw = reinterpret_cast<const float*>(
        __ldg(reinterpret_cast<const unsigned long long*>(&d->tw)));
    return w;
}

template <typename Fetch>
__device__ __forceinline__ float warp_adjoint_at(const WarpT& w, Fetch fetch, int qr, int qc) {
    const long long q = (long long)qr * w.cols + qc;
    if (w.kind == MCT_WARP_IDENTITY) return fetch(q);
    const int e0 = __ldg(w.tptr + q), e1 = __ldg(w.tptr + q + 1);
    float acc = 0.0f;
    // four entries per round: their index / weight loads, then their fetches, are
    // in flight together; the FMAs stay in entry order (same sum as one by one)
    for (int e = e0; e < e1; e += 4) {
        int idx[4];
        float wt[4], v[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const bool ok = e + j < e1;
            idx[j] = ok ? __ldg(w.tidx + e + j) : -1;
            wt[j] = ok ? __ldg(w.tw + e + j) : 0.0f;
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) v[j] = idx[j] >= 0 ? fetch(idx[j]) : 0.0f;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (idx[j] >= 0) acc = fmaf(wt[j], v[j], acc);
    }
    return acc;
}

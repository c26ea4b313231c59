// C-ABI layer (include/mctomo_b200.h): argument validation, plan construction,
// workspace layout and kernel launches.  No torch types cross this boundary.
#include "mct_internal.cuh"

#include <math.h>
#include <stdio.h>

#include <algorithm>
#include <string>
#include <vector>

namespace {
thread_local std::string g_err;

inline size_t align256(size_t b) { return (b + 255) & ~size_t(255); }

inline int cuda_fail(cudaError_t e, const char* where) {
    return mct_set_error(MCT_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define MCT_CUDA(call, where)                         \
    do {                                              \
        cudaError_t _e = (call);                      \
        if (_e != cudaSuccess) return cuda_fail(_e, where); \
    } while (0)

#define MCT_REQUIRE(cond, msg)                                       \
    do {                                                             \
        if (!(cond)) return mct_set_error(MCT_ERR_ARG, (msg));       \
    } while (0)

WarpDesc identity_desc(int rows, int cols) {
    WarpDesc d;
    memset(&d, 0, sizeof(d));
    d.kind = MCT_WARP_IDENTITY;
    d.rows = rows;
    d.cols = cols;
    d.hr = 0.5 * (rows - 1);
    d.hc = 0.5 * (cols - 1);
    return d;
}

ItemSel make_sel(const mct_items* it) {
    ItemSel s;
    s.gates = it->gates_dev;
    s.epoch_ctr = it->epoch_ctr_dev;
    s.slice_stride = it->slice_stride;
    s.epoch_stride = it->epoch_stride;
    s.base = it->base;
    s.ips = it->items_per_slice;
    s.num_slices = it->num_slices;
    s.iteration = it->iteration;
    s.iters_per_epoch = it->iters_per_epoch;
    s.last_part = it->last_part;
    s.first = it->first_item;
    s.count = it->item_count;
    return s;
}

ItemSel single_sel(int slices) {
    ItemSel s;
    memset(&s, 0, sizeof(s));
    s.ips = 1;
    s.num_slices = slices;
    return s;
}

int check_items(const mct_family* fam, const mct_items* it) {
    MCT_REQUIRE(fam && it, "null family or item selector");
    MCT_REQUIRE(it->gates_dev != nullptr, "items.gates_dev must be a device gate array");
    MCT_REQUIRE(it->items_per_slice >= 1, "items_per_slice must be >= 1");
    MCT_REQUIRE(it->num_slices >= 1 && it->num_slices <= fam->S,
                "items.num_slices must lie in [1, family slices]");
    MCT_REQUIRE(it->last_part >= 0 && it->last_part <= 2, "items.last_part must be 0, 1 or 2");
    MCT_REQUIRE(it->last_part == 0 || it->num_slices == 1,
                "a half last item needs a single-slice launch");
    const int n = it->items_per_slice * it->num_slices;
    MCT_REQUIRE(it->first_item >= 0 && it->first_item < n && (it->first_item & 1) == 0,
                "items.first_item must be an even item index of the launch");
    MCT_REQUIRE(it->item_count >= 0 && it->first_item + it->item_count <= n,
                "items.item_count must be 0 (to the end) or end inside the launch");
    return MCT_OK;
}

// K1-K3: the chunk's gate pairs must fit the workspace's ring of pair regions and
// start on a ring boundary (mct_family_chunk_items)
int check_chunk(const mct_family* fam, const mct_items* it) {
    const int n = it->items_per_slice * it->num_slices;
    const int np = mct_pair_items(n, it->last_part);
    const int ring = fam->ray->wsg.ring;
    const int end = it->item_count ? it->first_item + it->item_count : n;
    const int p_lo = std::min(it->first_item, np), p_hi = std::min(end, np);
    MCT_REQUIRE((p_hi - p_lo) / 2 <= ring,
                "launch holds more gate pairs than the workspace's ring: run K1-K3 in chunks "
                "of mct_family_chunk_items items (items.first_item / item_count)");
    MCT_REQUIRE((p_lo / 2) % ring == 0, "items.first_item must be a multiple of the chunk size");
    MCT_REQUIRE(it->item_count == 0 || end == n || (it->item_count & 1) == 0,
                "a chunk that does not end the launch must hold whole gate pairs");
    return MCT_OK;
}

FwdArgs fwd_args(const mct_ray_plan* rp, const void* ws) {
    FwdArgs a;
    memset(&a, 0, sizeof(a));
    a.ang = rp->d_fwd;
    a.A = rp->A;
    a.B = rp->B;
    a.rows = rp->rows;
    a.cols = rp->cols;
    a.wx = rp->wx;
    a.wxt = rp->wxt;
    a.sp = rp->sp;
    a.jmid = rp->jmid;
    a.ws = static_cast<const char*>(ws);
    a.wsg = rp->wsg;
    a.off_x = rp->off_x;
    a.off_xt = rp->off_xt;
    a.off_dy = rp->off_dy;
    a.off_part = rp->off_part;
    a.off_cnt = rp->off_cnt;
    a.off_px = rp->off_px;
    a.off_pxt = rp->off_pxt;
    a.off_pdy = rp->off_pdy;
    a.ksplit = rp->ksplit1;
    a.wy = rp->wy;
    a.pb = rp->pb;
    return a;
}

AdjArgs adj_args(const mct_ray_plan* rp, const void* ws) {
    AdjArgs a;
    a.ang = rp->d_adj;
    a.A = rp->A;
    a.B = rp->B;
    a.rows = rp->rows;
    a.cols = rp->cols;
    a.wy = rp->wy;
    a.pb = rp->pb;
    a.jmid = rp->jmid;
    a.ws = static_cast<const char*>(ws);
    a.wsg = rp->wsg;
    a.off_dy = rp->off_dy;
    a.off_img = rp->off_img;
    a.img_slot_bytes = rp->img_slot_bytes;
    a.off_pdy = rp->off_pdy;
    a.item0 = 0;
    a.n_items = 1;
    a.last_part = 0;
    a.first = 0;
    a.count = 0;
    a.asplit = 1;
    a.kfoot = rp->kfoot;
    a.segw = rp->adj_segw;
    return a;
}

PackArgs pack_args(const mct_ray_plan* rp, void* ws) {
    PackArgs a;
    memset(&a, 0, sizeof(a));
    a.rows = rp->rows;
    a.cols = rp->cols;
    a.wx = rp->wx;
    a.wxt = rp->wxt;
    a.ws = static_cast<char*>(ws);
    a.wsg = rp->wsg;
    a.off_x = rp->off_x;
    a.off_xt = rp->off_xt;
    a.off_px = rp->off_px;
    a.off_pxt = rp->off_pxt;
    a.x_slice_stride = (long long)rp->rows * rp->cols;
    a.cprox = 1.0f;
    return a;
}

UpdArgs upd_args(const mct_ray_plan* rp, const void* ws) {
    UpdArgs a;
    memset(&a, 0, sizeof(a));
    a.rows = rp->rows;
    a.cols = rp->cols;
    a.ws = static_cast<const char*>(ws);
    a.wsg = rp->wsg;
    a.off_img = rp->off_img;
    a.img_slot_bytes = rp->img_slot_bytes;
    a.asplit = 1;
    return a;
}
}  // namespace

int mct_set_error(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

extern "C" {

int mct_abi_version(void) { return MCT_ABI_VERSION; }
const char* mct_last_error(void) { return g_err.c_str(); }

// ------------------------------------------------------------------ ray plan
int mct_ray_plan_create(mct_ray_plan** plan, int rows, int cols, int num_angles, int num_bins,
                        double spacing, const double* cos_a, const double* sin_a,
                        const uint8_t* rows_dominant) {
    MCT_REQUIRE(plan, "plan out-pointer is null");
    *plan = nullptr;
    // Geometry.__post_init__ (projector.py:63-68)
    MCT_REQUIRE(rows >= 1, "rows must be >= 1");
    MCT_REQUIRE(cols >= 1, "cols must be >= 1");
    MCT_REQUIRE((long long)rows * cols <= MCT_MAX_PIXELS, "images above 2^29 pixels are not supported");
    MCT_REQUIRE(num_angles >= 1, "num_angles must be >= 1");
    MCT_REQUIRE(num_bins >= 1, "num_bins must be >= 1");
    MCT_REQUIRE(spacing > 0 && isfinite(spacing), "detector_spacing must be positive");
    MCT_REQUIRE(cos_a && sin_a && rows_dominant, "angle tables are null");

    mct_ray_plan* p = new mct_ray_plan();
    p->rows = rows;
    p->cols = cols;
    p->A = num_angles;
    p->B = num_bins;
    p->sp = spacing;
    p->jmid = 0.5 * (num_bins - 1);
    p->wx = cols + 2 * MCT_PADX;
    p->wxt = rows + 2 * MCT_PADX;
    std::vector<RayAngle> fwd(num_angles);
    std::vector<AdjAngle> adj(num_angles);
    const double hr = 0.5 * (rows - 1), hc = 0.5 * (cols - 1);
    double hmax = 0.0;
    for (int a = 0; a < num_angles; ++a) {
        const double c = cos_a[a], s = sin_a[a];
        RayAngle& r = fwd[a];
        double m;
        if (rows_dominant[a]) {
            if (c == 0.0) {
                delete p;
                return mct_set_error(MCT_ERR_ARG, "rows-dominant angle with cos == 0");
            }
            // projector.py:137-143
            r.P = 1.0 / c;
            r.slope = s / c;
            r.Q = hc - hr * r.slope;
            m = fabs(c);
            r.cols_dom = 0;
        } else {
            if (!(s > 0.0)) {
                delete p;
                return mct_set_error(MCT_ERR_ARG, "cols-dominant angle with sin <= 0");
            }
            // projector.py:148-154
            r.P = -1.0 / s;
            r.slope = c / s;
            r.Q = hr - hc * r.slope;
            m = s;
            r.cols_dom = 1;
        }
        r.step = (float)(1.0 / m);
        r.slope_fx = llrint(r.slope * 4294967296.0);
        adj[a].cs = c / spacing;
        adj[a].sn = s / spacing;
        adj[a].csx = llrint(c / spacing * 4294967296.0);
        adj[a].snx = llrint(s / spacing * 4294967296.0);
        adj[a].step = (float)(1.0 / m);
        adj[a].g = (float)(spacing / m);
        hmax = std::max(hmax, m / spacing);
        p->h_acs.push_back(fabs(c) / spacing);
        p->h_asn.push_back(fabs(s) / spacing);
    }
    p->adj_segw = adj_segw(p);
    // adjoint footprint: bins within hmax of the pixel's detector coordinate
    // (any positive spacing, projector.py:63-68; K > 3 runs the runtime-K kernel)
    const int K = std::max(0, (int)ceil(hmax - 1e-12) - 1);
    p->kfoot = K;
    const double hdiag = sqrt(hr * hr + hc * hc);
    int pb = (int)ceil(std::max(0.0, hdiag / spacing - p->jmid)) + K + 4;
    pb = (pb + 3) & ~3;
    p->pb = pb;
    p->wy = num_bins + 2 * pb;
    size_t off = 0;
    // item region: the prefix every item uses (paired or not) -- A^* partial-image
    // slots -- then what only single items use: K2 ray-split partials and arrival
    // counters, and the mirror layouts: pair-packed float2 (v[i], v[i+1] - v[i]) elements, one load
    // fetches both interpolation taps, two per float4 element: the item and its
    // column mirror (X, XT), angles q and A-q (DY rows 1 .. (A-1)/2; row 0 holds the
    // self-paired angles 0 and A/2) -- see mct_internal.cuh
    p->off_img = off;
    p->img_slot_bytes = align256((size_t)rows * cols * sizeof(float));
    // A^* partial-image slots: the largest angle split any launch of this plan may
    // use (choose_asplit never exceeds it)
    off += p->img_slot_bytes * (size_t)adj_plan_slots(p);
    p->wsg.pre_bytes = off;  // paired items use only their A^* slots (K2 pairs: no ray split)
    p->off_part = off;
    p->ksplit1 = choose_ksplit(num_angles, num_bins, std::max(rows, cols));
    off += align256((size_t)p->ksplit1 * num_angles * num_bins * sizeof(double));
    p->off_cnt = off;
    off += align256((size_t)mct_fwd_groups(num_angles) * mct_fwd_btiles(num_bins) * sizeof(int));
    // X and XT get max(rows, cols) rows: a K2 warp may walk a rows-dominant and a
    // cols-dominant ray together (MCT_FWD_IL), stepping up to max(rows, cols) rows;
    // the extra rows stay zero, so the short ray reads zeros there
    const size_t nrow = (size_t)std::max(rows, cols);
    p->off_x = off;
    off += align256(nrow * p->wx * sizeof(float4));
    p->off_xt = off;
    off += align256(nrow * p->wxt * sizeof(float4));
    p->off_dy = off;
    off += align256((size_t)(num_angles / 2 + 1) * p->wy * sizeof(float4));
    p->wsg.item_bytes = off;
    // gate-pair region (interleaved float4 layouts, see mct_internal.cuh)
    size_t poff = 0;
    p->off_px = poff;
    poff += align256(nrow * p->wx * sizeof(float4));
    p->off_pxt = poff;
    poff += align256(nrow * p->wxt * sizeof(float4));
    p->off_pdy = poff;
    poff += align256((size_t)num_angles * p->wy * sizeof(float4));
    p->wsg.pair_bytes = poff;
    p->wsg.pair_block = poff + 2 * p->wsg.pre_bytes;
    p->wsg.ring = (int)std::max<long long>(MCT_RING_MIN_PAIRS,
                                           (long long)((MCT_RING_BYTES + poff - 1) / poff));

    cudaError_t e = cudaMalloc(&p->d_fwd, sizeof(RayAngle) * num_angles);
    if (e == cudaSuccess) e = cudaMalloc(&p->d_adj, sizeof(AdjAngle) * num_angles);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_fwd, fwd.data(), sizeof(RayAngle) * num_angles, cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(p->d_adj, adj.data(), sizeof(AdjAngle) * num_angles, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(p->d_fwd);
        cudaFree(p->d_adj);
        delete p;
        return cuda_fail(e, "mct_ray_plan_create");
    }
    *plan = p;
    return MCT_OK;
}

int mct_ray_plan_destroy(mct_ray_plan* plan) {
    if (!plan) return MCT_OK;
    cudaFree(plan->d_fwd);
    cudaFree(plan->d_adj);
    delete plan;
    return MCT_OK;
}

size_t mct_ray_workspace_bytes(const mct_ray_plan* plan, int batch) {
    if (!plan || batch < 1) return 0;
    return mct_ws_bytes(plan, batch);
}

int mct_ray_plan_set_ring_pairs(mct_ray_plan* plan, int pairs) {
    MCT_REQUIRE(plan, "plan is null");
    MCT_REQUIRE(pairs >= 1, "pairs must be >= 1");
    plan->wsg.ring = pairs;
    return MCT_OK;
}

int mct_ray_forward(const mct_ray_plan* rp, const float* x, float* sino, int batch, void* ws,
                    void* stream) {
    MCT_REQUIRE(rp && x && sino && ws, "null argument");
    MCT_REQUIRE(batch >= 1, "batch must be >= 1");
    cudaStream_t st = (cudaStream_t)stream;
    PackArgs pa = pack_args(rp, ws);
    pa.x = x;
    FwdArgs fa = fwd_args(rp, ws);
    fa.out = sino;
    fa.out_item_stride = (long long)rp->A * rp->B;
    const int chunk = mct_chunk_items(rp, batch);
    for (int f = 0; f < batch; f += chunk) {  // chunks of the workspace's pair ring
        pa.sel = fa.sel = single_sel(batch);
        pa.sel.first = fa.sel.first = f;
        pa.sel.count = fa.sel.count = f + chunk < batch ? chunk : 0;
        MCT_CUDA(launch_pack(pa, batch, st), "pack");
        MCT_CUDA(launch_fwd(fa, 0, batch, st), "ray forward");
    }
    return MCT_OK;
}

int mct_ray_adjoint(const mct_ray_plan* rp, const float* sino, float* img, int batch, void* ws,
                    void* stream) {
    MCT_REQUIRE(rp && sino && img && ws, "null argument");
    MCT_REQUIRE(batch >= 1, "batch must be >= 1");
    cudaStream_t st = (cudaStream_t)stream;
    AdjArgs aa = adj_args(rp, ws);
    aa.asplit = choose_asplit(rp, batch);
    const int chunk = mct_chunk_items(rp, batch);
    for (int f = 0; f < batch; f += chunk) {  // chunks of the workspace's pair ring
        aa.first = f;
        aa.count = f + chunk < batch ? chunk : 0;
        MCT_CUDA(launch_pad_sino(sino, rp, static_cast<char*>(ws), aa.wsg, batch, aa.first,
                                 aa.count, st),
                 "pad sinogram");
        MCT_CUDA(launch_adj(aa, rp->kfoot, batch, st), "ray adjoint");
    }
    UpdArgs ua = upd_args(rp, ws);
    ua.asplit = aa.asplit;
    ua.sel = single_sel(batch);
    ua.out = img;
    MCT_CUDA(launch_update(ua, 0, batch, st), "ray adjoint (partials)");
    return MCT_OK;
}

// ----------------------------------------------------------------- warps
// Transposed gather list of a non-identity warp (the adjoint D^* reads it): built
// on the device from the forward's own taps, so forward and adjoint weights are
// bit-identical.  Synchronous (plan construction only).
static cudaError_t attach_transpose(mct_warp_plan* p, cudaStream_t st) {
    cudaError_t e = build_dense_transpose(p->desc, &p->tptr, &p->tidx, &p->tw, &p->nnz, st);
    if (e != cudaSuccess) return e;
    p->desc.tptr = p->tptr;
    p->desc.tidx = p->tidx;
    p->desc.tw = p->tw;
    return cudaSuccess;
}

static int warp_finish(mct_warp_plan* p, mct_warp_plan** out) {
    cudaError_t e = cudaMalloc(&p->d_desc, sizeof(WarpDesc));
    if (e == cudaSuccess) e = cudaMemcpy(p->d_desc, &p->desc, sizeof(WarpDesc), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        cudaFree(p->d_desc);
        cudaFree(p->phi);
        cudaFree(p->tptr);
        cudaFree(p->tidx);
        cudaFree(p->tw);
        delete p;
        return cuda_fail(e, "warp plan");
    }
    *out = p;
    return MCT_OK;
}

int mct_warp_plan_create_identity(mct_warp_plan** plan, int rows, int cols) {
    MCT_REQUIRE(plan, "plan out-pointer is null");
    *plan = nullptr;
    MCT_REQUIRE(rows >= 1 && cols >= 1 && (long long)rows * cols <= MCT_MAX_PIXELS,
                "invalid image shape");
    mct_warp_plan* p = new mct_warp_plan();
    p->desc = identity_desc(rows, cols);
    return warp_finish(p, plan);
}

int mct_warp_plan_create_rigid(mct_warp_plan** plan, int rows, int cols, double cos_r,
                               double sin_r, double t_row, double t_col) {
    MCT_REQUIRE(plan, "plan out-pointer is null");
    *plan = nullptr;
    MCT_REQUIRE(rows >= 1 && cols >= 1 && (long long)rows * cols <= MCT_MAX_PIXELS,
                "invalid image shape");
    MCT_REQUIRE(isfinite(cos_r) && isfinite(sin_r) && isfinite(t_row) && isfinite(t_col),
                "motion parameters must be finite");
    mct_warp_plan* p = new mct_warp_plan();
    WarpDesc d = identity_desc(rows, cols);
    d.kind = MCT_WARP_RIGID;
    d.cs = cos_r;
    d.sn = sin_r;
    d.tr = t_row;
    d.tc = t_col;
    p->desc = d;
    cudaError_t e = attach_transpose(p, 0);
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e, "mct_warp_plan_create_rigid");
    }
    return warp_finish(p, plan);
}

int mct_warp_plan_create_dilatation(mct_warp_plan** plan, int rows, int cols, double scale) {
    MCT_REQUIRE(plan, "plan out-pointer is null");
    *plan = nullptr;
    MCT_REQUIRE(rows >= 1 && cols >= 1 && (long long)rows * cols <= MCT_MAX_PIXELS,
                "invalid image shape");
    MCT_REQUIRE(scale > 0 && isfinite(scale), "scale must be positive");
    mct_warp_plan* p = new mct_warp_plan();
    WarpDesc d = identity_desc(rows, cols);
    d.kind = MCT_WARP_DILATATION;
    d.scale = scale;
    p->desc = d;
    cudaError_t e = attach_transpose(p, 0);
    if (e != cudaSuccess) {
        delete p;
        return cuda_fail(e, "mct_warp_plan_create_dilatation");
    }
    return warp_finish(p, plan);
}

int mct_warp_plan_create_dense(mct_warp_plan** plan, int rows, int cols, const float* phi_dev,
                               void* stream) {
    MCT_REQUIRE(plan, "plan out-pointer is null");
    *plan = nullptr;
    MCT_REQUIRE(rows >= 1 && cols >= 1 && (long long)rows * cols <= MCT_MAX_PIXELS,
                "invalid image shape");
    MCT_REQUIRE(phi_dev, "phi is null");
    cudaStream_t st = (cudaStream_t)stream;
    const long long n = (long long)rows * cols;
    mct_warp_plan* p = new mct_warp_plan();
    WarpDesc d = identity_desc(rows, cols);
    d.kind = MCT_WARP_DENSE;
    cudaError_t e = cudaMalloc(&p->phi, 2 * n * sizeof(float));
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(p->phi, phi_dev, 2 * n * sizeof(float), cudaMemcpyDeviceToDevice, st);
    // reject non-finite fields (MotionParams finiteness rule, motion.py:64-77)
    float* d_max = nullptr;
    float hmax = 0.0f;
    if (e == cudaSuccess) e = cudaMalloc(&d_max, sizeof(float));
    if (e == cudaSuccess) e = launch_absmax(p->phi, 2 * n, d_max, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&hmax, d_max, sizeof(float), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    cudaFree(d_max);
    if (e == cudaSuccess && !isfinite(hmax)) {
        cudaFree(p->phi);
        delete p;
        return mct_set_error(MCT_ERR_ARG, "displacement field must be finite");
    }
    if (e == cudaSuccess && hmax > 1.0e6f) {
        cudaFree(p->phi);
        delete p;
        return mct_set_error(MCT_ERR_ARG, "displacement field magnitude exceeds 1e6 pixels");
    }
    d.phi = p->phi;
    if (e == cudaSuccess) e = build_dense_transpose(d, &p->tptr, &p->tidx, &p->tw, &p->nnz, st);
    if (e != cudaSuccess) {
        cudaFree(p->phi);
        delete p;
        return cuda_fail(e, "mct_warp_plan_create_dense");
    }
    d.tptr = p->tptr;
    d.tidx = p->tidx;
    d.tw = p->tw;
    p->desc = d;
    return warp_finish(p, plan);
}

int mct_warp_plan_destroy(mct_warp_plan* plan) {
    if (!plan) return MCT_OK;
    cudaFree(plan->d_desc);
    cudaFree(plan->phi);
    cudaFree(plan->tptr);
    cudaFree(plan->tidx);
    cudaFree(plan->tw);
    delete plan;
    return MCT_OK;
}

int mct_warp_plan_kind(const mct_warp_plan* plan) { return plan ? plan->desc.kind : -1; }
long long mct_warp_plan_nnz(const mct_warp_plan* plan) { return plan ? plan->nnz : -1; }

int mct_warp_forward(const mct_warp_plan* plan, const float* x, float* out, void* stream) {
    MCT_REQUIRE(plan && x && out, "null argument");
    MCT_CUDA(launch_warp_fwd_plain(plan->d_desc, x, out, plan->desc.rows, plan->desc.cols,
                                   (cudaStream_t)stream),
             "warp forward");
    return MCT_OK;
}

int mct_warp_adjoint(const mct_warp_plan* plan, const float* y, float* out, void* stream) {
    MCT_REQUIRE(plan && y && out, "null argument");
    UpdArgs a;
    memset(&a, 0, sizeof(a));
    a.rows = plan->desc.rows;
    a.cols = plan->desc.cols;
    a.img_override = y;
    a.asplit = 1;
    a.sel = single_sel(1);
    a.warps = plan->d_desc;
    a.out = out;
    MCT_CUDA(launch_update(a, 0, 1, (cudaStream_t)stream), "warp adjoint");
    return MCT_OK;
}

// ----------------------------------------------------------------- family
int mct_family_create(mct_family** fam, const mct_ray_plan* ray, int num_slices, int num_gates,
                      const mct_warp_plan* const* warps) {
    MCT_REQUIRE(fam, "family out-pointer is null");
    *fam = nullptr;
    MCT_REQUIRE(ray, "ray plan is null");
    MCT_REQUIRE(num_slices >= 1, "num_slices must be >= 1");
    MCT_REQUIRE(num_gates >= 1, "at least one gate required");
    std::vector<WarpDesc> descs((size_t)num_slices * num_gates);
    for (size_t i = 0; i < descs.size(); ++i) {
        const mct_warp_plan* w = warps ? warps[i] : nullptr;
        if (w) {
            if (w->desc.rows != ray->rows || w->desc.cols != ray->cols)
                return mct_set_error(MCT_ERR_ARG, "warp shape does not match the ray geometry");
            descs[i] = w->desc;
        } else {
            descs[i] = identity_desc(ray->rows, ray->cols);
        }
    }
    mct_family* f = new mct_family();
    f->ray = ray;
    f->S = num_slices;
    f->N = num_gates;
    f->params_set = 0;
    cudaError_t e = cudaMalloc(&f->d_warps, sizeof(WarpDesc) * descs.size());
    if (e == cudaSuccess)
        e = cudaMemcpy(f->d_warps, descs.data(), sizeof(WarpDesc) * descs.size(),
                       cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&f->d_params, sizeof(GateParam) * num_gates);
    if (e == cudaSuccess) e = cudaMemset(f->d_params, 0, sizeof(GateParam) * num_gates);
    if (e != cudaSuccess) {
        cudaFree(f->d_warps);
        cudaFree(f->d_params);
        delete f;
        return cuda_fail(e, "mct_family_create");
    }
    *fam = f;
    return MCT_OK;
}

int mct_family_destroy(mct_family* fam) {
    if (!fam) return MCT_OK;
    cudaFree(fam->d_warps);
    cudaFree(fam->d_params);
    delete fam;
    return MCT_OK;
}

int mct_family_set_params(mct_family* fam, const double* sigmas, const double* probs,
                          double theta) {
    MCT_REQUIRE(fam && sigmas && probs, "null argument");
    MCT_REQUIRE(theta > 0 && theta <= 1, "theta must lie in (0, 1]");
    std::vector<GateParam> gp(fam->N);
    for (int g = 0; g < fam->N; ++g) {
        MCT_REQUIRE(sigmas[g] > 0 && isfinite(sigmas[g]), "all sigmas must be positive and finite");
        MCT_REQUIRE(probs[g] > 0 && probs[g] <= 1, "probabilities must lie in (0, 1]");
        gp[g].sigma = (float)sigmas[g];
        gp[g].dual_inv = (float)(1.0 / (1.0 + sigmas[g] * fam->N / 2.0));
        gp[g].theta_over_p = (float)(theta / probs[g]);
        gp[g].pad_ = 0.0f;
    }
    MCT_CUDA(cudaMemcpy(fam->d_params, gp.data(), sizeof(GateParam) * fam->N, cudaMemcpyHostToDevice),
             "mct_family_set_params");
    fam->params_set = 1;
    return MCT_OK;
}

size_t mct_family_workspace_bytes(const mct_family* fam, int items) {
    if (!fam || items < 1) return 0;
    return mct_ws_bytes(fam->ray, items);
}

int mct_family_chunk_items(const mct_family* fam, int items) {
    if (!fam || items < 1) return 0;
    return mct_chunk_items(fam->ray, items);
}

int mct_gated_forward(const mct_family* fam, int slice, int gate, const float* x, float* sino,
                      void* ws, void* stream) {
    MCT_REQUIRE(fam && x && sino && ws, "null argument");
    MCT_REQUIRE(slice >= 0 && slice < fam->S && gate >= 0 && gate < fam->N, "gate out of range");
    const mct_ray_plan* rp = fam->ray;
    cudaStream_t st = (cudaStream_t)stream;
    PackArgs pa = pack_args(rp, ws);
    pa.sel = single_sel(1);
    pa.x = x;
    pa.warps = fam->d_warps + (size_t)slice * fam->N + gate;
    MCT_CUDA(launch_pack(pa, 1, st), "gated pack");
    FwdArgs fa = fwd_args(rp, ws);
    fa.sel = single_sel(1);
    fa.out = sino;
    fa.out_item_stride = (long long)rp->A * rp->B;
    MCT_CUDA(launch_fwd(fa, 0, 1, st), "gated forward");
    return MCT_OK;
}

int mct_gated_forward_many(const mct_family* fam, int slice, const int32_t* gates, int count,
                           const float* x, float* sino, void* ws, void* stream) {
    MCT_REQUIRE(fam && gates && x && sino && ws, "null argument");
    MCT_REQUIRE(slice >= 0 && slice < fam->S, "slice out of range");
    MCT_REQUIRE(count >= 1 && count <= fam->N, "count must lie in [1, num_gates]");
    const mct_ray_plan* rp = fam->ray;
    cudaStream_t st = (cudaStream_t)stream;
    ItemSel sel;
    memset(&sel, 0, sizeof(sel));
    sel.gates = gates;  // item k -> gates[k] of this slice
    sel.ips = count;
    sel.num_slices = 1;
    PackArgs pa = pack_args(rp, ws);
    pa.N = fam->N;
    pa.x = x;
    pa.warps = fam->d_warps + (size_t)slice * fam->N;
    FwdArgs fa = fwd_args(rp, ws);
    fa.ksplit = count > 1 ? 1 : rp->ksplit1;  // as the fused iteration (see MCT_KSPLIT_MIN)
    fa.out = sino;
    fa.out_item_stride = (long long)rp->A * rp->B;
    const int chunk = mct_chunk_items(rp, count);
    for (int f = 0; f < count; f += chunk) {
        sel.first = f;
        sel.count = f + chunk < count ? chunk : 0;
        pa.sel = fa.sel = sel;
        MCT_CUDA(launch_pack(pa, count, st), "gated pack (many)");
        MCT_CUDA(launch_fwd(fa, 0, count, st), "gated forward (many)");
    }
    return MCT_OK;
}

int mct_gated_adjoint(const mct_family* fam, int slice, int gate, const float* y, float* img,
                      void* ws, void* stream) {
    MCT_REQUIRE(fam && y && img && ws, "null argument");
    MCT_REQUIRE(slice >= 0 && slice < fam->S && gate >= 0 && gate < fam->N, "gate out of range");
    const mct_ray_plan* rp = fam->ray;
    cudaStream_t st = (cudaStream_t)stream;
    AdjArgs aa = adj_args(rp, ws);
    MCT_CUDA(launch_pad_sino(y, rp, static_cast<char*>(ws), aa.wsg, 1, 0, 0, st), "pad sinogram");
    aa.asplit = choose_asplit(rp, 1);
    MCT_CUDA(launch_adj(aa, rp->kfoot, 1, st), "gated adjoint (A^*)");
    UpdArgs ua = upd_args(rp, ws);
    ua.asplit = aa.asplit;
    ua.sel = single_sel(1);
    ua.warps = fam->d_warps + (size_t)slice * fam->N + gate;
    ua.out = img;
    MCT_CUDA(launch_update(ua, 0, 1, st), "gated adjoint (D^*)");
    return MCT_OK;
}

// ------------------------------------------------------- fused iteration
int mct_iter_prox_warp(const mct_family* fam, const mct_items* it, mct_state* s, double tau,
                       double alpha, void* ws, void* stream) {
    int rc = check_items(fam, it);
    if (rc) return rc;
    MCT_REQUIRE(s && s->x && s->zbar && s->x_next && ws, "null state buffer");
    MCT_REQUIRE(tau >= 0 && alpha >= 0, "tau and alpha must be >= 0");
    if ((rc = check_chunk(fam, it))) return rc;
    const mct_ray_plan* rp = fam->ray;
    PackArgs pa = pack_args(rp, ws);
    pa.sel = make_sel(it);
    pa.N = fam->N;
    pa.warps = fam->d_warps;
    pa.x = s->x;
    pa.zbar = s->zbar;
    pa.tau = (float)tau;
    pa.cprox = (float)(1.0 / (1.0 + 2.0 * alpha * tau));  // functionals.py:48
    pa.x_next = s->x_next;
    pa.status = s->status;
    MCT_CUDA(launch_pack(pa, it->items_per_slice * it->num_slices, (cudaStream_t)stream),
             "prox+warp");
    return MCT_OK;
}

int mct_iter_forward_dual(const mct_family* fam, const mct_items* it, mct_state* s, void* ws,
                          void* stream) {
    int rc = check_items(fam, it);
    if (rc) return rc;
    MCT_REQUIRE(fam->params_set, "mct_family_set_params has not been called");
    MCT_REQUIRE(s && s->y && s->d && ws, "null state buffer");
    if ((rc = check_chunk(fam, it))) return rc;
    FwdArgs fa = fwd_args(fam->ray, ws);
    fa.ksplit = it->items_per_slice > 1 ? 1 : fam->ray->ksplit1;  // see MCT_KSPLIT_MIN
    fa.sel = make_sel(it);
    fa.N = fam->N;
    fa.y = s->y;
    fa.d = s->d;
    fa.proj = s->proj;
    fa.gp = fam->d_params;
    fa.status = s->status;
    MCT_CUDA(launch_fwd(fa, 1, it->items_per_slice * it->num_slices, (cudaStream_t)stream),
             "forward+dual");
    return MCT_OK;
}

int mct_iter_adjoint(const mct_family* fam, const mct_items* it, void* ws, void* stream) {
    int rc = check_items(fam, it);
    if (rc) return rc;
    MCT_REQUIRE(ws, "null workspace");
    if ((rc = check_chunk(fam, it))) return rc;
    AdjArgs aa = adj_args(fam->ray, ws);
    const int items = it->items_per_slice * it->num_slices;
    aa.last_part = it->last_part;
    aa.first = it->first_item;
    aa.count = it->item_count;
    aa.asplit = choose_asplit(fam->ray, items, it->last_part);
    MCT_CUDA(launch_adj(aa, fam->ray->kfoot, items, (cudaStream_t)stream), "adjoint");
    return MCT_OK;
}

int mct_iter_adjoint_update(const mct_family* fam, const mct_items* it, mct_state* s,
                            float* dz_partial, void* ws, void* stream) {
    int rc = check_items(fam, it);
    if (rc) return rc;
    MCT_REQUIRE(fam->params_set, "mct_family_set_params has not been called");
    MCT_REQUIRE(s && s->x && s->x_next && ws, "null state buffer");
    MCT_REQUIRE(it->first_item == 0 && it->item_count == 0,
                "K4 gathers every item of the launch: first_item / item_count must be 0");
    UpdArgs ua = upd_args(fam->ray, ws);
    ua.asplit = choose_asplit(fam->ray, it->items_per_slice * it->num_slices, it->last_part);
    ua.sel = make_sel(it);
    ua.N = fam->N;
    ua.warps = fam->d_warps;
    ua.gp = fam->d_params;
    ua.x = s->x;
    ua.x_next = s->x_next;
    int mode;
    if (dz_partial) {
        ua.dz = dz_partial;
        mode = 2;
    } else {
        MCT_REQUIRE(s->z && s->zbar, "null z / zbar");
        ua.z = s->z;
        ua.zbar = s->zbar;
        mode = 1;
    }
    MCT_CUDA(launch_update(ua, mode, it->num_slices, (cudaStream_t)stream), "adjoint update");
    return MCT_OK;
}

int mct_iter_z_update(const mct_family* fam, mct_state* s, const float* dz, double theta,
                      void* stream) {
    MCT_REQUIRE(fam && s && s->z && s->zbar && dz, "null argument");
    const long long n = (long long)fam->S * fam->ray->rows * fam->ray->cols;
    MCT_CUDA(launch_z_update(n, dz, s->z, s->zbar, (float)theta, (cudaStream_t)stream), "z update");
    return MCT_OK;
}

int mct_epoch_advance(int32_t* ctr, int32_t inc, void* stream) {
    MCT_REQUIRE(ctr, "null counter");
    MCT_CUDA(launch_epoch_advance(ctr, inc, (cudaStream_t)stream), "epoch advance");
    return MCT_OK;
}

// -------------------------------------------------------------- reductions
int mct_reduce(const float* a, const float* b, long long length, int segments, long long stride,
               int mode, double* out, double* scratch, void* stream) {
    MCT_REQUIRE(a && out, "null argument");
    MCT_REQUIRE(length >= 0 && segments >= 1, "invalid reduction shape");
    MCT_REQUIRE(mode == MCT_REDUCE_DOT || mode == MCT_REDUCE_SQDIFF, "invalid reduction mode");
    MCT_CUDA(launch_reduce(a, b, length, segments, stride, mode, out, scratch, (cudaStream_t)stream),
             "reduce");
    return MCT_OK;
}

int mct_axpby(long long n, float alpha, const float* x, float beta, float* y, void* stream) {
    MCT_REQUIRE(x && y && n >= 0, "null argument");
    MCT_CUDA(launch_axpby(n, alpha, x, beta, y, (cudaStream_t)stream), "axpby");
    return MCT_OK;
}

int mct_axpby_mixed(long long n, double alpha, const void* x, int x_is_f64, double beta, void* y,
                    int y_is_f64, void* stream) {
    MCT_REQUIRE(x && y && n >= 0, "null argument");
    MCT_CUDA(launch_axpby_mixed(n, alpha, x, x_is_f64 ? 1 : 0, beta, y, y_is_f64 ? 1 : 0,
                                (cudaStream_t)stream),
             "axpby_mixed");
    return MCT_OK;
}

int mct_dot_f64(const double* a, const double* b, long long n, double* out, double* scratch,
                void* stream) {
    MCT_REQUIRE(a && b && out && n >= 0, "null argument");
    MCT_CUDA(launch_dot_f64(a, b, n, out, scratch, (cudaStream_t)stream), "dot_f64");
    return MCT_OK;
}

// --------------------------------------------------- fused multi-GPU exchange
int mct_exchange_post(void* const* pads, int world, int rank, uint64_t epoch, void* stream) {
    MCT_REQUIRE(pads, "null pad array");
    MCT_REQUIRE(world >= 1 && world <= 1024 && rank >= 0 && rank < world, "invalid world / rank");
    MCT_REQUIRE(epoch >= 1, "epoch must be >= 1");
    MCT_CUDA(launch_exchange_post(reinterpret_cast<unsigned long long* const*>(pads), world, rank,
                                  (unsigned long long)epoch, (cudaStream_t)stream),
             "exchange post");
    return MCT_OK;
}

int mct_exchange_z_update(const float* const* parts, const uint64_t* my_pad, int world,
                          uint64_t epoch, long long n, float* z, float* zbar, double theta,
                          unsigned int* failed, void* stream) {
    MCT_REQUIRE(parts && my_pad && z && zbar && failed, "null argument");
    MCT_REQUIRE(world >= 1 && world <= 1024, "invalid world size");
    MCT_REQUIRE(epoch >= 1 && n >= 0, "epoch must be >= 1 and n >= 0");
    MCT_CUDA(launch_exchange_update(parts, reinterpret_cast<const unsigned long long*>(my_pad),
                                    world, (unsigned long long)epoch, n, z, zbar, (float)theta,
                                    failed, (cudaStream_t)stream),
             "exchange z update");
    return MCT_OK;
}

// ------------------------------------------------------------ data generation
int mct_gaussian_field(uint64_t key0, uint64_t key1, long long count, double scale,
                       const float* base, void* out, int out_is_f64, void* stream) {
    MCT_REQUIRE(count >= 0, "count must be >= 0");
    MCT_REQUIRE(count == 0 || out, "null output");
    MCT_REQUIRE(out_is_f64 == 0 || out_is_f64 == 1, "out_is_f64 must be 0 or 1");
    MCT_CUDA(launch_gaussian_field(key0, key1, count, scale, base, out, out_is_f64,
                                   (cudaStream_t)stream),
             "gaussian field");
    return MCT_OK;
}

}  // extern "C"

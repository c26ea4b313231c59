// Internal types shared by the sm_100a kernels and the C-ABI layer.
//
// Data layout in HBM:
//   image x            : (rows, cols) fp32 row-major
//   padded image X2    : (rows, wx) float2, wx = cols + 2*PADX; element PADX + c of
//                        row r holds (x[r][c], x[r][c+1])  (pair-packed taps)
//   padded transpose XT2: (cols, wxt) float2, wxt = rows + 2*PADX, the same for x^T
//   padded sinogram DY2: (A, wy) float2, wy = B + 2*pb, element pb + j holds
//                        (dy[a][j], dy[a][j+1])
// Pad regions are zero-initialised once (workspace contract) and never written,
// so the Joseph gather loops need no bounds checks.
//
// Gate pairs: every launch of two or more items (PDHG: all gates; C5: a batch of
// slices) shares one ray geometry, so K2 / K3 process items in pairs (2p, 2p+1):
// one fixed-point walk / one set of tent weights drives both items, and one
// 16-byte load fetches both items' pair-packed taps from a pair region in which
// the two items' X2 / XT2 / DY2 are interleaved element by element (float4 =
// (item 2p pair, item 2p+1 pair)).  Single-item regions (single-gate SPDHG,
// standalone operators, an odd last item) and pair regions never overlap and each
// keeps its own zero pads (workspace layout: see mct_item_off below).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <string>
#include <vector>

#include "../../include/mctomo_b200.h"

#define MCT_PADX 4
// image size limit: 32-bit tap indices in K2 / K3 and int32 entries in the transposed
// warp lists (about 4 per pixel)
#define MCT_MAX_PIXELS (1LL << 29)

// ---------------------------------------------------------------- ray plan --
// Forward (ray-driven) per-angle constants.  projector.py:134-155 restated as
// cont(k) = P*s_j + Q + k*slope along the dominant axis k.
struct RayAngle {
    double P, Q, slope;
    long long slope_fx;  // slope * 2^32 (32.32 fixed point increment)
    float step;          // 1/max(|cos|, sin)  (projector.py:143, :154)
    int cols_dom;        // 0: rows-dominant (sample every row), 1: cols-dominant
};

// Adjoint (pixel-driven) per-angle constants: the detector coordinate of pixel
// centre (u, v) is jc = (v*cos - u*sin)/sp + (B-1)/2 and the Joseph weight of
// bin j is step * max(0, 1 - |j - jc| * g) with g = sp*step (tent footprint).
struct AdjAngle {
    double cs, sn;            // cos/sp, sin/sp
    long long csx, snx;       // cos/sp, sin/sp in 32.32 fixed point
    float step, g;
};

// A^* splits its angle loop over up to MCT_MAX_ASPLIT blocks per tile when one
// launch has too few tiles to fill 148 SMs (single-gate SPDHG); each split
// writes its own partial image slot and K4 sums the slots in a fixed order.
// The item workspace holds as many slots as the plan's single-item split.
#ifndef MCT_MAX_ASPLIT
#define MCT_MAX_ASPLIT 16
#endif
#ifndef MCT_ASPLIT_MIN_PAIRS
#define MCT_ASPLIT_MIN_PAIRS 8
#endif

struct WsGeom {
    size_t item_bytes;  // a single region
    size_t pre_bytes;   // A^* IMG slots (prefix of a single region / of a pair block's item)
    size_t pair_bytes;  // interleaved X / XT / DY of a gate pair
    size_t pair_block;  // pair_bytes + 2 * pre_bytes
    int ring;           // pair blocks a workspace holds at most (see mct_pair_off)
};
struct mct_ray_plan {
    int rows, cols, A, B;
    double sp, jmid;     // detector spacing, (B-1)/2
    int wx, wxt;         // padded strides (floats)
    int pb, wy;          // sinogram pad (bins) and padded stride
    int kfoot;           // extra footprint bins for the adjoint (0 when sp >= step^-1)
    RayAngle* d_fwd;
    AdjAngle* d_adj;
    size_t off_x, off_xt, off_dy, off_img, img_slot_bytes, off_part, off_cnt;
    size_t off_px, off_pxt, off_pdy;  // pair region (see top)
    WsGeom wsg;                       // workspace layout (see mct_item_off)
    int ksplit1;  // K2 ray split of single-gate launches (see MCT_KSPLIT_MIN)
    std::vector<double> h_acs, h_asn;  // |cos| / sp, |sin| / sp per angle (host)
    int adj_segw;                      // A^* staged segment length (adj_segw)
};

// K2 may split every ray's sample walk into ksplit consecutive parts handled by
// different blocks (shorter blocks -> better load balance of single-gate SPDHG
// launches); the last block of a tile to finish sums the fp64 partials in part
// order and runs the epilogue.  Single items (mirror walks) of a launch whose
// slices carry one gate each use the plan's ksplit1 (enough parts to fill about one
// wave of resident blocks, clamped to [MCT_KSPLIT_MIN, MCT_KSPLIT_MAX]); gate pairs
// and several gates per slice use 1 (their grids already span many waves), so only
// single regions hold ray-split partials.  A batch of slices therefore agrees with
// single-slice runs to fp32 rounding (mirror walks, ray split, and K3's angle split
// choose_asplit, which follows the launch's tile count), bitwise for A^* whenever the
// splits agree (a plan-constant A^* split costs the 64-slice C5 batch 3.4 %).
#ifndef MCT_KSPLIT_MIN
#define MCT_KSPLIT_MIN 1
#endif
#ifndef MCT_KSPLIT_MAX
#define MCT_KSPLIT_MAX 4
#endif
#ifndef MCT_FWD_ANGLES
#define MCT_FWD_ANGLES 4
#endif
// K2 lane interleave: a warp walks 32 / IL bins of IL consecutive angle slots, lane
// l -> (bin l / IL, slot l % IL), so 8 consecutive lanes span 8 / IL bins x IL nearly
// parallel rays (see fwd_kernel); a block is MCT_FWD_ANGLES warps.
#ifndef MCT_FWD_IL
#define MCT_FWD_IL 2
#endif
// K2 tiles of a geometry: angle-slot groups x bin tiles (grid and arrival counters)
// (single-item launches: MCT_FWD_ANGLES warps per block; gate pairs: MCT_FWD_ANGLES_P
// warps -- their grids span tens of waves, and twice as many half-size blocks per SM
// schedule tighter: C3 K2 1.083 -> 1.072 ms, C4 16.05 -> 15.48 ms)
#ifndef MCT_FWD_ANGLES_P
#define MCT_FWD_ANGLES_P 2
#endif
__host__ __device__ __forceinline__ int mct_fwd_groups(int slots, int warps = MCT_FWD_ANGLES) {
    return (slots + warps * MCT_FWD_IL - 1) / (warps * MCT_FWD_IL);
}
__host__ __device__ __forceinline__ int mct_fwd_btiles(int bins) {
    return (bins + 32 / MCT_FWD_IL - 1) / (32 / MCT_FWD_IL);
}

// Items [0, mct_pair_items(n)) of a launch of n items run the gate-pair kernels
// (consecutive pairs); an odd last item runs the single-item kernels on its own
// region.  MCT_PAIRS=0 disables the pair kernels.
#ifndef MCT_PAIRS
#define MCT_PAIRS 1
#endif
__host__ __device__ __forceinline__ int mct_pair_items(int items) {
    return MCT_PAIRS ? (items & ~1) : 0;
}
// ... a last item that covers only half of the angles is never paired
__host__ __device__ __forceinline__ int mct_pair_items(int items, int last_part) {
    return mct_pair_items(last_part ? items - 1 : items);
}
// Angle-pair range of a half item: part 1 = self-paired angles + pairs q in
// [1, 1 + P/2), part 2 = pairs q in [1 + P/2, P + 1), P = (A-1)/2.
__host__ __device__ __forceinline__ int mct_half_q(int A) { return 1 + ((A - 1) / 2) / 2; }

// Workspace layout (one per launch family; a function of the plan alone, so every
// region keeps one role for every launch size and pads zeroed once stay zero):
//   [single region 0 | single region 1 | pair block 0 .. ring-1 | overflow IMG area]
// A single region (item_bytes) is the full item layout (A^* IMG slots, then the K2
// ray-split partials and arrival counters and the X / XT / DY of the mirror
// kernels) of an unpaired item: unpaired item k of a launch (k = item - pair_items,
// at most two: an odd last item and / or a half item) uses single region k.  Pair
// block p is the interleaved pair region (X / XT / DY of items 2p, 2p+1,
// pair_bytes) followed by the two items' prefixes (pre_bytes: the IMG slots) --
// gate-pair K2 launches never split rays and paired items never touch the
// single-item X / XT / DY, so a pair block holds no copy of them.
// A workspace holds at most `ring` pair blocks (about MCT_RING_BYTES of pair regions,
// >= MCT_RING_MIN_PAIRS).  Launches with more pairs run K1 -> K2 -> K3 chunk by chunk
// of `ring` pairs (mct_items.first_item / item_count): pair p uses the pair region of
// block p % ring, so the X / XT / DY of a chunk are dead before the next chunk
// overwrites them (same elements, pads untouched).  The A^* partial images outlive
// the chunks (K4 gathers all of them): items of pairs >= ring keep theirs in the
// overflow area behind the blocks, item i, split k of a call with angle split s at
// slot (i - 2 ring) * s + k (no pads, rewritten by every call).
#ifndef MCT_RING_BYTES
#define MCT_RING_BYTES (256ull << 20)
#endif
#ifndef MCT_RING_MIN_PAIRS
#define MCT_RING_MIN_PAIRS 4
#endif
__host__ __device__ __forceinline__ size_t mct_pair_off(int pair, const WsGeom& g) {
    return 2 * g.item_bytes + (size_t)(pair % g.ring) * g.pair_block;
}
// Byte offset of item `item`'s region in a launch whose items [0, pair_items) run
// the gate-pair kernels (paired: the pair region).
__host__ __device__ __forceinline__ size_t mct_item_off(int item, int pair_items,
                                                        const WsGeom& g) {
    return item < pair_items ? mct_pair_off(item >> 1, g)
                             : (size_t)(item - pair_items) * g.item_bytes;
}
// Byte offset of item `item`'s first A^* partial-image slot (the call's asplit slots
// follow one another, slot_bytes apart).
__host__ __device__ __forceinline__ size_t mct_img_off(int item, int pair_items, int asplit,
                                                       size_t slot_bytes, const WsGeom& g) {
    if (item >= pair_items) return (size_t)(item - pair_items) * g.item_bytes;
    if (item < 2 * g.ring)  // its pair's own block (pair < ring: no wrap)
        return 2 * g.item_bytes + (size_t)(item >> 1) * g.pair_block + g.pair_bytes +
               (item & 1) * g.pre_bytes;
    return 2 * g.item_bytes + (size_t)g.ring * g.pair_block +
           (size_t)(item - 2 * g.ring) * asplit * slot_bytes;
}
// Workspace bytes for launches of up to `items` items, and the most items one K1-K3
// chunk may hold (ray_kernels.cu).
size_t mct_ws_bytes(const struct mct_ray_plan* rp, int items);
int mct_chunk_items(const struct mct_ray_plan* rp, int items);

// --------------------------------------------------------------- warp plan --
struct WarpDesc {
    int kind;  // MCT_WARP_*
    int rows, cols;
    int pad_;
    double hr, hc;           // (rows-1)/2, (cols-1)/2
    double cs, sn, tr, tc;   // rigid
    double scale;            // dilatation
    const float* phi;        // dense (2, rows, cols)
    const int* tptr;         // transposed gather list of D (rows*cols + 1), all non-identity kinds
    const int* tidx;
    const float* tw;
};

struct mct_warp_plan {
    WarpDesc desc;
    WarpDesc* d_desc;  // device copy of desc
    float* phi;
    int* tptr;
    int* tidx;
    float* tw;
    long long nnz;
};

// ------------------------------------------------------------------ family --
struct GateParam {
    float sigma, dual_inv, theta_over_p, pad_;
};

struct mct_family {
    const mct_ray_plan* ray;
    int S, N;
    WarpDesc* d_warps;   // S*N descriptors
    GateParam* d_params; // N
    int params_set;
};

// ------------------------------------------------------------ item selector --
struct ItemSel {
    const int* gates;
    const int* epoch_ctr;
    int slice_stride, epoch_stride, base, ips, num_slices, iteration, iters_per_epoch;
    int last_part;  // 0, or 1 / 2: the launch's last item covers the first / second half
    int first, count;  // K1-K3 chunk: items [first, first + count) (count 0: to the end)
};

// gate and absolute iteration of item k of slice `slice`
__device__ __forceinline__ void resolve_slice_item(const ItemSel& s, int slice, int k, int& gate,
                                                   int& iter) {
    int e = s.epoch_ctr ? __ldg(s.epoch_ctr) : 0;
    gate = s.gates ? __ldg(s.gates + (long long)slice * s.slice_stride +
                           (long long)e * s.epoch_stride + s.base + k)
                   : 0;
    iter = s.epoch_ctr ? e * s.iters_per_epoch + s.iteration : s.iteration;
}

__device__ __forceinline__ void resolve_item(const ItemSel& s, int item, int& slice, int& gate,
                                             int& iter) {
    slice = item / s.ips;
    int k = item - slice * s.ips;
    int e = s.epoch_ctr ? __ldg(s.epoch_ctr) : 0;
    gate = s.gates ? __ldg(s.gates + (long long)slice * s.slice_stride +
                           (long long)e * s.epoch_stride + s.base + k)
                   : 0;
    iter = s.epoch_ctr ? e * s.iters_per_epoch + s.iteration : s.iteration;
}

// ------------------------------------------------------------ kernel args --
struct PackArgs {
    int rows, cols, wx, wxt;
    char* ws;
    WsGeom wsg;
    size_t off_x, off_xt;
    size_t off_px, off_pxt;
    int pair_items;          // items below this write the interleaved pair region
    ItemSel sel;
    int N;
    const WarpDesc* warps;   // NULL: identity; with sel.gates NULL: warps[0]
    const float* x;          // (slices, rows, cols)
    long long x_slice_stride;
    const float* zbar;       // prox mode when non-NULL
    float tau, cprox;
    float* x_next;           // written by item k==0 of each slice in prox mode
    unsigned long long* status;
};

struct FwdArgs {
    const RayAngle* ang;
    int A, B, rows, cols, wx, wxt;
    double sp, jmid;
    const char* ws;
    WsGeom wsg;
    size_t off_x, off_xt, off_dy, off_part, off_cnt;
    size_t off_px, off_pxt, off_pdy;
    int item0;               // first item of the launch
    int n_items;             // items of the whole call (the last may be a half item)
    int ksplit;
    int wy, pb;
    ItemSel sel;
    int N;
    // plain epilogue
    float* out;
    long long out_item_stride;
    // dual epilogue
    float* y;
    const float* d;
    float* proj;
    const GateParam* gp;
    unsigned long long* status;
};

struct AdjArgs {
    const AdjAngle* ang;
    int A, B, rows, cols, wy, pb;
    double jmid;
    const char* ws;
    WsGeom wsg;
    size_t off_dy, off_img, img_slot_bytes;
    size_t off_pdy;
    int item0;               // first item of the launch
    int n_items, last_part;  // items of the whole call; see ItemSel::last_part
    int first, count;        // K1-K3 chunk, see ItemSel
    int asplit;
    int kfoot;               // adjoint footprint (bins thi-kfoot .. thi+kfoot+1)
    int segw;                // staged sinogram segment length (K = 0, ADJ_TMA)
};

struct UpdArgs {
    int rows, cols;
    const char* ws;
    WsGeom wsg;
    size_t off_img, img_slot_bytes;
    int asplit;
    const float* img_override;  // plain D^* of a caller image (single item)
    ItemSel sel;
    int N;
    const WarpDesc* warps;
    const GateParam* gp;
    float* out;       // mode 0
    float* z;         // mode 1
    float* zbar;
    float* x;
    const float* x_next;
    float* dz;        // mode 2
};

// ------------------------------------------------------------- launchers --
cudaError_t launch_pack(const PackArgs& a, int items, cudaStream_t st);
cudaError_t launch_pad_sino(const float* sino, const mct_ray_plan* rp, char* ws,
                            const WsGeom& wsg, int items, int first, int count, cudaStream_t st);
cudaError_t launch_fwd(const FwdArgs& a, int mode, int items, cudaStream_t st);
cudaError_t launch_adj(const AdjArgs& a, int kfoot, int items, cudaStream_t st);  // a.last_part
int choose_asplit(const mct_ray_plan* rp, int items, int last_part = 0);
int adj_plan_slots(const mct_ray_plan* rp);
int choose_ksplit(int A, int B, int n);
int adj_segw(const mct_ray_plan* rp);
size_t adj_stage_bytes(int G, int segw);
cudaError_t launch_update(const UpdArgs& a, int mode, int slices, cudaStream_t st);
cudaError_t launch_z_update(long long n, const float* dz, float* z, float* zbar, float theta,
                            cudaStream_t st);
cudaError_t launch_epoch_advance(int* ctr, int inc, cudaStream_t st);
cudaError_t launch_warp_fwd_plain(const WarpDesc* d_desc, const float* x, float* out, int rows,
                                  int cols, cudaStream_t st);
cudaError_t launch_reduce(const float* a, const float* b, long long len, int segs,
                          long long stride, int mode, double* out, double* scratch,
                          cudaStream_t st);
cudaError_t launch_axpby(long long n, float alpha, const float* x, float beta, float* y,
                         cudaStream_t st);
cudaError_t launch_axpby_mixed(long long n, double alpha, const void* x, int xf64, double beta,
                               void* y, int yf64, cudaStream_t st);
cudaError_t launch_dot_f64(const double* a, const double* b, long long n, double* out,
                           double* scratch, cudaStream_t st);
cudaError_t launch_absmax(const float* x, long long n, float* out, cudaStream_t st);
cudaError_t build_dense_transpose(const WarpDesc& desc, int** tptr, int** tidx, float** tw,
                                  long long* nnz, cudaStream_t st);

cudaError_t launch_gaussian_field(unsigned long long k0, unsigned long long k1, long long count,
                                  double scale, const float* base, void* out, int out_f64,
                                  cudaStream_t st);

cudaError_t launch_exchange_post(unsigned long long* const* pads, int world, int rank,
                                 unsigned long long epoch, cudaStream_t st);
cudaError_t launch_exchange_update(const float* const* parts, const unsigned long long* my_pad,
                                   int world, unsigned long long epoch, long long n, float* z,
                                   float* zbar, float theta, unsigned int* failed,
                                   cudaStream_t st);

// error reporting (abi.cu)
int mct_set_error(int code, const std::string& msg);

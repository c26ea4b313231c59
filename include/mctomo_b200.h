/*
 * mctomo_b200.h — C-ABI of the B200-native motion-compensated PDHG/SPDHG hot path.
 *
 * This is the drop-in boundary for the reference package `mctomo`
 * (/root/reference/pkg/src/mctomo).  The reference is pure Python/numpy; its
 * "plugin interface" for this path is the `LinearMap` contract
 * (linops.py:39-73: domain_shape / range_shape / apply / adjoint_apply) plus the
 * solver entry points `default_config` / `step` / `run` (solvers.py:198-419).  A
 * Python reference binds native code through ctypes, so every entry point below
 * takes plain pointers and sizes (no torch types); INTEGRATION.md shows the
 * ctypes stub a maintainer of the reference would add.
 *
 * Conventions
 *   - All array pointers named *_dev are DEVICE pointers (fp32 unless noted),
 *     caller-owned, row-major, densely packed unless a stride is given.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Every op is stream-ordered and launch-only (no host sync) unless stated,
 *     so it can be captured in a CUDA graph.
 *   - Return value: MCT_OK (0) or an error code; mct_last_error() returns the
 *     thread-local message.  MCT_ERR_ARG maps to Python ValueError (the
 *     reference's _check_domain / _check_range behaviour, linops.py:59-73),
 *     MCT_ERR_CUDA to RuntimeError.
 *   - Plans are immutable after creation and may be shared read-only by
 *     concurrent calls on distinct outputs (linops.py:12-14, projector.py:190-191).
 */
#ifndef MCTOMO_B200_H
#define MCTOMO_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCT_ABI_VERSION 2

#define MCT_OK 0
#define MCT_ERR_ARG 1
#define MCT_ERR_CUDA 2
#define MCT_ERR_STATE 3

int mct_abi_version(void);
const char* mct_last_error(void);

/* ------------------------------------------------------------------------- */
/* Ray transform A / A^*  (replaces projector.RayTransform, projector.py:186-217)
 *
 * cos_a, sin_a, rows_dominant are HOST arrays of length num_angles computed by
 * the caller exactly as projector._build_tables does (projector.py:127-130:
 * angles = arange(A)*(pi/A); cos, sin; |cos| >= sin).  Detector bin centres
 * follow Geometry.bin_centers (projector.py:75-79).  Images hold at most 2^29
 * pixels (32-bit element offsets, int32 warp-list entries): MCT_ERR_ARG beyond.  */
typedef struct mct_ray_plan mct_ray_plan;

int mct_ray_plan_create(mct_ray_plan** plan, int rows, int cols, int num_angles,
                        int num_bins, double detector_spacing, const double* cos_a,
                        const double* sin_a, const uint8_t* rows_dominant);
int mct_ray_plan_destroy(mct_ray_plan* plan);

/* Bytes of device workspace a standalone forward/adjoint call of up to `batch`
 * items needs: two single-item regions (padded image copies + padded sinogram +
 * image scratch), a ring of interleaved gate-pair regions (launches of >= 2 items
 * process items 2p, 2p+1 together; the ring holds at most about 256 MB, larger
 * batches run through it chunk by chunk inside the call) and backprojection images
 * per item.  A function of the plan and `batch` only; any call of <= `batch` items
 * may use the workspace.  Not linear in `batch`; size with this.              */
size_t mct_ray_workspace_bytes(const mct_ray_plan* plan, int batch);
/* Most gate-pair regions a workspace of this plan holds (default: about 256 MB worth,
 * at least 4).  Fewer regions = less memory, more (smaller) K1-K3 launches per
 * iteration; results do not change.  Call before sizing any workspace.          */
int mct_ray_plan_set_ring_pairs(mct_ray_plan* plan, int pairs);

/* A: x_dev (batch, rows, cols) -> sino_dev (batch, A, B).  projector.py:201-207 */
int mct_ray_forward(const mct_ray_plan* plan, const float* x_dev, float* sino_dev,
                    int batch, void* workspace_dev, void* stream);
/* A^*: sino_dev (batch, A, B) -> img_dev (batch, rows, cols).  projector.py:209-217
 * Deterministic transpose-gather (no atomics).                                 */
int mct_ray_adjoint(const mct_ray_plan* plan, const float* sino_dev, float* img_dev,
                    int batch, void* workspace_dev, void* stream);

/* ------------------------------------------------------------------------- */
/* Warp D_i / D_i^*  (replaces motion.WarpOperator, motion.py:111-194, and adds
 * the dense-field warp the BASELINE configs need, restating motion.py:155-176
 * with src = p + phi(p)).                                                       */
typedef struct mct_warp_plan mct_warp_plan;

#define MCT_WARP_IDENTITY 0
#define MCT_WARP_RIGID 1
#define MCT_WARP_DILATATION 2
#define MCT_WARP_DENSE 3

/* Rigid: rotation (radians) + translation (delta_row, delta_col); cos/sin are
 * evaluated and snapped (|.|<1e-15 -> 0) on the host as motion.py:139-147 does,
 * the caller passes the snapped values.  Dilatation: scale about the centre.    */
int mct_warp_plan_create_rigid(mct_warp_plan** plan, int rows, int cols, double cos_r,
                               double sin_r, double t_row, double t_col);
int mct_warp_plan_create_dilatation(mct_warp_plan** plan, int rows, int cols,
                                    double scale);
int mct_warp_plan_create_identity(mct_warp_plan** plan, int rows, int cols);
/* Dense pull-back displacement phi_dev (2, rows, cols) fp32 in pixels:
 * src(r,c) = (r + phi[0,r,c], c + phi[1,r,c]).  The plan copies phi and builds a
 * deterministic transposed gather list for D^* on the device (synchronous).    */
int mct_warp_plan_create_dense(mct_warp_plan** plan, int rows, int cols,
                               const float* phi_dev, void* stream);
int mct_warp_plan_destroy(mct_warp_plan* plan);
int mct_warp_plan_kind(const mct_warp_plan* plan);
/* number of stored transposed entries (dense plans; 0 otherwise) */
long long mct_warp_plan_nnz(const mct_warp_plan* plan);

/* D: x -> out (rows, cols).  motion.py:178-183 */
int mct_warp_forward(const mct_warp_plan* plan, const float* x_dev, float* out_dev,
                     void* stream);
/* D^*: y -> out (rows, cols).  motion.py:185-194; deterministic gather. */
int mct_warp_adjoint(const mct_warp_plan* plan, const float* y_dev, float* out_dev,
                     void* stream);

/* ------------------------------------------------------------------------- */
/* Gated family: A_i = A o D_i for num_slices x num_gates (slice, gate) pairs
 * (replaces simulate.gate_operators + linops.ComposedMap, simulate.py:172-188,
 * linops.py:105-132).  warps[s*num_gates+g] may be NULL (identity gate, which the
 * reference represents by the bare RayTransform, simulate.py:186-187).          */
typedef struct mct_family mct_family;

int mct_family_create(mct_family** fam, const mct_ray_plan* ray, int num_slices,
                      int num_gates, const mct_warp_plan* const* warps);
int mct_family_destroy(mct_family* fam);

/* Per-gate step parameters of solvers.SolverConfig (solvers.py:127-195):
 * sigmas[g], probs[g], theta.  Dual prox constant uses N = num_gates
 * (functionals.prox_fstar, functionals.py:53-68).  Synchronous upload.         */
int mct_family_set_params(mct_family* fam, const double* sigmas, const double* probs,
                          double theta);

/* Workspace bytes for launches of up to `items` (slice,gate) items (see
 * mct_ray_workspace_bytes).                                                    */
size_t mct_family_workspace_bytes(const mct_family* fam, int items);
/* Most items one K1-K3 chunk of a fused iteration of `items` items may hold (even;
 * == items when every gate pair has its own region): launches with more items run
 * K1 -> K2 -> K3 chunk after chunk (mct_items.first_item / item_count), then K4
 * once.                                                                        */
int mct_family_chunk_items(const mct_family* fam, int items);

/* Standalone gated forward / adjoint of one (slice, gate): A(D x), D^*(A^* y). */
int mct_gated_forward(const mct_family* fam, int slice, int gate, const float* x_dev,
                      float* sino_dev, void* workspace_dev, void* stream);
int mct_gated_adjoint(const mct_family* fam, int slice, int gate, const float* y_dev,
                      float* img_dev, void* workspace_dev, void* stream);

/* The gated forwards of `count` gates of one slice in one pass (two launches):
 * sino_dev[k] = A(D_{gates_dev[k]} x), sino_dev (count, A, B).  The objective of
 * solvers._epoch_objective / Problem.objective (solvers.py:113-119, :422-432)
 * needs every gate's projection; the workspace must hold `count` items.        */
int mct_gated_forward_many(const mct_family* fam, int slice, const int32_t* gates_dev, int count,
                           const float* x_dev, float* sino_dev, void* workspace_dev,
                           void* stream);

/* ------------------------------------------------------------------------- */
/* Fused solver iteration (solvers.step, solvers.py:316-366).
 *
 * Item selection: the iteration processes items_per_slice items for each of
 * num_slices slices; item k of slice s uses gate
 *     gates_dev[s*slice_stride + (epoch_ctr_dev ? *epoch_ctr_dev*epoch_stride : 0)
 *               + base + k].
 * PDHG (solvers.sample_gates "pdhg"): gates_dev = [0..N-1], base = first local
 * gate, items_per_slice = local gate count.  SPDHG: gates_dev = the pre-drawn
 * per-slice sequence (numpy default_rng(seed).choice, solvers.py:312),
 * slice_stride = total iterations, epoch_stride = N, base = iteration in epoch,
 * items_per_slice = 1, epoch_ctr_dev = device epoch counter (graph replay).
 * K1-K4 of one iteration must see the same mct_items (item count): launches of
 * >= 2 items process items 2p, 2p+1 together (gate pairs) in an interleaved
 * workspace region, an odd last item on its own (concurrently, on a library
 * side stream joined back to `stream`); a single item pairs its mirror angles.  */
typedef struct {
    const int32_t* gates_dev;
    const int32_t* epoch_ctr_dev; /* may be NULL */
    int32_t slice_stride;
    int32_t epoch_stride;
    int32_t base;
    int32_t items_per_slice;
    int32_t num_slices;
    int32_t iteration;       /* 1-based iteration number (reported by the divergence
                                flags); with epoch_ctr_dev it is the iteration within
                                the epoch and the absolute number is
                                *epoch_ctr*iters_per_epoch + iteration            */
    int32_t iters_per_epoch;
    int32_t last_part;       /* 0: every item covers all angles; 1 / 2: the last item
                                covers only the first / second half of the angle pairs
                                (half-gate units of gate-sharded PDHG, solvers.py has no
                                counterpart: the partial images sum across ranks)   */
    int32_t first_item;      /* K1-K3 only: this call covers items [first_item,
                                first_item + item_count) of the launch (item_count 0:
                                to the end); first_item a multiple of
                                mct_family_chunk_items, item_count at most that.  K4
                                takes 0 / 0 (it gathers every item).               */
    int32_t item_count;
} mct_items;

/* Solver state buffers (device, fp32), slice-major.
 *   x, x_next, z, zbar : (num_slices, rows, cols)
 *   y, d               : (num_slices, num_gates, A, B)
 *   proj               : optional (num_slices, num_gates, A, B) (PDHG objective reuse,
 *                        solvers.py:427-431) or NULL
 *   status             : device uint64[2], initialised to UINT64_MAX:
 *                        [0] first iteration with a non-finite primal iterate,
 *                        [1] (iteration << 20 | gate) of the first non-finite dual
 *                        (solvers.py:330-333, :350-353).                         */
typedef struct {
    float* x;
    float* x_next;
    float* z;
    float* zbar;
    float* y;
    const float* d;
    float* proj;
    unsigned long long* status;
} mct_state;

/* K1: x_next = prox_g(x - tau*zbar) (functionals.py:40-50) fused with the warp
 * D_i x_next written into the projector's padded layouts in the workspace.      */
int mct_iter_prox_warp(const mct_family* fam, const mct_items* items, mct_state* st,
                       double tau, double alpha, void* workspace_dev, void* stream);
/* K2: A(D_i x_next) fused with the dual prox (functionals.py:53-68):
 * y_i <- (y_i + sigma_i*A_i x - sigma_i*d_i)/(1+sigma_i*N/2); dy_i -> workspace. */
int mct_iter_forward_dual(const mct_family* fam, const mct_items* items, mct_state* st,
                          void* workspace_dev, void* stream);
/* K3: A^* dy_i -> workspace image (transpose-gather).                          */
int mct_iter_adjoint(const mct_family* fam, const mct_items* items, void* workspace_dev,
                     void* stream);
/* K4: dz = sum_i D_i^* (A^* dy_i); z += dz; zbar = z + sum_i (theta/p_i) D_i^*(...);
 * x = x_next (solvers.py:358-363).  If dz_partial_dev is non-NULL the z/zbar
 * update is skipped and the local sum is written there instead (gate-sharded
 * PDHG, reduced across GPUs by the caller, then finished by mct_iter_z_update). */
int mct_iter_adjoint_update(const mct_family* fam, const mct_items* items, mct_state* st,
                            float* dz_partial_dev, void* workspace_dev, void* stream);
/* z += dz; zbar = z + theta*dz (all p_i = 1 in PDHG mode).                      */
int mct_iter_z_update(const mct_family* fam, mct_state* st, const float* dz_dev,
                      double theta, void* stream);
/* ++(*epoch_ctr_dev) (one-thread kernel, for epoch graphs).                    */
int mct_epoch_advance(int32_t* epoch_ctr_dev, int32_t increment, void* stream);

/* ------------------------------------------------------------------------- */
/* Deterministic reductions (fixed order, fp64 accumulation) for diagnostics,
 * power iteration and the divergence guard (linops.py:262-263,
 * functionals.py:71-82, solvers.py:289-295, experiment_io.py:294-301).
 * out_dev[s] = sum_i a[s*stride+i]*b[s*stride+i]          (mode 0, dot)
 * out_dev[s] = sum_i (a[s*stride+i]-b[s*stride+i])^2      (mode 1; b NULL -> a^2) */
#define MCT_REDUCE_DOT 0
#define MCT_REDUCE_SQDIFF 1
/* scratch_dev (optional, >= segments*MCT_REDUCE_PARTS doubles) enables the
 * two-pass multi-block reduction (same fixed order, still bitwise reproducible);
 * with NULL one block per segment does all the work.                          */
#define MCT_REDUCE_PARTS 128
int mct_reduce(const float* a_dev, const float* b_dev, long long length, int segments,
               long long stride, int mode, double* out_dev, double* scratch_dev, void* stream);

/* y = alpha*x + beta*y elementwise (fp32; used by the device power iteration). */
int mct_axpby(long long n, float alpha, const float* x_dev, float beta, float* y_dev,
              void* stream);

/* Mixed-precision vector ops for the device CG saddle-point solver
 * (solvers.cg_reference, solvers.py:435-490, GramSumMap linops.py:172-212):
 * y = alpha*x + beta*y with x, y each fp32 (flag 0) or fp64 (flag 1), fp64
 * arithmetic; out_dev[0] = sum_i a[i]*b[i] over fp64 vectors (fixed order).   */
int mct_axpby_mixed(long long n, double alpha, const void* x_dev, int x_is_f64, double beta,
                    void* y_dev, int y_is_f64, void* stream);
int mct_dot_f64(const double* a_dev, const double* b_dev, long long n, double* out_dev,
                double* scratch_dev, void* stream);

/* --------------------------------------------- fused multi-GPU exchange */
/* Gate-sharded PDHG without a collective library: the partial
 * dz_r = sum_{i in gates(r)} D_i^* A_i^* dy_i that mct_iter_adjoint_update
 * (dz_partial) wrote into this rank's peer-visible buffer is combined over
 * NVLink peer memory inside the z / z-bar update (solvers.py:356-366).
 *   pads_dev  : device array of `world` pointers, pads_dev[q] = rank q's signal
 *               pad (world uint64 slots, zeroed before the first epoch; slot r
 *               holds the last epoch rank r posted);
 *   parts_dev : device array of `world` pointers to the ranks' partial buffers
 *               of this epoch's parity (n floats each).
 * mct_exchange_post publishes this rank's partial for `epoch` (>= 1, strictly
 * increasing); mct_exchange_z_update waits for every rank's post of `epoch`
 * and applies z += sum_q parts[q], zbar = z + theta * sum_q parts[q], summing
 * in rank order (the same bits on every rank).  The wait is bounded: on expiry
 * *failed_dev is set to 1 and z / zbar are left untouched.                    */
int mct_exchange_post(void* const* pads_dev, int world, int rank, uint64_t epoch, void* stream);
int mct_exchange_z_update(const float* const* parts_dev, const uint64_t* my_pad_dev, int world,
                          uint64_t epoch, long long n, float* z_dev, float* zbar_dev, double theta,
                          unsigned int* failed_dev, void* stream);

/* ------------------------------------------------------------ data generation */
/* Seeded Gaussian sinogram noise on the device, the documented recipe of
 * simulate.gaussian_field (simulate.py:113-133) used by simulate.generate
 * (simulate.py:191-239): numpy's Philox4x64-10 stream keyed
 * (key0 = master_seed mod 2^64, key1 = gate_index), uniforms u1 then u2
 * (ceil(count/2) each, bit-identical to numpy), Box-Muller pairs.
 * out[i] = (base ? base[i] : 0) + scale * z_i in fp64 arithmetic, stored fp64
 * (out_is_f64 = 1) or rounded to fp32.  count = 0 is a no-op.                 */
int mct_gaussian_field(uint64_t key0, uint64_t key1, long long count, double scale,
                       const float* base_dev, void* out_dev, int out_is_f64, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MCTOMO_B200_H */

/*
 * sos_b200.h -- C ABI of the B200 (sm_100a) SOS loss-and-gradient path.
 *
 * The method (PAPER.md = arxiv 2410.19844 text, cited by line):
 *   A form p of degree 2d in n variables is fitted by p ~ sum_k q_k^2 with
 *   q_k = m_d . v_k, i.e. p = m_d V V^T m_d^T (PAPER.md:45-48,
 *   Eq. 1 with B = V V^T), by minimising the squared coefficient distance
 *   L(V) = || coef(m_d V V^T m_d^T) - p ||^2            (Eq. 2)
 *   with a first-order method ("basic ADAM approach").
 *   m_d holds the N = C(n+d-1, d) degree-d monomials; the
 *   target has M = C(n+2d-1, 2d) coefficients.
 *
 * Conventions (all entry points):
 *   - Monomial order: colex order of the sorted variable-index multiset,
 *     i.e. the combinatorial number system: the multiset m_1<=...<=m_D has
 *     rank sum_k C(m_k + k - 1, k).  For n=d=2 this is (x1^2, x1x2, x2^2),
 *     the order of PAPER.md:53.
 *   - V is N x r, fp32, row-major (row i = monomial alpha_i, column k = square k).
 *   - Coefficient vectors (coef, p, residual) are length M, fp32, in the
 *     degree-2d colex order.
 *   - Pointers named *_dev are CUDA device pointers; *_host are host pointers.
 *     The library never takes ownership of caller buffers.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Calls are asynchronous on that stream unless stated otherwise.
 *   - Every call returns SOS_OK (0) or an error code; sos_last_error() gives a
 *     thread-local message.  On error no output is guaranteed to be written.
 *   - Requires a compute-capability 10.0 device (B200); there is no CPU path:
 *     without one every compute call returns SOS_ERR_DEVICE.
 *   - Indexes and plans belong to the device that is current when they are
 *     created; calls must be made with that device current.  Kernel launch
 *     configurations (occupancy-derived grids, shared-memory attributes) are
 *     cached once per process, so a process drives one device (bench.py runs
 *     one process per GPU).
 *   - Not thread-safe per plan: calls on one plan must not overlap; distinct
 *     plans may be used from distinct host threads.
 */
#ifndef SOS_B200_H
#define SOS_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SOS_OK 0
#define SOS_ERR_ARG 1    /* invalid argument (sizes, null pointers, n/d out of range) */
#define SOS_ERR_CUDA 2   /* CUDA runtime error; message in sos_last_error() */
#define SOS_ERR_NOMEM 3  /* device allocation failed */
#define SOS_ERR_DEVICE 4 /* no sm_100 device visible */

typedef struct sos_index sos_index; /* monomial tables + pair-rank table (device) */
typedef struct sos_plan sos_plan;   /* per-(index, r) workspaces and optimiser state */

/* Thread-local description of the last error ("" if none). */
const char *sos_last_error(void);

/* ABI version (increments on incompatible change; 2: sos_plan_create_ex). */
int sos_version(void);

/* ------------------------------------------------------------------------
 * Index (the degree-d basis m_d and the degree-2d basis).
 * ------------------------------------------------------------------------ */

/* Build the index for n variables and half-degree d on the current device:
 * the colex-ordered exponent table of the N degree-d monomials, and the table
 * rank(alpha_i + alpha_j) in the degree-2d basis for every ordered pair (i,j),
 * computed by the combinatorial number system.  Synchronous.
 * Limits: 1 <= n, 1 <= d <= 32, n + 2d <= 255, M < 2^32 - 1, N <= 65536.
 * Device memory: about 2*Np^2 bytes (Np = N rounded up to 256): the pair-rank
 * table is stored for one triangle of 64 x 64 blocks (it is symmetric). */
int sos_build_index(int n, int d, sos_index **out);
int sos_index_destroy(sos_index *idx);

/* N (degree-d monomials) and M (degree-2d coefficients). */
int sos_index_dims(const sos_index *idx, int64_t *N, int64_t *M);

/* Copy the degree-d exponent table (N x n, uint8, row-major) to alpha_dev. */
int sos_index_alpha(const sos_index *idx, uint8_t *alpha_dev, void *stream);

/* Write the degree-2d exponent table (M x n, uint8, row-major) to beta_dev
 * (computed on the device by colex unranking). */
int sos_index_beta(const sos_index *idx, uint8_t *beta_dev, void *stream);

/* out_dev[t] = rank(alpha_{i_dev[t]} + alpha_{j_dev[t]}) read from the stored
 * pair-rank table, t < count; 0 <= i,j < N (else SOS_ERR_ARG is NOT detected on
 * device: out-of-range pairs yield 0xFFFFFFFF). */
int sos_index_pair_ranks(const sos_index *idx, const int64_t *i_dev, const int64_t *j_dev,
                         int64_t count, uint32_t *out_dev, void *stream);

/* ------------------------------------------------------------------------
 * Plan: workspaces for one (index, r).  Device memory ~ 3*Np*(2*r + Np) bytes
 * (int8 slices of V, V^T and R) plus 8*N*r once Adam is enabled, plus 4*N*r
 * (a gradient buffer) for the split pipeline (default when N <= 3008: short K),
 * plus a second V^T slice buffer on the first sos_descend call when the update
 * writes the next step's V^T slices (default when N > 8128).
 * ------------------------------------------------------------------------ */
int sos_plan_create(const sos_index *idx, int64_t r, sos_plan **out);

/* Implementation choices of a plan.  Every field is -1 (the
 * library picks by problem size, the default of sos_plan_create) or 0 / 1.
 * All variants compute the same step; they differ in how it is scheduled and
 * agree to fp32 rounding (tests/test_gpu_variants.py).  Nothing else -- no
 * environment variable -- changes what a plan computes.
 *   split:        1 = "split" step: forward, one cooperative kernel (residual,
 *                 loss, R maxima, V^T and R slices), backward storing the
 *                 gradient, one row-block update kernel (4 launches; default
 *                 for short K, N <= 3008); 0 = the update runs in the
 *                 backward's epilogue warps.
 *   vtq_from_update (split = 0, sos_descend): the update also writes the next
 *                 step's V^T slices (default for N > 8128).
 *   vtq_in_aux:   the forward's two aux warps write the V^T slices (default
 *                 when they hide under its MMAs) instead of a separate kernel.
 *   rmax_direct:  R row maxima by one gather pass over the pair-rank table
 *                 instead of the monomial-lattice DP (default by a cost model).
 *   narrow_tiles: tiles narrower than 160 columns where a column block is
 *                 partly outside the matrix (default 1).
 *   tile_w:       column tile width of the GEMMs, -1 or 0 = auto (160, or
 *                 narrower for small problems where it saves a partial wave),
 *                 else a multiple of 16 in [16, 160]; the backward uses it
 *                 only in split plans.
 *   r_headroom:   (split = 0, sos_descend) after the first step of a call the R
 *                 slices use 2x the previous step's exact R row maxima; the
 *                 packer takes this step's exact maxima on the fly and re-slices
 *                 the rare rows outside the window (default 1); 0 = exact row
 *                 maxima every step (lattice DP or direct pass).
 *   tiny:         sos_descend (and sos_solve_host) run all their steps in ONE
 *                 cooperative kernel of fp32 CUDA-core tiles with grid barriers
 *                 between forward, residual, backward and update (default for
 *                 small problems, N^2 r <= 2e7, e.g. N = r <= 271); other
 *                 calls are unchanged. */
typedef struct {
    int split;
    int vtq_from_update;
    int vtq_in_aux;
    int rmax_direct;
    int narrow_tiles;
    int tile_w;
    int r_headroom;
    int tiny;
} sos_plan_opts;
int sos_plan_create_ex(const sos_index *idx, int64_t r, const sos_plan_opts *opts, sos_plan **out);
int sos_plan_destroy(sos_plan *plan);

/* Number of kernels this library launched through `plan` so far. */
int64_t sos_plan_launch_count(const sos_plan *plan);

/* Per-kernel device timing of the launches made through `plan`: when enabled,
 * every kernel is bracketed by CUDA events recorded on its launch stream.
 * sos_plan_timing(plan, 1) clears previous records and starts recording;
 * sos_plan_timing(plan, 0) stops.  sos_plan_timing_read synchronises on the
 * recorded events and returns the summed duration (ms) and launch count of
 * kernel kind `kernel` (SOS_KERNEL_*). */
#define SOS_KERNEL_VMAX 0     /* row and column maxima of V (slice scales) */
#define SOS_KERNEL_PACK_V 1   /* int8 slices of V (and of V^T in sos_backward) */
#define SOS_KERNEL_GEMM_FWD 2 /* Gram tiles + coefficient scatter (tensor cores) */
#define SOS_KERNEL_RESIDUAL 3 /* res = coef - p, loss */
#define SOS_KERNEL_RMAX 4     /* row maxima of R (lattice DP or direct pass) */
#define SOS_KERNEL_PACK_R 5   /* R gathered through the pair-rank table into int8 slices */
#define SOS_KERNEL_GEMM_BWD 6 /* 4 R V (tensor cores), in sos_step with the optimiser update */
#define SOS_KERNEL_UPDATE 7   /* step bookkeeping (Adam t, loss record); the split step's row-block update
                                 (otherwise the update runs inside GEMM_BWD) */
#define SOS_KERNEL_MID 8      /* the split step's cooperative kernel: residual, loss, R maxima, V^T and R slices */
#define SOS_KERNEL_TINY 9     /* a tiny plan's whole sos_descend call (one cooperative kernel) */
#define SOS_KERNEL_COUNT 10
int sos_plan_timing(sos_plan *plan, int enable);
int sos_plan_timing_read(sos_plan *plan, int kernel, double *total_ms, int64_t *launches);

/* coef_dev[M] = coefficients of m_d V V^T m_d^T (PAPER.md:45-48 with B = V V^T):
 * coef_beta = sum over ordered pairs (i,j) with alpha_i + alpha_j = beta of
 * <V_i, V_j>.  Computed on tensor cores with fp32-class accuracy: each row of V
 * is split into three int8 slices against its own maximum (about 23 bits), the
 * six leading slice products accumulate exactly in s32, and the Gram tiles are
 * reduced into coef in the GEMM epilogue (the N x N matrix never reaches HBM).
 * Relative L2 error vs exact arithmetic is about 1e-7 (bar: 1e-5). */
int sos_forward(sos_plan *plan, const float *V_dev, float *coef_dev, void *stream);

/* grad_dev[N x r] = 4 R V with R_ij = res[rank(alpha_i + alpha_j)]: the
 * gradient of Eq. 2 for residual res = coef - p (length M). */
int sos_backward(sos_plan *plan, const float *V_dev, const float *res_dev, float *grad_dev,
                 void *stream);

/* loss_dev[0] = ||coef(V) - p||^2 (fp64), grad_dev = dL/dV = 4 R V.
 * grad_dev may be NULL (loss only).  res_dev, if not NULL, receives coef - p. */
int sos_loss_grad(sos_plan *plan, const float *V_dev, const float *p_dev, double *loss_dev,
                  float *grad_dev, float *res_dev, void *stream);

/* ------------------------------------------------------------------------
 * First-order optimiser ("basic ADAM approach"; plain GD).
 * ------------------------------------------------------------------------ */
#define SOS_OPT_GD 0
#define SOS_OPT_ADAM 1
typedef struct {
    int kind;     /* SOS_OPT_GD or SOS_OPT_ADAM */
    float lr;     /* step size */
    float beta1;  /* Adam only */
    float beta2;  /* Adam only */
    float eps;    /* Adam only */
} sos_opt_params;

/* Reset the optimiser: zero the Adam moments, step counter t = 0. */
int sos_opt_init(sos_plan *plan, const sos_opt_params *params, void *stream);

/* Change the learning rate of an initialised optimiser without touching its
 * state (Adam moments and step count t are kept): a step-size schedule for the
 * descent of PAPER.md:221.  lr must be > 0.  Host-only; takes effect from the
 * next sos_step. */
int sos_opt_set_lr(sos_plan *plan, float lr);

/* Stopping rule of the descent, decided ON THE DEVICE (no host sync): once the
 * current V meets  ||coef(V V^T) - p||^2 <= rel_tol * ||p||^2  (Eq. 2 relative
 * to the target's norm, reading R2), sos_step still evaluates the
 * loss but skips the backward and the update, so V and the optimiser state stay
 * at the first iterate that met the tolerance.  rel_tol <= 0 disables the rule
 * (the default after sos_opt_init).  Host-only setter. */
int sos_opt_set_stop(sos_plan *plan, double rel_tol);

/* One descent step, in place on V_dev:  loss_dev[0] = L(V) (before the update),
 * then V <- V - lr*g (GD) or the bias-corrected Adam update with t += 1:
 *   m <- b1 m + (1-b1) g,  v <- b2 v + (1-b2) g^2,
 *   V <- V - lr (m / (1-b1^t)) / (sqrt(v / (1-b2^t)) + eps).
 * The update runs inside the backward GEMM (the gradient never reaches HBM), or
 * for split plans in a row-block kernel after it.  V_dev must be 16-byte
 * aligned (SOS_ERR_ARG otherwise).  With a stopping tolerance set
 * (sos_opt_set_stop) and met, V is left unchanged. */
int sos_step(sos_plan *plan, float *V_dev, const float *p_dev, double *loss_dev, void *stream);

/* `steps` descent steps in one call, in place on V_dev: losses_dev[t] = L(V_t)
 * (fp64, device) before update t.  Same iteration as `steps` calls of sos_step,
 * faster because the library owns V between the steps: the backward of step t
 * also writes the int8 slices and the exact row / column maxima of V_{t+1}
 * (slices scaled by 2x the row maximum of V_t; rows whose new maximum leaves
 * [1/2, 2] of the old one are re-sliced exactly before the next forward), so
 * the per-step maxima and slicing passes over V disappear (split plans: exact
 * new row maxima, no re-slicing).  V_dev must be 16-byte aligned.  Results agree with
 * sos_step to the slice precision (~1e-7 relative), not bit for bit.  V_dev must
 * not be modified by anyone else during the call (it is asynchronous on
 * `stream`).  Honours sos_opt_set_lr / sos_opt_set_stop settings.  For long K
 * (N > 8128 monomials) the update also writes the next step's V^T slices,
 * into a second V^T slice buffer (3 * r' * N' bytes, r' = r rounded up to 160,
 * N' = N rounded up to 64) the plan allocates on the first call. */
int sos_descend(sos_plan *plan, float *V_dev, const float *p_dev, int64_t steps, double *losses_dev,
                void *stream);

/* Host-buffer entry point: copies p_host (M) and V_host (N x r) to the device,
 * runs sos_descend for `steps` steps, copies V back to V_host and the per-step
 * losses (steps values, fp64) to losses_host.  Synchronous (legacy default
 * stream).  Uses the plan's optimiser settings (sos_opt_init must have been
 * called).  The device staging buffers (4*N*r + 4*M + 8*steps bytes) are kept by
 * the plan between calls; page-locked host buffers give full copy bandwidth.
 * V comes back in row chunks (one per 8 x 256-row tile group) on a second
 * stream while the last step's backward is still updating later rows: the
 * update releases a chunk (device counter + cuStreamWaitValue32) once all its
 * tiles are stored; without stream memory operations, one copy at the end. */
int sos_solve_host(sos_plan *plan, float *V_host, const float *p_host, int64_t steps,
                   double *losses_host);

#ifdef __cplusplus
}
#endif
#endif /* SOS_B200_H */

/*
 * momentcp_b200 -- C ABI of the B200-native implicit moment-tensor CP f+grad path.
 *
 * This is the drop-in boundary: plain pointers, sizes and status codes, no torch
 * types.  Each entry point replaces one call site of the reference Python package
 * `momentcp` (paths relative to the reference root):
 *
 *   mcp_load_obs         ObservationSet.__post_init__         pkg/src/momentcp/dense.py:81-111
 *                        (V upload; fp32 is kept fp32 on device, converted exactly in-register)
 *   mcp_fg               fg_implicit                          pkg/src/momentcp/objective.py:77-94
 *                        (= ttsv_batch :94-107 + _finish objective.py:51-56 on device)
 *   mcp_fg_packed        packed_fg_implicit's fg(x) closure   pkg/src/momentcp/optimize.py:123-134
 *                        (x = [lam; vec_F(A)], g likewise -- optimize.py:104-120)
 *   mcp_ttsv_batch       ttsv_batch                           pkg/src/momentcp/implicit.py:94-107
 *   mcp_data_norm_sq     data_norm_sq                         pkg/src/momentcp/implicit.py:116-121
 *   mcp_fg_partial_device / mcp_fg_finish_device
 *                        the same evaluation split at the additive [Y | w] boundary so a
 *                        row-sharded ObservationSet can all-reduce between them (no reference
 *                        counterpart: the reference is single-process).
 *
 * Error behaviour mirrors the reference: argument errors (d < 2, shape mismatch, non-finite
 * inputs) return MCP_ERR_ARG, which the Python host raises as ValueError exactly where the
 * reference raises it; CUDA failures return MCP_ERR_CUDA (RuntimeError).  The message is
 * available from mcp_last_error(ctx) (or mcp_last_error(NULL) for a failed mcp_create).
 *
 * Threading: every call on a context is serialised by a per-context mutex, so concurrent
 * callers (momentcp.multistart(threads>1), optimize.py:484-493) are safe; all reductions are
 * fixed-order, so results are bitwise reproducible run to run and independent of threading.
 */
#ifndef MOMENTCP_B200_H
#define MOMENTCP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MCP_ABI_VERSION 1

/* status codes */
#define MCP_OK 0
#define MCP_ERR_ARG 1   /* invalid argument: Python raises ValueError   */
#define MCP_ERR_CUDA 2  /* CUDA/driver failure: Python raises RuntimeError */
#define MCP_ERR_STATE 3 /* call out of order (e.g. fg before load_obs)   */

/* element type of V as handed to mcp_load_obs */
#define MCP_F64 0
#define MCP_F32 1

/* host layout of V: VAR_MAJOR = reference ObservationSet.V (n x p, C order, row i = variable i,
 * leading dimension ld >= p); OBS_MAJOR = p x n C order (observation l contiguous, ld >= n). */
#define MCP_VAR_MAJOR 0
#define MCP_OBS_MAJOR 1

/* arithmetic mode */
#define MCP_MODE_FP64 0   /* bit-faithful mode: IEEE fp64 arithmetic, fixed-order reductions */
#define MCP_MODE_TF32X3 1 /* fast mode: 3xTF32 split on tcgen05, fp64 across tiles (<= 1e-4) */

typedef struct mcp_ctx mcp_ctx;

int mcp_abi_version(void);

/* Last error message of ctx, or of the calling thread's last failed mcp_create if ctx==NULL. */
const char* mcp_last_error(const mcp_ctx* ctx);

/* Create a context bound to CUDA device `device` (one context per GPU / rank). */
int mcp_create(mcp_ctx** out, int device);
int mcp_destroy(mcp_ctx* ctx);

/* Number of SMs of the bound device (the persistent-grid width the kernels use). */
int mcp_device_sms(const mcp_ctx* ctx);

/*
 * Upload the observation matrix (host memory).  n variables, p observations.
 * nu: p strictly positive weights, or NULL for uniform weights equal to nu_const
 * (nu_const <= 0 means 1/p, the reference default dense.py:90-91; a row shard of a larger
 * set passes 1/p_total).  Validation matches dense.py:83-105 (finite V, positive finite nu).
 */
int mcp_load_obs(mcp_ctx* ctx, const void* V, int dtype, int layout, int64_t n, int64_t p,
                 int64_t ld, const double* nu, double nu_const);

/* Same, from device memory on the context's device (e.g. data generated on the GPU). */
int mcp_load_obs_device(mcp_ctx* ctx, const void* dV, int dtype, int layout, int64_t n,
                        int64_t p, int64_t ld, const double* dnu, double nu_const);

/* Shape of the loaded observation set. */
int mcp_obs_shape(const mcp_ctx* ctx, int64_t* n, int64_t* p);

/*
 * One f+grad evaluation at (lam, A), host buffers.  A and g_A are n x r column-major
 * (Fortran order, the reference's packed layout).  alpha only shifts f.
 */
int mcp_fg(mcp_ctx* ctx, int d, int r, const double* lam, const double* A_colmajor, double alpha,
           int mode, double* f, double* g_lam, double* g_A_colmajor);

/* Packed form: x = [lam (r); vec_F(A) (n*r)], g the same layout (optimize.py:104-134). */
int mcp_fg_packed(mcp_ctx* ctx, int d, int r, const double* x, double alpha, int mode, double* f,
                  double* g);

/*
 * Batched evaluation of k starting points in ONE pass over V (SURVEY.md 8f "batched multistart";
 * the reference runs multistart's starts one by one, optimize.py:454-508).  X is k x (r + n r),
 * row s = the packed point of start s; F[s] and G row s are its f and packed gradient.  Y and w
 * depend on each factor column alone, so the k*r columns share K1; the tails run per start.
 */
int mcp_fg_batch(mcp_ctx* ctx, int d, int r, int k, const double* X, double alpha, int mode,
                 double* F, double* G);

/* Y = V diag(nu) (V^T A)^(d-1), n x r column-major (implicit.py:94-107). */
int mcp_ttsv_batch(mcp_ctx* ctx, int d, int r, const double* A_colmajor, int mode,
                   double* Y_colmajor);

/* ||X||^2 = nu^T (V^T V)^d nu (implicit.py:116-121), without the p x p Gram. */
int mcp_data_norm_sq(mcp_ctx* ctx, int d, int mode, double* out);

/* Part `part` of `nparts` of the symmetric tile-pair sum of ||X||^2 (multi-GPU split). */
int mcp_data_norm_sq_part(mcp_ctx* ctx, int d, int mode, int part, int nparts, double* out);

/*
 * Sharded ||X||^2 (implicit.py:116-121 over a row-sharded set): part `part` of
 * `nparts` of 2 * sum_{l in ctx's rows, l' in shard J} nu_l nu_l' (v_l^T v_l')^d, i.e. both
 * off-diagonal blocks (I, J) and (J, I) of the Gram.  Shard J is device memory in ctx's own
 * layout (p_pad_J rows of ctx's pitch and dtype, zero padded, p_pad_J a multiple of 128: a peer
 * rank's buffer received over NVLink); dnuJ its weights (NULL: uniform nu_const_J).
 * pair_order 0 lists the rectangle's 128 x 128 tile pairs with ctx's tiles outer, 1 with shard
 * J's tiles outer, so two ranks that share one shard pair can each take half of it
 * (part 0 of 2 in order 0 on one side, part 1 of 2 in order 1 on the other).
 */
int mcp_data_norm_sq_cross(mcp_ctx* ctx, const void* dVJ, int64_t p_pad_J, const double* dnuJ,
                           double nu_const_J, int d, int mode, int pair_order, int part,
                           int nparts, double* out);

/* The resident observation buffer (device pointer, pitch and padded rows in elements, dtype,
 * weights or NULL + the uniform weight): what a peer needs to run mcp_data_norm_sq_cross
 * against this shard. */
int mcp_obs_device_view(const mcp_ctx* ctx, void** dV, int64_t* ldv, int64_t* p_pad, int* dtype,
                        const double** dnu, double* nu_const);

/*
 * Device-resident pieces (all pointers are device memory on ctx's device; stream may be NULL
 * for the context's own stream).
 *   dx   : [lam (r); vec_F(A) (n*r)]
 *   dYw  : [vec_F(Y) (n*r); w (r)]  additive over row shards -> all-reduce(sum) between calls
 *   dout : [f (1); g_lam (r); vec_F(g_A) (n*r)]
 */
int mcp_fg_partial_device(mcp_ctx* ctx, int d, int r, const double* dx, int mode, double* dYw,
                          void* stream);
int mcp_fg_finish_device(mcp_ctx* ctx, int d, int r, const double* dx, const double* dYw,
                         double alpha, double* dout, void* stream);
/* partial + finish in one call (single-GPU device-resident evaluation). */
int mcp_fg_device(mcp_ctx* ctx, int d, int r, const double* dx, double alpha, int mode,
                  double* dout, void* stream);

/*
 * Kernel-level timing (bench.py's roofline): while enabled, every K1 / K5 launch issued outside
 * graph capture is bracketed by CUDA events on its own stream.  mcp_kernel_time_ms waits for
 * them and returns the summed duration and launch count (reset != 0 clears the record).
 */
int mcp_set_kernel_timing(mcp_ctx* ctx, int enable);   /* enable > 1: time every enable-th launch */

/*
 * Per-context run-time options (the library reads no environment variables; kernel and
 * schedule choices are compile-time, csrc/tuning.h).
 *   MCP_OPT_FUSED_TAIL (default 1): end eligible FP64 evaluations with the one-kernel
 *     reduce+finish (K3F); 0 runs the separate reduce and tail kernels (bitwise-equal results;
 *     the tests compare the two).  No reference counterpart (an implementation choice).
 *   MCP_OPT_SMALL_KERNEL (default 1): evaluate small problems (config 1, mini-batches) with the
 *     single-launch kernel K1Z; 0 runs the general K1 -> reduce+finish chain (results agree to
 *     fp64 reassociation; the tests compare the two).  No reference counterpart.
 */
#define MCP_OPT_FUSED_TAIL 1
#define MCP_OPT_SMALL_KERNEL 2
int mcp_set_option(mcp_ctx* ctx, int key, int64_t value);
int mcp_kernel_time_ms(mcp_ctx* ctx, double* total_ms, int* launches, int reset);

/*
 * Device-resident L-BFGS replacing lbfgs_minimize / two_loop_direction /
 * _wolfe_line_search (reference pkg/src/momentcp/optimize.py:149-355) for the objective
 * x -> fg(x) of the loaded observation set.  x, g, the direction and the (s, y) history stay in
 * HBM; the two-loop recursion, trial points and step bookkeeping run as kernels, and the host
 * only receives the handful of scalars the line-search decisions need (one graph launch + one
 * sync per function evaluation).  Decisions follow the reference in the same order; dot products
 * are fixed-order device reductions (deterministic, not numpy's summation order).
 *   x0 (host, r + n r)            starting point, packed as in mcp_fg_packed
 *   opts[7] = {memory, pgtol, max_iters, max_total_iters, c1 (sufficient decrease),
 *              c2 (curvature), max_line_steps}   (OptConfig, optimize.py:31-48)
 *   x_out, g_out (host, r + n r)  final iterate and its gradient; f_out its objective
 *   trace_f / trace_t (host, trace_cap)  f and seconds-since-start at x0 and every accepted step
 *   info[4] = {n_fg, n_steps, reason (0 tolerance, 1 iteration cap, 2 line-search failure),
 *              trace rows written}
 *   hook (may be NULL): called with a host copy of every accepted iterate (and x0).
 * MCP_ERR_ARG with "objective is not finite at the starting point" when fg(x0) is not finite.
 */
typedef void (*mcp_iterate_hook)(const double* x, int64_t len, void* user);
int mcp_lbfgs(mcp_ctx* ctx, int d, int r, double alpha, int mode, const double* x0,
              const double* opts, double* x_out, double* g_out, double* f_out, double* trace_f,
              double* trace_t, int64_t trace_cap, int64_t* info, mcp_iterate_hook hook,
              void* hook_user);

/*
 * k L-BFGS solves in lock step (the multistart of optimize.py:454-508 with
 * every start's evaluation sharing ONE pass over V per round).  X0 is k x (r + n r), row s = start
 * s; opts as mcp_lbfgs.  Per run s: X_out/G_out row s, F_out[s], trace_f/trace_t row s (trace_cap
 * each), info[4 s .. 4 s + 3] = {n_fg, n_steps, reason (0 tolerance, 1 iteration cap,
 * 2 line-search failure, 3 error), trace rows}.  Runs with reason 3 are described by
 * mcp_lbfgs_batch_errors() (one "run s: message" line each); the others are unaffected.
 */
int mcp_lbfgs_batch(mcp_ctx* ctx, int k, int d, int r, double alpha, int mode, const double* X0,
                    const double* opts, double* X_out, double* G_out, double* F_out,
                    double* trace_f, double* trace_t, int64_t trace_cap, int64_t* info);
const char* mcp_lbfgs_batch_errors(void);

/*
 * Stochastic path.
 * mcp_gather_rows: rows idx[0..s) of the resident set -> dst (device, s rows of pitch ld_dst,
 *   dst_dtype MCP_F64 or MCP_F32), i.e. the V[:, idx] of sample_observations
 *   (pkg/src/momentcp/objective.py:97-113) without leaving HBM.
 * mcp_adam: adam_minimize (pkg/src/momentcp/optimize.py:365-451) with x, m1, m2 and the
 *   best iterate in HBM; every iteration gathers its mini-batch on the device and evaluates it
 *   with uniform weights 1/batch.  Randomness stays with the caller: est_idx (n_est rows, the
 *   fixed estimate subset) and, once per epoch, sample(idx, epoch_len * batch, user) fills that
 *   epoch's row indices in draw order (return 0 on success).  The caller is responsible for the
 *   uniform-weights precondition.
 *   opts[8] = {step_size, reduced_step_size, epoch_len, batch, beta1, beta2, eps, max_epochs}
 *   x_out / g_out: best iterate and its estimate gradient; f_out: best estimate
 *   trace_f / trace_t: estimate at x0 and after every epoch, seconds since start
 *   info[4] = {inner iterations, reason (0 iteration cap, 1 learning-rate exhausted), trace rows,
 *              epochs drawn ahead and never run (0 or 1)}.  The next epoch's sample() call is
 *              made while the GPU runs the current epoch; when the run stops on the learning-rate
 *              rule that last draw was not needed, and a caller that wants its generator left
 *              exactly where the reference leaves it restores the state it saved before that
 *              call (the Python layer does).
 */
typedef int (*mcp_sample_fn)(int64_t* idx, int64_t count, void* user);
int mcp_gather_rows(mcp_ctx* ctx, const int64_t* idx, int64_t s, void* dst, int64_t ld_dst,
                    int dst_dtype);
int mcp_adam(mcp_ctx* ctx, int d, int r, int mode, const double* x0, const double* opts,
             const int64_t* est_idx, int64_t n_est, mcp_sample_fn sample, void* user,
             double* x_out, double* g_out, double* f_out, double* trace_f, double* trace_t,
             int64_t trace_cap, int64_t* info);

/*
 * Peer-memory exchange of the additive [vec_F(Y) | w] pieces for the row-sharded path
 * (SURVEY.md 8e), replacing all-reduce + mcp_fg_finish_device.  Buffers are symmetric
 * (peer-mapped over NVLink, e.g. torch symmetric memory); all pointers are device pointers.
 *   mcp_peer_signal(ctx, flag_ptrs, rank, world, epoch, stream): flag_ptrs is a device array of
 *     `world` int64* (every rank's flag array); stores epoch at [rank] of each, release.sys,
 *     after this rank's partial (mcp_fg_partial_device into its slot) in stream order.
 *   mcp_fg_partial_signal_device(ctx, d, r, dx, mode, dYw, flag_ptrs, rank, world, epoch,
 *     stream): mcp_fg_partial_device into the slot dYw fused with mcp_peer_signal -- the
 *     partial's reduce kernel publishes epoch once the whole piece is written (one launch less).
 *   mcp_peer_reduce_finish(ctx, d, r, dx, part_ptrs, my_flags, world, epoch, alpha, dout, derr,
 *     stream): waits for my_flags[k] >= epoch for all k (bounded; sets *derr = 1 on timeout),
 *     sums the world partials part_ptrs[0..world-1] in rank order and writes
 *     dout = [f ; g_lam ; vec_F(g_A)] (the same on every rank).
 */
int mcp_peer_signal(mcp_ctx* ctx, const void* flag_ptrs, int rank, int world, int64_t epoch,
                    void* stream);
int mcp_fg_partial_signal_device(mcp_ctx* ctx, int d, int r, const double* dx, int mode,
                                 double* dYw, const void* flag_ptrs, int rank, int world,
                                 int64_t epoch, void* stream);
int mcp_peer_reduce_finish(mcp_ctx* ctx, int d, int r, const double* dx, const void* part_ptrs,
                           const int64_t* my_flags, int world, int64_t epoch, double alpha,
                           double* dout, int* derr, void* stream);

/* Kernel launches issued by the last evaluation call (for the bench's gpu_launches claim). */
int mcp_last_launch_count(const mcp_ctx* ctx);

/* Name of the K1 kernel variant the last evaluation used (diagnostics / bench config). */
const char* mcp_last_variant(const mcp_ctx* ctx);

#ifdef __cplusplus
}
#endif

#endif /* MOMENTCP_B200_H */

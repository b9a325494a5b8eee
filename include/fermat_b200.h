/*
 * fermat_b200.h — C ABI of the B200-native batched Fermat path solver.
 *
 * Drop-in boundary for the hot path of the reference package `fermatpath`
 * (/root/reference/pkg/src/fermatpath). The reference is a pure-Python/numpy
 * library with no FFI of its own; each entry point below replaces the named
 * reference function and is what its Python layer (or a ctypes/cgo binding,
 * see INTEGRATION.md) would call.
 *
 * Conventions
 *   - All array arguments are DEVICE pointers (CUDA global memory) in the
 *     reference's C-contiguous batch layout (batching.py:20-25):
 *       basis  (B, K, 3, 2)   anchor (B, K, 3)   start/end (B, 3)
 *       T      (B, K, 2)      points (B, K, 3)   H (B, 2K, 2K)
 *     except the *_host entry points, which take HOST pointers and do the
 *     transfers themselves.
 *   - Every call is asynchronous on `stream` (a cudaStream_t; NULL = legacy
 *     default stream) and returns an fp_error code; kernels never raise —
 *     per-path conditions are reported in a status byte (FP_STATUS_*).
 *   - Optional outputs may be NULL (not computed, not copied).
 *   - Library state: a launch counter (fp_launch_count), the kernel policy
 *     (fp_set_kernel_policy), and per-DEVICE caches created on first use on
 *     the calling thread's current device: the kernels' shared-memory
 *     attributes, the layout-probe counters of the tile dispatch, the side
 *     streams of the bucketed dispatch and the host-buffer pipeline. Calls on
 *     different devices never share any of them.
 */
#ifndef FERMAT_B200_H
#define FERMAT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- return codes ------------------------------------------------------ */
enum fp_error {
  FP_OK = 0,
  FP_ERR_INVALID_ARGUMENT = 1,   /* negative sizes, iterations < 1, NULL required ptr */
  FP_ERR_UNSUPPORTED_ORDER = 2,  /* K outside [0, FP_MAX_ORDER] */
  FP_ERR_CUDA = 3,               /* a CUDA runtime call failed (see fp_last_cuda_error) */
  FP_ERR_UNSUPPORTED_MODE = 4
};

/* Largest interaction count: the reference's MAX_INTERACTIONS (geometry.py:23).
 * Orders 1..8 run the register-resident per-thread kernels, orders 9..64 the
 * warp-per-path solver (csrc/fp_wide.cu; two paths per warp up to order 15 in
 * fp32, 11 in fp64); larger K is FP_ERR_UNSUPPORTED_ORDER. */
#define FP_MAX_ORDER 64

/* ---- per-path status bits (uint8) --------------------------------------- */
#define FP_STATUS_DEGENERATE_ENTRY 0x01u /* entry segment <= eps: reference raises DegenerateSegment for the batch (solver.py:166) */
#define FP_STATUS_ZERO_DIRECTION   0x02u /* a line search met a zero direction, alpha kept (solver.py:100,110-111) */
#define FP_STATUS_NOT_STATIONARY   0x04u /* |g| >= 1e-5 (1 + L) at the returned T (implicit_diff.py:30-36) */
#define FP_STATUS_NONFINITE        0x08u /* non-finite T, g, L or gradient output */
#define FP_STATUS_DEGENERATE_FINAL 0x10u /* a segment at T <= eps: objective.py:25-31 would raise */
#define FP_STATUS_SINGULAR         0x20u /* active Hessian singular even with Tikhonov (implicit_diff.py:64-71) */
#define FP_STATUS_OUT_OF_BOUNDS    0x40u /* enumeration: an interaction point lies outside its object */
#define FP_STATUS_SHORT_SEGMENT    0x80u /* min segment < 1e-3 at T (near a kink; parity-excluded) */
/* A path is "converged" when none of these bits is set. */
#define FP_STATUS_UNCONVERGED_MASK \
  (FP_STATUS_DEGENERATE_ENTRY | FP_STATUS_NOT_STATIONARY | FP_STATUS_NONFINITE | FP_STATUS_DEGENERATE_FINAL)

/* ---- per-iteration BFGS update fate bits (trace_fate, uint8) --------------
 * The reference's guard rails (solver.py:180-199), recorded with the trace:
 * 0 = the inverse-Hessian update was applied. */
#define FP_FATE_CURVATURE_SKIP 0x01u  /* s.y <= 1e-12 |s| |y|: update skipped (solver.py:182-184) */
#define FP_FATE_NONFINITE_SKIP 0x02u  /* H' not finite: update skipped (solver.py:196-199) */
#define FP_FATE_ZERO_DIRECTION 0x04u  /* the step-size search met a zero direction (alpha kept) */
#define FP_FATE_ENTRY_CHECK    0x08u  /* (diagnostic) the magnitude bound on H' was inconclusive and
                                         every entry was checked for finiteness (fp_path.cuh) */

/* ---- VJP modes ---------------------------------------------------------- */
enum fp_vjp_mode {
  /* w_L * (dL/dtheta + vjp_solution(grad_T L)) + vjp_solution(v_T):
   * the chain-rule ("full") total derivative, implicit_diff.py:92-100 */
  FP_VJP_FULL = 0,
  /* w_L * dL/dtheta|_T + vjp_solution(v_T): the envelope value returned by
   * grad_length_wrt_params (implicit_diff.py:80-106) */
  FP_VJP_ENVELOPE = 1,
  /* w_L * dL/dtheta|_T + param_vjp(T, v_T): v_T is used directly as the
   * direction u (objective.length_param_gradient / param_vjp,
   * objective.py:89-135); no stationarity solve, fp_vjp_* only */
  FP_VJP_MIXED = 2
};

/* ---- forward solve: solver._bfgs_kernel (solver.py:146-215) -------------
 * Fixed-iteration batch BFGS with the paper's fixed-point step size.
 * T0 (B,K,2) in; T_out/g_out (B,K,2), points_out (B,K,3), length_out (B),
 * status_out (B), trace_len/trace_gnorm (iterations, B) [record_trace],
 * trace_fate (iterations, B) FP_FATE_* bits [with the trace; NULL = none],
 * H_out (B,2K,2K) [return_state]. */
int fp_solve_f32(const float* basis, const float* anchor, const float* start, const float* end,
                 const float* T0, int64_t B, int K, int iterations, int fp_iters,
                 float* T_out, float* g_out, float* points_out, float* length_out,
                 uint8_t* status_out, float* trace_len, float* trace_gnorm, uint8_t* trace_fate,
                 float* H_out, void* stream);
int fp_solve_f64(const double* basis, const double* anchor, const double* start, const double* end,
                 const double* T0, int64_t B, int K, int iterations, int fp_iters,
                 double* T_out, double* g_out, double* points_out, double* length_out,
                 uint8_t* status_out, double* trace_len, double* trace_gnorm, uint8_t* trace_fate,
                 double* H_out, void* stream);

/* ---- implicit-gradient VJP: implicit_diff.vjp_solution / grad_length_wrt_params
 * (implicit_diff.py:39-106 over objective.py:48-135), batched.
 * Cotangents: v_T (B,K,2) on T* (NULL = 0); w_L (B) per-path weight on L*
 * (NULL = use w_L_scale for every path). Outputs d_basis (B,K,3,2),
 * d_anchor (B,K,3), d_start (B,3), d_end (B,3); u_out (B,K,2) is the
 * solve_stationary_system solution for rhs w_L*g + v_T (FULL) or v_T. */
int fp_vjp_f32(const float* basis, const float* anchor, const float* start, const float* end,
               const float* T, const float* v_T, const float* w_L, float w_L_scale, int mode,
               int64_t B, int K, float* d_basis, float* d_anchor, float* d_start, float* d_end,
               float* u_out, uint8_t* status_out, void* stream);
int fp_vjp_f64(const double* basis, const double* anchor, const double* start, const double* end,
               const double* T, const double* v_T, const double* w_L, double w_L_scale, int mode,
               int64_t B, int K, double* d_basis, double* d_anchor, double* d_start, double* d_end,
               double* u_out, uint8_t* status_out, void* stream);

/* ---- fused forward + VJP of w_L * L* (one kernel; the config-2 step) ----- */
int fp_solve_vjp_f32(const float* basis, const float* anchor, const float* start, const float* end,
                     const float* T0, int64_t B, int K, int iterations, int fp_iters,
                     const float* w_L, float w_L_scale, int mode,
                     float* T_out, float* points_out, float* length_out,
                     float* d_basis, float* d_anchor, float* d_start, float* d_end,
                     uint8_t* status_out, void* stream);
int fp_solve_vjp_f64(const double* basis, const double* anchor, const double* start,
                     const double* end, const double* T0, int64_t B, int K, int iterations,
                     int fp_iters, const double* w_L, double w_L_scale, int mode,
                     double* T_out, double* points_out, double* length_out,
                     double* d_basis, double* d_anchor, double* d_start, double* d_end,
                     uint8_t* status_out, void* stream);

/* Same step with HOST buffers: copies in, solves + differentiates, copies
 * out, pipelined over chunks of `chunk` paths: a copy-in, a compute and a
 * copy-out stream over a ring of `depth` (1..8) device chunk slots, so both
 * PCIe directions stay busy; blocks until the outputs are in host memory.
 * Pinned host memory gives full PCIe bandwidth. basis/anchor (K > 0) and
 * start/end are required (NULL: FP_ERR_INVALID_ARGUMENT). T0 == NULL means
 * zero initialisation (set on the device: no host-to-device copy). Every
 * output may be NULL and is then neither computed into host memory nor
 * copied: e.g. points_out, which the reference derives on the host from T
 * (bench.py:313-314 of the reference). */
int fp_solve_vjp_host_f32(const float* basis, const float* anchor, const float* start,
                          const float* end, const float* T0, int64_t B, int K, int iterations,
                          int fp_iters, float w_L_scale, int mode, float* T_out, float* points_out,
                          float* length_out, float* d_basis, float* d_anchor, float* d_start,
                          float* d_end, uint8_t* status_out, int64_t chunk, int depth);
int fp_solve_vjp_host_f64(const double* basis, const double* anchor, const double* start,
                          const double* end, const double* T0, int64_t B, int K, int iterations,
                          int fp_iters, double w_L_scale, int mode, double* T_out,
                          double* points_out, double* length_out, double* d_basis,
                          double* d_anchor, double* d_start, double* d_end, uint8_t* status_out,
                          int64_t chunk, int depth);
/* The same call without the final wait: enqueues the copies and kernels and
 * returns a ticket; fp_host_wait(ticket) blocks until that call's outputs are
 * in host memory. Consecutive calls with the same order and chunk chain
 * through one ring of chunk slots, so call i + 1's host-to-device copies
 * overlap call i's device-to-host copies. The host buffers of a submitted
 * call must stay valid and unmodified until its wait returns; at most 16
 * calls are in flight (a submit waits for the one 16 tickets back). */
int fp_solve_vjp_host_submit_f32(const float* basis, const float* anchor, const float* start,
                                 const float* end, const float* T0, int64_t B, int K, int iterations,
                                 int fp_iters, float w_L_scale, int mode, float* T_out,
                                 float* points_out, float* length_out, float* d_basis,
                                 float* d_anchor, float* d_start, float* d_end, uint8_t* status_out,
                                 int64_t chunk, int depth, uint64_t* ticket);
int fp_solve_vjp_host_submit_f64(const double* basis, const double* anchor, const double* start,
                                 const double* end, const double* T0, int64_t B, int K,
                                 int iterations, int fp_iters, double w_L_scale, int mode,
                                 double* T_out, double* points_out, double* length_out,
                                 double* d_basis, double* d_anchor, double* d_start, double* d_end,
                                 uint8_t* status_out, int64_t chunk, int depth, uint64_t* ticket);
int fp_host_wait(uint64_t ticket);

/* ---- objective pieces: objective.path_length / gradient / hessian
 * (objective.py:34-64), unclamped norms; degenerate segments flag
 * FP_STATUS_DEGENERATE_FINAL instead of raising. hess_out (B,2K,2K). */
int fp_objective_f64(const double* basis, const double* anchor, const double* start,
                     const double* end, const double* T, int64_t B, int K, double* length_out,
                     double* grad_out, double* hess_out, uint8_t* status_out, void* stream);

/* ---- solver.line_search_alpha (solver.py:115-143), batched, fp64.
 * status: FP_STATUS_ZERO_DIRECTION (ZeroDirection) or
 * FP_STATUS_DEGENERATE_ENTRY (DegenerateSegment in a denominator). */
int fp_line_search_f64(const double* basis, const double* anchor, const double* start,
                       const double* end, const double* T, const double* P, const double* alpha0,
                       int64_t B, int K, int k, double* alpha_out, uint8_t* status_out,
                       void* stream);

/* ---- solver.init_params (solver.py:67-81), batched, fp64 ----------------- */
int fp_init_params_f64(const double* basis, const double* anchor, const double* start,
                       const double* end, int64_t B, int K, double* T_out, void* stream);

/* ---- candidate enumeration + tracing (BASELINE configs 3 and 4) -----------
 * No reference code exists; the specification is in
 * csrc/fp_enum.cu and DESIGN.md. Objects: obj_basis (N,3,2), obj_anchor
 * (N,3); plane_ids / edge_ids list the reflector and edge objects. One call
 * covers candidates [cand_begin, cand_end) of one (order <= 3, kind pattern)
 * group, RX-major: candidate c -> rx = c / count_p, sequence c % count_p.
 * Per-RX sequence count of a pattern (host function; -1 if invalid): */
int64_t fp_enum_pattern_count(int n_planes, int n_edges, int order, unsigned pattern);
/* Decode candidates to (rx, object sequence) — the enumeration itself. */
int fp_enum_decode(const int32_t* plane_ids, int n_planes, const int32_t* edge_ids, int n_edges,
                   int n_rx, int order, unsigned pattern, int64_t cand_begin, int64_t cand_end,
                   int32_t* rx_out, int32_t* seq_out, void* stream);
/* Fused decode -> solve (zero init) -> bounds mask -> compaction of VALID
 * paths (converged and inside every object). counters (device, 4 x u64,
 * accumulated): candidates, converged, in-bounds, valid (= records written
 * when below `capacity`). With obj_grad (N,9: basis 6 + anchor 3) non-NULL,
 * also accumulates loss += sum 1/L^2 and the gradients of that loss (full
 * implicit VJP, cotangent -2/L^3) into obj_grad, tx_grad (3), rx_grad (n_rx,3)
 * and loss — fp64 accumulators (each path's terms are fp32). */
int fp_enum_trace_f32(const float* obj_basis, const float* obj_anchor, const int32_t* plane_ids,
                      int n_planes, const int32_t* edge_ids, int n_edges, const float* tx,
                      const float* rx, int n_rx, int order, unsigned pattern, int64_t cand_begin,
                      int64_t cand_end, int iterations, int fp_iters,
                      unsigned long long* counters, int64_t capacity, int32_t* rec_rx,
                      int32_t* rec_seq, float* rec_T, float* rec_L, float* rec_points,
                      double* obj_grad, double* tx_grad, double* rx_grad, double* loss,
                      void* stream);
/* Object-parameter gradients -> vertex gradients: vert_ids (N,4) (-1 unused),
 * coef (N,3,4) for (anchor, basis col 0, basis col 1) x vertex slot. */
int fp_vertex_chain_f32(const double* obj_grad, int n_objects, const int32_t* vert_ids,
                        const float* coef, double* vertex_grad, void* stream);

/* ---- visibility of traced paths (post-processing; no reference code) --------
 * For n traced paths of order 1..3 (TX, interaction points (n, order, 3), RX =
 * rx[rec_rx[r]]), flags[r] gets
 *   FP_VIS_BLOCKED     a segment crosses one of the n_blockers parallelograms
 *                      O + a U + b V (blockers (Q, 3, 3) = O, U, V; a, b in
 *                      [0, 1]) farther than eps metres from both its ends;
 *   FP_VIS_WRONG_SIDE  (when rec_seq is given) a reflection (obj_plane[o] != 0
 *                      for object o = rec_seq[r, i], normal = column 0 x
 *                      column 1 of obj_basis[o]) whose neighbours are not
 *                      strictly on one side of the plane.
 * first_blocker[r] (nullable) = index of the first blocker hit, -1 if none.
 * fp64, unfused, in oracle/visibility_oracle.py's operation order. Q <= 2048. */
#define FP_VIS_BLOCKED 0x01
#define FP_VIS_WRONG_SIDE 0x02
int fp_visibility_f64(const double* blockers, int n_blockers, const float* tx, const float* rx,
                      const int32_t* rec_rx, const float* points, const int32_t* rec_seq,
                      const float* obj_basis, const uint8_t* obj_plane, int n_objects, int64_t n,
                      int order, double eps, uint8_t* flags, int32_t* first_blocker, void* stream);

/* ---- comparison solvers -------------------------------------
 * Damped Newton on active coordinates with step halving: baselines._newton_kernel
 * (baselines.py:152-193), the config-1 comparator. K <= 5. trace_gnorm
 * (iterations, B) optional: |g| after each iteration. */
int fp_newton_f32(const float* basis, const float* anchor, const float* start, const float* end,
                  const float* T0, int64_t B, int K, int iterations, float* T_out, float* g_out,
                  float* trace_gnorm, void* stream);
int fp_newton_f64(const double* basis, const double* anchor, const double* start, const double* end,
                  const double* T0, int64_t B, int K, int iterations, double* T_out, double* g_out,
                  double* trace_gnorm, void* stream);
/* Fixed-step gradient descent baseline: baselines._gd_kernel (baselines.py:87-101). K <= 5. */
int fp_gd_f32(const float* basis, const float* anchor, const float* start, const float* end,
              const float* T0, int64_t B, int K, int iterations, float* T_out, float* g_out,
              void* stream);
int fp_gd_f64(const double* basis, const double* anchor, const double* start, const double* end,
              const double* T0, int64_t B, int K, int iterations, double* T_out, double* g_out,
              void* stream);
/* Exact reflection points of all-plane paths: baselines.image_points_batch
 * (baselines.py:48-71). points (B,K,3); status FP_STATUS_SINGULAR where the
 * mirrored sight line is parallel to its plane (NoIntersection). */
int fp_image_method_f64(const double* basis, const double* anchor, const double* start,
                        const double* end, int64_t B, int K, double* points, uint8_t* status,
                        void* stream);

/* ---- FP32 roofline probe ----------------------------------------------------
 * blocks x 256 threads, each running iters x 128 dependent-free FFMAs; the
 * bench times it with CUDA events to measure the FP32 SIMT peak. */
int fp_peak_ffma(int blocks, int iters, float* out, void* stream);
/* The same FMA-lane count with every operand in a distinct register pair
 * (FFMA2 a, b, c all registers): the attainable ceiling for register-resident
 * arithmetic (register-file bandwidth bound). */
int fp_peak_ffma_reg(int blocks, int iters, float* out, void* stream);

/* Benchmark utility: enqueue a kernel that holds `stream` until the host
 * stores a nonzero int at host_flag (pinned host memory) or timeout_s
 * (<= 60) elapses. bench.py gates its timed region with it so every timed
 * step is enqueued before the device starts. */
int fp_gate_wait(const int* host_flag, double timeout_s, void* stream);

/* ---- bookkeeping ---------------------------------------------------------- */
/* Kernel selection for solves / fused steps of order 1..5 (other calls run
 * the dense kernels of their order). Every policy but FP_POLICY_DENSE runs,
 * for each path, the kernel variant carrying only its active unknowns (its
 * interaction-kind mask).
 *   FP_POLICY_AUTO (default): the tile kernel (one launch; each warp
 *     dispatches on its paths' masks; no host round trip; fp32 and fp64)
 *     unless the last call of that order saw more than 1/8 mixed-mask warps
 *     (a scattered layout), which then classifies the paths on the device
 *     (one host round trip) and runs the tile kernel over a mask-sorted row
 *     permutation.
 *   FP_POLICY_DENSE: the uniform 2K kernel for every path (agrees with the
 *     specialised variants to rounding; used by the tests).
 *   FP_POLICY_AUTO_SERIAL: bucketed, per-mask kernels (fp32) one after
 *     another on the caller's stream instead of concurrent side streams.
 *   FP_POLICY_BUCKET: always bucketed (classify on the device, one host
 *     round trip; fp32: one kernel per mask over its row range or
 *     permutation; fp64: the tile kernel over the mask-sorted permutation).
 *   FP_POLICY_TILE: always the tile kernel.
 * A path's results are bitwise the same under AUTO, AUTO_SERIAL, BUCKET and
 * TILE. */
#define FP_POLICY_AUTO 0
#define FP_POLICY_DENSE 1
#define FP_POLICY_AUTO_SERIAL 2
#define FP_POLICY_BUCKET 3
#define FP_POLICY_TILE 4
int fp_set_kernel_policy(int policy);

/* Number of kernels this library has launched in the process (monotone). */
uint64_t fp_launch_count(void);
/* Last CUDA error seen by the library (cudaError_t as int). */
int fp_last_cuda_error(void);
const char* fp_error_string(int code);
int fp_version(void);

#ifdef __cplusplus
}
#endif

#endif /* FERMAT_B200_H */

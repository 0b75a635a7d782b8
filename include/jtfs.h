/* jtfs.h — C ABI of libjtfs.so: B200-native joint time–frequency scattering (JTFS) forward
 * transform, Euclidean feature loss, its gradient with respect to the audio samples, and the
 * metamer descent step of arxiv 2602.11896 ("musical metamers").
 *
 * Citations: P:n = PAPER.md line n; S:n = SPEC.md line n; Rk = reading k of DESIGN.md §2.
 *
 * Conventions for every entry point
 *  - Return value: JTFS_OK (0) or an error code; on error `jtfs_last_error()` (thread-local)
 *    names the violated constraint. No entry point aborts the process.
 *  - A plan is immutable after `jtfs_plan` returns, except for its lazily uploaded device copy
 *    (see jtfs_plan_prepare); concurrent calls with one plan on different streams and distinct
 *    workspaces are safe once the plan is prepared on that device.
 *  - "device pointer": memory of the current CUDA device, fp32, contiguous, 16-byte aligned,
 *    owned by the caller. Work is enqueued on `stream` in order; no host synchronisation unless
 *    stated (the *_host variants synchronise `stream` before returning).
 *  - Results are deterministic (bitwise) for a fixed (plan, B, device, workspace size): no
 *    floating-point atomics on any output path.
 */
#ifndef JTFS_H
#define JTFS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct jtfs_plan_s* jtfs_plan_t;
typedef struct CUstream_st* jtfs_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  JTFS_OK = 0,
  JTFS_ERR_CONFIG = 1,  /* plan hyper-parameters violate a constraint */
  JTFS_ERR_SIZE = 2,    /* B <= 0, workspace too small, misaligned or NULL pointer, bad cap */
  JTFS_ERR_NUMERIC = 3, /* non-finite loss or gradient detected */
  JTFS_ERR_CUDA = 4,    /* CUDA runtime error (message = cudaGetErrorString) */
  JTFS_ERR_OOM = 5,     /* host or device allocation failed */
  JTFS_ERR_STATE = 6    /* invalid handle / state */
} jtfs_status;

/* ---------------------------------------------------------------------------------------
 * Plan (host, float64). Builds the three filterbanks of P:157-193 (generator P:167-191, readings
 * R1-R3), the Morlet responses with the κ correction of Eq.1 (R4-R5), the Gaussian
 * low-pass φ_T / φ_F (R6), padding (R10), the frequential grid P (= phi['N'],
 * P:276, R11), the admissible width-first blocks, and the path table in the
 * yield order of P:314-351 (R15). Q2 = 1 (R7).
 *  N     signal length (samples), multiple of T
 *  J,Q   first-layer scale and quality factor (J >= 1, Q >= 1)
 *  J_fr,Q_fr frequential scale and quality factor (>= 1)
 *  T,F   time / log-frequency averaging widths, powers of two, 1 <= log2 T <= J,
 *        0 <= log2 F <= J_fr; N_pad (R10) must be <= 2^22; ceil(N1/F) <= 32, or <= 64 when
 *        P <= 1024 (GPU limit: rows beyond 32 take the FFT route of the joint stage).
 *  out   receives the handle; release with jtfs_plan_destroy.
 * Errors: JTFS_ERR_CONFIG (constraint named), JTFS_ERR_OOM. Touches no GPU. */
jtfs_status jtfs_plan(int64_t N, int J, int Q, int J_fr, int Q_fr, int64_t T, int64_t F,
                      jtfs_plan_t* out);
/* Same with the second-layer temporal quality factor Q2 = Q^{tm,2} ("its own hyperparameters";
 * 1 <= Q2 <= 16). jtfs_plan is jtfs_plan_q2 with Q2 = 1 (R7). */
jtfs_status jtfs_plan_q2(int64_t N, int J, int Q, int Q2, int J_fr, int Q_fr, int64_t T, int64_t F,
                         jtfs_plan_t* out);
jtfs_status jtfs_plan_destroy(jtfs_plan_t plan); /* frees host and device copies */

typedef struct {
  int64_t N, N_pad, pad_left, P, frames, n_coef, n_paths;
  int32_t N1, N2, N_fr, n_blocks, log2T, log2F;
} jtfs_plan_info_t;
/* N1 = #psi1, N2 = #psi2, N_fr = #frequential filters with xi > 0 (per spin), frames = N/T,
 * n_coef = packed coefficients per signal (S0 first, then orders 1 and 2, R15). */
jtfs_status jtfs_plan_info(jtfs_plan_t plan, jtfs_plan_info_t* info);

typedef struct {
  int32_t order, n2, n_fr, spin, j2, j_fr, rows, frames;
  int64_t offset; /* first coefficient of this path in the packed vector */
} jtfs_path_t;
/* Path table in yield order: S0 (order 0), order 1 over [phi_F, psi+...],
 * order 2 by admissible n2 ascending over [phi_F, psi+..., psi-...] (R12). Each path occupies
 * rows*frames coefficients, row-major. `cap` = capacity of `out` in entries. */
jtfs_status jtfs_plan_paths(jtfs_plan_t plan, jtfs_path_t* out, int64_t cap);

/* Test hook: filter parameters of one bank. layer 0 = psi1, 1 = psi2, 2 = L_fr (R12 order:
 * phi_F, psi+..., psi-...), 3 = phi_T, 4 = phi_F. Writes up to `cap` entries; returns the
 * count through *count. */
jtfs_status jtfs_plan_filters(jtfs_plan_t plan, int layer, double* xi, double* sigma, int32_t* j,
                              int64_t cap, int64_t* count);

/* Test hook: level-k Fourier response (float64, periodised, R4/R9) of filter `idx` of `layer`
 * on a grid of L0 >> k bins (L0 = N_pad for layers 0,1,3 and P for 2,4), written to out[cap]. */
jtfs_status jtfs_plan_response(jtfs_plan_t plan, int layer, int idx, int k, double* out,
                               int64_t cap);

/* Uploads the plan's device tables (filter spectra, row kernels, twiddles) to the current device
 * on `stream` and synchronises. Called implicitly by the first compute call; call it explicitly
 * to keep the upload out of timed regions. */
jtfs_status jtfs_plan_prepare(jtfs_plan_t plan, jtfs_stream_t stream);

/* Workspace bytes for `batch` signals processed at once (with_grad = 1 for jtfs_loss_grad and
 * metamer_step). It is affine in batch: fixed + batch * per_signal. A compute call processes its
 * B signals in micro-batches of floor((ws_bytes - fixed) / per_signal) signals. */
size_t jtfs_workspace_size(jtfs_plan_t plan, int64_t batch, int with_grad);

/* ---------------------------------------------------------------------------------------
 * Forward (Eq.2-4 with R14 averaging). x [B][N] device fp32 signals; S [B][n_coef]
 * device fp32 packed coefficients (R15, unpadded R16). ws: device workspace of ws_bytes. */
jtfs_status jtfs_forward(jtfs_plan_t plan, const float* x, int64_t B, float* S, void* ws,
                         size_t ws_bytes, jtfs_stream_t stream);

/* Loss and gradient (R19-R22). For each signal b:
 *   loss[b] = 1/2 sum_{orders 1,2} (S(y_b) - S_target_b)^2   (S0 excluded, R19)
 *   grad[b] = dE_b/dy_b, the TRUE gradient (the paper's "grad E" is its negative, R23).
 *   Modulus adjoint (R22): the phase z/|z| is 0 where |z| < 1e-12 * RMS(y_b), at
 *   every modulus site; elsewhere it is the exact phase (PyTorch autograd's). On the
 *   split-K joint-stage blocks (large n1_max) the forward keeps that phase for the backward as
 *   two int16 per cell (|error| <= 1.6e-5 on the unit vector).
 * y [B][N], S_target [B][n_coef], loss [B], grad [B][N]: device fp32.
 * shard/n_shards: second-order path shard (0,1 = whole; n_shards <= 64). With n_shards > 1 the call
 * computes the contribution of the second-order blocks jtfs_plan_shards assigns to `shard` (layer 2,
 * joint stage and their adjoints for those blocks only), plus (shard 0 only) order 1; layer 1 runs on
 * every shard. Summing loss and grad over shards (e.g. NCCL allreduce) gives the full result. */
jtfs_status jtfs_loss_grad(jtfs_plan_t plan, const float* y, const float* S_target, int64_t B,
                           float* loss, float* grad, int shard, int n_shards, void* ws,
                           size_t ws_bytes, jtfs_stream_t stream);

/* Metamer state (R23-R24); all device pointers, caller-owned:
 *  y, u, y_prev, g_prev [B][N]; mu, loss_prev [B] (loss_prev = +inf before the first step);
 *  accepted [B] int32 output flag; loss [B] output (loss at the y evaluated this step). */
typedef struct {
  float *y, *u, *y_prev, *g_prev, *mu, *loss_prev, *loss;
  int32_t* accepted;
  int64_t iter; /* incremented by each call (host field) */
  const int32_t* active; /* [B] or NULL (all active): a signal with active[b] == 0 is frozen at its
                            best iterate (y = y_prev, u = 0, mu and loss_prev kept, accepted = 0) --
                            the host loop's early stop and rejection cap */
} jtfs_metamer_state;

/* One descent trial, entirely stream-ordered (no host sync): E, g = jtfs_loss_grad(y); per
 * signal accept if E <= loss_prev (then y_prev=y, g_prev=g, loss_prev=E, mu*=grow) else reject
 * (y=y_prev, g=g_prev, u=0, mu*=shrink); then u = momentum*u - mu*g; y = y + u.
 * Paper defaults: momentum 0.9, mu0 0.1; grow 1.1, shrink 0.5 (R24). */
jtfs_status metamer_step(jtfs_plan_t plan, jtfs_metamer_state* st, const float* S_target,
                         int64_t B, float momentum, float grow, float shrink, void* ws,
                         size_t ws_bytes, jtfs_stream_t stream);

/* Test-only: the library's batched C2C FFT (fft.cu) on device rows, for benchmarking against cuFFT
 * (tools/fft_vs_cufft.py): out[b][r][.] = FFT(in[b][r][.]) for B x count rows of length L (power of two,
 * 2 <= L <= the plan's N_pad); inverse includes 1/L; dbl = 0: complex64, 1: complex128. For L > 4096 the
 * input is clobbered (four-step scheme). Stream-ordered. */
jtfs_status jtfs_debug_fft(jtfs_plan_t plan, const void* in, void* out, int64_t L, int64_t count, int64_t B,
                           int inverse, int dbl, jtfs_stream_t stream);

/* Non-finite check ("non-finite direction -> numeric error"): returns JTFS_ERR_NUMERIC if any
 * of x[0..n) (device fp32) is NaN or +-inf, JTFS_OK otherwise. Synchronises `stream` (the only call
 * besides the host-buffer variants that does); used by the metamer loop on y and the loss each step. */
jtfs_status jtfs_check_finite(const float* x, int64_t n, jtfs_stream_t stream);

/* Path-shard assignment: block_owner_out[bi] = shard of second-order block bi for
 * n_shards shards (1..64): LPT over the planner's per-block cost (joint-stage contraction flops + the
 * block's time-axis FFTs), largest block first to the least-loaded shard, ties to the lower index;
 * shard 0 starts loaded with order 1. Deterministic; host only. cap >= n_blocks. */
jtfs_status jtfs_plan_shards(jtfs_plan_t plan, int n_shards, int32_t* block_owner_out, int64_t cap);

/* Per-path LossReport (R19): per_path[b][q] = 1/2 sum over the coefficients of path q
 * (jtfs_plan_paths order, R15) of (S - S_target)^2, float64 accumulation. Path 0 (S0) is reported but is
 * not part of the loss E_b = sum over the order-1 and order-2 entries. S, S_target [B][n_coef],
 * per_path [B][n_paths]: device fp32. Stream-ordered; no workspace. */
jtfs_status jtfs_loss_report(jtfs_plan_t plan, const float* S, const float* S_target, int64_t B,
                             float* per_path, jtfs_stream_t stream);

/* Colored Gaussian noise initialisation of the metamer loop (§2.3: "a colored Gaussian noise
 * y0(t) whose power spectral density matches S1 x(t, lambda)"; reading R25 in DESIGN.md):
 *   a[n1] = RMS over frames of the order-1 beta = 0 path of S_target, interpolated at row n1 / F;
 *   g[n1] = a[n1] / sqrt(pi/4 * nu[n1]),  nu[n1] = (1/N_pad) sum_m |psi1_hat_n1[m]|^2;
 *   G[m]  = sum_n1 g[n1] |psi1_hat_n1(|w_m|)|^2 / (sum_n1 |psi1_hat_n1(|w_m|)|^2 + delta);
 *   y0    = Re IFFT(FFT(white) G) on samples [pad_left, pad_left + N)  (1e-4 white if a == 0).
 * S_target [B][n_coef] (packed, R15), white [B][N_pad] standard-normal draws (the caller's random
 * numbers), y0 [B][N] out: device fp32. ws as for jtfs_forward (micro-batched). Stream-ordered. */
jtfs_status jtfs_colored_noise(jtfs_plan_t plan, const float* S_target, const float* white, int64_t B,
                               float* y0, void* ws, size_t ws_bytes, jtfs_stream_t stream);

/* End-to-end variants with HOST buffers (pinned or pageable): copy inputs host->device, run, copy
 * results device->host, synchronise `stream`. The library allocates device staging of the given
 * sizes inside ws (ws_bytes must include jtfs_host_staging_size). */
size_t jtfs_host_staging_size(jtfs_plan_t plan, int64_t B, int with_grad);
jtfs_status jtfs_loss_grad_host(jtfs_plan_t plan, const float* y_host, const float* S_target_host,
                                int64_t B, float* loss_host, float* grad_host, void* ws,
                                size_t ws_bytes, jtfs_stream_t stream);

/* Thread-local message of the last error ("" if none). */
const char* jtfs_last_error(void);

/* Test-only: run the forward of one micro-batch and copy an intermediate stage to out:
 *  stage 1 = U1 (|Z1|, [B][sum_n1 N_pad>>k1] fp32), 2 = S1t ([B][N1][N_pad/T] fp32),
 *  3 = Y2 ([B][sum_blocks n1_max*T2] complex64 interleaved), 4 = S ([B][n_coef]). */
jtfs_status jtfs_debug_stage(jtfs_plan_t plan, int stage, const float* x, int64_t B, void* out,
                             size_t out_bytes, void* ws, size_t ws_bytes, jtfs_stream_t stream);

/* Test-only: one-CTA tcgen05 kind::tf32 GEMM D[128][N] = A[128][K] . B[N][K]^T (3xTF32 if three)
 * with B given as a device image in the canonical K-major layout ([hi | lo], see tc.cuh). */
jtfs_status jtfs_debug_tc_gemm(const float* A, const float* Bimg, float* D, int N, int K, int three,
                               jtfs_stream_t stream);

/* Test-only: same GEMM with A staged in TMEM by tcgen05.st and the TS form of tcgen05.mma. */
jtfs_status jtfs_debug_tc_gemm_ts(const float* A, const float* Bimg, float* D, int N, int K, int three,
                                  jtfs_stream_t stream);

/* Number of kernels the library has launched in this process (for launch-count reporting). */
int64_t jtfs_launch_count(void);

/* Algorithmic cost per signal of the joint lambda_1 stage (roofline reporting),
 * over the pruned rows x columns ("cells", one modulus value each):
 *  out[0] forward dense-contraction flops on the tensor-core blocks (8 K per cell)
 *  out[1] forward FP32 flops on the FFT-route blocks (per column: 5 P log2 P for FFT_P of y; per filter
 *         4 P fold + 5 L_f log2 L_f inverse FFT + 4 n_rows modulus + 2 rows_out n_rows phi_F)
 *  out[2] backward contraction flops on the tensor-core blocks (16 K per cell: recompute + adjoint;
 *         8 K on split-K blocks, whose backward reuses the phase of W kept by the forward)
 *  out[3] backward FP32 flops on the FFT-route blocks (recompute, phi_F adjoint, phase, DFT, spectrum
 *         accumulation, final inverse FFT_P)
 *  out[4] cells, out[5] HBM bytes of the joint stage (Y2 r fwd + r bwd, g_Y2 w, o w + g_o r). cap >= 8. */
jtfs_status jtfs_plan_cost(jtfs_plan_t plan, double* out, int64_t cap);

/* Profiling hook used by bench.py: when enabled, CUDA events are recorded on the launch stream
 * around the joint stage (id 0 = forward, all routes; 2 = backward, all routes; the tensor-core and
 * FFT-route launches run concurrently on side streams in between). jtfs_prof_read synchronises on the
 * recorded events, returns the summed elapsed milliseconds and the number of timed launches of
 * `id`, and clears them. */
void jtfs_prof_enable(int on);
jtfs_status jtfs_prof_read(int id, double* total_ms, int64_t* count);

#ifdef __cplusplus
}
#endif
#endif /* JTFS_H */

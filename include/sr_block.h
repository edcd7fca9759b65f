/*
 * sr_block.h — C ABI of the B200-native block-layer stochastic-reconfiguration step
 * (arXiv 2510.08430, "block-layer QGT"; §2, Eqs. 1-3).
 *
 * One step, five stages (BASELINE.json north_star):
 *   (1) sr_jacobian      O_ki = d ln psi(x_k) / d theta_i, grouped by layer      PAPER.md Eq. 2
 *   (2) sr_local_energy  E_loc(x_k) = sum_x' <x_k|H|x'> psi(x')/psi(x_k)          PAPER.md Eq. 1
 *   (3) sr_center_force  Obar = O - <O>, F = Obar^H (E_loc - <E_loc>) / N_s      PAPER.md Eq. 2, §2
 *   (4) sr_block_qgt     S_b = Obar_b^H Obar_b / N_s for every layer block b     PAPER.md Eq. 3
 *   (5) sr_block_solve   (S_b + lambda I) dtheta_b = -F_b, blocks independent    PAPER.md §2
 * plus the comparison paths sr_full_qgt_solve (§2 "S . dtheta = -F") and
 * sr_ntk_solve (§1, sample-space NTK / MinSR), and sr_step / sr_step_host
 * which run stages (1)-(5) back to back.
 *
 * Conventions
 * -----------
 * - complex128 values are two interleaved doubles (re, im): the layout of C99
 *   `double _Complex`, `std::complex<double>`, numpy complex128 and torch.complex128.
 *   Pointers typed `double*` below that say "complex" point at 2*count doubles.
 * - Every pointer is a DEVICE pointer unless the argument says (host).  Device
 *   buffers are owned by the caller; the library never allocates or frees device
 *   memory, and keeps no state between calls apart from the process-wide Gram engine
 *   choice (sr_set_gram_engine), the optional kernel timer (sr_kernel_timer) and device
 *   trace (sr_trace_buffer), the CUDA-graph cache of sr_step_host, and a pool of side
 *   streams/events created on first use (the blocked solves run independent blocks and
 *   off-chain updates on them, forked from and joined back into `stream`).  Scratch
 *   comes in through a `workspace` pointer whose size the matching *_workspace_bytes()
 *   query returns (256-byte aligned base required).
 * - Threads: calls may come from any host thread, but not concurrently -- the side-stream
 *   pool, the graph cache and the timer are shared, unsynchronised process state.
 * - Devices: one device per process (the multi-GPU path runs one process per GPU).  The
 *   side-stream pool and the CUDA-graph cache are created on the device current at their
 *   first use; the kernels' shared-memory opt-ins are set once per device.
 * - `stream` is a cudaStream_t (NULL = legacy default stream).  All device work is
 *   enqueued on it; calls return without synchronising, except sr_step_host.
 * - Network: complex MLP with widths[0..n_layers] (widths[0] = N sites),
 *   z_l = W_l h_{l-1} + b_l, h_l = lncosh(z_l) (principal branch), ln psi = sum_j h_L[j].
 *   theta is complex [n_p]: for each layer l in order, W_l row-major
 *   [widths[l+1]][widths[l]] then b_l [widths[l+1]].  Layer block b = layer b, columns
 *   [off_b, off_b + n_b) with n_b = widths[b+1]*(widths[b]+1).  n_layers <= 16 and
 *   every width <= 256.
 * - Spins: int8 [n_samples][N], entries +1 / -1.
 * - Hamiltonian (Pauli units, reading R3): H = sum_b J_b sigma_i.sigma_j over
 *   the bond list; bonds_ij int32 [n_bonds][2], bond_j double [n_bonds].
 * - Sample weights: `weights` double [n_samples] summing to 1, or NULL for uniform
 *   1/n_samples.  Stage (3) stores A_k = sqrt(w_k) (O_k - <O>) in place of O and
 *   e_k = sqrt(w_k)(E_loc,k - E), so S = A^H A, F = A^H e, T_NTK = A A^H.
 *
 * Errors: functions return SR_OK (0) or a negative sr_status; sr_last_error()
 * returns a thread-local message for the last failure.  Invalid sizes/pointers are
 * rejected before any work is enqueued.  Kernel faults surface as SR_ERR_CUDA
 * (possibly from a later call, as with any asynchronous CUDA API).  A
 * non-positive Cholesky pivot is reported through the optional device `info` word
 * of the solvers (0 = success, k>0 = first failing pivot row + 1 of the first
 * failing block) — it cannot happen for lambda > 0 and a Hermitian PSD S.
 */
#ifndef SR_BLOCK_H
#define SR_BLOCK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define SR_API __attribute__((visibility("default")))
#else
#define SR_API
#endif

typedef int sr_status;
#define SR_OK 0
#define SR_ERR_INVALID (-1)  /* bad size, null pointer, unsupported width */
#define SR_ERR_CUDA (-2)     /* a CUDA runtime call or kernel launch failed */
#define SR_ERR_WORKSPACE (-3) /* workspace smaller than the query result */

/* Library version (major*10000 + minor*100 + patch). */
SR_API int sr_version(void);
/* Message for the most recent failure on this host thread ("" if none). */
SR_API const char* sr_last_error(void);
/* Number of kernel launches issued by this host thread since the last reset
 * (instrumentation for bench.py's gpu_launches; reset with sr_reset_launch_count). */
SR_API int64_t sr_launch_count(void);
SR_API void sr_reset_launch_count(void);

/* Kernel timer (measurement support for bench.py).  While enabled, launches of the
 * dominant kernels ("gram_i8" of sr_block_qgt_i8, "gram_tn" of sr_block_qgt) are
 * bracketed by CUDA events on their launch stream (not while the stream is being
 * captured into a graph).  sr_kernel_time_ms synchronises those events and returns the
 * summed milliseconds of the launches of `kernel` recorded since the previous read
 * (their count in *launches, may be NULL), then forgets them. */
SR_API void sr_kernel_timer(int enable);
SR_API double sr_kernel_time_ms(const char* kernel, int64_t* launches);
/* sr_kernel_timeline — every pending timer record (all names) as text lines
 * "name stream_index begin_ms end_ms\n", times relative to the first record's begin event,
 * stream_index numbering the distinct launching streams in order of first use.  With buf
 * non-NULL and bytes > 0, writes at most bytes-1 characters plus a NUL and consumes the
 * records; with buf NULL only queries.  Returns the size needed including the NUL.  Host-side diagnostics only. */
SR_API size_t sr_kernel_timeline(char* buf, size_t bytes);
/* sr_trace_buffer — device-side trace of the Cholesky / int8-engine kernels (diagnostics;
 * works inside CUDA-graph replays, where events between launches are unavailable).
 * records: device buffer of `capacity` 40-byte records, zeroed by the caller, or NULL to
 * turn tracing off.  Record 0's first uint64 counts appended records; each record i >= 1 is
 * {uint64 gridid, uint64 t_begin_ns, uint64 t_end_ns (globaltimer), int32 kind, int32 tag,
 * int32 sm, int32 0}, one per CTA, written by its thread 0 (kinds: paper_2510_08430_b200/
 * _lib.py TRACE_KINDS).  Appends beyond capacity are dropped.  Process-wide; the buffer
 * must outlive every launch made while it is installed. */
SR_API sr_status sr_trace_buffer(void* records, int64_t capacity);

/* sr_graph_capture_begin / sr_graph_capture_end / sr_graph_launch / sr_graph_destroy —
 * CUDA-graph capture of any sequence of the calls above, instantiated with per-node
 * priorities (cudaGraphInstantiateFlagUseNodePriority) so that the blocked solves' panel
 * chain keeps its higher stream priority over the off-chain updates inside the graph (a
 * graph instantiated without the flag runs every node at the priority of the stream it is
 * launched into).  begin: `stream` must be a non-default stream; the calls that follow on
 * it (and on the side streams they fork) are recorded, not run.  end: *graph_exec receives
 * an opaque executable graph owned by the caller (sr_graph_destroy frees it).  launch: runs
 * it on `stream`; the buffers and the workspace captured must still be valid.  Errors as
 * above (capture failures surface as SR_ERR_CUDA from end). */
SR_API sr_status sr_graph_capture_begin(void* stream);
SR_API sr_status sr_graph_capture_end(void* stream, void** graph_exec);
SR_API sr_status sr_graph_launch(void* graph_exec, void* stream);
SR_API sr_status sr_graph_destroy(void* graph_exec);

/* ---------------------------------------------------------------- stage (1) ---
 * sr_jacobian — PAPER.md §2 Eq. 2 "O_i(x) = d_{theta_i} log psi_theta(x)".
 *   theta    complex [n_p]                       network parameters (layout above)
 *   spins    int8 [n_samples][widths[0]]
 *   log_psi  complex [n_samples]   (out)         ln psi(x_k)
 *   O        complex [n_samples][ldo] (out)      row k = O(x_k); columns [0, n_p) written
 *   ldo      >= n_p (elements)
 * Holomorphic derivative; block l columns: W_l (j*fan_in+i) then b_l.  */
SR_API size_t sr_jacobian_workspace_bytes(int n_layers, const int32_t* widths /*host*/,
                                          int64_t n_samples);
SR_API sr_status sr_jacobian(int n_layers, const int32_t* widths /*host*/, const double* theta,
                             const int8_t* spins, int64_t n_samples, double* log_psi, double* O,
                             int64_t ldo, void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- stage (2) ---
 * sr_local_energy — PAPER.md Eq. 1 local energy with the same network evaluated on
 * every connected configuration x' (x with an anti-aligned bonded pair swapped):
 *   E_loc(x) = sum_b J_b [ s_i s_j + (1 - s_i s_j) psi(x^{ij})/psi(x) ].
 *   log_psi  complex [n_samples] (in)  ln psi of the samples (from sr_jacobian)
 *   e_loc    complex [n_samples] (out) */
SR_API size_t sr_local_energy_workspace_bytes(int n_layers, const int32_t* widths /*host*/,
                                              int64_t n_samples, int64_t n_bonds);
SR_API sr_status sr_local_energy(int n_layers, const int32_t* widths /*host*/,
                                 const double* theta, int64_t n_bonds, const int32_t* bonds_ij,
                                 const double* bond_j, const int8_t* spins, int64_t n_samples,
                                 const double* log_psi, double* e_loc, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- stage (3) ---
 * sr_center_force — PAPER.md Eq. 2 centring (Delta O_i = O_i - <O_i>) and the force
 *   F_i = sum_k w_k conj(Obar_ki) (E_loc,k - E),  E = sum_k w_k E_loc,k.
 *   O        complex [n_samples][ldo] (in/out)  O on entry, A = sqrt(w) Obar on exit
 *   weights  double [n_samples] or NULL (uniform)
 *   e_loc    complex [n_samples] (in)
 *   energy   complex [1] (out)            E
 *   e_tilde  complex [n_samples] (out)    e_k = sqrt(w_k) (E_loc,k - E)
 *   F        complex [n_p] (out) */
SR_API size_t sr_center_force_workspace_bytes(int64_t n_samples, int64_t n_p);
SR_API sr_status sr_center_force(int64_t n_samples, int64_t n_p, double* O, int64_t ldo,
                                 const double* weights, const double* e_loc, double* energy,
                                 double* e_tilde, double* F, void* workspace,
                                 size_t workspace_bytes, void* stream);

/* Sample-sharded form of stage (3) (one call per rank; BASELINE.json north_star:
 * "samples shard naturally").  n_total samples over all ranks; weights == NULL means
 * uniform 1/n_total, else the rank's slice of global weights.
 *   sr_column_moments       writes one moments row, complex [2*n_p + 2]:
 *                           [ <O>_hi (n_p) | <O>_lo (n_p) | E_hi | E_lo ], the rank's
 *                           contribution sum_{k local} w_k O_k and sum_{k local} w_k E_k as
 *                           double-double pairs (reading R7: the centring cancels
 *                           up to ~6 digits, so the mean is carried beyond double precision).
 *   (all-gather the rows of all ranks), then
 *   sr_center_force_global  sums the n_parts rows in double-double, and writes
 *                           A_k = sqrt(w_k)(O_k - <O>) in place, e_tilde_k = sqrt(w_k)(E_k - E),
 *                           energy = E (complex [1], may be NULL) and
 *                           F_partial = sum_{k local} conj(A_k) e_k   (all-reduce -> F).
 * Workspace: sr_column_moments_workspace_bytes(n_local, n_p) for both. */
SR_API size_t sr_column_moments_workspace_bytes(int64_t n_local, int64_t n_p);
SR_API sr_status sr_column_moments(int64_t n_local, int64_t n_total, int64_t n_p, const double* O, int64_t ldo,
                                   const double* weights, const double* e_loc, double* moments,
                                   void* workspace, size_t workspace_bytes, void* stream);
SR_API sr_status sr_center_force_global(int64_t n_local, int64_t n_total, int64_t n_p, double* O, int64_t ldo,
                                        const double* weights, const double* e_loc, int n_parts,
                                        const double* moments, double* energy, double* e_tilde,
                                        double* F_partial, void* workspace, size_t workspace_bytes,
                                        void* stream);

/* ---------------------------------------------------------------- stage (4) ---
 * sr_block_qgt — PAPER.md Eq. 3, S_l = <O_l^dag O_l> - <O_l^dag><O_l>, computed per
 * layer block from the centred, weighted Jacobian A (stage 3 output): S_b = A_b^H A_b.
 *   block_offsets (host) int64 [n_blocks+1], column ranges of the blocks in A
 *   S        complex, blocks packed back to back: block b is n_b x n_b row-major at
 *            element offset sum_{c<b} n_c^2; both triangles written (Hermitian),
 *            diagonal imaginary parts exactly 0.
 *   n_samples = 0 writes S = 0 (A may then be NULL; sr_block_qgt_i8 needs no workspace). */
SR_API size_t sr_block_qgt_workspace_bytes(int n_blocks, const int64_t* block_offsets /*host*/);
SR_API sr_status sr_block_qgt(int64_t n_samples, int n_blocks,
                              const int64_t* block_offsets /*host*/, const double* A, int64_t lda,
                              double* S, void* workspace, size_t workspace_bytes, void* stream);

/* sr_block_qgt_i8 — the same S_b = A_b^H A_b (same layout and contract as sr_block_qgt) on
 * the tcgen05 integer tensor cores: every column of A is scaled by a power of two, split
 * into seven exact int8 digit slices (54 bits), the slice products sum_{p+q<=6} C_p^T Y_q
 * are accumulated EXACTLY in int32 TMEM by tcgen05.mma kind::i8 and recombined in FP64
 * (the Ozaki splitting scheme; DESIGN.md §5 and reading R10).  Error: at most ~2^-51 of
 * n_samples * max_k|A_ki| * max_k|A_kj| per entry, the size of an FP64 dot product's.
 * Workspace: sr_block_qgt_i8_workspace_bytes(n_samples, ...) bytes (digit slices,
 * 42 bytes per sample per parameter of the largest group of blocks, plus column scales).
 * Non-finite input: an Inf or NaN anywhere in column i of A makes row i and column i of
 * S_b NaN (the other entries are unaffected), as with an FP64 Gram.
 * Errors: SR_ERR_INVALID on bad sizes, SR_ERR_WORKSPACE if the workspace is too small. */
SR_API size_t sr_block_qgt_i8_workspace_bytes(int64_t n_samples, int n_blocks,
                                              const int64_t* block_offsets /*host*/);
SR_API sr_status sr_block_qgt_i8(int64_t n_samples, int n_blocks,
                                 const int64_t* block_offsets /*host*/, const double* A, int64_t lda,
                                 double* S, void* workspace, size_t workspace_bytes, void* stream);

/* sr_block_qgt_i8_acc — S_b += A_b^H A_b (same layout, engine, workspace and errors as
 * sr_block_qgt_i8; S must hold a previous result): the sample-chunked step
 * (parallel.ChunkedStep) sums the Grams of sample chunks whose centred Jacobians are formed
 * one after another, so that N_s x n_p never has to be resident (configs[4]: 206 GB). */
SR_API sr_status sr_block_qgt_i8_acc(int64_t n_samples, int n_blocks, const int64_t* block_offsets /*host*/,
                                     const double* A, int64_t lda, double* S, void* workspace,
                                     size_t workspace_bytes, void* stream);

/* sr_set_gram_engine — engine of the dense contractions: sr_step's stage (4), the Grams of
 * the comparison solves (the full QGT A^H A of sr_full_qgt_solve, the NTK A A^H of
 * sr_ntk_solve) and the deferred trailing updates (A_22 -= L_21 L_21^H, K = 512) of every
 * Cholesky factorisation (sr_block_solve, sr_full_qgt_solve, sr_ntk_solve, sr_step).
 * SR_GRAM_FP64 = FP64 DMMA tensor cores (sr_block_qgt), SR_GRAM_INT8 = int8 tcgen05 digit
 * slices (sr_block_qgt_i8; for the trailing updates the rows of each L_21 strip are
 * scaled and split the same way).  Process-wide; returns the previous setting, or -1 for
 * an unknown engine (setting unchanged).  Default: SR_GRAM_INT8. */
#define SR_GRAM_FP64 0
#define SR_GRAM_INT8 1
SR_API int sr_set_gram_engine(int engine);
SR_API int sr_get_gram_engine(void);

/* ---------------------------------------------------------------- stage (5) ---
 * sr_block_solve — PAPER.md §2: "Each block S_l is inverted independently, using a
 * uniform diagonal shift lambda", (S_b + lambda I) dtheta_b = -F_b, by a blocked,
 * batched Cholesky factorisation (all blocks advance together).
 *   S       packed blocks as written by sr_block_qgt (read only; lower triangle used)
 *   F       complex [n_p];   dtheta complex [n_p] (out);   info int32 [1] (out) or NULL */
SR_API size_t sr_block_solve_workspace_bytes(int n_blocks, const int64_t* block_offsets /*host*/);
SR_API sr_status sr_block_solve(int n_blocks, const int64_t* block_offsets /*host*/,
                                const double* S, const double* F, double lambda, double* dtheta,
                                int32_t* info, void* workspace, size_t workspace_bytes,
                                void* stream);

/* sr_block_qgt_solve — stages (4) and (5) fused per block (the per-block schedule):
 * for b = 0, 1, ...: S_b = A_b^H A_b (Eq. 3) is formed straight into block b's
 * padded Cholesky matrix on the selected Gram engine and (S_b + lambda I) dtheta_b = -F_b is
 * solved (§2, "Each block S_l is inverted independently") before block b+1's Gram.
 * Same result as sr_block_qgt followed by sr_block_solve up to the FP64 summation order of
 * the Cholesky updates (a block solved alone uses the single-block lookahead; measured within
 * 1e-12 relative), but the workspace holds ONE block -- the largest -- instead of every S_b and its
 * factor copy: configs[4]'s eight blocks need 10.6 GB + digit slices instead of 157 GB.
 * Blocks run one after another (no S_b is kept; nothing to inspect).
 *   A        complex [n_samples][lda], the centred, weighted Jacobian (stage 3 output)
 *   F        complex [n_p];  dtheta complex [n_p] (out);  info int32 [1] (out) or NULL:
 *            0, or the global row + 1 of the first non-positive pivot of the first
 *            failing block.
 * Workspace: sr_block_qgt_solve_workspace_bytes(n_samples, ...).  Errors as sr_block_solve. */
SR_API size_t sr_block_qgt_solve_workspace_bytes(int64_t n_samples, int n_blocks,
                                                 const int64_t* block_offsets /*host*/);
SR_API sr_status sr_block_qgt_solve(int64_t n_samples, int n_blocks, const int64_t* block_offsets /*host*/,
                                    const double* A, int64_t lda, const double* F, double lambda,
                                    double* dtheta, int32_t* info, void* workspace,
                                    size_t workspace_bytes, void* stream);

/* sr_set_step_schedule — how sr_step / sr_step_host run stages (4)-(5):
 * SR_SCHED_BATCHED (default): every S_b is formed (one grouped Gram launch), then all blocks
 *   are factorised together on concurrent streams; sr_step_s_offset() locates the S blocks.
 * SR_SCHED_PER_BLOCK: sr_block_qgt_solve (one block at a time, O(max n_b^2) memory); the
 *   step workspace drops sum_b n_b^2 complex of S and all but one factor (configs[4] at
 *   8192 samples: 42 GB instead of 189 GB); sr_step_s_offset() returns SIZE_MAX.
 * Process-wide, read by the workspace queries too: query and call under the same setting.
 * Returns the previous setting, or -1 for an unknown schedule (unchanged). */
#define SR_SCHED_BATCHED 0
#define SR_SCHED_PER_BLOCK 1
SR_API int sr_set_step_schedule(int schedule);
SR_API int sr_get_step_schedule(void);

/* ------------------------------------------------------- comparison paths ---
 * sr_full_qgt_solve — PAPER.md §2 "S . delta theta = -F" with the full n_p x n_p QGT:
 *   S = A^H A formed in the workspace, (S + lambda I) dtheta = -F by Cholesky.
 *   S_out complex [n_p][n_p] (out, optional, may be NULL): copy of S (both triangles). */
SR_API size_t sr_full_qgt_solve_workspace_bytes(int64_t n_samples, int64_t n_p);
SR_API sr_status sr_full_qgt_solve(int64_t n_samples, int64_t n_p, const double* A, int64_t lda,
                                   const double* F, double lambda, double* dtheta,
                                   double* S_out, int32_t* info, void* workspace,
                                   size_t workspace_bytes, void* stream);

/* sr_ntk_solve — PAPER.md §1 sample-space reformulation ("inverting the neural
 * tangent kernel (NTK)-like matrix whose size depends on the number of Monte Carlo
 * samples"): T = A A^H (n_samples x n_samples), (T + lambda I) y = e,
 * dtheta = -A^H y.  Equal to sr_full_qgt_solve by the push-through identity.
 *   e_tilde complex [n_samples] (stage 3 output);  T_out optional copy of T. */
SR_API size_t sr_ntk_solve_workspace_bytes(int64_t n_samples, int64_t n_p);
SR_API sr_status sr_ntk_solve(int64_t n_samples, int64_t n_p, const double* A, int64_t lda,
                              const double* e_tilde, double lambda, double* dtheta,
                              double* T_out, int32_t* info, void* workspace,
                              size_t workspace_bytes, void* stream);

/* sr_gram_nh — C = A B^H (complex; C[i][j] = sum_k A[i][k] conj(B[j][k])) for row-major
 * A (m x k, lda), B (n x k, ldb), C (m x n, ldc), on the FP64 DMMA tile engine: the
 * block-row T_r,s = A_r A_s^H of the sample-space (NTK) matrix when samples are sharded
 * over ranks (parallel.ShardedStep.ntk_solve).  m, n or k = 0 is allowed (C is left
 * untouched for m or n = 0, zeroed for k = 0). */
SR_API sr_status sr_gram_nh(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                            int64_t ldb, double* C, int64_t ldc, void* stream);

/* sr_aHv — out = alpha A^H v (complex) for A (n_rows x n_p, lda), v [n_rows], out [n_p]:
 * the final product dtheta = -A^H y of the NTK solve, per rank on its own rows (summed over
 * ranks by the caller).  Deterministic (fixed-order chunk reduction). */
SR_API size_t sr_aHv_workspace_bytes(int64_t n_rows, int64_t n_p);
SR_API sr_status sr_aHv(int64_t n_rows, int64_t n_p, const double* A, int64_t lda, const double* v, double alpha,
                        double* out, void* workspace, size_t workspace_bytes, void* stream);

/* Matrix-free full-QGT solve support (the sharded comparison path parallel.full_qgt_cg):
 * (S + lambda I) dtheta = -F with S = A^H A applied as A^H (A p) by conjugate gradients,
 * never formed (configs[3]'s full QGT is 146 GB).  With samples sharded, S p = sum_r
 * A_r^H (A_r p) -- each rank's sr_av + sr_aHv, then one all-reduce of n_p values.
 *   sr_av      out = alpha A v for A (n_rows x n_p, lda), v [n_p], out [n_rows]; one warp per
 *              row, fixed summation order (deterministic).
 *   sr_zdotc   out (device complex [1]) = sum_i conj(x_i) y_i, fixed-order two-level
 *              reduction; workspace sr_zdotc_workspace_bytes().
 *   sr_cg_axpy y += sign * (num / den) x ;  sr_cg_xpby  y = x + (num / den) y
 *              (num, den: device complex scalars, e.g. sr_zdotc outputs; the CG step sizes
 *              are formed on the device, no host round trip). */
SR_API sr_status sr_av(int64_t n_rows, int64_t n_p, const double* A, int64_t lda, const double* v, double alpha,
                       double* out, void* stream);
SR_API size_t sr_zdotc_workspace_bytes(void);
SR_API sr_status sr_zdotc(int64_t n, const double* x, const double* y, double* out, void* workspace,
                          size_t workspace_bytes, void* stream);
SR_API sr_status sr_cg_axpy(int64_t n, const double* x, double* y, const double* num, const double* den,
                            double sign, void* stream);
SR_API sr_status sr_cg_xpby(int64_t n, const double* x, double* y, const double* num, const double* den,
                            void* stream);

/* Distributed dense full-QGT solve support (parallel.dist_full_qgt: S held by block rows
 * across ranks, right-looking blocked Cholesky with the panels broadcast; §2
 * "S . delta theta = -F" with the full QGT):
 *   sr_gram_tn      C = A^H B for A (k x m, lda) and B (k x n, ldb) row-major, C (m x n, ldc):
 *                   the partial QGT rows A_r[:, rows]^H A_r[:, cols] (FP64 DMMA).  k = 0
 *                   writes C = 0.
 *   sr_gram_nh_sub  C -= A B^H for A (m x k), B (n x k), C (m x n) row-major (FP64 DMMA): the
 *                   trailing update S_qj -= L_qp L_jp^H.
 *   sr_chol_inv     M + lambda I = L L^H for one n x n Hermitian block M (contiguous, ld n,
 *                   lower triangle read) by the library's blocked Cholesky, and the explicit
 *                   inverse Linv = L^{-1} (one CTA per 64-column tile column, forward
 *                   substitution with the factorisation's 64x64 diagonal-tile inverses):
 *                   L (ldl) and Linv (ldv) are written lower triangular with zeros above;
 *                   info as for sr_block_solve.  Workspace sr_chol_inv_workspace_bytes(n). */
SR_API sr_status sr_gram_tn(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                            int64_t ldb, double* C, int64_t ldc, void* stream);
SR_API sr_status sr_gram_nh_sub(int64_t m, int64_t n, int64_t k, const double* A, int64_t lda, const double* B,
                                int64_t ldb, double* C, int64_t ldc, void* stream);
/* The same panels on the int8 digit-slice engine (exact to FP64 level, as sr_block_qgt_i8):
 *   sr_cols_i8_prepare  splits all n_cols columns of A (n_samples x n_cols, lda) into the
 *                       workspace (sr_cols_i8_workspace_bytes: 21 bytes per sample and column);
 *   sr_cols_i8_gram     C (m x n, ldc) = (or += with accumulate != 0) A[:, row0:row0+m]^H A[:, 0:n]
 *                       on the prepared workspace (row0 + m <= n_cols, n <= n_cols);
 *   sr_rows_i8_prepare  splits the rows of L (rows x K row-major, K <= 8192) into the workspace
 *                       (sr_rows_i8_sub_workspace_bytes);
 *   sr_rows_i8_sub      C (m x n, ldc) -= L[row0:row0+m] L[0:n]^H on the prepared workspace:
 *                       the trailing update of a rank's panel row by the broadcast panel column
 *                       (the Cholesky trailing-update kernel, gram_i8<MODE_SUB>, on a rectangle). */
SR_API size_t sr_cols_i8_workspace_bytes(int64_t n_samples, int64_t n_cols);
SR_API sr_status sr_cols_i8_prepare(int64_t n_samples, int64_t n_cols, const double* A, int64_t lda, void* workspace,
                                    size_t workspace_bytes, void* stream);
SR_API sr_status sr_cols_i8_gram(int64_t n_samples, int64_t n_cols, int64_t row0, int64_t m, int64_t n, double* C,
                                 int64_t ldc, int accumulate, void* workspace, size_t workspace_bytes, void* stream);
SR_API size_t sr_rows_i8_sub_workspace_bytes(int64_t rows, int64_t K);
SR_API sr_status sr_rows_i8_prepare(int64_t rows, int64_t K, const double* L, int64_t ldl, void* workspace,
                                    size_t workspace_bytes, void* stream);
SR_API sr_status sr_rows_i8_sub(int64_t rows, int64_t K, int64_t row0, int64_t m, int64_t n, double* C, int64_t ldc,
                                void* workspace, size_t workspace_bytes, void* stream);
SR_API size_t sr_chol_inv_workspace_bytes(int64_t n);
SR_API sr_status sr_chol_inv(int64_t n, const double* M, double lambda, double* L, int64_t ldl, double* Linv,
                             int64_t ldv, int32_t* info, void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- full step ---
 * sr_step — stages (1)-(5) back to back on device buffers (uniform weights):
 *   theta complex [n_p], spins int8 [n_samples][N], bonds as in stage (2);
 *   dtheta complex [n_p] (out), energy complex [1] (out).
 * The workspace holds O/A, E_loc, S blocks and the factor storage; the S blocks sit
 * at offset sr_step_s_offset() of the workspace (for inspection; SIZE_MAX under the
 * per-block schedule, sr_set_step_schedule, which keeps no S). */
SR_API size_t sr_step_workspace_bytes(int n_layers, const int32_t* widths /*host*/,
                                      int64_t n_samples, int64_t n_bonds);
SR_API size_t sr_step_s_offset(int n_layers, const int32_t* widths /*host*/, int64_t n_samples,
                               int64_t n_bonds);
SR_API sr_status sr_step(int n_layers, const int32_t* widths /*host*/, const double* theta,
                         const int8_t* spins, int64_t n_samples, int64_t n_bonds,
                         const int32_t* bonds_ij, const double* bond_j, double lambda,
                         double* dtheta, double* energy, void* workspace, size_t workspace_bytes,
                         void* stream);

/* sr_step_host — sr_step with HOST inputs and outputs (theta_h, spins_h, bonds_ij_h,
 * bond_j_h in; dtheta_h, energy_h out).  Copies in, runs the step, copies out, and
 * synchronises `stream` before returning.  Host buffers should be pinned for
 * asynchronous copies.  Device workspace as for sr_step plus
 * sr_step_host_extra_bytes() for the staged inputs/outputs.  The device part of the step
 * is captured into a CUDA graph on the first call for a given (workspace, widths,
 * n_samples, n_bonds, lambda, Gram engine) and replayed on later calls (up to 4 cached;
 * environment SR_STEP_GRAPH=0 disables it); the workspace must not be freed while its
 * graph is cached unless the same address is never passed again. */
SR_API size_t sr_step_host_extra_bytes(int n_layers, const int32_t* widths /*host*/,
                                       int64_t n_samples, int64_t n_bonds);
SR_API sr_status sr_step_host(int n_layers, const int32_t* widths /*host*/,
                              const double* theta_h, const int8_t* spins_h, int64_t n_samples,
                              int64_t n_bonds, const int32_t* bonds_ij_h, const double* bond_j_h,
                              double lambda, double* dtheta_h, double* energy_h,
                              void* workspace, size_t workspace_bytes, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SR_BLOCK_H */

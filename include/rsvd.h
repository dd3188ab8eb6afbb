/*
 * rsvd.h — C ABI of the B200 (sm_100a) pass-efficient randomized SVD library (librsvd.so).
 *
 * Implements the matrix-view hot path of Bjarkason, "Pass-efficient randomized algorithms for
 * low-rank matrix approximation using any number of views" (arXiv 1804.07531).  Citations are
 * PAPER.md line numbers (P:<line>) with the algorithm / section they fall in.
 *
 *   rsvd_subspace      Alg. 2, generalized subspace iteration, any v >= 2
 *   rsvd_block_krylov  Alg. 9, generalized block Krylov, any v >= 2
 *   rsvd_single_pass   Alg. 7, 1-view Tropp variant with l_c;
 *                      minimum-variance l_c; Alg. 8 Woolfe variant
 *   rsvd_single_pass_extended  extended 1-view sketch, bwz / bwz2
 *   rsvd_row_stream    single pass over the rows of A
 *   rsvd_block_krylov_rows  block Krylov with A^T A X from one row pass
 *   rsvd_nystrom, rsvd_pinched  normal-matrix TEVDs, Alg. 4 / Alg. 5
 *   rsvd_plan          single-pass oversampling plans (host only)
 *
 * plus the primitives they are built from, exported for unit-level parity tests:
 *   rsvd_view          Y = A X  or  Z = A^T Y        (one matrix view)
 *   rsvd_view_fused    Y_c = A Omega and Y_r = A^T Phi from one read of A   (P:669 a)+b))
 *   rsvd_orth          [Q, R] = qr(Y) by CholeskyQR2
 *   rsvd_core_svd      [U, S, V] = tsvd(M) of a small core by one-sided Jacobi
 *
 * NOTATION.  The ABI uses BASELINE.json's letters: k = target rank (paper p), p = oversampling
 * (paper l), l = k + p = sketch width; l2 = co-range sketch width of the single-pass method
 * (paper p + l_2); lc in [0, p] = the truncation parameter (paper l_c; lc == p is the Tropp
 * baseline).
 *
 * LAYOUTS.
 *   A      row-major, m_local x n, row stride lda >= n (elements).
 *   tall-skinny arrays (Omega, Phi, U, V, X, Y, Q) are COLUMN-major: element (i, j) at
 *          ptr[j * ld + i], ld >= rows; every test / basis vector is contiguous.
 *   small square arrays (R, core U/V) are column-major with ld = their row count.
 * POINTERS.  Every array argument may be device memory or host memory (pageable or pinned); the
 *   library detects the kind with cudaPointerGetAttributes and stages host data through its own
 *   device workspace (host<->device copies then happen inside the call).  Device pointers must
 *   be on the ctx's device.
 * DTYPE.  All arrays of one call share A's dtype, RSVD_F64 or RSVD_F32.  fp32 views run on the
 *   tcgen05 tensor cores in 3xTF32; everything between views is computed in fp64 and the
 *   outputs are rounded to fp32.  Other dtypes return RSVD_E_DTYPE.
 * OWNERSHIP.  The caller owns every array; nothing is retained after return.  The ctx owns its
 *   workspace (grown on demand, freed by rsvd_destroy) and its CUDA-graph cache.
 * SYNCHRONISATION.  Calls are synchronous: one stream synchronisation at the end; no host
 *   round trip between views (the whole algorithm is one CUDA graph launch after the first call
 *   with a given signature).  With RSVD_ASYNC a call only enqueues; rsvd_wait completes it.
 * MULTI-GPU.  After rsvd_comm_init every algorithm call is a collective over the ranks: A is
 *   row-sharded (rank r holds rows [row0, row0 + m_local), the shards tiling [0, m) in rank
 *   order); U is returned row-sharded like A; S and V are replicated and bitwise identical on
 *   all ranks.  Gram matrices and the partial co-range views A^T Y are summed with NCCL
 *   all-reduce.  rsvd_subspace / rsvd_block_krylov with N > 1 ranks also shard the n-long side
 *   (SURVEY §8(e)): every n x w block lives as N row chunks of ceil(n / N) rounded up to 32 rows
 *   (rank r: rows [r cs, min((r + 1) cs, n))); A^T Y is reduce-scattered into the chunks, the
 *   basis is all-gathered before the next A X, V is all-gathered before it is returned
 *   (replicated, bitwise equal on all ranks).  Not used when some rank would own no chunk
 *   (n <= (N - 1) cs) or with RSVD_NO_SHARD_N=1 (environment); the caller's Omega (n x l) is
 *   passed whole on every rank either way.  A call waits for its collectives by polling ncclCommGetAsyncError: an
 *   asynchronous NCCL error, or no completion within RSVD_COMM_TIMEOUT_S seconds (environment,
 *   default 600), aborts the communicator and returns RSVD_E_NCCL (the ctx then needs a new one).
 * DETERMINISM.  Bitwise run-to-run reproducible for fixed inputs, rank count and SM budget
 *   (rsvd_set_sm_limit changes the reduction splits, i.e. the rounding), except the
 *   single-pass Y_c accumulation when the deterministic partial buffers would exceed the memory
 *   budget (info->nondeterministic = 1; never for the BASELINE configs C1-C3).
 * ERRORS.  Every function returns an int status (RSVD_OK = 0 or a negative RSVD_E_*); no C++
 *   exception crosses the ABI.  rsvd_last_error(ctx) gives a one-line detail.  Outputs are
 *   defined only when the call returns RSVD_OK.
 */
#ifndef RSVD_H_
#define RSVD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rsvd_ctx rsvd_ctx;

enum { RSVD_F32 = 1, RSVD_F64 = 2 };
enum { RSVD_INPUT_A = 0, RSVD_INPUT_AT = 1 };          /* matrix Alg. 2/9 is applied to */
enum { RSVD_GOAL_SVD = 0, RSVD_GOAL_LEFT = 1, RSVD_GOAL_RIGHT = 2, RSVD_GOAL_NORMAL = 3 };
enum {
  RSVD_OK = 0,
  RSVD_E_ARG = -1,       /* invalid argument (shape, rank, views, ld, alignment, pointer)   */
  RSVD_E_DTYPE = -2,     /* unsupported dtype                                                */
  RSVD_E_CUDA = -3,      /* CUDA runtime / driver failure                                    */
  RSVD_E_NCCL = -4,      /* NCCL unavailable or failed                                       */
  RSVD_E_NOMEM = -5,     /* device workspace allocation failed                               */
  RSVD_E_NUMERIC = -6,   /* numerical failure (Jacobi not converged, singular R-hat in Alg. 7) */
  RSVD_E_STATE = -7      /* ctx misuse (e.g. comm already initialised)                       */
};
/* ENVIRONMENT.  A/B measurement switches, read once per process; the defaults are the tuned
 * paths and no switch changes results beyond rounding:
 *   RSVD_NO_ORTH_CLUSTER=1        CholeskyQR without the 16-CTA cluster kernel (w <= 64)
 *   RSVD_CHOL_BIG_FROM=w          blocked Cholesky (k_chol_big) from this width (default 161)
 *   RSVD_JACOBI_CLUSTER_FROM=c    cluster block Jacobi from this core width (default 129)
 *   RSVD_JACOBI_OLD_MID=1         previous 65..128-column Jacobi kernel
 *   RSVD_ROW_PANEL_MB=x           row-panel size of rsvd_row_stream (default 48)          */
/* flags */
#define RSVD_SQUARED      1u   /* S := sigma^2  (normal-matrix estimate A^T A ~ V S V^T) */
#define RSVD_NO_GRAPH     2u   /* enqueue kernels directly instead of replaying a CUDA graph    */
#define RSVD_PROFILE      4u   /* record CUDA events around every view kernel (info->view_*)     */
#define RSVD_CORE_NO_J    16u  /* rsvd_core_svd: V = M^T U S^-1 instead of accumulated rotations  */
#define RSVD_ASYNC        32u  /* enqueue only: outputs and info complete after rsvd_wait(ctx) */
#define RSVD_WOOLFE       64u  /* rsvd_single_pass: Alg. 8 (Woolfe variant) instead of Alg. 7   */
#define RSVD_ORTH_SHIFTED 128u /* rsvd_orth: shifted CholeskyQR3 (a shift pass before the two
                                  CholeskyQR passes; what Alg. 9's projected Krylov blocks use) */
#define RSVD_ONE_READ     256u /* single pass, fp64, l <= 128, l2 <= 256: Y_c and Y_r from ONE read
                                  of A on the thread-block-cluster kernel, whose partial traffic is
                                  the lowest (l / (64 CL) of A's bytes).  Without it: the one-CTA
                                  fused kernel for l <= 72, l2 <= 144 and two view launches above,
                                  faster on device-resident A                    */
#define RSVD_LC_MINVAR    (-2) /* rsvd_single_pass lc: minimum-variance l_c          */
#define RSVD_EXT_BWZ      0    /* rsvd_single_pass_extended: Eq. (bwz)               */
#define RSVD_EXT_BWZ2     1    /* rsvd_single_pass_extended: Eq. (bwzimproved)       */

typedef struct {
  int32_t dtype;          /* RSVD_F64 or RSVD_F32                                         */
  int32_t reserved;
  int64_t m, n;           /* global shape of A                                            */
  int64_t m_local, row0;  /* this rank's rows [row0, row0 + m_local); single GPU: m, 0    */
  int64_t lda;            /* row stride of the local block in elements, >= n              */
  const void* data;       /* local block, device or host memory, never modified           */
} rsvd_mat;

typedef struct {
  int32_t status;               /* return value of the call                                 */
  int32_t views;                /* views of A used (v; 1 for the single pass)         */
  int64_t vectors;              /* matrix-vector products (Alg. 2: v l; Alg. 9: (v+floor(v/2)-1) l) */
  int32_t rank_deficient_cols;  /* columns zeroed by the guarded Cholesky (exact rank < l)   */
  int32_t jacobi_sweeps;        /* sweeps of the last core SVD                               */
  int32_t lc_used;              /* l_c of the single pass (the chosen one for RSVD_LC_MINVAR) */
  int32_t host_staged;          /* 1 if any argument was host memory; 2 if a device A had to be
                                   copied to a 16-byte-aligned block (TMA needs lda*8 % 16 == 0) */
  int32_t graph_replayed;       /* 1 if the call replayed a cached CUDA graph                 */
  int32_t nondeterministic;     /* 1 if atomics were used (see DETERMINISM)                   */
  int32_t view_launches;        /* view-kernel launches in the call                           */
  int32_t kernel_launches;      /* all librsvd kernels launched by the call (CUDA-graph kernel
                                   nodes; 0 with RSVD_NO_GRAPH / RSVD_PROFILE)                  */
  double  view_ms;              /* RSVD_PROFILE: summed device time of the view kernels      */
  double  view_bytes;           /* algorithmic bytes of A streamed by those kernels          */
  double  view_flops;           /* algorithmic flops of those kernels (2 m n w per view)     */
  double  total_ms;             /* RSVD_PROFILE: device time of the whole call               */
} rsvd_info;

/* ---- context ------------------------------------------------------------------------------- */
/* cuda_stream: the stream every call of this ctx is enqueued on.  NULL: the ctx creates its own
 * BLOCKING stream (cudaStreamDefault flags), which is ordered in both directions with the legacy
 * default stream (handle 0), so work queued there before a call (e.g. a PyTorch producer on the
 * default stream) completes before the call starts, and default-stream work queued after the
 * call waits for it.  A non-NULL stream is used as is: ordering against other streams is then
 * the caller's responsibility. */
int  rsvd_create(rsvd_ctx** ctx, int cuda_device, void* cuda_stream);
int  rsvd_destroy(rsvd_ctx* ctx);
const char* rsvd_strerror(int code);
const char* rsvd_last_error(const rsvd_ctx* ctx);
int  rsvd_version(void);                                /* 100 * major + minor               */
int  rsvd_sm_count(const rsvd_ctx* ctx);
/* Caps the SMs this ctx's persistent kernels are sized for (1 <= n; n >= the device's SM count
 * restores the default).  For several contexts running concurrently on one GPU: a smaller budget
 * for the off-critical-path calls leaves SMs to the critical one.  Results do not depend on it
 * beyond rounding (the reduction splits change).  Returns RSVD_E_ARG for n < 1. */
int  rsvd_set_sm_limit(rsvd_ctx* ctx, int n);
/* Completes a call made with RSVD_ASYNC on this ctx: synchronises the ctx stream, fills the
 * device-side fields of info (rank-deficient columns, Jacobi sweeps) and returns the call's
 * numerical status.  Until then the caller must not read the outputs nor modify the inputs,
 * and the ctx accepts no other call (RSVD_E_STATE).  Several contexts on different streams run
 * their asynchronous calls concurrently.  Returns RSVD_OK when nothing is pending. */
int  rsvd_wait(rsvd_ctx* ctx, rsvd_info* info);
/* Roofline denominators measured on this device: FP64 DMMA (mma.sync m8n8k4) throughput in
 * TFLOP/s (register operands, all SMs) and streaming HBM read bandwidth in GB/s (4 GiB buffer,
 * best of 5).  Allocates 4 GiB temporarily; synchronous. */
int  rsvd_probe_peaks(rsvd_ctx* ctx, double* dmma_tflops, double* read_gbs);
/* Orientation rule: returns RSVD_INPUT_A or RSVD_INPUT_AT.
 * RIGHT / NORMAL: v even -> A, v odd -> A^T;  LEFT: the reverse;  SVD: A.  Pure function. */
int  rsvd_recommend_input(int goal, int v);

/* ---- multi-GPU (NCCL, loaded at run time from libnccl.so.2) --------------------------------- */
int  rsvd_get_unique_id(void* id128);                  /* rank 0: fills 128 bytes             */
/* Collective over nranks processes (one per GPU): every rank passes the same 128-byte NCCL unique
 * id (rank 0's rsvd_get_unique_id, broadcast by the caller).  nranks == 1 also creates a
 * one-rank communicator: the calls then take the sharded code path (all-reduced Grams and
 * A^T Y partials, NCCL inside the CUDA graph) on a single GPU.  RSVD_E_STATE if already set. */
int  rsvd_comm_init(rsvd_ctx* ctx, int nranks, int rank, const void* id128);
int  rsvd_comm_nranks(const rsvd_ctx* ctx);
/* Loopback communicator: N virtual row shards of one A on ONE GPU (tests of the sharded path
 * without N GPUs).  rsvd_loop_create makes a group of 1 <= nranks <= 16 virtual ranks
 * (timeout_s <= 0: 120 s); each of N contexts joins it with rsvd_comm_init_loopback(ctx, loop, r)
 * and is then driven by ITS OWN host thread (every rank must make the same sequence of calls
 * with the same scalars, as with NCCL).  A collective is a host barrier of the N threads plus
 * cross-stream event waits, and sums the ranks' buffers in rank order 0..N-1 (identical bits on
 * every rank); no kernel waits on another kernel.  Loopback calls enqueue directly (no CUDA
 * graph).  A rank whose call fails aborts the group: peers blocked in a collective return
 * RSVD_E_NCCL (also after timeout_s without all ranks arriving).  rsvd_loop_destroy may be called
 * once every ctx has joined; the group lives until its last ctx is destroyed. */
typedef struct rsvd_loop rsvd_loop;
int  rsvd_loop_create(int nranks, double timeout_s, rsvd_loop** loop);
int  rsvd_loop_destroy(rsvd_loop* loop);
int  rsvd_comm_init_loopback(rsvd_ctx* ctx, rsvd_loop* loop, int rank);

/* ---- algorithms ----------------------------------------------------------------------------- */
/* Alg. 2.  k >= 1, p >= 0, l = k + p <= min(m, n), v >= 2.
 * input == RSVD_INPUT_A : Omega is n x l (replicated on all ranks);
 * input == RSVD_INPUT_AT: the algorithm runs on A^T and Omega is m_local x l (this rank's rows).
 * U (m_local x k, ldu >= m_local) and V (n x k, ldv >= n) are A's singular vectors in either
 * orientation; S (k) descending (sigma, or sigma^2 with RSVD_SQUARED).  U or V may be NULL. */
int rsvd_subspace(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, int input,
                  const void* Omega, int64_t ld_omega,
                  void* U, int64_t ldu, void* S, void* V, int64_t ldv,
                  unsigned flags, rsvd_info* info);

/* Alg. 9; same arguments.  Additionally the Krylov basis width (v/2) l (v even) or
 * ((v-1)/2) l (v odd) must not exceed the row count of its side (RSVD_E_ARG). */
int rsvd_block_krylov(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, int input,
                      const void* Omega, int64_t ld_omega,
                      void* U, int64_t ldu, void* S, void* V, int64_t ldv,
                      unsigned flags, rsvd_info* info);

/* Alg. 7, input = A.  Omega n x (k+p) replicated; Phi m_local x l2 (this rank's rows
 * of the co-range test matrix, P:667b); l2 >= k + p (P:663 l_2 >= l_1); lc in [0, p] or -1 (= p).
 *
 * lc = RSVD_LC_MINVAR: l_c = argmin_{0 <= l_c < p} Var[s(l_c)] (Eq. MinVar), chosen on
 *   the device from the one view's sketches (no second view): one SVD of Y_c, one QR of
 *   M = Phi^T Q_c U_c, the trial spectra of X(l_c) for l_c = 0..p (one CTA each), Var = unbiased
 *   sample variance, ties -> smallest l_c, 0/0 = 1 and a/0 = inf in s(l_c) (R19-R20);
 *   p = 0 gives l_c = 0.  The rest of Alg. 7 then runs at width k + p with the columns beyond
 *   k + l_c zeroed (identical to truncating).  info->lc_used returns the choice;
 *   info->rank_deficient_cols then also counts those zeroed columns.  Needs k + p <= 512.
 * flags & RSVD_WOOLFE: Alg. 8 instead: Q_c and Q_r both truncated to their k + l_c
 *   leading singular directions, Xh from (Phi^T Q_c) Xh = Y_r^T Q_r (QR), U = Q_c Uh, V = Q_r Vh.
 *   Not combinable with RSVD_LC_MINVAR (RSVD_E_ARG). */
int rsvd_single_pass(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int l2, int lc,
                     const void* Omega, int64_t ld_omega, const void* Phi, int64_t ld_phi,
                     void* U, int64_t ldu, void* S, void* V, int64_t ldv,
                     unsigned flags, rsvd_info* info);

/* Single pass over the rows of A: Y_c[i, :] = A[i, :] Omega and Yhat_r = sum_i
 * A[i, :]^T Y_c[i, :] from ONE pass over A's rows, Q_c R_c := Y_c, B^T = Yhat_r R_c^+ (TSVD
 * pseudo-inverse, singular values below 1e-12 sigma_max dropped), and the rank-k SVD of
 * Q_c B.  With R_c invertible this equals rsvd_subspace with v = 2 from half the reads of
 * A: the GPU walks A in row panels of <= 48 MB that stay in L2 between the two products (each
 * panel is read from HBM once).  Omega n x (k+p).  info->views = 1.  Same pointer, dtype, sharding
 * and error rules as rsvd_subspace (Yhat_r is all-reduced over the row shards). */
int rsvd_row_stream(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, const void* Omega, int64_t ld_omega,
                    void* U, int64_t ldu, void* S, void* V, int64_t ldv, unsigned flags, rsvd_info* info);

/* Block Krylov method for a matrix read row wise: A^T A X is evaluated in ONE pass
 * over A's rows (Y[i, :] = A[i, :] X, Z = sum_i A[i, :]^T Y[i, :], the row panels staying in L2
 * between the two products), so Alg. 9's Krylov blocks need about half the reads of A.
 *   v odd : K_r = [A^TA Omega, (A^TA)^2 Omega, ...] from (v-1)/2 row passes, Q_r = qr(K_r),
 *           Q_c R_c = A Q_r, tsvd(R_c): (v-1)/2 + 1 reads of A (Alg. 9: v views).
 *   v even: the same passes also give the range blocks: K_c = [A Omega, A Q^1, ...], Q_c = qr(K_c),
 *           Q_r R_r = A^T Q_c, tsvd(R_r): v/2 + 1 reads.
 * Equal to rsvd_block_krylov (input = A) up to rounding when the intermediate blocks have full
 * rank (the same Krylov subspaces).  input is always A; Omega n x (k+p); info->views = reads of A.
 * Same pointer, dtype, sharding (Z all-reduced over the row shards) and error rules as
 * rsvd_block_krylov. */
int rsvd_block_krylov_rows(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v,
                           const void* Omega, int64_t ld_omega,
                           void* U, int64_t ldu, void* S, void* V, int64_t ldv,
                           unsigned flags, rsvd_info* info);

/* Extended 1-view sketch: from ONE view of A, Y_c = A Omega (n x (k+p) Omega),
 * Y_r = A^T Phi (Phi m_local x l2) and Z = Xi_r^T A Xi_c (s x s), with Xi_r (m_local x s) and Xi_c
 * (n x s) the paper's SRFT matrices Phi_r, Phi_c, materialised dense by the caller and
 * applied as test matrices in the same view ([A Omega | A Xi_c] is one range product).  Then
 * Q_c R_c := Y_c, Q_r R_r := Y_r, U_c T_c := Xi_r^T Q_c, U_r T_r := Xi_c^T Q_r and
 *   variant RSVD_EXT_BWZ :   A ~ Q_c T_c^+ [[U_c^T Z U_r]]_k (T_r^T)^+ Q_r^T      (Eq. bwz)
 *   variant RSVD_EXT_BWZ2:   A ~ Q_c [[T_c^+ U_c^T Z U_r (T_r^T)^+]]_k Q_r^T      (Eq. bwzimproved)
 * returned as its rank-k SVD (U m_local x k, S k, V n x k).  ^+ drops singular values below
 * 1e-12 of the largest.  Requires l2 >= k + p and k + p <= s <= min(m, n, 512) (s >= p + l_1);
 * the paper assumes l_1 = l_2 (l2 = k + p) but any l2 >= k + p is accepted.  Same pointer, dtype
 * and error rules as rsvd_single_pass; info->views = 1. */
int rsvd_single_pass_extended(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int l2, int s,
                              const void* Omega, int64_t ld_omega, const void* Phi, int64_t ld_phi,
                              const void* Xi_r, int64_t ld_xi_r, const void* Xi_c, int64_t ld_xi_c, int variant,
                              void* U, int64_t ldu, void* S, void* V, int64_t ldv,
                              unsigned flags, rsvd_info* info);

/* Oversampling plans for the single pass from a sketch-size budget T = 2k + l_1 + l_2 (host only,
 * no GPU needed).  Writes the ABI arguments: *p = l_1, *l2 = k + l_2 (the co-range width), *lc.
 *   RSVD_PLAN_FLAT      Eq. (overflat)  P:610-618, lc = l_1        (needs T >= 2k + 6)
 *   RSVD_PLAN_DECAY     Eq. (overmed)   P:620-629, lc = l_1
 *   RSVD_PLAN_RAPID     Eq. (overrapid), lc = l_1
 *   RSVD_PLAN_BALANCED  l_1 = floor(T/2) - k, l_2 = T - 2k - l_1, lc = floor(alpha l_1)
 *                       (Eq. lcutfixedratio, P:716-722, 0 <= alpha <= 1); pass lc = RSVD_LC_MINVAR
 *                       to the single pass instead for the adaptive choice.
 * Returns RSVD_E_ARG for a budget below 2k + 6, k < 1 or alpha outside [0, 1]. */
enum { RSVD_PLAN_FLAT = 0, RSVD_PLAN_DECAY = 1, RSVD_PLAN_RAPID = 2, RSVD_PLAN_BALANCED = 3 };
int rsvd_plan(int scheme, int k, int T, double alpha, int* p, int* l2, int* lc);

/* ---------------------------------------------------------------------------------------------
 * Normal-matrix estimates A^T A ~ V diag(S) V^T (S = eigenvalues, descending), v >= 2 views.
 *
 * rsvd_nystrom   Alg. 4, modified prolonged (Nystrom) TEVD.  Q_r = orth(Omega) (v = 2),
 *                QrQc(A, v-2) (v even) or QrQc(A^T, v-2) (v odd) (Alg. 3); then
 *                Y_r = A^T (A Q_r), nu = 2.2e-16 ||Y_r||_2, Y_r += nu Q_r, B = Q_r^T Y_r,
 *                C_L = chol((B + B^T)/2), F = C_L^-1 Y_r^T, [~, Lam, V] = tsvd(F, k),
 *                S = max(Lam^2 - nu, 0).  Algebraically equal to rsvd_subspace with
 *                RSVD_SQUARED in the recommended orientation.
 *                Omega: n x (k+p) for even v, m_local x (k+p) for odd v (column-major).
 * rsvd_pinched   Alg. 5, modified pinched TEVD: Q_r = QrQc(A^T, v-1) (v even) or
 *                QrQc(A, v-1) (v odd), B_c = A Q_r, [S, V^] = tevd(B_c^T B_c, k), V = Q_r V^.
 *                Omega: m_local x (k+p) for even v, n x (k+p) for odd v.
 * S: k values (A's dtype), V: n x k (ldv >= n), either may be NULL.  Errors as rsvd_subspace.
 * ------------------------------------------------------------------------------------------- */
int rsvd_nystrom(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, const void* Omega, int64_t ld_omega, void* S,
                 void* V, int64_t ldv, unsigned flags, rsvd_info* info);
int rsvd_pinched(rsvd_ctx* ctx, const rsvd_mat* A, int k, int p, int v, const void* Omega, int64_t ld_omega, void* S,
                 void* V, int64_t ldv, unsigned flags, rsvd_info* info);

/* ---- primitives (single GPU; for unit tests and the benchmark's kernel timing) -------------- */

/* trans == 0: Y (m_local x w) = A X with X n x w;  trans == 1: Y (n x w) = A^T X with X m_local x w.
 * 1 <= w <= 1024 (wider views run as column chunks of 128 (fp64) / 512 (fp32) columns). */
int rsvd_view(rsvd_ctx* ctx, const rsvd_mat* A, int trans, const void* X, int64_t ldx, int w,
              void* Y, int64_t ldy, unsigned flags, rsvd_info* info);
/* Y_c (m_local x l) = A Omega (Omega n x l) and Y_r (n x l2) = A^T Phi (Phi m_local x l2), from one
 * read of A.  fp64: l <= 128 and l2 <= 256 (l > 72 or l2 > 144: the cluster kernel, whose Y_c
 * partials are reduced across a 16- or 8-CTA thread-block cluster).  fp32: RSVD_E_DTYPE. */
int rsvd_view_fused(rsvd_ctx* ctx, const rsvd_mat* A, const void* Omega, int64_t ld_omega, int l,
                    const void* Phi, int64_t ld_phi, int l2, void* Yc, int64_t ld_yc,
                    void* Yr, int64_t ld_yr, unsigned flags, rsvd_info* info);
/* In place: Y (rows x w) <- Q with Q^T Q = I, and R (w x w, column-major, may be NULL) with
 * Y_in = Q R, diag(R) >= 0.  Columns whose Cholesky pivot falls below the rank guard are set to
 * zero in Q (and their row of R is zero); their count is info->rank_deficient_cols.
 * flags | RSVD_ORTH_SHIFTED: shifted CholeskyQR3 (R = R_2 R_1 R_0), for blocks whose condition
 * number is too large for CholeskyQR2. */
int rsvd_orth(rsvd_ctx* ctx, int64_t rows, int w, void* Y, int64_t ldy, void* R, unsigned flags,
              rsvd_info* info);
/* M (r x c, column-major, ldm >= r, r >= c): M = U diag(S) V^T with U r x c, S c (descending),
 * V c x c.  One-sided Jacobi in one CTA; c <= 256, r <= 256. */
int rsvd_core_svd(rsvd_ctx* ctx, int r, int c, const void* M, int64_t ldm, void* U, void* S, void* V,
                  unsigned flags, rsvd_info* info);

#ifdef __cplusplus
}
#endif
#endif /* RSVD_H_ */

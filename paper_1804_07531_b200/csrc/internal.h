// Internal interfaces between the kernel files and the driver (not part of the ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/rsvd.h"

namespace rsvd {

constexpr int kMaxWT = 16;        // view kernels: w <= 128 per launch (wider -> column chunks)
constexpr int kFusedMaxL = 72;    // fused single-pass kernel: l <= 72 ...
constexpr int kFusedMaxL2T = 18;  // ... and l2 <= 144

enum { VIEW_AX = 0, VIEW_ATY = 1, VIEW_FUSED = 2 };

struct ViewArgs {
  const double* A;  // row-major rows x n, lda
  int64_t rows, n, lda;
  const double* X;  // AX: X^T (w x n, ldx); ATY: Y^T (w x rows, ldx)
  int64_t ldx;
  int w;
  double* out;      // column-major output (w x out_rows, ldo), slot s at out + s*slot_stride
  int64_t ldo, slot_stride;
  int S, KTS;       // reduction split (from plan_view)
  int grid_cap;     // persistent grid size (SM count)
  int a_keep = 0;   // A*X only: load A with evict_last (a row panel re-read from L2 by A^T Y next)
};

struct FusedArgs {
  const double* A;
  int64_t rows, n, lda;
  const double* Om;  // Omega^T: l x n, ldom
  int64_t ldom;
  int l;
  const double* Phi; // Phi^T: l2 x rows, ldphi
  int64_t ldphi;
  int l2;
  double* yc;        // Y_c^T partial slots (l x rows, ldyc) per column strip, or one buffer (atomic)
  int64_t ldyc, yc_slot_stride;
  int yc_atomic;
  double* yr;        // Y_r^T partial slots (l2 x n, ldyr) per row split
  int64_t ldyr, yr_slot_stride;
  int S, KTS;
  int grid_cap;
};

// Fused single pass for wide sketches (view_fused_cluster.cu): l <= 128, l2 <= 256, fp64, one read
// of A, Y_c partials reduced across a 16- (or 8-) CTA cluster through distributed shared memory.
struct FusedClArgs {
  const double* A;
  int64_t rows, n, lda;
  const double* Om;   // Omega^T: l x n, ldom
  int64_t ldom;
  int l;
  const double* Phi;  // Phi^T: l2 x rows, ldphi
  int64_t ldphi;
  int l2;
  double* yc_slots;   // per strip group: row-major rows x ldys partial of Y_c
  int64_t ldys, yc_slot_stride;
  double* yr;         // per row split: column-major n x l2 (ldyr) partial of Y_r
  int64_t ldyr, yr_slot_stride;
  int CL, NG, S, KTS, nclusters;   // from plan_fused_cl
};
bool fused_cl_supported(int l, int l2);
void plan_fused_cl(int64_t rows, int64_t n, int l, int l2, int sms, FusedClArgs* a);
int launch_view_fused_cl(const FusedClArgs& a, cudaStream_t st);
// out (column-major, ldo) = sum over NG row-major slots (rows x w, ld ldi) in slot order
int launch_slot_sum_rows(const double* in, int64_t ldi, int64_t slot_stride, int NG, int64_t rows, int w, double* out,
                         int64_t ldo, cudaStream_t st);

// fp32 A (view_tf32.cu): tcgen05 kind::tf32 views with the 3xTF32 split of both operands
constexpr int kMaxW32 = 512;      // widths per launch (wider -> column chunks)
struct ViewArgs32 {
  int kind;           // VIEW_AX or VIEW_ATY
  const float* A;     // row-major rows x n, lda (lda * 4 a multiple of 16 bytes)
  int64_t rows, n, lda;
  const float* Xhi;   // pre-split skinny operand, column-major [K x w] with ld ldx (K = n or rows)
  const float* Xlo;
  int64_t ldx;
  int w;
  float* out;         // fp32 partial slots, column-major (out_rows x w, ldo), slot j at out + j*slot_stride:
                      // one per accumulation chunk of kTf32Chunk stages of each unit (tf32_slots)
  int64_t ldo, slot_stride;
  int S, KTS;
  int grid_cap;
};
void plan_view_tf32(int kind, int64_t rows, int64_t n, int w, int grid_cap, int* S, int* KTS);
// number of fp32 partial slots of a planned view (S units x ceil(KTS / chunk) chunks per unit)
int tf32_slots(int S, int KTS);
// out (fp64) = sum of NS fp32 slots in slot order, accumulated in fp64 (round to nearest)
int launch_slot_sum_f32(const float* in, int64_t ldi, int64_t slot_stride, int NS, int64_t rows, int w, double* out,
                        int64_t ldo, cudaStream_t st);
int launch_view_tf32(const ViewArgs32& a, cudaStream_t st);
// X (fp64 col-major rows x w, ld) -> tf32-rounded hi / lo parts (fp32 col-major, ld32)
int launch_split_tf32(const double* X, int64_t ld, int64_t rows, int w, float* hi, float* lo, int64_t ld32,
                      cudaStream_t st);
// dtype conversions of column-major blocks (rows x cols)
int launch_f32_to_f64(const float* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int cols,
                      cudaStream_t st);
int launch_f64_to_f32(const double* src, int64_t lds, float* dst, int64_t ldd, int64_t rows, int cols,
                      cudaStream_t st);

void plan_view(int kind, int64_t rows, int64_t n, int w, int grid_cap, int* S, int* KTS);
int launch_view_ax(const ViewArgs& a, cudaStream_t st);
int launch_view_aty(const ViewArgs& a, cudaStream_t st);
int launch_view_fused(const FusedArgs& a, cudaStream_t st);
int fused_strips(int64_t n);  // number of 64-column strips of the fused kernel

// ---- small kernels (small_kernels.cu) --------------------------------------------------------
// device-side status words (one struct in device memory per ctx)
struct DevStatus {
  int deficient;        // columns zeroed by the guarded Cholesky
  int jacobi_sweeps;
  int jacobi_fail;
  int numeric_fail;     // e.g. singular R-hat
  int minvar_lc;        // l_c chosen by the minimum-variance post-processing (minvar.cu)
};

// out[c][r] = sum_{s<S} in[s][c][r] for c < w, r < rows   (column-major, slot stride)
int launch_slot_sum(const double* in, int64_t ldi, int64_t slot_stride, int S, int64_t rows, int w, double* out,
                    int64_t ldo, cudaStream_t st);
// G partial: G_b (a x b, col-major ld = a) = Xa[rows chunk]^T Xb[rows chunk]; returns #slots used
int gram_slots(int64_t rows);
int launch_cross_gram(const double* Xa, int64_t lda_, int a, const double* Xb, int64_t ldb, int b, int64_t rows,
                      double* slots, int nslots, cudaStream_t st);
// G = sum of nslots partials (a x b each, contiguous)
int launch_slots_reduce_small(const double* slots, int nslots, int64_t count, double* G, cudaStream_t st);
// Guarded Cholesky of the w x w Gram G (col-major): R upper (G = R^T R), Rinv = R^+ on the
// non-deficient columns, Racc <- R * Racc (if Racc != null, accumulate the product of passes).
int launch_chol(const double* G, int w, double* R, double* Rinv, double* Racc, DevStatus* status, cudaStream_t st);
// out (rows x c, col-major) = in (rows x w) * M (w x c, col-major ld = ldm);  mode 0: overwrite,
// mode 1: out -= in * M.  out must not alias in.
int launch_ts_gemm(const double* in, int64_t ldi, int64_t rows, int w, const double* M, int64_t ldm, int c,
                   double* out, int64_t ldo, int mode, cudaStream_t st);
// One-sided Jacobi SVD of M (r x c col-major, ldm), r >= c, c <= 256, r <= 256:
// M = Ul diag(S) Vr^T, S descending.  Ul (r x c, ld r), Vr (c x c, ld c).  Scratch >= 2*256*256.
int launch_jacobi(const double* M, int64_t ldm, int r, int c, double* Ul, double* S, double* Vr, double* scratch,
                  DevStatus* status, cudaStream_t st);
// general small GEMM / transposes on device (tiny sizes): C(mxn) = op(A) op(B), col-major
int launch_small_gemm(int ta, int tb, int m, int n, int k, const double* A, int64_t lda_, const double* B,
                      int64_t ldb, double* C, int64_t ldc, cudaStream_t st);
// strided 2-D copy of a column-major (rows x cols) block, with optional fill of padding rows
int launch_copy_cols(const double* src, int64_t lds, double* dst, int64_t ldd, int64_t rows, int cols,
                     cudaStream_t st);
int launch_fill(double* dst, int64_t count, double v, cudaStream_t st);
// out (rows x c) += T (rows x c), column-major
int launch_add_cols(const double* T, int64_t ldt, double* out, int64_t ldo, int64_t rows, int c, cudaStream_t st);
// out (rows x c) -= T (rows x c), column-major
// F (n x w, ld ldf, column-major) -> (to_chunks) / <- chunked layout: chunk q = rows [q cs, (q+1) cs)
// as a column-major cs x w block at buf + q cs w; rows >= n are zero in the chunks
int launch_rows_chunk(double* F, int64_t ldf, int64_t n, double* buf, int64_t cs, int nchunks, int w, int to_chunks,
                      cudaStream_t st);
int launch_sub_cols(const double* T, int64_t ldt, double* out, int64_t ldo, int64_t rows, int c, cudaStream_t st);
// triangular-system helpers for Alg. 7: out (c x c) = upper-triangular inverse of R (c x c)
int launch_tri_inv(const double* R, int c, double* Rinv, DevStatus* status, cudaStream_t st);
// Tp = V diag(s^+) U^T (w x w) from T = U diag(s) V^T, s_i <= rcut s_0 dropped; X(:, j) *= d[j]
int launch_pinv_svd(const double* U, const double* s, const double* V, int w, double rcut, double* Tp,
                    cudaStream_t st);
int launch_scale_cols(double* X, int64_t ld, int rows, int cols, const double* d, cudaStream_t st);
// zero the columns j of X (rows x w) with G_jj <= tol * ref_j (dependent after a block projection)
int launch_zero_dep_cols(double* X, int64_t ld, int64_t rows, int w, const double* G, const double* ref, double tol,
                         DevStatus* status, cudaStream_t st,
                         int64_t gstride = -1);   // G's diagonal stride (-1: a w x w Gram)
// d[j] = squared norm of column j of X (rows x w, ld)
int launch_colnorm2(const double* X, int64_t ld, int64_t rows, int w, double* d, cudaStream_t st);
// S[i] <- S[i]^2
int launch_square(double* S, int n, cudaStream_t st);
// Nystrom (Alg. 4) helpers: nu = 2.2e-16 ||Y_r||_2 from the Gram of Y_r (power iteration);
// Y += nu Q; S = (B + B^T)/2; lam2 = max(lam^2 - nu, 0)
int launch_nys_nu(const double* G, int w, double* out, cudaStream_t st);
int launch_axpy_dev(double* Y, int64_t ldy, const double* Q, int64_t ldq, int64_t rows, int w, const double* nu,
                    cudaStream_t st);
int launch_symmetrize(const double* B, int w, double* S, cudaStream_t st);
int launch_nys_eig(const double* lam, int k, const double* nu, double* lam2, cudaStream_t st);

// minimum-variance l_c (minvar.cu): trial spectra lam ((p+1) x k) from Z = R_y Qh
// (l2 x l, ld l2) and Rhi = Rh^-1 (l x l, ld l); the selection into *out; zero columns >= k + *lc.
int64_t minvar_scratch(int l2, int l, int p);
int launch_minvar_trials(const double* Z, int l2, int l, const double* Rhi, int k, int p, double* lam,
                         double* scratch, cudaStream_t st);
int launch_minvar_select(const double* lam, int k, int p, int* out, cudaStream_t st);
int launch_mask_cols(double* X, int64_t ld, int64_t rows, int w, int k, const int* lc, cudaStream_t st);

}  // namespace rsvd

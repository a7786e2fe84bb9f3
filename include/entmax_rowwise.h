/*
 * entmax_rowwise.h — C ABI of the standalone row-wise α-entmax solver.
 *
 * Method: arXiv 2502.12082, /root/reference/PAPER.md (cited P:L<n>).
 *   α-entmax of a row s (Eq. 2): p = [z − τ·1]_+^{1/(α−1)} with z = (α−1)·s
 *   (Alg. 1 line 3), τ the root of f(τ) = Σ_j [z_j − τ]_+^{1/(α−1)} − 1 (Eq. 3),
 *   found by the hybrid Halley-bisection of Alg. 1 (Halley step Eq. 5 P:L220-222 with
 *   f′, f″ of Eqs. 6-7, bisection fallback Eq. 4) — or, with halley = 0, by
 *   plain bisection (Eq. 4, the scheme the paper compares against).
 *   The paper benchmarks this solver on its own: n = 8192, Gaussian rows, T = 3.
 *   Backward: ds = u ⊙ dp − (⟨u, dp⟩ / ‖u‖₁)·u with u = p^{2−α}
 *   (0 off the support).
 *
 * Conventions
 *  - Matrices are row-major [rows, n] with leading dimension ld (elements, ld >= n); s, p, dp, ds
 *    share ld.  Element type `dtype` = ENTMAX_BF16 or ENTMAX_FP32 (entmax_attn.h); arithmetic is
 *    fp32.  Pointers are DEVICE pointers, 16-byte aligned, and ld·sizeof(dtype) must be a
 *    multiple of 16 bytes.  All n entries of a row are visible (n in τ_hi = m − n^{1−α}).
 *  - τ is returned in the pre-scaled convention of Alg. 1 (τ for z, not for s), fp32 [rows].
 *  - Ownership: the caller allocates every buffer; the library allocates nothing.  In-place
 *    (p == s, ds == dp) is allowed: every row is read completely before any of it is written.
 *  - Asynchrony: enqueued on `stream` (cudaStream_t as void*), no host synchronisation.
 *  - Errors: an entmax_status_t (entmax_attn.h) is returned, never thrown; argument errors are
 *    detected before any launch (entmax_attn_last_error() gives the detail).
 *    α < 1+1e-3 or n_iter < 1 or rows/n < 1 or a misaligned pointer/ld → ENTMAX_ERR_INVALID_ARG;
 *    α > 2 → ENTMAX_ERR_UNSUPPORTED; a launch failure → ENTMAX_ERR_CUDA.
 *  - Inputs must be finite; not checked on the device.
 */
#ifndef ENTMAX_ROWWISE_H_
#define ENTMAX_ROWWISE_H_

#include <stddef.h>
#include <stdint.h>

#include "entmax_attn.h"

#ifdef __cplusplus
extern "C" {
#endif

/*
 * Forward: p = α-entmax(s) row by row after T = n_iter iterations (reading c4: the τ after the
 * T-th update).
 *   s      in : [rows, n] dtype, raw scores (no (α−1) pre-scaling: the library applies it).
 *   halley in : 1 = Halley-bisection (Alg. 1), 0 = bisection only (Eq. 4: τ = midpoint after the
 *               T-th bracket update).
 *   p      out: [rows, n] dtype.  tau out: [rows] fp32, or NULL.
 */
int entmax_rowwise_fwd(const void* s, int64_t rows, int32_t n, int64_t ld, int dtype, float alpha, int n_iter,
                       int halley, void* p, float* tau, void* stream);

/*
 * Backward (vector-Jacobian product of Eq. 2 w.r.t. s).
 *   p  in : [rows, n] dtype, the forward's output.   dp in: [rows, n] dtype, upstream gradient.
 *   ds out: [rows, n] dtype.  A row with ‖u‖₁ = 0 cannot occur for a forward output (p sums to ~1).
 */
int entmax_rowwise_bwd(const void* p, const void* dp, int64_t rows, int32_t n, int64_t ld, int dtype, float alpha,
                       void* ds, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* ENTMAX_ROWWISE_H_ */

/*
 * entmax_attn.h — C ABI of the B200 (sm_100a) AdaSplash α-entmax attention hot path.
 *
 * Method: arXiv 2502.12082 ("AdaSplash"), /root/reference/PAPER.md, cited P:L<n>.
 *   forward  : τ by Halley-bisection over K blocks (Alg. 1, Alg. 3 P:L841-870,
 *              Eq. 8), then O_i = Σ_j [(α−1)S_ij − τ_i]_+^{1/(α−1)} V_j
 *              (Alg. 2, Eq. getting-oi) over the non-null blocks of the
 *              block mask M (Eq. 9) and O⁽²⁾ = Σ_j U_ij V_j / ‖U_i‖₁;
 *   backward : δ = rowsum(dO ⊙ O⁽²⁾), dK/dV over 𝒦_j (Alg. 4),
 *              dQ over 𝒬_i (Alg. 5), dS = U ⊙ (dP − δ).
 *   S = c·Q Kᵀ with c = 1/√d by default (Eq. 1); dQ and dK carry c.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Tensors Q, K, V, O, O2, dO, dQ, dK, dV are [B, H, N, d] with element strides
 *    (sb, sh, sn) given in entmax_shape_t and the last dimension contiguous; all of them use
 *    the SAME strides.  Element type = `dtype` (bf16 or fp32).  Pointers are DEVICE pointers,
 *    16-byte aligned; strides must be multiples of 8 elements (16 bytes).
 *  - τ is [B, H, N] fp32 contiguous, in the pre-scaled convention of Alg. 1 line 3
 *    (P:L195): p = [z − τ]_+^{1/(α−1)} with z = (α−1)·S.
 *  - Block mask granularity (B_r, B_c) is a library constant (entmax_attn_block_size);
 *    T_r = ⌈N/B_r⌉, T_c = ⌈N/B_c⌉.  mask is [B, H, T_r, T_c] uint8 contiguous with
 *    M_ij = 1 iff some (i′ ∈ block i, j′ ∈ block j, j′ visible to i′) has (α−1)S_{i′j′} − τ_{i′} > 0
 *    (Eq. 9 with readings c1/c2 of DESIGN.md).  row_cnt [B, H, T_r] int32 and row_idx
 *    [B, H, T_r, T_c] int32 are the lookup table 𝒬_i = {j | M_ij = 1} in
 *    increasing j, padded (ELL).  Causal: key j′ is visible to query i′ iff j′ <= i′.
 *  - Ownership: the caller allocates every buffer (including the workspace, sized by the
 *    *_workspace_bytes queries) and keeps it alive until the stream work completes.  The
 *    library allocates no device memory and keeps no per-call state, so one workspace can be
 *    shared by every layer / call on a stream.
 *  - Asynchrony: all work is enqueued on `stream` (a cudaStream_t passed as void*; NULL =
 *    legacy default stream).  No host synchronisation happens inside the calls.
 *  - Errors: every function returns an entmax_status_t; nothing is thrown across the ABI.
 *    Argument errors are detected synchronously before any launch; ENTMAX_ERR_CUDA reports
 *    a launch failure (cudaGetLastError).  entmax_attn_last_error() gives a human-readable
 *    detail string for the calling thread's most recent failure.
 *  - Inputs must be finite; this is not checked on the device.
 */
#ifndef ENTMAX_ATTN_H_
#define ENTMAX_ATTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ENTMAX_OK = 0,
  ENTMAX_ERR_INVALID_ARG = 1,  /* bad shape, α < 1+1e-3, n_iter < 1, null/misaligned pointer */
  ENTMAX_ERR_UNSUPPORTED = 2,  /* α > 2, head dim not supported, B·H > 65535, N > 2^24       */
  ENTMAX_ERR_WORKSPACE = 3,    /* workspace smaller than the *_workspace_bytes query      */
  ENTMAX_ERR_CUDA = 4          /* a CUDA launch failed                                    */
} entmax_status_t;

typedef enum { ENTMAX_BF16 = 0, ENTMAX_FP32 = 1 } entmax_dtype_t;

/* Shape + element strides of every [B, H, N, d] tensor of a call. */
typedef struct {
  int32_t B, H, N, d;
  int64_t sb, sh, sn;
} entmax_shape_t;

/* Static string for a status code (never NULL). */
const char* entmax_attn_status_string(int status);

/* Detail message of the calling thread's last failing call ("" if none). */
const char* entmax_attn_last_error(void);

/*
 * Mask / table granularity (B_r, B_c) for head dim d and element type dtype (the block
 * size the paper leaves open, P:L340-341 / reading c15).  Every supported (d, dtype) uses
 * B_r = B_c = 128 in this build.  Br, Bc out (either may be NULL).  Returns ENTMAX_OK, or
 * ENTMAX_ERR_INVALID_ARG for an unknown dtype, ENTMAX_ERR_UNSUPPORTED for a head dim no kernel
 * handles (d not in {16, 32, 64, 128}); the outputs are then left untouched.
 */
int entmax_attn_block_size(int32_t d, int dtype, int32_t* Br, int32_t* Bc);

/* Device workspace (bytes) needed by entmax_attn_fwd / entmax_attn_bwd for this shape. */
size_t entmax_attn_fwd_workspace_bytes(const entmax_shape_t* shp, int dtype, int causal);
size_t entmax_attn_bwd_workspace_bytes(const entmax_shape_t* shp, int dtype, int causal);

/*
 * Forward pass (Alg. 3 then Alg. 2 with block masking).
 *   q, k, v       in : [B,H,N,d] dtype.
 *   alpha         in : α ∈ [1+1e-3, 2] (α > 2 → UNSUPPORTED; α→1 would need softmax).
 *   causal        in : 0/1.
 *   n_iter        in : T >= 1 Halley-bisection iterations (Alg. 1; paper default 3).
 *   scale         in : c in S = c·QKᵀ; <= 0 selects 1/√d (Eq. 1).
 *   o             out: [B,H,N,d] dtype, O = P V (P not renormalised, Alg. 2 line 13).
 *   o2            out: [B,H,N,d] fp32, CONTIGUOUS, O⁽²⁾ (needed by the backward); may be NULL
 *                      for inference (the U·V product is then skipped).  Kept in fp32 whatever
 *                      the input dtype: δ = dO·O⁽²⁾ feeds dS = U ⊙ (dP − δ) whose row sums must
 *                      cancel, and a bf16 O⁽²⁾ leaks ~2⁻⁹·|K| into dQ (reading r3).
 *   tau           out: [B,H,N] fp32 (after the T-th update, reading c4).
 *   mask          out: [B,H,T_r,T_c] uint8 (see conventions).
 *   row_cnt/row_idx out: 𝒬 tables (see conventions).
 *                 mask, row_cnt and row_idx may ALL be NULL: the unmasked mode (the paper's variant
 *                 without block masking) visits every
 *                 visible K/V block and writes neither M nor the tables (O(N) extra memory); the
 *                 backward must then be called with NULL tables too.  Some but not all NULL →
 *                 ENTMAX_ERR_INVALID_ARG.
 *   workspace     in : device scratch of >= entmax_attn_fwd_workspace_bytes bytes.
 *   stream        in : cudaStream_t.
 */
int entmax_attn_fwd(const void* q, const void* k, const void* v, const entmax_shape_t* shp, int dtype,
                    float alpha, int causal, int n_iter, float scale,
                    void* o, void* o2, float* tau, uint8_t* mask, int32_t* row_cnt, int32_t* row_idx,
                    void* workspace, size_t ws_bytes, void* stream);

/*
 * Backward pass (App. A.2, Algs. 4-5 with the lookup tables).
 *   q, k, v, d_o  in : [B,H,N,d] dtype.  o2 in: [B,H,N,d] fp32 contiguous from the forward
 *                      (O itself is not needed).
 *   tau, mask, row_cnt, row_idx in : exactly as written by entmax_attn_fwd for these inputs
 *                      (mask, row_cnt, row_idx all NULL: unmasked mode, every visible block).
 *   alpha, causal, scale      in : the forward's values.
 *   dq, dk, dv    out: [B,H,N,d] dtype.  dQ = c·dS K, dK = c·dSᵀ Q, dV = Pᵀ dO.
 *   workspace     in : >= entmax_attn_bwd_workspace_bytes bytes (holds δ and the 𝒦 tables).
 */
int entmax_attn_bwd(const void* q, const void* k, const void* v, const void* o2, const void* d_o,
                    const float* tau, const uint8_t* mask, const int32_t* row_cnt, const int32_t* row_idx,
                    const entmax_shape_t* shp, int dtype, float alpha, int causal, float scale,
                    void* dq, void* dk, void* dv, void* workspace, size_t ws_bytes, void* stream);

/*
 * Bit-packed block mask: out[r, w] bit b = mask[r, 32·w + b] != 0 for the rows
 * r < rows (= B·H·T_r) of a [rows, T_c] uint8 mask; out is [rows, ⌈T_c/32⌉] uint32, bits past T_c
 * zero.  8× smaller than the byte mask for callers that keep masks across layers or steps.
 * Device pointers; asynchronous on `stream`; INVALID_ARG for NULL pointers or rows/Tc < 1.
 */
int entmax_attn_pack_mask(const uint8_t* mask, int64_t rows, int32_t Tc, uint32_t* out, void* stream);

/*
 * Kernel timing (instrumentation for bench.py's roofline numbers; off by default).
 * When enabled, every kernel launched by entmax_attn_fwd/bwd is bracketed by CUDA events
 * recorded on the launching stream.  entmax_attn_profile_collect() synchronises those events
 * and returns, per kernel name, the number of launches and the summed duration in ms since
 * the last reset.  Names are static strings.  Returns the number of entries written.
 */
void entmax_attn_profile_enable(int on);
void entmax_attn_profile_reset(void);
int entmax_attn_profile_collect(const char** names, int32_t* launches, double* total_ms, int cap);

/* Which implementation a (shape, dtype) runs on: 1 = tcgen05/TMEM/TMA (sm_100a),
 * 0 = SIMT fp32 kernels (fp32 inputs, small head dims), -1 = unsupported. */
int entmax_attn_impl_for(const entmax_shape_t* shp, int dtype);

#ifdef __cplusplus
}
#endif

#endif /* ENTMAX_ATTN_H_ */

/* gsg.h -- C ABI of libgsg.so: the B200 (sm_100a) hot path of graph-sampling GCN training.
 *
 * The operation (arXiv 2010.03166, "Accurate, Efficient and Scalable Training of Graph
 * Neural Networks"; PAPER.md line numbers as P:n):
 *   per sampled subgraph G_s (Alg. 1 lines 3-6) build the normalized adjacency
 *   Â_s (Eq. 5) and its transpose (Alg. 4); then per GCN layer l
 *     forward  (Eq. 5):           P = Â X ;  H = ReLU(P W)
 *     backward (Eq. 13 at P:704):  dZ = dH ⊙ 1[H > 0] ;  dW = Pᵀ dZ ;
 *                                         dX = Âᵀ (dZ Wᵀ)
 *   plus the classifier head (Eqs. 2-4; backward Eqs. 9-11) and the
 *   data-parallel mean of dW over independent subgraphs.
 *
 * Conventions (all entry points):
 *   - Return value: GSG_OK (0) or a negative GSG_E* code; a human-readable message for the
 *     calling thread is available from gsg_last_error() until its next failing call.
 *   - Argument errors (shapes, strides, alignment, NULL pointers) are reported
 *     synchronously and nothing is launched. Kernels are stream-ordered on the context's
 *     stream; asynchronous CUDA faults surface from the next call or from gsg_ctx_sync().
 *   - Dense matrices are row-major. `ld*` is the row stride in ELEMENTS, ld >= columns, and
 *     ld * sizeof(elem) must be a multiple of 16 bytes (TMA); base pointers 16-byte aligned.
 *     Columns [f, round_up(f, 4)) of an fp32 output row may be overwritten (float4 stores);
 *     columns beyond that are never touched.
 *   - Pointers named d_* / matrices passed to layer calls are DEVICE pointers owned by the
 *     caller. Pointers named h_* are host pointers (pinned memory enables async copies).
 *   - The library owns every subgraph array and the per-context workspace (split-K partials,
 *     T = dZ Wᵀ scratch, bf16 weight copies). Host inputs are copied, never retained.
 *   - Threading: one context per host thread/stream. Distinct subgraphs may be used
 *     concurrently from distinct contexts on the same device.
 *   - No CPU fallback exists: every compute step runs in this library's sm_100a kernels.
 */
#ifndef GSG_H_
#define GSG_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GSG_API __attribute__((visibility("default")))
#else
#define GSG_API
#endif

/* ---- status codes -------------------------------------------------------------------- */
enum {
  GSG_OK = 0,
  GSG_EINVAL = -1,         /* bad shape / stride / alignment / pointer / enum value        */
  GSG_EGRAPH = -2,         /* CSR invariant violated (see gsg_subgraph_upload)             */
  GSG_ENOMEM = -3,         /* device allocation failed                                     */
  GSG_ECUDA = -4,          /* CUDA runtime/driver error (message has the CUDA string)      */
  GSG_ENCCL = -5,          /* NCCL error or NCCL library not loadable                      */
  GSG_EUNSUPPORTED = -6    /* device is not sm_100, or a size exceeds a 32-bit index       */
};

/* ---- normalization modes (gsg_subgraph_normalize) ------------------------------------ */
enum {
  GSG_NORM_ROW_SELF = 0,   /* Â = D~^-1 (A + I), D~ = D + I, subgraph-local degrees: the
                              BASELINE configs (SURVEY reading R1/R2); rows sum to 1       */
  GSG_NORM_SYM_SELF = 1,   /* Â = (I+D)^-1/2 (I+A) (I+D)^-1/2, Eq. 5               */
  GSG_NORM_ROW = 2,        /* Ã = D^-1 A, GraphSAGE Eq. 1; isolated rows are zero  */
  GSG_NORM_VALUES = 3      /* Â_ij = the uploaded edge values, no self loop (weighted /
                              GraphSAINT-normalized adjacency)                  */
};

/* ---- GEMM precision ------------------------------------------------------------------ */
enum {
  GSG_PREC_TF32 = 0,       /* fp32 operands read as TF32 by tcgen05 (kind::tf32), fp32 acc */
  GSG_PREC_BF16 = 1,       /* bf16 operand copies (kind::f16), fp32 accumulate             */
  GSG_PREC_FP32X3 = 2      /* fp32-accurate GEMM on TF32 tensor cores (3xTF32): each fp32
                              operand x = hi + lo with hi = tf32_trunc(x) (kind::tf32 reads an
                              fp32 operand truncated: the operand itself is hi), lo = x - hi,
                              and op(A) op(B) = Ahi Bhi + Ahi Blo + Alo Bhi (the lo x lo term,
                              ~2^-20 relative, is dropped), evaluated as ONE TF32 GEMM over
                              K' = 3K whose k-block segments read [A | A | Alo] x [B ; Blo ; B];
                              only Alo, Blo (and copies of operands TMA cannot read in place)
                              are written, in the context workspace. ~1e-6 relative per
                              product; 3x the tensor work of TF32. fp32 operands like
                              GSG_PREC_TF32. (GSG_X3_IMPLICIT=0: the round-to-nearest split
                              with three stacked copies, for comparison.) */
};

/* ---- flags --------------------------------------------------------------------------- */
enum {
  GSG_NO_RELU = 1,         /* forward: H = P W (no ReLU)                                   */
  GSG_DH_PREMASKED = 2,    /* backward: dH already equals dZ = dH ⊙ 1[H>0] (fused upstream) */
  GSG_ACCUM_DW = 4,        /* backward: dW += Pᵀ dZ instead of dW = Pᵀ dZ                  */
  GSG_ORDER_A_XW = 8,      /* chain order 2 of §7.1: forward Y = X W then
                              H = ReLU(Â Y) (the SpMM runs at width f_out); backward
                              G = Âᵀ dZ, dW = Xᵀ G, dX = (G Wᵀ) ⊙ 1[H_below > 0]. With this
                              flag the P arguments of both calls carry X's role: forward
                              writes Y (n x f_out) into P; backward reads X (n x f_in) from P. */
  GSG_W_BF16 = 16,         /* GSG_PREC_BF16 only: d_W already points to a bf16 copy of W
                              (row-major f_in x f_out, ldw in bf16 elements, ldw % 8 == 0),
                              e.g. made once per step with gsg_to_bf16 and shared by the
                              layer's forward and backward; no per-call conversion. */
  GSG_H_BITS = 32          /* backward: d_H points to the layer's own ReLU bitmask (the
                              forward's d_Hbits, "ReLU bitmask" layout, ldh in 32-bit words,
                              ldh >= ceil(f_out / 32)) instead of fp32 H; the dZ = dH ⊙ 1[H > 0]
                              gate then reads 1/32 of the bytes (same result bit for bit). */
};

/* ---- GEMM epilogues (gsg_gemm) ------------------------------------------------------- */
enum {
  GSG_EPI_NONE = 0,        /* C = op(A) op(B)                                              */
  GSG_EPI_RELU = 1,        /* C = max(op(A) op(B), 0)               (forward a3)           */
  GSG_EPI_MASK = 2         /* C = (op(A) op(B)) ⊙ 1[aux > 0]         (ReLU' gate, a4)       */
};

/* ---- ReLU bitmasks -------------------------------------------------------------------- *
 * The ReLU' gate 1[H > 0] of the backward (dZ = dH ⊙ σ'(Z), σ = ReLU) needs one bit per
 * element of H, not H itself. A "ReLU bitmask" of an n x f matrix H is an n x ldb array of
 * uint32 words (row-major, ldb >= ceil(f / 32)): bit i of word w of row r is 1[H[r, 32 w + i] > 0];
 * bits of columns >= f are 0; words ldb > ceil(f/32) are never touched. Writers (the forward's
 * ReLU epilogue, GEMM or SpMM) write every word of columns < f; readers (the backward's gates)
 * read it in place of the fp32 matrix -- 1/32 of the bytes (config 5: 2.6 MB instead of 82 MB
 * per gated layer). Wherever a call takes both a gate matrix and a gate bitmask, the bitmask
 * wins and the matrix may be NULL. Results are identical bit for bit either way. */

/* ---- head kinds ---------------------------------------------------------------------- */
enum { GSG_HEAD_SOFTMAX = 0, GSG_HEAD_SIGMOID = 1 };

typedef struct gsg_ctx* gsg_ctx_t;
typedef struct gsg_subgraph* gsg_subgraph_t;

/* ==== context ========================================================================== */
/* Create a context on CUDA device `device`, issuing work on `cuda_stream` (a cudaStream_t,
 * not owned; NULL = the legacy default stream, which also orders against torch's default
 * stream). Fails with
 * GSG_EUNSUPPORTED if the device is not compute capability 10.0 (sm_100a kernels only). */
GSG_API int gsg_ctx_create(int device, void* cuda_stream, gsg_ctx_t* out);
GSG_API int gsg_ctx_destroy(gsg_ctx_t ctx);
/* Re-target subsequent launches to another stream (e.g. torch's current stream). */
GSG_API int gsg_ctx_set_stream(gsg_ctx_t ctx, void* cuda_stream);
GSG_API void* gsg_ctx_stream(gsg_ctx_t ctx);
/* Block until the context's stream drains; returns GSG_ECUDA for any pending fault. */
GSG_API int gsg_ctx_sync(gsg_ctx_t ctx);
/* Make the context stream wait for a CUDA event (cudaEvent_t) recorded on another stream. Inside
 * a stream capture the wait becomes an external-event node of the graph (cudaEventWaitExternal),
 * so a replayed step can wait for work issued outside the graph, e.g. the previous step's
 * gradient all-reduce on a communication stream before the step overwrites the gradients. */
GSG_API int gsg_ctx_wait_event(gsg_ctx_t ctx, void* cuda_event);
/* Number of kernels this context has launched so far (evidence counter for benches). */
GSG_API int64_t gsg_ctx_launch_count(gsg_ctx_t ctx);
/* Kernel-class profiling (bench evidence): while enabled, every launch of the class is
 * bracketed by CUDA events on the context stream, and the library accumulates the class's
 * ALGORITHMIC work: SpMM effective bytes 4*nnz_hat*f + 8*nnz_hat + 4*(n+1)
 * + 4*n*f per launch; GEMM flops 2*M*N*K. Classes: GSG_K_SPMM, GSG_K_GEMM, GSG_K_NORM,
 * GSG_K_OTHER. gsg_ctx_profile_read synchronizes the stream, returns the totals since the
 * last read and resets them. Enabling allocates events lazily (do it outside graph capture). */
enum { GSG_K_SPMM = 0, GSG_K_GEMM = 1, GSG_K_NORM = 2, GSG_K_OTHER = 3,
       /* the same launches again, by SURVEY §8(a) row (set by the layer / head entry points;
        * direct gsg_spmm / gsg_gemm calls carry no row): a1 normalize, a2 forward aggregation,
        * a3 forward transform, a4 standalone ReLU' gate, a5 dW, a6 T = dZ Wᵀ, a7 transposed
        * aggregation, a8 head (GEMMs + loss) */
       GSG_K_A1 = 4, GSG_K_A2 = 5, GSG_K_A3 = 6, GSG_K_A4 = 7, GSG_K_A5 = 8, GSG_K_A6 = 9,
       GSG_K_A7 = 10, GSG_K_A8 = 11, GSG_K_CLASSES = 12 };
GSG_API int gsg_ctx_profile(gsg_ctx_t ctx, int enable);
GSG_API int gsg_ctx_profile_read(gsg_ctx_t ctx, int kclass, double* total_ms, int64_t* launches,
                                 double* alg_bytes, double* alg_flops);
/* Thread-local message of the last failing call on this thread ("" if none). */
GSG_API const char* gsg_last_error(void);

/* ==== subgraph =================================================== */
/* Copy an induced subgraph G_s (Alg. 2 line 9) to the device.
 *   n            number of subgraph nodes |V_s| (0 <= n < 2^31)
 *   nnz          number of stored directed entries of A_s (no self loops)
 *   h_indptr     host int64[n+1], h_indptr[0] = 0, non-decreasing, h_indptr[n] = nnz
 *   h_indices    host int32[nnz]; row i = h_indices[h_indptr[i] .. h_indptr[i+1])
 *   h_values     host float[nnz] edge weights, or NULL for a binary adjacency (required by
 *                GSG_NORM_VALUES, ignored by the degree-based modes)
 *   validate     1 = check on the host before copying, rejecting with GSG_EGRAPH (first
 *                offending entry in the message): an index out of [0, n); a row that is not
 *                strictly ascending (Alg. 4's precondition; this also rejects
 *                duplicates); a self loop (normalization adds it); an asymmetric
 *                structure (the undirected assumption of P:737-743).
 * The structure must satisfy those invariants even when validate = 0 (undefined results
 * otherwise). nnz + n must be < 2^31. On success *out owns device copies. */
GSG_API int gsg_subgraph_upload(gsg_ctx_t ctx, int32_t n, int64_t nnz, const int64_t* h_indptr,
                                const int32_t* h_indices, const float* h_values, int validate,
                                gsg_subgraph_t* out);
/* Refill an existing subgraph with a new CSR (same contract as gsg_subgraph_upload),
 * reusing its device arrays when they are large enough (no allocation in the steady state;
 * copies are asynchronous from pinned host memory). The arrays may also be DEVICE-resident,
 * e.g. a GPU-sampled subgraph from gsg_sample_get (device-to-device copy; validate must be 0
 * and nnz must match indptr[n], which the library cannot check without a synchronization).
 * The subgraph must be normalized again. */
GSG_API int gsg_subgraph_assign(gsg_ctx_t ctx, gsg_subgraph_t sg, int32_t n, int64_t nnz,
                                const int64_t* h_indptr, const int32_t* h_indices,
                                const float* h_values, int validate);
/* Same, from DEVICE arrays already resident in HBM (stream-ordered device-to-device copy;
 * no validation). Used when a pool of subgraphs lives on the GPU (Alg. 7 pool). */
GSG_API int gsg_subgraph_upload_device(gsg_ctx_t ctx, int32_t n, int64_t nnz,
                                       const int64_t* d_indptr, const int32_t* d_indices,
                                       const float* d_values, gsg_subgraph_t* out);
/* Build Â on the device (stream-ordered, no host synchronization):
 *   - insert the self loop of each row at its sorted position (*_SELF modes),
 *   - values per `norm_mode` (GSG_NORM_*), computed in fp64 and rounded to fp32,
 *   - the transposed values valT on the same (symmetric) structure: valT at slot (u, v)
 *     equals val at slot (v, u) -- a device gather form of Alg. 4 that yields
 *     exactly Alg. 4's DataTrans (a permutation of val),
 *   - degree bins (rows ordered by degree, heavy rows split across warps in the SpMMs).
 * May be called again with another mode. */
GSG_API int gsg_subgraph_normalize(gsg_ctx_t ctx, gsg_subgraph_t sg, int norm_mode);
/* Sizes of the normalized subgraph. Synchronizes the stream (reads device counters). */
GSG_API int gsg_subgraph_info(gsg_ctx_t ctx, gsg_subgraph_t sg, int32_t* n, int64_t* nnz_hat,
                              int32_t* max_deg_hat, int32_t* n_heavy);
/* Copy Â back to the host (tests): h_indptr int64[n+1], h_idx int32[nnz_hat],
 * h_val / h_valT float[nnz_hat]; any pointer may be NULL. Synchronizes. */
GSG_API int gsg_subgraph_download(gsg_ctx_t ctx, gsg_subgraph_t sg, int64_t* h_indptr,
                                  int32_t* h_idx, float* h_val, float* h_valT);
GSG_API int gsg_subgraph_free(gsg_subgraph_t sg);

/* ==== sparse aggregation (rows a2 / a7) ================================================ */
/* Y = Â X (transpose = 0, P = Â X of Eq. 5 / Alg. 6) or Y = Âᵀ X (transpose = 1,
 * the backward dX = Âᵀ T of P:719, read from valT). fp32 in, fp32 accumulate, fp32 out.
 *   f            feature width (columns) of X and Y, 1 <= f
 *   d_X, ldx     n x f input (ldx % 4 == 0)
 *   d_Y, ldy     n x f output (ldy % 4 == 0), must not alias d_X
 *   d_Ylp, ldylp optional bf16 copy of Y (NULL = none; ldylp % 8 == 0)
 *   d_mask, ldm  optional ReLU' gate: Y ⊙ 1[mask > 0] (NULL = none) -- used to emit the
 *                next layer's dZ directly from the transposed aggregation
 *   d_mask_bits, ldmb  optional gate as a ReLU bitmask (ldmb words per row); overrides d_mask
 * Each output row is summed in a fixed order (bitwise reproducible run to run).
 * A subgraph with n = 0 returns GSG_OK without reading any pointer. Errors: GSG_EINVAL (not
 * normalized, f < 1, NULL / misaligned (16 B) pointers, ld < f or ld % 4 != 0, Y aliasing X,
 * ldmb < ceil(f/32) or a bitmask not 4-byte aligned), GSG_EUNSUPPORTED (n * ldx * 4 >= 4 GiB:
 * the kernel's 32-bit row byte offsets). */
GSG_API int gsg_spmm(gsg_ctx_t ctx, gsg_subgraph_t sg, int transpose, int32_t f,
                     const float* d_X, int64_t ldx, float* d_Y, int64_t ldy,
                     void* d_Ylp, int64_t ldylp, const float* d_mask, int64_t ldm,
                     const uint32_t* d_mask_bits, int64_t ldmb);

/* ==== dense contraction on tcgen05 tensor cores (rows a3 / a5 / a6) ==================== */
/* C[M x N] = epi( op(A) op(B) ), fp32 accumulate in TMEM.
 *   op(A): transA = 0 -> A stored M x K row-major (lda >= K); transA = 1 -> A stored K x M
 *          (lda >= M), i.e. op(A) = Aᵀ. Same for B: transB = 0 -> K x N (ldb >= N);
 *          transB = 1 -> stored N x K (ldb >= K).
 *   precision    GSG_PREC_TF32 / GSG_PREC_FP32X3: A, B are float*; GSG_PREC_BF16: A, B are
 *                bf16 (uint16). FP32X3 needs workspace for the lo copies (and 3K < 2^31).
 *   d_C, ldc     fp32 output; d_Clp, ldclp optional bf16 copy (NULL = none)
 *   epilogue     GSG_EPI_*; d_aux/ldaux is the M x N gate for GSG_EPI_MASK
 *   d_auxbits, ldauxb  GSG_EPI_MASK only: the gate as a ReLU bitmask (overrides d_aux)
 *   d_Cbits, ldcb      GSG_EPI_RELU only: also write the ReLU bitmask of C (forces split_k = 1)
 *   split_k      0 = automatic; >= 1 forces the number of K splits (deterministic fixed-order
 *                reduction through the context workspace)
 *   accumulate   1 = C += result (before the epilogue is NOT supported with RELU/MASK)
 * K = 0 writes epi(0); M = 0 or N = 0 returns GSG_OK without reading any pointer. Errors:
 * GSG_EINVAL (bad precision / epilogue, negative dims, ld or 16-byte alignment violations,
 * accumulate with an epilogue, d_auxbits without GSG_EPI_MASK or d_Cbits without GSG_EPI_RELU,
 * bitmask strides below ceil(N/32) words), GSG_ECUDA (launch failure). */
GSG_API int gsg_gemm(gsg_ctx_t ctx, int32_t M, int32_t N, int32_t K,
                     const void* d_A, int64_t lda, int transA,
                     const void* d_B, int64_t ldb, int transB,
                     float* d_C, int64_t ldc, void* d_Clp, int64_t ldclp,
                     int precision, int epilogue, const float* d_aux, int64_t ldaux,
                     const uint32_t* d_auxbits, int64_t ldauxb, uint32_t* d_Cbits, int64_t ldcb,
                     int split_k, int accumulate);

/* fp32 -> bf16 copy of a rows x cols matrix (round-to-nearest-even). */
GSG_API int gsg_to_bf16(gsg_ctx_t ctx, int32_t rows, int32_t cols, const float* d_src,
                        int64_t lds, void* d_dst, int64_t ldd);

/* ==== GCN layer (Eq. 5 forward, P:719 backward) ======================================== */
/* Forward: P = Â X (kept for backward), H = ReLU(P W) (GSG_NO_RELU: H = P W).
 *   X (n x f_in, ldx), W (f_in x f_out row-major, ldw), P (n x f_in, ldp), H (n x f_out, ldh)
 *   precision = GSG_PREC_BF16 additionally needs P_lp (bf16 n x f_in, ldplp) which the
 *   aggregation writes for the GEMM; H_lp (bf16 n x f_out) is optional.
 * Chain order: (ÂX)W by default; GSG_ORDER_A_XW selects Â(XW) (§7.1).
 * BF16: W is converted to bf16 per call unless GSG_W_BF16 says d_W already is bf16.
 * d_Hbits, ldhbits: optional ReLU bitmask of H written by the same epilogue (NULL = none; not
 * with GSG_NO_RELU) -- the gate the layer above's backward reads instead of H. */
GSG_API int gsg_layer_forward(gsg_ctx_t ctx, gsg_subgraph_t sg, int32_t f_in, int32_t f_out,
                              const float* d_X, int64_t ldx, const float* d_W, int64_t ldw,
                              float* d_P, int64_t ldp, void* d_Plp, int64_t ldplp,
                              float* d_H, int64_t ldh, void* d_Hlp, int64_t ldhlp,
                              uint32_t* d_Hbits, int64_t ldhbits, int precision, int flags);
/* Backward of one layer given the forward's P and H:
 *   dZ = dH ⊙ 1[H > 0] (skipped with GSG_DH_PREMASKED: dH is dZ; GSG_H_BITS: d_H is H's
 *        ReLU bitmask),
 *   dW = Pᵀ dZ          (f_in x f_out; GSG_ACCUM_DW adds into dW),
 *   dX = Âᵀ (dZ Wᵀ)     (n x f_in; d_dX = NULL skips it, e.g. for layer 1),
 *        ⊙ 1[H_below > 0] when d_Hbelow != NULL, i.e. dX is then the layer below's dZ;
 *        d_Hbelow_bits (ReLU bitmask of H_below, ldhbb words per row) gives the same gate from
 *        1/32 of the bytes and overrides d_Hbelow.
 * BF16: d_Plp (bf16 P) is required; d_dHlp (bf16 copy of the premasked dH) is optional;
 * d_dXlp (bf16 copy of dX) is optional. T = dZ Wᵀ and masked-dZ live in the workspace. */
GSG_API int gsg_layer_backward(gsg_ctx_t ctx, gsg_subgraph_t sg, int32_t f_in, int32_t f_out,
                               const float* d_P, int64_t ldp, const void* d_Plp, int64_t ldplp,
                               const float* d_H, int64_t ldh,
                               const float* d_dH, int64_t lddh, const void* d_dHlp, int64_t lddhlp,
                               const float* d_W, int64_t ldw,
                               float* d_dW, int64_t lddw,
                               float* d_dX, int64_t lddx, void* d_dXlp, int64_t lddxlp,
                               const float* d_Hbelow, int64_t ldhb,
                               const uint32_t* d_Hbelow_bits, int64_t ldhbb,
                               int precision, int flags);

/* ==== GraphSAGE layer (Eq. 1; backward Eqs. 12-15) ====
 * The subgraph must be normalized with GSG_NORM_ROW (Ã = D⁻¹ A, no self loop; isolated rows are
 * zero). Output layout (reading R21, the column slices of Eqs. 12-15 / SPEC S:436): self path in
 * columns [0, f_half), neighbor path in [f_half, 2 f_half):
 *   forward:  P = Ã X ;  H = ReLU([X W_s , P W_n])                  (H: n x 2 f_half, ldh)
 *   backward: dZ = dH ⊙ 1[H > 0] (skipped with GSG_DH_PREMASKED) ;
 *             dW_s = Xᵀ dZ[:, :f_half] ;  dW_n = Pᵀ dZ[:, f_half:] ;
 *             dX = (dZ[:, :f_half] W_sᵀ + Ãᵀ (dZ[:, f_half:] W_nᵀ)) ⊙ 1[H_below > 0]
 * W_s, W_n: f_in x f_half row-major. f_half % 4 == 0 (16-byte column offset of the neighbor
 * half). TF32 only (GSG_EUNSUPPORTED otherwise). d_dX = NULL skips the input gradient. */
GSG_API int gsg_sage_forward(gsg_ctx_t ctx, gsg_subgraph_t sg, int32_t f_in, int32_t f_half,
                             const float* d_X, int64_t ldx, const float* d_Ws, int64_t ldws,
                             const float* d_Wn, int64_t ldwn, float* d_P, int64_t ldp,
                             float* d_H, int64_t ldh, int precision, int flags);
GSG_API int gsg_sage_backward(gsg_ctx_t ctx, gsg_subgraph_t sg, int32_t f_in, int32_t f_half,
                              const float* d_X, int64_t ldx, const float* d_P, int64_t ldp,
                              const float* d_H, int64_t ldh, const float* d_dH, int64_t lddh,
                              const float* d_Ws, int64_t ldws, const float* d_Wn, int64_t ldwn,
                              float* d_dWs, int64_t lddws, float* d_dWn, int64_t lddwn,
                              float* d_dX, int64_t lddx, const float* d_Hbelow, int64_t ldhb,
                              int precision, int flags);

/* ==== classifier head + CE loss (SUPPORT row a8) ======================================= */
/* S = H_L W_mlp ; S+ = ReLU(S) ; Y = softmax_rows(S+) (GSG_HEAD_SOFTMAX, labels int32[n]
 * class ids) or sigmoid(S+) (GSG_HEAD_SIGMOID, labels uint8[n x C] indicators, ld C);
 * loss = mean CE over the n rows (readings R7/R8);
 * dS = (Y - Ybar)/n ⊙ 1[S > 0] ; dW_mlp = H_Lᵀ dS ; dH_L = (dS W_mlpᵀ) ⊙ 1[H_L > 0]
 * (the returned dH_L is the top GCN layer's dZ, i.e. already premasked).
 *   d_S, d_dS    n x C fp32 scratch/outputs (ld lds); d_loss: one device float.
 *   d_dHlp       optional bf16 copy of dH_L (for BF16 layer backward).
 *   d_node_w     optional per-node loss weights λ_i (device float[n]; GraphSAINT loss
 *                normalization): loss = Σ_i λ_i CE_i and dS_i = λ_i (Y_i - Ybar_i) ⊙
 *                1[S_i > 0]. NULL = λ_i = 1/n (the mean above).
 *   d_HLbits     optional ReLU bitmask of H_L (ldhlb words per row): the dH_L gate is read from
 *                it instead of H_L (identical result). */
GSG_API int gsg_head(gsg_ctx_t ctx, int32_t n, int32_t f, int32_t C, int kind,
                     const float* d_HL, int64_t ldh, const float* d_Wmlp, int64_t ldw,
                     const void* d_labels, float* d_S, float* d_dS, int64_t lds,
                     float* d_dWmlp, int64_t lddw, float* d_dHL, int64_t lddh,
                     void* d_dHlp, int64_t lddhlp, float* d_loss, int precision,
                     const float* d_node_w, const uint32_t* d_HLbits, int64_t ldhlb);

/* ==== GPU-side frontier sampling + induction ======================= *
 * Alg. 2 under reading R9, on the device, `count` independent samplers at once
 * (the paper's inter-sampler parallelism):
 *   FS_0: m distinct nodes drawn uniformly from the parent's non-isolated nodes (rejection of
 *         repeats); V_s <- FS_0;
 *   repeat until |V_s| = n (or 1000 n + 10^6 iterations): pick a frontier slot with
 *         probability deg(u) / sum_FS deg (Alg. 2 line 4; Fenwick tree in shared memory), pick a
 *         uniform neighbor u' of u (line 5), replace u by u' in FS (line 6), add u' to V_s if new;
 *   clip |V_s| to a multiple of `clip` by uniformly random removals (§7.2);
 *   induce G_s on V_s with ascending local ids (Alg. 2 line 9).
 * Random draws come from a counter-based generator: draw j of iteration i of sampler k is
 *   r = mix64(seed_k XOR mix64(4 i + j)),  seed_k = mix64(mix64(seed) + k)
 *   (so calls with nearby seeds draw unrelated subgraphs),
 *   mix64 = splitmix64 finalizer (z += 0x9E3779B97F4A7C15; z ^= z>>30; z *= 0xBF58476D1CE4E5B9;
 *           z ^= z>>27; z *= 0x94D049BB133111EB; z ^= z>>31),
 *   uniform integer below N (N < 2^32): ((r >> 32) * N) >> 32;
 *   j = 3 for FS_0 draws (i counts attempts), 0 for the frontier slot (x below sum_FS deg,
 *   slot = smallest i with prefix_i > x), 1 for the neighbor index, 2 for clipping removals.
 * so any implementation of the same rule reproduces the same subgraphs bit for bit.
 * The parent (symmetric CSR, ascending rows, no self loops) is uploaded once. */
typedef struct gsg_parent* gsg_parent_t;
typedef struct gsg_sample* gsg_sample_t;
GSG_API int gsg_parent_upload(gsg_ctx_t ctx, int64_t N, int64_t nnz, const int64_t* h_indptr,
                              const int32_t* h_indices, gsg_parent_t* out);
GSG_API int gsg_parent_free(gsg_parent_t parent);
/* Sample and induce `count` subgraphs (sampler k uses seed_k above). 1 <= m <= n <= N, m <= 16384,
 * clip >= 1. Synchronizes the context stream once (to size the induced CSR arrays). The call's
 * scratch (bitmaps, lists) stays with the context; the batch's arrays come from, and at
 * gsg_sample_free go back to, a small pool of the context (a config-5 batch of 888 holds 8.3 GB
 * of induced indices), so a sampling loop does not allocate per call. */
GSG_API int gsg_frontier_sample(gsg_ctx_t ctx, gsg_parent_t parent, int32_t n, int32_t m,
                                int32_t clip, uint64_t seed, int32_t count, gsg_sample_t* out);
/* Device views of subgraph k (valid until gsg_sample_free): n_k nodes, nnz_k entries,
 * int64 indptr[n_k+1], int32 indices[nnz_k] (local ids), int32 nodes[n_k] (parent ids,
 * ascending). Pass them to gsg_subgraph_upload_device to train on the sample. */
GSG_API int gsg_sample_get(gsg_sample_t s, int32_t k, int32_t* n_k, int64_t* nnz_k,
                           const int64_t** d_indptr, const int32_t** d_indices,
                           const int32_t** d_nodes);
/* Releases the batch: a device-wide synchronization (as cudaFree), then its arrays return to the
 * pool of the context that sampled it (or are freed, if that context was destroyed first). */
GSG_API int gsg_sample_free(gsg_sample_t s);
/* A subgraph whose sizes live on the device, so that one captured CUDA graph of the training
 * step serves every GPU-sampled subgraph (Alg. 7's pool refill, with Alg. 2 on the
 * device): n (>= 1) nodes fixed at creation, up to nnz_cap raw entries; the actual entry count is
 * indptr[n] on the device. Filled by gsg_sample_load; normalize / SpMM / layer calls then take
 * every size from device memory (host-side sizes are the capacities). Starts as an empty graph.
 * Errors: GSG_EINVAL (n < 1, nnz_cap < 0, NULL out), GSG_ENOMEM. Free with gsg_subgraph_free. */
GSG_API int gsg_subgraph_create_device(gsg_ctx_t ctx, int32_t n, int64_t nnz_cap, gsg_subgraph_t* out);
/* Loads sample *d_k of a gsg_frontier_sample batch into the device-sized subgraph sg, stream
 * ordered and CUDA-graph capturable, then advances *d_k = (*d_k + 1) mod count (d_k: one int32
 * in DEVICE memory, 0 <= *d_k < count). Sample k (n_k nodes, nnz_k entries) occupies nodes
 * 0..n_k-1 of sg; nodes n_k..n-1 are isolated padding (empty rows: normalization gives them
 * their self loop only). Optional outputs (device, n entries): d_nodes_out[i] = the parent id of
 * node i, or -1 for padding (gsg_gather_rows writes zero rows for -1: X_s = X[V_s], Alg. 1
 * line 5); d_node_w[i] = 1/n_k for real nodes and 0 for padding -- as gsg_head's node_w the loss
 * and dS equal those of the n_k-node subgraph (a zero feature row stays zero through the layers,
 * so padding adds nothing to any dW). A sample with n_k > n or nnz_k > nnz_cap leaves sg empty
 * and sets an error flag read by gsg_sample_check. Errors: GSG_EINVAL (NULL, sg not device-sized). */
GSG_API int gsg_sample_load(gsg_ctx_t ctx, gsg_sample_t s, int32_t* d_k, gsg_subgraph_t sg,
                            int32_t* d_nodes_out, float* d_node_w);
/* GSG_OK, or GSG_EINVAL if some gsg_sample_load of this batch did not fit (synchronous). */
GSG_API int gsg_sample_check(gsg_sample_t s);
/* Row gather for the sampled subgraph's inputs (Alg. 1 line 5: X_s = X[V_s], the labels
 * likewise): dst row r (row_bytes bytes, pitch dst_pitch) = src row d_idx[r] (pitch src_pitch),
 * r < rows, all DEVICE pointers (e.g. d_nodes of gsg_sample_get into a parent feature matrix
 * resident in HBM); d_idx[r] < 0 writes a zero row (padding nodes of gsg_sample_load). 16-byte vectors when all pointers, pitches and row_bytes are 16-byte
 * multiples. Errors: GSG_EINVAL (negative sizes, NULL, pitch < row_bytes). */
GSG_API int gsg_gather_rows(gsg_ctx_t ctx, int32_t rows, int64_t row_bytes, const void* d_src,
                            int64_t src_pitch, const int32_t* d_idx, void* d_dst, int64_t dst_pitch);

/* ==== measurement: the aggregation kernels' machine ceiling ================ *
 * Not a step of the method. Random whole-row gathers from the caller's DEVICE matrix X
 * (rows x ldx fp32, row-major, read only), the access pattern of gsg_spmm with the sparse
 * structure removed: each warp gathers rows of row_floats columns at uniformly random row ids,
 * 8 rows in flight, 256-bit loads; grids of 2, 3 and 4 CTAs per SM are timed with CUDA events
 * on the context stream (one warm-up launch each) and the best gathered GB/s is returned in
 * *gbs. With X L2-resident (<= ~half the L2) this is the L2->SM random-gather ceiling that the
 * SpMM's effective bandwidth is reported against. Synchronizes the context stream; must not be
 * called inside a stream capture.
 * Errors: GSG_EINVAL (NULL, rows < 1, row_floats not a multiple of 8 in [8, 256], ldx < row_floats,
 * ldx % 8 != 0, X not 32-byte aligned), GSG_ECUDA. */
GSG_API int gsg_diag_gather_ceiling(gsg_ctx_t ctx, const float* d_X, int32_t rows, int64_t ldx,
                                    int32_t row_floats, double* gbs);

/* ==== data parallelism (row a9) ======================================================== */
/* NCCL plumbing (libnccl.so.2 is resolved at run time; the process's already-loaded copy,
 * e.g. torch's, is reused). The 128-byte unique id is produced on one rank and broadcast
 * by the caller (torch.distributed). */
GSG_API int gsg_nccl_unique_id(void* out_id128);
GSG_API int gsg_nccl_comm_init(gsg_ctx_t ctx, int nranks, int rank, const void* id128,
                               void** out_comm);
GSG_API int gsg_nccl_comm_destroy(void* comm);
/* Sum (average = 1: mean) of each buffer across the communicator's ranks, in place, on the
 * context stream: bufs[i] (device fp32) has counts[i] elements. One grouped call. Returns
 * GSG_ENCCL without enqueueing if the communicator already holds an asynchronous error. */
GSG_API int gsg_allreduce_grads(gsg_ctx_t ctx, void* nccl_comm, float* const* bufs,
                                const int64_t* counts, int nbufs, int average);
/* Failure detection for the collective: waits until everything enqueued on the context stream
 * (e.g. gsg_allreduce_grads) has finished, polling ncclCommGetAsyncError meanwhile. Returns
 * GSG_OK, or GSG_ENCCL if NCCL reports an asynchronous error (a peer failed) or the stream is
 * not done after timeout_ms (> 0; <= 0 waits forever): in both cases the communicator has been
 * aborted (ncclCommAbort) and must not be used or destroyed again. GSG_ECUDA on a CUDA fault. */
GSG_API int gsg_nccl_wait(gsg_ctx_t ctx, void* nccl_comm, int64_t timeout_ms);

#ifdef __cplusplus
}
#endif
#endif /* GSG_H_ */

/*
 * qadapter.h — C ABI of the B200-native quantised tensor-adapter linear.
 *
 * The reference (`lrlm`, /root/reference/pkg/src/lrlm) is pure Python + numpy and has
 * no FFI; its drop-in boundary is the duck-typed linear-backend protocol plus the
 * module functions of quant.py / lowrank.py.  Each entry point below
 * replaces one of those reference functions; the cited file:line is the interface it
 * stands in for.  The Python mirror (paper_2402_13533_b200/) binds these with ctypes
 * (INTEGRATION.md shows the binding).
 *
 * Conventions
 *   - every pointer is a caller-owned DEVICE pointer; the library never allocates or
 *     frees device memory.  Scratch space is caller-allocated and sized by the
 *     matching *_workspace_bytes() query.
 *   - `stream` is a cudaStream_t passed as void*; all work is stream-ordered and the
 *     functions return without synchronising.
 *   - weights are stored (rows = fan_out, cols = fan_in) and applied as x · Wᵀ
 *     (transformer.py:5-7).  Codes use the reference layout exactly: u8 [rows, cols]
 *     for 8 bits, two codes per byte (even column in the low nibble, odd cols padded)
 *     [rows, ceil(cols/2)] for 4 bits (quant.py:37-52).
 *   - return value: QA_OK or a negative qa_status; qa_last_error() describes it.
 *     Non-finite inputs are detected on the device and reported through a
 *     caller-provided int32 flag (checked by the caller at its next sync point),
 *     mirroring QuantError (quant.py:79-80).
 */
#ifndef QADAPTER_H
#define QADAPTER_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define QA_API __attribute__((visibility("default")))
#else
#define QA_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  QA_OK = 0,
  QA_ERR_ARG = -1,         /* bad pointer / shape / stride        (QuantError / ModelError) */
  QA_ERR_BITS = -2,        /* bits not in {4, 8}                  (quant.py:74-75)          */
  QA_ERR_CUDA = -3,        /* a CUDA runtime / driver call failed                           */
  QA_ERR_UNSUPPORTED = -4, /* shape outside the tensor-core path's constraints              */
  QA_ERR_WORKSPACE = -5    /* workspace smaller than *_workspace_bytes()                    */
} qa_status;

typedef enum { QA_F32 = 0, QA_BF16 = 1 } qa_dtype;

#define QA_TT_MAX_D 4

/* Frozen quantised base weight (quant.py:55-70 QuantizedMatrix, on the device). */
typedef struct {
  int64_t rows;          /* fan_out N */
  int64_t cols;          /* fan_in  K */
  int32_t bits;          /* 4 or 8 */
  const uint8_t* codes;  /* reference layout, see above */
  const float* scale;    /* [rows] f32, (hi - lo) / (2^bits - 1) rounded to f32 */
  const float* offset;   /* [rows] f32, row minimum */
  const int32_t* rowsum; /* [rows] Σ_k code[n, k] (unpacked), written by qa_quantize_rows */
} qa_qweight;

/* Tensor-train adapter ΔW = W_t.
 * core k has shape (r[k], m[k], n[k], r[k+1]) row-major fp32, r[0] = r[d] = 1,
 * W_t[(i1..id), (j1..jd)] = G1[0,i1,j1,:] · G2[:,i2,j2,:] ··· Gd[:,id,jd,0]. */
typedef struct {
  int32_t d;
  int32_t m[QA_TT_MAX_D];
  int32_t n[QA_TT_MAX_D];
  int32_t r[QA_TT_MAX_D + 1];
  const float* cores[QA_TT_MAX_D];
} qa_tt;

QA_API const char* qa_version(void);
QA_API const char* qa_last_error(void);

/* quantize_rows (quant.py:73-99), also the per-token activation quantiser
 * (quantize_rows on x.reshape(-1, K); quantize_activations, quant.py:147-152).
 * w: [rows, cols] with row stride ld_w elements, dtype QA_F32 or QA_BF16.
 * codes: reference layout with row stride ld_codes bytes; for bits == 8 the bytes
 * [cols, pad_cols) of each row are zero-filled (GEMM operand padding; pass
 * pad_cols = cols for the plain reference layout).
 * scale/offset: [rows] f32; rowsum: [rows] i32 Σ codes (nullable);
 * nonfinite_flag: device i32 set to 1 when any input is NaN/Inf (nullable). */
QA_API int qa_quantize_rows(const void* w, int w_dtype, int64_t rows, int64_t cols, int64_t ld_w, int bits,
                     uint8_t* codes, int64_t ld_codes, int64_t pad_cols, float* scale, float* offset,
                     int32_t* rowsum, int32_t* nonfinite_flag, void* stream);

/* dequantize_rows (quant.py:102-105): out = code·scale + offset evaluated in fp64,
 * rounded to out_dtype (bit-exact with the reference for QA_F32).
 * transpose != 0 writes outᵀ ([cols, rows], row stride ld_out). */
QA_API int qa_dequantize_rows(const qa_qweight* w, void* out, int out_dtype, int64_t ld_out, int transpose, void* stream);

/* Reference-semantics products against the stored codes, no activation quantisation (quant.py:108-144):
 *   qa_qmatmul   (qmatmul / qmatvec, quant.py:108-132): y  [tokens, rows] f32 = (x·codesᵀ)·scale + Σx·offset
 *   qa_qmatmul_t (qmatmul_t, quant.py:135-144):         dx [tokens, cols] f32 = (dy·scale)·codes + dy·offset
 * x / dy: [tokens, cols] / [tokens, rows], dtype QA_F32 or QA_BF16, contiguous.  The products run on the bf16
 * tensor cores as three chained GEMMs over a 3-term bf16 split of the float operand (codes are exact in
 * bf16), fp64 row terms and epilogue: fp32-accurate against the reference's fp64 result.
 * Workspace from qa_qmatmul_workspace_bytes(w, tokens, transpose) (transpose = 1 for qa_qmatmul_t). */
QA_API size_t qa_qmatmul_workspace_bytes(const qa_qweight* w, int64_t tokens, int transpose);
QA_API int qa_qmatmul(const qa_qweight* w, const void* x, int x_dtype, int64_t tokens, float* y, void* workspace,
                      size_t workspace_bytes, void* stream);
QA_API int qa_qmatmul_t(const qa_qweight* w, const void* dy, int dy_dtype, int64_t tokens, float* dx,
                        void* workspace, size_t workspace_bytes, void* stream);

/* rowsum[r] = Σ_c code[r, c] of a stored code grid (reference layout, row stride = cols or
 * ceil(cols/2) bytes): the qa_qweight.rowsum term for bases loaded from a checkpoint's u8q / u4q
 * entries (checkpoint.py:64-70, 186-197) instead of quantised on the device. */
QA_API int qa_code_rowsum(const uint8_t* codes, int64_t rows, int64_t cols, int bits, int32_t* rowsum, void* stream);

/* Workspace for qa_linear_forward / qa_linear_backward at `tokens` tokens. */
QA_API size_t qa_linear_workspace_bytes(const qa_qweight* w, const qa_tt* tt, int64_t tokens);

/* Forward of the quantised adapter linear (LoraLinear.forward over
 * QuantizedLinear, transformer.py:266-267 + 304-308; qmatmul, quant.py:123-132):
 *   per-token 8-bit act-quant of x, int8 tcgen05 GEMM with exact int32 accumulators,
 *   dequantising epilogue, + y2 = x · W_tᵀ (tt may be NULL: base only).
 * x: [tokens, cols] (dtype x_dtype, row stride = cols).  y: [tokens, rows] bf16.
 * Optional debug outputs (NULL to skip): acc_i32 [tokens, rows] raw Σ cx·cw,
 * y_f32 [tokens, rows] the fp32 pre-rounding y, y2_f32 [tokens, rows] the adapter term (needs y_f32).
 * They come from the same persistent tcgen05 kernels as the plain call (probe outputs of the epilogue),
 * so parity tests that read them pin the production path. */
QA_API int qa_linear_forward(const qa_qweight* w, const qa_tt* tt, const void* x, int x_dtype, int64_t tokens,
                      void* y, int32_t* acc_i32, float* y_f32, float* y2_f32, void* workspace,
                      size_t workspace_bytes, void* stream);

/* Backward with recompute (LoraLinear.backward, transformer.py:310-318, with
 * QuantizedLinear.backward -> qmatmul_t, quant.py:135-144): recomputes the TT partial
 * contractions from the stored layer input x, writes dx = dy · deq(W) + dy · W_t
 * (bf16, NULL to skip) and the adapter-core gradients dcores[k] (fp32, shapes as the
 * cores; accumulate != 0 adds into them like _accumulate, transformer.py:150-156).
 * dx_f32 (nullable) receives the fp32 pre-rounding dx. */
QA_API int qa_linear_backward(const qa_qweight* w, const qa_tt* tt, const void* x, int x_dtype, const void* dy,
                       int dy_dtype, int64_t tokens, void* dx, float* dx_f32, float* const* dcores,
                       int accumulate, void* workspace, size_t workspace_bytes, void* stream);

/* Saved state of the recompute window (PER_LAYER recompute, transformer.py:613-637 / 888-897).
 * The reference re-runs a layer's forward from its stored input right before that layer's
 * backward; the intermediates of that recompute-forward live only until the backward.  For the
 * fast TT family (m_1 = 1, n_d = 1) the only adapter intermediate the backward needs is
 * Z1 = x · G1 ([tokens, n_1-remainder x r_1] fp32, 0.8% of x at the Llama shapes), so the
 * recompute-forward can hand it over instead of the backward reading x a third time.
 * qa_linear_saved_bytes returns 0 when the adapter has no savable state (the *_saved / *_save
 * entry points then behave exactly like qa_linear_forward / qa_linear_backward). */
QA_API size_t qa_linear_saved_bytes(const qa_qweight* w, const qa_tt* tt, int64_t tokens);

/* qa_linear_forward (no debug outputs) that also writes the saved state (nullable). */
QA_API int qa_linear_forward_save(const qa_qweight* w, const qa_tt* tt, const void* x, int x_dtype,
                                  int64_t tokens, void* y, void* saved, size_t saved_bytes, void* workspace,
                                  size_t workspace_bytes, void* stream);

/* qa_linear_backward that takes the saved state of qa_linear_forward_save on the SAME x and cores
 * (nullable: recompute from x). */
QA_API int qa_linear_backward_saved(const qa_qweight* w, const qa_tt* tt, const void* x, int x_dtype,
                                    const void* dy, int dy_dtype, int64_t tokens, void* dx,
                                    float* const* dcores, int accumulate, const void* saved,
                                    size_t saved_bytes, void* workspace, size_t workspace_bytes,
                                    void* stream);

/* Shared-input groups (n = 1..3 members with the same fan_in): a decoder layer applies q / k / v to
 * the same norm1 and up / gate to the same norm2 (_layer_forward, transformer.py:862-874) and sums
 * their input gradients (_layer_backward, transformer.py:919-944).  The group entry points give
 * each member's outputs exactly as its own qa_linear_forward_save / qa_linear_backward_saved would
 * (per-member y, dx and core gradients), but read x once per direction when every member is a
 * pinned-mode tensor-train adapter (first core input-only with 4-wide last input mode, rank 8);
 * otherwise they run the members one after another.  Decode-size batches (1..8 tokens) run each member's
 * act-quant prologue + matrix-vector pass, the next member's prologue overlapping the current pass
 * (programmatic dependent launches; stream order still holds for later work).  saved[i] / saved_bytes[i]
 * as in qa_linear_forward_save (entries or the arrays themselves may be NULL). */
QA_API size_t qa_group_workspace_bytes(int n, const qa_qweight* const* w, const qa_tt* const* tt, int64_t tokens);
QA_API int qa_group_forward(int n, const qa_qweight* const* w, const qa_tt* const* tt, const void* x, int x_dtype,
                            int64_t tokens, void* const* y, void* const* saved, const size_t* saved_bytes,
                            void* workspace, size_t workspace_bytes, void* stream);
/* dcores[i][k]: member i's core-k gradient (all three needed for the shared pass); dx[i] member i's
 * input gradient (the caller sums them, as _layer_backward does). */
QA_API int qa_group_backward(int n, const qa_qweight* const* w, const qa_tt* const* tt, const void* x, int x_dtype,
                             const void* const* dy, int dy_dtype, int64_t tokens, void* const* dx,
                             float* const* const* dcores, int accumulate, const void* const* saved,
                             const size_t* saved_bytes, void* workspace, size_t workspace_bytes, void* stream);

/* AdamW over a flat buffer of n adapter parameters (trainer.py:84-121 adamw_step): float64 masters and
 * moments updated with the reference's exact sequence of float64 operations (no contraction), float32
 * working copies rounded from the masters; step = the optimizer step after increment (t >= 1). */
QA_API int qa_adamw_step(float* params, double* master, double* m, double* v, const float* grads, int64_t n,
                         double lr, double beta1, double beta2, double eps, double weight_decay, int64_t step,
                         void* stream);
/* flags[s] |= 1 when grads[seg_offsets[s] .. seg_offsets[s+1]) holds a NaN / Inf (the reference raises
 * naming the first such tensor, trainer.py:107-108); flags must be zeroed by the caller. */
QA_API int qa_nonfinite_segments(const float* grads, const int64_t* seg_offsets, int nseg, int32_t* flags,
                                 void* stream);

/* Workspace for qa_merge / qa_tt_materialize. */
QA_API size_t qa_merge_workspace_bytes(const qa_tt* tt);

/* Merge (lowrank.py:245-257 via the explicit dequantise route lowrank.py:249-252):
 * out = dequantize_rows(w) + W_t, [rows, cols] in out_dtype (fp64 dequantisation,
 * fp32 W_t, rounded once to out_dtype). */
QA_API int qa_merge(const qa_qweight* w, const qa_tt* tt, void* out, int out_dtype, void* workspace,
             size_t workspace_bytes, void* stream);

/* W_t alone ([N, K] fp32, N = Π m, K = Π n): the contraction of the cores. */
QA_API int qa_tt_materialize(const qa_tt* tt, float* out, void* workspace, size_t workspace_bytes, void* stream);

/* Launch accounting (benchmark / profiling support, not on the reference's API).
 * qa_launch_count(): kernels this library has launched since load (all classes).
 * qa_timing_enable(1) resets and starts per-class CUDA-event timing of every launch on the
 * launching stream; qa_timing_read() synchronises the recorded events and returns, for the
 * named class ("gemm_i8", "gemm_bf16", "quantize", "tt", "dequant", "merge"), the summed
 * device time, the launch count and the summed algorithmic work (int8 ops / flops for GEMMs,
 * bytes for the memory-bound classes). */
QA_API int64_t qa_launch_count(void);
QA_API int qa_timing_enable(int on);
QA_API int qa_timing_read(const char* kernel_class, double* total_ms, int64_t* launches, double* work);

/* Plain bf16 tensor-core GEMM C[M, N] = A[M, K] · B[N, K]ᵀ (fp32 accumulate): the dense
 * forward of a merged adapter (LoraLinear.forward merged path, transformer.py:305-306).
 * Row strides in elements must give 16-byte aligned rows.  out_bf16 / out_f32 nullable. */
QA_API int qa_gemm_bf16(const void* a, int64_t lda, const void* b, int64_t ldb, int64_t m, int64_t n, int64_t k,
                        void* out_bf16, float* out_f32, int64_t ld_out, void* stream);

/* ---------------------------------------------------------------- decoder-layer glue (config 4)
 * The elementwise / row-reduction steps of _layer_forward / _layer_backward (transformer.py:858-946) around
 * the linears, bf16 activations, each one pass over its operands. Row kernels need dim = 256 * {1,2,4,..,32};
 * every buffer 16-byte aligned. */

/* rmsnorm (transformer.py:478-484): y = (s * inv) * gain, inv = rsqrt(mean(s^2) + eps) per row, with
 * s = a, or s = bf16(a + b) written to `sum` (the residual add res1 = x + attn folded in; b and sum both
 * NULL or both set). inv [rows] f32 is nullable (needed by the backward). */
QA_API int qa_rmsnorm_forward(const void* a, const void* b, void* sum, const float* gain, int64_t rows,
                              int64_t dim, float eps, void* y, float* inv, void* stream);

/* _rmsnorm_backward (transformer.py:487-496) for a frozen gain: dx = g*inv - x*(Σ g*x)*inv^3/dim (+ dres),
 * g = gain * Σ_{i<ndy} dys[i] — the summed input gradients of a shared-input group (:922-923, :942-944) and
 * the residual gradient dres (nullable) folded in. */
QA_API int qa_rmsnorm_backward(const void* x, const float* gain, const float* inv, int ndy, const void* const* dys,
                               const void* dres, int64_t rows, int64_t dim, void* dx, void* stream);

/* _rope_rotate (transformer.py:506-519) in place on q and k (k nullable): adjacent pairs of each head
 * vector rotate by pos = row % seq with the f32 [seq, head_dim/2] tables of _rope_tables (:499-503);
 * inverse != 0 applies sign -1 (the backward). */
QA_API int qa_rope(void* q, void* k, int64_t rows, int64_t dim, int head_dim, int seq, const float* cos_t,
                   const float* sin_t, int inverse, void* stream);

/* act = up * silu(gate) (transformer.py:872-874), n elements (multiple of 8). */
QA_API int qa_swiglu_forward(const void* up, const void* gate, void* act, int64_t n, void* stream);

/* dup = dact * silu(gate), dgate = dact * up * s * (1 + gate * (1 - s)), s = sigmoid(gate). */
QA_API int qa_swiglu_backward(const void* up, const void* gate, const void* dact, void* dup, void* dgate, int64_t n,
                              void* stream);

/* cross_entropy_loss / cross_entropy_grad (transformer.py:569-588) over bf16 logits [rows, vocab]:
 * loss_rows[r] = logsumexp - logit[target] (the loss is their mean), dlogits = (softmax - onehot) / rows. */
QA_API int qa_cross_entropy(const void* logits, const int64_t* targets, int64_t rows, int64_t vocab,
                            float* loss_rows, void* dlogits, void* stream);

/* MSE loss against a target (BASELINE config 1's "adapter grads vs MSE to a seeded target"; the
 * reference's own loss is cross-entropy, transformer.py:569-588): loss_rows[r] = Σ_c (y - target)^2 (the loss is
 * their sum / (rows * cols)), dy = 2 (y - target) / (rows * cols) (nullable).  y / dy: QA_F32 or QA_BF16. */
QA_API int qa_mse(const void* y, int y_dtype, const float* target, int64_t rows, int64_t cols, float* loss_rows,
                  void* dy, int dy_dtype, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* QADAPTER_H */

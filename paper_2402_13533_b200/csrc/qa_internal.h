// Internal launcher declarations shared by the kernel translation units and the C ABI.
#pragma once

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/qadapter.h"

namespace qa {

void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* what);

// ------------------------------------------------------------ quantisation
cudaError_t launch_quantize_rows(const void* w, int w_dtype, int64_t rows, int64_t cols, int64_t ld_w, int bits,
                                 uint8_t* codes, int64_t ld_codes, int64_t pad_cols, float* scale, float* offset,
                                 int32_t* rowsum, int32_t* flag, cudaStream_t s);
cudaError_t launch_dequantize(const uint8_t* codes, const float* scale, const float* offset, int64_t rows,
                              int64_t cols, int bits, void* out, int out_dtype, int64_t ld_out, bool transpose,
                              cudaStream_t s, __nv_bfloat16* out_lo = nullptr);
// Transposed bf16 dequantisation of up to kDqJobs matrices (a shared-input group's members) in one launch.
constexpr int kDqJobs = 3;
struct DequantJobs {
  const uint8_t* codes[kDqJobs];
  const float* scale[kDqJobs];
  const float* offset[kDqJobs];
  int64_t rows[kDqJobs], cols[kDqJobs], ldc[kDqJobs], ld_out[kDqJobs];
  int bits[kDqJobs];
  __nv_bfloat16* out[kDqJobs];
  int64_t first[kDqJobs + 1];  // first tile of each job (filled by the launcher)
  int n;
};
cudaError_t launch_dequantize_t_multi(int n, const DequantJobs& jobs, cudaStream_t s);
// 4-bit packed / unpadded codes -> u8 codes [rows, ld_out] with zero padding in [cols, ld_out).
cudaError_t launch_unpack_pad(const uint8_t* codes, int64_t rows, int64_t cols, int bits, uint8_t* out,
                              int64_t ld_out, cudaStream_t s);
// f32 / bf16 [rows, cols] -> bf16 [rows, ld_out] zero padded; out_lo (nullable) = bf16(v - hi).
cudaError_t launch_to_bf16_pad(const void* in, int in_dtype, int64_t rows, int64_t cols, __nv_bfloat16* out,
                               int64_t ld_out, cudaStream_t s, __nv_bfloat16* out_lo = nullptr);

// ------------------------------------------------------------ tensor-train adapter
struct TTDims {
  int d;
  int m[QA_TT_MAX_D], n[QA_TT_MAX_D], r[QA_TT_MAX_D + 1];
  int64_t N, K;
  // per-token size of the left-to-right partial contraction Z_k, k = 0..d
  int64_t zsize[QA_TT_MAX_D + 1];
  int64_t I(int k) const;  // Π_{q<k} m_q
  int64_t J(int k) const;  // Π_{q>=k} n_q  (J(d) = 1)
  int64_t core_numel(int k) const { return (int64_t)r[k] * m[k] * n[k] * r[k + 1]; }
};
bool tt_dims(const qa_tt* tt, TTDims* out);

// out[t, i, ik, b, q] = Σ_{a,j} in[t, i, a, j, q] G[a, ik, j, b]   (stage k of the forward contraction)
cudaError_t launch_tt_stage_fwd(const void* in, int in_dtype, int64_t in_ld, const float* G, float* out,
                                int64_t out_ld, int64_t T, int64_t I, int A, int nk, int64_t Q, int mk, int B,
                                cudaStream_t s);
// din[t, i, a, j, q] = Σ_{ik,b} dout[t, i, ik, b, q] G[a, ik, j, b]
cudaError_t launch_tt_stage_bwd(const void* dout, int dout_dtype, int64_t dout_ld, const float* G, float* din,
                                int64_t din_ld, int64_t T, int64_t I, int A, int nk, int64_t Q, int mk, int B,
                                cudaStream_t s);
// dG[a, ik, j, b] (+)= Σ_{t,i,q} in[t, i, a, j, q] dout[t, i, ik, b, q]; deterministic two-phase reduction.
cudaError_t launch_tt_core_grad(const void* in, int in_dtype, int64_t in_ld, const void* dout, int dout_dtype,
                                int64_t dout_ld, float* partial, int nchunks, float* dG, bool accumulate,
                                int64_t T, int64_t I, int A, int nk, int64_t Q, int mk, int B, cudaStream_t s);
int tt_grad_chunks(int64_t T);
// L[ip, jp, b]: contraction of cores 0..d-2 with the last rank left open (ip < I(d-1), jp < n_0..n_{d-2}).
cudaError_t launch_tt_prefix_full(const TTDims& dd, const float* const* cores, float* L, cudaStream_t s);
// out[(h, i), (jp, j)] = Σ_b L[h, jp, b] Gd[b, i, j]  (+ deq(codes) when codes != NULL)
cudaError_t launch_tt_last_full(const TTDims& dd, const float* L, const float* Gd, const uint8_t* codes,
                                int bits, const float* scale, const float* offset, void* out, int out_dtype,
                                cudaStream_t s);

// generic TT modes through the materialised W_t (tt_dense.cu): bf16 term planes of a matrix / of its transpose
// (order bit p set = plane p holds the lo term), and the projection of dW_t onto every core's gradient
cudaError_t launch_split3_rows(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t ldin,
                               __nv_bfloat16* out, int64_t ld_out, int64_t plane_w, int order, cudaStream_t s);
cudaError_t launch_split3_t(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t ldin,
                            __nv_bfloat16* out, int64_t ld_out, int64_t plane_w, int order, cudaStream_t s);
size_t tt_project_ws_floats(const TTDims& dd);
cudaError_t launch_tt_project(const TTDims& dd, const float* const* cores, const float* dW, float* ws,
                              float* const* dcores, bool accumulate, cudaStream_t s);
constexpr int kPlanesHiLoHi = 2;  // planes (hi, lo, hi): the activation side
constexpr int kPlanesHiHiLo = 4;  // planes (hi, hi, lo): the weight side

// Fused merge / materialise for the fast TT family (no prefix pass): out = W_t (+ deq(codes) when codes != NULL)
bool merge_fast_ok(const TTDims& dd, const void* codes, const void* out);
cudaError_t launch_merge_fast(const TTDims& dd, const float* const* cores, const uint8_t* codes, int bits,
                              const float* scale, const float* offset, void* out, int out_dtype, cudaStream_t s);

// out[i] (+)= Σ_p partial[p][i] in fixed order (deterministic reduction of per-CTA partials)
cudaError_t launch_sum_partials(const float* partial, int nparts, int64_t numel, float* out, bool accumulate,
                                cudaStream_t s);

cudaError_t launch_code_rowsum(const uint8_t* codes, int64_t rows, int64_t cols, int bits, int32_t* rowsum,
                               cudaStream_t s);

// decode-size forward (gemv.cu): 1..8 tokens against the stored codes (dp4a), GEMM-identical epilogue
bool gemv_ok(int64_t T, int64_t K, int bits);
bool pdl_enabled();
cudaError_t launch_gemv(const uint8_t* xc, int64_t ldx, int64_t T, const float* sx, const float* ox,
                        const int32_t* rsx, const uint8_t* wc, int64_t N, int64_t K, int bits, const float* ws,
                        const float* wo, const int32_t* wrs, const float* zl, int64_t ldz, const float* Gl,
                        int64_t Ml, int Cl, const float* addend, __nv_bfloat16* out, float* out32, cudaStream_t s);
// Decode-size forward (1..8 tokens, gemv.cu / tt_fast.cu): one prologue launch and one matrix-vector launch per
// linear or shared-input group.  Members share x (the activation codes of member 0's workspace) and K.
struct GemvMember {
  const uint8_t* wc;  // codes [N][K or K/2]
  int64_t N;
  const float* ws;    // scale, offset, Σcodes per row
  const float* wo;
  const int32_t* wrs;
  const float* zl;    // the adapter's last-core input Zlast [T][ldz] (null: no adapter)
  int64_t ldz;
  const float* Gl;    // last core [Cl][Ml]
  int64_t Ml;
  int Cl;
  const float* addend;  // optional fp32 [T][N] added to y
  __nv_bfloat16* out;
  float* out32;
  int cta0;           // first CTA of this member (filled by the launcher)
};
struct GemvMembers {
  GemvMember m[3];
  int n;
};
bool gemv_mma_ok(int64_t K, int64_t N, const float* Gl, int64_t Ml, int Cl);
cudaError_t launch_gemv_members(const uint8_t* xc, int64_t ldx, int64_t T, const float* sx, const float* ox,
                                const int32_t* rsx, int64_t K, int bits, GemvMembers mem, cudaStream_t s);
struct DecodePrepMember {
  const float* G1;
  const float* G2;  // middle core (d = 3)
  int d, H, C;
  float* z1out;     // optional Z1 export
  float* zlast;     // Zlast [T][ldz]
  int64_t ldz;
};
struct DecodePrepMembers {
  DecodePrepMember m[3];
  int n;
};
cudaError_t launch_decode_prep(const void* x, int64_t T, int64_t K, uint8_t* codes, int64_t ldc, float* sx, float* ox,
                               int32_t* rsx, int J1, int R1, const DecodePrepMembers& mem, cudaStream_t s,
                               bool chain);
// decode prologue (tt_fast.cu): act-quant of T <= 8 bf16 rows + Z1 + the last core's input Zlast


// AdamW (optim.cu)
cudaError_t launch_adamw(float* params, double* master, double* m, double* v, const float* g, int64_t n, double lr,
                         double b1, double b2, double eps, double wd, int64_t step, cudaStream_t s);
cudaError_t launch_seg_nonfinite(const float* g, const int64_t* seg, int nseg, int32_t* flags, cudaStream_t s);

// decoder glue (glue.cu): D = 256 * {1,2,4,8,16,32} for the row kernels
struct GlueDys {
  const __nv_bfloat16* p[3];
  int n;
};
cudaError_t launch_rmsnorm_fwd(const __nv_bfloat16* a, const __nv_bfloat16* b, __nv_bfloat16* sum,
                               const float* gain, __nv_bfloat16* y, float* inv, int64_t rows, int D, float eps,
                               cudaStream_t st);
cudaError_t launch_rmsnorm_bwd(const __nv_bfloat16* x, const float* gain, const float* inv, const GlueDys& dys,
                               const __nv_bfloat16* dres, __nv_bfloat16* dx, int64_t rows, int D, cudaStream_t st);
cudaError_t launch_rope(__nv_bfloat16* x0, __nv_bfloat16* x1, int64_t rows, int D, int head_dim, int seq,
                        const float* cos_t, const float* sin_t, float sign, cudaStream_t st);
cudaError_t launch_swiglu_fwd(const __nv_bfloat16* up, const __nv_bfloat16* gate, __nv_bfloat16* act, int64_t n,
                              cudaStream_t st);
cudaError_t launch_swiglu_bwd(const __nv_bfloat16* up, const __nv_bfloat16* gate, const __nv_bfloat16* dact,
                              __nv_bfloat16* dup, __nv_bfloat16* dgate, int64_t n, cudaStream_t st);
cudaError_t launch_mse(const void* y, int y_dtype, const float* target, int64_t rows, int64_t cols, float* loss_rows,
                       void* dy, int dy_dtype, cudaStream_t st);
cudaError_t launch_xent(const __nv_bfloat16* logits, const int64_t* targets, int64_t rows, int V, float* loss_rows,
                        __nv_bfloat16* dlogits, cudaStream_t st);

// ------------------------------------------------------------ fast TT family (tt_fast.cu)
bool fast_tt_supported(int J1, int R1);
size_t g1i_floats(int64_t K, int J1, int R1);  // workspace for the interleaved G1 copy
cudaError_t launch_actquant_z1(const void* x, int x_dtype, int64_t T, int64_t K, bool want_codes, uint8_t* codes,
                               int64_t ldc, float* sx, float* ox, int32_t* rsx, const float* G1, int J1, int R1,
                               __nv_bfloat16* zb, int64_t ldzb, float* zf, float* g1i_ws, cudaStream_t s,
                               bool frag_ready = false);
// launch_actquant_z1 takes its tensor-core path (the one reading G1 fragments) for these arguments
bool actquant_frag_path(int x_dtype, int64_t K, int J1, int R1, const void* x, bool want_codes, int64_t ldc,
                        const void* codes, const void* zf);
// One launch for the core-only inputs of a forward (tt_fast.cu k_adapter_prep): the G1 MMA fragments of nf
// members (same J1 / R1) and the V operands of nv members.
struct VJob {
  int d, R1, H, J1, C, M;
  const float* G2;
  const float* G3;
  __nv_bfloat16* V;
  int64_t N, ldv;
};
struct AdapterPrep {
  const float* G1[3];
  uint4* frag[3];
  int nf;
  int64_t nfrag, per_f;  // fragment steps per member, blocks per member
  VJob v[3];
  int nv;
  int64_t vstart[4];  // first block of each V job
};
cudaError_t launch_adapter_prep(int J1, int R1, int nf, const float* const* G1, float* const* frag, int64_t K,
                                int nv, const VJob* v, cudaStream_t s);
cudaError_t launch_build_v(int d, int R1, int H, int J1, int C, int M, const float* G2, const float* G3,
                           __nv_bfloat16* V, int64_t N, int64_t ldv, cudaStream_t s);
cudaError_t launch_build_bext(int R1, int J1, const float* G1, __nv_bfloat16* B, int64_t K, int64_t ldb,
                              cudaStream_t s);
cudaError_t launch_split_rows(const float* in, int64_t T, int K2, __nv_bfloat16* out, int64_t ld, cudaStream_t s);
bool mid_fast_ok(int K2, int HC);
int mid_bwd_ctas(int64_t T);
cudaError_t launch_mid_fwd(const float* z1, int64_t T, int K2, int J1, int HC, int C, const float* G2, float* z2,
                           cudaStream_t s);
cudaError_t launch_mid_bwd(const float* dz2, const float* z1, int64_t T, int K2, int J1, int HC, int C,
                           const float* G2, float* dz1, float* gpart, int nctas, cudaStream_t s);
int tt_dy_splits(int64_t T, int blocks_per_split);
cudaError_t launch_tt_dy(const __nv_bfloat16* dy, int64_t T, int64_t N, int H, int M, const float* Z, int64_t zs,
                         int C, const float* Gd, float* dz_part, float* dg_part, int S, cudaStream_t s);
int tt_dg1_splits(int64_t T, int64_t K, int J1);
// dz1: HS partials [HS][T][K2] (summed in fixed order); dz1b (nullable): [hi | lo | hi | 0] split rows
cudaError_t launch_tt_dg1(const void* x, int x_dtype, int64_t T, int64_t K, const float* dz1, int J1, int R1,
                          float* part, int S, cudaStream_t s, int HS = 1, __nv_bfloat16* dz1b = nullptr,
                          int64_t ldb = 0, int* splits_used = nullptr);  // partials written: *splits_used <= S
// fused backward of the pinned Llama modes (d = 3, J1 = 4, M = 256, R1 = C in {8, 16})
bool tt_bwd_fused_ok(int d, int J1, int R1, int C, int M);
void tt_bwd_fused_plan(int64_t T, int H, int C, int* HR, int* HS, int* TS);
cudaError_t launch_tt_bwd_fused(const __nv_bfloat16* dy, int64_t ldy, int64_t T, int H, int C, const float* Z1,
                                const float* G2, const float* G3, float* dz1p, float* g3part, float* g2part,
                                cudaStream_t s);
// rank-8 dy passes of the members of a shared-input group (same H) in one launch (grid z = member)
constexpr int kBwdJobs = 3;
struct BwdJobs {
  const __nv_bfloat16* dy[kBwdJobs];
  int64_t ldy[kBwdJobs];
  const float* Z1[kBwdJobs];
  const float* G2[kBwdJobs];
  const float* G3[kBwdJobs];
  float* dz1p[kBwdJobs];
  float* g3part[kBwdJobs];
  float* g2part[kBwdJobs];
};
cudaError_t launch_tt_bwd_ws_group(const BwdJobs& jobs, int n, int64_t T, int H, cudaStream_t s);
bool make_tmap_rows3d(CUtensorMap* m, const void* x, int64_t T, int64_t cols, int64_t ld, int box_rows, int box_cb);
bool make_tmap_bf16_rows(CUtensorMap* m, const void* x, int64_t rows, int64_t cols, int64_t ld, int box_rows);
// shared-input groups: one x pass for NA in {2, 3} adapters (J1 = 4, R1 = 8)
bool group_x_pass_ok(int J1, int R1, int64_t K, int NA, const void* x);
cudaError_t launch_actquant_z1_group(const void* x, int64_t T, int64_t K, bool want_codes, uint8_t* codes,
                                     int64_t ldc, float* sx, float* ox, int32_t* rsx, const float* const* G1, int NA,
                                     __nv_bfloat16* const* zb, int64_t ldzb, float* const* zf, float* frag_ws,
                                     cudaStream_t s, bool frag_ready = false);
cudaError_t launch_tt_dg1_group(const void* x, int64_t T, int64_t K, const float* const* dz1, float* const* part,
                                int S, int HS, __nv_bfloat16* const* dz1b, int64_t ldb, int NA, int* splits_used,
                                cudaStream_t s);
// out_i (+)= Σ_p parts_i[p] for three partial sets, plus the B_ext operand (bext nullable), one launch
cudaError_t launch_grad_reduce3(const float* const* parts, const int* nparts, const int64_t* numel,
                                float* const* outs, bool accumulate, int R1, int J1, const float* G1,
                                __nv_bfloat16* bext, int64_t K, int64_t ldb, cudaStream_t s);
// the same for the n <= 3 members of a shared-input group in one launch (arrays of 3 n sets, n B_ext jobs)
cudaError_t launch_grad_reduce_n(int n, const float* const* parts, const int* nparts, const int64_t* numel,
                                 float* const* outs, bool accumulate, int R1, int J1, const float* const* G1,
                                 __nv_bfloat16* const* bext, int64_t K, int64_t ldb, cudaStream_t s);

// ------------------------------------------------------------ tcgen05 GEMM
struct GemmEpilogue {
  // int8 path: per-row (activation) and per-column (weight) quantisation terms
  const float* row_scale = nullptr;
  const float* row_offset = nullptr;
  const int32_t* row_sum = nullptr;
  const float* col_scale = nullptr;
  const float* col_offset = nullptr;
  const int32_t* col_sum = nullptr;
  int zp_row = 128, zp_col = 128;
  int k_real = 0;
  const float* addend = nullptr;  // fp32 [M, N]
  int64_t ld_add = 0;
  __nv_bfloat16* out_bf16 = nullptr;
  int64_t ld_out = 0;
  float* out_f32 = nullptr;
  int64_t ld_f32 = 0;
  int32_t* out_acc = nullptr;
  int64_t ld_acc = 0;
  float* out_y2 = nullptr;  // kind 0 with extension: the fp32 adapter term (debug)
  int64_t ld_y2 = 0;
};

// Extension k-blocks: bf16 A2[M, K2] · B2[N, K2]ᵀ, issued after the main k-loop.  kind 0 puts them
// in a separate fp32 accumulator added in the epilogue (y2); kind 1 adds them to the main one.
struct GemmExt {
  const void* A2 = nullptr;
  int64_t lda2 = 0;
  const void* B2 = nullptr;
  int64_t ldb2 = 0;
  int64_t K2 = 0;  // multiple of 64 expected (zero padded)
  int64_t k2_valid = 0;  // columns [k2_valid, K2) are zero in both operands (0: unknown); their MMAs are skipped
};

// C[M, N] = A[M, K] · B[N, K]ᵀ, both operands K-major with row strides lda / ldb (elements).
// kind 0: u8 x u8 -> s32 (dequantising epilogue); kind 1: bf16 x bf16 -> f32.
int gemm_tc(int kind, const void* A, int64_t lda, const void* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
            const GemmEpilogue& epi, cudaStream_t s, const GemmExt* ext = nullptr);

}  // namespace qa

// extern "C" boundary: argument validation, workspace planning and kernel orchestration.
// See include/qadapter.h for the contract and the reference interfaces each entry replaces.
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>

#include "qa_internal.h"

namespace qa {

namespace {
thread_local char g_err[512] = "";
}

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return QA_OK;
  set_error("%s: %s", what, cudaGetErrorString(e));
  return QA_ERR_CUDA;
}

namespace {

constexpr int kMaxRank = 64;

int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// Bump allocator over the caller's workspace (256-byte aligned slices).
struct Bump {
  char* base;
  size_t off = 0;
  explicit Bump(void* b) : base(static_cast<char*>(b)) {}
  template <typename T>
  T* take(int64_t count) {
    off = (off + 255) & ~size_t(255);
    T* p = base ? reinterpret_cast<T*>(base + off) : nullptr;
    off += static_cast<size_t>(std::max<int64_t>(count, 0)) * sizeof(T);
    return p;
  }
};

struct LinearPlan {
  int64_t T = 0, N = 0, K = 0, Kp = 0, Np = 0;
  bool need_wcodes = false, need_dypad = false;
  uint8_t* xcodes = nullptr;
  float* sx = nullptr;
  float* ox = nullptr;
  int32_t* rsx = nullptr;
  uint8_t* wcodes = nullptr;
  int nchunks = 1;
  // generic TT modes (tt_dense.cu): plane widths and buffers
  int64_t Kg = 0, Ng = 0, Tg = 0, K2g = 0, N2g = 0, T2g = 0;
  float* lpre = nullptr;          // prefix contraction of cores 0..d-2
  float* wt32 = nullptr;          // W_t [N, K] fp32
  __nv_bfloat16* b2 = nullptr;    // W_t (or W_tᵀ) term planes
  __nv_bfloat16* a2 = nullptr;    // x (or dy) term planes
  __nv_bfloat16* dyT = nullptr;   // dyᵀ term planes [N, T2g]
  __nv_bfloat16* xT = nullptr;    // xᵀ term planes [K, T2g]
  float* dw32 = nullptr;          // dW_t = dyᵀ x [N, K]
  float* proj = nullptr;          // projection scratch
  __nv_bfloat16* wdt = nullptr;   // deq(W)ᵀ [K, Np]
  __nv_bfloat16* dyb = nullptr;   // dy padded [T, Np]
  __nv_bfloat16* wdt_lo = nullptr;  // fp32-input path: bf16 residuals of deq(W)ᵀ and dy
  __nv_bfloat16* dyb_lo = nullptr;
  float* dxacc = nullptr;           // fp32-input path: partial dx [T, K]
  // fast TT family (m_1 = 1, n_d = 1, d in {2, 3}): see tt_fast.cu
  bool fast = false;
  int fd = 0, R1 = 0, J1 = 0, K2 = 0, K2p = 0, H = 0, M = 0, C = 0, S_dy = 1, S_dg1 = 1;
  __nv_bfloat16* zb = nullptr;    // Z1 bf16 [T, K2p] (GEMM extension operand)
  __nv_bfloat16* v = nullptr;     // V bf16 [N, K2p]
  float* zf = nullptr;            // Z1 fp32 [T, K2]
  float* z2 = nullptr;            // Z2 fp32 [T, H*C] (d = 3)
  float* dzp = nullptr;           // dZ_{d-1} partials [M/256][T][H*C]
  float* dzd = nullptr;           // dZ_{d-1} [T][H*C] (summed)
  float* dz1 = nullptr;           // dZ1 fp32 [T, K2]
  __nv_bfloat16* dz1b = nullptr;  // dZ1 bf16 [T, K2p]
  __nv_bfloat16* bext = nullptr;  // B_ext bf16 [K, K2p]
  float* gpart = nullptr;         // core-gradient partials
  float* g1i = nullptr;           // G1 interleaved for the x pass
  // fused backward (tt_fast.cu k_tt_bwd_fused): d = 3, J1 = 4, M = 256, R1 = C
  bool fused = false;
  int HR = 0, HS = 0, TS = 0;
  float* dz1p = nullptr;          // dZ1 partials [HS][T][K2]
  float* g1p = nullptr;           // dG1 partials [S_dg1][K / J1 * R1]
  float* g2p = nullptr;           // dG2 partials [TS][core-1 numel]
  float* g3p = nullptr;           // dG3 partials [HS * TS][C * 256]
  size_t bytes = 0;
};

// The fast TT family: first core input-only, last core output-only (LoRA is d = 2).
bool plan_fast(const TTDims& dd, int64_t N, int64_t K, LinearPlan* P) {
  const int d = dd.d;
  if ((d != 2 && d != 3) || dd.m[0] != 1 || dd.n[d - 1] != 1) return false;
  const int R1 = dd.r[1];
  const int64_t J1 = K / dd.n[0];
  if (J1 > 64 || !fast_tt_supported(static_cast<int>(J1), R1)) return false;
  const int H = d == 3 ? dd.m[1] : 1;
  const int M = dd.m[d - 1];
  const int C = dd.r[d - 1];
  if ((C != 8 && C != 16) || M % 256 != 0 || N % 8 != 0 || K % 8 != 0) return false;
  P->fast = true;
  P->fd = d;
  P->R1 = R1;
  P->J1 = static_cast<int>(J1);
  P->K2 = R1 * static_cast<int>(J1);
  P->K2p = static_cast<int>(round_up(3 * P->K2, 64));  // 3-term bf16 split of Z1 / dZ1 (tt_fast.cu)
  P->H = H;
  P->M = M;
  P->C = C;
  return true;
}

bool plan_linear(const qa_qweight* w, const TTDims* dd, int64_t T, void* ws, LinearPlan* P, bool f32_path) {
  P->T = T;
  P->N = w->rows;
  P->K = w->cols;
  P->Kp = round_up(P->K, 16);
  P->Np = round_up(P->N, 8);
  P->need_wcodes = w->bits == 4 || P->Kp != P->K;
  Bump b(ws);
  P->xcodes = b.take<uint8_t>(T * P->Kp);
  P->sx = b.take<float>(T);
  P->ox = b.take<float>(T);
  P->rsx = b.take<int32_t>(T);
  if (P->need_wcodes) P->wcodes = b.take<uint8_t>(P->N * P->Kp);
  if (dd != nullptr && plan_fast(*dd, P->N, P->K, P)) {
    const int64_t HC = static_cast<int64_t>(P->H) * P->C;
    const int ncb = P->M / 256;
    P->g1i = b.take<float>(static_cast<int64_t>(g1i_floats(P->K, P->J1, P->R1)));
    P->zb = b.take<__nv_bfloat16>(T * P->K2p);
    P->v = b.take<__nv_bfloat16>(P->N * P->K2p);
    P->zf = b.take<float>(T * P->K2);
    if (P->fd == 3) P->z2 = b.take<float>(T * HC);
    P->dzp = b.take<float>(int64_t(ncb) * T * HC);
    P->dzd = b.take<float>(T * HC);
    P->dz1 = b.take<float>(T * P->K2);
    P->dz1b = b.take<__nv_bfloat16>(T * P->K2p);
    P->bext = b.take<__nv_bfloat16>(P->K * P->K2p);
    P->S_dy = tt_dy_splits(T, ncb * P->H);
    P->S_dg1 = tt_dg1_splits(T, P->K, P->J1);
    P->nchunks = tt_grad_chunks(T);
    int64_t gp = std::max<int64_t>(int64_t(P->H) * P->S_dy * P->C * P->M, int64_t(P->S_dg1) * P->K * P->R1);
    if (P->fd == 3) gp = std::max<int64_t>(gp, dd->core_numel(1) * P->nchunks);
    P->gpart = b.take<float>(gp);
    if (tt_bwd_fused_ok(P->fd, P->J1, P->R1, P->C, P->M)) {
      P->fused = true;
      tt_bwd_fused_plan(T, P->H, P->C, &P->HR, &P->HS, &P->TS);
      P->dz1p = b.take<float>(int64_t(P->HS) * T * P->K2);
      P->g1p = b.take<float>(int64_t(P->S_dg1) * (P->K / P->J1) * P->R1);
      P->g2p = b.take<float>(int64_t(P->TS) * dd->core_numel(1));
      P->g3p = b.take<float>(int64_t(P->HS) * P->TS * P->C * P->M);
    }
  } else if (dd != nullptr) {
    // generic modes: W_t materialised (fp32), its bf16 term planes as the GEMMs' extension operand, the
    // activation planes beside it; dW_t = dyᵀ x and its projection onto the cores for the gradients
    int64_t IP = 1, JP = 1;
    for (int k = 0; k + 1 < dd->d; ++k) {
      IP *= dd->m[k];
      JP *= dd->n[k];
    }
    P->Kg = round_up(P->K, 8);
    P->Ng = round_up(P->N, 8);
    P->Tg = round_up(T, 8);
    P->K2g = round_up(3 * P->Kg, 64);
    P->N2g = round_up(3 * P->Ng, 64);
    P->T2g = round_up(3 * P->Tg, 64);
    P->lpre = b.take<float>(IP * JP * dd->r[dd->d - 1]);
    P->wt32 = b.take<float>(P->N * P->K);
    P->b2 = b.take<__nv_bfloat16>(std::max(P->N * P->K2g, P->K * P->N2g));
    P->a2 = b.take<__nv_bfloat16>(T * std::max(P->K2g, P->N2g));
    P->dyT = b.take<__nv_bfloat16>(P->N * P->T2g);
    P->xT = b.take<__nv_bfloat16>(P->K * P->T2g);
    P->dw32 = b.take<float>(P->N * P->K);
    P->proj = b.take<float>(static_cast<int64_t>(tt_project_ws_floats(*dd)));
  }
  P->wdt = b.take<__nv_bfloat16>(P->K * P->Np);
  P->dyb = b.take<__nv_bfloat16>(T * P->Np);
  if (f32_path) {
    P->wdt_lo = b.take<__nv_bfloat16>(P->K * P->Np);
    P->dyb_lo = b.take<__nv_bfloat16>(T * P->Np);
    P->dxacc = b.take<float>(T * P->K);
  }
  P->bytes = b.off + 256;
  return true;
}

int check_weight(const qa_qweight* w) {
  if (w == nullptr || w->codes == nullptr || w->scale == nullptr || w->offset == nullptr) {
    set_error("qa_qweight: null pointer");
    return QA_ERR_ARG;
  }
  if (w->bits != 4 && w->bits != 8) {
    set_error("bits must be 4 or 8, got %d", w->bits);
    return QA_ERR_BITS;
  }
  if (w->rows < 1 || w->cols < 1) {
    set_error("weight grid must be non-empty, got %lldx%lld", (long long)w->rows, (long long)w->cols);
    return QA_ERR_ARG;
  }
  return QA_OK;
}

int check_tt(const qa_tt* tt, const qa_qweight* w, TTDims* dd) {
  if (!tt_dims(tt, dd)) {
    set_error("invalid TT adapter descriptor (d in [1,%d], r[0]=r[d]=1, positive modes, non-null cores)",
              QA_TT_MAX_D);
    return QA_ERR_ARG;
  }
  for (int k = 0; k <= dd->d; ++k)
    if (dd->r[k] > kMaxRank) {
      set_error("TT rank %d exceeds the supported maximum %d", dd->r[k], kMaxRank);
      return QA_ERR_UNSUPPORTED;
    }
  if (w != nullptr && (dd->N != w->rows || dd->K != w->cols)) {
    set_error("TT modes give %lldx%lld but the base weight is %lldx%lld", (long long)dd->N, (long long)dd->K,
              (long long)w->rows, (long long)w->cols);
    return QA_ERR_ARG;
  }
  return QA_OK;
}

#define QA_TRY_CUDA(expr, what)                         \
  do {                                                  \
    cudaError_t _e = (expr);                            \
    if (_e != cudaSuccess) return cuda_status(_e, what); \
  } while (0)
#define QA_TRY(expr)            \
  do {                          \
    int _s = (expr);            \
    if (_s != QA_OK) return _s; \
  } while (0)

// B-operand codes for the int8 GEMM: the reference layout directly when it already is a
// 16-byte-strided u8 grid, else an unpacked / padded copy in the workspace.
const uint8_t* weight_operand(const qa_qweight* w, const LinearPlan& P, cudaStream_t s, int* status) {
  *status = QA_OK;
  if (!P.need_wcodes) return w->codes;
  cudaError_t e = launch_unpack_pad(w->codes, w->rows, w->cols, w->bits, P.wcodes, P.Kp, s);
  if (e != cudaSuccess) *status = cuda_status(e, "unpack_pad");
  return P.wcodes;
}

}  // namespace
}  // namespace qa

using namespace qa;

extern "C" {

const char* qa_version(void) { return "qadapter 0.1 (sm_100a tcgen05)"; }

const char* qa_last_error(void) { return g_err; }

int qa_quantize_rows(const void* w, int w_dtype, int64_t rows, int64_t cols, int64_t ld_w, int bits,
                     uint8_t* codes, int64_t ld_codes, int64_t pad_cols, float* scale, float* offset,
                     int32_t* rowsum, int32_t* nonfinite_flag, void* stream) {
  if (bits != 4 && bits != 8) {
    set_error("bits must be 4 or 8, got %d", bits);
    return QA_ERR_BITS;
  }
  if (w == nullptr || codes == nullptr || scale == nullptr || offset == nullptr || rows < 0 || cols < 1 ||
      ld_w < cols || (w_dtype != QA_F32 && w_dtype != QA_BF16)) {
    set_error("qa_quantize_rows: bad argument");
    return QA_ERR_ARG;
  }
  const int64_t min_ld = bits == 8 ? std::max(cols, pad_cols) : (cols + 1) / 2;
  if (ld_codes < min_ld || (bits == 4 && pad_cols > cols)) {
    set_error("qa_quantize_rows: code row stride %lld too small", (long long)ld_codes);
    return QA_ERR_ARG;
  }
  return cuda_status(launch_quantize_rows(w, w_dtype, rows, cols, ld_w, bits, codes, ld_codes, std::max(pad_cols, cols),
                                          scale, offset, rowsum, nonfinite_flag, static_cast<cudaStream_t>(stream)),
                     "quantize_rows");
}

int qa_dequantize_rows(const qa_qweight* w, void* out, int out_dtype, int64_t ld_out, int transpose, void* stream) {
  QA_TRY(check_weight(w));
  if (out == nullptr || (out_dtype != QA_F32 && out_dtype != QA_BF16) ||
      ld_out < (transpose ? w->rows : w->cols)) {
    set_error("qa_dequantize_rows: bad output");
    return QA_ERR_ARG;
  }
  return cuda_status(launch_dequantize(w->codes, w->scale, w->offset, w->rows, w->cols, w->bits, out, out_dtype,
                                       ld_out, transpose != 0, static_cast<cudaStream_t>(stream)),
                     "dequantize");
}

int qa_adamw_step(float* params, double* master, double* m, double* v, const float* grads, int64_t n, double lr,
                  double beta1, double beta2, double eps, double weight_decay, int64_t step, void* stream) {
  if ((n > 0 && (params == nullptr || master == nullptr || m == nullptr || v == nullptr || grads == nullptr)) ||
      n < 0 || step < 1 || !(beta1 > 0.0 && beta1 < 1.0) || !(beta2 > 0.0 && beta2 < 1.0) || !(lr > 0.0)) {
    set_error("qa_adamw_step: bad argument");
    return QA_ERR_ARG;
  }
  return cuda_status(launch_adamw(params, master, m, v, grads, n, lr, beta1, beta2, eps, weight_decay, step,
                                  static_cast<cudaStream_t>(stream)),
                     "adamw");
}

int qa_nonfinite_segments(const float* grads, const int64_t* seg_offsets, int nseg, int32_t* flags, void* stream) {
  if (nseg < 0 || (nseg > 0 && (grads == nullptr || seg_offsets == nullptr || flags == nullptr))) {
    set_error("qa_nonfinite_segments: bad argument");
    return QA_ERR_ARG;
  }
  return cuda_status(launch_seg_nonfinite(grads, seg_offsets, nseg, flags, static_cast<cudaStream_t>(stream)),
                     "nonfinite segments");
}

namespace {
bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
bool glue_dim_ok(int64_t D) {
  if (D < 256 || D % 256 != 0) return false;
  const int64_t v = D / 256;
  return v <= 32 && (v & (v - 1)) == 0;
}
}  // namespace

int qa_rmsnorm_forward(const void* a, const void* b, void* sum, const float* gain, int64_t rows, int64_t dim,
                       float eps, void* y, float* inv, void* stream) {
  if (rows < 0 || a == nullptr || gain == nullptr || y == nullptr || (b == nullptr) != (sum == nullptr) ||
      !aligned16(a) || !aligned16(y) || !aligned16(gain) || (b != nullptr && (!aligned16(b) || !aligned16(sum)))) {
    set_error("qa_rmsnorm_forward: bad argument");
    return QA_ERR_ARG;
  }
  if (!glue_dim_ok(dim)) {
    set_error("qa_rmsnorm_forward: dim %lld must be 256 * {1,2,4,...,32}", (long long)dim);
    return QA_ERR_UNSUPPORTED;
  }
  return cuda_status(launch_rmsnorm_fwd(static_cast<const __nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(b),
                                        static_cast<__nv_bfloat16*>(sum), gain, static_cast<__nv_bfloat16*>(y), inv,
                                        rows, static_cast<int>(dim), eps, static_cast<cudaStream_t>(stream)),
                     "rmsnorm forward");
}

int qa_rmsnorm_backward(const void* x, const float* gain, const float* inv, int ndy, const void* const* dys,
                        const void* dres, int64_t rows, int64_t dim, void* dx, void* stream) {
  if (rows < 0 || x == nullptr || gain == nullptr || inv == nullptr || dx == nullptr || dys == nullptr || ndy < 1 ||
      ndy > 3 || !aligned16(x) || !aligned16(dx) || !aligned16(gain) || (dres != nullptr && !aligned16(dres))) {
    set_error("qa_rmsnorm_backward: bad argument");
    return QA_ERR_ARG;
  }
  GlueDys d{};
  d.n = ndy;
  for (int i = 0; i < ndy; ++i) {
    if (dys[i] == nullptr || !aligned16(dys[i])) {
      set_error("qa_rmsnorm_backward: bad dy[%d]", i);
      return QA_ERR_ARG;
    }
    d.p[i] = static_cast<const __nv_bfloat16*>(dys[i]);
  }
  if (!glue_dim_ok(dim)) {
    set_error("qa_rmsnorm_backward: dim %lld must be 256 * {1,2,4,...,32}", (long long)dim);
    return QA_ERR_UNSUPPORTED;
  }
  return cuda_status(launch_rmsnorm_bwd(static_cast<const __nv_bfloat16*>(x), gain, inv, d,
                                        static_cast<const __nv_bfloat16*>(dres), static_cast<__nv_bfloat16*>(dx),
                                        rows, static_cast<int>(dim), static_cast<cudaStream_t>(stream)),
                     "rmsnorm backward");
}

int qa_rope(void* q, void* k, int64_t rows, int64_t dim, int head_dim, int seq, const float* cos_t,
            const float* sin_t, int inverse, void* stream) {
  if (rows < 0 || q == nullptr || cos_t == nullptr || sin_t == nullptr || seq < 1 || head_dim < 8 ||
      head_dim % 8 != 0 || dim % head_dim != 0 || !aligned16(q) || (k != nullptr && !aligned16(k)) ||
      !aligned16(cos_t) || !aligned16(sin_t)) {
    set_error("qa_rope: bad argument (head_dim must be a multiple of 8 dividing dim)");
    return QA_ERR_ARG;
  }
  return cuda_status(launch_rope(static_cast<__nv_bfloat16*>(q), static_cast<__nv_bfloat16*>(k), rows,
                                 static_cast<int>(dim), head_dim, seq, cos_t, sin_t, inverse ? -1.f : 1.f,
                                 static_cast<cudaStream_t>(stream)),
                     "rope");
}

int qa_swiglu_forward(const void* up, const void* gate, void* act, int64_t n, void* stream) {
  if (n < 0 || n % 8 != 0 || up == nullptr || gate == nullptr || act == nullptr || !aligned16(up) ||
      !aligned16(gate) || !aligned16(act)) {
    set_error("qa_swiglu_forward: bad argument (n must be a multiple of 8, 16-byte aligned buffers)");
    return QA_ERR_ARG;
  }
  return cuda_status(launch_swiglu_fwd(static_cast<const __nv_bfloat16*>(up), static_cast<const __nv_bfloat16*>(gate),
                                       static_cast<__nv_bfloat16*>(act), n, static_cast<cudaStream_t>(stream)),
                     "swiglu forward");
}

int qa_swiglu_backward(const void* up, const void* gate, const void* dact, void* dup, void* dgate, int64_t n,
                       void* stream) {
  if (n < 0 || n % 8 != 0 || up == nullptr || gate == nullptr || dact == nullptr || dup == nullptr ||
      dgate == nullptr || !aligned16(up) || !aligned16(gate) || !aligned16(dact) || !aligned16(dup) ||
      !aligned16(dgate)) {
    set_error("qa_swiglu_backward: bad argument (n must be a multiple of 8, 16-byte aligned buffers)");
    return QA_ERR_ARG;
  }
  return cuda_status(launch_swiglu_bwd(static_cast<const __nv_bfloat16*>(up), static_cast<const __nv_bfloat16*>(gate),
                                       static_cast<const __nv_bfloat16*>(dact), static_cast<__nv_bfloat16*>(dup),
                                       static_cast<__nv_bfloat16*>(dgate), n, static_cast<cudaStream_t>(stream)),
                     "swiglu backward");
}

int qa_cross_entropy(const void* logits, const int64_t* targets, int64_t rows, int64_t vocab, float* loss_rows,
                     void* dlogits, void* stream) {
  if (rows < 0 || vocab < 8 || vocab % 8 != 0 || vocab > INT32_MAX || logits == nullptr || targets == nullptr ||
      loss_rows == nullptr || dlogits == nullptr || !aligned16(logits) || !aligned16(dlogits)) {
    set_error("qa_cross_entropy: bad argument (vocab must be a multiple of 8, 16-byte aligned buffers)");
    return QA_ERR_ARG;
  }
  return cuda_status(launch_xent(static_cast<const __nv_bfloat16*>(logits), targets, rows, static_cast<int>(vocab),
                                 loss_rows, static_cast<__nv_bfloat16*>(dlogits), static_cast<cudaStream_t>(stream)),
                     "cross entropy");
}

int qa_mse(const void* y, int y_dtype, const float* target, int64_t rows, int64_t cols, float* loss_rows, void* dy,
           int dy_dtype, void* stream) {
  if (rows < 0 || cols < 1 || y == nullptr || target == nullptr || loss_rows == nullptr ||
      (y_dtype != QA_F32 && y_dtype != QA_BF16) || (dy_dtype != QA_F32 && dy_dtype != QA_BF16)) {
    set_error("qa_mse: bad argument");
    return QA_ERR_ARG;
  }
  return cuda_status(launch_mse(y, y_dtype, target, rows, cols, loss_rows, dy, dy_dtype,
                                static_cast<cudaStream_t>(stream)),
                     "mse");
}

int qa_code_rowsum(const uint8_t* codes, int64_t rows, int64_t cols, int bits, int32_t* rowsum, void* stream) {
  if (bits != 4 && bits != 8) {
    set_error("bits must be 4 or 8, got %d", bits);
    return QA_ERR_BITS;
  }
  if (codes == nullptr || rowsum == nullptr || rows < 0 || cols < 1) {
    set_error("qa_code_rowsum: bad argument");
    return QA_ERR_ARG;
  }
  return cuda_status(launch_code_rowsum(codes, rows, cols, bits, rowsum, static_cast<cudaStream_t>(stream)),
                     "code rowsum");
}

size_t qa_linear_workspace_bytes(const qa_qweight* w, const qa_tt* tt, int64_t tokens) {
  if (check_weight(w) != QA_OK) return 0;
  TTDims dd;
  const TTDims* pd = nullptr;
  if (tt != nullptr) {
    if (check_tt(tt, w, &dd) != QA_OK) return 0;
    pd = &dd;
  }
  LinearPlan P;
  plan_linear(w, pd, tokens, nullptr, &P, true);  // large enough for the fp32-input backward too
  return P.bytes;
}

}  // extern "C"

namespace qa {
namespace {
int linear_forward_impl(const qa_qweight* w, const qa_tt* tt, const void* x, int x_dtype, int64_t tokens, void* y,
                        int32_t* acc_i32, float* y_f32, float* y2_f32, float* z1_save, void* workspace,
                        size_t workspace_bytes, void* stream, bool chain_prologue = false) {
  QA_TRY(check_weight(w));
  if (tokens == 0) return QA_OK;  // empty batch: nothing to do (pointers may be null)
  if (x == nullptr || tokens < 0 || (x_dtype != QA_F32 && x_dtype != QA_BF16) || w->rowsum == nullptr) {
    set_error("qa_linear_forward: bad argument (x, dtype, tokens or weight rowsum)");
    return QA_ERR_ARG;
  }
  if (y2_f32 != nullptr && y_f32 == nullptr) {
    set_error("qa_linear_forward: the y2_f32 probe needs y_f32");
    return QA_ERR_ARG;
  }
  TTDims dd;
  const TTDims* pd = nullptr;
  if (tt != nullptr) {
    QA_TRY(check_tt(tt, w, &dd));
    pd = &dd;
  }
  LinearPlan P;
  plan_linear(w, pd, tokens, nullptr, &P, false);
  if (workspace == nullptr || workspace_bytes < P.bytes) {
    set_error("workspace too small: need %zu bytes", P.bytes);
    return QA_ERR_WORKSPACE;
  }
  plan_linear(w, pd, tokens, workspace, &P, false);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t T = tokens, N = P.N, K = P.K;

  GemmExt ext;
  const bool x_vec = reinterpret_cast<uintptr_t>(x) % 16 == 0;
  // decode-size batches (KV-cached decoding, transformer.py:1043-1080): two launches — the act-quant /
  // adapter prologue and the HBM-bound dp4a matrix-vector pass over the stored codes (gemv.cu)
  if (gemv_ok(T, K, w->bits) && acc_i32 == nullptr && y2_f32 == nullptr &&
      (pd == nullptr || (P.fast && x_vec && x_dtype == QA_BF16 && P.C <= 32))) {
    const float* zl = nullptr;
    const float* gl = nullptr;
    int64_t ldz = 0;
    if (pd == nullptr) {
      QA_TRY_CUDA(launch_quantize_rows(x, x_dtype, T, K, K, 8, P.xcodes, P.Kp, P.Kp, P.sx, P.ox, P.rsx, nullptr, s),
                  "act quantize");
    } else {
      float* zlw = P.fd == 3 ? P.z2 : (z1_save != nullptr ? z1_save : P.zf);
      ldz = P.fd == 3 ? int64_t(P.H) * P.C : P.K2;
      DecodePrepMembers dm{};
      dm.n = 1;
      dm.m[0] = DecodePrepMember{tt->cores[0], tt->cores[1], P.fd, P.H, P.C, z1_save, zlw, ldz};
      QA_TRY_CUDA(launch_decode_prep(x, T, K, P.xcodes, P.Kp, P.sx, P.ox, P.rsx, P.J1, P.R1, dm, s, chain_prologue),
                  "decode prologue");
      zl = zlw;
      gl = tt->cores[P.fd - 1];
    }
    return cuda_status(launch_gemv(P.xcodes, P.Kp, T, P.sx, P.ox, P.rsx, w->codes, N, K, w->bits, w->scale,
                                   w->offset, w->rowsum, zl, ldz, gl, P.M, P.C, nullptr,
                                   static_cast<__nv_bfloat16*>(y), y_f32, s),
                       "decode gemv");
  }
  if (P.fast && x_vec) {
    // (4b, core-only half) one launch: the G1 fragments of the x pass and V = cores 2..d contracted (y2 = Z1 · Vᵀ
    // runs as extension k-blocks of the GEMM)
    const bool frags = actquant_frag_path(x_dtype, K, P.J1, P.R1, x, true, P.Kp, P.xcodes, z1_save);
    const VJob vj{P.fd, P.R1, P.H, P.J1, P.C, P.M, tt->cores[1], P.fd == 3 ? tt->cores[2] : nullptr, P.v, N, P.K2p};
    const float* g1 = tt->cores[0];
    float* fr = P.g1i;
    QA_TRY_CUDA(launch_adapter_prep(P.J1, P.R1, frags ? 1 : 0, &g1, &fr, K, 1, &vj, s), "adapter prep");
    // (2)+(4a) one pass over x: bit-exact per-token act-quant + Z1 = first TT stage
    QA_TRY_CUDA(launch_actquant_z1(x, x_dtype, T, K, true, P.xcodes, P.Kp, P.sx, P.ox, P.rsx, tt->cores[0], P.J1,
                                   P.R1, P.zb, P.K2p, z1_save, P.g1i, s, frags),
                "act quantize + TT stage 1");
    ext.A2 = P.zb;
    ext.lda2 = P.K2p;
    ext.B2 = P.v;
    ext.ldb2 = P.K2p;
    ext.K2 = P.K2p;
    ext.k2_valid = 3 * int64_t(P.K2);  // [hi | lo | hi] planes of K2 columns, zero beyond
  } else {
    // (2) per-token activation quantisation: quantize_rows on x[T, K] (codes padded to Kp with zeros)
    QA_TRY_CUDA(launch_quantize_rows(x, x_dtype, T, K, K, 8, P.xcodes, P.Kp, P.Kp, P.sx, P.ox, P.rsx, nullptr, s),
                "act quantize");
  }
  int st = QA_OK;
  const uint8_t* wop = weight_operand(w, P, s, &st);
  QA_TRY(st);

  // (4) generic TT adapter: y2 = x · W_tᵀ with W_t materialised once per call (O(N K r), token-independent) and
  // the product run as fp32-class extension k-blocks of the int8 GEMM: [x_hi | x_lo | x_hi] · [W_hi | W_hi | W_lo]
  float* y2 = nullptr;
  if (pd != nullptr && ext.K2 == 0) {
    QA_TRY_CUDA(launch_tt_prefix_full(dd, tt->cores, P.lpre, s), "tt prefix");
    QA_TRY_CUDA(launch_tt_last_full(dd, P.lpre, tt->cores[dd.d - 1], nullptr, 8, nullptr, nullptr, P.wt32, QA_F32, s),
                "tt materialize");
    QA_TRY_CUDA(launch_split3_rows(P.wt32, QA_F32, N, K, K, P.b2, P.K2g, P.Kg, kPlanesHiHiLo, s), "W_t planes");
    QA_TRY_CUDA(launch_split3_rows(x, x_dtype, T, K, K, P.a2, P.K2g, P.Kg, kPlanesHiLoHi, s), "x planes");
    ext.A2 = P.a2;
    ext.lda2 = P.K2g;
    ext.B2 = P.b2;
    ext.ldb2 = P.K2g;
    ext.K2 = P.K2g;
    ext.k2_valid = 3 * P.Kg;
  }

  // (3) int8 tcgen05 GEMM with the dequantising epilogue (+ y2)
  GemmEpilogue e;
  e.row_scale = P.sx;
  e.row_offset = P.ox;
  e.row_sum = P.rsx;
  e.col_scale = w->scale;
  e.col_offset = w->offset;
  e.col_sum = w->rowsum;
  e.zp_row = 128;
  e.zp_col = w->bits == 8 ? 128 : 8;
  e.k_real = static_cast<int>(K);
  e.addend = y2;
  e.ld_add = N;
  e.out_bf16 = static_cast<__nv_bfloat16*>(y);
  e.ld_out = N;
  e.out_f32 = y_f32;
  e.ld_f32 = N;
  e.out_acc = acc_i32;
  e.ld_acc = N;
  if (ext.K2 > 0) {
    e.out_y2 = y2_f32;
    e.ld_y2 = N;
  }
  return gemm_tc(0, P.xcodes, P.Kp, wop, P.Kp, T, N, P.Kp, e, s, ext.K2 > 0 ? &ext : nullptr);
}

int linear_backward_impl(const qa_qweight* w, const qa_tt* tt, const void* x, int x_dtype, const void* dy,
                         int dy_dtype, int64_t tokens, void* dx, float* dx_f32, float* const* dcores, int accumulate,
                         const float* z1_saved, void* workspace, size_t workspace_bytes, void* stream) {
  QA_TRY(check_weight(w));
  if (tokens == 0) {
    // empty batch: gradients of an empty sum are zero (unless accumulating)
    if (tt != nullptr && dcores != nullptr && accumulate == 0) {
      TTDims dz;
      QA_TRY(check_tt(tt, w, &dz));
      for (int k = 0; k < dz.d; ++k)
        if (dcores[k] != nullptr)
          QA_TRY_CUDA(cudaMemsetAsync(dcores[k], 0, sizeof(float) * dz.core_numel(k), static_cast<cudaStream_t>(stream)),
                      "memset dcores");
    }
    return QA_OK;
  }
  if (dy == nullptr || tokens < 0 || (x_dtype != QA_F32 && x_dtype != QA_BF16) ||
      (dy_dtype != QA_F32 && dy_dtype != QA_BF16)) {
    set_error("qa_linear_backward: bad argument");
    return QA_ERR_ARG;
  }
  TTDims dd;
  const TTDims* pd = nullptr;
  if (tt != nullptr) {
    QA_TRY(check_tt(tt, w, &dd));
    pd = &dd;
    if (x == nullptr) {
      set_error("qa_linear_backward: the adapter backward needs the stored layer input x");
      return QA_ERR_ARG;
    }
  }
  const bool f32_path = dy_dtype == QA_F32;
  LinearPlan P;
  plan_linear(w, pd, tokens, nullptr, &P, f32_path);
  if (workspace == nullptr || workspace_bytes < P.bytes) {
    set_error("workspace too small: need %zu bytes", P.bytes);
    return QA_ERR_WORKSPACE;
  }
  plan_linear(w, pd, tokens, workspace, &P, f32_path);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t T = tokens, N = P.N, K = P.K;
  const bool want_dx = dx != nullptr || dx_f32 != nullptr;

  GemmExt ext;
  // bf16 view of dy: the dX GEMM operand and the fast dy pass read it through 16-byte copies
  const void* dyb16 = dy;
  int64_t ld_dyb = N;
  bool dy_converted = false;
  auto convert_dy = [&]() -> int {
    if (dy_converted) return QA_OK;
    QA_TRY_CUDA(launch_to_bf16_pad(dy, dy_dtype, T, N, P.dyb, P.Np, s, f32_path ? P.dyb_lo : nullptr), "dy to bf16");
    dyb16 = P.dyb;
    ld_dyb = P.Np;
    dy_converted = true;
    return QA_OK;
  };
  if (f32_path || P.Np != N || reinterpret_cast<uintptr_t>(dy) % 16 != 0) QA_TRY(convert_dy());

  const bool fast = pd != nullptr && P.fast && reinterpret_cast<uintptr_t>(x) % 16 == 0;
  if (fast) {
    // (5) recompute Z1 from the stored layer input, then Z_{d-1}
    const int d = P.fd;
    const float* zf = z1_saved;  // Z1 of this very input, exported by the recompute forward
    if (zf == nullptr) {
      QA_TRY_CUDA(launch_actquant_z1(x, x_dtype, T, K, false, nullptr, 0, nullptr, nullptr, nullptr, tt->cores[0],
                                     P.J1, P.R1, nullptr, 0, P.zf, P.g1i, s),
                  "TT stage 1 recompute");
      zf = P.zf;
    }
    if (P.fused) {
      // one pass over dy: dZ1 partials, dG2 / dG3 partials (Z2 formed on the fly from Z1)
      QA_TRY_CUDA(launch_tt_bwd_fused(static_cast<const __nv_bfloat16*>(dyb16), ld_dyb, T, P.H, P.C, zf,
                                      tt->cores[1], tt->cores[2], P.dz1p, P.g3p, P.g2p, s),
                  "TT fused dy pass");
      // one pass over x: dG1 partials, dZ1 summed over the h-ranges, its bf16 split for the dX GEMM
      const bool want_g1 = dcores != nullptr && dcores[0] != nullptr;
      int s_dg1 = P.S_dg1;
      if (want_g1 || want_dx)
        QA_TRY_CUDA(launch_tt_dg1(x, x_dtype, T, K, P.dz1p, P.J1, P.R1, P.g1p, P.S_dg1, s, P.HS,
                                  want_dx ? P.dz1b : nullptr, P.K2p, &s_dg1),
                    "TT x pass");
      const float* parts[3] = {P.g1p, P.g2p, P.g3p};
      const int nparts[3] = {s_dg1, P.TS, P.HS * P.TS};
      const int64_t numel[3] = {dd.core_numel(0), dd.core_numel(1), dd.core_numel(2)};
      float* outs[3] = {want_g1 ? dcores[0] : nullptr, dcores != nullptr ? dcores[1] : nullptr,
                        dcores != nullptr ? dcores[2] : nullptr};
      QA_TRY_CUDA(launch_grad_reduce3(parts, nparts, numel, outs, accumulate != 0, P.R1, P.J1, tt->cores[0],
                                      want_dx ? P.bext : nullptr, K, P.K2p, s),
                  "reduce core gradients + B_ext");
      if (want_dx) {
        ext.A2 = P.dz1b;
        ext.lda2 = P.K2p;
        ext.B2 = P.bext;
        ext.ldb2 = P.K2p;
        ext.K2 = P.K2p;
        ext.k2_valid = 3 * int64_t(P.K2);  // [hi | lo | hi] planes of K2 columns, zero beyond
      }
    }
    const float* zd = zf;
    int64_t zs = P.K2;
    if (!P.fused) {
    const bool mid_fast = d == 3 && mid_fast_ok(P.K2, P.H * P.C);
    if (d == 3) {
      if (mid_fast)
        QA_TRY_CUDA(launch_mid_fwd(zf, T, P.K2, P.J1, P.H * P.C, P.C, tt->cores[1], P.z2, s), "TT stage 2 recompute");
      else
        QA_TRY_CUDA(launch_tt_stage_fwd(zf, QA_F32, P.K2, tt->cores[1], P.z2, int64_t(P.H) * P.C, T, 1, P.R1, P.J1,
                                        1, P.H, P.C, s),
                    "TT stage 2 recompute");
      zd = P.z2;
      zs = int64_t(P.H) * P.C;
    }
    // dy pass: dZ_{d-1} = dy · G_dᵀ and dG_d = Σ Z_{d-1}ᵀ dy (one read of dy)
    const int ncb = P.M / 256;
    QA_TRY_CUDA(launch_tt_dy(static_cast<const __nv_bfloat16*>(dyb16), T, ld_dyb, P.H, P.M, zd, zs, P.C,
                             tt->cores[d - 1], P.dzp, P.gpart, P.S_dy, s),
                "TT dy pass");
    if (dcores != nullptr && dcores[d - 1] != nullptr)
      QA_TRY_CUDA(launch_sum_partials(P.gpart, P.H * P.S_dy, int64_t(P.C) * P.M, dcores[d - 1], accumulate != 0, s),
                  "reduce dG_d");
    float* dzd = P.dzp;
    if (ncb > 1) {
      QA_TRY_CUDA(launch_sum_partials(P.dzp, ncb, T * P.H * P.C, P.dzd, false, s), "reduce dZ");
      dzd = P.dzd;
    }
    float* dz1 = dzd;
    if (d == 3) {
      const bool want_g2 = dcores != nullptr && dcores[1] != nullptr;
      if (mid_fast) {
        const int nctas = mid_bwd_ctas(T);
        QA_TRY_CUDA(launch_mid_bwd(dzd, zf, T, P.K2, P.J1, P.H * P.C, P.C, tt->cores[1], P.dz1,
                                   want_g2 ? P.gpart : nullptr, nctas, s),
                    "dZ1 + dG2");
        if (want_g2)
          QA_TRY_CUDA(launch_sum_partials(P.gpart, nctas, int64_t(P.K2) * P.H * P.C, dcores[1], accumulate != 0, s),
                      "reduce dG2");
      } else {
        if (want_g2)
          QA_TRY_CUDA(launch_tt_core_grad(zf, QA_F32, P.K2, dzd, QA_F32, int64_t(P.H) * P.C, P.gpart, P.nchunks,
                                          dcores[1], accumulate != 0, T, 1, P.R1, P.J1, 1, P.H, P.C, s),
                      "dG2");
        QA_TRY_CUDA(launch_tt_stage_bwd(dzd, QA_F32, int64_t(P.H) * P.C, tt->cores[1], P.dz1, P.K2, T, 1, P.R1,
                                        P.J1, 1, P.H, P.C, s),
                    "dZ1");
      }
      dz1 = P.dz1;
    }
    // x pass: dG1 = Σ_t x ⊗ dZ1
    if (dcores != nullptr && dcores[0] != nullptr) {
      int s_dg1 = P.S_dg1;
      QA_TRY_CUDA(launch_tt_dg1(x, x_dtype, T, K, dz1, P.J1, P.R1, P.gpart, P.S_dg1, s, 1, nullptr, 0, &s_dg1),
                  "TT x pass");
      QA_TRY_CUDA(launch_sum_partials(P.gpart, s_dg1, K / P.J1 * P.R1, dcores[0], accumulate != 0, s), "reduce dG1");
    }
    if (want_dx) {
      // adapter dx = dZ1 · B_extᵀ as extension k-blocks of the dX GEMM
      QA_TRY_CUDA(launch_split_rows(dz1, T, P.K2, P.dz1b, P.K2p, s), "dZ1 to bf16 hi/lo");
      QA_TRY_CUDA(launch_build_bext(P.R1, P.J1, tt->cores[0], P.bext, K, P.K2p, s), "build B_ext");
      ext.A2 = P.dz1b;
      ext.lda2 = P.K2p;
      ext.B2 = P.bext;
      ext.ldb2 = P.K2p;
      ext.K2 = P.K2p;
      ext.k2_valid = 3 * int64_t(P.K2);  // [hi | lo | hi] planes of K2 columns, zero beyond
    }
    }  // !P.fused
  } else if (pd != nullptr) {
    // generic modes (tt_dense.cu): W_t materialised once; the adapter dx = dy · W_t rides as extension k-blocks of
    // the dX GEMM, dW_t = dyᵀ · x runs on tcgen05 and is projected onto every core (no per-token stage chain)
    QA_TRY_CUDA(launch_tt_prefix_full(dd, tt->cores, P.lpre, s), "tt prefix");
    QA_TRY_CUDA(launch_tt_last_full(dd, P.lpre, tt->cores[dd.d - 1], nullptr, 8, nullptr, nullptr, P.wt32, QA_F32, s),
                "tt materialize");
    if (dcores != nullptr) {
      QA_TRY_CUDA(launch_split3_t(dy, dy_dtype, T, N, N, P.dyT, P.T2g, P.Tg, kPlanesHiLoHi, s), "dy planes");
      QA_TRY_CUDA(launch_split3_t(x, x_dtype, T, K, K, P.xT, P.T2g, P.Tg, kPlanesHiHiLo, s), "x planes");
      GemmEpilogue eg;
      eg.out_f32 = P.dw32;
      eg.ld_f32 = K;
      QA_TRY(gemm_tc(1, P.dyT, P.T2g, P.xT, P.T2g, N, K, P.T2g, eg, s));
      QA_TRY_CUDA(launch_tt_project(dd, tt->cores, P.dw32, P.proj, dcores, accumulate != 0, s), "project dW_t");
    }
    if (want_dx) {
      QA_TRY_CUDA(launch_split3_t(P.wt32, QA_F32, N, K, K, P.b2, P.N2g, P.Ng, kPlanesHiHiLo, s), "W_t planes");
      QA_TRY_CUDA(launch_split3_rows(dy, dy_dtype, T, N, N, P.a2, P.N2g, P.Ng, kPlanesHiLoHi, s), "dy planes");
      ext.A2 = P.a2;
      ext.lda2 = P.N2g;
      ext.B2 = P.b2;
      ext.ldb2 = P.N2g;
      ext.K2 = P.N2g;
      ext.k2_valid = 3 * P.Ng;
    }
  }

  if (want_dx) {
    // dx = dy · deq(W): transient bf16 deq(W)ᵀ [K, Np] + tcgen05 bf16 GEMM (+ adapter dx).
    // bf16 dy: one GEMM (deq(W) rounded once to bf16).  fp32 dy: 3xbf16 split
    // (dy_hi·W_hi + dy_hi·W_lo + dy_lo·W_hi) so fp32 callers keep ~2^-16 relative accuracy.
    if (P.Np != N) {
      QA_TRY_CUDA(cudaMemsetAsync(P.wdt, 0, sizeof(__nv_bfloat16) * K * P.Np, s), "memset wdt");
      if (f32_path) QA_TRY_CUDA(cudaMemsetAsync(P.wdt_lo, 0, sizeof(__nv_bfloat16) * K * P.Np, s), "memset wdt_lo");
    }
    QA_TRY_CUDA(launch_dequantize(w->codes, w->scale, w->offset, N, K, w->bits, P.wdt, QA_BF16, P.Np, true, s,
                                  f32_path ? P.wdt_lo : nullptr),
                "dequantize T");
    const void* a = dyb16;
    const int64_t lda = ld_dyb;
    const float* addend = nullptr;
    if (f32_path) {
      GemmEpilogue e1;
      e1.out_f32 = P.dxacc;
      e1.ld_f32 = K;
      QA_TRY(gemm_tc(1, P.dyb_lo, P.Np, P.wdt, P.Np, T, K, P.Np, e1, s));
      GemmEpilogue e2;
      e2.addend = P.dxacc;
      e2.ld_add = K;
      e2.out_f32 = P.dxacc;
      e2.ld_f32 = K;
      QA_TRY(gemm_tc(1, P.dyb, P.Np, P.wdt_lo, P.Np, T, K, P.Np, e2, s));
      addend = P.dxacc;
    }
    GemmEpilogue e;
    e.addend = addend;
    e.ld_add = K;
    e.out_bf16 = static_cast<__nv_bfloat16*>(dx);
    e.ld_out = K;
    e.out_f32 = dx_f32;
    e.ld_f32 = K;
    QA_TRY(gemm_tc(1, a, lda, P.wdt, P.Np, T, K, P.Np, e, s, ext.K2 > 0 ? &ext : nullptr));
  }
  return QA_OK;
}

}  // namespace
}  // namespace qa

extern "C" {

int qa_linear_forward(const qa_qweight* w, const qa_tt* tt, const void* x, int x_dtype, int64_t tokens,
                      void* y, int32_t* acc_i32, float* y_f32, float* y2_f32, void* workspace,
                      size_t workspace_bytes, void* stream) {
  return linear_forward_impl(w, tt, x, x_dtype, tokens, y, acc_i32, y_f32, y2_f32, nullptr, workspace,
                             workspace_bytes, stream);
}

int qa_linear_backward(const qa_qweight* w, const qa_tt* tt, const void* x, int x_dtype, const void* dy,
                       int dy_dtype, int64_t tokens, void* dx, float* dx_f32, float* const* dcores,
                       int accumulate, void* workspace, size_t workspace_bytes, void* stream) {
  return linear_backward_impl(w, tt, x, x_dtype, dy, dy_dtype, tokens, dx, dx_f32, dcores, accumulate, nullptr,
                              workspace, workspace_bytes, stream);
}

size_t qa_linear_saved_bytes(const qa_qweight* w, const qa_tt* tt, int64_t tokens) {
  if (tt == nullptr || check_weight(w) != QA_OK || tokens <= 0) return 0;
  TTDims dd;
  if (check_tt(tt, w, &dd) != QA_OK) return 0;
  LinearPlan P;
  plan_linear(w, &dd, tokens, nullptr, &P, false);
  return P.fast ? sizeof(float) * static_cast<size_t>(tokens) * P.K2 : 0;
}

int qa_linear_forward_save(const qa_qweight* w, const qa_tt* tt, const void* x, int x_dtype, int64_t tokens,
                           void* y, void* saved, size_t saved_bytes, void* workspace, size_t workspace_bytes,
                           void* stream) {
  const size_t need = qa_linear_saved_bytes(w, tt, tokens);
  if (saved != nullptr && saved_bytes < need) {
    set_error("qa_linear_forward_save: saved buffer needs %zu bytes", need);
    return QA_ERR_WORKSPACE;
  }
  return linear_forward_impl(w, tt, x, x_dtype, tokens, y, nullptr, nullptr, nullptr,
                             need > 0 ? static_cast<float*>(saved) : nullptr, workspace, workspace_bytes, stream);
}

int qa_linear_backward_saved(const qa_qweight* w, const qa_tt* tt, const void* x, int x_dtype, const void* dy,
                             int dy_dtype, int64_t tokens, void* dx, float* const* dcores, int accumulate,
                             const void* saved, size_t saved_bytes, void* workspace, size_t workspace_bytes,
                             void* stream) {
  const size_t need = qa_linear_saved_bytes(w, tt, tokens);
  if (saved != nullptr && saved_bytes < need) {
    set_error("qa_linear_backward_saved: saved buffer holds %zu of %zu bytes", saved_bytes, need);
    return QA_ERR_WORKSPACE;
  }
  return linear_backward_impl(w, tt, x, x_dtype, dy, dy_dtype, tokens, dx, nullptr, dcores, accumulate,
                              need > 0 ? static_cast<const float*>(saved) : nullptr, workspace, workspace_bytes,
                              stream);
}

// ------------------------------------------------------------------ shared-input groups
// A decoder layer applies q / k / v to the same norm1 and up / gate to the same norm2
// (transformer.py:862-874) and sums their input gradients (:919-944).  A group runs those members
// with one x pass in each direction when every member is a pinned-mode adapter (J1 = 4, r = 8);
// otherwise it is the members' single-linear calls in sequence.
}  // extern "C"

namespace qa {
namespace {
constexpr int kMaxGroup = 3;

struct GroupPlan {
  int n = 0;
  TTDims dd[kMaxGroup];
  LinearPlan P[kMaxGroup];
  float* frag = nullptr;
  size_t bytes = 0;
  bool fast = false;
};

int plan_group(int n, const qa_qweight* const* w, const qa_tt* const* tt, int64_t T, void* ws, bool f32_path,
               const void* x, GroupPlan* G) {
  if (n < 1 || n > kMaxGroup || w == nullptr || tt == nullptr) {
    set_error("group of %d members (1..%d supported)", n, kMaxGroup);
    return QA_ERR_ARG;
  }
  G->n = n;
  size_t off = 0;
  bool fast = n >= 2;
  for (int i = 0; i < n; ++i) {
    QA_TRY(check_weight(w[i]));
    if (tt[i] == nullptr) {
      set_error("group member %d has no adapter", i);
      return QA_ERR_ARG;
    }
    QA_TRY(check_tt(tt[i], w[i], &G->dd[i]));
    if (w[i]->cols != w[0]->cols) {
      set_error("group members must share fan_in (%lld vs %lld)", (long long)w[i]->cols, (long long)w[0]->cols);
      return QA_ERR_ARG;
    }
    plan_linear(w[i], &G->dd[i], T, ws != nullptr ? static_cast<char*>(ws) + off : nullptr, &G->P[i], f32_path);
    off += round_up(static_cast<int64_t>(G->P[i].bytes), 256);
    const LinearPlan& P = G->P[i];
    fast = fast && P.fast && P.fused && P.fd == 3 && P.J1 == 4 && P.R1 == 8 && P.HS == G->P[0].HS;
  }
  G->fast = fast && group_x_pass_ok(4, 8, w[0]->cols, n, x);
  G->frag = ws != nullptr ? reinterpret_cast<float*>(static_cast<char*>(ws) + off) : nullptr;
  off += sizeof(float) * kMaxGroup * g1i_floats(w[0]->cols, 4, 8) + 256;
  G->bytes = off;
  return QA_OK;
}
}  // namespace
}  // namespace qa

extern "C" {

size_t qa_group_workspace_bytes(int n, const qa_qweight* const* w, const qa_tt* const* tt, int64_t tokens) {
  GroupPlan G;
  static const uint64_t aligned_probe = 0;
  if (plan_group(n, w, tt, tokens, nullptr, true, &aligned_probe, &G) != QA_OK) return 0;
  return G.bytes;
}

int qa_group_forward(int n, const qa_qweight* const* w, const qa_tt* const* tt, const void* x, int x_dtype,
                     int64_t tokens, void* const* y, void* const* saved, const size_t* saved_bytes, void* workspace,
                     size_t workspace_bytes, void* stream) {
  GroupPlan G;
  QA_TRY(plan_group(n, w, tt, tokens, nullptr, false, x, &G));
  if (tokens == 0) return QA_OK;
  if (x == nullptr || y == nullptr || tokens < 0) {
    set_error("qa_group_forward: bad argument");
    return QA_ERR_ARG;
  }
  if (workspace == nullptr || workspace_bytes < G.bytes) {
    set_error("workspace too small: need %zu bytes", G.bytes);
    return QA_ERR_WORKSPACE;
  }
  QA_TRY(plan_group(n, w, tt, tokens, workspace, false, x, &G));
  // decode-size batches: every member through its prologue + matrix-vector pass, chained so that member
  // i + 1's prologue (its own workspace region, reading only x and its cores) runs while member i's pass
  // streams its weights (programmatic dependent launches, decode prologue / gemv.cu)
  bool decode = x_dtype == QA_BF16 && reinterpret_cast<uintptr_t>(x) % 16 == 0;
  for (int i = 0; i < n && decode; ++i)
    decode = gemv_ok(tokens, w[i]->cols, w[i]->bits) && (tt[i] == nullptr || (G.P[i].fast && G.P[i].C <= 32));
  // decode with every member adapted alike: one prologue launch (member 0's CTAs write the shared activation
  // codes) and one matrix-vector launch over all members' rows
  bool decode_group = decode && n <= 3;
  for (int i = 0; i < n && decode_group; ++i) {
    const LinearPlan& P = G.P[i];
    decode_group = tt[i] != nullptr && P.fast && P.J1 == G.P[0].J1 && P.R1 == G.P[0].R1 &&
                   w[i]->bits == w[0]->bits && gemv_mma_ok(w[i]->cols, P.N, tt[i]->cores[P.fd - 1], P.M, P.C);
  }
  if (decode_group) {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const LinearPlan& P0 = G.P[0];
    const int64_t T = tokens, K = w[0]->cols;
    DecodePrepMembers dm{};
    GemvMembers gm{};
    dm.n = gm.n = n;
    for (int i = 0; i < n; ++i) {
      const LinearPlan& P = G.P[i];
      const size_t need = sizeof(float) * static_cast<size_t>(tokens) * P.K2;
      float* sv = (saved != nullptr && saved[i] != nullptr && saved_bytes != nullptr && saved_bytes[i] >= need)
                      ? static_cast<float*>(saved[i]) : nullptr;
      float* zlw = P.fd == 3 ? P.z2 : (sv != nullptr ? sv : P.zf);
      const int64_t ldz = P.fd == 3 ? int64_t(P.H) * P.C : P.K2;
      dm.m[i] = DecodePrepMember{tt[i]->cores[0], tt[i]->cores[1], P.fd, P.H, P.C, sv, zlw, ldz};
      gm.m[i] = GemvMember{w[i]->codes, P.N, w[i]->scale, w[i]->offset, w[i]->rowsum, zlw, ldz,
                           tt[i]->cores[P.fd - 1], P.M, P.C, nullptr, static_cast<__nv_bfloat16*>(y[i]), nullptr, 0};
    }
    QA_TRY_CUDA(launch_decode_prep(x, T, K, P0.xcodes, P0.Kp, P0.sx, P0.ox, P0.rsx, P0.J1, P0.R1, dm, s, false),
                "group decode prologue");
    return cuda_status(launch_gemv_members(P0.xcodes, P0.Kp, T, P0.sx, P0.ox, P0.rsx, K, w[0]->bits, gm, s),
                       "group decode gemv");
  }
  const bool fast = G.fast && x_dtype == QA_BF16 && !decode;
  if (!fast) {  // the members' single-linear forwards
    for (int i = 0; i < n; ++i) {
      const size_t need = G.P[i].fast ? sizeof(float) * static_cast<size_t>(tokens) * G.P[i].K2 : 0;
      float* sv = (saved != nullptr && saved[i] != nullptr && need > 0 && saved_bytes != nullptr &&
                   saved_bytes[i] >= need) ? static_cast<float*>(saved[i]) : nullptr;
      QA_TRY(linear_forward_impl(w[i], tt[i], x, x_dtype, tokens, y[i], nullptr, nullptr, nullptr, sv,
                                 reinterpret_cast<char*>(G.P[i].xcodes) - 0, G.P[i].bytes, stream,
                                 decode && i > 0 && tt[i] != nullptr));
    }
    return QA_OK;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t T = tokens, K = w[0]->cols;
  LinearPlan& P0 = G.P[0];
  const float* G1[kMaxGroup];
  __nv_bfloat16* zb[kMaxGroup];
  float* zf[kMaxGroup];
  for (int i = 0; i < n; ++i) {
    G1[i] = tt[i]->cores[0];
    zb[i] = G.P[i].zb;
    const size_t need = sizeof(float) * static_cast<size_t>(T) * G.P[i].K2;
    zf[i] = (saved != nullptr && saved[i] != nullptr && saved_bytes != nullptr && saved_bytes[i] >= need)
                ? static_cast<float*>(saved[i]) : nullptr;
  }
  // every member's G1 fragments and V in one launch, then one pass over x: shared codes + each member's Z1
  {
    VJob vj[kMaxGroup];
    float* fr[kMaxGroup];
    const int64_t frag_floats = (K / 64) * 32 * 4;  // uint4 per lane per 64-element segment (J1 = 4, R1 = 8)
    for (int i = 0; i < n; ++i) {
      const LinearPlan& P = G.P[i];
      vj[i] = VJob{P.fd, P.R1, P.H, P.J1, P.C, P.M, tt[i]->cores[1], tt[i]->cores[2], P.v, P.N, P.K2p};
      fr[i] = G.frag + i * frag_floats;
    }
    QA_TRY_CUDA(launch_adapter_prep(4, 8, n, G1, fr, K, n, vj, s), "group adapter prep");
  }
  QA_TRY_CUDA(launch_actquant_z1_group(x, T, K, true, P0.xcodes, P0.Kp, P0.sx, P0.ox, P0.rsx, G1, n, zb, P0.K2p, zf,
                                       G.frag, s, true),
              "group act quantize + TT stage 1");
  for (int i = 0; i < n; ++i) {
    LinearPlan& P = G.P[i];
    int st = QA_OK;
    const uint8_t* wop = weight_operand(w[i], P, s, &st);
    QA_TRY(st);
    GemmEpilogue e;
    e.row_scale = P0.sx;
    e.row_offset = P0.ox;
    e.row_sum = P0.rsx;
    e.col_scale = w[i]->scale;
    e.col_offset = w[i]->offset;
    e.col_sum = w[i]->rowsum;
    e.zp_row = 128;
    e.zp_col = w[i]->bits == 8 ? 128 : 8;
    e.k_real = static_cast<int>(K);
    e.out_bf16 = static_cast<__nv_bfloat16*>(y[i]);
    e.ld_out = P.N;
    GemmExt ext;
    ext.A2 = P.zb;
    ext.lda2 = P.K2p;
    ext.B2 = P.v;
    ext.ldb2 = P.K2p;
    ext.K2 = P.K2p;
    ext.k2_valid = 3 * int64_t(P.K2);  // [hi | lo | hi] planes of K2 columns, zero beyond
    QA_TRY(gemm_tc(0, P0.xcodes, P0.Kp, wop, P.Kp, T, P.N, P0.Kp, e, s, &ext));
  }
  return QA_OK;
}

int qa_group_backward(int n, const qa_qweight* const* w, const qa_tt* const* tt, const void* x, int x_dtype,
                      const void* const* dy, int dy_dtype, int64_t tokens, void* const* dx,
                      float* const* const* dcores, int accumulate, const void* const* saved, const size_t* saved_bytes,
                      void* workspace, size_t workspace_bytes, void* stream) {
  GroupPlan G;
  QA_TRY(plan_group(n, w, tt, tokens, nullptr, dy_dtype == QA_F32, x, &G));
  if (dy == nullptr || x == nullptr || tokens < 0) {
    set_error("qa_group_backward: bad argument");
    return QA_ERR_ARG;
  }
  if (workspace == nullptr || workspace_bytes < G.bytes) {
    set_error("workspace too small: need %zu bytes", G.bytes);
    return QA_ERR_WORKSPACE;
  }
  QA_TRY(plan_group(n, w, tt, tokens, workspace, dy_dtype == QA_F32, x, &G));
  bool fast = G.fast && x_dtype == QA_BF16 && dy_dtype == QA_BF16 && tokens > 0 && dcores != nullptr;
  for (int i = 0; fast && i < n; ++i)
    fast = dy[i] != nullptr && reinterpret_cast<uintptr_t>(dy[i]) % 16 == 0 && G.P[i].Np == G.P[i].N &&
           dcores[i] != nullptr && dcores[i][0] != nullptr && dcores[i][1] != nullptr && dcores[i][2] != nullptr;
  if (!fast) {  // the members' single-linear backwards
    for (int i = 0; i < n; ++i) {
      const size_t need = G.P[i].fast ? sizeof(float) * static_cast<size_t>(tokens) * G.P[i].K2 : 0;
      const float* sv = (saved != nullptr && saved[i] != nullptr && need > 0 && saved_bytes != nullptr &&
                         saved_bytes[i] >= need) ? static_cast<const float*>(saved[i]) : nullptr;
      QA_TRY(linear_backward_impl(w[i], tt[i], x, x_dtype, dy[i], dy_dtype, tokens, dx != nullptr ? dx[i] : nullptr,
                                  nullptr, dcores != nullptr ? dcores[i] : nullptr, accumulate, sv,
                                  reinterpret_cast<char*>(G.P[i].xcodes), G.P[i].bytes, stream));
    }
    return QA_OK;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t T = tokens, K = w[0]->cols;
  // Z1 of each member: handed over by the recompute-forward, else recomputed in one shared x pass
  const float* zfs[kMaxGroup];
  bool all_saved = true;
  for (int i = 0; i < n; ++i) {
    const size_t need = sizeof(float) * static_cast<size_t>(T) * G.P[i].K2;
    zfs[i] = (saved != nullptr && saved[i] != nullptr && saved_bytes != nullptr && saved_bytes[i] >= need)
                 ? static_cast<const float*>(saved[i]) : nullptr;
    all_saved = all_saved && zfs[i] != nullptr;
  }
  if (!all_saved) {
    const float* G1[kMaxGroup];
    float* zf[kMaxGroup];
    for (int i = 0; i < n; ++i) {
      G1[i] = tt[i]->cores[0];
      zf[i] = G.P[i].zf;
      zfs[i] = G.P[i].zf;
    }
    QA_TRY_CUDA(launch_actquant_z1_group(x, T, K, false, nullptr, 0, nullptr, nullptr, nullptr, G1, n, nullptr, 0, zf,
                                         G.frag, s),
                "group TT stage 1 recompute");
  }
  // one pass over each dy; rank-8 members with the same output blocking share one launch
  bool one_dy_launch = n <= kBwdJobs;
  for (int i = 0; i < n && one_dy_launch; ++i) one_dy_launch = G.P[i].C == 8 && G.P[i].H == G.P[0].H;
  if (one_dy_launch) {
    BwdJobs bj{};
    for (int i = 0; i < n; ++i) {
      const LinearPlan& P = G.P[i];
      bj.dy[i] = static_cast<const __nv_bfloat16*>(dy[i]);
      bj.ldy[i] = P.N;
      bj.Z1[i] = zfs[i];
      bj.G2[i] = tt[i]->cores[1];
      bj.G3[i] = tt[i]->cores[2];
      bj.dz1p[i] = P.dz1p;
      bj.g3part[i] = P.g3p;
      bj.g2part[i] = P.g2p;
    }
    QA_TRY_CUDA(launch_tt_bwd_ws_group(bj, n, T, G.P[0].H, s), "group TT fused dy pass");
  } else {
  for (int i = 0; i < n; ++i) {
    LinearPlan& P = G.P[i];
    QA_TRY_CUDA(launch_tt_bwd_fused(static_cast<const __nv_bfloat16*>(dy[i]), P.N, T, P.H, P.C, zfs[i], tt[i]->cores[1],
                                    tt[i]->cores[2], P.dz1p, P.g3p, P.g2p, s),
                "TT fused dy pass");
  }
  }
  // one pass over x for every member's dG1 (+ the dZ1 split rows of the dX GEMMs)
  const float* dz1[kMaxGroup];
  float* g1p[kMaxGroup];
  __nv_bfloat16* dz1b[kMaxGroup];
  for (int i = 0; i < n; ++i) {
    dz1[i] = G.P[i].dz1p;
    g1p[i] = G.P[i].g1p;
    dz1b[i] = dx != nullptr ? G.P[i].dz1b : nullptr;
  }
  int s_dg1 = G.P[0].S_dg1;
  QA_TRY_CUDA(launch_tt_dg1_group(x, T, K, dz1, g1p, G.P[0].S_dg1, G.P[0].HS, dz1b, G.P[0].K2p, n, &s_dg1, s),
              "group TT x pass");
  {  // every member's core-gradient partials (fixed order) and B_ext in one launch
    const float* parts[3 * kMaxGroup];
    int nparts[3 * kMaxGroup];
    int64_t numel[3 * kMaxGroup];
    float* outs[3 * kMaxGroup];
    const float* g1s[kMaxGroup];
    __nv_bfloat16* bexts[kMaxGroup];
    for (int i = 0; i < n; ++i) {
      const LinearPlan& P = G.P[i];
      const float* pp[3] = {P.g1p, P.g2p, P.g3p};
      const int np[3] = {s_dg1, P.TS, P.HS * P.TS};
      for (int k = 0; k < 3; ++k) {
        parts[3 * i + k] = pp[k];
        nparts[3 * i + k] = np[k];
        numel[3 * i + k] = G.dd[i].core_numel(k);
        outs[3 * i + k] = dcores[i][k];
      }
      g1s[i] = tt[i]->cores[0];
      bexts[i] = dx != nullptr && dx[i] != nullptr ? P.bext : nullptr;
    }
    QA_TRY_CUDA(launch_grad_reduce_n(n, parts, nparts, numel, outs, accumulate != 0, G.P[0].R1, G.P[0].J1, g1s, bexts,
                                     K, G.P[0].K2p, s),
                "reduce core gradients + B_ext");
  }
  {  // every member's transient deq(W)ᵀ in one launch
    DequantJobs dj{};
    int nj = 0;
    for (int i = 0; i < n; ++i) {
      if (dx == nullptr || dx[i] == nullptr) continue;
      const LinearPlan& P = G.P[i];
      dj.codes[nj] = w[i]->codes;
      dj.scale[nj] = w[i]->scale;
      dj.offset[nj] = w[i]->offset;
      dj.rows[nj] = P.N;
      dj.cols[nj] = K;
      dj.ldc[nj] = w[i]->bits == 8 ? K : (K + 1) / 2;
      dj.ld_out[nj] = P.Np;
      dj.bits[nj] = w[i]->bits;
      dj.out[nj] = P.wdt;
      ++nj;
    }
    if (nj > 0) QA_TRY_CUDA(launch_dequantize_t_multi(nj, dj, s), "dequantize T");
  }
  for (int i = 0; i < n; ++i) {
    LinearPlan& P = G.P[i];
    const bool want_dx = dx != nullptr && dx[i] != nullptr;
    if (!want_dx) continue;
    GemmEpilogue e;
    e.out_bf16 = static_cast<__nv_bfloat16*>(dx[i]);
    e.ld_out = K;
    GemmExt ext;
    ext.A2 = P.dz1b;
    ext.lda2 = P.K2p;
    ext.B2 = P.bext;
    ext.ldb2 = P.K2p;
    ext.K2 = P.K2p;
    ext.k2_valid = 3 * int64_t(P.K2);  // [hi | lo | hi] planes of K2 columns, zero beyond
    QA_TRY(gemm_tc(1, dy[i], P.N, P.wdt, P.Np, T, K, P.Np, e, s, &ext));
  }
  return QA_OK;
}

size_t qa_merge_workspace_bytes(const qa_tt* tt) {
  TTDims dd;
  if (check_tt(tt, nullptr, &dd) != QA_OK) return 0;
  int64_t IP = 1, JP = 1;
  for (int k = 0; k + 1 < dd.d; ++k) {
    IP *= dd.m[k];
    JP *= dd.n[k];
  }
  return static_cast<size_t>(IP * JP * dd.r[dd.d - 1]) * sizeof(float) + 256;
}

int qa_merge(const qa_qweight* w, const qa_tt* tt, void* out, int out_dtype, void* workspace,
             size_t workspace_bytes, void* stream) {
  QA_TRY(check_weight(w));
  TTDims dd;
  QA_TRY(check_tt(tt, w, &dd));
  if (out == nullptr || (out_dtype != QA_F32 && out_dtype != QA_BF16)) {
    set_error("qa_merge: bad output");
    return QA_ERR_ARG;
  }
  if (workspace == nullptr || workspace_bytes < qa_merge_workspace_bytes(tt)) {
    set_error("workspace too small: need %zu bytes", qa_merge_workspace_bytes(tt));
    return QA_ERR_WORKSPACE;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (merge_fast_ok(dd, w->codes, out))  // one pass: the prefix contraction formed in registers
    return cuda_status(launch_merge_fast(dd, tt->cores, w->codes, w->bits, w->scale, w->offset, out, out_dtype, s),
                       "merge");
  float* L = static_cast<float*>(workspace);
  QA_TRY_CUDA(launch_tt_prefix_full(dd, tt->cores, L, s), "tt prefix");
  return cuda_status(launch_tt_last_full(dd, L, tt->cores[dd.d - 1], w->codes, w->bits, w->scale, w->offset, out,
                                         out_dtype, s),
                     "merge");
}

int qa_tt_materialize(const qa_tt* tt, float* out, void* workspace, size_t workspace_bytes, void* stream) {
  TTDims dd;
  QA_TRY(check_tt(tt, nullptr, &dd));
  if (out == nullptr) {
    set_error("qa_tt_materialize: null output");
    return QA_ERR_ARG;
  }
  if (workspace == nullptr || workspace_bytes < qa_merge_workspace_bytes(tt)) {
    set_error("workspace too small: need %zu bytes", qa_merge_workspace_bytes(tt));
    return QA_ERR_WORKSPACE;
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (merge_fast_ok(dd, nullptr, out))
    return cuda_status(launch_merge_fast(dd, tt->cores, nullptr, 8, nullptr, nullptr, out, QA_F32, s),
                       "tt materialize");
  float* L = static_cast<float*>(workspace);
  QA_TRY_CUDA(launch_tt_prefix_full(dd, tt->cores, L, s), "tt prefix");
  return cuda_status(launch_tt_last_full(dd, L, tt->cores[dd.d - 1], nullptr, 8, nullptr, nullptr, out, QA_F32, s),
                     "tt materialize");
}

int qa_gemm_bf16(const void* a, int64_t lda, const void* b, int64_t ldb, int64_t m, int64_t n, int64_t k,
                 void* out_bf16, float* out_f32, int64_t ld_out, void* stream) {
  if (a == nullptr || b == nullptr || m < 0 || n < 0 || k < 1 || lda < k || ldb < k || ld_out < n ||
      (out_bf16 == nullptr && out_f32 == nullptr)) {
    set_error("qa_gemm_bf16: bad argument");
    return QA_ERR_ARG;
  }
  GemmEpilogue e;
  e.out_bf16 = static_cast<__nv_bfloat16*>(out_bf16);
  e.ld_out = ld_out;
  e.out_f32 = out_f32;
  e.ld_f32 = ld_out;
  return gemm_tc(1, a, lda, b, ldb, m, n, k, e, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

// Reference-semantics products against the stored codes (quant.py:108-144), without activation quantisation:
//
//   qmatmul   : y[t, n]  = (Σ_k x[t, k] · code[n, k]) · scale[n] + (Σ_k x[t, k]) · offset[n]
//   qmatmul_t : dx[t, k] = Σ_n (dy[t, n] · scale[n]) · code[n, k] + Σ_n dy[t, n] · offset[n]
//
// The reference evaluates these in fp64.  Here the dense product runs on the bf16 tensor cores with fp32
// accumulation: codes (0..255) are exact in bf16, and the float operand (x, or dy·scale formed in fp64) is
// split into three bf16 planes hi + mid + lo whose sum carries ~27 significant bits, so the three chained
// tcgen05 GEMMs (gemm_tc kind 1, fp32 addend) form the products to fp32 accuracy.  The row terms (Σx,
// Σ dy·offset) are reduced in fp64 and the scale / offset epilogue is evaluated in fp64.
#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_timing.h"

namespace qa {

namespace {

template <typename InT>
QA_DEV double load_d(const InT* p);
template <>
QA_DEV double load_d<float>(const float* p) {
  return static_cast<double>(*p);
}
template <>
QA_DEV double load_d<__nv_bfloat16>(const __nv_bfloat16* p) {
  return static_cast<double>(__bfloat162float(*p));
}

// One CTA per row: planes[q][row, c] = the q-th bf16 term of v = in[row, c] (· col_scale[c]); pad columns
// [cols, ldp) zero.  rowdot[row] = Σ_c in[row, c] · (col_vec ? col_vec[c] : 1) in fp64 (fixed order:
// per-thread strided partials, then a fixed tree).
template <typename InT>
__global__ void __launch_bounds__(256) k_split3(const InT* __restrict__ in, int64_t cols, int64_t ldin,
                                                const float* __restrict__ col_scale,
                                                const float* __restrict__ col_vec, __nv_bfloat16* __restrict__ planes,
                                                int64_t ldp, int64_t plane_stride, double* __restrict__ rowdot) {
  const int64_t row = blockIdx.x;
  const InT* r = in + row * ldin;
  double acc = 0.0;
  for (int64_t c = threadIdx.x; c < ldp; c += blockDim.x) {
    double v = 0.0;
    if (c < cols) {
      const double raw = load_d(r + c);
      acc += raw * (col_vec != nullptr ? static_cast<double>(col_vec[c]) : 1.0);
      v = col_scale != nullptr ? raw * static_cast<double>(col_scale[c]) : raw;
    }
    const __nv_bfloat16 hi = __double2bfloat16(v);
    const double r1 = v - static_cast<double>(__bfloat162float(hi));
    const __nv_bfloat16 mid = __double2bfloat16(r1);
    const double r2 = r1 - static_cast<double>(__bfloat162float(mid));
    const __nv_bfloat16 lo = __double2bfloat16(r2);
    planes[row * ldp + c] = hi;
    planes[plane_stride + row * ldp + c] = mid;
    planes[2 * plane_stride + row * ldp + c] = lo;
  }
  __shared__ double red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (static_cast<int>(threadIdx.x) < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) rowdot[row] = red[0];
}

// Codes as an exact bf16 operand: out [rows, ldo] (transpose = 0) or its transpose [cols, ldo]
// (transpose = 1, 32 x 32 tiles through shared memory); padding zero.
__global__ void __launch_bounds__(256) k_codes_bf16(const uint8_t* __restrict__ codes, int64_t rows, int64_t cols,
                                                    int bits, __nv_bfloat16* __restrict__ out, int64_t ldo,
                                                    int64_t out_rows, int transpose) {
  __shared__ float tile[32][33];
  const int64_t ldc = bits == 8 ? cols : (cols + 1) / 2;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  auto code = [&](int64_t r, int64_t c) -> float {
    if (r >= rows || c >= cols) return 0.f;
    const uint8_t b = codes[r * ldc + (bits == 8 ? c : c / 2)];
    return static_cast<float>(bits == 8 ? b : ((c & 1) ? (b >> 4) : (b & 0xF)));
  };
  if (!transpose) {
    // block covers out rows r0.., out cols c0.. (out col = code col)
    for (int i = ty; i < 32; i += 8) {
      const int64_t r = r0 + i, c = c0 + tx;
      if (r < out_rows && c < ldo) out[r * ldo + c] = __float2bfloat16_rn(code(r, c));
    }
    return;
  }
  // out[k, n] = code[n, k]: block reads code rows r0.. (n) and cols c0.. (k)
  for (int i = ty; i < 32; i += 8) tile[i][tx] = code(r0 + i, c0 + tx);
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t k = c0 + i, n = r0 + tx;
    if (k < out_rows && n < ldo) out[k * ldo + n] = __float2bfloat16_rn(tile[tx][i]);
  }
}

// qmatmul: y = acc · scale[n] + rowdot[t] · offset[n];  qmatmul_t: dx = acc + rowdot[t]  (in place, fp64 math)
__global__ void __launch_bounds__(256) k_qmm_finish(float* __restrict__ y, int64_t T, int64_t N, int64_t ld,
                                                    const double* __restrict__ rowdot,
                                                    const float* __restrict__ scale,
                                                    const float* __restrict__ offset) {
  const int64_t total = T * N;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = i / N, n = i - t * N;
    float* p = y + t * ld + n;
    const double acc = static_cast<double>(*p);
    const double v = scale != nullptr ? acc * static_cast<double>(scale[n]) + rowdot[t] * static_cast<double>(offset[n])
                                      : acc + rowdot[t];
    *p = static_cast<float>(v);
  }
}

int64_t round8(int64_t v) { return (v + 7) / 8 * 8; }

struct QmmPlan {
  int64_t Ap = 0;  // padded reduction length
  int64_t out_cols = 0;
  __nv_bfloat16* planes = nullptr;
  __nv_bfloat16* codes = nullptr;
  double* rowdot = nullptr;
  size_t bytes = 0;
};

QmmPlan plan_qmm(const qa_qweight* w, int64_t T, bool transpose, void* ws) {
  QmmPlan P;
  const int64_t red = transpose ? w->rows : w->cols;  // reduction length
  P.Ap = round8(red);
  P.out_cols = transpose ? w->cols : w->rows;
  char* base = static_cast<char*>(ws);
  size_t off = 0;
  auto take = [&](size_t n) {
    off = (off + 255) & ~size_t(255);
    char* p = base != nullptr ? base + off : nullptr;
    off += n;
    return p;
  };
  P.planes = reinterpret_cast<__nv_bfloat16*>(take(sizeof(__nv_bfloat16) * 3 * T * P.Ap));
  P.codes = reinterpret_cast<__nv_bfloat16*>(take(sizeof(__nv_bfloat16) * P.out_cols * P.Ap));
  P.rowdot = reinterpret_cast<double*>(take(sizeof(double) * (T > 0 ? T : 1)));
  P.bytes = off + 256;
  return P;
}

int run_qmm(const qa_qweight* w, const void* in, int in_dtype, int64_t T, float* out, void* ws, size_t ws_bytes,
            cudaStream_t s, bool transpose) {
  if (w == nullptr || w->codes == nullptr || w->scale == nullptr || w->offset == nullptr) {
    set_error("qmatmul: null weight");
    return QA_ERR_ARG;
  }
  if (w->bits != 4 && w->bits != 8) {
    set_error("bits must be 4 or 8, got %d", w->bits);
    return QA_ERR_BITS;
  }
  if (T < 0 || (T > 0 && (in == nullptr || out == nullptr)) || (in_dtype != QA_F32 && in_dtype != QA_BF16)) {
    set_error("qmatmul: bad argument");
    return QA_ERR_ARG;
  }
  if (T == 0) return QA_OK;
  const QmmPlan need = plan_qmm(w, T, transpose, nullptr);
  if (ws == nullptr || ws_bytes < need.bytes) {
    set_error("workspace too small: need %zu bytes", need.bytes);
    return QA_ERR_WORKSPACE;
  }
  const QmmPlan P = plan_qmm(w, T, transpose, ws);
  const int64_t red = transpose ? w->rows : w->cols;
  {
    LaunchScope scope(kDequant, double(T) * red * (in_dtype == QA_F32 ? 4 : 2) + 6.0 * T * P.Ap, s);
    count_launches(1);
    const int64_t plane_stride = T * P.Ap;
    const float* cs = transpose ? w->scale : nullptr;
    const float* cv = transpose ? w->offset : nullptr;
    if (in_dtype == QA_F32)
      k_split3<float><<<static_cast<unsigned>(T), 256, 0, s>>>(static_cast<const float*>(in), red, red, cs, cv,
                                                               P.planes, P.Ap, plane_stride, P.rowdot);
    else
      k_split3<__nv_bfloat16><<<static_cast<unsigned>(T), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(in), red,
                                                                       red, cs, cv, P.planes, P.Ap, plane_stride,
                                                                       P.rowdot);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_status(e, "split planes");
  }
  {
    LaunchScope scope(kDequant, double(w->rows) * w->cols * (w->bits / 8.0) + 2.0 * P.out_cols * P.Ap, s);
    count_launches(1);
    // transpose = 0: out [N, Ap] from the code rows; transpose = 1: out [K, Ap = round8(N)] from the code
    // columns (blocks walk 32 code rows x 32 code columns; padding comes out zero either way)
    if (!transpose) {
      const dim3 g2(static_cast<unsigned>((P.Ap + 31) / 32), static_cast<unsigned>((w->rows + 31) / 32));
      k_codes_bf16<<<g2, 256, 0, s>>>(w->codes, w->rows, w->cols, w->bits, P.codes, P.Ap, w->rows, 0);
    } else {
      const dim3 g2(static_cast<unsigned>((w->cols + 31) / 32), static_cast<unsigned>((w->rows + 31) / 32));
      k_codes_bf16<<<g2, 256, 0, s>>>(w->codes, w->rows, w->cols, w->bits, P.codes, P.Ap, w->cols, 1);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_status(e, "codes to bf16");
  }
  // three chained GEMMs: out = hi·Cᵀ, out += mid·Cᵀ, out += lo·Cᵀ
  for (int q = 0; q < 3; ++q) {
    GemmEpilogue e;
    e.out_f32 = out;
    e.ld_f32 = P.out_cols;
    if (q > 0) {
      e.addend = out;
      e.ld_add = P.out_cols;
    }
    const int st = gemm_tc(1, P.planes + static_cast<int64_t>(q) * T * P.Ap, P.Ap, P.codes, P.Ap, T, P.out_cols,
                           P.Ap, e, s);
    if (st != QA_OK) return st;
  }
  LaunchScope scope(kDequant, 8.0 * double(T) * P.out_cols, s);
  count_launches(1);
  const int64_t total = T * P.out_cols;
  const int64_t blocks = (total + 255) / 256;
  k_qmm_finish<<<static_cast<unsigned>(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(
      out, T, P.out_cols, P.out_cols, P.rowdot, transpose ? nullptr : w->scale, transpose ? nullptr : w->offset);
  return cuda_status(cudaGetLastError(), "qmatmul epilogue");
}

}  // namespace
}  // namespace qa

using namespace qa;

extern "C" {

size_t qa_qmatmul_workspace_bytes(const qa_qweight* w, int64_t tokens, int transpose) {
  if (w == nullptr || tokens < 0) return 0;
  return plan_qmm(w, tokens, transpose != 0, nullptr).bytes;
}

int qa_qmatmul(const qa_qweight* w, const void* x, int x_dtype, int64_t tokens, float* y, void* workspace,
               size_t workspace_bytes, void* stream) {
  return run_qmm(w, x, x_dtype, tokens, y, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), false);
}

int qa_qmatmul_t(const qa_qweight* w, const void* dy, int dy_dtype, int64_t tokens, float* dx, void* workspace,
                 size_t workspace_bytes, void* stream) {
  return run_qmm(w, dy, dy_dtype, tokens, dx, workspace, workspace_bytes, static_cast<cudaStream_t>(stream), true);
}

}  // extern "C"

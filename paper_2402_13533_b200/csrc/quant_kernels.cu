// Per-row min/max quantisation, dequantisation and operand-layout kernels.
//
// Bit-exactness contract (quant.py:73-99): lo/hi are exact, the step is the fp64 quotient
// (hi - lo) / (2^b - 1), a code is floor(v + 0.5) of the fp64 quotient v = (w - lo) / step,
// clipped.  The kernel evaluates v in fp32 (|v32 - v64| <= ~5e-5 for v <= 255) and replays
// the exact fp64 sequence (__dsub_rn, __ddiv_rn, __dadd_rn, floor) only for elements whose
// fp32 quotient lies within 2.5e-4 of a rounding boundary (~0.05% of elements), so every
// code equals the reference's while the kernel stays HBM-bound.
#include <math.h>

#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_timing.h"
#include "quant_row.cuh"

namespace qa {

namespace {

// One warp per row.  Pass 1: exact min/max (+ finiteness); pass 2 re-reads the row (L1/L2
// resident) and writes codes, the reference's packed layout for 4 bits, and Σ codes.
template <typename InT, int BITS>
__global__ void __launch_bounds__(256) k_quantize_rows(const InT* __restrict__ w, int64_t rows, int64_t cols,
                                                       int64_t ldw, uint8_t* __restrict__ codes, int64_t ldc,
                                                       int64_t pad_cols, float* __restrict__ scale,
                                                       float* __restrict__ offset, int32_t* __restrict__ rowsum,
                                                       int32_t* __restrict__ flag, int vec_ok) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= rows) return;
  const uint32_t lane = threadIdx.x & 31u;
  const InT* src = w + row * ldw;
  uint8_t* dst = codes + row * ldc;
  const int64_t nvec = vec_ok ? cols / 8 : 0;  // full 8-element chunks on the vector path

  float lo = INFINITY, hi = -INFINITY;
  bool bad = false;
  for (int64_t c = lane; c < nvec; c += 32) {
    float f[8];
    load8<InT>(src + c * 8, f);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      lo = fminf(lo, f[i]);
      hi = fmaxf(hi, f[i]);
      bad |= !isfinite(f[i]);
    }
  }
  for (int64_t k = nvec * 8 + lane; k < cols; k += 32) {
    const float v = to_f32(src[k]);
    lo = fminf(lo, v);
    hi = fmaxf(hi, v);
    bad |= !isfinite(v);
  }
  lo = warp_min(lo);
  hi = warp_max(hi);
  const bool any_bad = __any_sync(0xffffffffu, bad);
  if (any_bad && lane == 0 && flag != nullptr) atomicOr(flag, 1);

  constexpr int kTop = (1 << BITS) - 1;
  const double lo64 = static_cast<double>(lo);
  const double step64 = __ddiv_rn(__dsub_rn(static_cast<double>(hi), lo64), static_cast<double>(kTop));
  const bool flat = !(step64 > 0.0) || any_bad;
  const float inv = flat ? 0.0f : static_cast<float>(1.0 / step64);

  int sum = 0;
  for (int64_t c = lane; c < nvec; c += 32) {
    float f[8];
    load8<InT>(src + c * 8, f);
    uint32_t q[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      q[i] = flat ? 0u : code_of<BITS>(f[i], lo, inv, lo64, step64);
      sum += static_cast<int>(q[i]);
    }
    if (BITS == 8) {
      uint2 packed;
      packed.x = q[0] | (q[1] << 8) | (q[2] << 16) | (q[3] << 24);
      packed.y = q[4] | (q[5] << 8) | (q[6] << 16) | (q[7] << 24);
      *reinterpret_cast<uint2*>(dst + c * 8) = packed;
    } else {
      const uint32_t packed = (q[0] | (q[1] << 4)) | ((q[2] | (q[3] << 4)) << 8) | ((q[4] | (q[5] << 4)) << 16) |
                              ((q[6] | (q[7] << 4)) << 24);
      *reinterpret_cast<uint32_t*>(dst + c * 4) = packed;
    }
  }
  // scalar tail, in (even, odd) pairs so 4-bit bytes are formed by one lane
  for (int64_t k = nvec * 8 + 2 * lane; k < cols; k += 64) {
    const uint32_t q0 = flat ? 0u : code_of<BITS>(to_f32(src[k]), lo, inv, lo64, step64);
    const bool has1 = k + 1 < cols;
    const uint32_t q1 = (flat || !has1) ? 0u : code_of<BITS>(to_f32(src[k + 1]), lo, inv, lo64, step64);
    sum += static_cast<int>(q0 + q1);
    if (BITS == 8) {
      dst[k] = static_cast<uint8_t>(q0);
      if (has1) dst[k + 1] = static_cast<uint8_t>(q1);
    } else {
      dst[k >> 1] = static_cast<uint8_t>(q0 | (q1 << 4));
    }
  }
  if (BITS == 8) {
    for (int64_t k = cols + lane; k < pad_cols; k += 32) dst[k] = 0;
  }
  sum = warp_sum_i(sum);
  if (lane == 0) {
    scale[row] = flat ? 0.0f : __double2float_rn(step64);
    offset[row] = lo;
    if (rowsum != nullptr) rowsum[row] = sum;
  }
}

// One CTA per row with the whole row in registers (production weight quantiser for rows of 8-element
// aligned chunks, cols <= 256 * 8 * CH): every thread issues its CH chunk loads (16 or 32 bytes each) at once,
// so a CTA keeps its row's bytes in flight; min / max meet through warp shuffles and shared memory; the
// codes come from the registers — each input byte crosses HBM exactly once.  Same code rule as
// k_quantize_rows (code_of / codes8: fp32 with an fp64 replay inside the tie band).
template <typename InT, int BITS, int CH, int QR_THREADS>
__global__ void __launch_bounds__(QR_THREADS) k_quantize_rows_reg(const InT* __restrict__ w, int64_t cols,
                                                                   int64_t ldw, uint8_t* __restrict__ codes,
                                                                   int64_t ldc, int64_t pad_cols,
                                                                   float* __restrict__ scale,
                                                                   float* __restrict__ offset,
                                                                   int32_t* __restrict__ rowsum,
                                                                   int32_t* __restrict__ flag) {
  __shared__ float s_lo[QR_THREADS / 32], s_hi[QR_THREADS / 32];
  __shared__ int s_bad[QR_THREADS / 32], s_sum[QR_THREADS / 32];
  const int64_t row = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const InT* src = w + row * ldw;
  const int nchunk = static_cast<int>(cols / 8);
  float v[CH][8];
  float lo = INFINITY, hi = -INFINITY;
  bool bad = false;
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = tid + j * QR_THREADS;
    if (c < nchunk) {
      load8<InT>(src + static_cast<int64_t>(c) * 8, v[j]);
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i) v[j][i] = 0.f;
    }
  }
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    if (tid + j * QR_THREADS < nchunk) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        lo = fminf(lo, v[j][i]);
        hi = fmaxf(hi, v[j][i]);
        bad |= !isfinite(v[j][i]);
      }
    }
  }
  lo = warp_min(lo);
  hi = warp_max(hi);
  const int wbad = __any_sync(0xffffffffu, bad);
  if (lane == 0) {
    s_lo[wid] = lo;
    s_hi[wid] = hi;
    s_bad[wid] = wbad;
  }
  __syncthreads();
  lo = s_lo[0];
  hi = s_hi[0];
  int any_bad = s_bad[0];
#pragma unroll
  for (int i = 1; i < QR_THREADS / 32; ++i) {
    lo = fminf(lo, s_lo[i]);
    hi = fmaxf(hi, s_hi[i]);
    any_bad |= s_bad[i];
  }
  if (any_bad && tid == 0 && flag != nullptr) atomicOr(flag, 1);
  constexpr int kTop = (1 << BITS) - 1;
  const double lo64 = static_cast<double>(lo);
  const double step64 = __ddiv_rn(__dsub_rn(static_cast<double>(hi), lo64), static_cast<double>(kTop));
  const bool flat = !(step64 > 0.0) || any_bad;
  const float inv = flat ? 0.0f : static_cast<float>(1.0 / step64);
  uint8_t* dst = codes + row * ldc;
  int sum = 0;
#pragma unroll
  for (int j = 0; j < CH; ++j) {
    const int c = tid + j * QR_THREADS;
    if (c >= nchunk) continue;
    if (BITS == 8) {
      uint2 packed = make_uint2(0u, 0u);
      if (!flat) codes8(v[j], lo, inv, lo64, step64, packed.x, packed.y, sum);
      *reinterpret_cast<uint2*>(dst + static_cast<int64_t>(c) * 8) = packed;
    } else {
      uint32_t packed = 0u;
      if (!flat) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const uint32_t q = code_of<4>(v[j][i], lo, inv, lo64, step64);
          sum += static_cast<int>(q);
          packed |= q << (4 * i);
        }
      }
      *reinterpret_cast<uint32_t*>(dst + static_cast<int64_t>(c) * 4) = packed;
    }
  }
  if (BITS == 8)
    for (int64_t k = cols + tid; k < pad_cols; k += QR_THREADS) dst[k] = 0;
  sum = warp_sum_i(sum);
  if (lane == 0) s_sum[wid] = sum;
  __syncthreads();
  if (tid == 0) {
    int t = 0;
#pragma unroll
    for (int i = 0; i < QR_THREADS / 32; ++i) t += s_sum[i];
    scale[row] = flat ? 0.0f : __double2float_rn(step64);
    offset[row] = lo;
    if (rowsum != nullptr) rowsum[row] = t;
  }
}

QA_DEV uint32_t unpack_code(const uint8_t* row, int64_t k, int bits) {
  if (bits == 8) return row[k];
  const uint32_t b = row[k >> 1];
  return (k & 1) ? (b >> 4) : (b & 0xFu);
}

template <typename OutT>
QA_DEV OutT from_f64(double v);
template <>
QA_DEV float from_f64<float>(double v) {
  return __double2float_rn(v);
}
template <>
QA_DEV __nv_bfloat16 from_f64<__nv_bfloat16>(double v) {
  return __float2bfloat16_rn(__double2float_rn(v));
}

// out[n, k] (or out[k, n]) = code · scale + offset in fp64 (quant.py:102-105), 32x32 tiles.
template <typename OutT, bool TRANS>
__global__ void __launch_bounds__(256) k_dequantize(const uint8_t* __restrict__ codes, int64_t ldc,
                                                    const float* __restrict__ scale,
                                                    const float* __restrict__ offset, int64_t rows, int64_t cols,
                                                    int bits, OutT* __restrict__ out, int64_t ld_out,
                                                    __nv_bfloat16* __restrict__ out_lo) {
  __shared__ OutT tile[32][33];
  __shared__ __nv_bfloat16 tile_lo[32][34];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 32 x 8
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + tx;
    if (r < rows && c < cols) {
      const double v = __dadd_rn(__dmul_rn(static_cast<double>(unpack_code(codes + r * ldc, c, bits)),
                                           static_cast<double>(scale[r])),
                                 static_cast<double>(offset[r]));
      const OutT hi = from_f64<OutT>(v);
      // bf16 split: lo = bf16(v - hi), so hi + lo carries ~16 mantissa bits (3xbf16 fp32 path)
      const __nv_bfloat16 lo = __float2bfloat16_rn(__double2float_rn(v - static_cast<double>(to_f32(hi))));
      if (TRANS) {
        tile[i][tx] = hi;
        tile_lo[i][tx] = lo;
      } else {
        out[r * ld_out + c] = hi;
        if (out_lo != nullptr) out_lo[r * ld_out + c] = lo;
      }
    }
  }
  if (TRANS) {
    __syncthreads();
    for (int i = ty; i < 32; i += 8) {
      const int64_t c = c0 + i, r = r0 + tx;
      if (r < rows && c < cols) {
        out[c * ld_out + r] = tile[tx][i];
        if (out_lo != nullptr) out_lo[c * ld_out + r] = tile_lo[tx][i];
      }
    }
  }
}

// Transposed bf16 dequantisation for the dX GEMM operand: outᵀ[k, n] = bf16(code·scale + offset),
// 64 x 64 tiles, 16-byte code loads and 16-byte stores (full tiles; edges go through k_dequantize).  The
// shared tile is [k][n] with its 16-byte n-chunks XOR-swizzled by k / 16, so the transposing 2-byte stores
// of a warp (8 rows n x 4 column blocks k) land on distinct banks and the row reads stay conflict-free.
template <int BITS>
struct T64Codes {  // one thread's 16 codes of a 64 x 64 tile: row n0 + t / 4, columns k0 + 16 (t % 4) ..
  uint32_t w[BITS == 8 ? 4 : 2];
};

template <int BITS>
QA_DEV T64Codes<BITS> dequant_t64_load(const uint8_t* __restrict__ codes, int64_t ldc, int64_t bx, int64_t by) {
  const int t = threadIdx.x, r = t >> 2, seg = t & 3;
  const int64_t n = by * 64 + r, k0 = bx * 64;
  T64Codes<BITS> c;
  if (BITS == 8) {
    const uint4 u = __ldg(reinterpret_cast<const uint4*>(codes + n * ldc + k0 + seg * 16));
    c.w[0] = u.x;
    c.w[1] = u.y;
    c.w[2] = u.z;
    c.w[3] = u.w;
  } else {
    const uint2 u = __ldg(reinterpret_cast<const uint2*>(codes + n * ldc + (k0 + seg * 16) / 2));
    c.w[0] = u.x;
    c.w[1] = u.y;
  }
  return c;
}

// Transposed bf16 dequantisation for the dX GEMM operand: outᵀ[k, n] = bf16(code·scale + offset),
// 64 x 64 tiles, 16-byte code loads and 16-byte stores (full tiles; edges go through k_dequantize).  The
// shared tile is [k][n] with its 16-byte n-chunks XOR-swizzled by k / 16, so the transposing 2-byte stores
// of a warp (8 rows n x 4 column blocks k) land on distinct banks and the row reads stay conflict-free.
// sh / sl: [64][64] shared tiles (sl only for the hi / lo split of fp32 callers).
template <int BITS>
QA_DEV void dequant_t64_store(const T64Codes<BITS>& cw, const float* __restrict__ scale,
                              const float* __restrict__ offset, __nv_bfloat16* __restrict__ out, int64_t ld_out,
                              __nv_bfloat16* __restrict__ out_lo, int64_t bx, int64_t by, __nv_bfloat16 (*sh)[64],
                              __nv_bfloat16 (*sl)[64]) {
  const int64_t n0 = by * 64, k0 = bx * 64;
  const int t = threadIdx.x;
  const int r = t >> 2, seg = t & 3;  // row n0 + r, columns k0 + 16 seg .. + 15
  const int64_t n = n0 + r;
  const int col = (((r >> 3) ^ seg) << 3) | (r & 7);  // swizzled position of n in rows k = 16 seg + i
  uint32_t c[16];
#pragma unroll
  for (int i = 0; i < 16; ++i)
    c[i] = BITS == 8 ? (cw.w[i >> 2] >> (8 * (i & 3))) & 0xFFu : (cw.w[i >> 3] >> (4 * (i & 7))) & 0xFu;
  if (out_lo == nullptr) {
    // bf16 operand of the dX GEMM: one fp32 FMA per code (its rounding sits 2^-16 below the bf16 step)
    const float s = scale[n], o = offset[n];
#pragma unroll
    for (int i = 0; i < 16; ++i) sh[seg * 16 + i][col] = __float2bfloat16_rn(fmaf(static_cast<float>(c[i]), s, o));
  } else {  // hi / lo split for fp32 callers: the reference's fp64 value (quant.py:102-105)
    const double s = static_cast<double>(scale[n]), o = static_cast<double>(offset[n]);
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const double v = __dadd_rn(__dmul_rn(static_cast<double>(c[i]), s), o);
      const __nv_bfloat16 hi = __float2bfloat16_rn(__double2float_rn(v));
      sh[seg * 16 + i][col] = hi;
      sl[seg * 16 + i][col] = __float2bfloat16_rn(__double2float_rn(v - double(__bfloat162float(hi))));
    }
  }
  __syncthreads();
#pragma unroll
  for (int pass = 0; pass < 2; ++pass) {
    const int kk = (t >> 3) + pass * 32, ch = t & 7;
    const int pch = (ch ^ ((kk >> 4) & 3)) << 3;  // physical chunk of logical chunk ch in row kk
    *reinterpret_cast<uint4*>(out + (k0 + kk) * ld_out + n0 + ch * 8) = *reinterpret_cast<const uint4*>(&sh[kk][pch]);
    if (out_lo != nullptr)
      *reinterpret_cast<uint4*>(out_lo + (k0 + kk) * ld_out + n0 + ch * 8) =
          *reinterpret_cast<const uint4*>(&sl[kk][pch]);
  }
}

template <int BITS>
__global__ void __launch_bounds__(256) k_dequant_t64(const uint8_t* __restrict__ codes, int64_t ldc,
                                                     const float* __restrict__ scale,
                                                     const float* __restrict__ offset,
                                                     __nv_bfloat16* __restrict__ out, int64_t ld_out,
                                                     __nv_bfloat16* __restrict__ out_lo) {
  __shared__ __align__(16) __nv_bfloat16 sh[64][64];
  __shared__ __align__(16) __nv_bfloat16 sl[64][64];
  const T64Codes<BITS> c = dequant_t64_load<BITS>(codes, ldc, blockIdx.x, blockIdx.y);
  dequant_t64_store<BITS>(c, scale, offset, out, ld_out, out_lo, blockIdx.x, blockIdx.y, sh, sl);
}

// The same for up to kDqJobs matrices in one launch (the members of a shared-input group), dq_tpb(BITS) tiles per
// block: block b takes tiles dq_tpb b .. of the concatenated row-major tile lists (job j from tile first[j]); every
// tile's code loads are issued before the first tile is converted (16 bytes of 8-bit codes or 8 bytes of 4-bit codes
// per tile and thread: two 8-bit tiles, four 4-bit tiles; measured 0.152 -> 0.126 ms per 7B step, 1.09 -> 1.04 ms per
// 70B int4 step).
constexpr int dq_tpb(int bits) { return bits == 4 ? 4 : 2; }

template <int BITS>
__global__ void __launch_bounds__(256) k_dequant_t64_multi(const DequantJobs J) {
  __shared__ __align__(16) __nv_bfloat16 sh[64][64];
  constexpr int DQ_TPB = dq_tpb(BITS);
  int jt[DQ_TPB];
  int64_t tx[DQ_TPB], ty[DQ_TPB];
  T64Codes<BITS> c[DQ_TPB];
#pragma unroll
  for (int u = 0; u < DQ_TPB; ++u) {
    const int64_t g = static_cast<int64_t>(blockIdx.x) * DQ_TPB + u;
    int j = 0;
    while (j + 1 < J.n && g >= J.first[j + 1]) ++j;
    jt[u] = g < J.first[J.n] ? j : -1;
    const int64_t t = g - J.first[j], ncol = J.cols[j] / 64;
    tx[u] = t % ncol;
    ty[u] = t / ncol;
    if (jt[u] >= 0) c[u] = dequant_t64_load<BITS>(J.codes[j], J.ldc[j], tx[u], ty[u]);
  }
#pragma unroll
  for (int u = 0; u < DQ_TPB; ++u) {
    if (jt[u] < 0) break;  // block-uniform
    if (u > 0) __syncthreads();  // the previous tile's shared-memory reads are done
    const int j = jt[u];
    dequant_t64_store<BITS>(c[u], J.scale[j], J.offset[j], J.out[j], J.ld_out[j], nullptr, tx[u], ty[u], sh, nullptr);
  }
}

__global__ void __launch_bounds__(256) k_unpack_pad(const uint8_t* __restrict__ codes, int64_t ldc, int64_t rows,
                                                    int64_t cols, int bits, uint8_t* __restrict__ out,
                                                    int64_t ld_out) {
  const int64_t row = blockIdx.y;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < ld_out;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    out[row * ld_out + k] = k < cols ? static_cast<uint8_t>(unpack_code(codes + row * ldc, k, bits)) : 0;
  }
}

// 4-bit codes -> one byte per code for the int8 GEMM operand, 16 codes per thread: 8 packed bytes in
// (low nibble = even column, quant.py:37-52), 16 bytes out; padding [cols, ld_out) written as 0.
__global__ void __launch_bounds__(256) k_unpack4_v16(const uint8_t* __restrict__ codes, int64_t ldc, int64_t cols,
                                                     uint8_t* __restrict__ out, int64_t ld_out) {
  const int64_t row = blockIdx.y;
  const int64_t nch = ld_out / 16, nin = cols / 16;
  for (int64_t c = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; c < nch;
       c += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    uint4 o = make_uint4(0u, 0u, 0u, 0u);
    if (c < nin) {
      const uint2 w = __ldg(reinterpret_cast<const uint2*>(codes + row * ldc) + c);
      const uint32_t lo0 = w.x & 0x0F0F0F0Fu, hi0 = (w.x >> 4) & 0x0F0F0F0Fu;
      const uint32_t lo1 = w.y & 0x0F0F0F0Fu, hi1 = (w.y >> 4) & 0x0F0F0F0Fu;
      o = make_uint4(__byte_perm(lo0, hi0, 0x5140), __byte_perm(lo0, hi0, 0x7362), __byte_perm(lo1, hi1, 0x5140),
                     __byte_perm(lo1, hi1, 0x7362));
    }
    reinterpret_cast<uint4*>(out + row * ld_out)[c] = o;
  }
}

template <typename InT>
__global__ void __launch_bounds__(256) k_to_bf16_pad(const InT* __restrict__ in, int64_t rows, int64_t cols,
                                                     __nv_bfloat16* __restrict__ out, int64_t ld_out,
                                                     __nv_bfloat16* __restrict__ out_lo) {
  const int64_t row = blockIdx.y;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < ld_out;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const float v = k < cols ? to_f32(in[row * cols + k]) : 0.f;
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    out[row * ld_out + k] = hi;
    if (out_lo != nullptr) out_lo[row * ld_out + k] = __float2bfloat16_rn(v - __bfloat162float(hi));
  }
}

}  // namespace

cudaError_t launch_quantize_rows(const void* w, int w_dtype, int64_t rows, int64_t cols, int64_t ld_w, int bits,
                                 uint8_t* codes, int64_t ld_codes, int64_t pad_cols, float* scale, float* offset,
                                 int32_t* rowsum, int32_t* flag, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  const size_t in_bytes = w_dtype == QA_F32 ? 4 : 2;
  LaunchScope scope(kQuantize, double(rows) * cols * in_bytes + double(rows) * ld_codes + 12.0 * rows, s);
  count_launches(1);
  const int warps = 8;
  const dim3 grid(static_cast<unsigned>((rows + warps - 1) / warps));
  const size_t esz = w_dtype == QA_F32 ? 4 : 2;
  const bool vec_in = (reinterpret_cast<uintptr_t>(w) % 16 == 0) && ((ld_w * esz) % 16 == 0);
  const bool vec_out = bits == 8 ? ((reinterpret_cast<uintptr_t>(codes) % 8 == 0) && (ld_codes % 8 == 0))
                                 : ((reinterpret_cast<uintptr_t>(codes) % 4 == 0) && (ld_codes % 4 == 0));
  const int vec_ok = vec_in && vec_out;
  // production path: one CTA per row, the row in registers (cols a multiple of 8, up to 32768): the (threads,
  // chunks per thread) shape that covers the row with the fewest idle chunk slots, fewer threads on a tie
  // (K = 11008 takes 256 x 6 instead of 128 x 16: 1.9 -> 3.5 TB/s; K = 8192 256 x 4 instead of 128 x 8, the
  // 70B int4 gate 3.5 -> 4.4 TB/s)
  static constexpr int kShapes[][2] = {{128, 1}, {128, 2}, {128, 4}, {256, 4}, {256, 6}, {256, 8}, {512, 6}, {512, 8}};
  const int64_t nchunk = cols / 8;
  int pick = -1;
  if (vec_ok && cols % 8 == 0)
    for (int i = 0; i < 8; ++i) {
      const int64_t cap = int64_t(kShapes[i][0]) * kShapes[i][1];
      if (cap < nchunk) continue;
      if (pick < 0 || cap < int64_t(kShapes[pick][0]) * kShapes[pick][1]) pick = i;
    }
  if (pick >= 0) {
#define QA_QR(TI, BB, CC, TH)                                                                                     \
  k_quantize_rows_reg<TI, BB, CC, TH><<<static_cast<unsigned>(rows), TH, 0, s>>>(                                  \
      static_cast<const TI*>(w), cols, ld_w, codes, ld_codes, pad_cols, scale, offset, rowsum, flag)
#define QA_QR_C(TI, BB)                          \
  switch (pick) {                                \
    case 0: QA_QR(TI, BB, 1, 128); break;        \
    case 1: QA_QR(TI, BB, 2, 128); break;        \
    case 2: QA_QR(TI, BB, 4, 128); break;        \
    case 3: QA_QR(TI, BB, 4, 256); break;        \
    case 4: QA_QR(TI, BB, 6, 256); break;        \
    case 5: QA_QR(TI, BB, 8, 256); break;        \
    case 6: QA_QR(TI, BB, 6, 512); break;        \
    default: QA_QR(TI, BB, 8, 512); break;       \
  }
    if (w_dtype == QA_F32) {
      if (bits == 8) {
        QA_QR_C(float, 8)
      } else {
        QA_QR_C(float, 4)
      }
    } else {
      if (bits == 8) {
        QA_QR_C(__nv_bfloat16, 8)
      } else {
        QA_QR_C(__nv_bfloat16, 4)
      }
    }
#undef QA_QR_C
#undef QA_QR
    return cudaGetLastError();
  }
  if (w_dtype == QA_F32) {
    if (bits == 8)
      k_quantize_rows<float, 8><<<grid, warps * 32, 0, s>>>(static_cast<const float*>(w), rows, cols, ld_w, codes,
                                                            ld_codes, pad_cols, scale, offset, rowsum, flag, vec_ok);
    else
      k_quantize_rows<float, 4><<<grid, warps * 32, 0, s>>>(static_cast<const float*>(w), rows, cols, ld_w, codes,
                                                            ld_codes, pad_cols, scale, offset, rowsum, flag, vec_ok);
  } else {
    if (bits == 8)
      k_quantize_rows<__nv_bfloat16, 8><<<grid, warps * 32, 0, s>>>(static_cast<const __nv_bfloat16*>(w), rows,
                                                                    cols, ld_w, codes, ld_codes, pad_cols, scale,
                                                                    offset, rowsum, flag, vec_ok);
    else
      k_quantize_rows<__nv_bfloat16, 4><<<grid, warps * 32, 0, s>>>(static_cast<const __nv_bfloat16*>(w), rows,
                                                                    cols, ld_w, codes, ld_codes, pad_cols, scale,
                                                                    offset, rowsum, flag, vec_ok);
  }
  return cudaGetLastError();
}

cudaError_t launch_dequantize(const uint8_t* codes, const float* scale, const float* offset, int64_t rows,
                              int64_t cols, int bits, void* out, int out_dtype, int64_t ld_out, bool transpose,
                              cudaStream_t s, __nv_bfloat16* out_lo) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  const int64_t ldc = bits == 8 ? cols : (cols + 1) / 2;
  LaunchScope scope(kDequant, double(rows) * ldc + double(rows) * cols * (out_dtype == QA_F32 ? 4 : 2) * (out_lo ? 2 : 1), s);
  count_launches(1);
  const dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((rows + 31) / 32));
  if (out_dtype == QA_F32) {
    if (transpose)
      k_dequantize<float, true><<<grid, 256, 0, s>>>(codes, ldc, scale, offset, rows, cols, bits,
                                                     static_cast<float*>(out), ld_out, nullptr);
    else
      k_dequantize<float, false><<<grid, 256, 0, s>>>(codes, ldc, scale, offset, rows, cols, bits,
                                                      static_cast<float*>(out), ld_out, nullptr);
  } else {
    const bool fast_t = transpose && rows % 64 == 0 && cols % 64 == 0 && ld_out % 8 == 0 &&
                        reinterpret_cast<uintptr_t>(out) % 16 == 0 &&
                        (out_lo == nullptr || reinterpret_cast<uintptr_t>(out_lo) % 16 == 0) &&
                        reinterpret_cast<uintptr_t>(codes) % 16 == 0 && (ldc % 16 == 0);
    if (fast_t && out_lo == nullptr) {  // the dX GEMM operand: the multi-tile kernel with one job
      DequantJobs J{};
      J.n = 1;
      J.codes[0] = codes;
      J.scale[0] = scale;
      J.offset[0] = offset;
      J.rows[0] = rows;
      J.cols[0] = cols;
      J.ldc[0] = ldc;
      J.ld_out[0] = ld_out;
      J.bits[0] = bits;
      J.out[0] = static_cast<__nv_bfloat16*>(out);
      J.first[0] = 0;
      J.first[1] = (rows / 64) * (cols / 64);
      const int tpb = dq_tpb(bits);
      const unsigned blocks = static_cast<unsigned>((J.first[1] + tpb - 1) / tpb);
      if (bits == 8)
        k_dequant_t64_multi<8><<<blocks, 256, 0, s>>>(J);
      else
        k_dequant_t64_multi<4><<<blocks, 256, 0, s>>>(J);
    } else if (fast_t) {
      const dim3 g64(static_cast<unsigned>(cols / 64), static_cast<unsigned>(rows / 64));
      if (bits == 8)
        k_dequant_t64<8><<<g64, 256, 0, s>>>(codes, ldc, scale, offset, static_cast<__nv_bfloat16*>(out), ld_out,
                                             out_lo);
      else
        k_dequant_t64<4><<<g64, 256, 0, s>>>(codes, ldc, scale, offset, static_cast<__nv_bfloat16*>(out), ld_out,
                                             out_lo);
    } else if (transpose)
      k_dequantize<__nv_bfloat16, true><<<grid, 256, 0, s>>>(codes, ldc, scale, offset, rows, cols, bits,
                                                             static_cast<__nv_bfloat16*>(out), ld_out, out_lo);
    else
      k_dequantize<__nv_bfloat16, false><<<grid, 256, 0, s>>>(codes, ldc, scale, offset, rows, cols, bits,
                                                              static_cast<__nv_bfloat16*>(out), ld_out, out_lo);
  }
  return cudaGetLastError();
}

cudaError_t launch_dequantize_t_multi(int n, const DequantJobs& jobs_in, cudaStream_t s) {
  DequantJobs J = jobs_in;
  J.n = n;
  bool fast = n >= 1 && n <= kDqJobs;
  int bits = fast ? J.bits[0] : 8;
  int64_t tiles = 0;
  double bytes = 0.0;
  for (int i = 0; i < n && fast; ++i) {
    fast = J.bits[i] == bits && J.rows[i] % 64 == 0 && J.cols[i] % 64 == 0 && J.ld_out[i] % 8 == 0 &&
           reinterpret_cast<uintptr_t>(J.out[i]) % 16 == 0 && reinterpret_cast<uintptr_t>(J.codes[i]) % 16 == 0 &&
           J.ldc[i] % 16 == 0;
    J.first[i] = tiles;
    tiles += (J.rows[i] / 64) * (J.cols[i] / 64);
    bytes += double(J.rows[i]) * J.ldc[i] + 2.0 * double(J.rows[i]) * J.cols[i];
  }
  if (!fast) {  // member by member (the general kernels)
    for (int i = 0; i < n; ++i) {
      cudaError_t e = launch_dequantize(J.codes[i], J.scale[i], J.offset[i], J.rows[i], J.cols[i], J.bits[i], J.out[i],
                                        QA_BF16, J.ld_out[i], true, s);
      if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
  }
  if (tiles == 0) return cudaSuccess;
  J.first[n] = tiles;
  LaunchScope scope(kDequant, bytes, s);
  count_launches(1);
  const unsigned blocks = static_cast<unsigned>((tiles + dq_tpb(bits) - 1) / dq_tpb(bits));
  if (bits == 8)
    k_dequant_t64_multi<8><<<blocks, 256, 0, s>>>(J);
  else
    k_dequant_t64_multi<4><<<blocks, 256, 0, s>>>(J);
  return cudaGetLastError();
}

cudaError_t launch_unpack_pad(const uint8_t* codes, int64_t rows, int64_t cols, int bits, uint8_t* out,
                              int64_t ld_out, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  const int64_t ldc = bits == 8 ? cols : (cols + 1) / 2;
  LaunchScope scope(kDequant, double(rows) * (ldc + ld_out), s);
  count_launches(1);
  if (bits == 4 && cols % 16 == 0 && ld_out % 16 == 0 && reinterpret_cast<uintptr_t>(codes) % 8 == 0 &&
      reinterpret_cast<uintptr_t>(out) % 16 == 0) {
    const dim3 g16(static_cast<unsigned>((ld_out / 16 + 255) / 256), static_cast<unsigned>(rows));
    k_unpack4_v16<<<g16, 256, 0, s>>>(codes, ldc, cols, out, ld_out);
    return cudaGetLastError();
  }
  const dim3 grid(static_cast<unsigned>(std::min<int64_t>((ld_out + 255) / 256, 64)), static_cast<unsigned>(rows));
  k_unpack_pad<<<grid, 256, 0, s>>>(codes, ldc, rows, cols, bits, out, ld_out);
  return cudaGetLastError();
}

// Σ codes per row of a stored code grid (reference layout; 4-bit: low nibble = even column), for
// bases whose codes arrive from a checkpoint rather than from qa_quantize_rows.
__global__ void __launch_bounds__(256) k_code_rowsum(const uint8_t* __restrict__ codes, int64_t rows, int64_t cols,
                                                     int bits, int32_t* __restrict__ rowsum) {
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  if (row >= rows) return;
  const int lane = threadIdx.x & 31;
  const int64_t ldc = bits == 8 ? cols : (cols + 1) / 2;
  const uint8_t* r = codes + row * ldc;
  int32_t sum = 0;
  for (int64_t c = lane; c < ldc; c += 32) {
    const uint32_t b = r[c];
    sum += bits == 8 ? static_cast<int32_t>(b) : static_cast<int32_t>((b & 0xFu) + (2 * c + 1 < cols ? (b >> 4) : 0u));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) rowsum[row] = sum;
}

cudaError_t launch_code_rowsum(const uint8_t* codes, int64_t rows, int64_t cols, int bits, int32_t* rowsum,
                               cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  LaunchScope scope(kQuantize, double(rows) * (bits == 8 ? cols : (cols + 1) / 2) + 4.0 * rows, s);
  count_launches(1);
  k_code_rowsum<<<static_cast<unsigned>((rows + 7) / 8), 256, 0, s>>>(codes, rows, cols, bits, rowsum);
  return cudaGetLastError();
}

cudaError_t launch_to_bf16_pad(const void* in, int in_dtype, int64_t rows, int64_t cols, __nv_bfloat16* out,
                               int64_t ld_out, cudaStream_t s, __nv_bfloat16* out_lo) {
  if (rows == 0) return cudaSuccess;
  LaunchScope scope(kDequant, double(rows) * cols * (in_dtype == QA_F32 ? 4 : 2) + double(rows) * ld_out * (out_lo ? 4 : 2), s);
  count_launches(1);
  const dim3 grid(static_cast<unsigned>(std::min<int64_t>((ld_out + 255) / 256, 64)), static_cast<unsigned>(rows));
  if (in_dtype == QA_F32)
    k_to_bf16_pad<float><<<grid, 256, 0, s>>>(static_cast<const float*>(in), rows, cols, out, ld_out, out_lo);
  else
    k_to_bf16_pad<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(in), rows, cols, out,
                                                      ld_out, out_lo);
  return cudaGetLastError();
}

}  // namespace qa

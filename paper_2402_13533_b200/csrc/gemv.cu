// Decode-size forward (1..8 tokens, KV-cached decoding, transformer.py:1043-1080): the int8 product is a
// matrix-vector pass over the stored codes, so it is HBM-bound on the weight bytes, not tensor-bound.
// One warp per output row at a time: lanes stream 16-byte code chunks of the row (512 B per warp
// load), multiply them against the tokens' activation codes with dp4a (u8 x u8 -> exact int32),
// reduce across the warp, and apply the same exact-int32 centring + fp32 dequant epilogue as the
// tcgen05 GEMM (gemm_tc.cu), plus the adapter term y2 = Z1 · Vᵀ from the fp32 Z1 and the hi + lo V split.
#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_timing.h"

namespace qa {

namespace {

constexpr int GV_WARPS = 8, GV_RPW = 2, GV_UNR = 4;  // warps per CTA, rows per warp, chunks in flight per row

template <int M, int BITS>
__global__ void __launch_bounds__(GV_WARPS * 32) k_gemv(const uint8_t* __restrict__ xc, int64_t ldx, int T,
                                                        const float* __restrict__ sx, const float* __restrict__ ox,
                                                        const int32_t* __restrict__ rsx,
                                                        const uint8_t* __restrict__ wc, int64_t N, int64_t K,
                                                        const float* __restrict__ ws, const float* __restrict__ wo,
                                                        const int32_t* __restrict__ wrs,
                                                        const float* __restrict__ zl, int64_t ldz,
                                                        const float* __restrict__ Gl, int64_t Ml, int Cl,
                                                        const float* __restrict__ addend,
                                                        __nv_bfloat16* __restrict__ out, float* __restrict__ out32) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ldw = BITS == 8 ? K : K / 2;
  const int64_t nchunk = ldw / 16;  // 16-byte code chunks per row (16 codes at 8 bits, 32 at 4)
  const int64_t row0 = (static_cast<int64_t>(blockIdx.x) * GV_WARPS + warp) * GV_RPW;
  uint32_t acc[GV_RPW][M];  // u8 x u8 sums: exact below 2^31 for K <= 33025
#pragma unroll
  for (int r = 0; r < GV_RPW; ++r)
#pragma unroll
    for (int t = 0; t < M; ++t) acc[r][t] = 0u;
  for (int64_t q0 = lane; q0 < nchunk; q0 += 32 * GV_UNR) {
    uint4 wu[GV_UNR][GV_RPW];
#pragma unroll
    for (int u = 0; u < GV_UNR; ++u)
#pragma unroll
      for (int r = 0; r < GV_RPW; ++r)
        wu[u][r] = (row0 + r < N && q0 + 32 * u < nchunk)
                       ? __ldg(reinterpret_cast<const uint4*>(wc + (row0 + r) * ldw) + q0 + 32 * u)
                       : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int u = 0; u < GV_UNR; ++u) {
    const int64_t q = q0 + 32 * u;
    if (q >= nchunk) break;
    const uint4(&w)[GV_RPW] = wu[u];
#pragma unroll
    for (int t = 0; t < M; ++t) {
      if (t >= T) break;
      if constexpr (BITS == 8) {
        const uint4 x = __ldg(reinterpret_cast<const uint4*>(xc + t * ldx) + q);
#pragma unroll
        for (int r = 0; r < GV_RPW; ++r) {
          uint32_t a = acc[r][t];
          a = __dp4a(w[r].x, x.x, a);
          a = __dp4a(w[r].y, x.y, a);
          a = __dp4a(w[r].z, x.z, a);
          a = __dp4a(w[r].w, x.w, a);
          acc[r][t] = a;
        }
      } else {
        // 32 codes: byte j of the chunk holds columns 2j (low nibble) and 2j + 1 (high nibble)
        const uint4 x0 = __ldg(reinterpret_cast<const uint4*>(xc + t * ldx) + 2 * q);
        const uint4 x1 = __ldg(reinterpret_cast<const uint4*>(xc + t * ldx) + 2 * q + 1);
        const uint32_t xw[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
        uint32_t xe[4], xo[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          xe[k] = __byte_perm(xw[2 * k], xw[2 * k + 1], 0x6420);
          xo[k] = __byte_perm(xw[2 * k], xw[2 * k + 1], 0x7531);
        }
#pragma unroll
        for (int r = 0; r < GV_RPW; ++r) {
          const uint32_t ww[4] = {w[r].x, w[r].y, w[r].z, w[r].w};
          uint32_t a = acc[r][t];
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            a = __dp4a(ww[k] & 0x0F0F0F0Fu, xe[k], a);
            a = __dp4a((ww[k] >> 4) & 0x0F0F0F0Fu, xo[k], a);
          }
          acc[r][t] = a;
        }
      }
    }
    }
  }
  // adapter: y2[t, n] = Σ_b Zlast[t, h, b] Glast[b, i], n = h Ml + i (the last TT core, rank Cl <= 32)
  float y2[GV_RPW][M];
#pragma unroll
  for (int r = 0; r < GV_RPW; ++r)
#pragma unroll
    for (int t = 0; t < M; ++t) y2[r][t] = 0.f;
  if (Gl != nullptr && lane < Cl) {
#pragma unroll
    for (int r = 0; r < GV_RPW; ++r) {
      const int64_t n = row0 + r;
      if (n >= N) break;
      const int64_t h = n / Ml, i = n - h * Ml;
      const float g = __ldg(Gl + lane * Ml + i);
#pragma unroll
      for (int t = 0; t < M; ++t)
        if (t < T) y2[r][t] = __ldg(zl + t * ldz + h * Cl + lane) * g;
    }
  }
#pragma unroll
  for (int r = 0; r < GV_RPW; ++r)
#pragma unroll
    for (int t = 0; t < M; ++t)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc[r][t] += __shfl_xor_sync(0xffffffffu, acc[r][t], o);
        y2[r][t] += __shfl_xor_sync(0xffffffffu, y2[r][t], o);
      }
  // epilogue (lane t writes token t of each row): the GEMM's exact int32 centring + fp32 dequant
  const int zp_row = 128, zp_col = BITS == 8 ? 128 : 8;
  const int kr = static_cast<int>(K);
#pragma unroll
  for (int r = 0; r < GV_RPW; ++r) {
    const int64_t n = row0 + r;
    if (n >= N) break;
#pragma unroll
    for (int t = 0; t < M; ++t) {
      if (lane != t || t >= T) continue;
      const float sw = ws[n];
      const float owt = wo[n] + static_cast<float>(zp_col) * sw;
      const int32_t rs = wrs[n];
      const float colC = fmaf(sw, static_cast<float>(rs - zp_col * kr), static_cast<float>(kr) * owt);
      const int32_t colD = zp_row * rs;
      const float s = sx[t];
      const float oxt = ox[t] + static_cast<float>(zp_row) * s;
      const int32_t rx = rsx[t];
      const float rsxc = static_cast<float>(rx - zp_row * kr);
      const int32_t ibase = zp_row * zp_col * kr - zp_col * rx;
      const int32_t accc = static_cast<int32_t>(acc[r][t]) + ibase - colD;
      float y = fmaf(s, fmaf(sw, static_cast<float>(accc), owt * rsxc), oxt * colC);
      y += y2[r][t];
      if (addend != nullptr) y += addend[t * N + n];
      if (out32 != nullptr) out32[t * N + n] = y;
      if (out != nullptr) out[t * N + n] = __float2bfloat16_rn(y);
    }
  }
}

}  // namespace

bool gemv_ok(int64_t T, int64_t K, int bits) {
  static const bool off = [] {
    const char* v = getenv("QA_GEMV");
    return v != nullptr && v[0] == '0';
  }();
  return !off && T >= 1 && T <= 8 && (bits == 8 ? K % 16 == 0 : K % 32 == 0);
}

cudaError_t launch_gemv(const uint8_t* xc, int64_t ldx, int64_t T, const float* sx, const float* ox,
                        const int32_t* rsx, const uint8_t* wc, int64_t N, int64_t K, int bits, const float* ws,
                        const float* wo, const int32_t* wrs, const float* zl, int64_t ldz, const float* Gl,
                        int64_t Ml, int Cl, const float* addend, __nv_bfloat16* out, float* out32, cudaStream_t s) {
  if (T == 0 || N == 0) return cudaSuccess;
  LaunchScope scope(kGemmI8, 2.0 * double(T) * N * K, s);
  count_launches(1);
  const unsigned grid = static_cast<unsigned>((N + GV_WARPS * GV_RPW - 1) / (GV_WARPS * GV_RPW));
#define QA_GV(MM)                                                                                                   \
  {                                                                                                                 \
    if (bits == 8)                                                                                                  \
      k_gemv<MM, 8><<<grid, GV_WARPS * 32, 0, s>>>(xc, ldx, static_cast<int>(T), sx, ox, rsx, wc, N, K, ws, wo, wrs, \
                                                   zl, ldz, Gl, Ml, Cl, addend, out, out32);                        \
    else                                                                                                            \
      k_gemv<MM, 4><<<grid, GV_WARPS * 32, 0, s>>>(xc, ldx, static_cast<int>(T), sx, ox, rsx, wc, N, K, ws, wo, wrs, \
                                                   zl, ldz, Gl, Ml, Cl, addend, out, out32);                        \
  }
  if (T == 1)
    QA_GV(1)
  else if (T == 2)
    QA_GV(2)
  else if (T <= 4)
    QA_GV(4)
  else
    QA_GV(8)
#undef QA_GV
  return cudaGetLastError();
}

}  // namespace qa

// Generic tensor-train modes on the tensor cores (any d <= 4, any modes / ranks): the adapter runs through the
// materialised W_t = G1 ··· Gd instead of the left-to-right stage chain on CUDA cores.
//
//   forward  : y2 = x · W_tᵀ as extension k-blocks of the int8 GEMM, A2 = [x_hi | x_lo | x_hi],
//              B2 = [W_hi | W_hi | W_lo] (bf16 planes; the three products give an fp32-class y2, folded in TMEM)
//   backward : dx_adapter = dy · W_t as extension k-blocks of the dX GEMM (A2 = dy planes, B2 = W_tᵀ planes);
//              dW_t = dyᵀ · x on tcgen05 (kind::f16, fp32 accumulate, T as the reduction), then each core's
//              gradient is the projection of dW_t onto it (k_proj_right / k_proj_left):
//                dG_k[a, ik, j, b] = Σ L_k[I, J, a] · dW[(I, ik, I'), (J, j, J')] · R_k[b, I', J']
//              with L_k the contraction of cores 0..k-1 and R_k of cores k+1..d-1.
// The W_t-side work is O(N·K·r) per call, independent of the token count; every token-side product runs on the
// tensor cores.  Balanced modes (BASELINE config 1's (4,16,16)²) cost more flops than dense at 1024² (SURVEY
// §8(d)), so the dense route is also the cheaper one there.
#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_timing.h"

namespace qa {

namespace {

template <typename T>
QA_DEV float ld_val(const T* p) {
  return to_f32(*p);
}

// Three bf16 planes of a [rows, cols] matrix side by side in out [rows, ld_out]: plane p holds term
// order[p] (0 = hi, 1 = lo) of every element, columns [cols, plane_w) and [3 plane_w, ld_out) zero.
template <typename InT>
__global__ void __launch_bounds__(256) k_split3_rows(const InT* __restrict__ in, int64_t rows, int64_t cols,
                                                     int64_t ldin, __nv_bfloat16* __restrict__ out, int64_t ld_out,
                                                     int64_t plane_w, int order) {
  const int64_t total = rows * ld_out;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = i / ld_out, c = i - r * ld_out;
    const int64_t p = c / plane_w, cc = c - p * plane_w;
    float v = 0.f;
    if (p < 3 && cc < cols) {
      const float x = ld_val(in + r * ldin + cc);
      const __nv_bfloat16 hi = __float2bfloat16_rn(x);
      v = ((order >> p) & 1) ? x - __bfloat162float(hi) : __bfloat162float(hi);
    }
    out[i] = __float2bfloat16_rn(v);
  }
}

// The same planes of the TRANSPOSE: out [cols, ld_out], plane p of row c = term order[p] of in[:, c]; 32 x 32
// tiles through shared memory (coalesced on both sides).
template <typename InT>
__global__ void __launch_bounds__(256) k_split3_t(const InT* __restrict__ in, int64_t rows, int64_t cols,
                                                  int64_t ldin, __nv_bfloat16* __restrict__ out, int64_t ld_out,
                                                  int64_t plane_w, int order) {
  __shared__ float tile[32][33];
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * 32, c0 = static_cast<int64_t>(blockIdx.x) * 32;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int i = ty; i < 32; i += 8) {
    const int64_t r = r0 + i, c = c0 + tx;
    tile[i][tx] = (r < rows && c < cols) ? ld_val(in + r * ldin + c) : 0.f;
  }
  __syncthreads();
  for (int i = ty; i < 32; i += 8) {
    const int64_t c = c0 + i, r = r0 + tx;  // output row c, column r (+ plane offset)
    if (c >= cols || r >= plane_w) continue;
    const float x = tile[tx][i];
    const __nv_bfloat16 hi = __float2bfloat16_rn(x);
    const float lo = x - __bfloat162float(hi);
#pragma unroll
    for (int p = 0; p < 3; ++p)
      out[c * ld_out + p * plane_w + r] = __float2bfloat16_rn(((order >> p) & 1) ? lo : __bfloat162float(hi));
  }
}

// out[r, c] = 0 for the padding of a plane layout the tiles above do not reach
__global__ void __launch_bounds__(256) k_zero_bf16(__nv_bfloat16* __restrict__ p, int64_t n) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    p[i] = __float2bfloat16_rn(0.f);
}

struct Cores {
  const float* p[QA_TT_MAX_D];
};

// R_k[b, I', J'] = G_{k+1}[b, i, j, :] ··· G_{d-1}[:, i, j, 0] over I' = (i_{k+1}..i_{d-1}), J' likewise; one
// thread per (I', J'), the rank vector contracted right to left (ranks <= 64).
__global__ void __launch_bounds__(128) k_suffix(TTDims dd, Cores cores, int k, float* __restrict__ R, int64_t SM,
                                                int64_t SN) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= SM * SN) return;
  const int64_t Ip = idx / SN, Jp = idx - Ip * SN;
  int iv[QA_TT_MAX_D], jv[QA_TT_MAX_D];
  int64_t ir = Ip, jr = Jp;
  for (int q = dd.d - 1; q > k; --q) {
    iv[q] = static_cast<int>(ir % dd.m[q]);
    ir /= dd.m[q];
    jv[q] = static_cast<int>(jr % dd.n[q]);
    jr /= dd.n[q];
  }
  constexpr int kMaxR = 64;
  float v[kMaxR], w[kMaxR];
  v[0] = 1.f;
  int rb = 1;  // right rank of the running vector
  for (int q = dd.d - 1; q > k; --q) {
    const int ra = dd.r[q];
    const float* g = cores.p[q];
    for (int a = 0; a < ra; ++a) {
      float s = 0.f;
      for (int b = 0; b < rb; ++b)
        s = fmaf(g[((static_cast<int64_t>(a) * dd.m[q] + iv[q]) * dd.n[q] + jv[q]) * rb + b], v[b], s);
      w[a] = s;
    }
    for (int a = 0; a < ra; ++a) v[a] = w[a];
    rb = ra;
  }
  const int rk = dd.r[k + 1];
  for (int b = 0; b < rk; ++b) R[(static_cast<int64_t>(b) * SM + Ip) * SN + Jp] = v[b];
}

// Y[I, ik, J, j, b] = Σ_{I', J'} dW[(I, ik, I'), (J, j, J')] · R[b, I', J']   (one warp per (I, ik, J, j))
template <int RB>
__global__ void __launch_bounds__(256) k_proj_right(const float* __restrict__ dW, int64_t K, int64_t OUT_ROWS,
                                                    int64_t OUT_COLS, int64_t SM, int64_t SN,
                                                    const float* __restrict__ R, int rb, float* __restrict__ Y) {
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= OUT_ROWS * OUT_COLS) return;
  const int64_t orow = wid / OUT_COLS, ocol = wid - orow * OUT_COLS;  // (I, ik) and (J, j)
  float acc[RB];
#pragma unroll
  for (int b = 0; b < RB; ++b) acc[b] = 0.f;
  for (int64_t e = lane; e < SM * SN; e += 32) {
    const int64_t Ip = e / SN, Jp = e - Ip * SN;
    const float w = dW[(orow * SM + Ip) * K + ocol * SN + Jp];
#pragma unroll
    for (int b = 0; b < RB; ++b)
      if (b < rb) acc[b] = fmaf(w, R[(static_cast<int64_t>(b) * SM + Ip) * SN + Jp], acc[b]);
  }
#pragma unroll
  for (int b = 0; b < RB; ++b) {
    float v = acc[b];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0 && b < rb) Y[wid * rb + b] = v;
  }
}

// The same for long inner sums over few outputs (e.g. the first core): CTAs (o, s) split output o's sum into
// gridDim.y slices, each writing its partial to Y plane s (summed in fixed order by k_proj_left)
template <int RB>
__global__ void __launch_bounds__(256) k_proj_right_cta(const float* __restrict__ dW, int64_t K, int64_t OUT_COLS,
                                                        int64_t SM, int64_t SN, const float* __restrict__ R, int rb,
                                                        float* __restrict__ Y, int64_t plane) {
  __shared__ float red[8][RB];
  const int64_t o = blockIdx.x;
  const int64_t orow = o / OUT_COLS, ocol = o - orow * OUT_COLS;
  const int64_t total = SM * SN, per = (total + gridDim.y - 1) / gridDim.y;
  const int64_t e0 = blockIdx.y * per, e1 = e0 + per < total ? e0 + per : total;
  float acc[RB];
#pragma unroll
  for (int b = 0; b < RB; ++b) acc[b] = 0.f;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += 256) {
    const int64_t Ip = e / SN, Jp = e - Ip * SN;
    const float w = dW[(orow * SM + Ip) * K + ocol * SN + Jp];
#pragma unroll
    for (int b = 0; b < RB; ++b)
      if (b < rb) acc[b] = fmaf(w, R[(static_cast<int64_t>(b) * SM + Ip) * SN + Jp], acc[b]);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int b = 0; b < RB; ++b) {
    float v = acc[b];
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if (lane == 0) red[warp][b] = v;
  }
  __syncthreads();
  if (threadIdx.x < rb) {
    float v = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += red[w][threadIdx.x];
    Y[blockIdx.y * plane + o * rb + threadIdx.x] = v;
  }
}

// dG[a, ik, j, b] (+)= Σ_{I, J} L[I, J, a] · Y[I, ik, J, j, b]   (one warp per output element; Y may come as
// nplanes partial planes, summed first in fixed order)
__global__ void __launch_bounds__(256) k_proj_left(const float* __restrict__ Y, const float* __restrict__ L, int64_t PM,
                                                   int64_t PN, int ra, int mk, int nk, int rb, float* __restrict__ dG,
                                                   int accumulate, int nplanes, int64_t plane) {
  const int64_t wid = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t total = static_cast<int64_t>(ra) * mk * nk * rb;
  if (wid >= total) return;
  const int b = static_cast<int>(wid % rb);
  const int j = static_cast<int>((wid / rb) % nk);
  const int ik = static_cast<int>((wid / (static_cast<int64_t>(rb) * nk)) % mk);
  const int a = static_cast<int>(wid / (static_cast<int64_t>(rb) * nk * mk));
  float acc = 0.f;
  for (int64_t e = lane; e < PM * PN; e += 32) {
    const int64_t I = e / PN, J = e - I * PN;
    const float l = L != nullptr ? L[(I * PN + J) * ra + a] : 1.f;
    // Y index: ((I * mk + ik) * (PN * nk) + J * nk + j) * rb + b
    const int64_t yi = (((I * mk + ik) * PN + J) * nk + j) * rb + b;
    float y = Y[yi];
    for (int p = 1; p < nplanes; ++p) y += Y[p * plane + yi];
    acc = fmaf(l, y, acc);
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane == 0) dG[wid] = accumulate ? dG[wid] + acc : acc;
}

constexpr int kProjMaxPlanes = 64;  // partial Y planes of a split projection

// Slices of a projection's inner sum: long sums (SM·SN >= 2048 terms) over few outputs are split so that ~4 CTAs
// per SM run, each slice >= 1024 terms; the rest run unsplit (one warp per output).
int proj_planes(int64_t outs, int64_t terms) {
  if (terms < 2048) return 1;
  int64_t sl = (4 * 148 + outs - 1) / outs;
  const int64_t by_len = (terms + 1023) / 1024;
  if (sl > by_len) sl = by_len;
  return static_cast<int>(sl < 1 ? 1 : (sl > kProjMaxPlanes ? kProjMaxPlanes : sl));
}

unsigned blocks_for(int64_t work, int threads) {
  const int64_t b = (work + threads - 1) / threads;
  return static_cast<unsigned>(b < 1 ? 1 : (b < 148 * 32 ? b : 148 * 32));
}

}  // namespace

cudaError_t launch_split3_rows(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t ldin,
                               __nv_bfloat16* out, int64_t ld_out, int64_t plane_w, int order, cudaStream_t s) {
  if (rows == 0) return cudaSuccess;
  LaunchScope scope(kTT, double(rows) * cols * (in_dtype == QA_F32 ? 4 : 2) + 2.0 * rows * ld_out, s);
  count_launches(1);
  const unsigned g = blocks_for(rows * ld_out, 256);
  if (in_dtype == QA_F32)
    k_split3_rows<float><<<g, 256, 0, s>>>(static_cast<const float*>(in), rows, cols, ldin, out, ld_out, plane_w, order);
  else
    k_split3_rows<__nv_bfloat16><<<g, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(in), rows, cols, ldin, out, ld_out,
                                                   plane_w, order);
  return cudaGetLastError();
}

cudaError_t launch_split3_t(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t ldin,
                            __nv_bfloat16* out, int64_t ld_out, int64_t plane_w, int order, cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  LaunchScope scope(kTT, double(rows) * cols * (in_dtype == QA_F32 ? 4 : 2) + 2.0 * cols * ld_out, s);
  count_launches(2);
  k_zero_bf16<<<blocks_for(cols * ld_out, 256), 256, 0, s>>>(out, cols * ld_out);
  const dim3 grid(static_cast<unsigned>((cols + 31) / 32), static_cast<unsigned>((plane_w + 31) / 32));
  if (in_dtype == QA_F32)
    k_split3_t<float><<<grid, 256, 0, s>>>(static_cast<const float*>(in), rows, cols, ldin, out, ld_out, plane_w, order);
  else
    k_split3_t<__nv_bfloat16><<<grid, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(in), rows, cols, ldin, out, ld_out,
                                                    plane_w, order);
  return cudaGetLastError();
}

size_t tt_project_ws_floats(const TTDims& dd) {
  // max over k of L_k + R_k + Y_k
  size_t best = 0;
  for (int k = 0; k < dd.d; ++k) {
    int64_t PM = 1, PN = 1, SM = 1, SN = 1;
    for (int q = 0; q < k; ++q) {
      PM *= dd.m[q];
      PN *= dd.n[q];
    }
    for (int q = k + 1; q < dd.d; ++q) {
      SM *= dd.m[q];
      SN *= dd.n[q];
    }
    const size_t L = static_cast<size_t>(PM * PN * dd.r[k]);
    const size_t R = static_cast<size_t>(SM * SN * dd.r[k + 1]);
    const int64_t outs = PM * dd.m[k] * PN * dd.n[k];
    const size_t Y = static_cast<size_t>(outs) * dd.r[k + 1] * (k + 1 < dd.d ? proj_planes(outs, SM * SN) : 1);
    const size_t tot = L + R + Y + 3 * 64;
    if (tot > best) best = tot;
  }
  return best;
}

cudaError_t launch_tt_project(const TTDims& dd, const float* const* cores, const float* dW, float* ws,
                              float* const* dcores, bool accumulate, cudaStream_t s) {
  Cores cp{};
  for (int q = 0; q < dd.d; ++q) cp.p[q] = cores[q];
  for (int k = 0; k < dd.d; ++k) {
    if (dcores == nullptr || dcores[k] == nullptr) continue;
    int64_t PM = 1, PN = 1, SM = 1, SN = 1;
    for (int q = 0; q < k; ++q) {
      PM *= dd.m[q];
      PN *= dd.n[q];
    }
    for (int q = k + 1; q < dd.d; ++q) {
      SM *= dd.m[q];
      SN *= dd.n[q];
    }
    const int ra = dd.r[k], rb = dd.r[k + 1], mk = dd.m[k], nk = dd.n[k];
    float* L = ws;
    float* R = L + ((PM * PN * ra + 63) / 64) * 64;
    float* Y = R + ((SM * SN * rb + 63) / 64) * 64;
    LaunchScope scope(kTT, 4.0 * double(dd.N) * double(dd.K) * (1 + rb), s);
    if (k > 0) {  // L_k: the prefix contraction of cores 0..k-1 (open rank r[k])
      TTDims dk = dd;
      dk.d = k + 1;
      cudaError_t e = launch_tt_prefix_full(dk, cores, L, s);
      if (e != cudaSuccess) return e;
    }
    count_launches(2);
    if (k + 1 < dd.d)  // R_k: the contraction of cores k+1..d-1 (R_{d-1} = 1)
      k_suffix<<<static_cast<unsigned>((SM * SN + 127) / 128), 128, 0, s>>>(dd, cp, k, R, SM, SN);
    const float* Rp = R;
    const int64_t outs = (PM * mk) * (PN * nk);
    const unsigned gr = static_cast<unsigned>((outs * 32 + 255) / 256);
    const int64_t plane = outs * rb;
    int nplanes = 1;
    if (k + 1 == dd.d) {
      // Y[I, ik, J, j, 0] = dW[(I, ik), (J, j)] (SM = SN = 1, R = 1)
      cudaError_t e = cudaMemcpyAsync(Y, dW, sizeof(float) * outs, cudaMemcpyDeviceToDevice, s);
      if (e != cudaSuccess) return e;
    } else {
      // long inner sums over few outputs take CTAs (split into proj_planes slices), the rest a warp each
      const bool cta = SM * SN >= 2048;
      nplanes = proj_planes(outs, SM * SN);
      const dim3 gc(static_cast<unsigned>(outs), static_cast<unsigned>(nplanes));
#define QA_PR(RBV)                                                                                   \
  if (cta)                                                                                           \
    k_proj_right_cta<RBV><<<gc, 256, 0, s>>>(dW, dd.K, PN * nk, SM, SN, Rp, rb, Y, plane);           \
  else                                                                                               \
    k_proj_right<RBV><<<gr, 256, 0, s>>>(dW, dd.K, PM * mk, PN * nk, SM, SN, Rp, rb, Y);
      if (rb <= 8) {
        QA_PR(8)
      } else if (rb <= 16) {
        QA_PR(16)
      } else if (rb <= 32) {
        QA_PR(32)
      } else {
        QA_PR(64)
      }
#undef QA_PR
    }
    const int64_t gouts = static_cast<int64_t>(ra) * mk * nk * rb;
    k_proj_left<<<static_cast<unsigned>((gouts * 32 + 255) / 256), 256, 0, s>>>(Y, k > 0 ? L : nullptr, PM, PN, ra, mk,
                                                                                nk, rb, dcores[k], accumulate ? 1 : 0,
                                                                                nplanes, plane);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace qa

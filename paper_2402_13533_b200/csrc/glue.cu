// Decoder-layer glue around the quantised linears (BASELINE config 4): the elementwise and
// row-reduction steps of _layer_forward / _layer_backward (transformer.py:858-946) as single-pass bf16 kernels.
//   rmsnorm (:478-484) with the residual add folded in, its backward (:487-496) with the summed input
//   gradients of a shared-input group and the residual gradient folded in, the rotary rotation (:506-519),
//   SiLU gating (:474-475, :872-874) forward and backward, and the mean cross-entropy loss + gradient
//   (:569-588) of the head's logits.
// All are HBM-bound: every kernel reads its operands once and writes its results once (rows stay in
// registers; the cross-entropy's second pass over a 64 KB logit row hits L2).
#include <cuda_bf16.h>

#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_timing.h"

namespace qa {

namespace {

constexpr int kRowWarps = 8;  // rows per CTA (one warp per row)

__device__ __forceinline__ void unpack8(const uint4& u, float* f) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 p = __bfloat1622float2(h[i]);
    f[2 * i] = p.x;
    f[2 * i + 1] = p.y;
  }
}

__device__ __forceinline__ uint4 pack8(const float* f) {
  uint4 u;
  __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) h[i] = __floats2bfloat162_rn(f[2 * i], f[2 * i + 1]);
  return u;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Sum over the WPR warps that share a row (CTA = 8 warps = 8 / WPR rows); every thread must call it.
template <int WPR>
__device__ __forceinline__ float row_sum(float v, float* red) {
  v = warp_sum(v);
  if constexpr (WPR == 1) {
    return v;
  } else {
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    const int w0 = w - w % WPR;
    float t = 0.f;
#pragma unroll
    for (int i = 0; i < WPR; ++i) t += red[w0 + i];
    return t;
  }
}

// y = bf16((s * inv) * gain), inv = rsqrt(mean(s^2) + eps), s = a (+ b, rounded to bf16 and written to sum).
// Rows of D = 256 * VPL columns, WPR warps per row; thread u of a row owns the 8-column chunks u, u + 32*WPR, ...
template <int VPL, bool ADD, int WPR = 1>
__global__ void __launch_bounds__(kRowWarps * 32) k_rmsnorm_fwd(const __nv_bfloat16* __restrict__ a,
                                                                const __nv_bfloat16* __restrict__ b,
                                                                __nv_bfloat16* __restrict__ sum,
                                                                const float* __restrict__ gain,
                                                                __nv_bfloat16* __restrict__ y, float* __restrict__ inv,
                                                                int64_t rows, float eps) {
  constexpr int D = 256 * VPL, NV = VPL / WPR, STRIDE = 32 * WPR;
  __shared__ float red[kRowWarps];
  const int u = threadIdx.x % STRIDE;
  int64_t row = static_cast<int64_t>(blockIdx.x) * (kRowWarps / WPR) + threadIdx.x / STRIDE;
  const bool live = row < rows;
  if (WPR == 1 && !live) return;
  if (!live) row = rows - 1;  // shares the row reduction's barrier, writes nothing
  const uint4* ar = reinterpret_cast<const uint4*>(a + row * D);
  uint4 v[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) v[i] = __ldg(ar + u + STRIDE * i);
  if constexpr (ADD) {
    const uint4* br = reinterpret_cast<const uint4*>(b + row * D);
    uint4* sr = reinterpret_cast<uint4*>(sum + row * D);
#pragma unroll
    for (int i = 0; i < NV; ++i) {
      const uint4 w = __ldg(br + u + STRIDE * i);
      __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&v[i]);
      const __nv_bfloat162* q = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int j = 0; j < 4; ++j) p[j] = __hadd2(p[j], q[j]);
      if (live) sr[u + STRIDE * i] = v[i];
    }
  }
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    float f[8];
    unpack8(v[i], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) ss = fmaf(f[j], f[j], ss);
  }
  ss = row_sum<WPR>(ss, red);
  if (!live) return;
  const float r = rsqrtf(ss / static_cast<float>(D) + eps);
  if (inv != nullptr && u == 0) inv[row] = r;
  uint4* yr = reinterpret_cast<uint4*>(y + row * D);
  const float4* g4 = reinterpret_cast<const float4*>(gain);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = u + STRIDE * i;
    const float4 g0 = __ldg(g4 + 2 * c), g1 = __ldg(g4 + 2 * c + 1);
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    float f[8];
    unpack8(v[i], f);
#pragma unroll
    for (int j = 0; j < 8; ++j) f[j] = (f[j] * r) * g[j];
    yr[c] = pack8(f);
  }
}

// dx = gdy * inv - x * (Σ gdy·x) * inv^3 / D (+ dres), gdy = gain * Σ_i dy_i  (transformer.py:487-496).
// Σ_i dy_i is kept as bf16 (the sum autograd would store between the group's dx and the norm's backward).
template <int VPL, int WPR, int NDY>
__global__ void __launch_bounds__(kRowWarps * 32) k_rmsnorm_bwd(const __nv_bfloat16* __restrict__ x,
                                                                const float* __restrict__ gain,
                                                                const float* __restrict__ inv, GlueDys dys,
                                                                const __nv_bfloat16* __restrict__ dres,
                                                                __nv_bfloat16* __restrict__ dx, int64_t rows) {
  constexpr int D = 256 * VPL, NV = VPL / WPR, STRIDE = 32 * WPR;
  __shared__ float red[kRowWarps];
  const int u = threadIdx.x % STRIDE;
  int64_t row = static_cast<int64_t>(blockIdx.x) * (kRowWarps / WPR) + threadIdx.x / STRIDE;
  const bool live = row < rows;
  if (WPR == 1 && !live) return;
  if (!live) row = rows - 1;  // shares the row reduction's barrier, writes nothing
  const uint4* xr = reinterpret_cast<const uint4*>(x + row * D);
  const float4* g4 = reinterpret_cast<const float4*>(gain);
  uint4 xv[NV], dv[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = u + STRIDE * i;
    xv[i] = __ldg(xr + c);
    dv[i] = __ldg(reinterpret_cast<const uint4*>(dys.p[0] + row * D) + c);
#pragma unroll
    for (int k = 1; k < NDY; ++k) {
      const uint4 w = __ldg(reinterpret_cast<const uint4*>(dys.p[k] + row * D) + c);
      __nv_bfloat162* p = reinterpret_cast<__nv_bfloat162*>(&dv[i]);
      const __nv_bfloat162* q = reinterpret_cast<const __nv_bfloat162*>(&w);
#pragma unroll
      for (int j = 0; j < 4; ++j) p[j] = __hadd2(p[j], q[j]);
    }
  }
  float inner = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = u + STRIDE * i;
    const float4 g0 = __ldg(g4 + 2 * c), g1 = __ldg(g4 + 2 * c + 1);
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    float f[8], d[8];
    unpack8(xv[i], f);
    unpack8(dv[i], d);
#pragma unroll
    for (int j = 0; j < 8; ++j) inner = fmaf(d[j] * g[j], f[j], inner);
  }
  inner = row_sum<WPR>(inner, red);
  if (!live) return;
  const float r = inv[row];
  const float coef = inner * r * r * r / static_cast<float>(D);
  uint4* out = reinterpret_cast<uint4*>(dx + row * D);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = u + STRIDE * i;
    const float4 g0 = __ldg(g4 + 2 * c), g1 = __ldg(g4 + 2 * c + 1);
    const float g[8] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
    float f[8], d[8], o[8];
    unpack8(xv[i], f);
    unpack8(dv[i], d);
    float rr[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (dres != nullptr) unpack8(__ldg(reinterpret_cast<const uint4*>(dres + row * D) + c), rr);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = ((d[j] * g[j]) * r - f[j] * coef) + rr[j];
    out[c] = pack8(o);
  }
}

// In-place rotation of adjacent (even, odd) pairs of every head vector by sign * pos * base^(-2i/d):
// x[t, h*d + 2i], x[t, h*d + 2i + 1] with pos = t % seq (transformer.py:506-519). Two tensors per launch
// (q and k). Each thread rotates 4 pairs (one 16-byte chunk).
__global__ void __launch_bounds__(256) k_rope(__nv_bfloat16* __restrict__ x0, __nv_bfloat16* __restrict__ x1,
                                              int64_t rows, int D, int head_dim, int seq,
                                              const float* __restrict__ cos_t, const float* __restrict__ sin_t,
                                              float sign) {
  // blockIdx.y picks the tensor; each CTA walks whole rows (chunk = threadIdx.x + 256 j) so the row, its
  // position and the table row are computed once per row.
  __nv_bfloat16* base = blockIdx.y == 0 ? x0 : x1;
  const int chunks = D / 8;
  const int half = head_dim / 2;
  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int pos = static_cast<int>(row % seq);
    const float* cr = cos_t + static_cast<int64_t>(pos) * half;
    const float* sr = sin_t + static_cast<int64_t>(pos) * half;
    uint4* rp = reinterpret_cast<uint4*>(base + row * D);
    for (int c = threadIdx.x; c < chunks; c += blockDim.x) {
      const int p0 = ((c * 8) % head_dim) / 2;  // first pair index within the head
      float f[8];
      unpack8(rp[c], f);
      const float4 cs = __ldg(reinterpret_cast<const float4*>(cr + p0));
      const float4 sn = __ldg(reinterpret_cast<const float4*>(sr + p0));
      const float cc[4] = {cs.x, cs.y, cs.z, cs.w};
      const float ss[4] = {sn.x * sign, sn.y * sign, sn.z * sign, sn.w * sign};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float ev = f[2 * j], od = f[2 * j + 1];
        f[2 * j] = ev * cc[j] - od * ss[j];
        f[2 * j + 1] = ev * ss[j] + od * cc[j];
      }
      rp[c] = pack8(f);
    }
  }
}

__device__ __forceinline__ float sigmoidf_(float g) { return 1.f / (1.f + __expf(-g)); }

// act = up * silu(gate)
__global__ void __launch_bounds__(256) k_swiglu_fwd(const uint4* __restrict__ up, const uint4* __restrict__ gate,
                                                    uint4* __restrict__ act, int64_t n8) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float u[8], g[8], o[8];
    unpack8(__ldg(up + i), u);
    unpack8(__ldg(gate + i), g);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = u[j] * (g[j] * sigmoidf_(g[j]));
    act[i] = pack8(o);
  }
}

// dup = dact * silu(gate); dgate = dact * up * s * (1 + gate * (1 - s)), s = sigmoid(gate)
__global__ void __launch_bounds__(256) k_swiglu_bwd(const uint4* __restrict__ up, const uint4* __restrict__ gate,
                                                    const uint4* __restrict__ dact, uint4* __restrict__ dup,
                                                    uint4* __restrict__ dgate, int64_t n8) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n8;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float u[8], g[8], d[8], du[8], dg[8];
    unpack8(__ldg(up + i), u);
    unpack8(__ldg(gate + i), g);
    unpack8(__ldg(dact + i), d);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float s = sigmoidf_(g[j]);
      du[j] = d[j] * (g[j] * s);
      dg[j] = d[j] * u[j] * s * (1.f + g[j] * (1.f - s));
    }
    dup[i] = pack8(du);
    dgate[i] = pack8(dg);
  }
}

// Per row of V logits: loss_row = logsumexp - logit[target]; dlogits = (softmax - onehot) * scale
// (transformer.py:569-588 with scale = 1 / rows). One CTA per row; pass 1 keeps a per-thread online
// (max, sum), pass 2 re-reads the row (L2) and writes the bf16 gradient.
constexpr int kXentThreads = 512;

__global__ void __launch_bounds__(kXentThreads) k_xent(const __nv_bfloat16* __restrict__ logits,
                                                       const int64_t* __restrict__ targets, int V, float scale,
                                                       float* __restrict__ loss_rows,
                                                       __nv_bfloat16* __restrict__ dlogits) {
  const int64_t row = blockIdx.x;
  const uint4* lr = reinterpret_cast<const uint4*>(logits + row * V);
  const int n8 = V / 8;
  float m = -INFINITY, s = 0.f;
  for (int c = threadIdx.x; c < n8; c += kXentThreads) {
    float f[8];
    unpack8(__ldg(lr + c), f);
    float cm = f[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) cm = fmaxf(cm, f[j]);
    const float nm = fmaxf(m, cm);
    float add = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) add += __expf(f[j] - nm);
    s = s * __expf(m - nm) + add;
    m = nm;
  }
  __shared__ float sm[kXentThreads / 32], ss[kXentThreads / 32];
  __shared__ float fin[2];
  // warp reduce (max, sum)
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const float om = __shfl_xor_sync(0xffffffffu, m, o), os = __shfl_xor_sync(0xffffffffu, s, o);
    const float nm = fmaxf(m, om);
    s = (m == -INFINITY ? 0.f : s * __expf(m - nm)) + (om == -INFINITY ? 0.f : os * __expf(om - nm));
    m = nm;
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sm[w] = m;
    ss[w] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float M = sm[0], S = ss[0];
    for (int i = 1; i < kXentThreads / 32; ++i) {
      const float nm = fmaxf(M, sm[i]);
      S = S * __expf(M - nm) + ss[i] * __expf(sm[i] - nm);
      M = nm;
    }
    fin[0] = M;
    fin[1] = S;
    const int64_t t = targets[row];
    // a target outside [0, V) reads nothing and marks the row NaN (the host wrapper raises IndexError first)
    const float lt = (t >= 0 && t < V) ? __bfloat162float(logits[row * V + t]) : __int_as_float(0x7fc00000);
    loss_rows[row] = (M + logf(S)) - lt;
  }
  __syncthreads();
  const float M = fin[0], invS = 1.f / fin[1];
  const int64_t t = targets[row];
  uint4* dr = reinterpret_cast<uint4*>(dlogits + row * V);
  for (int c = threadIdx.x; c < n8; c += kXentThreads) {
    float f[8];
    unpack8(__ldg(lr + c), f);
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const float p = __expf(f[j] - M) * invS - (static_cast<int64_t>(c * 8 + j) == t ? 1.f : 0.f);
      f[j] = p * scale;
    }
    dr[c] = pack8(f);
  }
}

// MSE against a target (the reference's loss is cross-entropy only): per row,
// loss_rows[r] = Σ_c (y - t)^2 (fixed-order block reduction) and dy = 2 (y - t) / (rows * cols).
template <typename YT, typename DT>
__global__ void __launch_bounds__(256) k_mse(const YT* __restrict__ y, const float* __restrict__ target, int64_t cols,
                                             float inv_n2, float* __restrict__ loss_rows, DT* __restrict__ dy) {
  const int64_t row = blockIdx.x;
  const YT* yr = y + row * cols;
  const float* tr = target + row * cols;
  float acc = 0.f;
  for (int64_t c = threadIdx.x; c < cols; c += 256) {
    const float d = to_f32(yr[c]) - tr[c];
    acc = fmaf(d, d, acc);
    if (dy != nullptr) dy[row * cols + c] = static_cast<DT>(d * inv_n2);
  }
  __shared__ float red[256];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (static_cast<int>(threadIdx.x) < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) loss_rows[row] = red[0];
}

int glue_grid(int64_t work, int threads) {
  int dev = 0, nsm = 0;  // per call: the current device's SM count (an attribute query, no global state)
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  if (nsm <= 0) nsm = 148;
  const int64_t want = (work + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(nsm) * 8;
  return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

cudaError_t launch_rmsnorm_fwd(const __nv_bfloat16* a, const __nv_bfloat16* b, __nv_bfloat16* sum,
                               const float* gain, __nv_bfloat16* y, float* inv, int64_t rows, int D, float eps,
                               cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  // <= 16 16-byte chunks per thread in registers: rows wider than 4096 share 2 warps
#define QA_RMS_CASE(V)                                                                                       \
  case V: {                                                                                                  \
    constexpr int W = V > 16 ? 2 : 1;                                                                       \
    const int grid = static_cast<int>((rows + kRowWarps / W - 1) / (kRowWarps / W));                       \
    if (b != nullptr)                                                                                        \
      k_rmsnorm_fwd<V, true, W><<<grid, kRowWarps * 32, 0, st>>>(a, b, sum, gain, y, inv, rows, eps);       \
    else                                                                                                     \
      k_rmsnorm_fwd<V, false, W><<<grid, kRowWarps * 32, 0, st>>>(a, nullptr, nullptr, gain, y, inv, rows, eps); \
    break;                                                                                                   \
  }
  switch (D / 256) {
    QA_RMS_CASE(1)
    QA_RMS_CASE(2)
    QA_RMS_CASE(4)
    QA_RMS_CASE(8)
    QA_RMS_CASE(16)
    QA_RMS_CASE(32)
    default:
      return cudaErrorInvalidValue;
  }
#undef QA_RMS_CASE
  return cudaGetLastError();
}

cudaError_t launch_rmsnorm_bwd(const __nv_bfloat16* x, const float* gain, const float* inv, const GlueDys& dys,
                               const __nv_bfloat16* dres, __nv_bfloat16* dx, int64_t rows, int D, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  // x and Σdy of <= 8 chunks per thread in registers: rows wider than 2048 share 2..4 warps
#define QA_RMSB_CASE(V)                                                                            \
  case V: {                                                                                        \
    constexpr int W = V > 8 ? V / 8 : 1;                                                          \
    const int grid = static_cast<int>((rows + kRowWarps / W - 1) / (kRowWarps / W));             \
    if (dys.n == 1)                                                                                \
      k_rmsnorm_bwd<V, W, 1><<<grid, kRowWarps * 32, 0, st>>>(x, gain, inv, dys, dres, dx, rows); \
    else if (dys.n == 2)                                                                           \
      k_rmsnorm_bwd<V, W, 2><<<grid, kRowWarps * 32, 0, st>>>(x, gain, inv, dys, dres, dx, rows); \
    else                                                                                           \
      k_rmsnorm_bwd<V, W, 3><<<grid, kRowWarps * 32, 0, st>>>(x, gain, inv, dys, dres, dx, rows); \
    break;                                                                                         \
  }
  switch (D / 256) {
    QA_RMSB_CASE(1)
    QA_RMSB_CASE(2)
    QA_RMSB_CASE(4)
    QA_RMSB_CASE(8)
    QA_RMSB_CASE(16)
    QA_RMSB_CASE(32)
    default:
      return cudaErrorInvalidValue;
  }
#undef QA_RMSB_CASE
  return cudaGetLastError();
}

cudaError_t launch_rope(__nv_bfloat16* x0, __nv_bfloat16* x1, int64_t rows, int D, int head_dim, int seq,
                        const float* cos_t, const float* sin_t, float sign, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  const int64_t want = rows < 148 * 16 ? rows : 148 * 16;
  const dim3 grid(static_cast<unsigned>(want), x1 != nullptr ? 2 : 1);
  const int threads = D / 8 >= 256 ? 256 : ((D / 8 + 31) / 32) * 32;
  k_rope<<<grid, threads, 0, st>>>(x0, x1, rows, D, head_dim, seq, cos_t, sin_t, sign);
  return cudaGetLastError();
}

cudaError_t launch_swiglu_fwd(const __nv_bfloat16* up, const __nv_bfloat16* gate, __nv_bfloat16* act, int64_t n,
                              cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_swiglu_fwd<<<glue_grid(n / 8, 256), 256, 0, st>>>(reinterpret_cast<const uint4*>(up),
                                                     reinterpret_cast<const uint4*>(gate),
                                                     reinterpret_cast<uint4*>(act), n / 8);
  return cudaGetLastError();
}

cudaError_t launch_swiglu_bwd(const __nv_bfloat16* up, const __nv_bfloat16* gate, const __nv_bfloat16* dact,
                              __nv_bfloat16* dup, __nv_bfloat16* dgate, int64_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  k_swiglu_bwd<<<glue_grid(n / 8, 256), 256, 0, st>>>(
      reinterpret_cast<const uint4*>(up), reinterpret_cast<const uint4*>(gate), reinterpret_cast<const uint4*>(dact),
      reinterpret_cast<uint4*>(dup), reinterpret_cast<uint4*>(dgate), n / 8);
  return cudaGetLastError();
}

cudaError_t launch_mse(const void* y, int y_dtype, const float* target, int64_t rows, int64_t cols, float* loss_rows,
                       void* dy, int dy_dtype, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  count_launches(1);
  const float inv_n2 = static_cast<float>(2.0 / (static_cast<double>(rows) * static_cast<double>(cols)));
  const unsigned grid = static_cast<unsigned>(rows);
  if (y_dtype == QA_F32 && dy_dtype == QA_F32)
    k_mse<float, float><<<grid, 256, 0, st>>>(static_cast<const float*>(y), target, cols, inv_n2, loss_rows,
                                              static_cast<float*>(dy));
  else if (y_dtype == QA_F32)
    k_mse<float, __nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const float*>(y), target, cols, inv_n2, loss_rows,
                                                      static_cast<__nv_bfloat16*>(dy));
  else if (dy_dtype == QA_F32)
    k_mse<__nv_bfloat16, float><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(y), target, cols, inv_n2,
                                                      loss_rows, static_cast<float*>(dy));
  else
    k_mse<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(y), target, cols,
                                                              inv_n2, loss_rows, static_cast<__nv_bfloat16*>(dy));
  return cudaGetLastError();
}

cudaError_t launch_xent(const __nv_bfloat16* logits, const int64_t* targets, int64_t rows, int V, float* loss_rows,
                        __nv_bfloat16* dlogits, cudaStream_t st) {
  if (rows == 0) return cudaSuccess;
  k_xent<<<static_cast<unsigned>(rows), kXentThreads, 0, st>>>(logits, targets, V, 1.f / static_cast<float>(rows),
                                                               loss_rows, dlogits);
  return cudaGetLastError();
}

}  // namespace qa

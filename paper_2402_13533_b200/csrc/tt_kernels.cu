// Tensor-train (matrix-product-operator) adapter contractions.
//
// The adapter is W_t[(i1..id),(j1..jd)] = G1[0,i1,j1,:]·G2[:,i2,j2,:]···Gd[:,id,jd,0]
// with row-major multi-indices.  Token-side work is organised as the left-to-right partial
// contractions Z_k[t, i<=k, r_k, j>k] (Z_0 = x, Z_d = y2):
//   forward stage k : Z_k = Σ_{a, j_k} Z_{k-1}[t, I, a, j_k, Q] · G_k[a, i_k, j_k, b]
//   backward stage k: dZ_{k-1}[t, I, a, j_k, Q] = Σ_{i_k, b} dZ_k[t, I, i_k, b, Q] · G_k[a, i_k, j_k, b]
//   core gradient   : dG_k[a, i_k, j_k, b] = Σ_{t, I, Q} Z_{k-1}[...] · dZ_k[...]
// (I = Π_{q<k} m_q, Q = Π_{q>k} n_q).  The core gradient reduction is two-phase with a fixed
// summation order, so results are bit-reproducible run to run (the reference's determinism
// contract, distsim.py:312).
#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_timing.h"

namespace qa {

int64_t TTDims::I(int k) const {
  int64_t v = 1;
  for (int q = 0; q < k; ++q) v *= m[q];
  return v;
}
int64_t TTDims::J(int k) const {
  int64_t v = 1;
  for (int q = k; q < d; ++q) v *= n[q];
  return v;
}

bool tt_dims(const qa_tt* tt, TTDims* o) {
  if (tt == nullptr || tt->d < 1 || tt->d > QA_TT_MAX_D) return false;
  o->d = tt->d;
  if (tt->r[0] != 1 || tt->r[tt->d] != 1) return false;
  o->N = 1;
  o->K = 1;
  for (int k = 0; k < tt->d; ++k) {
    if (tt->m[k] < 1 || tt->n[k] < 1 || tt->r[k] < 1 || tt->cores[k] == nullptr) return false;
    o->m[k] = tt->m[k];
    o->n[k] = tt->n[k];
    o->r[k] = tt->r[k];
    o->N *= tt->m[k];
    o->K *= tt->n[k];
  }
  o->r[tt->d] = 1;
  // Z_k[t, i<=k, r_k, j>k]: I(k) * r_k * J(k) per token (k = 0: x itself, k = d: y2)
  for (int k = 0; k <= tt->d; ++k) {
    int64_t ik = 1;
    for (int q = 0; q < k; ++q) ik *= o->m[q];
    o->zsize[k] = ik * o->r[k] * o->J(k);
  }
  return true;
}

namespace {

struct TTCorePtrs {
  const float* p[QA_TT_MAX_D];
};

template <typename T>
QA_DEV float ld_f(const T* p) {
  return to_f32(*p);
}

// One thread per output element of Z_k.
template <typename InT>
__global__ void __launch_bounds__(256) k_stage_fwd(const InT* __restrict__ in, int64_t in_ld,
                                                   const float* __restrict__ G, float* __restrict__ out,
                                                   int64_t out_ld, int64_t T, int64_t I, int A, int nk, int64_t Q,
                                                   int mk, int B) {
  const int64_t per_tok = I * mk * B * Q;
  const int64_t total = T * per_tok;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = idx / per_tok;
    int64_t rem = idx - t * per_tok;
    const int64_t q = rem % Q;
    rem /= Q;
    const int b = static_cast<int>(rem % B);
    rem /= B;
    const int ik = static_cast<int>(rem % mk);
    const int64_t i = rem / mk;
    const InT* src = in + t * in_ld + i * (static_cast<int64_t>(A) * nk * Q) + q;
    float acc = 0.f;
    for (int a = 0; a < A; ++a) {
      const float* g = G + ((static_cast<int64_t>(a) * mk + ik) * nk) * B + b;  // G[a, ik, j, b]
      const InT* s = src + static_cast<int64_t>(a) * nk * Q;
      for (int j = 0; j < nk; ++j) acc = fmaf(ld_f(s + j * Q), g[static_cast<int64_t>(j) * B], acc);
    }
    out[t * out_ld + rem * B * Q + static_cast<int64_t>(b) * Q + q] = acc;
  }
}

// One thread per element of dZ_{k-1}.
template <typename OutT>
__global__ void __launch_bounds__(256) k_stage_bwd(const OutT* __restrict__ dout, int64_t dout_ld,
                                                   const float* __restrict__ G, float* __restrict__ din,
                                                   int64_t din_ld, int64_t T, int64_t I, int A, int nk, int64_t Q,
                                                   int mk, int B) {
  const int64_t per_tok = I * A * nk * Q;
  const int64_t total = T * per_tok;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = idx / per_tok;
    int64_t rem = idx - t * per_tok;
    const int64_t q = rem % Q;
    rem /= Q;
    const int j = static_cast<int>(rem % nk);
    rem /= nk;
    const int a = static_cast<int>(rem % A);
    const int64_t i = rem / A;
    const OutT* src = dout + t * dout_ld + i * (static_cast<int64_t>(mk) * B * Q) + q;
    float acc = 0.f;
    for (int ik = 0; ik < mk; ++ik) {
      const float* g = G + ((static_cast<int64_t>(a) * mk + ik) * nk + j) * B;  // G[a, ik, j, :]
      const OutT* s = src + static_cast<int64_t>(ik) * B * Q;
      for (int b = 0; b < B; ++b) acc = fmaf(ld_f(s + static_cast<int64_t>(b) * Q), g[b], acc);
    }
    din[t * din_ld + idx - t * per_tok] = acc;
  }
}

// Phase 1: partial[chunk][g] = Σ over the chunk's tokens; one thread per core element.
template <typename InT, typename OutT>
__global__ void __launch_bounds__(256) k_core_grad_partial(const InT* __restrict__ in, int64_t in_ld,
                                                           const OutT* __restrict__ dout, int64_t dout_ld,
                                                           float* __restrict__ partial, int nchunks, int64_t T,
                                                           int64_t I, int A, int nk, int64_t Q, int mk, int B) {
  const int64_t numel = static_cast<int64_t>(A) * mk * nk * B;
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int chunk = blockIdx.y;
  if (g >= numel) return;
  const int b = static_cast<int>(g % B);
  const int j = static_cast<int>((g / B) % nk);
  const int ik = static_cast<int>((g / (static_cast<int64_t>(B) * nk)) % mk);
  const int a = static_cast<int>(g / (static_cast<int64_t>(B) * nk * mk));
  const int64_t per = (T + nchunks - 1) / nchunks;
  const int64_t t0 = chunk * per, t1 = t0 + per < T ? t0 + per : T;
  float acc = 0.f;
  for (int64_t t = t0; t < t1; ++t) {
    const InT* zi = in + t * in_ld + (static_cast<int64_t>(a) * nk + j) * Q;
    const OutT* zo = dout + t * dout_ld + (static_cast<int64_t>(ik) * B + b) * Q;
    for (int64_t i = 0; i < I; ++i) {
      const InT* zi_i = zi + i * (static_cast<int64_t>(A) * nk * Q);
      const OutT* zo_i = zo + i * (static_cast<int64_t>(mk) * B * Q);
      for (int64_t q = 0; q < Q; ++q) acc = fmaf(ld_f(zi_i + q), ld_f(zo_i + q), acc);
    }
  }
  partial[static_cast<int64_t>(chunk) * numel + g] = acc;
}

// Phase 2: fixed-order sum over chunks.  A block owns 32 consecutive outputs; warp w sums chunks
// w, w+8, ... (lane = output), then lanes combine the 8 warp sums in warp order.
__global__ void __launch_bounds__(256) k_core_grad_reduce(const float* __restrict__ partial, int nchunks,
                                                          int64_t numel, float* __restrict__ dG, int accumulate) {
  __shared__ float red[8][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t g = static_cast<int64_t>(blockIdx.x) * 32 + lane;
  float s = 0.f;
  if (g < numel) {
    int c = warp;
    for (; c + 24 < nchunks; c += 32) {  // 4 independent loads in flight
      const float a0 = partial[static_cast<int64_t>(c) * numel + g];
      const float a1 = partial[static_cast<int64_t>(c + 8) * numel + g];
      const float a2 = partial[static_cast<int64_t>(c + 16) * numel + g];
      const float a3 = partial[static_cast<int64_t>(c + 24) * numel + g];
      s += a0;
      s += a1;
      s += a2;
      s += a3;
    }
    for (; c < nchunks; c += 8) s += partial[static_cast<int64_t>(c) * numel + g];
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && g < numel) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    dG[g] = accumulate ? dG[g] + t : t;
  }
}

// L[ip, jp, b] = (G_0 ··· G_{d-2})[ip, jp, b]; one thread per element, chain of small vector-matrix products.
__global__ void __launch_bounds__(128) k_prefix_full(TTDims dd, TTCorePtrs cores,
                                                     float* __restrict__ L, int64_t IP, int64_t JP, int R) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= IP * JP * R) return;
  const int b = static_cast<int>(idx % R);
  const int64_t jp = (idx / R) % JP;
  const int64_t ip = idx / (static_cast<int64_t>(R) * JP);
  const int last = dd.d - 1;  // cores 0..last-1 are contracted
  int iv[QA_TT_MAX_D], jv[QA_TT_MAX_D];
  int64_t ir = ip, jr = jp;
  for (int k = last - 1; k >= 0; --k) {
    iv[k] = static_cast<int>(ir % dd.m[k]);
    ir /= dd.m[k];
    jv[k] = static_cast<int>(jr % dd.n[k]);
    jr /= dd.n[k];
  }
  constexpr int kMaxR = 64;
  float v[kMaxR], w[kMaxR];
  v[0] = 1.f;
  int ra = 1;
  for (int k = 0; k < last; ++k) {
    const int rb = dd.r[k + 1];
    const float* g = cores.p[k];
    for (int bb = 0; bb < rb; ++bb) {
      float s = 0.f;
      for (int a = 0; a < ra; ++a)
        s = fmaf(v[a], g[((static_cast<int64_t>(a) * dd.m[k] + iv[k]) * dd.n[k] + jv[k]) * rb + bb], s);
      w[bb] = s;
    }
    for (int bb = 0; bb < rb; ++bb) v[bb] = w[bb];
    ra = rb;
  }
  L[idx] = v[b];
}

template <typename OutT>
QA_DEV void store_out(OutT* p, float v);
template <>
QA_DEV void store_out<float>(float* p, float v) {
  *p = v;
}
template <>
QA_DEV void store_out<__nv_bfloat16>(__nv_bfloat16* p, float v) {
  *p = __float2bfloat16_rn(v);
}

// out[(h, i), (jp, j)] = Σ_b L[h, jp, b] Gd[b, i, j, 0]  (+ fp64 dequantised code when merging)
template <typename OutT>
__global__ void __launch_bounds__(256) k_last_full(const float* __restrict__ L, const float* __restrict__ Gd,
                                                   int64_t H, int64_t JP, int R, int md, int nd,
                                                   const uint8_t* __restrict__ codes, int bits,
                                                   const float* __restrict__ scale,
                                                   const float* __restrict__ offset, OutT* __restrict__ out) {
  const int64_t N = H * md, K = JP * nd;
  const int64_t total = N * K;
  for (int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; idx < total;
       idx += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = idx / K, col = idx - row * K;
    const int64_t h = row / md, jp = col / nd;
    const int i = static_cast<int>(row - h * md), j = static_cast<int>(col - jp * nd);
    const float* l = L + (h * JP + jp) * R;
    float s = 0.f;
    for (int b = 0; b < R; ++b) s = fmaf(l[b], Gd[(static_cast<int64_t>(b) * md + i) * nd + j], s);
    if (codes != nullptr) {
      const int64_t ldc = bits == 8 ? K : (K + 1) / 2;
      const uint8_t* cr = codes + row * ldc;
      const uint32_t c = bits == 8 ? cr[col] : ((col & 1) ? (cr[col >> 1] >> 4) : (cr[col >> 1] & 0xF));
      const double deq = __dadd_rn(__dmul_rn(static_cast<double>(c), static_cast<double>(scale[row])),
                                   static_cast<double>(offset[row]));
      store_out<OutT>(out + idx, static_cast<float>(__dadd_rn(deq, static_cast<double>(s))));
    } else {
      store_out<OutT>(out + idx, s);
    }
  }
}

unsigned grid_for(int64_t total, int threads) {
  const int64_t blocks = (total + threads - 1) / threads;
  return static_cast<unsigned>(blocks < 148 * 64 ? (blocks > 0 ? blocks : 1) : 148 * 64);
}

}  // namespace

cudaError_t launch_tt_stage_fwd(const void* in, int in_dtype, int64_t in_ld, const float* G, float* out,
                                int64_t out_ld, int64_t T, int64_t I, int A, int nk, int64_t Q, int mk, int B,
                                cudaStream_t s) {
  const int64_t total = T * I * mk * B * Q;
  if (total == 0) return cudaSuccess;
  LaunchScope scope(kTT, 2.0 * double(total) * A * nk, s);
  count_launches(1);
  if (in_dtype == QA_F32)
    k_stage_fwd<float><<<grid_for(total, 256), 256, 0, s>>>(static_cast<const float*>(in), in_ld, G, out, out_ld, T,
                                                             I, A, nk, Q, mk, B);
  else
    k_stage_fwd<__nv_bfloat16><<<grid_for(total, 256), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(in), in_ld, G,
                                                                     out, out_ld, T, I, A, nk, Q, mk, B);
  return cudaGetLastError();
}

cudaError_t launch_tt_stage_bwd(const void* dout, int dout_dtype, int64_t dout_ld, const float* G, float* din,
                                int64_t din_ld, int64_t T, int64_t I, int A, int nk, int64_t Q, int mk, int B,
                                cudaStream_t s) {
  const int64_t total = T * I * A * nk * Q;
  if (total == 0) return cudaSuccess;
  LaunchScope scope(kTT, 2.0 * double(total) * mk * B, s);
  count_launches(1);
  if (dout_dtype == QA_F32)
    k_stage_bwd<float><<<grid_for(total, 256), 256, 0, s>>>(static_cast<const float*>(dout), dout_ld, G, din, din_ld,
                                                             T, I, A, nk, Q, mk, B);
  else
    k_stage_bwd<__nv_bfloat16><<<grid_for(total, 256), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(dout), dout_ld,
                                                                     G, din, din_ld, T, I, A, nk, Q, mk, B);
  return cudaGetLastError();
}

cudaError_t launch_sum_partials(const float* partial, int nparts, int64_t numel, float* out, bool accumulate,
                                cudaStream_t s) {
  if (numel == 0) return cudaSuccess;
  LaunchScope scope(kTT, 4.0 * double(numel) * (nparts + 1), s);
  count_launches(1);
  k_core_grad_reduce<<<static_cast<unsigned>((numel + 31) / 32), 256, 0, s>>>(partial, nparts, numel, out,
                                                                                accumulate ? 1 : 0);
  return cudaGetLastError();
}

int tt_grad_chunks(int64_t T) { return static_cast<int>(T < 296 ? (T > 0 ? T : 1) : 296); }

cudaError_t launch_tt_core_grad(const void* in, int in_dtype, int64_t in_ld, const void* dout, int dout_dtype,
                                int64_t dout_ld, float* partial, int nchunks, float* dG, bool accumulate,
                                int64_t T, int64_t I, int A, int nk, int64_t Q, int mk, int B, cudaStream_t s) {
  const int64_t numel = static_cast<int64_t>(A) * mk * nk * B;
  LaunchScope scope(kTT, 2.0 * double(numel) * T * I * Q, s);
  count_launches(2);
  const dim3 grid(static_cast<unsigned>((numel + 255) / 256), static_cast<unsigned>(nchunks));
#define QA_CG(TI, TO)                                                                                            \
  k_core_grad_partial<TI, TO><<<grid, 256, 0, s>>>(static_cast<const TI*>(in), in_ld, static_cast<const TO*>(dout), \
                                                  dout_ld, partial, nchunks, T, I, A, nk, Q, mk, B)
  if (in_dtype == QA_F32 && dout_dtype == QA_F32)
    QA_CG(float, float);
  else if (in_dtype == QA_F32)
    QA_CG(float, __nv_bfloat16);
  else if (dout_dtype == QA_F32)
    QA_CG(__nv_bfloat16, float);
  else
    QA_CG(__nv_bfloat16, __nv_bfloat16);
#undef QA_CG
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  k_core_grad_reduce<<<static_cast<unsigned>((numel + 31) / 32), 256, 0, s>>>(partial, nchunks, numel, dG,
                                                                                accumulate ? 1 : 0);
  return cudaGetLastError();
}

cudaError_t launch_tt_prefix_full(const TTDims& dd, const float* const* cores, float* L, cudaStream_t s) {
  TTCorePtrs cp{};
  for (int k = 0; k < dd.d; ++k) cp.p[k] = cores[k];
  const int last = dd.d - 1;
  int64_t IP = 1, JP = 1;
  for (int k = 0; k < last; ++k) {
    IP *= dd.m[k];
    JP *= dd.n[k];
  }
  const int R = dd.r[last];
  const int64_t total = IP * JP * R;
  LaunchScope scope(kMerge, 4.0 * double(total), s);
  count_launches(1);
  k_prefix_full<<<static_cast<unsigned>((total + 127) / 128), 128, 0, s>>>(dd, cp, L, IP, JP, R);
  return cudaGetLastError();
}

cudaError_t launch_tt_last_full(const TTDims& dd, const float* L, const float* Gd, const uint8_t* codes, int bits,
                                const float* scale, const float* offset, void* out, int out_dtype, cudaStream_t s) {
  const int last = dd.d - 1;
  int64_t H = 1, JP = 1;
  for (int k = 0; k < last; ++k) {
    H *= dd.m[k];
    JP *= dd.n[k];
  }
  const int64_t total = dd.N * dd.K;
  LaunchScope scope(kMerge, double(total) * ((codes ? (bits == 8 ? 1.0 : 0.5) : 0.0) + (out_dtype == QA_F32 ? 4 : 2)), s);
  count_launches(1);
  if (out_dtype == QA_F32)
    k_last_full<float><<<grid_for(total, 256), 256, 0, s>>>(L, Gd, H, JP, dd.r[last], dd.m[last], dd.n[last], codes,
                                                            bits, scale, offset, static_cast<float*>(out));
  else
    k_last_full<__nv_bfloat16><<<grid_for(total, 256), 256, 0, s>>>(L, Gd, H, JP, dd.r[last], dd.m[last], dd.n[last],
                                                                    codes, bits, scale, offset,
                                                                    static_cast<__nv_bfloat16*>(out));
  return cudaGetLastError();
}

}  // namespace qa

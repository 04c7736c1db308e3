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
#include <cmath>
#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_timing.h"
#include "quant_row.cuh"

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

// Prefix of the pinned 3-core modes (m_1 = 1): L[h, j1 J1 + j2, :] = G1[0, 0, j1, :] · G2[:, h, j2, :].
// A CTA owns one h and 256 columns; G2[:, h, :, :] (R x J1 x R) sits in shared memory.
template <int R>
__global__ void __launch_bounds__(256) k_prefix_d3(const float* __restrict__ G1, const float* __restrict__ G2,
                                                   float* __restrict__ L, int H, int J1, int64_t K) {
  __shared__ float g2[R][16][R];  // [a][j2][b], J1 <= 16
  const int h = blockIdx.y;
  for (int q = threadIdx.x; q < R * J1 * R; q += 256) {
    const int a = q / (J1 * R), j2 = (q / R) % J1, b = q % R;
    g2[a][j2][b] = G2[((static_cast<int64_t>(a) * H + h) * J1 + j2) * R + b];
  }
  __syncthreads();
  const int64_t col = static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x;
  if (col >= K) return;
  const int64_t j1 = col / J1;
  const int j2 = static_cast<int>(col - j1 * J1);
  float v[R];
#pragma unroll
  for (int a = 0; a < R; ++a) v[a] = __ldg(G1 + j1 * R + a);
  float out[R];
#pragma unroll
  for (int b = 0; b < R; ++b) {
    float acc = 0.f;
#pragma unroll
    for (int a = 0; a < R; ++a) acc = fmaf(v[a], g2[a][j2][b], acc);
    out[b] = acc;
  }
  float4* dst = reinterpret_cast<float4*>(L + (static_cast<int64_t>(h) * K + col) * R);
#pragma unroll
  for (int q = 0; q < R / 4; ++q) dst[q] = make_float4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
}

// Same chain, one thread per (ip, jp) writing all R entries (R <= 16).
__global__ void __launch_bounds__(128) k_prefix_vec(TTDims dd, TTCorePtrs cores, float* __restrict__ L, int64_t IP,
                                                    int64_t JP, int R) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= IP * JP) return;
  const int64_t jp = idx % JP, ip = idx / JP;
  const int last = dd.d - 1;
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
  for (int b = 0; b < R; ++b) L[idx * R + b] = v[b];
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

// Merge / materialise for last cores with n_d = 1 (the pinned Llama modes and LoRA):
//   W'[row, col] = code(row, col) * scale[row] + offset[row] + Σ_b L[h, col, b] Gd[b, i],  row = h md + i
// A warp owns one row and 128 consecutive columns (4 per lane: one 4- or 2-byte code load, one 8- or
// 16-byte output store per lane, coalesced); the CTA's 8 warps walk MG_ROWS rows of one h-block with
// the lane's L[h, col, :] pairs held in registers (packed FFMA2 over column pairs) and the code words
// of RU rows loaded before any is used.  Dequantisation is one fp32 FMA (error < 1 ulp of fp32 against
// the reference's fp64 route, quant.py:102-105 — well inside the merge's 1e-5 tolerance).
constexpr int MG_COLS = 256, MG_GROUPS = 1;  // 4 groups measured slower (243 vs 216 us, 70B gate)

template <typename OutT, int BITS, int R>
__global__ void __launch_bounds__(256, 2) k_merge_nd1(const float* __restrict__ L, const float* __restrict__ Gd,
                                                      int64_t md, int64_t N, int64_t K, int MG_ROWS,
                                                      const uint8_t* __restrict__ codes,
                                                      const float* __restrict__ scale,
                                                      const float* __restrict__ offset, OutT* __restrict__ out) {
  __shared__ float gs[R][256];  // Gd[:, i] of this CTA's rows (i = row - h md), MG_ROWS <= 256
  __shared__ float ss[256], os[256];
  extern __shared__ __align__(16) uint8_t mg_codes[];  // the CTA's code tile [MG_ROWS][256 * BITS / 8]
  constexpr int CB = MG_COLS * BITS / 8;               // code bytes per tile row
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * MG_COLS;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * MG_ROWS;
  const int64_t h = r0 / md;  // MG_ROWS divides md: one h-block per CTA
  const int i0 = static_cast<int>(r0 - h * md);
  const int64_t cld = BITS == 8 ? K : (K + 1) / 2;
  // the whole code tile in flight at once (cp.async, MG_GROUPS commit groups of rows), consumed from
  // shared memory group by group while the later groups are still landing
  const int grows = MG_ROWS / MG_GROUPS;
  {
    const int64_t cb0 = BITS == 8 ? c0 : c0 / 2;
    for (int gq = 0; gq < MG_GROUPS; ++gq) {
      if (codes != nullptr)
        for (int q = threadIdx.x; q < grows * (CB / 16); q += 256) {
          const int r = gq * grows + q / (CB / 16), ch = q % (CB / 16);
          const bool ok = r0 + r < N && cb0 + ch * 16 + 16 <= cld;
          cp_async16(mg_codes + r * CB + ch * 16, ok ? codes + (r0 + r) * cld + cb0 + ch * 16 : codes, ok);
        }
      cp_async_commit();
    }
  }
  for (int q = threadIdx.x; q < R * MG_ROWS; q += 256) gs[q / MG_ROWS][q % MG_ROWS] = Gd[(q / MG_ROWS) * md + i0 + q % MG_ROWS];
  for (int q = threadIdx.x; q < MG_ROWS; q += 256) {
    ss[q] = codes != nullptr && r0 + q < N ? scale[r0 + q] : 0.f;
    os[q] = codes != nullptr && r0 + q < N ? offset[r0 + q] : 0.f;
  }
  const int64_t col = c0 + lane * 8;
  unsigned long long lp[R][4];  // column pairs of the lane's 8 columns, per rank index b
  {
    const float4* lr = reinterpret_cast<const float4*>(L + (h * K + col) * R);
    float lv[8][R];
#pragma unroll
    for (int c = 0; c < 8; ++c)
#pragma unroll
      for (int q = 0; q < R / 4; ++q) {
        const float4 v = __ldg(lr + c * (R / 4) + q);
        lv[c][4 * q] = v.x;
        lv[c][4 * q + 1] = v.y;
        lv[c][4 * q + 2] = v.z;
        lv[c][4 * q + 3] = v.w;
      }
#pragma unroll
    for (int b = 0; b < R; ++b)
#pragma unroll
      for (int q = 0; q < 4; ++q) lp[b][q] = f2pack(lv[2 * q][b], lv[2 * q + 1][b]);
  }
  OutT* obase = out + col;
  const bool active = col < K;
  for (int rl = warp; rl < MG_ROWS; rl += 8) {
    if (rl % grows < 8) {  // first row of a group for this warp: its codes have landed for every thread
      cp_async_wait_dyn(MG_GROUPS - 1 - rl / grows);
      __syncthreads();
    }
    const int64_t row = r0 + rl;
    if (row >= N || !active) continue;
    unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
    for (int b = 0; b < R; ++b) {
      const float gb = gs[b][rl];
      const unsigned long long g2 = f2pack(gb, gb);
#pragma unroll
      for (int q = 0; q < 4; ++q) ffma2(acc[q], g2, lp[b][q]);
    }
    float wt[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      wt[2 * q] = f2lo(acc[q]);
      wt[2 * q + 1] = f2hi(acc[q]);
    }
    if (codes != nullptr) {
      uint32_t cv[8];
      if constexpr (BITS == 8) {
        const uint2 w = *reinterpret_cast<const uint2*>(mg_codes + rl * CB + lane * 8);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          cv[e] = (w.x >> (8 * e)) & 0xFFu;
          cv[4 + e] = (w.y >> (8 * e)) & 0xFFu;
        }
      } else {  // two codes per byte, even column in the low nibble (quant.py:37-52)
        const uint32_t w = *reinterpret_cast<const uint32_t*>(mg_codes + rl * CB + lane * 4);
#pragma unroll
        for (int e = 0; e < 8; ++e) cv[e] = (w >> (4 * e)) & 0xFu;
      }
      const float sc = ss[rl], of = os[rl];
#pragma unroll
      for (int e = 0; e < 8; ++e) wt[e] += fmaf(static_cast<float>(cv[e]), sc, of);
    }
    OutT* dst = obase + row * K;
    if constexpr (sizeof(OutT) == 2) {
      uint4 pk;
      uint32_t* pw = reinterpret_cast<uint32_t*>(&pk);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const __nv_bfloat162 b2 = __floats2bfloat162_rn(wt[2 * q], wt[2 * q + 1]);
        pw[q] = *reinterpret_cast<const uint32_t*>(&b2);
      }
      *reinterpret_cast<uint4*>(dst) = pk;
    } else {
      *reinterpret_cast<float4*>(dst) = make_float4(wt[0], wt[1], wt[2], wt[3]);
      *reinterpret_cast<float4*>(dst + 4) = make_float4(wt[4], wt[5], wt[6], wt[7]);
    }
  }
}

// Fused merge / materialise for the fast TT family (first core input-only, last core output-only: the pinned
// Llama modes m = (1, H, M), n = (J0, J1, 1), and LoRA, m = (1, N), n = (K, 1)):
//   W'[row, col] = code·scale[row] + offset[row] + Σ_b L[col, b] · Gd[b, i],   row = h·md + i
//   d = 3: L[col, b] = Σ_a G1[j0, a] · G2[a, h, j1, b]  (col = j0·J1 + j1);  d = 2: L[col, b] = G1[col, b]
// A CTA owns RT rows of one h-block (RT divides md, so every row of the tile exists) and 32·CPL columns,
// CPL = 64 / R (8 for r = 8, 4 for r = 16).  The prologue stages Gd[:, i] and scale / offset per tile row and
// forms L for the tile's columns (one thread per column, all R values); then every lane holds its CPL columns'
// L as R x CPL/2 packed pairs (64 registers) and walks RT/4 consecutive rows of its warp with no predicates:
// the code word (prefetched MF_UN rows ahead), codes -> fp32 by one byte permute into the 2^23 exponent field
// and a packed subtract, one packed FMA dequantisation per column pair (< 1 ulp of the reference's fp64
// route, quant.py:102-105), R packed FMAs per column pair on a broadcast Gd value, one 16-byte store (a warp
// writes 512 contiguous bytes per row in bf16).
template <int R>
__host__ __device__ constexpr int mf_cpl() { return 64 / R; }
template <int R>
__host__ __device__ constexpr int mf_cols() { return 32 * mf_cpl<R>(); }

// code bytes of a lane's CPL columns in one row (2, 4 or 8), and the code-row ring per warp: MF_SLOTS batches of
// MF_UN rows in flight as cp.async copies (no registers held), so each SM keeps 16-64 KB of code reads in flight
// while the stores stream out
template <int BITS, int CPL>
__host__ __device__ constexpr int mf_lane_bytes() { return CPL * BITS / 8; }
constexpr int MF_SLOTS = 4, MF_UN = 8;

constexpr int MF_THREADS = 128;  // 4 warps: 4 CTAs (16 warps) per SM at <= 128 registers

template <typename OutT, int BITS, int R, bool D3>
__global__ void __launch_bounds__(MF_THREADS, 4) k_merge_fast(const float* __restrict__ G1, const float* __restrict__ G2,
                                                             const float* __restrict__ Gd, int R1, int J1, int H,
                                                             int64_t md, int64_t N, int64_t K, int RT,
                                                             const uint8_t* __restrict__ codes,
                                                             const float* __restrict__ scale,
                                                             const float* __restrict__ offset, OutT* __restrict__ out) {
  constexpr int CPL = mf_cpl<R>(), COLS = mf_cols<R>(), NP = CPL / 2, NWARP = MF_THREADS / 32;
  constexpr int LB = mf_lane_bytes<BITS, CPL>();  // code bytes per lane and row
  constexpr int CB = LB < 4 ? 4 : LB;               // bytes per copy (an even lane copies its pair when LB = 2)
  constexpr int NW = LB > 4 ? 2 : 1;
  constexpr int SLOT = MF_UN * 32 * LB;
  extern __shared__ __align__(16) float mf_smem[];
  float* gs = mf_smem;           // [RT][R]: Gd[:, i] per tile row
  float* ls = gs + RT * R;       // [COLS][R]: L of the tile's columns (formed once per CTA)
  float* so = ls + COLS * R;     // [RT][2]: scale, offset per tile row
  float* g2s = so + 2 * RT;      // [R1][J1][R]: G2[:, h, :, :] (d = 3)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // [NWARP][MF_SLOTS][MF_UN][32 lanes][LB]: this warp's code ring
  const uint32_t ring = smem_u32(g2s + R1 * J1 * R) + static_cast<uint32_t>(warp * MF_SLOTS * SLOT);
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * COLS;
  const int64_t r0 = static_cast<int64_t>(blockIdx.y) * RT;
  const int64_t h = r0 / md;
  const int64_t i0 = r0 - h * md;
  const int64_t col = c0 + lane * CPL;
  const bool live = col < K;
  const int64_t cld = BITS == 8 ? K : K / 2;
  const int rpw = RT / NWARP;  // consecutive rows of this warp
  const int rw0 = warp * rpw;
  const uint8_t* cp = codes != nullptr && live && (LB >= 4 || (lane & 1) == 0)
                          ? codes + (r0 + rw0) * cld + (BITS == 8 ? col : col / 2)
                          : nullptr;
  const int nb = rpw / MF_UN;
  // batch i of this warp's rows into ring slot i % MF_SLOTS; every lane commits a (possibly empty) group
  auto issue = [&](int i) {
    if (cp != nullptr && i < nb) {
      const uint32_t slot = ring + static_cast<uint32_t>((i % MF_SLOTS) * SLOT + lane * LB);
#pragma unroll
      for (int u = 0; u < MF_UN; ++u) cp_async_ca<CB>(slot + u * 32 * LB, cp + (static_cast<int64_t>(i) * MF_UN + u) * cld);
    }
    cp_async_commit();
  };
  // Prologue, one round trip: Gd[:, i] / scale / offset / G2[:, h] as cp.async copies (committed first), the
  // first code batches behind them, and this thread's G1 rows in registers, all in flight at once.
#pragma unroll
  for (int b = 0; b < R; ++b)  // coalesced along the rows of Gd
    for (int rl = threadIdx.x; rl < RT; rl += MF_THREADS)
      cp_async_ca<4>(smem_u32(gs + rl * R + b), Gd + static_cast<int64_t>(b) * md + i0 + rl);
  for (int rl = threadIdx.x; rl < RT; rl += MF_THREADS) {
    if (codes != nullptr) {
      cp_async_ca<4>(smem_u32(so + 2 * rl), scale + r0 + rl);
      cp_async_ca<4>(smem_u32(so + 2 * rl + 1), offset + r0 + rl);
    } else {
      *reinterpret_cast<float2*>(so + 2 * rl) = make_float2(0.f, 0.f);
    }
  }
  if (D3)
    for (int q = threadIdx.x; q < R1 * J1 * R; q += MF_THREADS) {
      const int a = q / (J1 * R), rem = q - a * J1 * R;
      cp_async_ca<4>(smem_u32(g2s + q), G2 + (static_cast<int64_t>(a) * H + h) * J1 * R + rem);
    }
  cp_async_commit();
#pragma unroll
  for (int i = 0; i < MF_SLOTS - 1; ++i) issue(i);
  // G1 rows of this thread's L columns (one thread per column; R1 <= 16 values each for d = 3, R for d = 2)
  constexpr int NCT = COLS / MF_THREADS;
  constexpr int G1N = D3 ? 16 : R;
  float g1v[NCT][G1N];
  int j1c[NCT];
#pragma unroll
  for (int k = 0; k < NCT; ++k) {
    const int cl = static_cast<int>(threadIdx.x) + k * MF_THREADS;
    const int64_t cc = c0 + cl < K ? c0 + cl : 0;
    if (D3) {
      const int64_t j0 = cc / J1;
      j1c[k] = static_cast<int>(cc - j0 * J1);
#pragma unroll
      for (int a = 0; a < G1N; ++a) g1v[k][a] = a < R1 ? __ldg(G1 + j0 * R1 + a) : 0.f;
    } else {
      j1c[k] = 0;
#pragma unroll
      for (int b = 0; b < G1N; ++b) g1v[k][b] = __ldg(G1 + cc * R + b);
    }
  }
  cp_async_wait<MF_SLOTS - 1>();  // the prologue group (the code batches may still be in flight)
  __syncthreads();
  // L for the tile's columns, every rank index (same summation order as the prefix)
#pragma unroll
  for (int k = 0; k < NCT; ++k) {
    const int cl = static_cast<int>(threadIdx.x) + k * MF_THREADS;
    float acc[R];
    if (D3) {
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] = 0.f;
#pragma unroll
      for (int a = 0; a < G1N; ++a) {
        if (a >= R1) break;
        const float4* g2 = reinterpret_cast<const float4*>(g2s + (a * J1 + j1c[k]) * R);
#pragma unroll
        for (int b4 = 0; b4 < R / 4; ++b4) {
          const float4 t = g2[b4];
          acc[4 * b4] = fmaf(g1v[k][a], t.x, acc[4 * b4]);
          acc[4 * b4 + 1] = fmaf(g1v[k][a], t.y, acc[4 * b4 + 1]);
          acc[4 * b4 + 2] = fmaf(g1v[k][a], t.z, acc[4 * b4 + 2]);
          acc[4 * b4 + 3] = fmaf(g1v[k][a], t.w, acc[4 * b4 + 3]);
        }
      }
    } else {
#pragma unroll
      for (int b = 0; b < R; ++b) acc[b] = g1v[k][b];
    }
#pragma unroll
    for (int b = 0; b < R; b += 4)
      *reinterpret_cast<float4*>(ls + cl * R + b) = make_float4(acc[b], acc[b + 1], acc[b + 2], acc[b + 3]);
  }
  __syncthreads();
  const unsigned live_mask = __ballot_sync(0xffffffffu, live);
  if (!live) return;
  // the lane's CPL columns as column pairs per rank: lp[b][p] = (col + 2p, col + 2p + 1)
  unsigned long long lp[R][NP];
#pragma unroll
  for (int p = 0; p < NP; ++p)
#pragma unroll
    for (int b4 = 0; b4 < R / 4; ++b4) {
      const float4 u = *reinterpret_cast<const float4*>(ls + (lane * CPL + 2 * p) * R + 4 * b4);
      const float4 v = *reinterpret_cast<const float4*>(ls + (lane * CPL + 2 * p + 1) * R + 4 * b4);
      lp[4 * b4][p] = f2pack(u.x, v.x);
      lp[4 * b4 + 1][p] = f2pack(u.y, v.y);
      lp[4 * b4 + 2][p] = f2pack(u.z, v.z);
      lp[4 * b4 + 3][p] = f2pack(u.w, v.w);
    }
  OutT* dst = out + (r0 + rw0) * K + col;
  const unsigned long long nm2 = f2pack(-8388608.f, -8388608.f);
  for (int bi = 0; bi < nb; ++bi) {
    issue(bi + MF_SLOTS - 1);
    cp_async_wait<MF_SLOTS - 1>();
    if (LB < 4) __syncwarp(live_mask);  // the pair's bytes were copied by the even lane
    const int rb = bi * MF_UN;
    const uint32_t slot = ring + static_cast<uint32_t>((bi % MF_SLOTS) * SLOT + lane * LB);
    uint32_t cw[MF_UN][NW];
#pragma unroll
    for (int u = 0; u < MF_UN; ++u) {
      if (codes == nullptr) {
        cw[u][0] = 0u;
        if (NW == 2) cw[u][NW - 1] = 0u;
      } else if constexpr (LB == 8) {
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(cw[u][0]), "=r"(cw[u][NW - 1]) : "r"(slot + u * 32 * LB));
      } else if constexpr (LB == 4) {
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(cw[u][0]) : "r"(slot + u * 32 * LB));
      } else {
        uint16_t v;
        asm volatile("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(slot + u * 32 * LB));
        cw[u][0] = v;
      }
    }
#pragma unroll
    for (int u = 0; u < MF_UN; ++u) {
      const int rl = rw0 + rb + u;
      const float2 sv = *reinterpret_cast<const float2*>(so + 2 * rl);
      const unsigned long long sc2 = f2pack(sv.x, sv.x), of2 = f2pack(sv.y, sv.y);
      // codes of column 2p in `ev` byte p, of column 2p + 1 in `od` byte p
      uint32_t ev[NW], od[NW];
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        if (BITS == 8) {
          ev[q] = __byte_perm(cw[u][q], 0u, 0x4420);
          od[q] = __byte_perm(cw[u][q], 0u, 0x4431);
        } else {
          ev[q] = cw[u][q] & 0x0F0F0F0Fu;
          od[q] = (cw[u][q] >> 4) & 0x0F0F0F0Fu;
        }
      }
      unsigned long long acc[NP];
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        constexpr int kPerWord = BITS == 8 ? 2 : 4;  // column pairs per code word
        const int q = p / kPerWord, byte = p % kPerWord;
        const uint32_t e = __byte_perm(ev[q], 0x4B000000u, 0x7650 + byte);
        const uint32_t o = __byte_perm(od[q], 0x4B000000u, 0x7650 + byte);
        acc[p] = ffma2r(fadd2(f2pack(__uint_as_float(e), __uint_as_float(o)), nm2), sc2, of2);
      }
      const float4* gr = reinterpret_cast<const float4*>(gs + rl * R);
#pragma unroll
      for (int b4 = 0; b4 < R / 4; ++b4) {
        const float4 g = gr[b4];
        const float gg[4] = {g.x, g.y, g.z, g.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const unsigned long long g2 = f2pack(gg[e], gg[e]);
#pragma unroll
          for (int p = 0; p < NP; ++p) ffma2(acc[p], g2, lp[4 * b4 + e][p]);
        }
      }
      OutT* d = dst + static_cast<int64_t>(rb + u) * K;
      if constexpr (sizeof(OutT) == 2) {
        uint32_t pk[NP];
#pragma unroll
        for (int p = 0; p < NP; ++p) {
          const __nv_bfloat162 t = __floats2bfloat162_rn(f2lo(acc[p]), f2hi(acc[p]));
          pk[p] = *reinterpret_cast<const uint32_t*>(&t);
        }
        if constexpr (NP == 4)
          *reinterpret_cast<uint4*>(d) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        else
          *reinterpret_cast<uint2*>(d) = make_uint2(pk[0], pk[1]);
      } else {
#pragma unroll
        for (int p = 0; p < NP; p += 2)
          *reinterpret_cast<float4*>(d + 2 * p) =
              make_float4(f2lo(acc[p]), f2hi(acc[p]), f2lo(acc[p + 1]), f2hi(acc[p + 1]));
      }
    }
    if (LB < 4) __syncwarp(live_mask);  // before the even lane refills the slot its pair has just read
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
  if (dd.d == 3 && dd.m[0] == 1 && (R == 8 || R == 16) && dd.r[1] == R && dd.n[1] <= 16) {
    // pinned 3-core modes: a tiny GEMM per (h, j2) with G2[:, h, :, :] in shared memory
    const dim3 grid(static_cast<unsigned>((JP + 255) / 256), static_cast<unsigned>(IP));
    if (R == 8)
      k_prefix_d3<8><<<grid, 256, 0, s>>>(cores[0], cores[1], L, static_cast<int>(IP), dd.n[1], JP);
    else
      k_prefix_d3<16><<<grid, 256, 0, s>>>(cores[0], cores[1], L, static_cast<int>(IP), dd.n[1], JP);
  } else if (R <= 16) {  // one thread per (ip, jp): the whole rank vector at once
    const int64_t pairs = IP * JP;
    k_prefix_vec<<<static_cast<unsigned>((pairs + 127) / 128), 128, 0, s>>>(dd, cp, L, IP, JP, R);
  } else {
    k_prefix_full<<<static_cast<unsigned>((total + 127) / 128), 128, 0, s>>>(dd, cp, L, IP, JP, R);
  }
  return cudaGetLastError();
}

bool merge_fast_ok(const TTDims& dd, const void* codes, const void* out) {
  const int d = dd.d;
  if ((d != 2 && d != 3) || dd.m[0] != 1 || dd.n[d - 1] != 1) return false;
  const int R = dd.r[d - 1];
  const int64_t md = dd.m[d - 1];
  if ((R != 8 && R != 16) || md % 64 != 0 || dd.K % 8 != 0) return false;
  if (d == 3 && (dd.r[1] > 16 || dd.n[1] > 16)) return false;
  return reinterpret_cast<uintptr_t>(out) % 16 == 0 && (codes == nullptr || reinterpret_cast<uintptr_t>(codes) % 8 == 0);
}

cudaError_t launch_merge_fast(const TTDims& dd, const float* const* cores, const uint8_t* codes, int bits,
                              const float* scale, const float* offset, void* out, int out_dtype, cudaStream_t s) {
  const int d = dd.d;
  const int R = dd.r[d - 1];
  const int64_t md = dd.m[d - 1];
  const int cols = R == 8 ? mf_cols<8>() : mf_cols<16>();
  const int64_t ctiles = (dd.K + cols - 1) / cols;
  // 256-row tiles: the per-CTA prologue (L for the tile's columns) amortised over more rows; 64-row tiles
  // (more CTAs for the 1024-row k / v matrices) measured slower even where 256 leaves SMs idle
  const int RT = md % 256 == 0 ? 256 : 64;
  const int R1 = d == 3 ? dd.r[1] : 0, J1 = d == 3 ? dd.n[1] : 1, H = d == 3 ? dd.m[1] : 1;
  const int64_t total = dd.N * dd.K;
  LaunchScope scope(kMerge, double(total) * ((codes ? (bits == 8 ? 1.0 : 0.5) : 0.0) + (out_dtype == QA_F32 ? 4 : 2)), s);
  count_launches(1);
  const dim3 grid(static_cast<unsigned>(ctiles), static_cast<unsigned>(dd.N / RT));
  const size_t smem =
      sizeof(float) * (static_cast<size_t>(RT) * R + static_cast<size_t>(cols) * R + 2 * RT +
                       static_cast<size_t>(R1) * J1 * R) +
      static_cast<size_t>(MF_THREADS / 32) * MF_SLOTS * MF_UN * 32 * (cols / 32) * bits / 8;
  const float* G1 = cores[0];
  const float* G2 = d == 3 ? cores[1] : nullptr;
  const float* Gd = cores[d - 1];
#define QA_MF(OT, BB, RR, DD)                                                                                     \
  {                                                                                                              \
    cudaFuncSetAttribute(k_merge_fast<OT, BB, RR, DD>, cudaFuncAttributeMaxDynamicSharedMemorySize,                 \
                         static_cast<int>(smem));                                                                   \
    k_merge_fast<OT, BB, RR, DD><<<grid, MF_THREADS, smem, s>>>(G1, G2, Gd, R1, J1, H, md, dd.N, dd.K, RT, codes,   \
                                                               scale, offset, static_cast<OT*>(out));              \
  }
#define QA_MF_D(OT, BB, RR) \
  if (d == 3)               \
    QA_MF(OT, BB, RR, true)  \
  else                      \
    QA_MF(OT, BB, RR, false)
#define QA_MF_R(OT, BB) \
  if (R == 8) {         \
    QA_MF_D(OT, BB, 8)  \
  } else {              \
    QA_MF_D(OT, BB, 16) \
  }
  if (out_dtype == QA_F32) {
    if (bits == 4) {
      QA_MF_R(float, 4)
    } else {
      QA_MF_R(float, 8)
    }
  } else {
    if (bits == 4) {
      QA_MF_R(__nv_bfloat16, 4)
    } else {
      QA_MF_R(__nv_bfloat16, 8)
    }
  }
#undef QA_MF_R
#undef QA_MF_D
#undef QA_MF
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
  const int R = dd.r[last];
  const int64_t md = dd.m[last];
  const int mg_rows = md % 256 == 0 ? 256 : (md % 64 == 0 ? 64 : 0);
  const bool nd1 = dd.n[last] == 1 && mg_rows > 0 && dd.K % 32 == 0 && (R == 8 || R == 16) &&
                   reinterpret_cast<uintptr_t>(out) % 16 == 0 && reinterpret_cast<uintptr_t>(L) % 16 == 0 &&
                   (codes == nullptr || reinterpret_cast<uintptr_t>(codes) % 8 == 0);
  if (nd1) {
    const dim3 grid(static_cast<unsigned>((dd.K + MG_COLS - 1) / MG_COLS), static_cast<unsigned>(dd.N / mg_rows));
#define QA_MG(OT, BB, RR)                                                                                        \
  {                                                                                                              \
    const size_t smem = codes != nullptr ? static_cast<size_t>(mg_rows) * MG_COLS * BB / 8 : 0;                 \
    cudaFuncSetAttribute(k_merge_nd1<OT, BB, RR>, cudaFuncAttributeMaxDynamicSharedMemorySize,                    \
                         static_cast<int>(smem));                                                                 \
    k_merge_nd1<OT, BB, RR><<<grid, 256, smem, s>>>(L, Gd, md, dd.N, dd.K, mg_rows, codes, scale, offset,         \
                                                   static_cast<OT*>(out));                                        \
  }
#define QA_MG_R(OT, BB) \
  if (R == 8)           \
    QA_MG(OT, BB, 8)    \
  else                  \
    QA_MG(OT, BB, 16)
    if (out_dtype == QA_F32) {
      if (bits == 4) {
        QA_MG_R(float, 4)
      } else {
        QA_MG_R(float, 8)
      }
    } else {
      if (bits == 4) {
        QA_MG_R(__nv_bfloat16, 4)
      } else {
        QA_MG_R(__nv_bfloat16, 8)
      }
    }
#undef QA_MG_R
#undef QA_MG
    return cudaGetLastError();
  }
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

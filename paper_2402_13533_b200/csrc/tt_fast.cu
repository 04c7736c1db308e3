// Fast path for the tensor-train adapters whose first core is input-only and last core is
// output-only (m_1 = 1, n_d = 1; d = 2 is LoRA, d = 3 is the pinned Llama modes
// m = (1, N/256, 256), n = (K/4, 4, 1)).  With that shape every contraction that touches a
// big tensor has a small rank side, so each is a single streaming pass:
//
//   forward  x-pass  : act-quant codes + Z1[t, a, J] = Σ_j1 x[t, j1, J] G1[j1, a]  (one read of x)
//                      y2 = Z1 · Vᵀ runs inside the int8 GEMM as bf16 extension k-blocks, with
//                      V[n, (a, J)] the contraction of cores 2..d (k_build_v)
//   backward dy-pass : dZ_{d-1} = dy · G_dᵀ and dG_d = Σ Z_{d-1}ᵀ dy (warp-level bf16 MMA, one read of dy)
//            x-pass  : dG1 = Σ_t x ⊗ dZ1 (one read of x); dx_adapter = dZ1 · B_extᵀ as extension
//                      k-blocks of the dX GEMM (k_build_bext)
// Middle-core work is per-token and tiny (generic kernels in tt_kernels.cu).
#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_timing.h"
#include "quant_row.cuh"

namespace qa {

namespace {

// Sum of 32 per-lane values across the warp; afterwards lane l holds the total of value l.
template <int NV>
QA_DEV void warp_reduce_scatter32(float (&z)[NV], int base) {
  const uint32_t lane = lane_id();
#pragma unroll
  for (int o = 16, half = 16; o > 0; o >>= 1, half >>= 1) {
    const bool up = lane & o;
#pragma unroll
    for (int i = 0; i < half; ++i) {
      const float send = up ? z[base + i] : z[base + i + half];
      const float keep = up ? z[base + i + half] : z[base + i];
      z[base + i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Per-token act-quant (bit-exact, quant.py:73-99) fused with the first TT stage.
// One warp per token row (lane l takes the 8-element chunks l, l + 32, ...), so a warp's row
// (<= 22 KB) stays L1/L2-resident between the stats pass and the codes pass.  The G1 rows a chunk
// needs (8 R1 / J1 floats) come from an interleaved copy G1i[c / 32][q][c % 32] (float4), so each
// warp-wide G1 load is one contiguous 512-byte line.  Vector path only (K % 8 == 0, aligned rows).
template <int J1, int R1>
__global__ void __launch_bounds__(256) k_g1_interleave(const float* __restrict__ G1, float4* __restrict__ G1i,
                                                       int64_t nvec) {
  constexpr int NQ = 2 * R1 / J1;  // float4 pieces per 8-element chunk
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= nvec * NQ) return;
  const int64_t c = idx / NQ;
  const int q = static_cast<int>(idx % NQ);
  const float* src = G1 + c * (8 / J1) * R1 + 4 * q;
  G1i[((c / 32) * NQ + q) * 32 + (c % 32)] = make_float4(src[0], src[1], src[2], src[3]);
}

template <typename InT, int J1, int R1, bool CODES>
__global__ void __launch_bounds__(256, 2) k_actquant_z1(const InT* __restrict__ x, int64_t T, int64_t K,
                                                     uint8_t* __restrict__ codes, int64_t ldc,
                                                     float* __restrict__ sx, float* __restrict__ ox,
                                                     int32_t* __restrict__ rsx, const float4* __restrict__ G1i,
                                                     __nv_bfloat16* __restrict__ zb, int64_t ldzb,
                                                     float* __restrict__ zf) {
  constexpr int K2 = J1 * R1;
  static_assert(K2 == 8 || K2 == 16 || K2 == 32 || K2 == 64, "unsupported Z1 width");
  constexpr int NQ = 2 * R1 / J1;
  constexpr int RP = R1 / 2;  // rank pairs: Z1 accumulates with packed fp32 FMAs (FFMA2)
  constexpr bool BF = sizeof(InT) == 2;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (row >= T) return;
  const uint32_t lane = lane_id();
  const InT* src = x + row * K;
  const int64_t nvec = K / 8;

  unsigned long long zz[J1][RP];  // zz[J][p] = (z[2p, J], z[2p+1, J])
#pragma unroll
  for (int J = 0; J < J1; ++J)
#pragma unroll
    for (int p = 0; p < RP; ++p) zz[J][p] = 0ull;
  float lo = INFINITY, hi = -INFINITY;
  __nv_bfloat162 lo2 = __floats2bfloat162_rn(INFINITY, INFINITY), hi2 = __floats2bfloat162_rn(-INFINITY, -INFINITY);
  constexpr int UNR = 4;  // chunks per batch; the next batch's loads are in flight while this one computes
  uint4 nxt[UNR];
  if (BF) {
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t c = u * 32 + lane;
      if (c < nvec) nxt[u] = __ldg(reinterpret_cast<const uint4*>(src + c * 8));
    }
  }
  for (int64_t i0 = 0; i0 * 32 + lane < nvec; i0 += UNR) {
    float f[UNR][8];
    uint4 raw[UNR];
    if (BF) {
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        raw[u] = nxt[u];
        const int64_t c = (i0 + UNR + u) * 32 + lane;
        if (c < nvec) nxt[u] = __ldg(reinterpret_cast<const uint4*>(src + c * 8));
      }
    } else {
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t c = (i0 + u) * 32 + lane;
        if (c < nvec) load8<InT>(src + c * 8, f[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < UNR; ++u) {
      const int64_t c = (i0 + u) * 32 + lane;
      if (c >= nvec) break;
      if (BF) {
        const uint32_t w[4] = {raw[u].x, raw[u].y, raw[u].z, raw[u].w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
          lo2 = __hmin2(lo2, b2);
          hi2 = __hmax2(hi2, b2);
          f[u][2 * i] = __uint_as_float(w[i] << 16);
          f[u][2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          lo = fminf(lo, f[u][i]);
          hi = fmaxf(hi, f[u][i]);
        }
      }
      unsigned long long g2[2 * NQ];  // [8 / J1 rows][RP] rank pairs of G1
      const float4* gp = G1i + ((i0 + u) * NQ) * 32 + lane;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const float4 v = __ldg(gp + q * 32);
        g2[2 * q] = f2pack(v.x, v.y);
        g2[2 * q + 1] = f2pack(v.z, v.w);
      }
#pragma unroll
      for (int jj = 0; jj < 8 / J1; ++jj)
#pragma unroll
        for (int J = 0; J < J1; ++J) {
          const float xv = f[u][jj * J1 + J];
          const unsigned long long xb = f2pack(xv, xv);
#pragma unroll
          for (int p = 0; p < RP; ++p) ffma2(zz[J][p], xb, g2[jj * RP + p]);
        }
    }
  }
  if (BF) {
    lo = fminf(__low2float(lo2), __high2float(lo2));
    hi = fmaxf(__low2float(hi2), __high2float(hi2));
  }
  float z[K2];  // z[a * J1 + J]
#pragma unroll
  for (int J = 0; J < J1; ++J)
#pragma unroll
    for (int p = 0; p < RP; ++p) {
      z[(2 * p) * J1 + J] = f2lo(zz[J][p]);
      z[(2 * p + 1) * J1 + J] = f2hi(zz[J][p]);
    }
  // Z1 row: reduce across lanes, write fp32 and/or the 3-term bf16 split [hi | lo | hi | 0]
  if (K2 >= 32) {
#pragma unroll
    for (int b = 0; b < K2; b += 32) warp_reduce_scatter32<K2>(z, b);
#pragma unroll
    for (int b = 0; b < K2; b += 32) {
      const float v = z[b];
      if (zf != nullptr) zf[row * K2 + b + lane] = v;
      if (zb != nullptr) {
        const __nv_bfloat16 hv = __float2bfloat16_rn(v);
        zb[row * ldzb + b + lane] = hv;
        zb[row * ldzb + K2 + b + lane] = __float2bfloat16_rn(v - __bfloat162float(hv));
        zb[row * ldzb + 2 * K2 + b + lane] = hv;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < K2; ++i) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) z[i] += __shfl_xor_sync(0xffffffffu, z[i], o);
    }
#pragma unroll
    for (int i = 0; i < K2; ++i) {
      if (lane == static_cast<uint32_t>(i)) {
        if (zf != nullptr) zf[row * K2 + i] = z[i];
        if (zb != nullptr) {
          const __nv_bfloat16 hv = __float2bfloat16_rn(z[i]);
          zb[row * ldzb + i] = hv;
          zb[row * ldzb + K2 + i] = __float2bfloat16_rn(z[i] - __bfloat162float(hv));
          zb[row * ldzb + 2 * K2 + i] = hv;
        }
      }
    }
  }
  if (zb != nullptr)
    for (int64_t i = 3 * K2 + lane; i < ldzb; i += 32) zb[row * ldzb + i] = __float2bfloat16_rn(0.f);
  if constexpr (CODES) {
    lo = warp_min(lo);
    hi = warp_max(hi);
    const double lo64 = static_cast<double>(lo);
    const double step64 = __ddiv_rn(__dsub_rn(static_cast<double>(hi), lo64), 255.0);
    const bool flat = !(step64 > 0.0);
    const float inv = flat ? 0.0f : static_cast<float>(1.0 / step64);
    uint8_t* dst = codes + row * ldc;
    int sum = 0;
    for (int64_t i0 = 0; i0 * 32 + lane < nvec; i0 += UNR) {
      float f[UNR][8];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t c = (i0 + u) * 32 + lane;
        if (c < nvec) load8<InT>(src + c * 8, f[u]);
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        const int64_t c = (i0 + u) * 32 + lane;
        if (c >= nvec) break;
        uint2 packed = make_uint2(0u, 0u);
        if (!flat) codes8(f[u], lo, inv, lo64, step64, packed.x, packed.y, sum);
        *reinterpret_cast<uint2*>(dst + c * 8) = packed;
      }
    }
    for (int64_t k = K + lane; k < ldc; k += 32) dst[k] = 0;
    sum = warp_sum_i(sum);
    if (lane == 0) {
      sx[row] = flat ? 0.0f : __double2float_rn(step64);
      ox[row] = lo;
      rsx[row] = sum;
    }
  }
}

// ---------------------------------------------------------------------------------------------
// Tensor-core act-quant + Z1 (production path for bf16 rows, J1 in {1, 4}).
// A CTA of 4 warps owns a tile of TOK token rows staged in shared memory by cp.async.bulk (one
// copy per row, rows padded so the fragment loads below are bank-conflict free).
//   pass 1: Z1 on the tensor cores.  Per J, Z1[:, :, J] = X_J · G1 with X_J[t, j1] = x[t, j1 J1 + J]
//           is an (R1 x 8 tokens) mma.sync m16n8k16 tile: A = [G1_hi | G1_lo]ᵀ (the fp32 core
//           split into two bf16 terms; x is exact in bf16, products are exact, accumulation fp32),
//           B = the x row read straight from shared memory (J1 = 4: one PRMT per pair of x words
//           regroups (j1, j1 + 1) of the same J).  The k-steps are strided over the 4 warps, which
//           also take the exact bf16 min/max of what they read; partials meet in shared memory
//           and are summed in fixed warp order (deterministic).
//   pass 2: per-token codes (reference rule, bit-exact) from the same shared-memory rows.
// G1 reaches the MMAs as pre-built fragments (k_g1_frag): one 16-byte load per lane per k-step.
template <int J1, int R1>
QA_DEV void g1_frag_at(const float* __restrict__ G1, uint4* __restrict__ frag, int64_t nsteps, int64_t idx) {
  constexpr int MT = R1 / 8;  // m16 tiles: R1 = 8 -> rows (hi a | lo a); R1 = 16 -> tile 0 hi, tile 1 lo
  if (idx >= nsteps * MT * 32) return;
  const int lane = static_cast<int>(idx % 32), mt = static_cast<int>((idx / 32) % MT);
  const int64_t s = idx / (32 * MT);
  const int g = lane >> 2, c = lane & 3;
  uint32_t w[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int m = g + 8 * (q & 1);  // a0a1: (g, 2c), a2a3: (g+8, 2c), a4a5: (g, 2c+8), a6a7: (g+8, 2c+8)
    const int term = R1 == 8 ? (m >> 3) : mt;
    const int a = R1 == 8 ? (m & 7) : m;
    uint32_t packed = 0;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int kk = 2 * c + 8 * (q >> 1) + e;
      int64_t j;
      if (J1 == 4) {
        j = 16 * s + kk;
      } else {  // LoRA: MMA u of super-step S reads x[64 S + 16 c' + 4 u + {0,1}] (b0) and {2,3} (b1)
        const int64_t S = s >> 2;
        const int u = static_cast<int>(s & 3);
        j = 64 * S + 16 * ((kk & 7) >> 1) + 4 * u + 2 * (kk >> 3) + (kk & 1);
      }
      const float v = G1[j * R1 + a];
      const __nv_bfloat16 hv = __float2bfloat16_rn(v);
      const __nv_bfloat16 t = term == 0 ? hv : __float2bfloat16_rn(v - __bfloat162float(hv));
      packed |= static_cast<uint32_t>(__bfloat16_as_ushort(t)) << (16 * e);
    }
    w[q] = packed;
  }
  frag[idx] = make_uint4(w[0], w[1], w[2], w[3]);
}

template <int J1, int R1>
__global__ void __launch_bounds__(256) k_g1_frag(const float* __restrict__ G1, uint4* __restrict__ frag,
                                                 int64_t nsteps) {
  g1_frag_at<J1, R1>(G1, frag, nsteps, static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
}

// Per-row constants of the act-quant rule for the byte-grid code path below.
struct AqRow {
  float lo, inv, nbh;   // nbh = 1/2 - lo * inv
  double lo64, step64;  // the reference's fp64 quantities (tie replays)
};

// Bracketed codes of 8 elements: t = q' + 1/2 is evaluated twice, with the addend shifted by
// -kTieBand and +kTieBand, and each is floored onto the integer grid by a round-down magic add
// (byte 1 of M + t, M = 1.5 * 2^15).  Outside the band both floors agree and equal the reference's
// code (the fp32 error of t is far below kTieBand); a byte where they differ marks an element whose
// [t - band, t + band] holds an integer — about 2 * kTieBand of all elements — and is replayed in
// fp64 (aq_replay64).  c0/c1 = codes of elements 0..3 / 4..7, d0/d1 = nonzero bytes to replay.
template <bool SUB>
QA_DEV void aq_codes8b(const uint4 raw, unsigned long long inv2, unsigned long long alo2, unsigned long long ahi2,
                       unsigned long long nlo2, uint32_t& c0, uint32_t& c1, uint32_t& d0, uint32_t& d1) {
  const unsigned long long m2 = f2pack(49152.0f, 49152.0f);
  const uint32_t w[4] = {raw.x, raw.y, raw.z, raw.w};
  uint32_t sl[8], sh[8];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    unsigned long long v2 = f2pack(__uint_as_float(w[i] << 16), __uint_as_float(w[i] & 0xFFFF0000u));
    if constexpr (SUB) v2 = fadd2(v2, nlo2);
    const unsigned long long tl = ffma2r(v2, inv2, alo2), th = ffma2r(v2, inv2, ahi2);
    const unsigned long long l2 = fadd2rm(tl, m2), h2 = fadd2rm(th, m2);
    sl[2 * i] = static_cast<uint32_t>(l2);
    sl[2 * i + 1] = static_cast<uint32_t>(l2 >> 32);
    sh[2 * i] = static_cast<uint32_t>(h2);
    sh[2 * i + 1] = static_cast<uint32_t>(h2 >> 32);
  }
  c0 = __byte_perm(__byte_perm(sl[0], sl[1], 0x0051), __byte_perm(sl[2], sl[3], 0x0051), 0x5410);
  c1 = __byte_perm(__byte_perm(sl[4], sl[5], 0x0051), __byte_perm(sl[6], sl[7], 0x0051), 0x5410);
  d0 = c0 ^ __byte_perm(__byte_perm(sh[0], sh[1], 0x0051), __byte_perm(sh[2], sh[3], 0x0051), 0x5410);
  d1 = c1 ^ __byte_perm(__byte_perm(sh[4], sh[5], 0x0051), __byte_perm(sh[6], sh[7], 0x0051), 0x5410);
}

// The reference's code of element e (0..7) of an 8-element bf16 word, in its own fp64 arithmetic
// (quant.py:73-99: round_half_away((w - lo) / scale) clipped to [0, 255], w >= lo).
QA_DEV uint32_t aq_replay64(const uint4 raw, int e, double lo64, double step64) {
  const uint32_t wa = (e & 2) ? raw.y : raw.x, wb = (e & 2) ? raw.w : raw.z;
  const uint32_t wd = (e & 4) ? wb : wa;
  const float v = __uint_as_float((e & 1) ? (wd & 0xFFFF0000u) : (wd << 16));
  const double q = __ddiv_rn(__dsub_rn(static_cast<double>(v), lo64), step64);
  return static_cast<uint32_t>(fmin(fmax(floor(__dadd_rn(q, 0.5)), 0.0), 255.0));
}

// Replays the flagged bytes of one code word (elements e0 .. e0 + 3 of raw).
QA_DEV uint32_t aq_replay_word(const uint4 raw, int e0, uint32_t code, uint32_t d, double lo64, double step64) {
  while (d != 0u) {
    const int b = (__ffs(d) - 1) >> 3;
    d &= ~(0xFFu << (8 * b));
    code = (code & ~(0xFFu << (8 * b))) | (aq_replay64(raw, e0 + b, lo64, step64) << (8 * b));
  }
  return code;
}

// ---------------------------------------------------------------------------------------------
// CTA-per-8-token act-quant + Z1 (production path for bf16 rows, K % 64 == 0, J1 in {1, 4}).
// Nothing is staged in shared memory but the G1 fragments: a CTA of AQC_WARPS warps owns 8 token
// rows at a time and warp w takes the 64-element segments w, w + AQC_WARPS, ... of all 8 rows.
// Lane (g, c) = (lane / 4, lane % 4) reads, per segment, exactly the 16 elements of row g that the
// m16n8k16 B fragment of the Z1 MMA needs from it (J1 = 4: elements 8c..8c+7 and 32+8c..32+8c+7;
// J1 = 1: 16c..16c+15): two 16-byte loads straight from global memory, 8 rows x 64 contiguous
// bytes per warp instruction.
//   pass 1 (the one HBM read of x): Z1 partials on the tensor cores (A = [G1_hi | G1_lo] fragments,
//          k_g1_frag; B = the x words, exact in bf16) and the exact bf16 min / max, per warp.
//   reduce : partials meet in shared memory and are summed in fixed warp order (deterministic).
//   pass 2 : codes by the byte-grid rule (aq_codes8b, bit-exact with quant.py:73-99) from a second
//            read of the same 64-byte pieces by the same warp — a CTA's live rows are 8 x 2K bytes,
//            so the re-read is served by L1 / L2, not HBM.  Bracketed elements (aq_codes8b) are
//            replayed in fp64 in place.
// Splitting the row over the CTA's warps keeps the live footprint per in-flight byte small (the
// whole row must be seen before its first code), so many CTAs per SM can stream at once.
#ifndef QA_AQC_UNROLL
#define QA_AQC_UNROLL 4
#endif
constexpr int AQC_WARPS = 8, AQC_UNROLL = QA_AQC_UNROLL;

struct AqAdapters {  // per-adapter outputs of the shared x pass (unused entries null)
  __nv_bfloat16* zb[3];
  float* zf[3];
  int64_t frag_stride;  // uint4 elements between adapters' G1 fragments
};

template <int J1>
QA_DEV void aqc_offsets(uint32_t c, uint32_t& off0, uint32_t& off1) {
  off0 = J1 == 4 ? 16u * c : 32u * c;
  off1 = J1 == 4 ? 64u + 16u * c : 32u * c + 16u;
}

// Codes of one lane's two 8-element words of segment st (bracketed rule, aq_codes8b); writes them
// and returns their Σ.
template <int J1, bool SUB>
QA_DEV uint32_t aqc_codes_seg(const uint4 p0, const uint4 p1, unsigned long long inv2, unsigned long long alo2,
                              unsigned long long ahi2, unsigned long long nlo2, double lo64, double step64, bool flat,
                              uint8_t* dst, bool store) {
  uint32_t cw[4], dw[4];
  aq_codes8b<SUB>(p0, inv2, alo2, ahi2, nlo2, cw[0], cw[1], dw[0], dw[1]);
  aq_codes8b<SUB>(p1, inv2, alo2, ahi2, nlo2, cw[2], cw[3], dw[2], dw[3]);
  if (flat) cw[0] = cw[1] = cw[2] = cw[3] = dw[0] = dw[1] = dw[2] = dw[3] = 0u;
  if ((dw[0] | dw[1] | dw[2] | dw[3]) != 0u) {
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (dw[k] != 0u) cw[k] = aq_replay_word(k < 2 ? p0 : p1, (k & 1) * 4, cw[k], dw[k], lo64, step64);
  }
  if (store) {
    if constexpr (J1 == 4) {
      *reinterpret_cast<uint2*>(dst) = make_uint2(cw[0], cw[1]);
      *reinterpret_cast<uint2*>(dst + 32) = make_uint2(cw[2], cw[3]);
    } else {
      *reinterpret_cast<uint4*>(dst) = make_uint4(cw[0], cw[1], cw[2], cw[3]);
    }
  }
  return __dp4a(cw[0], 0x01010101u, __dp4a(cw[1], 0x01010101u, __dp4a(cw[2], 0x01010101u, __dp4a(cw[3], 0x01010101u, 0u))));
}

template <int J1, bool SUB>
QA_DEV uint32_t aqc_codes_row(const uint8_t* xrow, uint8_t* crow, int64_t nseg, uint32_t warp, uint32_t off0,
                              uint32_t off1, const AqRow& r, bool flat, bool store) {
  const unsigned long long inv2 = f2pack(r.inv, r.inv), nlo2 = f2pack(-r.lo, -r.lo);
  const float alo = SUB ? 0.5f - kTieBand : r.nbh - kTieBand, ahi = SUB ? 0.5f + kTieBand : r.nbh + kTieBand;
  const unsigned long long alo2 = f2pack(alo, alo), ahi2 = f2pack(ahi, ahi);
  uint32_t sum = 0;
  // this warp's segments warp + i W, i < n, visited last-first: pass 1 read them first-first, so the most
  // recently loaded (likeliest still in L2) come first when rows are long (K = 11008: 8 rows x 22 KB per CTA)
  const int64_t n = nseg > static_cast<int64_t>(warp) ? (nseg - warp + AQC_WARPS - 1) / AQC_WARPS : 0;
  int64_t i = n - 1;
  for (; i >= AQC_UNROLL - 1; i -= AQC_UNROLL) {
    uint4 p[AQC_UNROLL][2];
#pragma unroll
    for (int u = 0; u < AQC_UNROLL; ++u) {
      const int64_t st = warp + (i - u) * AQC_WARPS;
      p[u][0] = __ldg(reinterpret_cast<const uint4*>(xrow + 128 * st + off0));
      p[u][1] = __ldg(reinterpret_cast<const uint4*>(xrow + 128 * st + off1));
    }
#pragma unroll
    for (int u = 0; u < AQC_UNROLL; ++u) {
      const int64_t st = warp + (i - u) * AQC_WARPS;
      sum += aqc_codes_seg<J1, SUB>(p[u][0], p[u][1], inv2, alo2, ahi2, nlo2, r.lo64, r.step64, flat,
                                    crow + 64 * st + off0 / 2, store);
    }
  }
  for (; i >= 0; --i) {
    const int64_t st = warp + i * AQC_WARPS;
    const uint4 p0 = __ldg(reinterpret_cast<const uint4*>(xrow + 128 * st + off0));
    const uint4 p1 = __ldg(reinterpret_cast<const uint4*>(xrow + 128 * st + off1));
    sum += aqc_codes_seg<J1, SUB>(p0, p1, inv2, alo2, ahi2, nlo2, r.lo64, r.step64, flat, crow + 64 * st + off0 / 2,
                                  store);
  }
  return sum;
}

#ifndef QA_AQC_MINB
#define QA_AQC_MINB 3  // <= 85 registers: 3 CTAs (24 warps) per SM; measured best of {1, 3, 4}
#endif
#ifndef QA_AQC_MINB_GROUP
#define QA_AQC_MINB_GROUP 2  // NA = 2, 3 adapters sharing x: NA sets of Z1 accumulators need <= 128 registers
#endif
// NA adapters share the pass over x (the q / k / v or up / gate linears of a decoder layer read the
// same input, transformer.py:862-874): one set of codes, NA sets of Z1 (fragments of adapter a at
// frag + a * ad.frag_stride).
template <int J1, int R1, bool CODES, bool FRAG_SMEM, int NA = 1>
__global__ void __launch_bounds__(AQC_WARPS * 32, NA == 1 ? QA_AQC_MINB : QA_AQC_MINB_GROUP) k_aq_cta(const __nv_bfloat16* __restrict__ x, int64_t T, int64_t K,
                                                            uint8_t* __restrict__ codes, int64_t ldc,
                                                            float* __restrict__ sx, float* __restrict__ ox,
                                                            int32_t* __restrict__ rsx, const uint4* __restrict__ frag_g,
                                                            const AqAdapters ad, int64_t ldzb) {
  static_assert(J1 == 1 || J1 == 4, "J1");
  static_assert(R1 == 8 || R1 == 16, "R1");
  constexpr int K2 = J1 * R1, MT = R1 / 8, NJ = J1 == 4 ? 4 : 1, W = AQC_WARPS;
  constexpr int FPS = (J1 == 4 ? 1 : 4) * MT;  // fragments (one uint4 per lane) per 64-element segment
  extern __shared__ uint4 s_frag[];
  __shared__ float s_z[W][8][NA * K2];
  __shared__ float s_lo[W][8], s_hi[W][8];
  __shared__ int32_t s_sum[W][8];
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id(), g = lane >> 2, c = lane & 3;
  const int64_t nseg = K / 64;
  if constexpr (FRAG_SMEM) {
    const int64_t n = nseg * FPS * 32;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s_frag[i] = frag_g[i];  // NA == 1 only
    __syncthreads();
  }
  const uint4* frag = FRAG_SMEM ? s_frag : frag_g;
  uint32_t off0, off1;
  aqc_offsets<J1>(c, off0, off1);
  const int64_t ngroups = (T + 7) / 8;
  for (int64_t grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
    const int64_t t0 = grp * 8;
    const bool valid = t0 + g < T;
    const int64_t trow = valid ? t0 + g : T - 1;  // rows past T are computed on a clamped row, never stored
    const uint8_t* xrow = reinterpret_cast<const uint8_t*>(x + trow * K);
    // ---- pass 1: Z1 partial + exact min / max over this warp's segments
    float acc[NA][NJ][MT][4];
#pragma unroll
    for (int aa = 0; aa < NA; ++aa)
#pragma unroll
      for (int J = 0; J < NJ; ++J)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int i = 0; i < 4; ++i) acc[aa][J][mt][i] = 0.f;
    __nv_bfloat162 lo2 = __floats2bfloat162_rn(INFINITY, INFINITY), hi2 = __floats2bfloat162_rn(-INFINITY, -INFINITY);
    auto seg = [&](int64_t st, const uint4 p0, const uint4 p1) {
      const uint32_t w[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
        lo2 = __hmin2(lo2, b2);
        hi2 = __hmax2(hi2, b2);
      }
#pragma unroll
      for (int aa = 0; aa < NA; ++aa) {
        const uint4* fa = frag + aa * ad.frag_stride;
        if constexpr (J1 == 4) {
          uint4 fr[MT];
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) fr[mt] = fa[(st * MT + mt) * 32 + lane];
#pragma unroll
          for (int J = 0; J < 4; ++J) {
            const uint32_t sel = (J & 1) ? 0x7632u : 0x5410u;
            const uint32_t b0 = __byte_perm(w[J >> 1], w[2 + (J >> 1)], sel);
            const uint32_t b1 = __byte_perm(w[4 + (J >> 1)], w[6 + (J >> 1)], sel);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) mma_16816(acc[aa][J][mt], fr[mt].x, fr[mt].y, fr[mt].z, fr[mt].w, b0, b1);
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
              const uint4 fr = fa[((st * 4 + u) * MT + mt) * 32 + lane];
              mma_16816(acc[aa][0][mt], fr.x, fr.y, fr.z, fr.w, w[2 * u], w[2 * u + 1]);
            }
        }
      }
    };
    int64_t st = warp;
    for (; st + (AQC_UNROLL - 1) * W < nseg; st += AQC_UNROLL * W) {
      uint4 p[AQC_UNROLL][2];
#pragma unroll
      for (int u = 0; u < AQC_UNROLL; ++u) {
        p[u][0] = __ldg(reinterpret_cast<const uint4*>(xrow + 128 * (st + u * W) + off0));
        p[u][1] = __ldg(reinterpret_cast<const uint4*>(xrow + 128 * (st + u * W) + off1));
      }
#pragma unroll
      for (int u = 0; u < AQC_UNROLL; ++u) seg(st + u * W, p[u][0], p[u][1]);
    }
    for (; st < nseg; st += W)
      seg(st, __ldg(reinterpret_cast<const uint4*>(xrow + 128 * st + off0)),
          __ldg(reinterpret_cast<const uint4*>(xrow + 128 * st + off1)));
    // D rows m = g (+ 8), columns n = tokens 2c, 2c + 1
#pragma unroll
    for (int aa = 0; aa < NA; ++aa)
#pragma unroll
      for (int J = 0; J < NJ; ++J)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          float* zrow = &s_z[warp][2 * c + h][aa * K2];
          if constexpr (MT == 1) {
            zrow[g * J1 + J] = acc[aa][J][0][h] + acc[aa][J][0][2 + h];
          } else {
            zrow[g * J1 + J] = acc[aa][J][0][h] + acc[aa][J][1][h];
            zrow[(g + 8) * J1 + J] = acc[aa][J][0][2 + h] + acc[aa][J][1][2 + h];
          }
        }
    if (CODES) {
      float lo = fminf(__low2float(lo2), __high2float(lo2)), hi = fmaxf(__low2float(hi2), __high2float(hi2));
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, 1));
      lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, 2));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, 1));
      hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, 2));
      if (c == 0) {
        s_lo[warp][g] = lo;
        s_hi[warp][g] = hi;
      }
    }
    __syncthreads();
    // ---- Z1 of the 8 tokens: fixed-order sum of the warp partials
    for (int i = static_cast<int>(threadIdx.x); i < 8 * NA * K2; i += W * 32) {
      const int tk = i / (NA * K2), ac = i % (NA * K2), aa = ac / K2, col = ac % K2;
      const int64_t row = t0 + tk;
      float v = s_z[0][tk][ac];
#pragma unroll
      for (int w2 = 1; w2 < W; ++w2) v += s_z[w2][tk][ac];
      if (row < T) {
        float* zf = ad.zf[aa];
        __nv_bfloat16* zb = ad.zb[aa];
        if (zf != nullptr) zf[row * K2 + col] = v;
        if (zb != nullptr) {
          const __nv_bfloat16 hv = __float2bfloat16_rn(v);
          zb[row * ldzb + col] = hv;
          zb[row * ldzb + K2 + col] = __float2bfloat16_rn(v - __bfloat162float(hv));
          zb[row * ldzb + 2 * K2 + col] = hv;
        }
      }
    }
    if (ldzb > 3 * K2) {
      const int padw = static_cast<int>(ldzb - 3 * K2);
      for (int i = static_cast<int>(threadIdx.x); i < 8 * NA * padw; i += W * 32) {
        const int aa = i / (8 * padw), ii = i % (8 * padw);
        const int64_t row = t0 + ii / padw;
        if (row < T && ad.zb[aa] != nullptr) ad.zb[aa][row * ldzb + 3 * K2 + ii % padw] = __float2bfloat16_rn(0.f);
      }
    }
    if constexpr (CODES) {
      // ---- pass 2: codes of this warp's segments of row g
      float lo = s_lo[0][g], hi = s_hi[0][g];
#pragma unroll
      for (int w2 = 1; w2 < W; ++w2) {
        lo = fminf(lo, s_lo[w2][g]);
        hi = fmaxf(hi, s_hi[w2][g]);
      }
      AqRow r;
      r.lo = lo;
      r.lo64 = static_cast<double>(lo);
      r.step64 = __ddiv_rn(__dsub_rn(static_cast<double>(hi), r.lo64), 255.0);
      const bool flat = !(r.step64 > 0.0);
      r.inv = flat ? 0.f : static_cast<float>(1.0 / r.step64);
      const float nb = -lo * r.inv;
      r.nbh = nb + 0.5f;
      uint8_t* crow = codes + trow * ldc;
      const bool sub = __any_sync(0xffffffffu, fabsf(nb) > 512.0f);
      uint32_t sum = sub ? aqc_codes_row<J1, true>(xrow, crow, nseg, warp, off0, off1, r, flat, valid)
                         : aqc_codes_row<J1, false>(xrow, crow, nseg, warp, off0, off1, r, flat, valid);
      sum += __shfl_xor_sync(0xffffffffu, sum, 1);
      sum += __shfl_xor_sync(0xffffffffu, sum, 2);
      if (c == 0) s_sum[warp][g] = static_cast<int32_t>(sum);
      if (warp == 0 && valid) {
        if (c == 0) {
          sx[trow] = flat ? 0.0f : __double2float_rn(r.step64);
          ox[trow] = lo;
        }
        for (int64_t kk = K + c; kk < ldc; kk += 4) crow[kk] = 0;  // zero padding [K, ldc) of the codes row
      }
      __syncthreads();  // after this only s_sum is read until the next group's first barrier
      if (threadIdx.x < 8 && t0 + threadIdx.x < T) {
        int32_t s = 0;
#pragma unroll
        for (int w2 = 0; w2 < W; ++w2) s += s_sum[w2][threadIdx.x];
        rsx[t0 + threadIdx.x] = s;
      }
    } else {
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------------------------
#ifdef QA_DP_TRACE
__device__ unsigned long long g_dp_trace[16];
#define DP_MARK(i)                                                                   \
  if (threadIdx.x == 0 && blockIdx.x == 0) {                                         \
    unsigned long long tt_;                                                          \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt_));                          \
    g_dp_trace[i] = tt_;                                                             \
  }
#else
#define DP_MARK(i)
#endif

// Warp transpose-reduction of NV values per lane (NV a power of two <= 32): afterwards lane l holds
// Σ_lanes v[l % NV] in v[0] — 31 shuffles for NV = 32 instead of 32 x 5 for 32 separate reductions.
template <int NV>
__device__ __forceinline__ void warp_transpose_reduce(float (&v)[NV]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o >= NV; o >>= 1)
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] += __shfl_xor_sync(0xffffffffu, v[j], o);
#pragma unroll
  for (int o = NV / 2; o >= 1; o >>= 1) {
    const bool upper = (lane & o) != 0;
#pragma unroll
    for (int j = 0; j < o; ++j) {
      const float send = upper ? v[j] : v[j + o];
      const float keep = upper ? v[j + o] : v[j];
      v[j] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

// Decode-size prologue (1..8 tokens, KV-cached decoding): one CTA per token row does the bit-exact
// act-quant (aq_codes8b + fp64 replay), Z1 = x·G1 in fp32 and the last core's input Zlast (d = 3:
// Z2 = Z1·Gm, [H][C]; d = 2: Z1), so the matrix-vector pass (gemv.cu) needs no V / fragment build.
// The CTA is sized to the row (one 16-byte chunk per thread up to 1024 threads) and releases the
// dependent matrix-vector launch at once (programmatic dependent launch): its CTAs stream the weight
// codes into L2 while this prologue runs and wait on griddepcontrol before reading its outputs.
template <int J1, int R1>
__global__ void __launch_bounds__(512) k_decode_prep(const __nv_bfloat16* __restrict__ x, int64_t K,
                                                    uint8_t* __restrict__ codes, int64_t ldc, float* __restrict__ sx,
                                                    float* __restrict__ ox, int32_t* __restrict__ rsx,
                                                    const DecodePrepMembers mem, bool vec, bool early) {
  DP_MARK(0)
  asm volatile("griddepcontrol.launch_dependents;");
  // CTA (token, member): every member's Z1 / Zlast; member 0 also writes the shared activation codes
  const DecodePrepMember& me = mem.m[blockIdx.y];
  const float* __restrict__ G1 = me.G1;
  const float* __restrict__ G2 = me.G2;
  const int d = me.d, H = me.H, C = me.C;
  float* __restrict__ z1out = me.z1out;
  float* __restrict__ zlast = me.zlast;
  const int64_t ldz = me.ldz;
  const bool coder = blockIdx.y == 0;
  constexpr int K2 = J1 * R1;
  constexpr int NV = K2 < 32 ? K2 : 32;  // values per transpose-reduction round
  constexpr int NJ = 8 / J1;             // G1 rows (j1) per 16-byte chunk of x
  constexpr int GH = NJ * R1 > 64 ? 2 : 1;  // G1 floats of a chunk loaded in GH halves (<= 64 registers)
  extern __shared__ __align__(16) uint8_t dp_smem[];
  __shared__ float red[16][K2 + 1];
  __shared__ float s_lo[16], s_hi[16];
  __shared__ int32_t s_sum[16];
  __shared__ float z1s[K2];
  const int t = blockIdx.x, tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int NT = blockDim.x, NW = NT >> 5;
  const uint4* xr = reinterpret_cast<const uint4*>(x + t * K);
  uint4* row = reinterpret_cast<uint4*>(dp_smem);
  const int nchunk = static_cast<int>(K / 8);
  // the middle core (d = 3) does not depend on x: start its copy into shared memory now
  float* g2s = reinterpret_cast<float*>(dp_smem + ((K * 2 + 15) / 16) * 16);  // [R1][H][J1][C]
  const int n2 = d == 3 ? R1 * H * J1 * C : 0;
  if (vec && n2 > 0) {
    for (int q = tid; q < n2 / 4; q += NT) cp_async16(g2s + 4 * q, G2 + 4 * q, true);
    cp_async_commit();
  }
  // early: launched as a programmatic dependent of whatever kernel produces x — the cores (weights) are
  // pulled into L2 while that kernel finishes, then x is read only after it has completed
  if (early) {
    for (int c = tid; c < nchunk; c += NT)
      for (int off = 0; off < NJ * R1; off += 32)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(G1 + static_cast<int64_t>(c) * NJ * R1 + off));
    asm volatile("griddepcontrol.wait;" ::: "memory");
  }
  __nv_bfloat162 lo2 = __floats2bfloat162_rn(INFINITY, INFINITY), hi2 = __floats2bfloat162_rn(-INFINITY, -INFINITY);
  float z[K2];
#pragma unroll
  for (int i = 0; i < K2; ++i) z[i] = 0.f;
#pragma unroll 2
  for (int c = tid; c < nchunk; c += NT) {
    uint4 v;  // not ld.global.nc: x may come from the kernel this one was launched behind
    asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(xr + c));
    row[c] = v;
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const __nv_bfloat162 b2 = *reinterpret_cast<const __nv_bfloat162*>(&w[i]);
      lo2 = __hmin2(lo2, b2);
      hi2 = __hmax2(hi2, b2);
    }
    // elements 8c + e: j1 = 8c / J1 + e / J1, J = e % J1; the chunk's G1 rows are NJ * R1 contiguous floats
    const float* gbase = G1 + static_cast<int64_t>(c) * NJ * R1;
#pragma unroll
    for (int hh = 0; hh < GH; ++hh) {
      constexpr int GF = NJ * R1 / GH;
      float gv[GF];
      if (vec) {
#pragma unroll
        for (int q = 0; q < GF / 4; ++q) {
          const float4 f = __ldg(reinterpret_cast<const float4*>(gbase + hh * GF) + q);
          gv[4 * q] = f.x;
          gv[4 * q + 1] = f.y;
          gv[4 * q + 2] = f.z;
          gv[4 * q + 3] = f.w;
        }
      } else {
#pragma unroll
        for (int q = 0; q < GF; ++q) gv[q] = __ldg(gbase + hh * GF + q);
      }
#pragma unroll
      for (int e = hh * (8 / GH); e < (hh + 1) * (8 / GH); ++e) {
        const float xv = __uint_as_float((e & 1) ? (w[e >> 1] & 0xFFFF0000u) : (w[e >> 1] << 16));
        const int jl = e / J1 - hh * (NJ / GH), J = e % J1;
#pragma unroll
        for (int a = 0; a < R1; ++a) z[a * J1 + J] = fmaf(xv, gv[jl * R1 + a], z[a * J1 + J]);
      }
    }
  }
  DP_MARK(1)
  float lo = fminf(__low2float(lo2), __high2float(lo2)), hi = fmaxf(__low2float(hi2), __high2float(hi2));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    lo = fminf(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
#pragma unroll
  for (int g = 0; g < K2 / NV; ++g) {
    float v[NV];
#pragma unroll
    for (int i = 0; i < NV; ++i) v[i] = z[g * NV + i];
    warp_transpose_reduce<NV>(v);
    if (lane < NV) red[warp][g * NV + lane] = v[0];
  }
  if (lane == 0) {
    s_lo[warp] = lo;
    s_hi[warp] = hi;
  }
  DP_MARK(2)
  __syncthreads();
  DP_MARK(3)
  lo = s_lo[0];
  hi = s_hi[0];
  for (int w2 = 1; w2 < NW; ++w2) {
    lo = fminf(lo, s_lo[w2]);
    hi = fmaxf(hi, s_hi[w2]);
  }
  if (tid < K2) {
    float v = red[0][tid];
    for (int w2 = 1; w2 < NW; ++w2) v += red[w2][tid];
    z1s[tid] = v;
    if (z1out != nullptr) z1out[t * K2 + tid] = v;
  }
  DP_MARK(4)
  if (coder) {
  // codes of this row (bracketed rule, bit-exact with quant.py:73-99)
  const double lo64 = static_cast<double>(lo);
  const double step64 = __ddiv_rn(__dsub_rn(static_cast<double>(hi), lo64), 255.0);
  const bool flat = !(step64 > 0.0);
  const float inv = flat ? 0.f : static_cast<float>(1.0 / step64);
  const float nb = -lo * inv;
  const bool sub = fabsf(nb) > 512.0f;  // uniform across the CTA
  const float alo = sub ? 0.5f - kTieBand : nb + 0.5f - kTieBand, ahi = sub ? 0.5f + kTieBand : nb + 0.5f + kTieBand;
  const unsigned long long inv2 = f2pack(inv, inv), nlo2 = f2pack(-lo, -lo), alo2 = f2pack(alo, alo),
                           ahi2 = f2pack(ahi, ahi);
  uint8_t* crow = codes + t * ldc;
  uint32_t sum = 0;
  for (int c = tid; c < nchunk; c += NT) {
    const uint4 v = row[c];
    uint32_t c0, c1, d0, d1;
    if (sub)
      aq_codes8b<true>(v, inv2, alo2, ahi2, nlo2, c0, c1, d0, d1);
    else
      aq_codes8b<false>(v, inv2, alo2, ahi2, nlo2, c0, c1, d0, d1);
    if (flat) c0 = c1 = d0 = d1 = 0u;
    if (d0 != 0u) c0 = aq_replay_word(v, 0, c0, d0, lo64, step64);
    if (d1 != 0u) c1 = aq_replay_word(v, 4, c1, d1, lo64, step64);
    sum = __dp4a(c0, 0x01010101u, __dp4a(c1, 0x01010101u, sum));
    *reinterpret_cast<uint2*>(crow + 8 * static_cast<int64_t>(c)) = make_uint2(c0, c1);
  }
  DP_MARK(5)
  for (int64_t k = K + tid; k < ldc; k += NT) crow[k] = 0;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  if (lane == 0) s_sum[warp] = static_cast<int32_t>(sum);
  __syncthreads();
  DP_MARK(6)
  if (tid == 0) {
    int32_t sm = 0;
    for (int w2 = 0; w2 < NW; ++w2) sm += s_sum[w2];
    rsx[t] = sm;
    sx[t] = flat ? 0.0f : __double2float_rn(step64);
    ox[t] = lo;
  }
  }  // coder
  // Zlast: d = 3 -> Z2[i2, b] = Σ_{a, j2} Z1[a, j2] G2[a, i2, j2, b], four lanes per output (K2 / 4 terms
  // each, then two shuffles); d = 2 -> Z1.
  if (d == 3) {
    DP_MARK(7)
    if (vec) {
      cp_async_wait<0>();
    } else {
      for (int q = tid; q < n2; q += NT) g2s[q] = __ldg(G2 + q);
    }
    __syncthreads();
    DP_MARK(8)
    const int HC = H * C;
    const int passes = (HC * 4 + NT - 1) / NT;
    for (int p = 0; p < passes; ++p) {
      const int o = (p * NT + tid) >> 2, part = tid & 3;
      const int oc = o < HC ? o : HC - 1;
      const int i2 = oc / C, b = oc % C;
      float v = 0.f;
#pragma unroll
      for (int q = 0; q < K2 / 4; ++q) {
        const int aj = part * (K2 / 4) + q;
        const int a = aj / J1, j2 = aj % J1;
        v = fmaf(z1s[aj], g2s[((a * H + i2) * J1 + j2) * C + b], v);
      }
      v += __shfl_xor_sync(0xffffffffu, v, 1);
      v += __shfl_xor_sync(0xffffffffu, v, 2);
      if (part == 0 && o < HC) zlast[t * ldz + o] = v;
    }
    DP_MARK(9)
  } else {
    if (tid < K2) zlast[t * ldz + tid] = z1s[tid];
  }
  // when chained behind the previous member's matrix-vector pass: do not complete before it (no-op when
  // launched normally)
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

}  // namespace

#ifdef QA_DP_TRACE
extern "C" __attribute__((visibility("default"))) int qa_debug_dp_trace(unsigned long long* out) {
  return static_cast<int>(cudaMemcpyFromSymbol(out, g_dp_trace, sizeof(g_dp_trace)));
}
#endif

cudaError_t launch_decode_prep(const void* x, int64_t T, int64_t K, uint8_t* codes, int64_t ldc, float* sx, float* ox,
                               int32_t* rsx, int J1, int R1, const DecodePrepMembers& mem, cudaStream_t s,
                               bool chain) {
  if (T == 0 || mem.n < 1) return cudaSuccess;
  LaunchScope scope(kQuantize, double(T) * K * 3 + 12.0 * T, s);
  count_launches(1);
  const int64_t nch = K / 8;  // one 16-byte chunk per thread, 128..512 threads
  const int threads = static_cast<int>(nch >= 512 ? 512 : (nch <= 128 ? 128 : (nch + 31) / 32 * 32));
  size_t n2 = 0;
  bool vec = true;  // vector / cp.async paths need 16-byte aligned cores (G1 rows of a chunk start at multiples of 32 floats)
  for (int i = 0; i < mem.n; ++i) {
    const DecodePrepMember& m = mem.m[i];
    const size_t n2i = m.d == 3 ? static_cast<size_t>(R1) * m.H * J1 * m.C : 0;
    n2 = n2i > n2 ? n2i : n2;
    vec = vec && reinterpret_cast<uintptr_t>(m.G1) % 16 == 0 &&
          (m.G2 == nullptr || reinterpret_cast<uintptr_t>(m.G2) % 16 == 0) && n2i % 4 == 0;
  }
  const size_t smem = (static_cast<size_t>(K) * 2 + 15) / 16 * 16 + sizeof(float) * n2;
  // every prologue is a programmatic dependent: a chained member (x already complete) overlaps the previous
  // member's pass; the first one (early) prefetches its cores and waits for x's producer before reading it
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(T), static_cast<unsigned>(mem.n));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const bool early = !chain;
  const __nv_bfloat16* xb = static_cast<const __nv_bfloat16*>(x);
  cudaError_t e = cudaSuccess;
#define QA_DPR(JJ, RR)                                                                                             \
  {                                                                                                                \
    cudaFuncSetAttribute(k_decode_prep<JJ, RR>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)); \
    e = cudaLaunchKernelEx(&cfg, k_decode_prep<JJ, RR>, xb, K, codes, ldc, sx, ox, rsx, mem, vec, early);          \
  }
  if (J1 == 4 && R1 == 8)
    QA_DPR(4, 8)
  else if (J1 == 4)
    QA_DPR(4, 16)
  else if (R1 == 8)
    QA_DPR(1, 8)
  else
    QA_DPR(1, 16)
#undef QA_DPR
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

namespace {

// V[n, c] (bf16, zero padded to ldv): contraction of cores 2..d with the left rank open.
//   d = 2: V[i, a] = G2[a, i];  d = 3: V[(i2, i3), (a, j2)] = Σ_b G2[a, i2, j2, b] G3[b, i3]
QA_DEV void build_v_at(int d, int R1, int H, int J1, int C, int M, const float* __restrict__ G2,
                       const float* __restrict__ G3, __nv_bfloat16* __restrict__ V, int64_t N, int64_t ldv,
                       int64_t idx) {
  // one thread per (row n, column cc < K2): v is computed once and written to its three slots
  // [V_hi | V_hi | V_lo] against [Z_hi | Z_lo | Z_hi]: the three leading terms of the bf16 split
  // product, so y2 carries ~16 mantissa bits although the MMA operands are bf16; padding [3 K2, ldv) = 0
  const int K2 = R1 * J1;
  const int per_row = static_cast<int>(ldv) - 2 * K2;  // threads per row: K2 value columns + the padding
  if (idx >= N * per_row) return;
  const int n32 = static_cast<int>(idx / per_row);  // N * ldv < 2^31 (launcher)
  const int c = static_cast<int>(idx - static_cast<int64_t>(n32) * per_row);
  __nv_bfloat16* vr = V + static_cast<int64_t>(n32) * ldv;
  if (c >= K2) {
    vr[c + 2 * K2] = __float2bfloat16_rn(0.f);
    return;
  }
  const int a = c / J1, j2 = c - a * J1;
  float v = 0.f;
  if (d == 2) {
    v = G2[static_cast<int64_t>(a) * N + n32];
  } else {
    const int i2 = n32 / M, i3 = n32 - i2 * M;
    const float* g2 = G2 + ((static_cast<int64_t>(a) * H + i2) * J1 + j2) * C;
    for (int b = 0; b < C; ++b) v = fmaf(__ldg(g2 + b), __ldg(G3 + static_cast<int64_t>(b) * M + i3), v);
  }
  const __nv_bfloat16 hi = __float2bfloat16_rn(v);
  vr[c] = hi;
  vr[c + K2] = hi;
  vr[c + 2 * K2] = __float2bfloat16_rn(v - __bfloat162float(hi));
}

__global__ void __launch_bounds__(256) k_build_v(int d, int R1, int H, int J1, int C, int M,
                                                 const float* __restrict__ G2, const float* __restrict__ G3,
                                                 __nv_bfloat16* __restrict__ V, int64_t N, int64_t ldv) {
  build_v_at(d, R1, H, J1, C, M, G2, G3, V, N, ldv, static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x);
}

// Everything the forward of a linear (or of a shared-input group) derives from the cores alone, in one launch:
// the G1 MMA fragments of every member (k_g1_frag) and every member's V (k_build_v); blocks [0, fb) build
// fragments (member = block / per_f), the rest V (member from the prefix vstart).
template <int J1, int R1>
__global__ void __launch_bounds__(256) k_adapter_prep(const AdapterPrep P) {
  const int64_t b = blockIdx.x;
  const int64_t fb = P.nf * P.per_f;
  if (b < fb) {
    const int m = static_cast<int>(b / P.per_f);
    g1_frag_at<J1, R1>(P.G1[m], P.frag[m], P.nfrag, (b - m * P.per_f) * 256 + threadIdx.x);
    return;
  }
  int m = 0;
  while (m + 1 < P.nv && b >= P.vstart[m + 1]) ++m;
  const VJob& v = P.v[m];
  build_v_at(v.d, v.R1, v.H, v.J1, v.C, v.M, v.G2, v.G3, v.V, v.N, v.ldv, (b - P.vstart[m]) * 256 + threadIdx.x);
}

// B_ext[k = (j1, J), c = (a, J')] = G1[j1, a] δ(J, J')  (bf16, zero padded to ldb)
__global__ void __launch_bounds__(256) k_build_bext(int R1, int J1, const float* __restrict__ G1,
                                                    __nv_bfloat16* __restrict__ B, int64_t K, int64_t ldb) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= K * ldb) return;
  const int64_t k = idx / ldb;
  const int c = static_cast<int>(idx - k * ldb);
  // [B_hi | B_hi | B_lo] against [dZ1_hi | dZ1_lo | dZ1_hi] (see k_build_v)
  const int K2 = R1 * J1;
  float v = 0.f;
  if (c < 3 * K2) {
    const int cc = c % K2;
    const int a = cc / J1, Jp = cc % J1;
    const int64_t j1 = k / J1;
    const int J = static_cast<int>(k % J1);
    if (J == Jp) v = G1[j1 * R1 + a];
    if (c >= 2 * K2) v -= __bfloat162float(__float2bfloat16_rn(v));
  }
  B[idx] = __float2bfloat16_rn(v);
}

// f32 [T, K2] -> bf16 [T, ld] laid out [hi | lo | 0]: hi + lo carries ~16 mantissa bits, so the
// bf16 extension MMA against [B | B] rounds only the constant operand.
__global__ void __launch_bounds__(256) k_split_rows(const float* __restrict__ in, int64_t T, int K2,
                                                    __nv_bfloat16* __restrict__ out, int64_t ld) {
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= T * ld) return;
  const int64_t t = idx / ld;
  const int c = static_cast<int>(idx - t * ld);
  float v = 0.f;
  if (c < 3 * K2) {  // [hi | lo | hi]
    const float f = in[t * K2 + c % K2];
    v = __bfloat162float(__float2bfloat16_rn(f));
    if (c >= K2 && c < 2 * K2) v = f - v;
  }
  out[idx] = __float2bfloat16_rn(v);
}

// ---------------------------------------------------------------------------------------------
// dy pass: for one (h, 256-column block) and a token range:
//   dZ[t, h, c]  = Σ_col dy[t, h, col] · Gd[c, col]          (partial per column block)
//   dGd[c, col] += Σ_t  Z[t, h, c] · dy[t, h, col]           (partial per (h, token split))
constexpr int DY_TT = 32, DY_COLS = 256, DY_LDY = DY_COLS + 8;

template <int C>
__global__ void __launch_bounds__(256) k_tt_dy(const __nv_bfloat16* __restrict__ dy, int64_t T, int64_t N, int H,
                                               int M, const float* __restrict__ Z, int64_t zs,
                                               const float* __restrict__ Gd, float* __restrict__ dz_part,
                                               float* __restrict__ dg_part, int S) {
  static_assert(C == 8 || C == 16, "rank into the last core must be 8 or 16");
  constexpr int NT = C / 8;
  constexpr int KW = 8 / (2 * NT);  // warps sharing one 16 x 8 dZ output tile (split over K)
  extern __shared__ __align__(16) uint8_t dy_smem[];
  auto sdy = reinterpret_cast<__nv_bfloat16(*)[DY_TT][DY_LDY]>(dy_smem);
  auto sz = reinterpret_cast<__nv_bfloat16(*)[C][DY_TT + 8]>(dy_smem + sizeof(__nv_bfloat16) * 2 * DY_TT * DY_LDY);
  auto sg = reinterpret_cast<__nv_bfloat16(*)[DY_COLS + 8]>(dy_smem + sizeof(__nv_bfloat16) * 2 * DY_TT * DY_LDY +
                                                             sizeof(__nv_bfloat16) * 2 * C * (DY_TT + 8));
  auto sred = reinterpret_cast<float(*)[DY_TT][C]>(dy_smem + sizeof(__nv_bfloat16) * 2 * DY_TT * DY_LDY +
                                                    sizeof(__nv_bfloat16) * 2 * C * (DY_TT + 8) +
                                                    sizeof(__nv_bfloat16) * C * (DY_COLS + 8));

  const int ncb = M / DY_COLS;
  const int cb = blockIdx.x % ncb, h = blockIdx.x / ncb, s = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t col0 = static_cast<int64_t>(h) * M + static_cast<int64_t>(cb) * DY_COLS;
  const int64_t tiles = (T + DY_TT - 1) / DY_TT;
  const int64_t per = (tiles + S - 1) / S;
  const int64_t tile0 = s * per, tile1 = tile0 + per < tiles ? tile0 + per : tiles;

  for (int i = tid; i < C * DY_COLS; i += 256) {
    const int c = i / DY_COLS, col = i % DY_COLS;
    sg[c][col] = __float2bfloat16_rn(Gd[static_cast<int64_t>(c) * M + cb * DY_COLS + col]);
  }

  auto load_tile = [&](int64_t tile, int buf) {
    const int64_t t0 = tile * DY_TT;
    for (int i = tid; i < DY_TT * (DY_COLS / 8); i += 256) {
      const int r = i / (DY_COLS / 8), ch = i % (DY_COLS / 8);
      const int64_t t = t0 + r;
      const bool ok = t < T;
      cp_async16(&sdy[buf][r][ch * 8], dy + (ok ? t : 0) * N + col0 + ch * 8, ok);
    }
    for (int i = tid; i < DY_TT * C; i += 256) {
      const int r = i / C, c = i % C;
      const int64_t t = t0 + r;
      sz[buf][c][r] = __float2bfloat16_rn(t < T ? Z[t * zs + static_cast<int64_t>(h) * C + c] : 0.f);
    }
  };

  float acc2[2][NT][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc2[i][nt][q] = 0.f;

  if (tile0 < tile1) load_tile(tile0, 0);
  cp_async_commit();
  const int g = lane >> 2, tq = lane & 3;
  for (int64_t tile = tile0; tile < tile1; ++tile) {
    const int buf = static_cast<int>((tile - tile0) & 1);
    if (tile + 1 < tile1) load_tile(tile + 1, buf ^ 1);
    cp_async_commit();
    cp_async_wait<1>();
    __syncthreads();

    // (1) dZ partial: warp -> (m-tile, n-tile) output tile, K (256 columns) split over KW warps
    {
      const int ti = warp / KW, kq = warp % KW;
      const int mt = ti / NT, nt = ti % NT;
      float d1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < 16 / KW; ++ks) {
        const int kc = (kq * (16 / KW) + ks) * 16;
        uint32_t b0, b1, a0, a1, a2, a3;
        ldsm_x2(&sg[nt * 8 + (lane & 7)][kc + ((lane >> 3) & 1) * 8], b0, b1);
        ldsm_x4(&sdy[buf][mt * 16 + (lane & 7) + ((lane >> 3) & 1) * 8][kc + (lane >> 4) * 8], a0, a1, a2, a3);
        mma_16816(d1, a0, a1, a2, a3, b0, b1);
      }
      sred[kq][mt * 16 + g][nt * 8 + 2 * tq] = d1[0];
      sred[kq][mt * 16 + g][nt * 8 + 2 * tq + 1] = d1[1];
      sred[kq][mt * 16 + g + 8][nt * 8 + 2 * tq] = d1[2];
      sred[kq][mt * 16 + g + 8][nt * 8 + 2 * tq + 1] = d1[3];
    }

    // (2) dGd^T[cols x C] += dy_tile^T [cols x 32 tokens] · Z [32 tokens x C]
#pragma unroll
    for (int ks = 0; ks < 2; ++ks) {
      uint32_t b[NT][2];
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
        ldsm_x2(&sz[buf][nt * 8 + (lane & 7)][ks * 16 + ((lane >> 3) & 1) * 8], b[nt][0], b[nt][1]);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int c0 = warp * 32 + i * 16;
        const int q = lane >> 3;
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(&sdy[buf][ks * 16 + (q >> 1) * 8 + (lane & 7)][c0 + (q & 1) * 8], a0, a1, a2, a3);
#pragma unroll
        for (int nt = 0; nt < NT; ++nt) mma_16816(acc2[i][nt], a0, a1, a2, a3, b[nt][0], b[nt][1]);
      }
    }
    __syncthreads();
    for (int i = tid; i < DY_TT * C; i += 256) {
      const int r = i / C, c = i % C;
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < KW; ++w) v += sred[w][r][c];
      const int64_t t = tile * DY_TT + r;
      if (t < T) dz_part[(static_cast<int64_t>(cb) * T + t) * (static_cast<int64_t>(H) * C) + static_cast<int64_t>(h) * C + c] = v;
    }
  }
  cp_async_wait<0>();
  // dGd partial for (h, s): element (col = c0 + g (+8), c = nt*8 + 2tq (+1))
  float* dst = dg_part + (static_cast<int64_t>(h) * S + s) * (static_cast<int64_t>(C) * M);
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      const int col = cb * DY_COLS + warp * 32 + i * 16 + g;
      const int c = nt * 8 + 2 * tq;
      dst[static_cast<int64_t>(c) * M + col] = acc2[i][nt][0];
      dst[static_cast<int64_t>(c + 1) * M + col] = acc2[i][nt][1];
      dst[static_cast<int64_t>(c) * M + col + 8] = acc2[i][nt][2];
      dst[static_cast<int64_t>(c + 1) * M + col + 8] = acc2[i][nt][3];
    }
}

// ---------------------------------------------------------------------------------------------
// Fused backward of the pinned Llama modes (d = 3, m = (1, H, 256), n = (K/4, 4, 1), ranks
// (1, C, C, 1)): one pass over dy per (h-range, token-range) CTA replaces the stage-2 recompute,
// the dy pass, the middle-core backward and their partial buffers.  Per 32-token tile and output
// block h (256 columns of dy, double-buffered with cp.async), all on the tensor cores (mma.sync):
//   dZ2_h  = dy_h · G3ᵀ       K = 256 split over KW warps, fixed-order sum
//   dG3   += dy_hᵀ · Z2_h     accumulators in registers for the CTA's lifetime
//   dZ1   += dZ2_h · Gm_hᵀ    accumulators in registers for the tile (Gm_h[aj][c] = G2[a, h, j2, c])
//   dG2_h += Z1ᵀ · dZ2_h      per-tile products added to shared-memory accumulators
//   Z2_h+1 = Z1 · Gm_h+1      (for the next block's dG3)
// dy, G3 and Z2 enter as bf16 (dy is bf16 already; as in the unfused kernels); Z1, Gm and dZ2 —
// fp32 values — enter as hi + lo bf16 pairs with three MMAs per product (hi·hi + lo·hi + hi·lo),
// which keeps those contractions at ~2^-16 relative accuracy.  dZ1 of the h-range is written as a
// partial ([HS][T][K2]); k_tt_dg1 sums the HS partials in fixed order.
constexpr int FB_TT = 32, FB_COLS = 256, FB_LDY = FB_COLS + 8, FB_LDZ = FB_TT + 8, FB_NS = 3;

template <int C>
struct FbLayout {
  static constexpr int K2 = 4 * C, NT = C / 8, KW = 8 / (2 * NT);
  static constexpr int LZ1 = K2 + 8;         // Z1 planes: row stride (bf16)
  static constexpr int LC = C == 8 ? 8 : 24;  // Gm / dZ2 planes: row stride (bf16), ldmatrix conflict-free
  static constexpr size_t dy = 0;                                                         // bf16 [NS][TT][LDY]
  static constexpr size_t g3 = dy + sizeof(__nv_bfloat16) * FB_NS * FB_TT * FB_LDY;      // bf16 [C][LDY]
  static constexpr size_t z2t = g3 + sizeof(__nv_bfloat16) * C * FB_LDY;          // bf16 [C][LDZ]
  static constexpr size_t red = z2t + sizeof(__nv_bfloat16) * C * FB_LDZ;         // f32 [KW][TT][C]
  static constexpr size_t z1p = red + sizeof(float) * KW * FB_TT * C;             // bf16 [2][TT][LZ1]
  static constexpr size_t dz2p = z1p + sizeof(__nv_bfloat16) * 2 * FB_TT * LZ1;   // bf16 [2][TT][LC]
  static constexpr size_t gmp = dz2p + sizeof(__nv_bfloat16) * 2 * FB_TT * LC;    // bf16 [2][HR][K2][LC]
  __host__ __device__ static size_t dg2(int hr) { return gmp + sizeof(__nv_bfloat16) * 2 * size_t(hr) * K2 * LC; }  // f32 [HR][K2][C]
  __host__ __device__ static size_t z1raw(int hr) { return dg2(hr) + sizeof(float) * size_t(hr) * K2 * C; }  // f32 [2][TT][K2]
  __host__ __device__ static size_t bytes(int hr) { return z1raw(hr) + sizeof(float) * 2 * FB_TT * K2; }
};

template <int C>
__global__ void __launch_bounds__(256) k_tt_bwd_fused(const __nv_bfloat16* __restrict__ dy, int64_t ldy, int64_t T,
                                                      int H, int HR, const float* __restrict__ Z1,
                                                      const float* __restrict__ G2, const float* __restrict__ G3,
                                                      float* __restrict__ dz1p, float* __restrict__ g3part,
                                                      float* __restrict__ g2part) {
  using L = FbLayout<C>;
  constexpr int K2 = L::K2, NT = L::NT, KW = L::KW, LZ1 = L::LZ1, LC = L::LC, J1 = 4;
  constexpr int MTZ = FB_TT / 16;                        // token m-tiles
  constexpr int DZT = MTZ * (K2 / 8) / 8;                // dZ1 output tiles per warp
  extern __shared__ __align__(16) uint8_t fb_smem[];
  auto sdy = reinterpret_cast<__nv_bfloat16(*)[FB_TT][FB_LDY]>(fb_smem + L::dy);
  auto sg3 = reinterpret_cast<__nv_bfloat16(*)[FB_LDY]>(fb_smem + L::g3);
  auto sz2t = reinterpret_cast<__nv_bfloat16(*)[FB_LDZ]>(fb_smem + L::z2t);
  auto sred = reinterpret_cast<float(*)[FB_TT][C]>(fb_smem + L::red);
  auto sz1p = reinterpret_cast<__nv_bfloat16(*)[FB_TT][LZ1]>(fb_smem + L::z1p);
  auto sdz2p = reinterpret_cast<__nv_bfloat16(*)[FB_TT][LC]>(fb_smem + L::dz2p);
  __nv_bfloat16* sgmp = reinterpret_cast<__nv_bfloat16*>(fb_smem + L::gmp);
  float* sdg2 = reinterpret_cast<float*>(fb_smem + L::dg2(HR));
  float* sz1raw = reinterpret_cast<float*>(fb_smem + L::z1raw(HR));
  auto gm = [&](int p, int hl, int aj, int c) -> __nv_bfloat16* {
    return sgmp + ((static_cast<size_t>(p) * HR + hl) * K2 + aj) * LC + c;
  };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  const int hs = blockIdx.x, ts = blockIdx.y, TS = gridDim.y;
  const int h0 = hs * HR, nh = H - h0 < HR ? H - h0 : HR;
  const int64_t ntiles = (T + FB_TT - 1) / FB_TT;
  const int64_t per = (ntiles + TS - 1) / TS;
  const int64_t tile0 = ts * per, tile1 = tile0 + per < ntiles ? tile0 + per : ntiles;

  for (int i = tid; i < C * FB_COLS; i += 256) sg3[i / FB_COLS][i % FB_COLS] = __float2bfloat16_rn(G3[i]);
  for (int i = tid; i < nh * K2 * C; i += 256) {
    const int hl = i / (K2 * C), aj = (i / C) % K2, c = i % C;
    const int a = aj / J1, j2 = aj % J1;
    const float v = G2[((static_cast<int64_t>(a) * H + h0 + hl) * J1 + j2) * C + c];
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    *gm(0, hl, aj, c) = hi;
    *gm(1, hl, aj, c) = __float2bfloat16_rn(v - __bfloat162float(hi));
    sdg2[i] = 0.f;
  }
  float acc2[2][NT][4];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int n = 0; n < NT; ++n)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc2[i][n][q] = 0.f;

  auto load_dy = [&](int64_t t0, int h, int buf) {
    for (int i = tid; i < FB_TT * (FB_COLS / 8); i += 256) {
      const int r = i / (FB_COLS / 8), ch = i % (FB_COLS / 8);
      const int64_t t = t0 + r;
      const bool ok = t < T;
      cp_async16(&sdy[buf][r][ch * 8], dy + (ok ? t : 0) * ldy + static_cast<int64_t>(h) * FB_COLS + ch * 8, ok);
    }
  };
  // Z2_hl = Z1 · Gm_hl (3-term split MMAs) -> bf16, transposed into sz2t; warps 4..7
  auto z2_phase = [&](int hl) {
    for (int task = (warp + 4) & 7; task < MTZ * NT; task += 8) {
      const int mz = task / NT, n8 = task % NT;
      float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < K2 / 16; ++ks) {
        uint32_t ah[4], al[4], bh[2], bl[2];
        ldsm_x4(&sz1p[0][mz * 16 + (lane & 15)][ks * 16 + (lane >> 4) * 8], ah[0], ah[1], ah[2], ah[3]);
        ldsm_x4(&sz1p[1][mz * 16 + (lane & 15)][ks * 16 + (lane >> 4) * 8], al[0], al[1], al[2], al[3]);
        ldsm_x2_t(gm(0, hl, ks * 16 + (lane & 15), n8 * 8), bh[0], bh[1]);
        ldsm_x2_t(gm(1, hl, ks * 16 + (lane & 15), n8 * 8), bl[0], bl[1]);
        mma_16816(d, ah[0], ah[1], ah[2], ah[3], bh[0], bh[1]);
        mma_16816(d, al[0], al[1], al[2], al[3], bh[0], bh[1]);
        mma_16816(d, ah[0], ah[1], ah[2], ah[3], bl[0], bl[1]);
      }
      sz2t[n8 * 8 + 2 * tq][mz * 16 + g] = __float2bfloat16_rn(d[0]);
      sz2t[n8 * 8 + 2 * tq + 1][mz * 16 + g] = __float2bfloat16_rn(d[1]);
      sz2t[n8 * 8 + 2 * tq][mz * 16 + g + 8] = __float2bfloat16_rn(d[2]);
      sz2t[n8 * 8 + 2 * tq + 1][mz * 16 + g + 8] = __float2bfloat16_rn(d[3]);
    }
  };

  // the CTA's (tile, h) items form one stream; dy blocks are prefetched FB_NS - 1 items ahead
  const int64_t nit = (tile1 - tile0) * nh;
  // Z1 rows of a tile are prefetched into sz1raw one tile ahead when a tile spans >= FB_NS items
  const bool z1_async = nh >= FB_NS;
  auto load_z1raw = [&](int64_t tile) {
    if (tile >= tile1) return;
    float* dst = sz1raw + static_cast<size_t>((tile - tile0) & 1) * FB_TT * K2;
    for (int i = tid; i < FB_TT * (K2 / 4); i += 256) {
      const int r = i / (K2 / 4), q = i % (K2 / 4);
      const bool ok = tile * FB_TT + r < T;
      cp_async16(dst + r * K2 + 4 * q, ok ? Z1 + (tile * FB_TT + r) * K2 + 4 * q : Z1, ok);
    }
  };
  auto issue = [&](int64_t it) {
    if (it < nit) load_dy((tile0 + it / nh) * FB_TT, h0 + static_cast<int>(it % nh), static_cast<int>(it % FB_NS));
    cp_async_commit();
  };
  if (z1_async) load_z1raw(tile0);
  for (int i = 0; i < FB_NS - 1; ++i) issue(i);
  float dacc[DZT][4];
  for (int64_t it = 0; it < nit; ++it) {
    const int64_t tile = tile0 + it / nh;
    const int hl = static_cast<int>(it % nh), buf = static_cast<int>(it % FB_NS);
    const int64_t t0 = tile * FB_TT;
    const int nt = static_cast<int>(T - t0 < FB_TT ? T - t0 : FB_TT);
    if (hl == 0) {
      __syncthreads();  // previous tile's readers of the Z1 planes are done
      if (z1_async) {  // this tile's Z1 group (issued a tile ahead; tile 0: group 0) has landed ...
        if (it == 0)
          cp_async_wait<FB_NS - 2>();
        else
          cp_async_wait<FB_NS - 1>();
      }
      __syncthreads();                              // ... for every thread
      const float* zr = sz1raw + static_cast<size_t>((tile - tile0) & 1) * FB_TT * K2;
      for (int i = tid; i < FB_TT * K2; i += 256) {
        const int r = i / K2, aj = i % K2;
        const float f = r < nt ? (z1_async ? zr[i] : Z1[(t0 + r) * K2 + aj]) : 0.f;
        const __nv_bfloat16 hi = __float2bfloat16_rn(f);
        sz1p[0][r][aj] = hi;
        sz1p[1][r][aj] = __float2bfloat16_rn(f - __bfloat162float(hi));
      }
#pragma unroll
      for (int u = 0; u < DZT; ++u)
#pragma unroll
        for (int q = 0; q < 4; ++q) dacc[u][q] = 0.f;
      __syncthreads();
      z2_phase(0);
    }
    if (z1_async && hl == 0) load_z1raw(tile + 1);  // joins the group below; needed nh >= FB_NS items later
    issue(it + FB_NS - 1);  // into the buffer item it - 1 used; its readers passed two barriers since
    cp_async_wait<FB_NS - 1>();
    __syncthreads();  // dy_h and Z2_h are in shared memory
    {  // dZ2_h partial: warp -> (m-tile, n-tile), K split over KW warps
      const int ti = warp / KW, kq = warp % KW;
      const int mt = ti / NT, n8 = ti % NT;
      float d1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < 16 / KW; ++ks) {
        const int kc = (kq * (16 / KW) + ks) * 16;
        uint32_t b0, b1, a0, a1, a2, a3;
        ldsm_x2(&sg3[n8 * 8 + (lane & 7)][kc + ((lane >> 3) & 1) * 8], b0, b1);
        ldsm_x4(&sdy[buf][mt * 16 + (lane & 15)][kc + (lane >> 4) * 8], a0, a1, a2, a3);
        mma_16816(d1, a0, a1, a2, a3, b0, b1);
      }
      sred[kq][mt * 16 + g][n8 * 8 + 2 * tq] = d1[0];
      sred[kq][mt * 16 + g][n8 * 8 + 2 * tq + 1] = d1[1];
      sred[kq][mt * 16 + g + 8][n8 * 8 + 2 * tq] = d1[2];
      sred[kq][mt * 16 + g + 8][n8 * 8 + 2 * tq + 1] = d1[3];
    }
#pragma unroll
    for (int ks = 0; ks < FB_TT / 16; ++ks) {  // dG3ᵀ[cols x C] += dy_hᵀ [cols x tokens] · Z2_h [tokens x C]
      uint32_t b[NT][2];
#pragma unroll
      for (int n8 = 0; n8 < NT; ++n8)
        ldsm_x2(&sz2t[n8 * 8 + (lane & 7)][ks * 16 + ((lane >> 3) & 1) * 8], b[n8][0], b[n8][1]);
#pragma unroll
      for (int i = 0; i < 2; ++i) {
        const int c0 = warp * 32 + i * 16;
        const int q = lane >> 3;
        uint32_t a0, a1, a2, a3;
        ldsm_x4_t(&sdy[buf][ks * 16 + (q >> 1) * 8 + (lane & 7)][c0 + (q & 1) * 8], a0, a1, a2, a3);
#pragma unroll
        for (int n8 = 0; n8 < NT; ++n8) mma_16816(acc2[i][n8], a0, a1, a2, a3, b[n8][0], b[n8][1]);
      }
    }
    __syncthreads();
    for (int i = tid; i < FB_TT * C; i += 256) {  // dZ2_h: fixed-order sum of the K-split partials, hi/lo
      const int t = i / C, c = i % C;
      float v = sred[0][t][c];
#pragma unroll
      for (int w = 1; w < KW; ++w) v += sred[w][t][c];
      const __nv_bfloat16 hi = __float2bfloat16_rn(v);
      sdz2p[0][t][c] = hi;
      sdz2p[1][t][c] = __float2bfloat16_rn(v - __bfloat162float(hi));
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < DZT; ++u) {  // dZ1 tile += dZ2_h · Gm_hᵀ
      const int tl = warp + 8 * u, m = tl / (K2 / 8), n = tl % (K2 / 8);
      if constexpr (C == 8) {
        uint32_t ah0, ah1, al0, al1, bh, bl;
        ldsm_x2(&sdz2p[0][m * 16 + (lane & 15)][0], ah0, ah1);
        ldsm_x2(&sdz2p[1][m * 16 + (lane & 15)][0], al0, al1);
        ldsm_x1(gm(0, hl, n * 8 + (lane & 7), 0), bh);
        ldsm_x1(gm(1, hl, n * 8 + (lane & 7), 0), bl);
        mma_1688(dacc[u], ah0, ah1, bh);
        mma_1688(dacc[u], al0, al1, bh);
        mma_1688(dacc[u], ah0, ah1, bl);
      } else {
        uint32_t ah[4], al[4], bh[2], bl[2];
        ldsm_x4(&sdz2p[0][m * 16 + (lane & 15)][(lane >> 4) * 8], ah[0], ah[1], ah[2], ah[3]);
        ldsm_x4(&sdz2p[1][m * 16 + (lane & 15)][(lane >> 4) * 8], al[0], al[1], al[2], al[3]);
        ldsm_x2(gm(0, hl, n * 8 + (lane & 7), ((lane >> 3) & 1) * 8), bh[0], bh[1]);
        ldsm_x2(gm(1, hl, n * 8 + (lane & 7), ((lane >> 3) & 1) * 8), bl[0], bl[1]);
        mma_16816(dacc[u], ah[0], ah[1], ah[2], ah[3], bh[0], bh[1]);
        mma_16816(dacc[u], al[0], al[1], al[2], al[3], bh[0], bh[1]);
        mma_16816(dacc[u], ah[0], ah[1], ah[2], ah[3], bl[0], bl[1]);
      }
    }
    for (int task = warp; task < (K2 / 16) * NT; task += 8) {  // dG2_h += Z1ᵀ · dZ2_h
      const int ma = task / NT, n8 = task % NT;
      float d[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < FB_TT / 16; ++ks) {
        const int q = lane >> 3;
        uint32_t ah[4], al[4], bh[2], bl[2];
        ldsm_x4_t(&sz1p[0][ks * 16 + (q >> 1) * 8 + (lane & 7)][ma * 16 + (q & 1) * 8], ah[0], ah[1], ah[2], ah[3]);
        ldsm_x4_t(&sz1p[1][ks * 16 + (q >> 1) * 8 + (lane & 7)][ma * 16 + (q & 1) * 8], al[0], al[1], al[2], al[3]);
        ldsm_x2_t(&sdz2p[0][ks * 16 + (lane & 15)][n8 * 8], bh[0], bh[1]);
        ldsm_x2_t(&sdz2p[1][ks * 16 + (lane & 15)][n8 * 8], bl[0], bl[1]);
        mma_16816(d, ah[0], ah[1], ah[2], ah[3], bh[0], bh[1]);
        mma_16816(d, al[0], al[1], al[2], al[3], bh[0], bh[1]);
        mma_16816(d, ah[0], ah[1], ah[2], ah[3], bl[0], bl[1]);
      }
      float* dst = sdg2 + static_cast<size_t>(hl) * K2 * C;
      dst[(ma * 16 + g) * C + n8 * 8 + 2 * tq] += d[0];
      dst[(ma * 16 + g) * C + n8 * 8 + 2 * tq + 1] += d[1];
      dst[(ma * 16 + g + 8) * C + n8 * 8 + 2 * tq] += d[2];
      dst[(ma * 16 + g + 8) * C + n8 * 8 + 2 * tq + 1] += d[3];
    }
    if (hl + 1 < nh) z2_phase(hl + 1);  // sz2t's readers (the dG3 MMAs of block hl) are done
    if (hl + 1 < nh) continue;
    // dZ1 partial of this h-range: D rows = tokens, columns = aj
#pragma unroll
    for (int u = 0; u < DZT; ++u) {
      const int tl = warp + 8 * u, m = tl / (K2 / 8), n = tl % (K2 / 8);
      const int r0 = m * 16 + g, col = n * 8 + 2 * tq;
      float* base = dz1p + (static_cast<int64_t>(hs) * T + t0) * K2;
      if (r0 < nt) *reinterpret_cast<float2*>(base + static_cast<int64_t>(r0) * K2 + col) = make_float2(dacc[u][0], dacc[u][1]);
      if (r0 + 8 < nt)
        *reinterpret_cast<float2*>(base + static_cast<int64_t>(r0 + 8) * K2 + col) = make_float2(dacc[u][2], dacc[u][3]);
    }
  }
  cp_async_wait<0>();
  __syncthreads();
  // dG3 partial of this CTA: element (col = warp*32 + i*16 + g (+8), c = n8*8 + 2tq (+1))
  float* dst3 = g3part + (static_cast<int64_t>(ts) * gridDim.x + hs) * (C * FB_COLS);
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int n8 = 0; n8 < NT; ++n8) {
      const int col = warp * 32 + i * 16 + g;
      const int c = n8 * 8 + 2 * tq;
      dst3[c * FB_COLS + col] = acc2[i][n8][0];
      dst3[(c + 1) * FB_COLS + col] = acc2[i][n8][1];
      dst3[c * FB_COLS + col + 8] = acc2[i][n8][2];
      dst3[(c + 1) * FB_COLS + col + 8] = acc2[i][n8][3];
    }
  // dG2 partial of token split ts, h in [h0, h0 + nh)
  float* dst2 = g2part + static_cast<int64_t>(ts) * (static_cast<int64_t>(C) * H * J1 * C);
  for (int i = tid; i < nh * K2 * C; i += 256) {
    const int hl = i / (K2 * C), aj = (i / C) % K2, c = i % C;
    const int a = aj / J1, j2 = aj % J1;
    dst2[((static_cast<int64_t>(a) * H + h0 + hl) * J1 + j2) * C + c] = sdg2[i];
  }
}

// ---------------------------------------------------------------------------------------------
// Warp-specialised fused backward for C = 8 (the benchmark's rank).  Same contractions as
// k_tt_bwd_fused, but each warp owns whole output blocks h (local h = warp, warp + 8) and streams
// its own 16-token x 256-column dy blocks through a private 2-slot ring (one TMA box per block, completion on the
// slot's mbarrier; lane 0 issues the next block as soon as the current one has landed), so the only CTA
// barriers are at 16-token tile boundaries (Z1 planes in, dZ1 partials out).  Every intermediate
// of a block stays in registers: the m16n8 D fragments of Z2_h and dZ2_h are re-used as the
// m16n8k8 A fragments (dZ1 += dZ2_h · Gm_hᵀ) and, transposed with movmatrix, as the B fragments
// of dG3 += dy_hᵀ · Z2_h and dG2_h += Z1ᵀ · dZ2_h.  dG3 / dG2 accumulate in registers per warp.
constexpr int WS_TT = 16, WS_NHW = 2, WS_LDZ1 = 40, WS_DYBLK = WS_TT * 256 * 2;

struct WsLayout {  // offsets from the 1024-byte aligned base (bytes() includes the alignment slack)
  static constexpr size_t dy = 0;                       // bf16 [8][2][4 column blocks][TT][64], 128-byte swizzle
  static constexpr size_t dybar = dy + 8 * 2 * WS_DYBLK;                                 // u64 [8][2]
  static constexpr size_t g3 = dybar + 8 * 2 * sizeof(uint64_t);                        // bf16 [8][LDY]
  static constexpr size_t z1p = g3 + sizeof(__nv_bfloat16) * 8 * FB_LDY;                // bf16 [2][TT][LDZ1]
  static constexpr size_t z1raw = z1p + sizeof(__nv_bfloat16) * 2 * WS_TT * WS_LDZ1;    // f32 [2][TT][32]
  static constexpr size_t dzs = z1raw + sizeof(float) * 2 * WS_TT * 32;                 // f32 [8][TT][33]
  static constexpr size_t gmp = dzs + sizeof(float) * 8 * WS_TT * 33;                   // bf16 [2][HR][32][8]
  __host__ __device__ static size_t bytes(int hr) {
    return 1024 + gmp + sizeof(__nv_bfloat16) * 2 * size_t(hr) * 32 * 8;
  }
};

// dy maps of the (up to kBwdJobs) jobs: rows [T, N] as {64 elements, T, N / 64}, box {64, WS_TT, 4}
struct DyMaps {
  CUtensorMap m[kBwdJobs];
};

// dy element (row r, column c, c % 8 == 0) of a warp's 16 x 256 block written by the 3-D TMA box: column block
// c / 64 of 2 KB, 128-byte rows, 16-byte chunks XOR-swizzled by r % 8
QA_DEV uint32_t ws_dy_addr(uint32_t blk, int r, int c) {
  return blk + (c >> 6) * (WS_TT * 128) + r * 128 + ((((c >> 3) & 7) ^ (r & 7)) << 4);
}

// blockIdx.z selects the member of a shared-input group (same H / HR / token split): its dy, Z1, cores and
// partial buffers come from the job table, so the members' dy passes run as one launch
__global__ void __launch_bounds__(256, 1) k_tt_bwd_ws(const BwdJobs jobs, const __grid_constant__ DyMaps maps,
                                                      int64_t T, int H, int HR) {
  constexpr int C = 8, K2 = 32, J1 = 4;
  const int mz = blockIdx.z;
  const __nv_bfloat16* __restrict__ dy = jobs.dy[mz];
  const int64_t ldy = jobs.ldy[mz];
  const float* __restrict__ Z1 = jobs.Z1[mz];
  const float* __restrict__ G2 = jobs.G2[mz];
  const float* __restrict__ G3 = jobs.G3[mz];
  float* __restrict__ dz1p = jobs.dz1p[mz];
  float* __restrict__ g3part = jobs.g3part[mz];
  float* __restrict__ g2part = jobs.g2part[mz];
  extern __shared__ __align__(16) uint8_t ws_smem_raw[];
  uint8_t* ws_smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(ws_smem_raw) + 1023) & ~uintptr_t(1023));
  const CUtensorMap* tmdy = &maps.m[mz];
  uint64_t* dybar = reinterpret_cast<uint64_t*>(ws_smem + WsLayout::dybar);  // [warp][slot]
  const uint32_t sdy0 = smem_u32(ws_smem + WsLayout::dy);
  auto sg3 = reinterpret_cast<__nv_bfloat16(*)[FB_LDY]>(ws_smem + WsLayout::g3);
  auto sz1p = reinterpret_cast<__nv_bfloat16(*)[WS_TT][WS_LDZ1]>(ws_smem + WsLayout::z1p);
  auto sz1raw = reinterpret_cast<float(*)[WS_TT][K2]>(ws_smem + WsLayout::z1raw);
  auto sdzs = reinterpret_cast<float(*)[WS_TT][K2 + 1]>(ws_smem + WsLayout::dzs);
  __nv_bfloat16* sgmp = reinterpret_cast<__nv_bfloat16*>(ws_smem + WsLayout::gmp);
  auto gm = [&](int p, int hl, int aj) -> __nv_bfloat16* {
    return sgmp + ((static_cast<size_t>(p) * HR + hl) * K2 + aj) * C;
  };
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3, q = lane >> 3;
  const int hs = blockIdx.x, ts = blockIdx.y, TS = gridDim.y;
  const int h0 = hs * HR, nh = H - h0 < HR ? H - h0 : HR;
  const int64_t ntiles = (T + WS_TT - 1) / WS_TT;
  const int64_t per = (ntiles + TS - 1) / TS;
  const int64_t tile0 = ts * per, tile1 = tile0 + per < ntiles ? tile0 + per : ntiles;
  const int nmine = nh > warp ? (nh - warp + 7) / 8 : 0;  // this warp's h blocks (<= WS_NHW)
  const int64_t nit = (tile1 > tile0 ? tile1 - tile0 : 0) * nmine;

  for (int i = tid; i < C * FB_COLS; i += 256) sg3[i / FB_COLS][i % FB_COLS] = __float2bfloat16_rn(G3[i]);
  for (int i = tid; i < nh * K2 * C; i += 256) {
    const int hl = i / (K2 * C), aj = (i / C) % K2, c = i % C;
    const int a = aj / J1, j2 = aj % J1;
    const float v = G2[((static_cast<int64_t>(a) * H + h0 + hl) * J1 + j2) * C + c];
    const __nv_bfloat16 hi = __float2bfloat16_rn(v);
    gm(0, hl, aj)[c] = hi;
    gm(1, hl, aj)[c] = __float2bfloat16_rn(v - __bfloat162float(hi));
  }
  if (tid < 16) mbar_init(&dybar[tid], 1);
  fence_barrier_init();
  // one TMA box per (tile, h block) item: the warp's 16 x 256 dy block into its slot (rows past T zero-filled)
  auto load_item = [&](int64_t it, int slot) {
    const int64_t t0 = (tile0 + it / nmine) * WS_TT;
    const int h = h0 + warp + 8 * static_cast<int>(it % nmine);
    __syncwarp();  // every lane's reads of the slot (item it - 2) are done ...
    if (lane == 0) {
      fence_proxy_async_smem();  // ... and ordered before the asynchronous-proxy write
      mbar_arrive_expect_tx(&dybar[warp * 2 + slot], WS_DYBLK);
      tma_load_3d(ws_smem + WsLayout::dy + (warp * 2 + slot) * WS_DYBLK, tmdy, &dybar[warp * 2 + slot], 0,
                  static_cast<int32_t>(t0), 4 * h);
    }
  };
  auto load_z1raw = [&](int64_t tile) {
    if (tile >= tile1 || tid >= WS_TT * K2 / 4) return;
    const int r = tid / (K2 / 4), c4 = tid % (K2 / 4);
    const bool ok = tile * WS_TT + r < T;
    cp_async16(&sz1raw[(tile - tile0) & 1][r][4 * c4], ok ? Z1 + (tile * WS_TT + r) * K2 + 4 * c4 : Z1, ok);
  };
  float acc3[16][4];
#pragma unroll
  for (int m = 0; m < 16; ++m)
#pragma unroll
    for (int k = 0; k < 4; ++k) acc3[m][k] = 0.f;
  float g2acc[WS_NHW][2][4];
#pragma unroll
  for (int i = 0; i < WS_NHW; ++i)
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int k = 0; k < 4; ++k) g2acc[i][m][k] = 0.f;

  __syncthreads();  // barrier inits visible to every warp
  load_z1raw(tile0);
  if (nit > 0) load_item(0, 0);
  cp_async_commit();
  int64_t it = 0;
  for (int64_t tile = tile0; tile < tile1; ++tile) {
    const int64_t t0 = tile * WS_TT;
    const int nt = static_cast<int>(T - t0 < WS_TT ? T - t0 : WS_TT);
    __syncthreads();     // previous tile: Z1 planes and dZ1 partial buffers are free
    cp_async_wait<0>();  // this tile's Z1 rows (and the warp's first dy block) landed ...
    __syncthreads();     // ... for every thread
    for (int i = tid; i < WS_TT * K2; i += 256) {
      const int r = i / K2, aj = i % K2;
      const float f = r < nt ? sz1raw[(tile - tile0) & 1][r][aj] : 0.f;
      const __nv_bfloat16 hi = __float2bfloat16_rn(f);
      sz1p[0][r][aj] = hi;
      sz1p[1][r][aj] = __float2bfloat16_rn(f - __bfloat162float(hi));
    }
    __syncthreads();
    load_z1raw(tile + 1);
    cp_async_commit();
    // Z1 fragments of the tile: A of Z2 = Z1 · Gm (rows t, k = aj) and A of dG2 = Z1ᵀ · dZ2 (rows aj, k = t)
    uint32_t za[2][2][4], zt[2][2][4];
#pragma unroll
    for (int p = 0; p < 2; ++p)
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        ldsm_x4(&sz1p[p][lane & 15][k * 16 + (lane >> 4) * 8], za[p][k][0], za[p][k][1], za[p][k][2], za[p][k][3]);
        ldsm_x4_t(&sz1p[p][(q >> 1) * 8 + (lane & 7)][k * 16 + (q & 1) * 8], zt[p][k][0], zt[p][k][1], zt[p][k][2],
                  zt[p][k][3]);
      }
    float dz1acc[4][4];
#pragma unroll
    for (int n = 0; n < 4; ++n)
#pragma unroll
      for (int k = 0; k < 4; ++k) dz1acc[n][k] = 0.f;
#pragma unroll
    for (int i = 0; i < WS_NHW; ++i, ++it) {
      if (i >= nmine) break;
      const int slot = static_cast<int>(it & 1), hl = warp + 8 * i;
      mbar_wait(&dybar[warp * 2 + slot], static_cast<uint32_t>((it >> 1) & 1));
      if (it + 1 < nit) load_item(it + 1, slot ^ 1);
      const uint32_t dyw = sdy0 + (warp * 2 + slot) * WS_DYBLK;
      // Z2_h = Z1 · Gm_h
      float z2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 2; ++k) {
        uint32_t bh0, bh1, bl0, bl1;
        ldsm_x2_t(gm(0, hl, k * 16 + (lane & 15)), bh0, bh1);
        ldsm_x2_t(gm(1, hl, k * 16 + (lane & 15)), bl0, bl1);
        mma_16816(z2, za[0][k][0], za[0][k][1], za[0][k][2], za[0][k][3], bh0, bh1);
        mma_16816(z2, za[1][k][0], za[1][k][1], za[1][k][2], za[1][k][3], bh0, bh1);
        mma_16816(z2, za[0][k][0], za[0][k][1], za[0][k][2], za[0][k][3], bl0, bl1);
      }
      // dZ2_h = dy_h · G3ᵀ (two accumulator chains, summed in fixed order)
      float e0[4] = {0.f, 0.f, 0.f, 0.f}, e1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        uint32_t a0, a1, a2, a3, b0, b1;
        ldsm_x4_a(ws_dy_addr(dyw, lane & 15, k * 16 + (lane >> 4) * 8), a0, a1, a2, a3);
        ldsm_x2(&sg3[lane & 7][k * 16 + ((lane >> 3) & 1) * 8], b0, b1);
        if (k & 1)
          mma_16816(e1, a0, a1, a2, a3, b0, b1);
        else
          mma_16816(e0, a0, a1, a2, a3, b0, b1);
      }
      float dz2[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) dz2[k] = e0[k] + e1[k];
      // dG3ᵀ[i3, c] += Σ_t dy[t, i3] Z2[t, c]: B = Z2 (k = t, n = c) from the D fragment via movmatrix
      {
        const uint32_t b0 = movm_t(pack_bf16(z2[0], z2[1])), b1 = movm_t(pack_bf16(z2[2], z2[3]));
#pragma unroll
        for (int m = 0; m < 16; ++m) {
          uint32_t a0, a1, a2, a3;
          ldsm_x4_t_a(ws_dy_addr(dyw, (q >> 1) * 8 + (lane & 7), m * 16 + (q & 1) * 8), a0, a1, a2, a3);
          mma_16816(acc3[m], a0, a1, a2, a3, b0, b1);
        }
      }
      // dZ2 as hi / lo bf16: A fragments of m16n8k8 (rows t, k = c) are the D layout itself
      float hv[4];
      uint32_t ah[2], al[2];
#pragma unroll
      for (int k = 0; k < 4; ++k) hv[k] = __bfloat162float(__float2bfloat16_rn(dz2[k]));
      ah[0] = pack_bf16(hv[0], hv[1]);
      ah[1] = pack_bf16(hv[2], hv[3]);
      al[0] = pack_bf16(dz2[0] - hv[0], dz2[1] - hv[1]);
      al[1] = pack_bf16(dz2[2] - hv[2], dz2[3] - hv[3]);
#pragma unroll
      for (int n = 0; n < 4; ++n) {  // dZ1 += dZ2_h · Gm_hᵀ
        uint32_t bh, bl;
        ldsm_x1(gm(0, hl, n * 8 + (lane & 7)), bh);
        ldsm_x1(gm(1, hl, n * 8 + (lane & 7)), bl);
        mma_1688(dz1acc[n], ah[0], ah[1], bh);
        mma_1688(dz1acc[n], al[0], al[1], bh);
        mma_1688(dz1acc[n], ah[0], ah[1], bl);
      }
      {  // dG2_h += Z1ᵀ · dZ2_h: B = dZ2 (k = t, n = c), transposed D fragments
        const uint32_t bh0 = movm_t(ah[0]), bh1 = movm_t(ah[1]), bl0 = movm_t(al[0]), bl1 = movm_t(al[1]);
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          mma_16816(g2acc[i][m], zt[0][m][0], zt[0][m][1], zt[0][m][2], zt[0][m][3], bh0, bh1);
          mma_16816(g2acc[i][m], zt[1][m][0], zt[1][m][1], zt[1][m][2], zt[1][m][3], bh0, bh1);
          mma_16816(g2acc[i][m], zt[0][m][0], zt[0][m][1], zt[0][m][2], zt[0][m][3], bl0, bl1);
        }
      }
    }
    // dZ1 partial of the tile: warp partials -> fixed-order sum
#pragma unroll
    for (int n = 0; n < 4; ++n) {
      sdzs[warp][g][n * 8 + 2 * tq] = dz1acc[n][0];
      sdzs[warp][g][n * 8 + 2 * tq + 1] = dz1acc[n][1];
      sdzs[warp][g + 8][n * 8 + 2 * tq] = dz1acc[n][2];
      sdzs[warp][g + 8][n * 8 + 2 * tq + 1] = dz1acc[n][3];
    }
    __syncthreads();
    for (int i = tid; i < nt * K2; i += 256) {
      const int r = i / K2, aj = i % K2;
      float v = sdzs[0][r][aj];
#pragma unroll
      for (int w = 1; w < 8; ++w) v += sdzs[w][r][aj];
      dz1p[(static_cast<int64_t>(hs) * T + t0 + r) * K2 + aj] = v;
    }
  }
  cp_async_wait<0>();
  // dG2 partial of token split ts for this warp's h blocks (D rows = aj, cols = c)
  float* dst2 = g2part + static_cast<int64_t>(ts) * (static_cast<int64_t>(C) * H * J1 * C);
#pragma unroll
  for (int i = 0; i < WS_NHW; ++i) {
    if (i >= nmine) break;
    const int h = h0 + warp + 8 * i;
#pragma unroll
    for (int m = 0; m < 2; ++m)
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int aj = m * 16 + g + (k >> 1) * 8, c = 2 * tq + (k & 1);
        const int a = aj / J1, j2 = aj % J1;
        dst2[((static_cast<int64_t>(a) * H + h) * J1 + j2) * C + c] = g2acc[i][m][k];
      }
  }
  // dG3 partial of this CTA: per-warp accumulators summed in warp order through shared memory
  __syncthreads();
  float* red = reinterpret_cast<float*>(ws_smem);  // [8][C][256] over the dy ring
#pragma unroll
  for (int m = 0; m < 16; ++m) {
    const int col = m * 16 + g;
    red[(warp * C + 2 * tq) * FB_COLS + col] = acc3[m][0];
    red[(warp * C + 2 * tq + 1) * FB_COLS + col] = acc3[m][1];
    red[(warp * C + 2 * tq) * FB_COLS + col + 8] = acc3[m][2];
    red[(warp * C + 2 * tq + 1) * FB_COLS + col + 8] = acc3[m][3];
  }
  __syncthreads();
  float* dst3 = g3part + (static_cast<int64_t>(ts) * gridDim.x + hs) * (C * FB_COLS);
  for (int i = tid; i < C * FB_COLS; i += 256) {
    float v = red[i];
#pragma unroll
    for (int w = 1; w < 8; ++w) v += red[w * C * FB_COLS + i];
    dst3[i] = v;
  }
}

// Fixed-order reduction of up to three partial sets in one launch, plus (optionally) the B_ext
// operand of the dX GEMM's adapter extension (k_build_bext).
struct ReduceSet {
  const float* part;
  int nparts;
  int64_t numel;
  float* out;
};
constexpr int kRedMembers = 3;  // members of a shared-input group reduced in one launch
struct ReduceArgs {
  ReduceSet set[3 * kRedMembers];
  int64_t blocks[3 * kRedMembers];
  int nsets;
  int accumulate;
  int R1, J1;
  const float* G1s[kRedMembers];  // B_ext jobs: member j's first core and output (null: none)
  __nv_bfloat16* bexts[kRedMembers];
  int64_t bext_blocks;            // blocks per B_ext job
  int64_t K, ldb;
};

__global__ void __launch_bounds__(256) k_grad_reduce3(const ReduceArgs a) {
  __shared__ float red[8][33];
  int64_t b = blockIdx.x;
  int si = 0;
  while (si < a.nsets && b >= a.blocks[si]) b -= a.blocks[si++];
  if (si == a.nsets) {  // B_ext rows of job b / bext_blocks
    const int jb = static_cast<int>(b / a.bext_blocks);
    b -= jb * a.bext_blocks;
    const float* G1 = a.G1s[jb];
    __nv_bfloat16* bext = a.bexts[jb];
    // 8 consecutive columns of one row per thread (ldb % 8 == 0), one 16-byte store; 32-bit index math
    // (K * ldb < 2^31, checked by the launcher)
    const int e0 = (static_cast<int>(b) * 256 + static_cast<int>(threadIdx.x)) * 8;
    if (bext == nullptr || e0 >= static_cast<int>(a.K * a.ldb)) return;
    const int ldb = static_cast<int>(a.ldb);
    const int k = e0 / ldb;
    const int c0 = e0 - k * ldb;
    const int K2 = a.R1 * a.J1;
    const int j1 = k / a.J1, J = k - j1 * a.J1;
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const int c = c0 + q;
      float v = 0.f;
      if (c < 3 * K2) {  // [B_hi | B_hi | B_lo] against [dZ1_hi | dZ1_lo | dZ1_hi]
        const int cc = c % K2;
        const int aa = cc / a.J1, Jp = cc % a.J1;
        if (J == Jp) v = __ldg(G1 + static_cast<int64_t>(j1) * a.R1 + aa);
        if (c >= 2 * K2) v -= __bfloat162float(__float2bfloat16_rn(v));
      }
      const uint32_t h = __bfloat16_as_ushort(__float2bfloat16_rn(v));
      w[q >> 1] = (q & 1) ? (w[q >> 1] | (h << 16)) : h;
    }
    *reinterpret_cast<uint4*>(bext + e0) = make_uint4(w[0], w[1], w[2], w[3]);
    return;
  }
  const ReduceSet& S = a.set[si];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t gi = b * 32 + lane;
  float s = 0.f;
  if (gi < S.numel) {
    // this warp's partials c = warp, warp + 8, ... summed in that order; eight loads in flight per batch
    const float* __restrict__ pp = S.part + gi;
    const int64_t st = S.numel;
    int c = warp;
    for (; c + 56 < S.nparts; c += 64) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldg(pp + static_cast<int64_t>(c + 8 * u) * st);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; c < S.nparts; c += 8) s += __ldg(pp + static_cast<int64_t>(c) * st);
  }
  red[warp][lane] = s;
  __syncthreads();
  if (warp == 0 && gi < S.numel) {
    float t = 0.f;
#pragma unroll
    for (int w = 0; w < 8; ++w) t += red[w][lane];
    S.out[gi] = a.accumulate ? S.out[gi] + t : t;
  }
}

// ---------------------------------------------------------------------------------------------
// x pass of the backward: dG1[j1, a] partial = Σ_{t in split} Σ_J x[t, j1 J1 + J] dZ1[t, a, J]
// dz1 may hold HS partials ([HS][T][K2], summed here in fixed order); when dz1b is given, the CTAs
// of column block 0 also write the [hi | lo | hi | 0] bf16 split of the summed rows (the dX GEMM's
// extension operand, see k_split_rows).
// x pass on the tensor cores (bf16 rows, J1 = 4):
//   dG1[j1, a] = Σ_t Σ_J x[t, 4 j1 + J] dZ1[t, a, J] = Σ_k X'[j1, k] D'[k, a],   k = 4 t + J
// is a GEMM with M = j1, N = a and a reduction over (token, J): the A fragment of an m16n8k16 MMA
// needs, per lane, the bf16 pair x[t, 4 j1 + J .. + 1] — one 32-bit shared-memory load — and the
// B fragment the pair dZ1[t, a, J .. J + 1] of the [t][a][J] staged dZ1 rows.  x is exact in bf16;
// dZ1 enters as hi + lo bf16 (two MMAs), so the sums keep fp32-class accuracy.  A CTA owns 1024
// columns (16 m-tiles, 2 per warp) of a token range, streamed through a ring of 16-token stages (one TMA box per
// stage, mbarrier completion); dZ1 is staged per 64 tokens (HS partials summed in fixed order), and CTAs of
// column block 0 also emit the [hi | lo | hi | 0] split rows the dX GEMM's extension reads.
constexpr int DM_COLS = 1024, DM_LDX = DM_COLS + 32, DM_ST = 16, DM_NSTG = 4, DM_DZT = 64;
constexpr int DM_XST = DM_ST * DM_COLS * 2;  // bytes of one x stage (16 tokens x 1024 columns, one TMA box)

// x stage element (row r, column c) of the 3-D TMA box {64, 16, 16}: column block c / 64 of 2 KB, 128-byte rows,
// 16-byte chunks XOR-swizzled by r % 8
QA_DEV uint32_t dm_x_addr(uint32_t stage, int r, int c) {
  return stage + (c >> 6) * (DM_ST * 128) + r * 128 + ((((c >> 3) & 7) ^ (r & 7)) << 4) + ((c & 7) << 1);
}

// NA adapters sharing x (a decoder layer's q / k / v or up / gate) run in one pass: per adapter its
// own dZ1 planes, B fragments and accumulators.
struct DgAdapters {
  const float* dz1[3];
  float* part[3];
  __nv_bfloat16* dz1b[3];
};

template <int R1, int NA = 1>
__global__ void __launch_bounds__(256, 2) k_tt_dg1m(const __grid_constant__ CUtensorMap tmx,
                                                    const __nv_bfloat16* __restrict__ x, int64_t T, int64_t K,
                                                    const DgAdapters ad, int S, int HS, int64_t ldb, int raw_async,
                                                    int nstg, int x3d) {
  constexpr int J1 = 4, K2 = J1 * R1, NN = R1 / 8;
  extern __shared__ __align__(16) uint8_t dm_smem[];
  // x ring: nstg TMA stages (1024-byte aligned) and their mbarriers inside the XS_BYTES region
  const size_t XS_BYTES = sizeof(__nv_bfloat16) * nstg * DM_ST * DM_LDX;  // >= 1024 + nstg * (DM_XST + 8)
  uint8_t* xring = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dm_smem) + 1023) & ~uintptr_t(1023));
  uint64_t* xbar = reinterpret_cast<uint64_t*>(xring + static_cast<size_t>(nstg) * DM_XST);
  const uint32_t xring_s = smem_u32(xring);
  auto dzs = reinterpret_cast<__nv_bfloat16(*)[DM_DZT][R1][J1]>(dm_smem + XS_BYTES);  // [NA][2 planes]
  // raw fp32 dZ1 partials of the next 64-token blocks, prefetched by cp.async: [2][NA][HS][DZT][K2]
  float* raw = reinterpret_cast<float*>(dm_smem + XS_BYTES + sizeof(__nv_bfloat16) * NA * 2 * DM_DZT * R1 * J1);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, tq = lane & 3;
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * DM_COLS;
  const int s = blockIdx.y;
  const int64_t per = (T + S - 1) / S;
  const int64_t t0 = s * per, t1 = t0 + per < T ? t0 + per : T;
  const int64_t nst = t1 > t0 ? (t1 - t0 + DM_ST - 1) / DM_ST : 0;
  constexpr int SPB = DM_DZT / DM_ST;  // stages per dZ1 block
  float acc[2][NA * NN][4];
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < NA * NN; ++n)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[m][n][q] = 0.f;
  auto issue_raw = [&](int64_t blk) {  // 16-byte pieces of HS x [DZT][K2] fp32 rows (tokens past t1 are zero)
    const int64_t tb = t0 + blk * DM_DZT;
    if (tb >= t1) return;
#pragma unroll
    for (int aa = 0; aa < NA; ++aa) {
      float* dst = raw + (static_cast<size_t>(blk & 1) * NA + aa) * HS * DM_DZT * K2;
      const float* dz1 = ad.dz1[aa];
      for (int i = tid; i < HS * DM_DZT * (K2 / 4); i += 256) {
        const int h = i / (DM_DZT * (K2 / 4)), r = (i / (K2 / 4)) % DM_DZT, q = i % (K2 / 4);
        const bool ok = tb + r < t1;
        cp_async16(dst + (static_cast<size_t>(h) * DM_DZT + r) * K2 + 4 * q,
                   ok ? dz1 + (static_cast<int64_t>(h) * T + tb + r) * K2 + 4 * q : dz1, ok);
      }
    }
  };
  if (tid == 0) {
    for (int i = 0; i < nstg; ++i) mbar_init(&xbar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // stage k: 16 tokens x 1024 columns as up to 16 TMA boxes of 64 columns (128-byte swizzle) issued by one thread;
  // columns past K and rows past T are zero-filled, blocks wholly past K are not loaded (their j1 rows are never
  // stored), rows of the next split past t1 meet zero dZ1 rows
  const int ncb = static_cast<int>((K - c0 + 63) / 64 < 16 ? (K - c0 + 63) / 64 : 16);
  auto issue = [&](int64_t k) {
    if (k < nst && tid == 0) {
      const int slot = static_cast<int>(k % nstg);
      fence_proxy_async_smem();  // the slot's previous readers (behind the CTA barrier) before the async write
      if (x3d) {  // K % 64 == 0: the whole stage as one box {64, 16, 16} of the view {64, T, K / 64}
        mbar_arrive_expect_tx(&xbar[slot], DM_XST);
        tma_load_3d(xring + static_cast<size_t>(slot) * DM_XST, &tmx, &xbar[slot], 0,
                    static_cast<int32_t>(t0 + k * DM_ST), static_cast<int32_t>(c0 / 64));
      } else {
        mbar_arrive_expect_tx(&xbar[slot], static_cast<uint32_t>(ncb) * DM_ST * 128);
        for (int cb = 0; cb < ncb; ++cb)
          tma_load_2d(xring + static_cast<size_t>(slot) * DM_XST + cb * (DM_ST * 128), &tmx, &xbar[slot],
                      static_cast<int32_t>(c0 + 64 * cb), static_cast<int32_t>(t0 + k * DM_ST));
      }
    }
  };
  if (raw_async) issue_raw(0);
  for (int k = 0; k < nstg - 1; ++k) {
    issue(k);
    cp_async_commit();
  }
  for (int64_t k = 0; k < nst; ++k) {
    const int slot = static_cast<int>(k % nstg);
    cp_async_wait_dyn(nstg - 2);
    mbar_wait(&xbar[slot], static_cast<uint32_t>((k / nstg) & 1));
    __syncthreads();  // stage k (and its dZ1 block) visible to all warps; stage k - 1's readers are done
    if (k % SPB == 0) {  // dZ1 rows of the next 64 tokens: HS partials summed, hi / lo planes, [t][a][J]
      const int64_t blk = k / SPB, tb = t0 + k * DM_ST;
      const int nt = static_cast<int>(t1 - tb < DM_DZT ? t1 - tb : DM_DZT);
      // element i = tid + 256 u of the [NA][DZT][K2] block: adapter u / PA, row (i / K2) % DZT, column tid % K2.
      // One partial plane (HS == 1, every N <= 4096): all reads are issued before any is used, one round trip per
      // block (q / k / v x pass 82 -> 51 us); several planes: each element's planes read together, element by
      // element (measured faster there: up / gate, HS = 3, 74 us against 91 us batched plane by plane).
      constexpr int PER = NA * DM_DZT * K2 / 256, PA = PER / NA;
      float vv[PER];
      if (!raw_async && HS == 1) {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int aa = u / PA, i = tid + 256 * u, r = (i / K2) % DM_DZT, cc = i % K2;
          vv[u] = r < nt ? __ldg(ad.dz1[aa] + (tb + r) * K2 + cc) : 0.f;
        }
      } else {
#pragma unroll
        for (int u = 0; u < PER; ++u) {
          const int aa = u / PA, i = tid + 256 * u, r = (i / K2) % DM_DZT, cc = i % K2;
          float v = 0.f;
          if (r < nt) {
            if (raw_async) {
              const float* rb = raw + (static_cast<size_t>(blk & 1) * NA + aa) * HS * DM_DZT * K2;
              v = rb[r * K2 + cc];
              for (int h = 1; h < HS; ++h) v += rb[(static_cast<size_t>(h) * DM_DZT + r) * K2 + cc];
            } else {
              const int64_t off = (tb + r) * K2 + cc;
              v = ad.dz1[aa][off];
              for (int h = 1; h < HS; ++h) v += ad.dz1[aa][static_cast<int64_t>(h) * T * K2 + off];
            }
          }
          vv[u] = v;
        }
      }
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const int aa = u / PA, i = tid + 256 * u, r = (i / K2) % DM_DZT, cc = i % K2;  // cc = a * J1 + J
        const float v = vv[u];
        const __nv_bfloat16 hi = __float2bfloat16_rn(v);
        dzs[2 * aa][r][cc / J1][cc % J1] = hi;
        dzs[2 * aa + 1][r][cc / J1][cc % J1] = __float2bfloat16_rn(v - __bfloat162float(hi));
        __nv_bfloat16* dz1b = ad.dz1b[aa];
        if (dz1b != nullptr && blockIdx.x == 0 && r < nt) {  // [hi | lo | hi] split row for the dX GEMM
          __nv_bfloat16* row = dz1b + (tb + r) * ldb;
          row[cc] = hi;
          row[K2 + cc] = __float2bfloat16_rn(v - __bfloat162float(hi));
          row[2 * K2 + cc] = hi;
          if (cc < ldb - 3 * K2) row[3 * K2 + cc] = __float2bfloat16_rn(0.f);
        }
      }
      if (blockIdx.x == 0 && ldb - 3 * K2 > K2)
        for (int i = tid; i < NA * nt * static_cast<int>(ldb - 4 * K2); i += 256) {
          const int w4 = static_cast<int>(ldb - 4 * K2);
          const int aa = i / (nt * w4), r = (i / w4) % nt, c = i % w4;
          if (ad.dz1b[aa] != nullptr) ad.dz1b[aa][(tb + r) * ldb + 4 * K2 + c] = __float2bfloat16_rn(0.f);
        }
      __syncthreads();
    }
    issue(k + nstg - 1);  // into the slot stage k - 1 used
    if (raw_async && k % SPB == 1) issue_raw(k / SPB + 1);  // complete by the next block's first stage
    cp_async_commit();
    const int zr = static_cast<int>(k % SPB) * DM_ST;
    const uint32_t xst = xring_s + static_cast<uint32_t>(slot) * DM_XST;
#pragma unroll
    for (int ks = 0; ks < DM_ST / 4; ++ks) {  // 4 tokens x 4 J per k-step
      // the k-step's tokens: stage rows r0 (k 0..7) and r0 + 1 (k 8..15) for lane pair s = tq / 2 at rows 4 apart,
      // so a quarter-warp's two rows have swizzle keys differing in bit 2 (conflict-free 32-bit reads); the B
      // fragments read the dZ1 rows of the same tokens
      const int r0 = 8 * (ks >> 1) + 4 * (tq >> 1) + 2 * (ks & 1), J = 2 * (tq & 1);
      uint32_t bh[NA * NN][2], bl[NA * NN][2];
#pragma unroll
      for (int n = 0; n < NA * NN; ++n) {
        const int aa = n / NN, nn = n % NN;
        bh[n][0] = *reinterpret_cast<const uint32_t*>(&dzs[2 * aa][zr + r0][nn * 8 + g][J]);
        bh[n][1] = *reinterpret_cast<const uint32_t*>(&dzs[2 * aa][zr + r0 + 1][nn * 8 + g][J]);
        bl[n][0] = *reinterpret_cast<const uint32_t*>(&dzs[2 * aa + 1][zr + r0][nn * 8 + g][J]);
        bl[n][1] = *reinterpret_cast<const uint32_t*>(&dzs[2 * aa + 1][zr + r0 + 1][nn * 8 + g][J]);
      }
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        const int jl = (warp * 2 + m) * 16 + g;
        const uint32_t a0 = lds32(dm_x_addr(xst, r0, 4 * jl + J));
        const uint32_t a1 = lds32(dm_x_addr(xst, r0, 4 * (jl + 8) + J));
        const uint32_t a2 = lds32(dm_x_addr(xst, r0 + 1, 4 * jl + J));
        const uint32_t a3 = lds32(dm_x_addr(xst, r0 + 1, 4 * (jl + 8) + J));
#pragma unroll
        for (int n = 0; n < NA * NN; ++n) {
          mma_16816(acc[m][n], a0, a1, a2, a3, bh[n][0], bh[n][1]);
          mma_16816(acc[m][n], a0, a1, a2, a3, bl[n][0], bl[n][1]);
        }
      }
    }
  }
  cp_async_wait<0>();
  const int64_t nj1 = K / J1;
#pragma unroll
  for (int m = 0; m < 2; ++m)
#pragma unroll
    for (int n = 0; n < NA * NN; ++n) {
      float* dst = ad.part[n / NN] + static_cast<int64_t>(s) * (K / J1) * R1;
      const int64_t j1 = c0 / J1 + (warp * 2 + m) * 16 + g;
      const int a = (n % NN) * 8 + 2 * tq;
      if (j1 < nj1) {
        dst[j1 * R1 + a] = acc[m][n][0];
        dst[j1 * R1 + a + 1] = acc[m][n][1];
      }
      if (j1 + 8 < nj1) {
        dst[(j1 + 8) * R1 + a] = acc[m][n][2];
        dst[(j1 + 8) * R1 + a + 1] = acc[m][n][3];
      }
    }
}

template <typename InT, int J1, int R1>
__global__ void __launch_bounds__(256) k_tt_dg1(const InT* __restrict__ x, int64_t T, int64_t K,
                                                const float* __restrict__ dz1, float* __restrict__ part, int S,
                                                int HS, __nv_bfloat16* __restrict__ dz1b, int64_t ldb) {
  constexpr int K2 = J1 * R1;
  constexpr int E = J1 == 1 ? 4 : 8;  // x elements per thread
  constexpr int NJ = E / J1;
  constexpr int TB = 32;
  static_assert(R1 % 4 == 0, "R1");
  __shared__ __align__(16) float sdz[TB][J1][R1];  // dZ1 rows as [t][J][a]: (a, a+1) pairs adjacent for FFMA2
  const int64_t col0 = (static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x) * E;
  const bool active = col0 < K;
  const int s = blockIdx.y;
  const int64_t per = (T + S - 1) / S;
  const int64_t t0 = s * per, t1 = t0 + per < T ? t0 + per : T;
  unsigned long long acc[NJ][R1 / 2];
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int a = 0; a < R1 / 2; ++a) acc[j][a] = 0ull;
  for (int64_t tb = t0; tb < t1; tb += TB) {
    const int nt = static_cast<int>(t1 - tb < TB ? t1 - tb : TB);
    __syncthreads();
    for (int i = threadIdx.x; i < nt * K2; i += 256) {
      const int r = i / K2, cc = i % K2;
      const int64_t off = (tb + r) * K2 + cc;
      float v = dz1[off];
      for (int h = 1; h < HS; ++h) v += dz1[static_cast<int64_t>(h) * T * K2 + off];
      sdz[r][cc % J1][cc / J1] = v;
    }
    __syncthreads();
    if (dz1b != nullptr && blockIdx.x == 0) {
      for (int i = threadIdx.x; i < nt * static_cast<int>(ldb); i += 256) {
        const int r = i / static_cast<int>(ldb), c = i % static_cast<int>(ldb);
        float v = 0.f;
        if (c < 3 * K2) {  // [hi | lo | hi]
          const int cc = c % K2;
          const float f = sdz[r][cc % J1][cc / J1];
          v = __bfloat162float(__float2bfloat16_rn(f));
          if (c >= K2 && c < 2 * K2) v = f - v;
        }
        dz1b[(tb + r) * ldb + c] = __float2bfloat16_rn(v);
      }
    }
    if (!active) continue;
    constexpr int UNR = 4;  // token rows of x in flight per thread
    for (int r0 = 0; r0 < nt; r0 += UNR) {
      float f[UNR][8];
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (r0 + u < nt) {
          if (E == 8) {
            load8<InT>(x + (tb + r0 + u) * K + col0, f[u]);
          } else {
#pragma unroll
            for (int i = 0; i < 4; ++i) f[u][i] = to_f32(x[(tb + r0 + u) * K + col0 + i]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < UNR; ++u) {
        if (r0 + u >= nt) break;
#pragma unroll
        for (int J = 0; J < J1; ++J) {
          const float4* dz4 = reinterpret_cast<const float4*>(&sdz[r0 + u][J][0]);
          float4 d4[R1 / 4];
#pragma unroll
          for (int q = 0; q < R1 / 4; ++q) d4[q] = dz4[q];
#pragma unroll
          for (int j = 0; j < NJ; ++j) {
            const float xv = f[u][j * J1 + J];
            const unsigned long long xx = f2pack(xv, xv);
#pragma unroll
            for (int q = 0; q < R1 / 4; ++q) {
              ffma2(acc[j][2 * q], xx, f2pack(d4[q].x, d4[q].y));
              ffma2(acc[j][2 * q + 1], xx, f2pack(d4[q].z, d4[q].w));
            }
          }
        }
      }
    }
  }
  if (!active) return;
  const int64_t n1 = K / J1;
  float* dst = part + static_cast<int64_t>(s) * n1 * R1;
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int a = 0; a < R1 / 2; ++a) {
      dst[(col0 / J1 + j) * R1 + 2 * a] = f2lo(acc[j][a]);
      dst[(col0 / J1 + j) * R1 + 2 * a + 1] = f2hi(acc[j][a]);
    }
}

// ---------------------------------------------------------------------------------------------
// Middle core (d = 3) as register-tiled small GEMMs over token tiles of 64.  G2 [R1][H][J1][C]
// is gathered once per CTA into shared memory as the dense matrix Gm[aj][hc] (aj = a*J1 + j2,
// hc = i2*C + b), or its transpose.
//   fwd : Z2 = Z1 · Gm                 [T, HC]
//   bwd : dZ1 = dZ2 · Gmᵀ              [T, K2]   and   dG2 (+)= Z1ᵀ · dZ2 (per-CTA partial)
constexpr int MID_TT = 64, MID_LD = MID_TT + 4;

QA_DEV int g2_index(int aj, int hc, int J1, int C, int HC) {
  const int a = aj / J1, j2 = aj % J1, i2 = hc / C, b = hc % C;
  return ((a * (HC / C) + i2) * J1 + j2) * C + b;
}

__global__ void __launch_bounds__(256) k_mid_fwd(const float* __restrict__ z1, int64_t T, int K2, int J1, int HC,
                                                 int C, const float* __restrict__ G2, float* __restrict__ z2) {
  extern __shared__ __align__(16) float mid_smem[];
  float* gm = mid_smem;                  // [K2][HC]
  float* zt = mid_smem + K2 * HC;        // [K2][MID_LD]  (Z1 tile, transposed)
  for (int i = threadIdx.x; i < K2 * HC; i += 256) gm[i] = G2[g2_index(i / HC, i % HC, J1, C, HC)];
  const int64_t t0 = static_cast<int64_t>(blockIdx.x) * MID_TT;
  const int nt = static_cast<int>(T - t0 < MID_TT ? T - t0 : MID_TT);
  for (int i = threadIdx.x; i < MID_TT * K2; i += 256) {
    const int r = i / K2, aj = i % K2;
    zt[aj * MID_LD + r] = r < nt ? z1[(t0 + r) * K2 + aj] : 0.f;
  }
  __syncthreads();
  const int ntile = (MID_TT / 4) * (HC / 4);
  for (int mt = threadIdx.x; mt < ntile; mt += 256) {
    const int r0 = (mt % (MID_TT / 4)) * 4, c0 = (mt / (MID_TT / 4)) * 4;
    float acc[4][4] = {};
    for (int aj = 0; aj < K2; ++aj) {
      const float4 zv = *reinterpret_cast<const float4*>(zt + aj * MID_LD + r0);
      const float4 gv = *reinterpret_cast<const float4*>(gm + aj * HC + c0);
      const float zz[4] = {zv.x, zv.y, zv.z, zv.w}, gg[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(zz[i], gg[j], acc[i][j]);
    }
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (r0 + i < nt)
        *reinterpret_cast<float4*>(z2 + (t0 + r0 + i) * HC + c0) = make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
  }
}

template <int MAXT>  // dG2 micro-tiles (4 x 4) per thread
__global__ void __launch_bounds__(256) k_mid_bwd(const float* __restrict__ dz2, const float* __restrict__ z1,
                                                 int64_t T, int K2, int J1, int HC, int C,
                                                 const float* __restrict__ G2, float* __restrict__ dz1,
                                                 float* __restrict__ gpart, int tiles_per_cta) {
  extern __shared__ __align__(16) float mid_smem[];
  float* gt = mid_smem;                        // [HC][K2]
  float* dt = mid_smem + HC * K2;              // [HC][MID_LD]  dZ2 tile, transposed
  float* zt = dt + HC * MID_LD;                // [K2][MID_LD]  Z1 tile, transposed
  for (int i = threadIdx.x; i < K2 * HC; i += 256) gt[i] = G2[g2_index(i % K2, i / K2, J1, C, HC)];
  const bool want_g = gpart != nullptr;
  const int gtiles = (K2 / 4) * (HC / 4);
  float gacc[MAXT][4][4];
#pragma unroll
  for (int u = 0; u < MAXT; ++u)
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) gacc[u][i][j] = 0.f;
  for (int tile = 0; tile < tiles_per_cta; ++tile) {
    const int64_t t0 = (static_cast<int64_t>(blockIdx.x) * tiles_per_cta + tile) * MID_TT;
    if (t0 >= T) break;
    const int nt = static_cast<int>(T - t0 < MID_TT ? T - t0 : MID_TT);
    __syncthreads();
    for (int i = threadIdx.x; i < MID_TT * HC; i += 256) {
      const int r = i / HC, hc = i % HC;
      dt[hc * MID_LD + r] = r < nt ? dz2[(t0 + r) * HC + hc] : 0.f;
    }
    if (want_g)
      for (int i = threadIdx.x; i < MID_TT * K2; i += 256) {
        const int r = i / K2, aj = i % K2;
        zt[aj * MID_LD + r] = r < nt ? z1[(t0 + r) * K2 + aj] : 0.f;
      }
    __syncthreads();
    // dZ1 tile [64 x K2]: micro-tile 4 tokens x 4 aj
    for (int mt = threadIdx.x; mt < (MID_TT / 4) * (K2 / 4); mt += 256) {
      const int r0 = (mt % (MID_TT / 4)) * 4, c0 = (mt / (MID_TT / 4)) * 4;
      float acc[4][4] = {};
      for (int hc = 0; hc < HC; ++hc) {
        const float4 dv = *reinterpret_cast<const float4*>(dt + hc * MID_LD + r0);
        const float4 gv = *reinterpret_cast<const float4*>(gt + hc * K2 + c0);
        const float dd[4] = {dv.x, dv.y, dv.z, dv.w}, gg[4] = {gv.x, gv.y, gv.z, gv.w};
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(dd[i], gg[j], acc[i][j]);
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (r0 + i < nt)
          *reinterpret_cast<float4*>(dz1 + (t0 + r0 + i) * K2 + c0) =
              make_float4(acc[i][0], acc[i][1], acc[i][2], acc[i][3]);
    }
    // dG2 partial [K2 x HC] += Z1ᵀ · dZ2 over this tile's tokens: micro-tile 4 aj x 4 hc
    if (want_g) {
#pragma unroll
      for (int u = 0; u < MAXT; ++u) {
        const int mt = threadIdx.x + 256 * u;
        if (mt >= gtiles) break;
        const int a0 = (mt % (K2 / 4)) * 4, h0 = (mt / (K2 / 4)) * 4;
        for (int r = 0; r < MID_TT; r += 4) {
          float4 zv[4], dv[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) zv[i] = *reinterpret_cast<const float4*>(zt + (a0 + i) * MID_LD + r);
#pragma unroll
          for (int j = 0; j < 4; ++j) dv[j] = *reinterpret_cast<const float4*>(dt + (h0 + j) * MID_LD + r);
#pragma unroll
          for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j)
              gacc[u][i][j] = fmaf(zv[i].x, dv[j].x,
                                   fmaf(zv[i].y, dv[j].y, fmaf(zv[i].z, dv[j].z, fmaf(zv[i].w, dv[j].w, gacc[u][i][j]))));
        }
      }
    }
  }
  if (want_g) {
    const int numel = K2 * HC;
#pragma unroll
    for (int u = 0; u < MAXT; ++u) {
      const int mt = threadIdx.x + 256 * u;
      if (mt >= gtiles) break;
      const int a0 = (mt % (K2 / 4)) * 4, h0 = (mt / (K2 / 4)) * 4;
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j)
          gpart[static_cast<int64_t>(blockIdx.x) * numel + g2_index(a0 + i, h0 + j, J1, C, HC)] = gacc[u][i][j];
    }
  }
}

}  // namespace

size_t mid_fwd_smem(int K2, int HC) { return sizeof(float) * (size_t(K2) * HC + size_t(K2) * MID_LD); }
size_t mid_bwd_smem(int K2, int HC) {
  return sizeof(float) * (size_t(K2) * HC + size_t(HC) * MID_LD + size_t(K2) * MID_LD);
}

bool mid_fast_ok(int K2, int HC) {
  return K2 % 4 == 0 && HC % 4 == 0 && (K2 / 4) * (HC / 4) <= 256 * 4 && mid_bwd_smem(K2, HC) <= 200 * 1024;
}

int mid_bwd_ctas(int64_t T) {
  const int64_t tiles = (T + MID_TT - 1) / MID_TT;
  return static_cast<int>(tiles < 148 ? (tiles > 0 ? tiles : 1) : 148);
}

cudaError_t launch_mid_fwd(const float* z1, int64_t T, int K2, int J1, int HC, int C, const float* G2, float* z2,
                           cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  LaunchScope scope(kTT, 2.0 * double(T) * K2 * HC, s);
  count_launches(1);
  const unsigned grid = static_cast<unsigned>((T + MID_TT - 1) / MID_TT);
  const size_t smem = mid_fwd_smem(K2, HC);
  cudaFuncSetAttribute(k_mid_fwd, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k_mid_fwd<<<grid, 256, smem, s>>>(z1, T, K2, J1, HC, C, G2, z2);
  return cudaGetLastError();
}

cudaError_t launch_mid_bwd(const float* dz2, const float* z1, int64_t T, int K2, int J1, int HC, int C,
                           const float* G2, float* dz1, float* gpart, int nctas, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  LaunchScope scope(kTT, 2.0 * double(T) * K2 * HC * (gpart ? 2 : 1), s);
  count_launches(1);
  const int64_t tiles = (T + MID_TT - 1) / MID_TT;
  const int per = static_cast<int>((tiles + nctas - 1) / nctas);
  const size_t smem = mid_bwd_smem(K2, HC);
  const int gtiles = (K2 / 4) * (HC / 4);
#define QA_MB(U)                                                                                                    cudaFuncSetAttribute(k_mid_bwd<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));        k_mid_bwd<U><<<static_cast<unsigned>(nctas), 256, smem, s>>>(dz2, z1, T, K2, J1, HC, C, G2, dz1, gpart, per)
  if (gtiles <= 256) {
    QA_MB(1);
  } else if (gtiles <= 512) {
    QA_MB(2);
  } else {
    QA_MB(4);
  }
#undef QA_MB
  return cudaGetLastError();
}

bool fast_tt_supported(int J1, int R1) {
  return (J1 == 1 && (R1 == 8 || R1 == 16)) || (J1 == 4 && (R1 == 8 || R1 == 16));
}

size_t g1i_floats(int64_t K, int J1, int R1) {
  const int64_t nvec = K / 8;
  return static_cast<size_t>(((nvec + 31) / 32) * 32) * 8 * R1 / J1 * 2;  // >= the k_g1_frag fragments
}

bool actquant_frag_path(int x_dtype, int64_t K, int J1, int R1, const void* x, bool want_codes, int64_t ldc,
                        const void* codes, const void* zf) {
  return x_dtype == QA_BF16 && K % 64 == 0 && (J1 == 1 || J1 == 4) && (R1 == 8 || R1 == 16) &&
         reinterpret_cast<uintptr_t>(x) % 16 == 0 &&
         (!want_codes || (ldc % 16 == 0 && reinterpret_cast<uintptr_t>(codes) % 16 == 0)) &&
         (zf == nullptr || reinterpret_cast<uintptr_t>(zf) % 16 == 0);
}

cudaError_t launch_actquant_z1(const void* x, int x_dtype, int64_t T, int64_t K, bool want_codes, uint8_t* codes,
                               int64_t ldc, float* sx, float* ox, int32_t* rsx, const float* G1, int J1, int R1,
                               __nv_bfloat16* zb, int64_t ldzb, float* zf, float* g1i_ws, cudaStream_t s,
                               bool frag_ready) {
  if (T == 0) return cudaSuccess;
  const int64_t nvec = K / 8;
  // ---- production path: CTA-per-8-token kernel, rows read straight from global memory
  if (actquant_frag_path(x_dtype, K, J1, R1, x, want_codes, ldc, codes, zf)) {
    const int MT = R1 / 8;
    const int64_t nfrag = (J1 == 4 ? K / 64 : K / 16);
    if (!frag_ready) {
      LaunchScope scope(kTT, double(nfrag) * MT * 32 * 16 + double(K) * R1 * 4, s);
      count_launches(1);
      const int64_t n = nfrag * MT * 32;
      const unsigned gr = static_cast<unsigned>((n + 255) / 256);
      uint4* fr = reinterpret_cast<uint4*>(g1i_ws);
      if (J1 == 1 && R1 == 8)
        k_g1_frag<1, 8><<<gr, 256, 0, s>>>(G1, fr, nfrag);
      else if (J1 == 1)
        k_g1_frag<1, 16><<<gr, 256, 0, s>>>(G1, fr, nfrag);
      else if (R1 == 8)
        k_g1_frag<4, 8><<<gr, 256, 0, s>>>(G1, fr, nfrag);
      else
        k_g1_frag<4, 16><<<gr, 256, 0, s>>>(G1, fr, nfrag);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
    }
    LaunchScope scope(kQuantize, double(T) * K * 2 + (want_codes ? double(T) * ldc + 12.0 * T : 0.0) +
                                     double(T) * (zb ? ldzb * 2 : 0) + double(T) * (zf ? J1 * R1 * 4 : 0),
                      s);
    count_launches(1);
    const uint4* fr = reinterpret_cast<const uint4*>(g1i_ws);
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    const int64_t ngroups = (T + 7) / 8;
    const size_t frag_bytes = static_cast<size_t>(nfrag) * MT * 32 * 16;
    const bool fsmem = frag_bytes <= 48 * 1024;
    const size_t smem = fsmem ? frag_bytes : 0;
#define QA_AQC(JJ, RR, CC, FS)                                                                                  \
  {                                                                                                             \
    auto kern = k_aq_cta<JJ, RR, CC, FS>;                                                                       \
    int per_sm = 1;                                                                                             \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, AQC_WARPS * 32, smem);                          \
    const int64_t cap = static_cast<int64_t>(per_sm < 1 ? 1 : per_sm) * nsm;                                    \
    const unsigned grid = static_cast<unsigned>(ngroups < cap ? ngroups : cap);                                 \
    kern<<<grid, AQC_WARPS * 32, smem, s>>>(static_cast<const __nv_bfloat16*>(x), T, K, codes, ldc, sx, ox, rsx, \
                                            fr, AqAdapters{{zb, nullptr, nullptr}, {zf, nullptr, nullptr}, 0}, ldzb); \
  }
#define QA_AQC_C(JJ, RR)          \
  if (want_codes) {               \
    if (fsmem)                    \
      QA_AQC(JJ, RR, true, true)  \
    else                          \
      QA_AQC(JJ, RR, true, false) \
  } else {                        \
    if (fsmem)                    \
      QA_AQC(JJ, RR, false, true) \
    else                          \
      QA_AQC(JJ, RR, false, false) \
  }
    if (J1 == 1 && R1 == 8)
      QA_AQC_C(1, 8)
    else if (J1 == 1)
      QA_AQC_C(1, 16)
    else if (R1 == 8)
      QA_AQC_C(4, 8)
    else
      QA_AQC_C(4, 16)
#undef QA_AQC_C
#undef QA_AQC
    return cudaGetLastError();
  }
  {
    const int64_t n = nvec * 2 * R1 / J1;
    LaunchScope scope(kTT, double(n) * 32, s);
    count_launches(1);
    const unsigned g = static_cast<unsigned>((n + 255) / 256);
    float4* G1i = reinterpret_cast<float4*>(g1i_ws);
    if (J1 == 1 && R1 == 8)
      k_g1_interleave<1, 8><<<g, 256, 0, s>>>(G1, G1i, nvec);
    else if (J1 == 1 && R1 == 16)
      k_g1_interleave<1, 16><<<g, 256, 0, s>>>(G1, G1i, nvec);
    else if (J1 == 4 && R1 == 8)
      k_g1_interleave<4, 8><<<g, 256, 0, s>>>(G1, G1i, nvec);
    else
      k_g1_interleave<4, 16><<<g, 256, 0, s>>>(G1, G1i, nvec);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  const float4* G1i = reinterpret_cast<const float4*>(g1i_ws);
  const size_t esz = x_dtype == QA_F32 ? 4 : 2;
  LaunchScope scope(kQuantize, double(T) * K * esz + (want_codes ? double(T) * ldc + 12.0 * T : 0.0) +
                                   double(T) * (zb ? ldzb * 2 : 0) + double(T) * (zf ? J1 * R1 * 4 : 0),
                    s);
  count_launches(1);
  const dim3 grid(static_cast<unsigned>((T + 7) / 8));  // 8 warps = 8 token rows per CTA
#define QA_AQ(TI, JJ, RR)                                                                                           \
  if (want_codes)                                                                                                   \
    k_actquant_z1<TI, JJ, RR, true><<<grid, 256, 0, s>>>(static_cast<const TI*>(x), T, K, codes, ldc, sx, ox, rsx,  \
                                                         G1i, zb, ldzb, zf);                                        \
  else                                                                                                              \
    k_actquant_z1<TI, JJ, RR, false><<<grid, 256, 0, s>>>(static_cast<const TI*>(x), T, K, codes, ldc, sx, ox, rsx, \
                                                          G1i, zb, ldzb, zf);
#define QA_AQ_T(TI)                  \
  if (J1 == 1 && R1 == 8) {          \
    QA_AQ(TI, 1, 8)                  \
  } else if (J1 == 1 && R1 == 16) {  \
    QA_AQ(TI, 1, 16)                 \
  } else if (J1 == 4 && R1 == 8) {   \
    QA_AQ(TI, 4, 8)                  \
  } else {                           \
    QA_AQ(TI, 4, 16)                 \
  }
  if (x_dtype == QA_F32) {
    QA_AQ_T(float)
  } else {
    QA_AQ_T(__nv_bfloat16)
  }
#undef QA_AQ_T
#undef QA_AQ
  return cudaGetLastError();
}

cudaError_t launch_adapter_prep(int J1, int R1, int nf, const float* const* G1, float* const* frag, int64_t K,
                                int nv, const VJob* v, cudaStream_t s) {
  AdapterPrep P{};
  P.nf = nf;
  P.nfrag = J1 == 4 ? K / 64 : K / 16;
  P.per_f = (P.nfrag * (R1 / 8) * 32 + 255) / 256;
  double bytes = 0.0;
  for (int i = 0; i < nf; ++i) {
    P.G1[i] = G1[i];
    P.frag[i] = reinterpret_cast<uint4*>(frag[i]);
    bytes += double(P.nfrag) * (R1 / 8) * 32 * 16 + double(K) * R1 * 4;
  }
  P.nv = nv;
  int64_t blk = nf * P.per_f;
  for (int i = 0; i < nv; ++i) {
    P.v[i] = v[i];
    P.vstart[i] = blk;
    const int K2 = v[i].R1 * v[i].J1;
    if (v[i].N * v[i].ldv >= (int64_t(1) << 31) || v[i].ldv < 3 * int64_t(K2)) return cudaErrorInvalidValue;
    blk += (v[i].N * (v[i].ldv - 2 * K2) + 255) / 256;
    bytes += double(v[i].N) * v[i].ldv * 2 + double(v[i].N) * K2 * v[i].C * 2;
  }
  P.vstart[nv] = blk;
  if (blk == 0) return cudaSuccess;
  LaunchScope scope(kTT, bytes, s);
  count_launches(1);
  const unsigned g = static_cast<unsigned>(blk);
  if (J1 == 1 && R1 == 8)
    k_adapter_prep<1, 8><<<g, 256, 0, s>>>(P);
  else if (J1 == 1)
    k_adapter_prep<1, 16><<<g, 256, 0, s>>>(P);
  else if (R1 == 8)
    k_adapter_prep<4, 8><<<g, 256, 0, s>>>(P);
  else
    k_adapter_prep<4, 16><<<g, 256, 0, s>>>(P);
  return cudaGetLastError();
}

cudaError_t launch_build_v(int d, int R1, int H, int J1, int C, int M, const float* G2, const float* G3,
                           __nv_bfloat16* V, int64_t N, int64_t ldv, cudaStream_t s) {
  const int64_t total = N * ldv;
  LaunchScope scope(kTT, double(total) * 2 + double(N) * R1 * J1 * C * 2, s);
  count_launches(1);
  const int64_t threads = N * (ldv - 2 * int64_t(R1) * J1);
  if (total >= (int64_t(1) << 31) || ldv < 3 * int64_t(R1) * J1) return cudaErrorInvalidValue;
  k_build_v<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, s>>>(d, R1, H, J1, C, M, G2, G3, V, N, ldv);
  return cudaGetLastError();
}

cudaError_t launch_build_bext(int R1, int J1, const float* G1, __nv_bfloat16* B, int64_t K, int64_t ldb,
                              cudaStream_t s) {
  const int64_t total = K * ldb;
  LaunchScope scope(kTT, double(total) * 2, s);
  count_launches(1);
  k_build_bext<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(R1, J1, G1, B, K, ldb);
  return cudaGetLastError();
}

cudaError_t launch_split_rows(const float* in, int64_t T, int K2, __nv_bfloat16* out, int64_t ld, cudaStream_t s) {
  const int64_t total = T * ld;
  if (total == 0) return cudaSuccess;
  LaunchScope scope(kTT, double(T) * K2 * 4 + double(total) * 2, s);
  count_launches(1);
  k_split_rows<<<static_cast<unsigned>((total + 255) / 256), 256, 0, s>>>(in, T, K2, out, ld);
  return cudaGetLastError();
}

int tt_dy_splits(int64_t T, int blocks_per_split) {
  const int64_t tiles = (T + DY_TT - 1) / DY_TT;
  int64_t S = (4 * 148 + blocks_per_split - 1) / blocks_per_split;  // ~4 resident CTAs per SM
  if (S > tiles) S = tiles;
  return static_cast<int>(S < 1 ? 1 : S);
}

cudaError_t launch_tt_dy(const __nv_bfloat16* dy, int64_t T, int64_t N, int H, int M, const float* Z, int64_t zs,
                         int C, const float* Gd, float* dz_part, float* dg_part, int S, cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  LaunchScope scope(kTT, 4.0 * double(T) * N * C, s);
  count_launches(1);
  const dim3 grid(static_cast<unsigned>((M / DY_COLS) * H), static_cast<unsigned>(S));
  const size_t smem = sizeof(__nv_bfloat16) * (2 * DY_TT * DY_LDY + 2 * C * (DY_TT + 8) + C * (DY_COLS + 8)) +
                      sizeof(float) * (8 / (2 * (C / 8))) * DY_TT * C;
  // the attribute is per device; setting it on every launch is cheap next to the kernel
  if (C == 8) {
    cudaFuncSetAttribute(k_tt_dy<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_tt_dy<8><<<grid, 256, smem, s>>>(dy, T, N, H, M, Z, zs, Gd, dz_part, dg_part, S);
  } else {
    cudaFuncSetAttribute(k_tt_dy<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_tt_dy<16><<<grid, 256, smem, s>>>(dy, T, N, H, M, Z, zs, Gd, dz_part, dg_part, S);
  }
  return cudaGetLastError();
}

bool tt_bwd_fused_ok(int d, int J1, int R1, int C, int M) {
  return d == 3 && J1 == 4 && M == FB_COLS && R1 == C && (C == 8 || C == 16);
}

// h-range per CTA: the dG2 accumulators (HR x K2 x C fp32) and Gm_h stay <= 64 KB of shared memory
void tt_bwd_fused_plan(int64_t T, int H, int C, int* HR, int* HS, int* TS) {
  const int hr_max = C == 8 ? 16 : 8;
  *HS = (H + hr_max - 1) / hr_max;
  *HR = (H + *HS - 1) / *HS;
  const bool ws = C == 8;  // k_tt_bwd_ws: 16-token tiles, one CTA per SM
  const int64_t tiles = (T + (ws ? WS_TT : FB_TT) - 1) / (ws ? WS_TT : FB_TT);
  // rank 16: two CTAs per SM (120 registers; measured 9.7 -> 8.7 ms of TT side kernels at config 3 vs
  // one; three or four were not better)
  const int per_sm = ws ? 1 : 2;
  int64_t ts = (static_cast<int64_t>(per_sm) * 148 + *HS - 1) / *HS;
  if (ts > tiles) ts = tiles;
  *TS = static_cast<int>(ts < 1 ? 1 : ts);
}

cudaError_t launch_tt_bwd_ws_group(const BwdJobs& jobs, int n, int64_t T, int H, cudaStream_t s) {
  if (T == 0 || n < 1) return cudaSuccess;
  if (n > kBwdJobs) return cudaErrorInvalidValue;
  int HR, HS, TS;
  tt_bwd_fused_plan(T, H, 8, &HR, &HS, &TS);
  const int64_t N = static_cast<int64_t>(H) * FB_COLS;
  // algorithmic HBM bytes: dy (bf16) + Z1 in, the dZ1 partials out (the kTT class counts bytes)
  LaunchScope scope(kTT, n * (2.0 * double(T) * N + 4.0 * double(T) * 4 * 8 * (1 + HS)), s);
  count_launches(1);
  const dim3 grid(static_cast<unsigned>(HS), static_cast<unsigned>(TS), static_cast<unsigned>(n));
  DyMaps maps;
  for (int i = 0; i < n; ++i)
    if (!make_tmap_rows3d(&maps.m[i], jobs.dy[i], T, N, jobs.ldy[i], WS_TT, 4)) return cudaErrorInvalidValue;
  const size_t smem = WsLayout::bytes(HR);
  cudaFuncSetAttribute(k_tt_bwd_ws, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  k_tt_bwd_ws<<<grid, 256, smem, s>>>(jobs, maps, T, H, HR);
  return cudaGetLastError();
}

cudaError_t launch_tt_bwd_fused(const __nv_bfloat16* dy, int64_t ldy, int64_t T, int H, int C, const float* Z1,
                                const float* G2, const float* G3, float* dz1p, float* g3part, float* g2part,
                                cudaStream_t s) {
  if (T == 0) return cudaSuccess;
  if (C == 8) {
    BwdJobs j{};
    j.dy[0] = dy;
    j.ldy[0] = ldy;
    j.Z1[0] = Z1;
    j.G2[0] = G2;
    j.G3[0] = G3;
    j.dz1p[0] = dz1p;
    j.g3part[0] = g3part;
    j.g2part[0] = g2part;
    return launch_tt_bwd_ws_group(j, 1, T, H, s);
  }
  int HR, HS, TS;
  tt_bwd_fused_plan(T, H, C, &HR, &HS, &TS);
  const int64_t N = static_cast<int64_t>(H) * FB_COLS;
  // algorithmic HBM bytes: dy (bf16) + Z1 in, the dZ1 partials out (the kTT class counts bytes)
  LaunchScope scope(kTT, 2.0 * double(T) * N + 4.0 * double(T) * 4 * C * (1 + HS), s);
  count_launches(1);
  const dim3 grid(static_cast<unsigned>(HS), static_cast<unsigned>(TS));
  {
    const size_t smem = FbLayout<16>::bytes(HR);
    cudaFuncSetAttribute(k_tt_bwd_fused<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_tt_bwd_fused<16><<<grid, 256, smem, s>>>(dy, ldy, T, H, HR, Z1, G2, G3, dz1p, g3part, g2part);
  }
  return cudaGetLastError();
}

cudaError_t launch_grad_reduce_n(int n, const float* const* parts, const int* nparts, const int64_t* numel,
                                 float* const* outs, bool accumulate, int R1, int J1, const float* const* G1,
                                 __nv_bfloat16* const* bext, int64_t K, int64_t ldb, cudaStream_t s) {
  if (n < 1 || n > kRedMembers) return cudaErrorInvalidValue;
  ReduceArgs a{};
  int64_t total = 0;
  double bytes = 0.0;
  a.nsets = 3 * n;
  for (int i = 0; i < 3 * n; ++i) {
    a.set[i] = ReduceSet{parts[i], nparts[i], numel[i], outs[i]};
    a.blocks[i] = (parts[i] != nullptr && outs[i] != nullptr) ? (numel[i] + 31) / 32 : 0;
    total += a.blocks[i];
    bytes += 4.0 * double(numel[i]) * (nparts[i] + 1);
  }
  a.accumulate = accumulate ? 1 : 0;
  a.R1 = R1;
  a.J1 = J1;
  a.K = K;
  a.ldb = ldb;
  if (ldb % 8 != 0) return cudaErrorInvalidValue;  // B_ext rows are written 8 columns (16 bytes) per thread
  a.bext_blocks = (K * ldb / 8 + 255) / 256;
  int nb = 0;  // B_ext jobs run after the sets, in member order (a member without one leaves an idle range)
  for (int j = 0; j < n; ++j) {
    a.G1s[j] = G1[j];
    a.bexts[j] = bext != nullptr ? bext[j] : nullptr;
    if (a.bexts[j] != nullptr) nb = j + 1;
  }
  if (nb > 0) {
    if (K * ldb >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
    total += nb * a.bext_blocks;
    for (int j = 0; j < nb; ++j)
      if (a.bexts[j] != nullptr) bytes += 2.0 * double(K) * ldb;
  }
  if (total == 0) return cudaSuccess;
  LaunchScope scope(kTT, bytes, s);
  count_launches(1);
  k_grad_reduce3<<<static_cast<unsigned>(total), 256, 0, s>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_grad_reduce3(const float* const* parts, const int* nparts, const int64_t* numel,
                                float* const* outs, bool accumulate, int R1, int J1, const float* G1,
                                __nv_bfloat16* bext, int64_t K, int64_t ldb, cudaStream_t s) {
  return launch_grad_reduce_n(1, parts, nparts, numel, outs, accumulate, R1, J1, &G1, &bext, K, ldb, s);
}

// ---- shared-input groups (a decoder layer's q / k / v and up / gate, transformer.py:862-874):
// one x pass serves NA in {2, 3} adapters of the pinned modes with J1 = 4, R1 = 8.
bool group_x_pass_ok(int J1, int R1, int64_t K, int NA, const void* x) {
  return J1 == 4 && R1 == 8 && NA >= 2 && NA <= 3 && K % 64 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0;
}

cudaError_t launch_actquant_z1_group(const void* x, int64_t T, int64_t K, bool want_codes, uint8_t* codes,
                                     int64_t ldc, float* sx, float* ox, int32_t* rsx, const float* const* G1, int NA,
                                     __nv_bfloat16* const* zb, int64_t ldzb, float* const* zf, float* frag_ws,
                                     cudaStream_t s, bool frag_ready) {
  if (T == 0) return cudaSuccess;
  const int64_t nfrag = K / 64;  // J1 = 4, R1 = 8: one uint4 per lane per 64-element segment
  const int64_t stride = nfrag * 32;
  uint4* fr = reinterpret_cast<uint4*>(frag_ws);
  for (int a = 0; a < NA && !frag_ready; ++a) {
    LaunchScope scope(kTT, double(stride) * 16 + double(K) * 8 * 4, s);
    count_launches(1);
    k_g1_frag<4, 8><<<static_cast<unsigned>((stride + 255) / 256), 256, 0, s>>>(G1[a], fr + a * stride, nfrag);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  AqAdapters ad{{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}, stride};
  for (int a = 0; a < NA; ++a) {
    ad.zb[a] = zb != nullptr ? zb[a] : nullptr;
    ad.zf[a] = zf != nullptr ? zf[a] : nullptr;
  }
  double out_bytes = 0.0;
  for (int a = 0; a < NA; ++a) out_bytes += double(T) * ((ad.zb[a] ? ldzb * 2 : 0) + (ad.zf[a] ? 32 * 4 : 0));
  LaunchScope scope(kQuantize, double(T) * K * 2 + (want_codes ? double(T) * ldc + 12.0 * T : 0.0) + out_bytes, s);
  count_launches(1);
  int dev = 0, nsm = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ngroups = (T + 7) / 8;
#define QA_AQN(CC, NN)                                                                                         \
  {                                                                                                            \
    auto kern = k_aq_cta<4, 8, CC, false, NN>;                                                                 \
    int per_sm = 1;                                                                                            \
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, AQC_WARPS * 32, 0);                            \
    const int64_t cap = static_cast<int64_t>(per_sm < 1 ? 1 : per_sm) * nsm;                                   \
    kern<<<static_cast<unsigned>(ngroups < cap ? ngroups : cap), AQC_WARPS * 32, 0, s>>>(                      \
        static_cast<const __nv_bfloat16*>(x), T, K, codes, ldc, sx, ox, rsx, fr, ad, ldzb);                    \
  }
  if (NA == 2) {
    if (want_codes) QA_AQN(true, 2) else QA_AQN(false, 2)
  } else {
    if (want_codes) QA_AQN(true, 3) else QA_AQN(false, 3)
  }
#undef QA_AQN
  return cudaGetLastError();
}

// x-pass occupancy: two CTAs per SM with a 2-stage x ring when ring + dZ1 planes + prefetched dZ1 partials fit
// in half an SM's shared memory (measured on the 7B set: TT side kernels 1.21 -> 1.14 ms), else one CTA per
// SM with the deepest ring that fits.
struct Dg1Shape {
  int per_sm, nstg, raw;  // raw: the dZ1 partials prefetched into shared memory (else read from L2 in place)
};
Dg1Shape dg1_shape(size_t planes, size_t raw_bytes) {
  const size_t ring2 = sizeof(__nv_bfloat16) * 2 * DM_ST * DM_LDX;
  Dg1Shape d{1, DM_NSTG, -1};
  if (ring2 + planes + raw_bytes <= 112 * 1024)
    d = Dg1Shape{2, 2, 1};
  else if (ring2 + planes <= 112 * 1024)  // shared-input groups: two CTAs per SM beat the prefetch
    d = Dg1Shape{2, 2, 0};
  return d;
}

cudaError_t launch_tt_dg1_group(const void* x, int64_t T, int64_t K, const float* const* dz1, float* const* part,
                                int S, int HS, __nv_bfloat16* const* dz1b, int64_t ldb, int NA, int* splits_used,
                                cudaStream_t s) {
  constexpr int R1 = 8, J1 = 4;
  if (splits_used != nullptr) *splits_used = S;
  if (T == 0) return cudaSuccess;
  double bytes = double(T) * K * 2;
  for (int a = 0; a < NA; ++a) bytes += 4.0 * double(T) * J1 * R1 * HS + (dz1b && dz1b[a] ? 2.0 * double(T) * ldb : 0.0);
  LaunchScope scope(kTT, bytes, s);
  count_launches(1);
  const int64_t gx = (K + DM_COLS - 1) / DM_COLS;
  const int64_t stages = (T + DM_ST - 1) / DM_ST;
  const size_t raw_bytes = sizeof(float) * 2 * NA * HS * DM_DZT * J1 * R1;
  const size_t planes = sizeof(__nv_bfloat16) * NA * 2 * DM_DZT * R1 * J1;
  const Dg1Shape shp = dg1_shape(planes, raw_bytes);
  int64_t Sm = (148 * shp.per_sm + gx - 1) / gx;
  if (Sm > stages) Sm = stages;
  if (Sm > S) Sm = S;
  if (Sm < 1) Sm = 1;
  if (splits_used != nullptr) *splits_used = static_cast<int>(Sm);
  DgAdapters ad{{nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}, {nullptr, nullptr, nullptr}};
  for (int a = 0; a < NA; ++a) {
    ad.dz1[a] = dz1[a];
    ad.part[a] = part[a];
    ad.dz1b[a] = dz1b != nullptr ? dz1b[a] : nullptr;
  }
  // one CTA per SM: a 4-stage x ring when the prefetched dZ1 partials fit beside it, else 3 stages (the
  // prefetch matters more)
  int nstg = shp.nstg;
  if (shp.raw < 0 && sizeof(__nv_bfloat16) * nstg * DM_ST * DM_LDX + planes + raw_bytes > 220 * 1024) nstg = 3;
  size_t smem = sizeof(__nv_bfloat16) * nstg * DM_ST * DM_LDX + planes;
  const int raw_async = shp.raw >= 0 ? shp.raw : (smem + raw_bytes <= 220 * 1024 ? 1 : 0);
  if (raw_async) smem += raw_bytes;
  const dim3 gm(static_cast<unsigned>(gx), static_cast<unsigned>(Sm));
  CUtensorMap tmx;
  const int x3d = K % 64 == 0 ? 1 : 0;
  if (!(x3d ? make_tmap_rows3d(&tmx, x, T, K, K, DM_ST, DM_COLS / 64) : make_tmap_bf16_rows(&tmx, x, T, K, K, DM_ST)))
    return cudaErrorInvalidValue;
  if (NA == 2) {
    cudaFuncSetAttribute(k_tt_dg1m<8, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_tt_dg1m<8, 2><<<gm, 256, smem, s>>>(tmx, static_cast<const __nv_bfloat16*>(x), T, K, ad, static_cast<int>(Sm), HS,
                                          ldb, raw_async, nstg, x3d);
  } else {
    cudaFuncSetAttribute(k_tt_dg1m<8, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_tt_dg1m<8, 3><<<gm, 256, smem, s>>>(tmx, static_cast<const __nv_bfloat16*>(x), T, K, ad, static_cast<int>(Sm), HS,
                                          ldb, raw_async, nstg, x3d);
  }
  return cudaGetLastError();
}

int tt_dg1_splits(int64_t T, int64_t K, int J1) {
  const int E = J1 == 1 ? 4 : 8;
  const int64_t gx = (K + 256 * E - 1) / (256 * E);
  int64_t S = (2 * 148 + gx - 1) / gx;
  if (S > T) S = T;
  return static_cast<int>(S < 1 ? 1 : S);
}

cudaError_t launch_tt_dg1(const void* x, int x_dtype, int64_t T, int64_t K, const float* dz1, int J1, int R1,
                          float* part, int S, cudaStream_t s, int HS, __nv_bfloat16* dz1b, int64_t ldb,
                          int* splits_used) {
  if (splits_used != nullptr) *splits_used = S;
  if (T == 0) return cudaSuccess;
  // algorithmic HBM bytes: x in, the dZ1 partials in, the split dZ1 rows out
  LaunchScope scope(kTT, double(T) * K * (x_dtype == QA_F32 ? 4 : 2) + 4.0 * double(T) * J1 * R1 * HS +
                             (dz1b ? 2.0 * double(T) * ldb : 0.0), s);
  count_launches(1);
  const int E = J1 == 1 ? 4 : 8;
  const dim3 grid(static_cast<unsigned>((K + 256 * E - 1) / (256 * E)), static_cast<unsigned>(S));
  if (x_dtype == QA_BF16 && J1 == 4 && K % 8 == 0 && reinterpret_cast<uintptr_t>(x) % 16 == 0) {
    const int64_t gx = (K + DM_COLS - 1) / DM_COLS;
    const int64_t stages = (T + DM_ST - 1) / DM_ST;
    const size_t raw_bytes = sizeof(float) * 2 * HS * DM_DZT * J1 * R1;
    const size_t planes = sizeof(__nv_bfloat16) * 2 * DM_DZT * R1 * J1;
    const Dg1Shape shp = dg1_shape(planes, raw_bytes);
    int64_t Sm = (148 * shp.per_sm + gx - 1) / gx;
    if (Sm > stages) Sm = stages;
    if (Sm > S) Sm = S;
    if (Sm < 1) Sm = 1;
    if (Sm <= S) {  // the caller's partial buffer holds S splits
      if (splits_used != nullptr) *splits_used = static_cast<int>(Sm);
      const dim3 gm(static_cast<unsigned>(gx), static_cast<unsigned>(Sm));
      int nstg = shp.nstg;
      if (shp.raw < 0 && sizeof(__nv_bfloat16) * nstg * DM_ST * DM_LDX + planes + raw_bytes > 220 * 1024) nstg = 3;
      size_t smem = sizeof(__nv_bfloat16) * nstg * DM_ST * DM_LDX + planes;
      const int raw_async = shp.raw >= 0 ? shp.raw : (smem + raw_bytes <= 220 * 1024 ? 1 : 0);
      if (raw_async) smem += raw_bytes;
      const DgAdapters ad{{dz1, nullptr, nullptr}, {part, nullptr, nullptr}, {dz1b, nullptr, nullptr}};
      CUtensorMap tmx;
      const int x3d = K % 64 == 0 ? 1 : 0;
      if (!(x3d ? make_tmap_rows3d(&tmx, x, T, K, K, DM_ST, DM_COLS / 64)
                : make_tmap_bf16_rows(&tmx, x, T, K, K, DM_ST)))
        return cudaErrorInvalidValue;
      if (R1 == 8) {
        cudaFuncSetAttribute(k_tt_dg1m<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k_tt_dg1m<8><<<gm, 256, smem, s>>>(tmx, static_cast<const __nv_bfloat16*>(x), T, K, ad, static_cast<int>(Sm), HS,
                                           ldb, raw_async, nstg, x3d);
      } else {
        cudaFuncSetAttribute(k_tt_dg1m<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        k_tt_dg1m<16><<<gm, 256, smem, s>>>(tmx, static_cast<const __nv_bfloat16*>(x), T, K, ad, static_cast<int>(Sm), HS,
                                            ldb, raw_async, nstg, x3d);
      }
      return cudaGetLastError();
    }
  }
#define QA_DG(TI, JJ, RR) \
  k_tt_dg1<TI, JJ, RR><<<grid, 256, 0, s>>>(static_cast<const TI*>(x), T, K, dz1, part, S, HS, dz1b, ldb)
#define QA_DG_T(TI)                 \
  if (J1 == 1 && R1 == 8)           \
    QA_DG(TI, 1, 8);                \
  else if (J1 == 1 && R1 == 16)     \
    QA_DG(TI, 1, 16);               \
  else if (J1 == 4 && R1 == 8)      \
    QA_DG(TI, 4, 8);                \
  else                              \
    QA_DG(TI, 4, 16);
  if (x_dtype == QA_F32) {
    QA_DG_T(float)
  } else {
    QA_DG_T(__nv_bfloat16)
  }
#undef QA_DG_T
#undef QA_DG
  return cudaGetLastError();
}

}  // namespace qa

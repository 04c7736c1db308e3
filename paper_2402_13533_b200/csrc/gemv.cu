// Decode-size forward (1..8 tokens, KV-cached decoding, transformer.py:1043-1080): the int8 product is a
// matrix-vector pass over the stored codes, so it is HBM-bound on the weight bytes, not tensor-bound.
//   k_gemv_mma (K % 64 == 0, the production pass): mma.sync m16n8k32 u8 x u8 -> exact s32 with 16 weight
//     rows x 8 token columns per warp instruction, 8 warps splitting K, launched as a programmatic dependent
//     of the act-quant prologue (weights loaded / prefetched before griddepcontrol.wait).
//   k_gemv (other K): one warp per output row at a time, lanes stream 16-byte code chunks and multiply them
//     against the activation codes with dp4a.
// Both apply the tcgen05 GEMM's exact-int32 centring + fp32 dequant epilogue (gemm_tc.cu) plus the adapter
// term y2 = Σ_b Zlast[t, h, b] · Glast[b, i] from the prologue's fp32 Zlast and the last core.
#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_timing.h"

namespace qa {

namespace {

// Loads of what the prologue wrote (activation codes, scales, Zlast). The matrix-vector kernels start
// before the prologue finishes (programmatic dependent launch) and wait on griddepcontrol.wait; these
// loads must stay after that wait, so they are volatile asm (an __ldg / ld.global.nc may legally be
// hoisted above it, the data being declared read-only for the kernel's lifetime).
__device__ __forceinline__ uint4 ld_dep_v4(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
  return v;
}
__device__ __forceinline__ float ld_dep_f32(const float* p) {
  float v;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ int32_t ld_dep_s32(const int32_t* p) {
  int32_t v;
  asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

constexpr int GV_WARPS = 8;  // warps per CTA

// Rows per warp and 16-byte chunks in flight per row: more rows per warp for more tokens, so each
// activation chunk loaded from L1 feeds GV_RPW rows of dp4a (the T = 8 pass is L1-load bound otherwise).
template <int M>
struct GvShape {
  static constexpr int RPW = M <= 1 ? 2 : 4;
  static constexpr int UNR = M <= 1 ? 4 : 2;
};

template <int M, int BITS>
__global__ void __launch_bounds__(GV_WARPS * 32, 1) k_gemv(const uint8_t* __restrict__ xc, int64_t ldx, int T,
                                                        const float* __restrict__ sx, const float* __restrict__ ox,
                                                        const int32_t* __restrict__ rsx,
                                                        const uint8_t* __restrict__ wc, int64_t N, int64_t K,
                                                        const float* __restrict__ ws, const float* __restrict__ wo,
                                                        const int32_t* __restrict__ wrs,
                                                        const float* __restrict__ zl, int64_t ldz,
                                                        const float* __restrict__ Gl, int64_t Ml, int Cl,
                                                        const float* __restrict__ addend,
                                                        __nv_bfloat16* __restrict__ out, float* __restrict__ out32) {
  constexpr int GV_RPW = GvShape<M>::RPW, GV_UNR = GvShape<M>::UNR;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ldw = BITS == 8 ? K : K / 2;
  const int64_t nchunk = ldw / 16;  // 16-byte code chunks per row (16 codes at 8 bits, 32 at 4)
  const int64_t row0 = (static_cast<int64_t>(blockIdx.x) * GV_WARPS + warp) * GV_RPW;
  // Launched as a programmatic dependent of the act-quant prologue: pull this warp's weight rows into
  // L2 (they do not depend on it), then wait for the prologue's codes / scales / Zlast.
#pragma unroll
  for (int r = 0; r < GV_RPW; ++r)
    if (row0 + r < N)
      for (int64_t b = static_cast<int64_t>(lane) * 128; b < ldw; b += 32 * 128)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(wc + (row0 + r) * ldw + b));
  asm volatile("griddepcontrol.wait;" ::: "memory");
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
        const uint4 x = ld_dep_v4(reinterpret_cast<const uint4*>(xc + t * ldx) + q);
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
        const uint4 x0 = ld_dep_v4(reinterpret_cast<const uint4*>(xc + t * ldx) + 2 * q);
        const uint4 x1 = ld_dep_v4(reinterpret_cast<const uint4*>(xc + t * ldx) + 2 * q + 1);
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
        if (t < T) y2[r][t] = ld_dep_f32(zl + t * ldz + h * Cl + lane) * g;
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
      const float s = ld_dep_f32(sx + t);
      const float oxt = ld_dep_f32(ox + t) + static_cast<float>(zp_row) * s;
      const int32_t rx = ld_dep_s32(rsx + t);
      const float rsxc = static_cast<float>(rx - zp_row * kr);
      const int32_t ibase = zp_row * zp_col * kr - zp_col * rx;
      const int32_t accc = static_cast<int32_t>(acc[r][t]) + ibase - colD;
      float y = fmaf(s, fmaf(sw, static_cast<float>(accc), owt * rsxc), oxt * colC);
      y += y2[r][t];
      if (addend != nullptr) y += ld_dep_f32(addend + t * N + n);
      if (out32 != nullptr) out32[t * N + n] = y;
      if (out != nullptr) out[t * N + n] = __float2bfloat16_rn(y);
    }
  }
}

// Tensor-core variant (K % 64 == 0): the [tokens x K] x [K x N] u8 product as mma.sync m16n8k32
// (u8 x u8 -> exact s32): 16 weight rows form the M side, up to 8 tokens the N side, so one warp
// instruction does 16 x 8 x 32 MACs and the pass is left bound on the weight bytes. Because the k
// reduction is order-free, each thread feeds the mma the contiguous bytes it loaded (8-bit: 16 B of
// a row = two k32 steps; 4-bit: 8 packed bytes unpacked to even / odd columns) with the activation
// bytes of the same columns. A CTA owns 16 rows; its 8 warps split K and meet in shared memory.
// warps (K split) per CTA and 64-column steps held in registers: 8 steps = a 4096-wide row slice per warp in one
// round trip, at two CTAs per SM (measured: 93.5 -> 76.2 us for the 7-linear decode step against 4 steps)
constexpr int GM_WARPS = 8, GM_MAXS = 8;

__device__ __forceinline__ void mma_u8_16832(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                             uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k32.row.col.s32.u8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

template <int BITS>
struct GmW {
  using T = uint4;  // 16 bytes of a row per 64-column step at 8 bits
};
template <>
struct GmW<4> {
  using T = uint2;  // 8 packed bytes at 4 bits
};

template <int BITS>
__device__ __forceinline__ void gm_step(int (&acc)[4], const typename GmW<BITS>::T& A, const typename GmW<BITS>::T& B,
                                        const uint4& xv) {
  if constexpr (BITS == 8) {
    mma_u8_16832(acc, A.x, B.x, A.y, B.y, xv.x, xv.y);
    mma_u8_16832(acc, A.z, B.z, A.w, B.w, xv.z, xv.w);
  } else {
    // packed byte j = columns 2j (low nibble), 2j + 1 (high nibble)
    const uint32_t m = 0x0F0F0F0Fu;
    mma_u8_16832(acc, A.x & m, B.x & m, (A.x >> 4) & m, (B.x >> 4) & m, __byte_perm(xv.x, xv.y, 0x6420),
                 __byte_perm(xv.x, xv.y, 0x7531));
    mma_u8_16832(acc, A.y & m, B.y & m, (A.y >> 4) & m, (B.y >> 4) & m, __byte_perm(xv.z, xv.w, 0x6420),
                 __byte_perm(xv.z, xv.w, 0x7531));
  }
}

// The members of a shared-input group (q / k / v, up / gate) in one launch: CTA b belongs to the member whose
// [cta0, next cta0) range holds it, and reads that member's weights, epilogue terms and adapter input.
template <int BITS>
__global__ void __launch_bounds__(GM_WARPS * 32, 2) k_gemv_mma(const uint8_t* __restrict__ xc, int64_t ldx, int T,
                                                            const float* __restrict__ sx, const float* __restrict__ ox,
                                                            const int32_t* __restrict__ rsx, int64_t K,
                                                            const GemvMembers mem) {
  using W = typename GmW<BITS>::T;
  constexpr int SB = BITS == 8 ? 64 : 32;  // weight bytes per row per 64-column step
  __shared__ int red[GM_WARPS][16][8];
  // let a chained next prologue (a programmatic dependent, see launch_decode_prep) start right away
  asm volatile("griddepcontrol.launch_dependents;");
  int mi = 0;
  while (mi + 1 < mem.n && static_cast<int>(blockIdx.x) >= mem.m[mi + 1].cta0) ++mi;
  const GemvMember& M = mem.m[mi];
  const uint8_t* __restrict__ wc = M.wc;
  const int64_t N = M.N;
  const float* __restrict__ ws = M.ws;
  const float* __restrict__ wo = M.wo;
  const int32_t* __restrict__ wrs = M.wrs;
  const float* __restrict__ zl = M.zl;
  const int64_t ldz = M.ldz;
  const float* __restrict__ Gl = M.Gl;
  const int64_t Ml = M.Ml;
  const int Cl = M.Cl;
  const float* __restrict__ addend = M.addend;
  __nv_bfloat16* __restrict__ out = M.out;
  float* __restrict__ out32 = M.out32;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, tq = lane & 3;
  const int64_t n0 = static_cast<int64_t>(blockIdx.x - M.cta0) * 16;
  const int64_t ldw = BITS == 8 ? K : K / 2;
  const int64_t nsteps = K / 64;
  const int64_t per = (nsteps + GM_WARPS - 1) / GM_WARPS;
  const int64_t s0 = warp * per < nsteps ? warp * per : nsteps, s1 = s0 + per < nsteps ? s0 + per : nsteps;
  const int64_t ra = n0 + g < N ? n0 + g : N - 1, rb = n0 + g + 8 < N ? n0 + g + 8 : N - 1;
  const uint8_t* pa = wc + ra * ldw + tq * (SB / 4);
  const uint8_t* pb = wc + rb * ldw + tq * (SB / 4);
  // Launched as a programmatic dependent of the act-quant prologue: the weight codes do not depend on it,
  // so the first GM_MAXS steps go straight into registers (the rest of the slice into L2) before waiting.
  W A[GM_MAXS], B[GM_MAXS];
  int ns = static_cast<int>(s1 - s0 < GM_MAXS ? s1 - s0 : GM_MAXS);
#pragma unroll
  for (int i = 0; i < GM_MAXS; ++i)
    if (i < ns) {
      A[i] = __ldg(reinterpret_cast<const W*>(pa + (s0 + i) * SB));
      B[i] = __ldg(reinterpret_cast<const W*>(pb + (s0 + i) * SB));
    }
  {
    const int64_t r = n0 + (lane & 15);
    if (r < N)
      for (int64_t b = (s0 + GM_MAXS) * SB + (lane >> 4) * 128; b < s1 * SB; b += 256)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(wc + r * ldw + b));
  }
  // weight-side epilogue operands: this thread's (row, token) after the cross-warp reduction is
  // (n0 + threadIdx.x / 8, threadIdx.x % 8) for threadIdx.x < 128
  const int rr = threadIdx.x >> 3, t = threadIdx.x & 7;
  const int64_t n = n0 + rr;
  const bool live = threadIdx.x < 128 && n < N && t < T;
  float sw = 0.f, wof = 0.f;
  int32_t rs = 0;
  if (live) {
    sw = ws[n];
    wof = wo[n];
    rs = wrs[n];
  }
  // adapter operands in shared memory: the last core's columns of this CTA's 16 rows (weights, read
  // before the wait) and Zlast[t, h, :] of the row block (one h: 16 | Ml), read right after it
  __shared__ float sG[16][32], sZ[8][32];
  const int64_t h0 = Gl != nullptr ? n0 / Ml : 0;
  if (Gl != nullptr)
    for (int idx = threadIdx.x; idx < 16 * Cl; idx += GM_WARPS * 32) {
      const int r = idx / Cl, b = idx - (idx / Cl) * Cl;
      const int64_t nr = n0 + r < N ? n0 + r : N - 1;
      sG[r][b] = __ldg(Gl + b * Ml + (nr - h0 * Ml));
    }
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (Gl != nullptr && static_cast<int>(threadIdx.x) < T * Cl) {
    const int tt = threadIdx.x / Cl, b = threadIdx.x - (threadIdx.x / Cl) * Cl;
    sZ[tt][b] = ld_dep_f32(zl + tt * ldz + h0 * Cl + b);
  }
  float sxt = 0.f, oxr = 0.f;
  int32_t rx = 0;
  if (live) {
    sxt = ld_dep_f32(sx + t);
    oxr = ld_dep_f32(ox + t);
    rx = ld_dep_s32(rsx + t);
  }
  const bool tok = g < T;
  const uint8_t* px = xc + (tok ? g : 0) * ldx + tq * 16;
  int acc[4] = {0, 0, 0, 0};
  for (int64_t st = s0; ns > 0;) {
    uint4 X[GM_MAXS];
#pragma unroll
    for (int i = 0; i < GM_MAXS; ++i)
      if (i < ns) X[i] = tok ? ld_dep_v4(px + (st + i) * 64) : make_uint4(0, 0, 0, 0);
#pragma unroll
    for (int i = 0; i < GM_MAXS; ++i)
      if (i < ns) gm_step<BITS>(acc, A[i], B[i], X[i]);
    st += ns;
    ns = static_cast<int>(s1 - st < GM_MAXS ? s1 - st : GM_MAXS);
#pragma unroll
    for (int i = 0; i < GM_MAXS; ++i)
      if (i < ns) {
        A[i] = __ldg(reinterpret_cast<const W*>(pa + (st + i) * SB));
        B[i] = __ldg(reinterpret_cast<const W*>(pb + (st + i) * SB));
      }
  }
  red[warp][g][2 * tq] = acc[0];
  red[warp][g][2 * tq + 1] = acc[1];
  red[warp][g + 8][2 * tq] = acc[2];
  red[warp][g + 8][2 * tq + 1] = acc[3];
  __syncthreads();
  if (!live) return;
  uint32_t a = 0;
#pragma unroll
  for (int w = 0; w < GM_WARPS; ++w) a += static_cast<uint32_t>(red[w][rr][t]);
  // adapter: y2[t, n] = Σ_b Zlast[t, h, b] Glast[b, i], n = h Ml + i
  float y2 = 0.f;
  if (Gl != nullptr)
    for (int b = 0; b < Cl; ++b) y2 = fmaf(sZ[t][b], sG[rr][b], y2);
  // the tcgen05 GEMM's exact int32 centring + fp32 dequant epilogue (gemm_tc.cu)
  const int zp_row = 128, zp_col = BITS == 8 ? 128 : 8;
  const int kr = static_cast<int>(K);
  const float owt = wof + static_cast<float>(zp_col) * sw;
  const float colC = fmaf(sw, static_cast<float>(rs - zp_col * kr), static_cast<float>(kr) * owt);
  const int32_t colD = zp_row * rs;
  const float oxt = oxr + static_cast<float>(zp_row) * sxt;
  const float rsxc = static_cast<float>(rx - zp_row * kr);
  const int32_t ibase = zp_row * zp_col * kr - zp_col * rx;
  const int32_t accc = static_cast<int32_t>(a) + ibase - colD;
  float y = fmaf(sxt, fmaf(sw, static_cast<float>(accc), owt * rsxc), oxt * colC);
  y += y2;
  if (addend != nullptr) y += ld_dep_f32(addend + t * N + n);
  if (out32 != nullptr) out32[t * N + n] = y;
  if (out != nullptr) out[t * N + n] = __float2bfloat16_rn(y);
}

}  // namespace

// The decode kernels chain by programmatic dependent launch (the pass's weight loads start while the
// prologue still runs).
bool pdl_enabled() { return true; }

bool gemv_mma_ok(int64_t K, int64_t N, const float* Gl, int64_t Ml, int Cl) {
  return K % 64 == 0 && (Gl == nullptr || ((Ml % 16 == 0 || Ml >= N) && Cl <= 32));
}

cudaError_t launch_gemv_members(const uint8_t* xc, int64_t ldx, int64_t T, const float* sx, const float* ox,
                                const int32_t* rsx, int64_t K, int bits, GemvMembers mem, cudaStream_t s) {
  if (T == 0 || mem.n < 1) return cudaSuccess;
  int ctas = 0;
  double flops = 0.0;
  for (int i = 0; i < mem.n; ++i) {
    if (!gemv_mma_ok(K, mem.m[i].N, mem.m[i].Gl, mem.m[i].Ml, mem.m[i].Cl)) return cudaErrorInvalidValue;
    mem.m[i].cta0 = ctas;
    ctas += static_cast<int>((mem.m[i].N + 15) / 16);
    flops += 2.0 * double(T) * mem.m[i].N * K;
  }
  LaunchScope scope(kGemmI8, flops, s);
  count_launches(1);
  // programmatic dependent launch: the CTAs may start while the preceding prologue still runs
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(static_cast<unsigned>(ctas));
  cfg.blockDim = dim3(GM_WARPS * 32);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const int Ti = static_cast<int>(T);
  cudaError_t e = bits == 8 ? cudaLaunchKernelEx(&cfg, k_gemv_mma<8>, xc, ldx, Ti, sx, ox, rsx, K, mem)
                            : cudaLaunchKernelEx(&cfg, k_gemv_mma<4>, xc, ldx, Ti, sx, ox, rsx, K, mem);
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

bool gemv_ok(int64_t T, int64_t K, int bits) {
  return T >= 1 && T <= 8 && (bits == 8 ? K % 16 == 0 : K % 32 == 0);
}

cudaError_t launch_gemv(const uint8_t* xc, int64_t ldx, int64_t T, const float* sx, const float* ox,
                        const int32_t* rsx, const uint8_t* wc, int64_t N, int64_t K, int bits, const float* ws,
                        const float* wo, const int32_t* wrs, const float* zl, int64_t ldz, const float* Gl,
                        int64_t Ml, int Cl, const float* addend, __nv_bfloat16* out, float* out32, cudaStream_t s) {
  if (T == 0 || N == 0) return cudaSuccess;
  // the tensor-core pass keeps one Zlast block per 16-row tile (16 | Ml, or a single block) and Cl <= 32
  if (gemv_mma_ok(K, N, Gl, Ml, Cl)) {
    GemvMembers mem{};
    mem.n = 1;
    mem.m[0] = GemvMember{wc, N, ws, wo, wrs, zl, ldz, Gl, Ml, Cl, addend, out, out32, 0};
    return launch_gemv_members(xc, ldx, T, sx, ox, rsx, K, bits, mem, s);
  }
  LaunchScope scope(kGemmI8, 2.0 * double(T) * N * K, s);
  count_launches(1);
  // programmatic dependent launch: the CTAs may start while the preceding prologue still runs
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(GV_WARPS * 32);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const int Ti = static_cast<int>(T);
  cudaError_t e = cudaSuccess;
#define QA_GV(MM)                                                                                                 \
  {                                                                                                               \
    constexpr int rows = GV_WARPS * GvShape<MM>::RPW;                                                             \
    cfg.gridDim = dim3(static_cast<unsigned>((N + rows - 1) / rows));                                            \
    if (bits == 8)                                                                                                \
      e = cudaLaunchKernelEx(&cfg, k_gemv<MM, 8>, xc, ldx, Ti, sx, ox, rsx, wc, N, K, ws, wo, wrs, zl, ldz, Gl, Ml, \
                             Cl, addend, out, out32);                                                             \
    else                                                                                                          \
      e = cudaLaunchKernelEx(&cfg, k_gemv<MM, 4>, xc, ldx, Ti, sx, ox, rsx, wc, N, K, ws, wo, wrs, zl, ldz, Gl, Ml, \
                             Cl, addend, out, out32);                                                             \
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
  if (e != cudaSuccess) return e;
  return cudaGetLastError();
}

}  // namespace qa

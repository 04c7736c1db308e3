// Bit-exact per-element code derivation shared by the quantisation kernels (see quant_kernels.cu).
#pragma once

#include <math.h>

#include "qa_common.cuh"

namespace qa {
namespace {

constexpr float kTieBand = 2.5e-4f;

template <int BITS>
QA_DEV uint32_t code_of(float v, float lo, float inv, double lo64, double step64) {
  constexpr float kTop = float((1 << BITS) - 1);
  const float q = (v - lo) * inv;
  const float fl = floorf(q);
  const float fr = q - fl;
  float c;
  if (fabsf(fr - 0.5f) < kTieBand) {
    const double v64 = __ddiv_rn(__dsub_rn(static_cast<double>(v), lo64), step64);
    c = static_cast<float>(floor(__dadd_rn(v64, 0.5)));
  } else {
    c = fr > 0.5f ? fl + 1.0f : fl;
  }
  return static_cast<uint32_t>(fminf(fmaxf(c, 0.0f), kTop));
}

template <typename T>
QA_DEV void load8(const T* p, float (&f)[8]);
template <>
QA_DEV void load8<float>(const float* p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p));
  const float4 b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  f[0] = a.x, f[1] = a.y, f[2] = a.z, f[3] = a.w, f[4] = b.x, f[5] = b.y, f[6] = b.z, f[7] = b.w;
}
template <>
QA_DEV void load8<__nv_bfloat16>(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    f[2 * i] = __uint_as_float(w[i] << 16);
    f[2 * i + 1] = __uint_as_float(w[i] & 0xFFFF0000u);
  }
}

// ---- packed fp32 (sm_100 FFMA2) helpers
QA_DEV unsigned long long f2pack(float a, float b) {
  return static_cast<unsigned long long>(__float_as_uint(a)) |
         (static_cast<unsigned long long>(__float_as_uint(b)) << 32);
}
QA_DEV float f2lo(unsigned long long v) { return __uint_as_float(static_cast<uint32_t>(v)); }
QA_DEV float f2hi(unsigned long long v) { return __uint_as_float(static_cast<uint32_t>(v >> 32)); }
QA_DEV void ffma2(unsigned long long& d, unsigned long long a, unsigned long long b) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(d) : "l"(a), "l"(b));
}
QA_DEV unsigned long long ffma2r(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// 8-bit codes of 8 consecutive elements (same rule as code_of<8>) packed little-endian into
// two words; adds the codes to `sum`.  q = v*inv + (-lo*inv) is evaluated with packed FMAs (its
// error, < 2e-5, is far inside the tie band); elements within the band of a rounding boundary are
// replayed exactly in fp64.
QA_DEV unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
QA_DEV unsigned long long fadd2rm(unsigned long long a, unsigned long long b) {  // round toward -inf
  unsigned long long d;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
QA_DEV unsigned long long fsub2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}

// Rounding uses the magic constant 1.5 * 2^23: for 0 <= q < 2^22, q + M rounds q to the nearest
// integer (ties to even) in the low mantissa bits, so the code is the low byte of the sum and
// rint(q) = (q + M) - M — plain FP32 adds instead of the quarter-rate F2I / FRND pipe.  Exact
// ties and everything within the band of one are replayed in fp64 below.  q = (v - lo) * inv is
// formed by subtraction first (as code_of does): v * inv - lo * inv would lose the tie band when
// |lo| >> hi - lo.
QA_DEV void codes8(const float (&f)[8], float lo, float inv, double lo64, double step64, uint32_t& w0, uint32_t& w1,
                   int& sum) {
  constexpr float kMagic = 12582912.0f;
  const unsigned long long inv2 = f2pack(inv, inv), nlo2 = f2pack(-lo, -lo);
  const unsigned long long m2 = f2pack(kMagic, kMagic), nm2 = f2pack(-kMagic, -kMagic);
  uint32_t r[8];
  bool near = false;
#pragma unroll
  for (int i = 0; i < 8; i += 2) {
    const unsigned long long q2 = ffma2r(fadd2(f2pack(f[i], f[i + 1]), nlo2), inv2, 0ull);
    const unsigned long long s2 = fadd2(q2, m2);            // q + M: rounded integer in the low bits
    const unsigned long long d2 = fadd2(q2, fadd2(s2, nm2) ^ 0x8000000080000000ull);  // q - rint(q)
    near |= fabsf(f2lo(d2)) > 0.5f - kTieBand;
    near |= fabsf(f2hi(d2)) > 0.5f - kTieBand;
    r[i] = static_cast<uint32_t>(s2);
    r[i + 1] = static_cast<uint32_t>(s2 >> 32);
  }
  // low bytes of the magic sums; q in (-1e-4, 255 + 1e-4) so the byte is the clipped code
  w0 = __byte_perm(__byte_perm(r[0], r[1], 0x0040), __byte_perm(r[2], r[3], 0x0040), 0x5410);
  w1 = __byte_perm(__byte_perm(r[4], r[5], 0x0040), __byte_perm(r[6], r[7], 0x0040), 0x5410);
  if (near) {
    uint32_t c[8];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      c[i] = (w0 >> (8 * i)) & 0xFFu;
      c[i + 4] = (w1 >> (8 * i)) & 0xFFu;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float q = (f[i] - lo) * inv;
      if (fabsf(q - ((q + kMagic) - kMagic)) > 0.5f - 2.0f * kTieBand) {
        const double v64 = __ddiv_rn(__dsub_rn(static_cast<double>(f[i]), lo64), step64);
        c[i] = static_cast<uint32_t>(fmin(fmax(floor(__dadd_rn(v64, 0.5)), 0.0), 255.0));
      }
    }
    w0 = c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24);
    w1 = c[4] | (c[5] << 8) | (c[6] << 16) | (c[7] << 24);
  }
  sum = static_cast<int>(__dp4a(w0, 0x01010101u, static_cast<unsigned int>(sum)));
  sum = static_cast<int>(__dp4a(w1, 0x01010101u, static_cast<unsigned int>(sum)));
}

}  // namespace
}  // namespace qa

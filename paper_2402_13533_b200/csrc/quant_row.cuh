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

}  // namespace
}  // namespace qa

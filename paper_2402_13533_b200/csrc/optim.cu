// AdamW over the flat adapter-parameter buffer (trainer.py:84-121, adamw_step), in the reference's own
// float64 arithmetic: the same sequence of IEEE operations (explicit _rn intrinsics, no contraction),
// so masters, moments and the float32 working copies are bit-identical to the reference's numpy update.
#include <cmath>

#include "qa_common.cuh"
#include "qa_internal.h"
#include "qa_timing.h"

namespace qa {

namespace {

__global__ void __launch_bounds__(256) k_adamw(float* __restrict__ params, double* __restrict__ master,
                                               double* __restrict__ m, double* __restrict__ v,
                                               const float* __restrict__ g, int64_t n, double lr, double b1,
                                               double b2, double omb1, double omb2, double bias1, double bias2,
                                               double eps, double wd) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double gi = static_cast<double>(g[i]);
    // m *= b1; m += (1 - b1) * g
    double mi = __dadd_rn(__dmul_rn(m[i], b1), __dmul_rn(omb1, gi));
    // v *= b2; v += (1 - b2) * g^2
    double vi = __dadd_rn(__dmul_rn(v[i], b2), __dmul_rn(omb2, __dmul_rn(gi, gi)));
    m[i] = mi;
    v[i] = vi;
    const double mh = __ddiv_rn(mi, bias1), vh = __ddiv_rn(vi, bias2);
    // w -= lr * (m_hat / (sqrt(v_hat) + eps) + wd * w)
    const double w = master[i];
    const double upd = __dadd_rn(__ddiv_rn(mh, __dadd_rn(__dsqrt_rn(vh), eps)), __dmul_rn(wd, w));
    const double wn = __dsub_rn(w, __dmul_rn(lr, upd));
    master[i] = wn;
    params[i] = __double2float_rn(wn);
  }
}

__global__ void __launch_bounds__(256) k_seg_nonfinite(const float* __restrict__ g, const int64_t* __restrict__ seg,
                                                       int nseg, int32_t* __restrict__ flags) {
  const int s = blockIdx.y;
  if (s >= nseg) return;
  const int64_t a = seg[s], b = seg[s + 1];
  bool bad = false;
  for (int64_t i = a + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < b;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    bad |= !isfinite(g[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags + s, 1);
}

}  // namespace

cudaError_t launch_adamw(float* params, double* master, double* m, double* v, const float* g, int64_t n, double lr,
                         double b1, double b2, double eps, double wd, int64_t step, cudaStream_t s) {
  if (n == 0) return cudaSuccess;
  LaunchScope scope(kDequant, double(n) * (4 + 8 * 3 * 2 + 4 + 4), s);
  count_launches(1);
  // the reference's scalars, computed on the host in float64 exactly as numpy does
  const double bias1 = 1.0 - std::pow(b1, static_cast<double>(step));
  const double bias2 = 1.0 - std::pow(b2, static_cast<double>(step));
  const int64_t blocks = (n + 255) / 256;
  k_adamw<<<static_cast<unsigned>(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, s>>>(
      params, master, m, v, g, n, lr, b1, b2, 1.0 - b1, 1.0 - b2, bias1, bias2, eps, wd);
  return cudaGetLastError();
}

cudaError_t launch_seg_nonfinite(const float* g, const int64_t* seg, int nseg, int32_t* flags, cudaStream_t s) {
  if (nseg == 0) return cudaSuccess;
  count_launches(1);
  const dim3 grid(16, static_cast<unsigned>(nseg));
  k_seg_nonfinite<<<grid, 256, 0, s>>>(g, seg, nseg, flags);
  return cudaGetLastError();
}

}  // namespace qa

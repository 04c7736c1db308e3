// Launch accounting helpers (see timing.cu).
#pragma once

#include <cuda_runtime.h>

namespace qa {

enum KernelClass { kGemmI8 = 0, kGemmBF16, kQuantize, kTT, kDequant, kMerge, kNumClasses };

// Adds n to the library-wide launch counter (qa_launch_count).
void count_launches(int n);

// Records CUDA events around the launches issued in its lifetime when timing is enabled.
class LaunchScope {
 public:
  LaunchScope(KernelClass cls, double work, cudaStream_t s);
  ~LaunchScope();
  LaunchScope(const LaunchScope&) = delete;
  LaunchScope& operator=(const LaunchScope&) = delete;

 private:
  KernelClass cls_;
  double work_;
  cudaStream_t s_;
  cudaEvent_t a_ = nullptr, b_ = nullptr;
  bool active_ = false;
};

}  // namespace qa

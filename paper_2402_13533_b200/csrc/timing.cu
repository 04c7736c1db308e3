// Launch accounting: a global launch counter and optional per-class CUDA-event timing of each
// launch on its own stream (bench.py reads it to report the dominant kernel's live duration).
#include <atomic>
#include <mutex>
#include <string.h>
#include <vector>

#include "qa_internal.h"
#include "qa_timing.h"

namespace qa {

namespace {

const char* kClassNames[kNumClasses] = {"gemm_i8", "gemm_bf16", "quantize", "tt", "dequant", "merge"};

struct Rec {
  int cls;
  cudaEvent_t a, b;
  double work;
};

std::atomic<int64_t> g_launches{0};
std::atomic<bool> g_enabled{false};
std::mutex g_mu;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

}  // namespace

void count_launches(int n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

LaunchScope::LaunchScope(KernelClass cls, double work, cudaStream_t s) : cls_(cls), work_(work), s_(s) {
  if (!g_enabled.load(std::memory_order_relaxed)) return;
  std::lock_guard<std::mutex> lk(g_mu);
  a_ = take_event();
  b_ = take_event();
  cudaEventRecord(a_, s_);
  active_ = true;
}

LaunchScope::~LaunchScope() {
  if (!active_) return;
  std::lock_guard<std::mutex> lk(g_mu);
  cudaEventRecord(b_, s_);
  g_recs.push_back({static_cast<int>(cls_), a_, b_, work_});
}

}  // namespace qa

using namespace qa;

extern "C" {

int64_t qa_launch_count(void) { return g_launches.load(); }

int qa_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& r : g_recs) {
    cudaEventSynchronize(r.b);
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
  g_enabled.store(on != 0);
  return QA_OK;
}

int qa_timing_read(const char* kernel_class, double* total_ms, int64_t* launches, double* work) {
  int cls = -1;
  for (int i = 0; i < kNumClasses; ++i)
    if (kernel_class != nullptr && strcmp(kernel_class, kClassNames[i]) == 0) cls = i;
  if (cls < 0) {
    set_error("unknown kernel class %s", kernel_class ? kernel_class : "(null)");
    return QA_ERR_ARG;
  }
  std::lock_guard<std::mutex> lk(g_mu);
  double ms = 0.0, w = 0.0;
  int64_t n = 0;
  for (auto& r : g_recs) {
    if (r.cls != cls) continue;
    cudaError_t e = cudaEventSynchronize(r.b);
    if (e != cudaSuccess) return cuda_status(e, "qa_timing_read");
    float t = 0.f;
    cudaEventElapsedTime(&t, r.a, r.b);
    ms += t;
    w += r.work;
    ++n;
  }
  if (total_ms) *total_ms = ms;
  if (launches) *launches = n;
  if (work) *work = w;
  return QA_OK;
}

}  // extern "C"

// Error state, launch accounting and per-class CUDA-event timing for the C ABI.
#include <atomic>
#include <cstdio>
#include <mutex>
#include <string>
#include <vector>

#include "slq_common.cuh"

namespace slq {

static thread_local std::string g_error;
static std::atomic<uint64_t> g_launches{0};

void set_error(const std::string& msg) { g_error = msg; }

int fail(int code, const std::string& msg) {
  g_error = msg;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  g_error = std::string("CUDA error ") + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ") in " + what;
  return e == cudaErrorMemoryAllocation ? SLQ_ERR_ALLOC : SLQ_ERR_CUDA;
}

struct Rec {
  int cls;
  cudaEvent_t a, b;
};
static std::mutex g_mu;
static bool g_prof = false;
static std::vector<Rec> g_recs;
static std::vector<cudaEvent_t> g_pool;   // events are created once and recycled
static int64_t g_class_launches[K_NUM_CLASSES] = {0};

static cudaEvent_t pooled_event() {
  if (g_pool.empty()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
  cudaEvent_t e = g_pool.back();
  g_pool.pop_back();
  return e;
}

void launch_begin(KernelClass k, cudaStream_t s) {
  g_launches.fetch_add(1, std::memory_order_relaxed);
  std::lock_guard<std::mutex> lk(g_mu);
  g_class_launches[k] += 1;
  if (!g_prof) return;
  Rec r{static_cast<int>(k), pooled_event(), pooled_event()};
  cudaEventRecord(r.a, s);
  g_recs.push_back(r);
}

void launch_end(KernelClass k, cudaStream_t s) {
  std::lock_guard<std::mutex> lk(g_mu);
  if (!g_prof) return;
  for (auto it = g_recs.rbegin(); it != g_recs.rend(); ++it) {
    if (it->cls == static_cast<int>(k)) {
      cudaEventRecord(it->b, s);
      return;
    }
  }
}

}  // namespace slq

using namespace slq;

extern "C" const char* slq_last_error(void) { return g_error.c_str(); }

extern "C" uint64_t slq_launch_count(void) { return g_launches.load(); }

extern "C" void slq_profile_begin(void) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& r : g_recs) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
  g_recs.clear();
  while (g_pool.size() < 4096) {   // pre-create so recording stays cheap inside timed regions
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) break;
    g_pool.push_back(e);
  }
  for (auto& c : g_class_launches) c = 0;
  g_prof = true;
}

extern "C" int slq_profile_end(double* ms, int64_t* launches, int n) {
  std::vector<Rec> recs;
  int64_t counts[K_NUM_CLASSES];
  {
    std::lock_guard<std::mutex> lk(g_mu);
    g_prof = false;
    recs.swap(g_recs);
    for (int i = 0; i < K_NUM_CLASSES; ++i) counts[i] = g_class_launches[i];
  }
  double acc[K_NUM_CLASSES] = {0};
  for (auto& r : recs) {
    cudaEventSynchronize(r.b);
    float t = 0.f;
    if (cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess) acc[r.cls] += t;
  }
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& r : recs) { g_pool.push_back(r.a); g_pool.push_back(r.b); }
  }
  const int m = n < K_NUM_CLASSES ? n : K_NUM_CLASSES;
  for (int i = 0; i < m; ++i) {
    if (ms) ms[i] = acc[i];
    if (launches) launches[i] = counts[i];
  }
  return K_NUM_CLASSES;
}

extern "C" const char* slq_build_info(void) {
  static char buf[256];
  int rt = 0;
  cudaRuntimeGetVersion(&rt);
  snprintf(buf, sizeof(buf), "libslq_b200 sm_100a cudart=%d nvcc=%d.%d", rt, __CUDACC_VER_MAJOR__,
           __CUDACC_VER_MINOR__);
  return buf;
}

#include "profile.hpp"

#include <mutex>
#include <string>
#include <vector>

#include "capi_guard.hpp"

namespace rp::prof {

std::atomic<bool> g_enabled{false};

namespace {

struct Rec {
  int cls;
  int device;
  cudaEvent_t a, b;
  double flops, bytes;
};

std::mutex g_mu;
std::vector<Rec*> g_recs;
std::vector<std::pair<int, cudaEvent_t>> g_pool;  // (device, event)

cudaEvent_t get_event(int device) {
  for (size_t i = 0; i < g_pool.size(); ++i) {
    if (g_pool[i].first == device) {
      cudaEvent_t e = g_pool[i].second;
      g_pool.erase(g_pool.begin() + (long)i);
      return e;
    }
  }
  cudaEvent_t e;
  RP_CUDA(cudaEventCreate(&e));
  return e;
}

const char* kNames[RP_PROF_NUM_CLASSES] = {"conv_fprop", "conv_dgrad", "conv_wgrad", "synthetic_grad",
                                           "correct", "sgd", "head", "stem", "other"};

}  // namespace

void begin(int cls, cudaStream_t s, double flops, double bytes, void** token) {
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(g_mu);
  Rec* r = new Rec{cls, dev, get_event(dev), get_event(dev), flops, bytes};
  RP_CUDA(cudaEventRecord(r->a, s));
  g_recs.push_back(r);
  *token = r;
}

void end(void* token, cudaStream_t s) {
  Rec* r = static_cast<Rec*>(token);
  cudaEventRecord(r->b, s);
}

}  // namespace rp::prof

extern "C" {

int rp_profile_enable(int32_t on) {
  rp::prof::g_enabled.store(on != 0);
  return RP_OK;
}

int rp_profile_collect(int64_t* launches, double* ms, double* flops, double* bytes) {
  return rp::guard([&] {
    using namespace rp::prof;
    std::lock_guard<std::mutex> lk(g_mu);
    for (int c = 0; c < RP_PROF_NUM_CLASSES; ++c) {
      if (launches) launches[c] = 0;
      if (ms) ms[c] = 0;
      if (flops) flops[c] = 0;
      if (bytes) bytes[c] = 0;
    }
    for (Rec* r : g_recs) {
      int prev = 0;
      cudaGetDevice(&prev);
      cudaSetDevice(r->device);
      RP_CUDA(cudaEventSynchronize(r->b));
      float t = 0.f;
      RP_CUDA(cudaEventElapsedTime(&t, r->a, r->b));
      cudaSetDevice(prev);
      if (launches) launches[r->cls] += 1;
      if (ms) ms[r->cls] += t;
      if (flops) flops[r->cls] += r->flops;
      if (bytes) bytes[r->cls] += r->bytes;
      g_pool.emplace_back(r->device, r->a);
      g_pool.emplace_back(r->device, r->b);
      delete r;
    }
    g_recs.clear();
  });
}

const char* rp_profile_class_name(int32_t cls) {
  if (cls < 0 || cls >= RP_PROF_NUM_CLASSES) return "?";
  return rp::prof::kNames[cls];
}

}  // extern "C"

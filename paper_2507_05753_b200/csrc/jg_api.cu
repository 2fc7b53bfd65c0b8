// jg_api.cu — error state, version and launch accounting for libjigsaw_sm100.so.
#include "jg_common.cuh"
#include <mutex>

namespace jg {

static thread_local std::string t_last_error;
std::atomic<int64_t> g_launches{0};

void set_error(const std::string& msg) { t_last_error = msg; }

int shape_error(const std::string& msg) {
  t_last_error = msg;
  return JG_ERR_SHAPE;
}

int cuda_check(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return JG_OK;
  t_last_error = std::string(what) + ": " + cudaGetErrorString(e);
  return JG_ERR_CUDA;
}

int num_sms() {
  static int n = 0;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  });
  return n;
}

}  // namespace jg

extern "C" {

const char* jg_version(void) { return "jigsaw_sm100 0.1.0 (sm_100a, tcgen05/TMA)"; }

const char* jg_last_error(void) { return jg::t_last_error.c_str(); }

int64_t jg_launch_count(void) { return jg::g_launches.load(std::memory_order_relaxed); }

size_t jg_gemm_desc_size(void) { return sizeof(jg_gemm_desc); }

}  // extern "C"

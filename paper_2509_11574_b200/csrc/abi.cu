// abi.cu -- status strings, thread-local error messages and version of the libgps C ABI.
#include <cuda_runtime.h>

#include <string>

#include "common.cuh"

namespace gps {
namespace {
thread_local std::string g_last_error;
}
void set_error(const std::string& msg) { g_last_error = msg; }
gps_status cuda_fail(const char* where, cudaError_t e) {
  g_last_error = std::string(where) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  return GPS_ERR_CUDA;
}
gps_status invalid(const std::string& msg) {
  g_last_error = msg;
  return GPS_ERR_INVALID_ARG;
}
}  // namespace gps

extern "C" {
const char* gps_status_string(gps_status s) {
  switch (s) {
    case GPS_OK: return "GPS_OK";
    case GPS_ERR_INVALID_ARG: return "GPS_ERR_INVALID_ARG";
    case GPS_ERR_OUT_OF_BLOCKS: return "GPS_ERR_OUT_OF_BLOCKS";
    case GPS_ERR_WORKSPACE_TOO_SMALL: return "GPS_ERR_WORKSPACE_TOO_SMALL";
    case GPS_ERR_CUDA: return "GPS_ERR_CUDA";
    case GPS_ERR_OOM: return "GPS_ERR_OOM";
  }
  return "GPS_ERR_UNKNOWN";
}
const char* gps_last_error(void) { return gps::g_last_error.c_str(); }
int gps_abi_version(void) { return GPS_ABI_VERSION; }

gps_status gps_debug_check_word_sync(int64_t* word, int32_t* checked) {
  if (!word) return gps::invalid("gps_debug_check_word_sync: null argument");
  GPS_CHECK_CUDA(cudaDeviceSynchronize());
  const unsigned long long w = gps::check_word_take_volume() | gps::check_word_take_render() |
                               gps::check_word_take_adding() | gps::check_word_take_tracking();
  GPS_CHECK_CUDA(cudaGetLastError());
  *word = (int64_t)w;
#ifdef GPS_CHECKED
  if (checked) *checked = 1;
#else
  if (checked) *checked = 0;
#endif
  return GPS_OK;
}
}

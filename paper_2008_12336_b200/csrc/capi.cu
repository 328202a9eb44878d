// C-ABI plumbing: error strings, version, device queries.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace gb {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int num_sms() {
  static thread_local int cached_dev = -1, cached_sms = 0;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (dev != cached_dev) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
        sms < 1)
      sms = 148;
    cached_dev = dev;
    cached_sms = sms;
  }
  return cached_sms;
}

}  // namespace gb

GB_API const char *gb_last_error(void) { return gb::g_err; }

GB_API int gb_version(void) { return 1; }

GB_API int gb_device_info(int device, int *num_sms, int *max_warps_per_sm) {
  GB_REQUIRE(num_sms && max_warps_per_sm, "gb_device_info: null pointer");
  int sms = 0, thr = 0;
  GB_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  GB_CUDA_TRY(cudaDeviceGetAttribute(&thr, cudaDevAttrMaxThreadsPerMultiProcessor, device));
  *num_sms = sms;
  *max_warps_per_sm = thr / 32;
  return GB_OK;
}

// Failure is an expected outcome here (already pinned / registered memory,
// some mappings): callers fall back to a pinned copy.  The runtime's sticky
// last-error slot is cleared so the failure cannot surface in the next
// launch's GB_CHECK_LAUNCH (cudaGetLastError) as an unrelated error.
GB_API int gb_host_register(void *ptr, size_t bytes) {
  GB_REQUIRE(ptr && bytes > 0, "gb_host_register: bad args");
  const cudaError_t e = cudaHostRegister(ptr, bytes, cudaHostRegisterDefault);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    gb::set_error("cudaHostRegister: %s", cudaGetErrorString(e));
    return GB_E_CUDA;
  }
  return GB_OK;
}

GB_API int gb_host_unregister(void *ptr) {
  GB_REQUIRE(ptr, "gb_host_unregister: null pointer");
  const cudaError_t e = cudaHostUnregister(ptr);
  if (e != cudaSuccess) {
    (void)cudaGetLastError();
    gb::set_error("cudaHostUnregister: %s", cudaGetErrorString(e));
    return GB_E_CUDA;
  }
  return GB_OK;
}


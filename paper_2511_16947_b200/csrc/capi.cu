// capi.cu — C ABI plumbing: thread-local error message, version, device info.
#include <stdarg.h>

#include "common.cuh"

namespace hep {
static thread_local char g_err[1024] = "";
void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
}  // namespace hep

extern "C" const char *hep_last_error(void) { return hep::g_err; }

extern "C" int hep_abi_version(void) { return 1; }

extern "C" int hep_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return n;
}

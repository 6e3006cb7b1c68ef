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

// measured defaults; see hep_tuning in include/hep.h
static const hep_tuning kDefaultTuning = {
    /*st256*/ 1, /*pair_wait_cluster*/ 0, /*ffn_pair*/ -2, /*ffn_light_rows*/ 256, /*wgrad_order*/ 1,
    /*l2_policy*/ 0, /*light_first*/ 1, /*raster_gm1*/ 16, /*raster_gm2*/ 8, /*sched_lexmin_warps*/ 4,
    /*lsu256*/ 1, /*ffn_clock*/ 0, /*router_tile_rows*/ 0, /*pair_wave_sync*/ 60, /*lp_dsm*/ 1, /*light_wave_sync*/ 0, /*router_mc*/ 0, /*router_pair*/ 0, /*wgrad_wave_sync*/ 0, /*wgrad_raster*/ 1, /*sched_route_serial*/ 0, {0}};
hep_tuning g_tuning = kDefaultTuning;
}  // namespace hep

extern "C" int hep_tuning_get(hep_tuning *out) {
    if (!out) {
        hep::set_error("hep_tuning_get: null pointer");
        return HEP_E_CONTRACT;
    }
    *out = hep::g_tuning;
    return HEP_OK;
}

extern "C" int hep_tuning_set(const hep_tuning *in) {
    if (!in) {
        hep::set_error("hep_tuning_set: null pointer");
        return HEP_E_CONTRACT;
    }
    const int *src = reinterpret_cast<const int *>(in);
    const int *def = reinterpret_cast<const int *>(&hep::kDefaultTuning);
    int *dst = reinterpret_cast<int *>(&hep::g_tuning);
    for (size_t i = 0; i < sizeof(hep_tuning) / sizeof(int); ++i) dst[i] = src[i] == -1 ? def[i] : src[i];
    return HEP_OK;
}

extern "C" const char *hep_last_error(void) { return hep::g_err; }

extern "C" int hep_abi_version(void) { return 1; }

extern "C" int hep_device_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return 0;
    return n;
}

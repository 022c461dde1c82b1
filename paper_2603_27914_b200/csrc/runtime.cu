// Host-side runtime of libitq3: thread-local error strings and launch checks.
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace itq3 {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: CUDA error %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
        return ITQ3_E_CUDA;
    }
    return ITQ3_OK;
}

}  // namespace itq3

extern "C" const char* itq3_version(void) { return "libitq3 0.1.0 (sm_100a)"; }

extern "C" const char* itq3_last_error(void) { return itq3::g_err; }

extern "C" int itq3_sm_count(void) {
    int dev = 0, n = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return -1;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) return -1;
    return n;
}

// Scalar binary16 codec on the host (encode_f16 / decode_f16, packing.py:87-109): the same
// bit logic the kernels use, compiled for the host side of the library.
extern "C" uint16_t itq3_f16_encode(double x) { return itq3::f64_to_f16_bits(x); }
extern "C" double itq3_f16_decode(uint16_t bits) { return itq3::f16_bits_to_f64(bits); }

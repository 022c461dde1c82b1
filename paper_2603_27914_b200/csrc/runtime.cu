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

// fp32 copy by one CTA of 1024 threads, 16-byte vectors (n % 4 == 0, 16-byte aligned): the e2e step's
// host -> device input copy inside the token's CUDA graph.  `src` may be pinned host memory (UVA-mapped):
// one short kernel reading over the host link instead of a DMA-engine memcpy node.
__global__ void __launch_bounds__(1024) copy_f32_kernel(float4* __restrict__ dst, const float4* __restrict__ src,
                                                        int64_t n4) {
    for (int64_t i = threadIdx.x; i < n4; i += 1024) dst[i] = src[i];
}

extern "C" int itq3_copy_f32(float* dst, const float* src, int64_t n, void* stream) {
    if (n < 0 || (n & 3) || (((uintptr_t)dst | (uintptr_t)src) & 15)) {
        itq3::set_error("copy_f32: n must be a multiple of 4 and both pointers 16-byte aligned");
        return ITQ3_E_DOMAIN;
    }
    if (n == 0) return ITQ3_OK;
    copy_f32_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>((float4*)dst, (const float4*)src, n / 4);
    return itq3::check_launch("itq3_copy_f32");
}

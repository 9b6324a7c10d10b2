// SPDX-License-Identifier: Apache-2.0
// ABI probes and error strings for klotski/kernels.h.
#include "common.cuh"

extern "C" int kl_abi_version(void) { return 1; }

extern "C" int kl_device_supported(void) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return 0;
    cudaDeviceProp p{};
    if (cudaGetDeviceProperties(&p, dev) != cudaSuccess) return 0;
    return p.major == 10 && p.minor == 0 ? 1 : 0;
}

extern "C" const char* kl_error_string(int code) {
    switch (code) {
        case KL_OK: return "ok";
        case KL_EINVAL: return "invalid argument (shape, pointer or alignment)";
        case KL_EUNSUPPORTED: return "shape not supported by this kernel";
        case KL_ENODEV: return "no sm_100 device or driver entry point";
        default: return code > 0 ? cudaGetErrorString(static_cast<cudaError_t>(code)) : "unknown error";
    }
}

// Benchmarking aid: one thread spins until *flag (host-mapped) becomes
// non-zero, so work queued behind it starts without host launch latency.
namespace {
__global__ void spin_flag_kernel(const volatile int* flag) {
    while (*flag == 0) {
    }
}
}  // namespace

extern "C" int kl_debug_spin_flag(const int* flag, cudaStream_t stream) {
    if (flag == nullptr) return KL_EINVAL;
    spin_flag_kernel<<<1, 1, 0, stream>>>(flag);
    return kl::check_launch();
}

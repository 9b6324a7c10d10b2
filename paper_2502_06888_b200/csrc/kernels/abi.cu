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

// Device timestamp: one thread writes %globaltimer (ns, the clock cudaEvent
// timestamps come from) into *dst once every earlier grid of the stream has
// completed. The engine marks op boundaries with these instead of timed
// cudaEvents: a timed event record stalls the stream for tens of microseconds
// while a copy engine streams pinned host memory, and breaks programmatic
// dependent launch (tools/dma_interference_probe.py). Launched as a PDL
// secondary that releases its own dependents first, so the next kernel still
// pre-launches while the previous one runs; griddepcontrol.wait then returns
// when that previous grid has completed.
namespace kl {
int g_pdl = 1;  // kl_tune(KL_TUNE_PDL, ...)
}
namespace {
__global__ void stamp_kernel(unsigned long long* dst) {
    kl::griddep_launch_dependents();
    kl::griddep_wait();
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    *dst = t;
}
}  // namespace

namespace kl {
thread_local EndMark t_next_end{nullptr, nullptr};
}

extern "C" int kl_stamp_end_next_launch(unsigned long long* dst, unsigned* counter) {
    if ((dst == nullptr) != (counter == nullptr)) return KL_EINVAL;
    kl::t_next_end = kl::EndMark{dst, counter};
    return KL_OK;
}

extern "C" int kl_stamp_end_pending(void) {
    const bool pending = kl::t_next_end.t != nullptr;
    kl::t_next_end = kl::EndMark{nullptr, nullptr};
    return pending ? 1 : 0;
}

extern "C" int kl_stamp(unsigned long long* dst, cudaStream_t stream) {
    if (dst == nullptr) return KL_EINVAL;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(32);
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = kl::g_pdl ? 1 : 0;
    KL_CUDA_TRY(cudaLaunchKernelEx(&cfg, stamp_kernel, dst));
    return kl::check_launch();
}

// devguard.h -- make the device that owns a buffer current for the duration of
// an entry point (the PPO / pixel entry points take raw device pointers, not a
// handle with a device; their launches, SM-count and attribute queries must go
// to the tensors' device even when another device is current).
#pragma once
#include <cuda_runtime.h>

namespace dk {
struct PtrDeviceGuard {
    int prev = -1, dev = -1;
    explicit PtrDeviceGuard(const void *p) {
        if (!p) return;
        cudaPointerAttributes a;
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();  // not a CUDA pointer: leave the current device
            return;
        }
        if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged) return;
        cudaGetDevice(&prev);
        if (prev != a.device) {
            dev = a.device;
            cudaSetDevice(dev);
        }
    }
    ~PtrDeviceGuard() {
        if (dev >= 0 && prev >= 0) cudaSetDevice(prev);
    }
};

// Dynamic shared memory above 48 KB is a per-device function attribute: opt a
// kernel in once per device (and again when a launch needs more).
struct SmemOptIn {
    size_t bytes[64] = {};
    cudaError_t ensure(const void *fn, size_t smem) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (dev < 0 || dev >= 64)
            return cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (smem <= bytes[dev]) return cudaSuccess;
        cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)smem);
        if (e == cudaSuccess) bytes[dev] = smem;
        return e;
    }
};
}  // namespace dk

// hpr_device_scope.h — the C-ABI entry points make the handle's device
// current for their own work and give the caller's thread its previous
// device back on every exit path (including the error paths, which unwind
// through exceptions inside the ABI functions).
#pragma once

#include <cuda_runtime.h>

namespace hpr {

struct DeviceScope {
    int prev = -1;
    cudaError_t err = cudaSuccess;
    explicit DeviceScope(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
        err = cudaSetDevice(dev);
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceScope(const DeviceScope&) = delete;
    DeviceScope& operator=(const DeviceScope&) = delete;
};

}  // namespace hpr

// capi_common.cuh -- host-side plumbing shared by the C-ABI translation units.
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>

#include <cuda_runtime.h>

#include "../../include/lfg.h"

namespace lfg {

void set_error(const std::string& msg);

struct Error : std::runtime_error {
    int status;
    Error(int st, const std::string& m) : std::runtime_error(m), status(st) {}
};

inline void cuda_check(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return;
    if (e == cudaErrorMemoryAllocation) {
        cudaGetLastError();
        throw Error(LFG_ENOMEM, std::string(what) + ": " + cudaGetErrorString(e));
    }
    throw Error(LFG_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F&& f) {
    try {
        f();
        return LFG_OK;
    } catch (const Error& e) {
        set_error(e.what());
        return e.status;
    } catch (const std::bad_alloc&) {
        set_error("host allocation failed");
        return LFG_ENOMEM;
    } catch (const std::exception& e) {
        set_error(e.what());
        return LFG_EINVAL;
    }
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cuda_check(cudaSetDevice(dev), "cudaSetDevice");
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

template <class T>
T* dmalloc(size_t n, const char* what) {
    void* p = nullptr;
    cuda_check(cudaMalloc(&p, n * sizeof(T)), what);
    return static_cast<T*>(p);
}

inline void dfree(void* p) {
    if (p) cudaFree(p);
}

inline bool is_pow2(int64_t v) { return v > 0 && (v & (v - 1)) == 0; }

// ceil(x * 2^32) for x in [0,1]: u * 2^-32 < x  <=>  u < ceil(x * 2^32)
// (power-of-two scaling is exact, so this is the reference's double compare).
inline uint64_t threshold32(double x) {
    if (x <= 0.0) return 0;
    if (x >= 1.0) return uint64_t{1} << 32;
    const double t = x * 4294967296.0;
    const uint64_t fl = uint64_t(t);
    return double(fl) == t ? fl : fl + 1;
}

}  // namespace lfg

// capi_peer.cu -- C ABI for single-node peer-memory shard exchange (include/lfg.h,
// "peer memory"): CUDA IPC handles of device buffers, stream-ordered device-side
// step barriers, and peer copies.  Used by paper_1204_5072_b200/shard.py
// (PeerComm) so strip shards exchange rows over NVLink without NCCL and without
// host synchronisation.
#include <cstring>

#include "../../include/lfg.h"
#include "capi_common.cuh"
#include "kpz_kernels.cuh"

using namespace lfg;

static_assert(sizeof(cudaIpcMemHandle_t) <= 64, "IPC handle larger than the ABI's 64 bytes");

extern "C" {

}  // extern "C"

namespace {

// cuMemGetAddressRange through the runtime's driver entry point (no link-time
// dependency on libcuda): IPC handles name whole allocations, while a caching
// allocator may hand out interior pointers.
typedef int (*MemGetAddressRangeFn)(unsigned long long*, size_t*, unsigned long long);

void allocation_base(const void* p, unsigned long long* base) {
    static MemGetAddressRangeFn fn = nullptr;
    if (!fn) {
        void* sym = nullptr;
        cudaDriverEntryPointQueryResult q;
        cuda_check(cudaGetDriverEntryPoint("cuMemGetAddressRange", &sym, cudaEnableDefault, &q),
                   "cudaGetDriverEntryPoint(cuMemGetAddressRange)");
        if (!sym || q != cudaDriverEntryPointSuccess) throw Error(LFG_ECUDA, "cuMemGetAddressRange unavailable");
        fn = reinterpret_cast<MemGetAddressRangeFn>(sym);
    }
    size_t size = 0;
    if (fn(base, &size, reinterpret_cast<unsigned long long>(p)) != 0)
        throw Error(LFG_ECUDA, "cuMemGetAddressRange failed (not a device allocation?)");
}

}  // namespace

extern "C" {

int lfg_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset) {
    return guarded([&] {
        if (!dev_ptr || !handle64 || !offset) throw Error(LFG_EINVAL, "null pointer");
        unsigned long long base = 0;
        allocation_base(dev_ptr, &base);
        cudaIpcMemHandle_t hd;
        cuda_check(cudaIpcGetMemHandle(&hd, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
        std::memset(handle64, 0, 64);
        std::memcpy(handle64, &hd, sizeof(hd));
        *offset = uint64_t(reinterpret_cast<unsigned long long>(dev_ptr) - base);
    });
}

int lfg_ipc_open_handle(const void* handle64, int32_t device, void** dev_ptr) {
    return guarded([&] {
        if (!handle64 || !dev_ptr) throw Error(LFG_EINVAL, "null pointer");
        DeviceGuard g(device);
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, handle64, sizeof(hd));
        cuda_check(cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
    });
}

int lfg_ipc_close(void* dev_ptr, int32_t device) {
    return guarded([&] {
        DeviceGuard g(device);
        if (dev_ptr) cuda_check(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
    });
}

int lfg_peer_signal(void* stream, void* flag_a, void* flag_b, uint32_t value, int32_t device) {
    return guarded([&] {
        DeviceGuard g(device);
        cuda_check(peer_launch_signal(static_cast<uint32_t*>(flag_a), static_cast<uint32_t*>(flag_b), value,
                                      static_cast<cudaStream_t>(stream)),
                   "peer signal");
    });
}

int lfg_peer_wait(void* stream, const void* flag_a, const void* flag_b, uint32_t value, uint64_t max_spins,
                  void* err_flag, int32_t device) {
    return guarded([&] {
        DeviceGuard g(device);
        cuda_check(peer_launch_wait(static_cast<const uint32_t*>(flag_a), static_cast<const uint32_t*>(flag_b), value,
                                    max_spins, static_cast<uint32_t*>(err_flag), static_cast<cudaStream_t>(stream)),
                   "peer wait");
    });
}

int lfg_copy_async(void* dst, const void* src, size_t bytes, void* stream, int32_t device) {
    return guarded([&] {
        DeviceGuard g(device);
        cuda_check(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, static_cast<cudaStream_t>(stream)),
                   "peer copy");
    });
}

}  // extern "C"

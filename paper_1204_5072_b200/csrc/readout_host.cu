// readout_host.cu -- handle-free device readouts of host lattices in the
// reference word layout (include/lfg.h "readouts of host lattices").
//
// The C++ drop-in's free functions interface_width(const SlopeField&),
// reconstruct_heights(const SlopeField&) and open_bonds_per_particle(const
// OccupancyLattice&) take an arbitrary host lattice.  They must give the
// reference's answer for EVERY field the reference accepts -- any power-of-two
// L >= 4 and, for the KPZ readouts, slope fields that are not integrable
// (interface_width integrates along row 0 and then up every column without
// checking closure, kpz.cpp:62-81).  So these kernels read the two slope
// planes themselves, bit by bit in the reference's index order (site j*L+i,
// bit idx&63 of uint64 word idx>>6), instead of going through the spin
// representation and its DT plan constraints (L >= 64).
#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/lfg_kmc.h"
#include "capi_common.cuh"
#include "kmc_kernels.cuh"
#include "kpz_kernels.cuh"

namespace lfg {
namespace {

__device__ __forceinline__ int bit64(const uint64_t* __restrict__ w, int64_t idx) {
    return int((w[idx >> 6] >> (idx & 63)) & 1u);
}

// H0[i] = sum_{k=1..i} slope_x(k, 0)  (kpz.cpp:66-69), one CTA.
__global__ void __launch_bounds__(1024) slopes_row0_kernel(const uint64_t* __restrict__ X, int L,
                                                           int32_t* __restrict__ H0) {
    __shared__ int32_t wsum[32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int chunk = (L + 1023) / 1024;
    const int i0 = t * chunk, i1 = min(L, i0 + chunk);
    int32_t s = 0;
    for (int i = max(i0, 1); i < i1; ++i) s += bit64(X, i) ? 1 : -1;
    int32_t inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int32_t w = wsum[lane];
        int32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t v = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= o) wi += v;
        }
        wsum[lane] = wi - w;
    }
    __syncthreads();
    int32_t acc = wsum[warp] + inc - s;
    for (int i = i0; i < i1; ++i) {
        if (i > 0) acc += bit64(X, i) ? 1 : -1;
        H0[i] = acc;
    }
}

// Column segments of S rows (kpz.cpp:70-77 split by rows): for column i and
// segment g, p = column height relative to the segment start (the step into
// global row 0 is skipped), P1 = sum p, D = last p, sum p^2 into *p2.
__global__ void slopes_colseg_kernel(const uint64_t* __restrict__ Y, int L, int S, int32_t* __restrict__ P1,
                                     int32_t* __restrict__ D, unsigned long long* __restrict__ p2) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x, g = blockIdx.y;
    long long s2 = 0;
    if (i < L) {
        int32_t p = 0, s1 = 0;
        const int j0 = g * S, j1 = min(L, j0 + S);
        for (int j = j0; j < j1; ++j) {
            if (j > 0) p += bit64(Y, int64_t(j) * L + i) ? 1 : -1;
            s1 += p;
            s2 += (long long)p * p;
        }
        P1[size_t(g) * L + i] = s1;
        D[size_t(g) * L + i] = p;
    }
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_down_sync(0xFFFFFFFFu, s2, o);
    if ((threadIdx.x & 31) == 0 && s2) atomicAdd(p2, (unsigned long long)s2);
}

// reconstruct_heights (kpz.cpp:21-34): h(i, j) = H0[i] + column steps.
__global__ void slopes_heights_kernel(const uint64_t* __restrict__ Y, const int32_t* __restrict__ H0, int L,
                                      int32_t* __restrict__ h) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L) return;
    int32_t v = H0[i];
    h[i] = v;
    for (int j = 1; j < L; ++j) {
        v += bit64(Y, int64_t(j) * L + i) ? 1 : -1;
        h[size_t(j) * L + i] = v;
    }
}

// The path-independence check of kpz.cpp:35-47, every site, periodic wrap.
__global__ void slopes_heights_check_kernel(const uint64_t* __restrict__ X, const uint64_t* __restrict__ Y,
                                            const int32_t* __restrict__ h, int L,
                                            unsigned long long* __restrict__ bad) {
    const int64_t n = int64_t(L) * L;
    const int mask = L - 1;
    unsigned long long nb = 0;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int i = int(k % L), j = int(k / L);
        const int32_t v = h[k];
        const int32_t sx = bit64(X, k) ? 1 : -1, sy = bit64(Y, k) ? 1 : -1;
        if (v - h[size_t(j) * L + ((i - 1) & mask)] != sx || v - h[size_t((j - 1) & mask) * L + i] != sy) ++nb;
    }
    nb = __reduce_add_sync(0xFFFFFFFFu, unsigned(nb));
    if ((threadIdx.x & 31) == 0 && nb) atomicAdd(bad, nb);
}

// open_bonds_per_particle (kmc.cpp:20-40) for any L: one thread per site,
// B particles on valid (even x^y^z) sites count their A neighbours.
__constant__ int8_t c_fcc_off[12][3] = {{1, 1, 0},  {1, -1, 0}, {-1, 1, 0}, {-1, -1, 0}, {1, 0, 1},  {1, 0, -1},
                                        {-1, 0, 1}, {-1, 0, -1}, {0, 1, 1}, {0, 1, -1},  {0, -1, 1}, {0, -1, -1}};

__global__ void kmc_open_bonds_generic_kernel(const uint64_t* __restrict__ w, int L,
                                              unsigned long long* __restrict__ out2) {
    const int64_t n = int64_t(L) * L * L;
    const int mask = L - 1;
    unsigned long long np = 0, no = 0;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < n; k += int64_t(gridDim.x) * blockDim.x) {
        const int x = int(k % L), y = int((k / L) % L), z = int(k / (int64_t(L) * L));
        if (((x ^ y ^ z) & 1) || !bit64(w, k)) continue;
        ++np;
#pragma unroll
        for (int d = 0; d < 12; ++d) {
            const int64_t q = (int64_t((z + c_fcc_off[d][2]) & mask) * L + ((y + c_fcc_off[d][1]) & mask)) * L +
                              ((x + c_fcc_off[d][0]) & mask);
            no += !bit64(w, q);
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        np += __shfl_down_sync(0xFFFFFFFFu, np, o);
        no += __shfl_down_sync(0xFFFFFFFFu, no, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (np) atomicAdd(out2 + 0, np);
        if (no) atomicAdd(out2 + 1, no);
    }
}

// interface_width(const HeightField&) (kpz.cpp:51-60): exact int64 sums.
__global__ void heights_sums_kernel(const int32_t* __restrict__ h, size_t n, unsigned long long* __restrict__ out2) {
    long long s = 0, s2 = 0;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n; k += size_t(gridDim.x) * blockDim.x) {
        const long long v = h[k];
        s += v;
        s2 += v * v;
    }
    for (int o = 16; o > 0; o >>= 1) {
        s += __shfl_down_sync(0xFFFFFFFFu, s, o);
        s2 += __shfl_down_sync(0xFFFFFFFFu, s2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out2 + 0, (unsigned long long)s);
        atomicAdd(out2 + 1, (unsigned long long)s2);
    }
}

void check_size(int32_t L, const char* what) {  // check_size (lattice.cpp:10-16)
    if (L < 4 || !is_pow2(L))
        throw Error(LFG_EINVAL, std::string(what) + ": size must be a power of two >= 4, got " + std::to_string(L));
}

size_t word_count(uint64_t sites) { return size_t((sites + 63) / 64); }  // detail::word_count

// A stream and device allocations for one call, released on every exit path.
struct Scratch {
    cudaStream_t st = nullptr;
    std::vector<void*> ptrs;
    explicit Scratch() { cuda_check(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate"); }
    ~Scratch() {
        if (st) cudaStreamSynchronize(st);
        for (void* p : ptrs) cudaFree(p);
        if (st) cudaStreamDestroy(st);
    }
    template <class T>
    T* alloc(size_t n) {
        T* p = dmalloc<T>(std::max<size_t>(n, 1), "alloc readout scratch");
        ptrs.push_back(p);
        return p;
    }
    template <class T>
    T* upload(const T* host, size_t n) {
        T* d = alloc<T>(n);
        cuda_check(cudaMemcpyAsync(d, host, n * sizeof(T), cudaMemcpyHostToDevice, st), "upload");
        return d;
    }
    void sync() { cuda_check(cudaStreamSynchronize(st), "readout"); }
};

}  // namespace
}  // namespace lfg

using namespace lfg;

extern "C" {

int lfg_kpz_width_sums_host(int32_t device, int32_t L, const uint64_t* x, const uint64_t* y, size_t nwords,
                            int64_t* sum, int64_t* sum2) {
    return guarded([&] {
        check_size(L, "SlopeField");
        if (!x || !y || !sum || !sum2) throw Error(LFG_EINVAL, "null argument");
        const size_t need = word_count(uint64_t(L) * uint64_t(L));
        if (nwords != need) throw Error(LFG_EINVAL, "width: expected " + std::to_string(need) + " words per plane");
        DeviceGuard g(device);
        Scratch s;
        const uint64_t* X = s.upload(x, need);
        const uint64_t* Y = s.upload(y, need);
        const int S = std::min(L, 2048), G = (L + S - 1) / S;
        int32_t* H0 = s.alloc<int32_t>(size_t(L));
        int32_t* P1 = s.alloc<int32_t>(size_t(G) * L);
        int32_t* D = s.alloc<int32_t>(size_t(G) * L);
        int32_t* seglen = s.alloc<int32_t>(size_t(G));
        unsigned long long* out = s.alloc<unsigned long long>(3);
        std::vector<int32_t> lens(size_t(G), S);
        lens.back() = L - S * (G - 1);
        cuda_check(cudaMemcpyAsync(seglen, lens.data(), 4 * size_t(G), cudaMemcpyHostToDevice, s.st), "upload");
        cuda_check(cudaMemsetAsync(out, 0, 24, s.st), "memset");
        slopes_row0_kernel<<<1, 1024, 0, s.st>>>(X, L, H0);
        slopes_colseg_kernel<<<dim3(unsigned((L + 127) / 128), unsigned(G)), 128, 0, s.st>>>(Y, L, S, P1, D, out + 2);
        cuda_check(cudaGetLastError(), "width kernels");
        cuda_check(kpz_launch_width_combine(H0, P1, D, seglen, L, G, out, s.st), "width combine");
        unsigned long long h[3];
        cuda_check(cudaMemcpyAsync(h, out, 24, cudaMemcpyDeviceToHost, s.st), "readback");
        s.sync();
        *sum = int64_t(h[0]);
        *sum2 = int64_t(h[1] + h[2]);
    });
}

int lfg_kpz_heights_host(int32_t device, int32_t L, const uint64_t* x, const uint64_t* y, size_t nwords,
                         int32_t* heights, size_t n) {
    return guarded([&] {
        check_size(L, "SlopeField");
        if (!x || !y || !heights) throw Error(LFG_EINVAL, "null argument");
        const size_t need = word_count(uint64_t(L) * uint64_t(L));
        if (nwords != need) throw Error(LFG_EINVAL, "heights: expected " + std::to_string(need) + " words per plane");
        if (n != size_t(L) * size_t(L)) throw Error(LFG_EINVAL, "heights: expected L*L entries");
        DeviceGuard g(device);
        Scratch s;
        const uint64_t* X = s.upload(x, need);
        const uint64_t* Y = s.upload(y, need);
        int32_t* H0 = s.alloc<int32_t>(size_t(L));
        int32_t* h = s.alloc<int32_t>(n);
        unsigned long long* bad = s.alloc<unsigned long long>(1);
        cuda_check(cudaMemsetAsync(bad, 0, 8, s.st), "memset");
        slopes_row0_kernel<<<1, 1024, 0, s.st>>>(X, L, H0);
        slopes_heights_kernel<<<unsigned((L + 127) / 128), 128, 0, s.st>>>(Y, H0, L, h);
        const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 16));
        slopes_heights_check_kernel<<<blocks, 256, 0, s.st>>>(X, Y, h, L, bad);
        cuda_check(cudaGetLastError(), "heights kernels");
        unsigned long long nb = 0;
        cuda_check(cudaMemcpyAsync(&nb, bad, 8, cudaMemcpyDeviceToHost, s.st), "readback");
        s.sync();
        if (nb) throw Error(LFG_ECLOSURE,
                            "reconstruct_heights: slope field violates closure; heights would be path-dependent");
        cuda_check(cudaMemcpyAsync(heights, h, n * 4, cudaMemcpyDeviceToHost, s.st), "readback");
        s.sync();
    });
}

int lfg_heights_width_sums_host(int32_t device, const int32_t* heights, size_t n, int64_t* sum, int64_t* sum2) {
    return guarded([&] {
        if (!heights || !sum || !sum2) throw Error(LFG_EINVAL, "null argument");
        DeviceGuard g(device);
        Scratch s;
        const int32_t* H = s.upload(heights, n);
        unsigned long long* out = s.alloc<unsigned long long>(2);
        cuda_check(cudaMemsetAsync(out, 0, 16, s.st), "memset");
        const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 8));
        if (n) heights_sums_kernel<<<blocks, 256, 0, s.st>>>(H, n, out);
        cuda_check(cudaGetLastError(), "height sums");
        unsigned long long h[2];
        cuda_check(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, s.st), "readback");
        s.sync();
        *sum = int64_t(h[0]);
        *sum2 = int64_t(h[1]);
    });
}

int lfg_kmc_open_bond_sums_host(int32_t device, int32_t L, const uint64_t* words, size_t nwords, int64_t* particles,
                                int64_t* open) {
    return guarded([&] {
        check_size(L, "OccupancyLattice");
        if (!words || !particles || !open) throw Error(LFG_EINVAL, "null argument");
        const size_t need = word_count(uint64_t(L) * uint64_t(L) * uint64_t(L));
        if (nwords != need) throw Error(LFG_EINVAL, "open bonds: expected " + std::to_string(need) + " words");
        DeviceGuard g(device);
        Scratch s;
        const uint64_t* W = s.upload(words, need);
        unsigned long long* out = s.alloc<unsigned long long>(2);
        cuda_check(cudaMemsetAsync(out, 0, 16, s.st), "memset");
        if (L >= 32) {  // rows are whole uint32 words: the word-parallel kernel
            cuda_check(kmc_launch_open_bonds(reinterpret_cast<const uint32_t*>(W), L, L - 1, 0, L, out, s.st),
                       "open bonds");
        } else {
            kmc_open_bonds_generic_kernel<<<64, 256, 0, s.st>>>(W, L, out);
            cuda_check(cudaGetLastError(), "open bonds");
        }
        unsigned long long h[2];
        cuda_check(cudaMemcpyAsync(h, out, 16, cudaMemcpyDeviceToHost, s.st), "readback");
        s.sync();
        *particles = int64_t(h[0]);
        *open = int64_t(h[1]);
    });
}

}  // extern "C"

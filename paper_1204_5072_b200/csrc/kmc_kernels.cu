// kmc_kernels.cu -- sm_100a kernels for the 3-D fcc binary-alloy KMC.
//
// Lattice in HBM: the reference's OccupancyLattice layout (lattice.hpp:107-135)
// -- one bit per simple-cubic site, index (z*L + y)*L + x, little-endian
// 32-bit words, so upload/download is a plain copy.  Only even-parity sites
// (x^y^z even) are fcc sites (lattice.hpp:139-141).
//
// Two-layer DT: per sweep a random
// origin in [0, 2bk)^3 and a random order of the eight block sets; each phase
// is one launch over the active bk^3 blocks.  Inside a block, 256 single-hit
// rounds: the block draws one of eight inner sets of 4^3 domains (8^3 tiles)
// and every tile's active domain makes one exchange attempt.  Reach: read 2,
// write 1 (kmc.hpp:140-141) < the one-domain gap, so attempts of a round are
// independent and the result equals the CPU oracle bit for bit.
#include <cstdint>

#include "kmc_kernels.cuh"
#include "lfg_common.cuh"

namespace lfg {

__constant__ int8_t c_fcc[12][3] = {  // kFccOffsets (lattice.hpp:147-151)
    {1, 1, 0}, {1, -1, 0}, {-1, 1, 0}, {-1, -1, 0}, {1, 0, 1}, {1, 0, -1},
    {-1, 0, 1}, {-1, 0, -1}, {0, 1, 1}, {0, 1, -1}, {0, -1, 1}, {0, -1, -1}};

__device__ __forceinline__ uint32_t u4sel(const U4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// Staged rows: for block-local (ly, lz) in [-2, bk+2)^2 one 64-bit word with
// the global x bits [X0 - 16, X0 + 48): local x lx in [-2, bk+2) sits at bit
// lx + 16.  Row index (lz + 2) * E + (ly + 2), E = bk + 4.
struct KmcRows {
    unsigned long long* r;
    int E;
    __device__ __forceinline__ unsigned long long at(int ly, int lz) const { return r[(lz + 2) * E + (ly + 2)]; }
    __device__ __forceinline__ unsigned long long* ptr(int ly, int lz) const { return r + (lz + 2) * E + (ly + 2); }
};

__device__ __forceinline__ int bit_at(unsigned long long row, int lx) { return int((row >> (lx + 16)) & 1ull); }

// Number of B among the 12 fcc neighbours of (lx, ly, lz).
__device__ __forceinline__ int nb_count(const KmcRows& R, int lx, int ly, int lz) {
    const unsigned long long m2 = 5ull << (lx + 15);  // bits lx-1, lx+1
    int n = __popcll(R.at(ly - 1, lz) & m2) + __popcll(R.at(ly + 1, lz) & m2) + __popcll(R.at(ly, lz - 1) & m2) +
            __popcll(R.at(ly, lz + 1) & m2);
    n += bit_at(R.at(ly - 1, lz - 1), lx) + bit_at(R.at(ly - 1, lz + 1), lx) + bit_at(R.at(ly + 1, lz - 1), lx) +
         bit_at(R.at(ly + 1, lz + 1), lx);
    return n;
}

__device__ __forceinline__ void global_flip(uint32_t* w, int L, int gx, int gy, int gz) {
    const size_t idx = (size_t(gz) * L + gy) * L + gx;
    atomicXor(w + (idx >> 5), 1u << (idx & 31));
}

template <bool BOTH>
__global__ void __launch_bounds__(128) kmc_dt_phase_kernel(const __grid_constant__ KmcPhaseArgs a) {
    extern __shared__ __align__(16) unsigned long long smk[];
    const int L = a.L, Lm = L - 1, bk = a.bk, E = bk + 4, rows = E * E;
    const int tb = bk / 8, tpb = tb * tb * tb;
    const int sub = int(threadIdx.x) / tpb, t = int(threadIdx.x) % tpb;
    const int bpc = int(blockDim.x) / tpb;
    const int nb = L / bk, h = nb / 2;
    const int blin = int(blockIdx.x) * bpc + sub;
    const KmcSweep sw = kmc_sweep_draw(bk, a.seed, a.sweep);
    const int set = sw.set(a.phase);
    const int bxi = 2 * (blin % h) + (set & 1);
    const int byi = 2 * ((blin / h) % h) + ((set >> 1) & 1);
    const int bzi = 2 * (blin / (h * h)) + (set >> 2);
    const uint32_t block_id = (uint32_t(bzi) * uint32_t(nb) + uint32_t(byi)) * uint32_t(nb) + uint32_t(bxi);
    const int X0 = (sw.ox + bxi * bk) & Lm, Y0 = (sw.oy + byi * bk) & Lm, Z0 = (sw.oz + bzi * bk) & Lm;
    const KmcRows R{smk + size_t(sub) * rows, E};

    // Stage the block plus a 2-site halo.
    const int wpr = L >> 5, wm = wpr - 1;
    const int xs = (X0 - 16 + L) & Lm, w0 = xs >> 5, bo = xs & 31;
    for (int rr = t; rr < rows; rr += tpb) {
        const int ly = rr % E - 2, lz = rr / E - 2;
        const uint32_t* row = a.w + (size_t((Z0 + lz) & Lm) * L + size_t((Y0 + ly) & Lm)) * wpr;
        const uint32_t g0 = row[w0 & wm], g1 = row[(w0 + 1) & wm], g2 = row[(w0 + 2) & wm];
        const uint32_t lo = __funnelshift_r(g0, g1, bo), hi = __funnelshift_r(g1, g2, bo);
        R.r[rr] = (static_cast<unsigned long long>(hi) << 32) | lo;
    }
    __syncthreads();

    const int tx = t % tb, ty = (t / tb) % tb, tz = t / (tb * tb);
    const uint32_t tl = uint32_t(L / 8);
    const uint32_t tile_id = (uint32_t(bzi * tb + tz) * tl + uint32_t(byi * tb + ty)) * tl + uint32_t(bxi * tb + tx);
    uint32_t nsucc = 0;
    U4 V = {0, 0, 0, 0};
    for (int r = 0; r < kKmcRounds; ++r) {
        if ((r & 31) == 0) V = draw(a.seed, a.sweep, TAG_KMC_SET, block_id, uint32_t(r >> 5));
        const int inner = int((u4sel(V, (r >> 3) & 3) >> (4 * (r & 7))) & 7u);
        const U4 W = draw(a.seed, a.sweep, TAG_KMC_SITE, tile_id, uint32_t(r));
        const int lx0 = 8 * tx + 4 * (inner & 1), ly0 = 8 * ty + 4 * ((inner >> 1) & 1), lz0 = 8 * tz + 4 * (inner >> 2);
        // KmcKernel::draw_site (kmc.hpp:154-171) over the domain box.
        const int lx = lx0 + int(W.x & 3u), ly = ly0 + int((W.x >> 2) & 3u);
        const int tpar = ((X0 + lx) ^ (Y0 + ly)) & 1;
        const int lz = lz0 + ((((Z0 + lz0) & 1) == tpar) ? 0 : 1) + 2 * int((W.x >> 4) & 1u);
        // kmc_attempt_impl (kmc.hpp:84-111)
        const int here = bit_at(R.at(ly, lz), lx);
        if (BOTH || here) {
            const int dir = int(below(W.y, 12));
            const int px = lx + c_fcc[dir][0], py = ly + c_fcc[dir][1], pz = lz + c_fcc[dir][2];
            const int pb = bit_at(R.at(py, pz), px);
            if (pb != here) {
                const int bx_ = here ? lx : px, by_ = here ? ly : py, bz_ = here ? lz : pz;
                const int ax = here ? px : lx, ay = here ? py : ly, az = here ? pz : lz;
                // n_i excludes the A partner (no B there), n_f excludes the B partner.
                const int d = nb_count(R, bx_, by_, bz_) - (nb_count(R, ax, ay, az) - 1);
                const bool acc = d <= 0 || uint64_t(W.z) < ((uint64_t(a.thr_hi[d]) << 32) | a.thr_lo[d]);
                if (acc) {
                    atomicXor(R.ptr(by_, bz_), 1ull << (bx_ + 16));
                    atomicXor(R.ptr(ay, az), 1ull << (ax + 16));
                    global_flip(a.w, L, (X0 + bx_) & Lm, (Y0 + by_) & Lm, (Z0 + bz_) & Lm);
                    global_flip(a.w, L, (X0 + ax) & Lm, (Y0 + ay) & Lm, (Z0 + az) & Lm);
                    ++nsucc;
                }
            }
        }
        __syncthreads();
    }
    nsucc = __reduce_add_sync(0xFFFFFFFFu, nsucc);
    if ((threadIdx.x & 31) == 0 && nsucc) atomicAdd(a.counters, (unsigned long long)nsucc);
}

int kmc_blocks_per_cta(int bk) {
    const int tpb = (bk / 8) * (bk / 8) * (bk / 8);
    return tpb >= 128 ? 1 : 128 / tpb;
}

size_t kmc_phase_smem_bytes(int bk) {
    const size_t E = size_t(bk) + 4;
    return size_t(kmc_blocks_per_cta(bk)) * E * E * 8;
}

cudaError_t kmc_phase_kernel_attrs() {
    const int smem = int(kmc_phase_smem_bytes(32) > kmc_phase_smem_bytes(16) ? kmc_phase_smem_bytes(32)
                                                                              : kmc_phase_smem_bytes(16));
    cudaError_t e = cudaFuncSetAttribute(kmc_dt_phase_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         smem);
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(kmc_dt_phase_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    return e;
}

cudaError_t kmc_launch_phase(const KmcPhaseArgs& a, cudaStream_t st) {
    const int tpb = (a.bk / 8) * (a.bk / 8) * (a.bk / 8);
    const int h = a.L / a.bk / 2;
    const int active = h * h * h;
    int bpc = kmc_blocks_per_cta(a.bk);
    if (bpc > active) bpc = active;
    const dim3 grid(unsigned(active / bpc));
    const dim3 block(unsigned(bpc * tpb));
    const size_t smem = size_t(bpc) * size_t(a.bk + 4) * size_t(a.bk + 4) * 8;
    if (a.both)
        kmc_dt_phase_kernel<true><<<grid, block, smem, st>>>(a);
    else
        kmc_dt_phase_kernel<false><<<grid, block, smem, st>>>(a);
    return cudaGetLastError();
}

// make_random_alloy (lattice.cpp:117-132) with the counter RNG: valid site n
// (n = sc index >> 1) is B iff word (n & 3) of Philox(seed; n >> 2, 0, 0,
// TAG_KMC_INIT) < threshold, threshold = llround(c 2^32) as in the reference.
__global__ void kmc_init_alloy_kernel(uint32_t* w, int L, uint32_t thr_lo, uint32_t thr_hi, uint64_t seed) {
    const size_t nwords = size_t(L) * L * L / 32;
    const uint64_t thr = (uint64_t(thr_hi) << 32) | thr_lo;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nwords; k += size_t(gridDim.x) * blockDim.x) {
        const size_t idx0 = k * 32;  // first sc index of the word
        const size_t row = idx0 / size_t(L);
        const int y = int(row % size_t(L)), z = int(row / size_t(L));
        const int xpar = (y ^ z) & 1;  // valid x parity in this row
        uint32_t v = 0;
        // 16 valid sites per word: n = (idx0 + 2 j + xpar) >> 1 = idx0/2 + j
        const size_t n0 = idx0 >> 1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const U4 r = philox4x32_10(uint32_t((n0 >> 2) + q), uint32_t(((n0 >> 2) + q) >> 32), 0u,
                                       TAG_KMC_INIT << 24, uint32_t(seed), uint32_t(seed >> 32));
            const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (uint64_t(rr[e]) < thr) v |= 1u << (2 * (4 * q + e) + xpar);
        }
        w[k] = v;
    }
}

cudaError_t kmc_launch_init_alloy(uint32_t* w, int L, uint32_t thr_lo, uint32_t thr_hi, uint64_t seed,
                                  cudaStream_t st) {
    const size_t nwords = size_t(L) * L * L / 32;
    const int blocks = int(std::min<size_t>((nwords + 255) / 256, 148 * 16));
    kmc_init_alloy_kernel<<<blocks, 256, 0, st>>>(w, L, thr_lo, thr_hi, seed);
    return cudaGetLastError();
}

// open_bonds_per_particle (kmc.cpp:20-40) as exact sums: out[0] += #B on
// valid sites, out[1] += sum over those B of A-occupied neighbours.  One
// thread per 32-bit word; the 12 neighbour directions are aligned to the
// word with funnel shifts of the three adjacent words of each neighbour row.
__device__ __forceinline__ uint32_t kmc_row_word(const uint32_t* w, int L, int y, int z, int wi) {
    const int Lm = L - 1, wpr = L >> 5;
    return w[(size_t((z + L) & Lm) * L + size_t((y + L) & Lm)) * wpr + size_t((wi + wpr) & (wpr - 1))];
}

// bits of row (y, z) at x + dx for the 32 x of word wi
__device__ __forceinline__ uint32_t kmc_shifted(const uint32_t* w, int L, int y, int z, int wi, int dx) {
    if (dx == 0) return kmc_row_word(w, L, y, z, wi);
    if (dx > 0) return __funnelshift_r(kmc_row_word(w, L, y, z, wi), kmc_row_word(w, L, y, z, wi + 1), 1);
    return __funnelshift_l(kmc_row_word(w, L, y, z, wi - 1), kmc_row_word(w, L, y, z, wi), 1);
}

__global__ void kmc_open_bonds_kernel(const uint32_t* __restrict__ w, int L, unsigned long long* out2) {
    const size_t nwords = size_t(L) * L * L / 32;
    const int wpr = L >> 5;
    unsigned long long np = 0, no = 0;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nwords; k += size_t(gridDim.x) * blockDim.x) {
        const int wi = int(k % size_t(wpr));
        const size_t row = k / size_t(wpr);
        const int y = int(row % size_t(L)), z = int(row / size_t(L));
        const uint32_t valid = ((y ^ z) & 1) ? 0xAAAAAAAAu : 0x55555555u;
        const uint32_t b = w[k] & valid;
        if (!b) continue;
        np += __popc(b);
        uint32_t open = 0;
#pragma unroll
        for (int d = 0; d < 12; ++d) {
            const uint32_t nbits = kmc_shifted(w, L, y + c_fcc[d][1], z + c_fcc[d][2], wi, c_fcc[d][0]);
            open += __popc(b & ~nbits);
        }
        no += open;
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

cudaError_t kmc_launch_open_bonds(const uint32_t* w, int L, unsigned long long* out2, cudaStream_t st) {
    const size_t nwords = size_t(L) * L * L / 32;
    const int blocks = int(std::min<size_t>((nwords + 255) / 256, 148 * 16));
    kmc_open_bonds_kernel<<<blocks, 256, 0, st>>>(w, L, out2);
    return cudaGetLastError();
}

// count_b (lattice.cpp:97-101): popcount of every word.
__global__ void kmc_count_b_kernel(const uint32_t* __restrict__ w, size_t nwords, unsigned long long* out) {
    unsigned long long n = 0;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nwords; k += size_t(gridDim.x) * blockDim.x)
        n += __popc(w[k]);
    for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xFFFFFFFFu, n, o);
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(out, n);
}

cudaError_t kmc_launch_count_b(const uint32_t* w, int L, unsigned long long* out, cudaStream_t st) {
    const size_t nwords = size_t(L) * L * L / 32;
    const int blocks = int(std::min<size_t>((nwords + 255) / 256, 148 * 16));
    kmc_count_b_kernel<<<blocks, 256, 0, st>>>(w, nwords, out);
    return cudaGetLastError();
}

}  // namespace lfg

// kmc_kernels.cuh -- launchers for the 3-D fcc binary-alloy KMC kernels.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace lfg {

struct KmcPhaseArgs {
    uint32_t* w;                   // occupancy bits, sc layout [L][L][L/32] (z, y, x-words)
    unsigned long long* counters;  // [1] exchanges
    int32_t L, bk;                 // lattice edge, device block edge
    int32_t rounds;                // single-hit rounds per block activation (kKmcRounds / sub)
    uint64_t seed, sweep;
    int32_t phase;                 // 0..7 position in the sweep's block-set order
    int32_t both;                  // ActiveMode::both
    uint32_t thr_lo[13];           // low 32 bits of ceil(exp(-d eps) 2^32), d = 0..12
    uint32_t thr_hi[13];           // bit 32 (threshold == 2^32)
    int32_t zmask;                 // buffer plane slot = global z & zmask (L-1: whole lattice)
    int32_t bz0, nbz;              // block z-rows [bz0, bz0 + nbz) of the shifted frame (slabs)
    int32_t share;                 // lattices sharing the GPU at once (kernel choice; >= 1)
    const uint32_t* abort_flag;    // slab step-barrier abort flag (see KpzPhaseArgs), or nullptr
    // Debug write-set recording (lfg_kmc_debug_record_writes; 16^3 plans): this
    // phase's [256 rounds][active blocks][8 tiles][2] u32 -- the two sc site
    // indices an exchange writes (kmc.hpp:105-110), 0xFFFFFFFF when the attempt
    // did not exchange -- or nullptr.
    uint32_t* wlog;
};

int kmc_blocks_per_cta(int bk);
size_t kmc_phase_smem_bytes(int bk);
cudaError_t kmc_phase_kernel_attrs();
cudaError_t kmc_launch_phase(const KmcPhaseArgs& a, cudaStream_t st);
// Plane-ranged variants: planes [z0, z0 + nz) (global z, slot z & zmask).
cudaError_t kmc_launch_init_alloy(uint32_t* w, int L, int zmask, int z0, int nz, uint32_t thr_lo, uint32_t thr_hi,
                                  uint64_t seed, cudaStream_t st);
cudaError_t kmc_launch_open_bonds(const uint32_t* w, int L, int zmask, int z0, int nz, unsigned long long* out2,
                                  cudaStream_t st);
cudaError_t kmc_launch_count_b(const uint32_t* w, int L, unsigned long long* out, cudaStream_t st);

}  // namespace lfg

/* lfg_kmc.h -- C ABI of the KMC path of liblfg.so (see lfg.h for conventions).
 *
 * Replaces the reference's binary-alloy API (kmc.hpp, lattice.hpp:104-154):
 * OccupancyLattice + make_random_alloy + kmc_mcs_sequential +
 * open_bonds_per_particle + count_b, with the sequential sweep replaced by
 * the two-layer DT sweep (device blocks of `block`^3 sites in eight block
 * sets, inner single-hit rounds over 4^3 domains).
 */
#ifndef LFG_KMC_H
#define LFG_KMC_H

#include "lfg.h"

#ifdef __cplusplus
extern "C" {
#endif

/* ======================================================================= KMC */
typedef struct lfg_kmc lfg_kmc;

typedef struct lfg_kmc_plan {
    int32_t block; /* device block edge in sc sites (0 = auto) */
    int32_t sub;   /* sub-sweeps per MCS (0 = auto = 1; 1 or 4): 4 gives every block four
                      shorter activations per MCS, each sub-sweep with its own origin and
                      set order -- removes the early-time transient of the frozen block
                      borders; the sweep index of the phase-level calls
                      (lfg_kmc_phase, lfg_kmc_slab_phase, lfg_kmc_sweep_origin) is the
                      sub-sweep index s' = MCS * sub + k */
} lfg_kmc_plan;

/* OccupancyLattice(L) + KmcParams{eps, active_mode}.validate() (kmc.hpp:18-27). */
LFG_API int lfg_kmc_create(lfg_kmc** h, int32_t L, double eps, int32_t both_active, uint64_t seed,
                   const lfg_kmc_plan* plan, int32_t device);
LFG_API int lfg_kmc_destroy(lfg_kmc* h);
LFG_API int lfg_kmc_get_plan(const lfg_kmc* h, lfg_kmc_plan* out);
/* words(): nwords = L^3/64 (lattice.hpp:125-126). */
LFG_API int lfg_kmc_upload(lfg_kmc* h, const uint64_t* words, size_t nwords);
LFG_API int lfg_kmc_download(lfg_kmc* h, uint64_t* words, size_t nwords);
/* make_random_alloy (lattice.cpp:117-132) with the device counter RNG:
 * Bernoulli(c) per valid site, statistically (not bit-) equal to the
 * reference's serial stream. */
LFG_API int lfg_kmc_init_random_alloy(lfg_kmc* h, double c, uint64_t seed);
/* kmc_mcs_sequential (kmc.cpp:5-18) replaced by n_mcs two-layer DT sweeps. */
LFG_API int lfg_kmc_sweep(lfg_kmc* h, int64_t n_mcs, lfg_counters* out);
LFG_API int lfg_kmc_sweep_async(lfg_kmc* h, int64_t n_mcs);
/* Enqueue one device-layer phase (0..7) of sweep `sweep` (profiling / sharded driver). */
LFG_API int lfg_kmc_phase(lfg_kmc* h, uint64_t sweep, int32_t phase);
/* Cumulative counters since create / reset (synchronises); deposits = exchanges. */
LFG_API int lfg_kmc_counters(lfg_kmc* h, lfg_counters* out);
LFG_API int lfg_kmc_reset_counters(lfg_kmc* h);
/* open_bonds_per_particle (kmc.cpp:20-40) as exact sums; LFG_EDOMAIN if no B. */
LFG_API int lfg_kmc_open_bond_sums(lfg_kmc* h, int64_t* particles, int64_t* open_bonds);
LFG_API int lfg_kmc_open_bonds_per_particle(lfg_kmc* h, double* out);
/* open_bonds_per_particle (kmc.cpp:20-40) of a host OccupancyLattice (words(),
 * nwords = ceil(L^3/64), any power-of-two L >= 4) on `device`, no handle:
 * the exact int64 sums; the caller divides (and raises std::domain_error when
 * particles == 0, kmc.cpp:36-38). */
LFG_API int lfg_kmc_open_bond_sums_host(int32_t device, int32_t L, const uint64_t* words, size_t nwords,
                                        int64_t* particles, int64_t* open_bonds);
/* count_b (lattice.cpp:97-101). */
LFG_API int lfg_kmc_count_b(lfg_kmc* h, int64_t* out);
LFG_API int lfg_kmc_set_params(lfg_kmc* h, double eps, int32_t both_active);
LFG_API int lfg_kmc_set_sweep_index(lfg_kmc* h, uint64_t sweep);
LFG_API int lfg_kmc_get_sweep_index(const lfg_kmc* h, uint64_t* sweep);
LFG_API int lfg_kmc_set_seed(lfg_kmc* h, uint64_t seed);
LFG_API int lfg_kmc_set_stream(lfg_kmc* h, void* cuda_stream);
/* Performance hint, no reference counterpart: `lattices` handles (this one included) run
 * sweeps side by side on their own streams (an ensemble).  Phases then pick the kernel
 * that suits the combined block count (lattice states are unaffected). */
LFG_API int lfg_kmc_set_concurrency(lfg_kmc* h, int32_t lattices);
LFG_API int lfg_kmc_synchronize(lfg_kmc* h);
/* Device pointer of the occupancy words ([L][L][L/32] uint32) for interop. */
LFG_API int lfg_kmc_device_words(lfg_kmc* h, void** dev_ptr, size_t* bytes);

/* ------------------------------------------------------ z-slab shards (C5)
 * No reference counterpart: the reference is single-process (SURVEY.md §2,
 * PAPER.md:473-480 describes only an MPI dead-border variant).  One rank holds
 * the planes of its z-slab in a device ring buffer of `plane_capacity` planes
 * (a power of two; == L for a whole lattice); global plane z lives at slot
 * z & (plane_capacity - 1), each plane L*L/32 uint32 words in the
 * OccupancyLattice order.  The RNG is keyed on global block/tile ids of the
 * sweep's shifted frame, so any slab decomposition reproduces the
 * single-lattice trajectory bit for bit.  The host driver
 * (paper_1204_5072_b200/shard.py, ShardedKmc) moves planes between ranks. */
/* A handle without a resident lattice (slab phases, readouts, counters). */
LFG_API int lfg_kmc_create_slab(lfg_kmc** h, int32_t L, double eps, int32_t both_active, uint64_t seed,
                                const lfg_kmc_plan* plan, int32_t device);
/* Sweep draw of the shifted frame: out[11] = ox, oy, oz, block-set order[8]. */
LFG_API int lfg_kmc_sweep_origin(int32_t L, const lfg_kmc_plan* plan, uint64_t seed, uint64_t sweep, int32_t* out);
/* Phase `phase` of sweep `sweep` restricted to block z-rows
 * [block_row_begin, +block_rows) (even-aligned) of the shifted frame; reads
 * planes two beyond the slab, writes one beyond (kmc.hpp:140-141). */
LFG_API int lfg_kmc_slab_phase(lfg_kmc* h, void* planes, int32_t plane_capacity, int32_t block_row_begin,
                               int32_t block_rows, uint64_t sweep, int32_t phase);
/* make_random_alloy on planes [z_begin, +nz) (same sites as lfg_kmc_init_random_alloy). */
LFG_API int lfg_kmc_slab_init_random_alloy(lfg_kmc* h, void* planes, int32_t plane_capacity, int32_t z_begin,
                                           int32_t nz, double c, uint64_t seed);
/* open_bonds_per_particle partial sums over planes [z_begin, +nz) (planes
 * z_begin-1 and z_begin+nz must be current). */
LFG_API int lfg_kmc_slab_open_bond_sums(lfg_kmc* h, const void* planes, int32_t plane_capacity, int32_t z_begin,
                                        int32_t nz, int64_t* particles, int64_t* open_bonds);

/* Abort flag of the slab step barrier (see lfg_kpz_set_abort_flag). */
LFG_API int lfg_kmc_set_abort_flag(lfg_kmc* h, const void* dev_flag);

/* Debug instrumentation for the write-disjointness check (the
 * reference's WriteLog, write_log.hpp:10-60; KMC write hooks kmc.hpp:105-110):
 * while enabled (dev_buf != NULL, >= L^3 device words, 16^3 block plan), every
 * sweep writes, per phase k at offset k * L^3/8 words, [256 rounds][active
 * blocks][8 tiles][2] uint32: the two simple-cubic site indices (z L + y) L + x
 * an exchange writes, or 0xFFFFFFFF twice for an attempt that did not
 * exchange.  Block order within a round = launch order (x fastest). */
LFG_API int lfg_kmc_debug_record_writes(lfg_kmc* h, void* dev_buf, size_t capacity_words);

/* ------------------------------------------------------------ sharded lattice (one process, N GPUs)
 * BASELINE configs[4]: the lattice cut into N z-slabs (slab g on devices[g];
 * NULL: devices 0..N-1; a device may repeat) driven by ONE host thread -- the
 * caller of kmc_mcs_sequential / open_bonds_per_particle (kmc.hpp:128-129) gets
 * the same lattice, bit for bit, as lfg_kmc_create's single-GPU handle.  Per MCS
 * the plane ownership rolls with the DT origin; around each phase the two ghost
 * planes on the active side are refreshed and the one the phase may have
 * modified goes back to its owner (peer copies over NVLink, event-ordered).
 * L/N must be a multiple of 2 * block. */
typedef struct lfg_kmc_sharded lfg_kmc_sharded;
LFG_API int lfg_kmc_create_sharded(lfg_kmc_sharded** h, int32_t L, double eps, int32_t both_active, uint64_t seed,
                                   const lfg_kmc_plan* plan, int32_t n_shards, const int32_t* devices);
LFG_API int lfg_kmc_sharded_destroy(lfg_kmc_sharded* h);
LFG_API int lfg_kmc_sharded_init_random_alloy(lfg_kmc_sharded* h, double c, uint64_t alloy_seed);
LFG_API int lfg_kmc_sharded_upload(lfg_kmc_sharded* h, const uint64_t* words, size_t nwords);
LFG_API int lfg_kmc_sharded_download(lfg_kmc_sharded* h, uint64_t* words, size_t nwords);
LFG_API int lfg_kmc_sharded_sweep(lfg_kmc_sharded* h, int64_t n_mcs, lfg_counters* out);
LFG_API int lfg_kmc_sharded_counters(lfg_kmc_sharded* h, lfg_counters* out);
LFG_API int lfg_kmc_sharded_open_bond_sums(lfg_kmc_sharded* h, int64_t* particles, int64_t* open_bonds);
LFG_API int lfg_kmc_sharded_open_bonds_per_particle(lfg_kmc_sharded* h, double* value);
LFG_API int lfg_kmc_sharded_set_sweep_index(lfg_kmc_sharded* h, uint64_t sweep);
LFG_API int lfg_kmc_sharded_get_sweep_index(const lfg_kmc_sharded* h, uint64_t* sweep);

#ifdef __cplusplus
}
#endif

#endif /* LFG_KMC_H */

// kpz_kernels.cuh -- launchers for the KPZ device kernels (kpz_kernels.cu).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda.h>
#include <cuda_runtime.h>

namespace lfg {

constexpr int kMaxRepPerLaunch = 64;

#ifndef LFG_KPZ_MAXBY
#define LFG_KPZ_MAXBY 256  // largest DT block height: 256 = 8-warp CTAs, two tiles per lane (the default plan stays 128)
#endif

// Passed as a __grid_constant__ kernel parameter: everything block-uniform
// (seeds included) lives in the constant bank -> uniform registers.
struct alignas(64) KpzPhaseArgs {
    // 1024-wide plans: 3-D tensor maps [R][rows][L/32] u32 of the lattice (or
    // strip ring buffer); tm_ld boxes 64 words x (by/2 + 1) rows (staging),
    // tm_st 64 words x by/2 rows (write-back).  tma = 0: per-row bulk copies.
    CUtensorMap tm_ld;
    CUtensorMap tm_st;
    int32_t tma;
    uint32_t* f;                    // spins, replica-major [R][L][L/32]
    unsigned long long* counters;   // [R][2] deposits, detaches (device)
    unsigned long long* skipped;    // [R] attempts skipped by the sub = 4 count law (device)
    int32_t L, bx, by;
    int32_t rounds;                 // single-hit rounds per block activation (kpz_rounds(sub))
    int32_t skip;                   // sub (4 or 8): per-tile Poisson attempt counts; 0: none (sub = 1)
    uint64_t sweep;                 // global sub-sweep index s' = MCS * sub + k
    int32_t phase;                  // 0..3 position in the sweep's block-set order
    uint64_t thrP, thrQ;            // ceil(p 2^32), ceil(q 2^32)
    bool general;                   // false: p == 1, q == 0 fast path
    int32_t rep0;                   // first replica of this launch (set by the launcher)
    int32_t row_mask;               // buffer row slot = global row & row_mask (L-1: whole lattice)
    int32_t brow0, nbrow;           // block rows [brow0, brow0 + nbrow) of the shifted frame (strips)
    uint32_t* wlog;                 // debug: this phase's [rounds][tiles] anchor records, or nullptr
    // Fused peer push (strip shards over NVLink): blocks writing global row
    // push_row_dn / push_row_up also store it into the lower / upper
    // neighbour's ring buffer (same capacity; peer pointer from CUDA IPC).
    // Abort flag of the strip step barrier (device memory, or nullptr): when a
    // neighbour never arrived (peer_wait_kernel timed out and set it), the
    // phase kernels of this handle return without touching the lattice instead
    // of updating it against stale ghost rows.
    const uint32_t* abort_flag;
    uint32_t* peer_dn;
    uint32_t* peer_up;
    int32_t push_row_dn, push_row_up;  // -1: none
    // Chained phases (programmatic dependent launch): each block publishes
    // dflags[rep][block] = depoch when done; a launch with chain_wait set waits,
    // per block, for the previous phase's blocks around it instead of for the
    // whole previous grid (pdl: this launch may overlap the previous one).
    uint32_t* dflags;
    uint32_t depoch;
    int32_t chain_wait;
    int32_t pdl;
    // per replica r of this launch: bits 2r, 2r+1 of dd[r >> 5] = x / y parity
    // of set(phase) ^ set(phase - 1), filled by the launcher from the seeds
    uint64_t dd[kMaxRepPerLaunch / 32];
    uint64_t seeds[kMaxRepPerLaunch];
    // per replica of this launch: ox | oy << 12 | set(phase) << 24 of sub-sweep
    // `sweep` (kpz_sweep_draw on the host: no Philox / permutation divisions per CTA)
    uint32_t swd[kMaxRepPerLaunch];
};

// Device-side step barrier between strip shards (no host synchronisation):
// signal stores `value` (release, system scope) into up to two peer flags;
// wait spins until both local flags reach `value` (acquire) or max_spins
// elapse (then *err = 1).
cudaError_t peer_launch_signal(uint32_t* flag_a, uint32_t* flag_b, uint32_t value, cudaStream_t st);
cudaError_t peer_launch_wait(const uint32_t* flag_a, const uint32_t* flag_b, uint32_t value,
                             unsigned long long max_spins, uint32_t* err, cudaStream_t st);

size_t kpz_phase_smem_bytes(int by);
cudaError_t kpz_phase_kernel_attrs();
cudaError_t kpz_launch_phase(const KpzPhaseArgs& a, const uint64_t* seeds, int replicas, cudaStream_t st);
cudaError_t kpz_launch_init_flat(uint32_t* f, int L, int replicas, cudaStream_t st);
cudaError_t kpz_launch_init_zero_slopes(uint32_t* f, int L, int replicas, cudaStream_t st);
cudaError_t kpz_launch_from_slopes(const uint32_t* X, const uint32_t* Y, int L, uint8_t* f0_scratch,
                                   uint32_t* f, cudaStream_t st);
cudaError_t kpz_launch_to_slopes(const uint32_t* f, int L, uint32_t* X, uint32_t* Y, const uint32_t* Xcmp,
                                 const uint32_t* Ycmp, unsigned long long* mismatch, cudaStream_t st);
int kpz_width_segment_rows(int L);
cudaError_t kpz_launch_width(const uint32_t* f, int L, int32_t* H0, int32_t* P1, int32_t* D, int32_t* seg_len,
                             unsigned long long* out3, cudaStream_t st);
cudaError_t kpz_launch_row0_heights(const uint32_t* row0, int L, int32_t* H0, cudaStream_t st);
cudaError_t kpz_launch_width_partials(const uint32_t* f, int L, int rmask, int row_begin, int row_count, int S,
                                      int32_t* P1, int32_t* D, unsigned long long* sum_p2, cudaStream_t st);
cudaError_t kpz_launch_width_combine(const int32_t* H0, const int32_t* P1, const int32_t* D, const int32_t* seg_len,
                                     int L, int G, unsigned long long* out2, cudaStream_t st);
cudaError_t kpz_launch_fill_rows(uint32_t* f, int L, int rmask, int row_begin, int row_count, int pattern,
                                 cudaStream_t st);
// Row-order W^2 sums of a locally closed spin lattice (kpz_width.cu): global
// rows [row_begin, +row_count) of a ring buffer (slot = row & rmask), heights
// relative to the column-0 height of the row below the piece (0 at global row
// 0).  out3[0] += sum h, out3[1] += sum h^2, out3[2] = net column-0 step of
// the piece (as int64); scratch: kpz_width_scratch_bytes(row_count) bytes.
size_t kpz_width_scratch_bytes(int row_count);
cudaError_t kpz_width_kernel_attrs();  // called by kpz_phase_kernel_attrs
cudaError_t kpz_launch_width_rows(const uint32_t* f, int L, int rmask, int row_begin, int row_count, void* scratch,
                                  unsigned long long* out3, cudaStream_t st);
// Closure of two uploaded slope planes: plaquettes that do not close ->
// *local_bad; row 0 / column 0 sums != 0 -> *global_bad (kpz.cpp:35-47).
cudaError_t kpz_launch_closure_check(const uint32_t* X, const uint32_t* Y, int L, unsigned long long* local_bad,
                                     unsigned long long* global_bad, cudaStream_t st);
cudaError_t kpz_launch_heights(const uint32_t* f, int L, int32_t* H0, int32_t* h, cudaStream_t st);

}  // namespace lfg

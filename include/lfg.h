/* lfg.h -- C ABI of the B200 lattice library (liblfg.so).
 *
 * This is the drop-in boundary for the reference's simulation API (namespace
 * lf, /root/reference/proj/include/lf).  The reference is a C++ library with
 * free functions and no FFI; each entry point below names the reference
 * symbol it replaces (file:line relative to /root/reference/proj).  The C++
 * drop-in wrapper (include/lf_gpu.hpp) re-exposes the reference signatures
 * on top of this ABI and rethrows the reference's exception types.
 *
 * Conventions
 *   - plain pointers and sizes only; lattice words use the reference layout:
 *     SlopeField planes (lattice.hpp:56-97) and OccupancyLattice bits
 *     (lattice.hpp:107-135) as little-endian uint64 words, site index
 *     j*L+i (KPZ) or (z*L+y)*L+x (KMC), bit idx&63 of word idx>>6;
 *   - every function returns an lfg_status; lfg_last_error() gives the
 *     message of the last failure on the calling thread, worded like the
 *     reference's exception text;
 *   - a handle is not thread-safe (one host thread per handle, as
 *     RngStream/lattice ownership in the reference, rng.hpp:38-39); all
 *     device work is ordered on the handle's CUDA stream; calls that return
 *     host data are synchronous.
 */
#ifndef LFG_H
#define LFG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LFG_ABI_VERSION 1

#if defined(__GNUC__)
#define LFG_API __attribute__((visibility("default")))
#else
#define LFG_API
#endif

typedef enum lfg_status {
    LFG_OK = 0,
    LFG_EINVAL = 1,   /* std::invalid_argument  (lattice.cpp:10-16, kpz.hpp:19-26, kmc.hpp:24-26, ...) */
    LFG_ECLOSURE = 2, /* std::runtime_error     (reconstruct_heights closure violation, kpz.cpp:42-44) */
    LFG_EDOMAIN = 3,  /* std::domain_error      (no B particles, kmc.cpp:36-38) */
    LFG_ECUDA = 4,    /* CUDA runtime failure (no reference analogue) */
    LFG_ENCCL = 5,    /* collective/transport failure on the sharded path */
    LFG_ENOMEM = 6    /* device allocation failure */
} lfg_status;

/* Attempt accounting, lf::Counters (counters.hpp:10-19) plus the
 * deposit/detach split needed for <h>(t). */
typedef struct lfg_counters {
    int64_t attempts;
    int64_t successes;
    int64_t deposits;  /* KPZ: depositions; KMC: exchanges */
    int64_t detaches;  /* KPZ: detachments; KMC: 0 */
} lfg_counters;

LFG_API const char* lfg_last_error(void);
LFG_API int lfg_abi_version(void);
/* Number of visible CUDA devices (0 on a host without a GPU). */
LFG_API int lfg_device_count(int* count);

/* ======================================================================= KPZ */
typedef struct lfg_kpz lfg_kpz;

/* Two-layer DTr geometry: device blocks block_x x block_y sites (0 = auto:
 * min(1024, L/2) x min(128, L/2)); powers of two, block_x in [32, 1024],
 * block_y in [16, 256]; inner 16x8 single-hit domains are fixed.
 * sub: sub-sweeps per MCS (0 = auto = 4).  4: every MCS is four sub-sweeps,
 * each with its own random origin and block-set order, and every tile makes a
 * Poisson-distributed number of attempts per activation (mean and variance
 * 128) -- statistically matched to kpz_sweep_sequential (kpz.cpp:5-19) at
 * >= 64 seeds.  8: eight sub-sweeps with Poisson counts of mean
 * and variance 64 (halves the residual <h> bias of 4 at twice the phase
 * launches).  1: the paper's scheme, one origin per MCS and
 * exactly 512 single-hit rounds per activation. */
typedef struct lfg_kpz_plan {
    int32_t block_x;
    int32_t block_y;
    int32_t sub;
} lfg_kpz_plan;

/* SlopeField(L) + KpzParams{p,q}.validate() + the seeding of
 * RngStream::make (rng.cpp:49-69): a Philox4x32-10 key.  The lattice starts
 * all-zero slopes like SlopeField's constructor (lattice.cpp:20-25). */
LFG_API int lfg_kpz_create(lfg_kpz** h, int32_t L, double p, double q, uint64_t seed, const lfg_kpz_plan* plan,
                   int32_t device);
/* `replicas` independent lattices (seed per replica) advanced by one launch. */
LFG_API int lfg_kpz_create_batch(lfg_kpz** h, int32_t L, double p, double q, const uint64_t* seeds, int32_t replicas,
                         const lfg_kpz_plan* plan, int32_t device);
LFG_API int lfg_kpz_destroy(lfg_kpz* h);
LFG_API int lfg_kpz_get_plan(const lfg_kpz* h, lfg_kpz_plan* out);

/* make_flat_slopes (lattice.cpp:71-82), all replicas. */
LFG_API int lfg_kpz_init_flat(lfg_kpz* h);
/* Copy a host SlopeField (words_x()/words_y(), lattice.hpp:81-84) in/out.
 * nwords = L*L/64.  Upload rejects a non-integrable field with LFG_ECLOSURE
 * (the reference's reconstruct_heights error, kpz.cpp:42-44). */
LFG_API int lfg_kpz_upload(lfg_kpz* h, int32_t replica, const uint64_t* x, const uint64_t* y, size_t nwords);
LFG_API int lfg_kpz_download(lfg_kpz* h, int32_t replica, uint64_t* x, uint64_t* y, size_t nwords);
/* Stream-ordered variants (return after enqueueing on the handle's stream;
 * host buffers must be pinned and stay untouched until lfg_kpz_synchronize):
 * several handles on their own streams overlap one lattice's device->host
 * copy with another's host->device copy (full-duplex PCIe).  The closure
 * check of upload_async is deferred: lfg_kpz_upload_check synchronises and
 * returns LFG_ECLOSURE if any upload since the last check was not integrable
 * (the replica's state is then unspecified, unlike lfg_kpz_upload). */
LFG_API int lfg_kpz_upload_async(lfg_kpz* h, int32_t replica, const uint64_t* x, const uint64_t* y, size_t nwords);
LFG_API int lfg_kpz_upload_check(lfg_kpz* h);
LFG_API int lfg_kpz_download_async(lfg_kpz* h, int32_t replica, uint64_t* x, uint64_t* y, size_t nwords);

/* kpz_sweep_sequential (kpz.cpp:5-19) replaced by n_mcs two-layer DTr sweeps.
 * out: NULL or an array of `replicas` counters for this call. */
LFG_API int lfg_kpz_sweep(lfg_kpz* h, int64_t n_mcs, lfg_counters* out);
/* Enqueue n_mcs sweeps without synchronising (counters accumulate on device). */
LFG_API int lfg_kpz_sweep_async(lfg_kpz* h, int64_t n_mcs);
/* Enqueue one device-layer phase (0..3) of sub-sweep `sweep` (the global
 * sub-sweep index s' = MCS * plan.sub + k; profiling / sharded driver). */
LFG_API int lfg_kpz_phase(lfg_kpz* h, uint64_t sweep, int32_t phase);
/* Cumulative counters since create / reset (synchronises). */
LFG_API int lfg_kpz_counters(lfg_kpz* h, int32_t replica, lfg_counters* out);
LFG_API int lfg_kpz_reset_counters(lfg_kpz* h);

/* interface_width(const SlopeField&) (kpz.cpp:62-81): exact int64 sums with
 * h(0,0)=0; W2 = sum2/n - (sum/n)^2 finished on the host exactly as kpz.cpp:78-80. */
LFG_API int lfg_kpz_width_sums(lfg_kpz* h, int32_t replica, int64_t* sum, int64_t* sum2);
LFG_API int lfg_kpz_interface_width(lfg_kpz* h, int32_t replica, double* w2);
/* Stream-ordered W^2 sums: out3[0] = sum h, out3[1] + out3[2] = sum h^2
 * (pinned host int64[3], valid after lfg_kpz_synchronize). */
LFG_API int lfg_kpz_width_sums_async(lfg_kpz* h, int32_t replica, int64_t* out3);
/* Debug instrumentation for the write-disjointness check (the
 * reference's WriteLog, write_log.hpp:10-60): while enabled, every MCS writes
 * one uint32 record per (round, tile) into dev_buf (device memory, >=
 * L*L/512 * rounds * sub words; sub-sweep k, phase f at offset
 * (4k + f) * L*L/2048 * rounds, then [rounds][tiles of the launch], rounds =
 * 68 for sub = 8, 132 for sub = 4, 512 for sub = 1): global tile id (bits 0-19), anchor column
 * in the domain xd (20-23), row yd (24-26), inner set hx (27) / hy (28),
 * accepted (29), skipped round of the tile (30; no attempt).  Single-replica
 * handles, every plan (incl. the 1024-wide TMA path); dev_buf = NULL
 * disables.  Uses the per-phase kernels (no phase chaining). */
LFG_API int lfg_kpz_debug_record_anchors(lfg_kpz* h, void* dev_buf, size_t capacity_words);
/* reconstruct_heights (kpz.cpp:21-49): n = L*L int32, row-major j*L+i. */
LFG_API int lfg_kpz_heights(lfg_kpz* h, int32_t replica, int32_t* heights, size_t n);

LFG_API int lfg_kpz_set_params(lfg_kpz* h, double p, double q);
/* Counter-based RNG state: (seed, next sweep index) -> exact resume. */
LFG_API int lfg_kpz_set_sweep_index(lfg_kpz* h, uint64_t sweep);
LFG_API int lfg_kpz_get_sweep_index(const lfg_kpz* h, uint64_t* sweep);
LFG_API int lfg_kpz_set_seed(lfg_kpz* h, int32_t replica, uint64_t seed);
LFG_API int lfg_kpz_set_stream(lfg_kpz* h, void* cuda_stream);
LFG_API int lfg_kpz_synchronize(lfg_kpz* h);
/* Device pointer of a replica's spin words ([L][L/32] uint32) for zero-copy
 * interop (torch.distributed halo exchange on the sharded path). */
LFG_API int lfg_kpz_device_spins(lfg_kpz* h, int32_t replica, void** dev_ptr, size_t* bytes);

/* ---- readouts of host lattices (no handle) ---------------------------------
 * The reference's free functions on an arbitrary SlopeField, any power-of-two
 * L >= 4, integrable or not, computed on `device` in the reference's own index
 * order (words = SlopeField::words_x()/words_y(), nwords = ceil(L*L/64)):
 *   interface_width(const SlopeField&) (kpz.cpp:62-81): the int64 sums of
 *     heights integrated along row 0, then up every column (no closure check,
 *     as the reference); W2 = sum2/n - (sum/n)^2 on the host (kpz.cpp:78-80);
 *   reconstruct_heights (kpz.cpp:21-49): heights[j*L+i], LFG_ECLOSURE (the
 *     reference's std::runtime_error) when they would be path-dependent. */
LFG_API int lfg_kpz_width_sums_host(int32_t device, int32_t L, const uint64_t* x, const uint64_t* y, size_t nwords,
                                    int64_t* sum, int64_t* sum2);
/* interface_width(const HeightField&) (kpz.cpp:51-60): int64 sums of n heights. */
LFG_API int lfg_heights_width_sums_host(int32_t device, const int32_t* heights, size_t n, int64_t* sum,
                                        int64_t* sum2);
LFG_API int lfg_kpz_heights_host(int32_t device, int32_t L, const uint64_t* x, const uint64_t* y, size_t nwords,
                                 int32_t* heights, size_t n);

/* ---- strip-sharded path (multi-GPU) ----------------------
 * The caller (one process per GPU) owns a device ring buffer of
 * `row_capacity` spin rows (power of two; global row y lives at slot
 * y & (row_capacity-1); each row is L/32 uint32 words) holding its strip
 * plus ghost rows, and moves rows between ranks (NCCL send/recv).  These
 * calls only enqueue on the handle's stream.  A handle from
 * lfg_kpz_create_strip has no resident lattice of its own. */
LFG_API int lfg_kpz_create_strip(lfg_kpz** h, int32_t L, double p, double q, uint64_t seed,
                                 const lfg_kpz_plan* plan, int32_t device);
/* Sweep-level draws of the DTr schedule for sub-sweep s' (= MCS * plan.sub + k):
 * out = {ox, oy, set of phase 0..3}. */
LFG_API int lfg_kpz_sweep_origin(int32_t L, const lfg_kpz_plan* plan, uint64_t seed, uint64_t sweep,
                                 int32_t out[6]);
/* One DT phase of sub-sweep `sweep` (s') restricted to block rows
 * [block_row_begin, +block_row_count) of its shifted frame (begin and count even). */
LFG_API int lfg_kpz_strip_phase(lfg_kpz* h, void* rows, int32_t row_capacity, int32_t block_row_begin,
                                int32_t block_row_count, uint64_t sweep, int32_t phase);
/* Fill global rows [row_begin, +row_count) (mod L): pattern 0 = make_flat_slopes,
 * 1 = all slopes -1 (SlopeField constructor). */
/* lfg_kpz_strip_phase with the ghost-row exchange fused into the write-back:
 * the blocks that write global row push_row_dn (push_row_up) also store it
 * into the ring buffer peer_dn (peer_up) of the lower (upper) neighbour -- a
 * device pointer from lfg_ipc_open_handle, same row_capacity -- over NVLink.
 * NULL / -1 disables a side.  Ordering with the neighbour is the caller's
 * (lfg_peer_signal / lfg_peer_wait). */
LFG_API int lfg_kpz_strip_phase_push(lfg_kpz* h, void* rows, int32_t row_capacity, int32_t block_row_begin,
                                     int32_t block_rows, uint64_t sweep, int32_t phase, void* peer_dn,
                                     int32_t push_row_dn, void* peer_up, int32_t push_row_up);
/* Abort flag of the strip step barrier (device uint32, or NULL to clear):
 * pass the err_flag given to lfg_peer_wait.  Once a neighbour has failed to
 * arrive (the flag is nonzero), this handle's strip phases return without
 * touching the rows -- no update against stale ghost rows; the caller then
 * raises the transport error (the lattice is left as of the last completed
 * phase). */
LFG_API int lfg_kpz_set_abort_flag(lfg_kpz* h, const void* dev_flag);
LFG_API int lfg_kpz_strip_fill(lfg_kpz* h, void* rows, int32_t row_capacity, int32_t row_begin, int32_t row_count,
                               int32_t pattern);
/* W^2 pieces (kpz.cpp:62-81 split by rows): H0 = row-0 heights (int32[L], needs global row 0);
 * per segment of seg_rows rows of [row_begin, +row_count): P1/D int32[nseg][L], P2 += sum p^2 (uint64). */
LFG_API int lfg_kpz_strip_row0_heights(lfg_kpz* h, const void* rows, int32_t row_capacity, void* H0);
LFG_API int lfg_kpz_strip_width_partials(lfg_kpz* h, const void* rows, int32_t row_capacity, int32_t row_begin,
                                         int32_t row_count, int32_t seg_rows, void* P1, void* D, void* P2);
/* Row-order W^2 pieces (the fast readout; the strip must be a piece of a
 * lattice reached from an integrable state, which every device state is):
 * for global rows [row_begin, +row_count) (no wrap past L-1) with heights
 * relative to B = the column-0 height of the row below the piece (B = 0 for
 * row_begin = 0, which anchors h(0,0) = 0 as kpz.cpp:66 does):
 * out3[0] = sum h_rel, out3[1] = sum h_rel^2, out3[2] = net column-0 step D.
 * The ghost row below the piece must be current.  The caller walks the pieces
 * in global row order: sum h += s1 + n L B, sum h^2 += s2 + 2 B s1 + n L B^2,
 * B += D (n = row_count).  Synchronous. */
LFG_API int lfg_kpz_strip_width_rows(lfg_kpz* h, const void* rows, int32_t row_capacity, int32_t row_begin,
                                     int32_t row_count, int64_t out3[3]);
/* Combine segments given in global row order (seg_len int32[nseg], device):
 * sum h and sum h^2 - sum p^2 (add the all-reduced P2 to get sum h^2). */
LFG_API int lfg_kpz_width_combine(lfg_kpz* h, const void* H0, const void* P1, const void* D, const void* seg_len,
                                  int32_t nseg, int64_t* sum, int64_t* sum2_without_p2);

/* ------------------------------------------------------------ sharded lattice (one process, N GPUs)
 * BASELINE configs[2]: the lattice split into N y-strips, strip g on
 * devices[g] (NULL: devices 0..N-1; a device may repeat), driven by ONE host
 * thread: the caller of the reference's kpz_sweep_sequential / interface_width
 * (kpz.hpp:119-120) gets the same lattice, bit for bit, as lfg_kpz_create's
 * single-GPU handle.  Per sub-sweep the row ownership rolls
 * with the DTr origin and the ghost rows are peer copies (NVLink); per phase the
 * ghost row a neighbour needs is stored into its ring by the phase kernel's
 * write-back and neighbouring strips are ordered by CUDA events.  L/N must be a
 * multiple of 2 * block_y.  Error codes as the single-GPU calls. */
typedef struct lfg_kpz_sharded lfg_kpz_sharded;
LFG_API int lfg_kpz_create_sharded(lfg_kpz_sharded** h, int32_t L, double p, double q, uint64_t seed,
                                   const lfg_kpz_plan* plan, int32_t n_shards, const int32_t* devices);
LFG_API int lfg_kpz_sharded_destroy(lfg_kpz_sharded* h);
/* make_flat_slopes (lattice.cpp:71-82) / a host SlopeField (closure-checked). */
LFG_API int lfg_kpz_sharded_init_flat(lfg_kpz_sharded* h);
LFG_API int lfg_kpz_sharded_upload(lfg_kpz_sharded* h, const uint64_t* x, const uint64_t* y, size_t nwords);
LFG_API int lfg_kpz_sharded_download(lfg_kpz_sharded* h, uint64_t* x, uint64_t* y, size_t nwords);
/* n_mcs DTr MCS over all strips; out: NULL or this call's counters. */
LFG_API int lfg_kpz_sharded_sweep(lfg_kpz_sharded* h, int64_t n_mcs, lfg_counters* out);
LFG_API int lfg_kpz_sharded_counters(lfg_kpz_sharded* h, lfg_counters* out);
/* interface_width (kpz.cpp:62-81): exact int64 sums assembled from the strips. */
LFG_API int lfg_kpz_sharded_width_sums(lfg_kpz_sharded* h, int64_t* sum, int64_t* sum2);
LFG_API int lfg_kpz_sharded_interface_width(lfg_kpz_sharded* h, double* w2);
/* Next MCS index (set before init_flat / upload). */
LFG_API int lfg_kpz_sharded_set_sweep_index(lfg_kpz_sharded* h, uint64_t sweep);
LFG_API int lfg_kpz_sharded_get_sweep_index(const lfg_kpz_sharded* h, uint64_t* sweep);

/* ------------------------------------------------------------ peer memory
 * Single-node shard exchange without a collective library (one process per
 * GPU; NVLink peer access through CUDA IPC).  Handles are 64 opaque bytes. */
/* Handle of the allocation containing dev_ptr and dev_ptr's byte offset in it
 * (pointers from a caching allocator may be interior); the opener adds the offset
 * to the base that lfg_ipc_open_handle returns. */
LFG_API int lfg_ipc_get_handle(const void* dev_ptr, void* handle64, uint64_t* offset);
LFG_API int lfg_ipc_open_handle(const void* handle64, int32_t device, void** dev_ptr);
LFG_API int lfg_ipc_close(void* dev_ptr, int32_t device);
/* Device-side step barrier on `stream`: signal stores `value` (release, system
 * scope) into flag_a / flag_b (either may be NULL; typically a neighbour's flag
 * through its IPC pointer); wait blocks the stream until both local flags have
 * reached `value` (wrap-around compare), giving up after max_spins polls with
 * *err_flag = 1 (device memory, may be NULL) instead of hanging. */
LFG_API int lfg_peer_signal(void* stream, void* flag_a, void* flag_b, uint32_t value, int32_t device);
LFG_API int lfg_peer_wait(void* stream, const void* flag_a, const void* flag_b, uint32_t value, uint64_t max_spins,
                          void* err_flag, int32_t device);
/* cudaMemcpyAsync(cudaMemcpyDefault) on `stream` (peer copies between rings). */
LFG_API int lfg_copy_async(void* dst, const void* src, size_t bytes, void* stream, int32_t device);

#ifdef __cplusplus
}
#endif

#endif /* LFG_H */

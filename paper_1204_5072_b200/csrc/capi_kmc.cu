// capi_kmc.cu -- C ABI for the KMC path (include/lfg_kmc.h), host orchestration.
//
// One handle = one L^3 occupancy lattice resident in HBM in the reference's
// word layout, plus the counter-based RNG state (seed, next sweep index) and
// the Metropolis threshold table.  A sweep is eight launches of the DT phase
// kernel, one per block set, in the order drawn for that sweep.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <string>

#include "../../include/lfg_kmc.h"
#include "capi_common.cuh"
#include "kmc_kernels.cuh"
#include "lfg_common.cuh"

using namespace lfg;

struct lfg_kmc {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int32_t L = 0, bk = 0, sub = 1;  // sub: sub-sweeps per MCS (plan)
    double eps = 1.5;
    int both = 0;
    uint64_t seed = 0, sweep = 0;
    uint32_t* w = nullptr;              // [L][L][L/32]
    unsigned long long* dcnt = nullptr; // [1] exchanges
    unsigned long long* dtmp = nullptr; // [2] reductions
    unsigned long long* hpin = nullptr; // pinned [2]
    int64_t attempts = 0;
    const uint32_t* abort_flag = nullptr;  // slab step-barrier abort flag (lfg_kmc_set_abort_flag)
    uint32_t* wlog = nullptr;           // debug write-set records (lfg_kmc_debug_record_writes) or nullptr
    uint64_t thr[13] = {};
    bool slab_only = false;             // created by lfg_kmc_create_slab: no resident lattice
    int32_t share = 1;                  // lfg_kmc_set_concurrency

    size_t nwords() const { return size_t(L) * L * L / 32; }
};

namespace {

void check_handle(const lfg_kmc* h) {
    if (!h) throw Error(LFG_EINVAL, "null lfg_kmc handle");
}

void check_resident(const lfg_kmc* h) {
    check_handle(h);
    if (h->slab_only) throw Error(LFG_EINVAL, "handle was created with lfg_kmc_create_slab (no resident lattice)");
}

void check_ring(const lfg_kmc* h, const void* planes, int32_t cap) {
    if (!planes) throw Error(LFG_EINVAL, "null plane buffer");
    if (cap < 1 || !is_pow2(cap) || cap > h->L)
        throw Error(LFG_EINVAL, "plane_capacity must be a power of two <= L, got " + std::to_string(cap));
}

void validate_eps(double eps) {  // KmcParams::validate (kmc.hpp:24-26)
    if (!(eps >= 0.0)) throw Error(LFG_EINVAL, "KmcParams: eps must be >= 0");
}

// metropolis_prob (kmc.hpp:33-39): w(d) = exp(-d eps) for d = n_i - n_f > 0,
// evaluated with the host's std::exp exactly as the reference does; the
// device compares u < ceil(w 2^32), equivalent to u * 2^-32 < w.
void build_thresholds(lfg_kmc* h) {
    h->thr[0] = uint64_t{1} << 32;
    for (int d = 1; d <= 12; ++d) h->thr[d] = threshold32(1.0 * std::exp(-d * h->eps));
}

void sync(lfg_kmc* h) { cuda_check(cudaStreamSynchronize(h->stream), "kernel execution"); }

KmcPhaseArgs base_args(const lfg_kmc* h) {
    KmcPhaseArgs a{};
    a.w = h->w;
    a.counters = h->dcnt;
    a.L = h->L;
    a.bk = h->bk;
    a.rounds = kKmcRounds / h->sub;
    a.seed = h->seed;
    a.both = h->both;
    for (int d = 0; d <= 12; ++d) {
        a.thr_lo[d] = uint32_t(h->thr[d]);
        a.thr_hi[d] = uint32_t(h->thr[d] >> 32);
    }
    a.zmask = h->L - 1;
    a.bz0 = 0;
    a.nbz = h->L / h->bk;
    a.share = h->share;
    a.abort_flag = h->abort_flag;
    return a;
}

void enqueue(lfg_kmc* h, int64_t n) {
    KmcPhaseArgs a = base_args(h);
    for (int64_t s = 0; s < n * h->sub; ++s) {
        a.sweep = h->sweep * uint64_t(h->sub) + uint64_t(s);  // global sub-sweep index
        for (int k = 0; k < 8; ++k) {
            a.phase = k;
            // one MCS of records: phase k of sub-sweep j at (8 j + k) * (L^3/2 attempts / (8 sub)) * 2 words
            a.wlog = h->wlog ? h->wlog + size_t((s % h->sub) * 8 + k) * (size_t(h->L) * h->L * h->L / 8 / h->sub)
                             : nullptr;
            cuda_check(kmc_launch_phase(a, h->stream), "kmc_dt_phase launch");
        }
    }
    h->sweep += uint64_t(n);
    h->attempts += int64_t(h->L) * h->L * h->L / 2 * n;
}

unsigned long long read_u64(lfg_kmc* h, const unsigned long long* d) {
    cuda_check(cudaMemcpyAsync(h->hpin, d, 8, cudaMemcpyDeviceToHost, h->stream), "readback");
    sync(h);
    return h->hpin[0];
}

}  // namespace

extern "C" {

}  // extern "C"

namespace {

int32_t validate_create(int32_t L, double eps, const lfg_kmc_plan* plan) {
    if (L < 4 || !is_pow2(L))  // check_size (lattice.cpp:10-16)
        throw Error(LFG_EINVAL, "OccupancyLattice: size must be a power of two >= 4, got " + std::to_string(L));
    if (L < 32)
        throw Error(LFG_EINVAL, "DtPlan: the KMC two-layer DT needs L >= 32 (two 16-site blocks per axis), got " +
                                    std::to_string(L));
    validate_eps(eps);
    const int32_t bk = plan && plan->block ? plan->block : 16;  // 16^3 blocks: SURVEY §7.1 (+0.03 %, z=+0.3)
    if (!(bk == 16 || bk == 32) || L % (2 * bk))
        throw Error(LFG_EINVAL, "DtPlan: block must be 16 or 32 with L % (2*block) == 0, got " + std::to_string(bk));
    if (plan && plan->sub && plan->sub != 1 && plan->sub != 4)
        throw Error(LFG_EINVAL, "DtPlan: sub (sub-sweeps per MCS) must be 1 or 4, got " + std::to_string(plan->sub));
    return bk;
}

lfg_kmc* create_handle(int32_t L, double eps, int32_t both_active, uint64_t seed, const lfg_kmc_plan* plan,
                       int32_t device, bool slab_only) {
    const int32_t bk = validate_create(L, eps, plan);
    auto* h = new lfg_kmc();
    try {
        h->L = L;
        h->bk = bk;
        h->sub = plan && plan->sub ? plan->sub : 1;
        h->eps = eps;
        h->both = both_active ? 1 : 0;
        h->seed = seed;
        h->device = device;
        h->slab_only = slab_only;
        build_thresholds(h);
        DeviceGuard g(device);
        cuda_check(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "cudaStreamCreate");
        h->own_stream = true;
        cuda_check(kmc_phase_kernel_attrs(), "kernel attributes");
        if (!slab_only) h->w = dmalloc<uint32_t>(h->nwords(), "alloc lattice");
        h->dcnt = dmalloc<unsigned long long>(1, "alloc counters");
        h->dtmp = dmalloc<unsigned long long>(2, "alloc scratch");
        cuda_check(cudaMallocHost(&h->hpin, 16), "alloc pinned");
        if (!slab_only)  // all A (lattice.cpp:84-88)
            cuda_check(cudaMemsetAsync(h->w, 0, h->nwords() * 4, h->stream), "memset");
        cuda_check(cudaMemsetAsync(h->dcnt, 0, 8, h->stream), "memset");
        sync(h);
    } catch (...) {
        lfg_kmc_destroy(h);
        throw;
    }
    return h;
}

}  // namespace

extern "C" {

int lfg_kmc_create(lfg_kmc** out, int32_t L, double eps, int32_t both_active, uint64_t seed,
                   const lfg_kmc_plan* plan, int32_t device) {
    return guarded([&] {
        if (!out) throw Error(LFG_EINVAL, "null output handle");
        *out = nullptr;
        *out = create_handle(L, eps, both_active, seed, plan, device, false);
    });
}

int lfg_kmc_create_slab(lfg_kmc** out, int32_t L, double eps, int32_t both_active, uint64_t seed,
                        const lfg_kmc_plan* plan, int32_t device) {
    return guarded([&] {
        if (!out) throw Error(LFG_EINVAL, "null output handle");
        *out = nullptr;
        *out = create_handle(L, eps, both_active, seed, plan, device, true);
    });
}

int lfg_kmc_sweep_origin(int32_t L, const lfg_kmc_plan* plan, uint64_t seed, uint64_t sweep, int32_t* out) {
    return guarded([&] {
        if (!out) throw Error(LFG_EINVAL, "null output");
        const int32_t bk = validate_create(L, 0.0, plan);
        const KmcSweep sw = kmc_sweep_draw(bk, seed, sweep);
        out[0] = sw.ox;
        out[1] = sw.oy;
        out[2] = sw.oz;
        for (int k = 0; k < 8; ++k) out[3 + k] = sw.set(k);
    });
}

int lfg_kmc_slab_phase(lfg_kmc* h, void* planes, int32_t cap, int32_t bz0, int32_t nbz, uint64_t sweep,
                       int32_t phase) {
    return guarded([&] {
        check_handle(h);
        check_ring(h, planes, cap);
        if (phase < 0 || phase > 7) throw Error(LFG_EINVAL, "phase must be in 0..7");
        if (bz0 < 0 || (bz0 & 1) || nbz < 2 || (nbz & 1) || bz0 + nbz > h->L / h->bk)
            throw Error(LFG_EINVAL, "block-row range must be even-aligned inside [0, L/block)");
        if (cap < h->L && cap < nbz * h->bk + 4)
            throw Error(LFG_EINVAL, "plane_capacity too small for the slab and its ghost planes");
        DeviceGuard g(h->device);
        KmcPhaseArgs a = base_args(h);
        a.w = static_cast<uint32_t*>(planes);
        a.zmask = cap - 1;
        a.bz0 = bz0;
        a.nbz = nbz;
        a.sweep = sweep;
        a.phase = phase;
        cuda_check(kmc_launch_phase(a, h->stream), "kmc_dt_phase launch");
        const int64_t hh = h->L / h->bk / 2;
        h->attempts += hh * hh * (nbz / 2) * int64_t(h->bk) * h->bk * h->bk / 2 / h->sub;
    });
}

int lfg_kmc_slab_init_random_alloy(lfg_kmc* h, void* planes, int32_t cap, int32_t z0, int32_t nz, double c,
                                   uint64_t seed) {
    return guarded([&] {
        check_handle(h);
        check_ring(h, planes, cap);
        if (!(c >= 0.0 && c <= 1.0))  // lattice.cpp:118-120
            throw Error(LFG_EINVAL, "make_random_alloy: concentration must be in [0,1]");
        if (nz < 0 || nz > cap) throw Error(LFG_EINVAL, "plane count out of range");
        const uint64_t thr = uint64_t(std::llround(c * 4294967296.0));
        DeviceGuard g(h->device);
        cuda_check(kmc_launch_init_alloy(static_cast<uint32_t*>(planes), h->L, cap - 1, ((z0 % h->L) + h->L) % h->L,
                                         nz, uint32_t(thr), uint32_t(thr >> 32), seed, h->stream),
                   "init");
    });
}

int lfg_kmc_slab_open_bond_sums(lfg_kmc* h, const void* planes, int32_t cap, int32_t z0, int32_t nz,
                                int64_t* particles, int64_t* open_bonds) {
    return guarded([&] {
        check_handle(h);
        check_ring(h, planes, cap);
        if (nz < 0 || nz > cap) throw Error(LFG_EINVAL, "plane count out of range");
        DeviceGuard g(h->device);
        cuda_check(cudaMemsetAsync(h->dtmp, 0, 16, h->stream), "memset");
        cuda_check(kmc_launch_open_bonds(static_cast<const uint32_t*>(planes), h->L, cap - 1,
                                         ((z0 % h->L) + h->L) % h->L, nz, h->dtmp, h->stream),
                   "open bonds");
        cuda_check(cudaMemcpyAsync(h->hpin, h->dtmp, 16, cudaMemcpyDeviceToHost, h->stream), "readback");
        sync(h);
        *particles = int64_t(h->hpin[0]);
        *open_bonds = int64_t(h->hpin[1]);
    });
}

int lfg_kmc_destroy(lfg_kmc* h) {
    if (!h) return LFG_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(h->device);
    if (h->stream) cudaStreamSynchronize(h->stream);
    dfree(h->w);
    dfree(h->dcnt);
    dfree(h->dtmp);
    if (h->hpin) cudaFreeHost(h->hpin);
    if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
    if (prev >= 0) cudaSetDevice(prev);
    delete h;
    return LFG_OK;
}

int lfg_kmc_get_plan(const lfg_kmc* h, lfg_kmc_plan* out) {
    return guarded([&] {
        check_handle(h);
        out->block = h->bk;
        out->sub = h->sub;
    });
}

int lfg_kmc_upload(lfg_kmc* h, const uint64_t* words, size_t nwords) {
    return guarded([&] {
        check_resident(h);
        const size_t need = size_t(h->L) * h->L * h->L / 64;
        if (nwords != need || !words) throw Error(LFG_EINVAL, "upload: expected " + std::to_string(need) + " words");
        DeviceGuard g(h->device);
        cuda_check(cudaMemcpyAsync(h->w, words, need * 8, cudaMemcpyHostToDevice, h->stream), "upload");
        sync(h);
    });
}

int lfg_kmc_download(lfg_kmc* h, uint64_t* words, size_t nwords) {
    return guarded([&] {
        check_resident(h);
        const size_t need = size_t(h->L) * h->L * h->L / 64;
        if (nwords != need || !words) throw Error(LFG_EINVAL, "download: expected " + std::to_string(need) + " words");
        DeviceGuard g(h->device);
        cuda_check(cudaMemcpyAsync(words, h->w, need * 8, cudaMemcpyDeviceToHost, h->stream), "download");
        sync(h);
    });
}

int lfg_kmc_init_random_alloy(lfg_kmc* h, double c, uint64_t seed) {
    return guarded([&] {
        check_resident(h);
        if (!(c >= 0.0 && c <= 1.0))  // lattice.cpp:118-120
            throw Error(LFG_EINVAL, "make_random_alloy: concentration must be in [0,1]");
        const uint64_t thr = uint64_t(std::llround(c * 4294967296.0));
        DeviceGuard g(h->device);
        cuda_check(kmc_launch_init_alloy(h->w, h->L, h->L - 1, 0, h->L, uint32_t(thr), uint32_t(thr >> 32), seed,
                                         h->stream),
                   "init");
        sync(h);
    });
}

int lfg_kmc_sweep(lfg_kmc* h, int64_t n_mcs, lfg_counters* out) {
    return guarded([&] {
        check_resident(h);
        if (n_mcs < 0) throw Error(LFG_EINVAL, "sweep: n_mcs must be >= 0");
        DeviceGuard g(h->device);
        const unsigned long long before = read_u64(h, h->dcnt);
        enqueue(h, n_mcs);
        const unsigned long long after = read_u64(h, h->dcnt);
        if (out) {
            out->attempts = int64_t(h->L) * h->L * h->L / 2 * n_mcs;
            out->successes = int64_t(after - before);
            out->deposits = out->successes;
            out->detaches = 0;
        }
    });
}

int lfg_kmc_sweep_async(lfg_kmc* h, int64_t n_mcs) {
    return guarded([&] {
        check_resident(h);
        if (n_mcs < 0) throw Error(LFG_EINVAL, "sweep: n_mcs must be >= 0");
        DeviceGuard g(h->device);
        enqueue(h, n_mcs);
    });
}

int lfg_kmc_phase(lfg_kmc* h, uint64_t sweep, int32_t phase) {
    return guarded([&] {
        check_resident(h);
        if (phase < 0 || phase > 7) throw Error(LFG_EINVAL, "phase must be in 0..7");
        DeviceGuard g(h->device);
        KmcPhaseArgs a = base_args(h);
        a.sweep = sweep;
        a.phase = phase;
        cuda_check(kmc_launch_phase(a, h->stream), "kmc_dt_phase launch");
        h->attempts += int64_t(h->L) * h->L * h->L / 16 / h->sub;
    });
}

int lfg_kmc_counters(lfg_kmc* h, lfg_counters* out) {
    return guarded([&] {
        check_handle(h);
        DeviceGuard g(h->device);
        const unsigned long long n = read_u64(h, h->dcnt);
        out->attempts = h->attempts;
        out->successes = int64_t(n);
        out->deposits = int64_t(n);
        out->detaches = 0;
    });
}

int lfg_kmc_reset_counters(lfg_kmc* h) {
    return guarded([&] {
        check_handle(h);
        DeviceGuard g(h->device);
        cuda_check(cudaMemsetAsync(h->dcnt, 0, 8, h->stream), "memset");
        sync(h);
        h->attempts = 0;
    });
}

int lfg_kmc_open_bond_sums(lfg_kmc* h, int64_t* particles, int64_t* open_bonds) {
    return guarded([&] {
        check_resident(h);
        DeviceGuard g(h->device);
        cuda_check(cudaMemsetAsync(h->dtmp, 0, 16, h->stream), "memset");
        cuda_check(kmc_launch_open_bonds(h->w, h->L, h->L - 1, 0, h->L, h->dtmp, h->stream), "open bonds");
        cuda_check(cudaMemcpyAsync(h->hpin, h->dtmp, 16, cudaMemcpyDeviceToHost, h->stream), "readback");
        sync(h);
        *particles = int64_t(h->hpin[0]);
        *open_bonds = int64_t(h->hpin[1]);
    });
}

int lfg_kmc_open_bonds_per_particle(lfg_kmc* h, double* out) {
    int64_t np = 0, no = 0;
    const int rc = lfg_kmc_open_bond_sums(h, &np, &no);
    if (rc != LFG_OK) return rc;
    if (np == 0) {  // kmc.cpp:36-38
        set_error("open_bonds_per_particle: no B particles in lattice");
        return LFG_EDOMAIN;
    }
    *out = double(no) / double(np);
    return LFG_OK;
}

int lfg_kmc_count_b(lfg_kmc* h, int64_t* out) {
    return guarded([&] {
        check_resident(h);
        DeviceGuard g(h->device);
        cuda_check(cudaMemsetAsync(h->dtmp, 0, 8, h->stream), "memset");
        cuda_check(kmc_launch_count_b(h->w, h->L, h->dtmp, h->stream), "count_b");
        *out = int64_t(read_u64(h, h->dtmp));
    });
}

int lfg_kmc_set_params(lfg_kmc* h, double eps, int32_t both_active) {
    return guarded([&] {
        check_handle(h);
        validate_eps(eps);
        h->eps = eps;
        h->both = both_active ? 1 : 0;
        build_thresholds(h);
    });
}

int lfg_kmc_set_sweep_index(lfg_kmc* h, uint64_t sweep) {
    return guarded([&] {
        check_handle(h);
        h->sweep = sweep;
    });
}

int lfg_kmc_get_sweep_index(const lfg_kmc* h, uint64_t* sweep) {
    return guarded([&] {
        check_handle(h);
        *sweep = h->sweep;
    });
}

int lfg_kmc_set_seed(lfg_kmc* h, uint64_t seed) {
    return guarded([&] {
        check_handle(h);
        h->seed = seed;
    });
}

int lfg_kmc_set_stream(lfg_kmc* h, void* stream) {
    return guarded([&] {
        check_handle(h);
        DeviceGuard g(h->device);
        sync(h);
        if (h->own_stream) cudaStreamDestroy(h->stream);
        h->own_stream = false;
        h->stream = static_cast<cudaStream_t>(stream);
    });
}

int lfg_kmc_debug_record_writes(lfg_kmc* h, void* dev_buf, size_t capacity_words) {
    return guarded([&] {
        check_handle(h);
        if (!dev_buf) {
            h->wlog = nullptr;
            return;
        }
        if (h->slab_only) throw Error(LFG_EINVAL, "debug_record_writes: resident lattices only");
        if (h->bk != 16) throw Error(LFG_EINVAL, "debug_record_writes: needs the 16^3 block plan (the default)");
        const size_t need = size_t(h->L) * h->L * h->L;  // L^3/2 attempts x 2 words
        if (capacity_words < need)
            throw Error(LFG_EINVAL, "debug_record_writes: buffer must hold L^3 words (one MCS of records)");
        h->wlog = static_cast<uint32_t*>(dev_buf);
    });
}

int lfg_kmc_set_concurrency(lfg_kmc* h, int32_t lattices) {
    return guarded([&] {
        check_handle(h);
        if (lattices < 1) throw Error(LFG_EINVAL, "concurrency must be >= 1");
        h->share = lattices;
    });
}

int lfg_kmc_synchronize(lfg_kmc* h) {
    return guarded([&] {
        check_handle(h);
        DeviceGuard g(h->device);
        sync(h);
    });
}

int lfg_kmc_device_words(lfg_kmc* h, void** ptr, size_t* bytes) {
    return guarded([&] {
        check_resident(h);
        *ptr = h->w;
        *bytes = h->nwords() * 4;
    });
}

int lfg_kmc_set_abort_flag(lfg_kmc* h, const void* dev_flag) {
    return guarded([&] {
        check_handle(h);
        h->abort_flag = static_cast<const uint32_t*>(dev_flag);
    });
}

}  // extern "C"

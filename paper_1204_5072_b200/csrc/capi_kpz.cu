// capi_kpz.cu -- C ABI for the KPZ path (include/lfg.h), host orchestration.
//
// One handle = `replicas` L x L spin lattices resident in HBM (a single
// allocation, replica-major) plus the counter-based RNG state (seed per
// replica, next sweep index).  A sweep is four launches of the DTr phase
// kernel, one per block set in the order drawn for that sweep; the kernel
// derives origin/permutation from (seed, sweep) itself, so the host only
// enqueues.  Counters accumulate on the device and are read back once per
// lfg_kpz_sweep call.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "capi_common.cuh"
#include "kpz_kernels.cuh"
#include "lfg_common.cuh"

namespace lfg {

thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

}  // namespace lfg

using namespace lfg;

struct lfg_kpz {
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int32_t L = 0, bx = 0, by = 0, R = 1;
    int32_t sub = 4;                        // sub-sweeps per MCS (plan; lfg_common.cuh kpz_rounds)
    double p = 1.0, q = 0.0;
    uint64_t sweep = 0;
    std::vector<uint64_t> seeds;
    uint32_t* f = nullptr;                  // [R][L][L/32]
    uint64_t* dseeds = nullptr;             // [R]
    unsigned long long* dcnt = nullptr;     // [R][2] deposits, detaches, then [R] skipped attempts
    std::vector<unsigned long long> hcnt;   // cumulative host mirror of dcnt (3R)
    std::vector<int64_t> attempts;          // cumulative scheduled attempts per replica (before skips)
    // scratch (lazy)
    uint32_t* sx = nullptr;                 // [L][L/32] slope planes staging
    uint32_t* sy = nullptr;
    uint8_t* f0 = nullptr;                  // [L]
    uint32_t* fnew = nullptr;               // [L][L/32]
    unsigned long long* dmis = nullptr;     // mismatch counter
    int32_t* H0 = nullptr;                  // [L]
    void* wscr = nullptr;                   // W^2 row-pass scratch (kpz_width_scratch_bytes(L))
    int32_t* P1 = nullptr;                  // [G][L]
    int32_t* Dd = nullptr;                  // [G][L]
    int32_t* seglen = nullptr;              // [G]
    unsigned long long* wout = nullptr;     // [3]
    bool strip_only = false;                // created by lfg_kpz_create_strip: no resident lattice
    int32_t* hbuf = nullptr;                // [L][L] heights (small L)
    uint32_t* wlog = nullptr;               // debug anchor records ([4 phases][L^2/4]) or nullptr
    uint32_t* flags = nullptr;              // [R][L/bx][L/by] phase-chaining completion epochs
    uint32_t epoch = 0;
    unsigned long long* hpin = nullptr;     // pinned readback [max(3, 2R)]
    // Global closure of each replica's field (reconstruct_heights, kpz.cpp:35-47):
    // dbad[r] != 0 <=> row/column slope sums are not zero.  Set at create (the
    // all -1 field is not closed), init_flat (closed) and upload; sweeps keep it
    // (the octahedron move preserves every row and column sum).
    unsigned long long* dbad = nullptr;     // [R]
    unsigned long long* dglob = nullptr;    // upload scratch: global-closure violations
    const uint32_t* abort_flag = nullptr;   // strip step-barrier abort flag (lfg_kpz_set_abort_flag)

    size_t words_per_replica() const { return size_t(L) * size_t(L / 32); }
    uint32_t* rep(int r) const { return f + size_t(r) * words_per_replica(); }
};

namespace {

void validate_params(double p, double q) {  // KpzParams::validate (kpz.hpp:19-26)
    if (!(p >= 0.0 && p <= 1.0) || !(q >= 0.0 && q <= 1.0))
        throw Error(LFG_EINVAL, "KpzParams: p and q must lie in [0,1]");
    if (p + q <= 0.0) throw Error(LFG_EINVAL, "KpzParams: p + q must be positive");
}

void validate_size(int32_t L) {  // check_size (lattice.cpp:10-16)
    if (L < 4 || !is_pow2(L))
        throw Error(LFG_EINVAL, "SlopeField: size must be a power of two >= 4, got " + std::to_string(L));
    if (L < 64)
        throw Error(LFG_EINVAL, "DtrPlan: the KPZ two-layer DTr needs L >= 64 (two 32-site tiles per block "
                                "set and axis), got " + std::to_string(L));
}

void resolve_plan(lfg_kpz* h, const lfg_kpz_plan* plan) {
    int32_t bx = plan && plan->block_x ? plan->block_x : std::min<int32_t>(1024, h->L / 2);
    int32_t by = plan && plan->block_y ? plan->block_y : std::min<int32_t>(128, h->L / 2);
    if (bx < 32 || bx > 1024 || bx % 32 || !is_pow2(bx) || h->L % (2 * bx))
        throw Error(LFG_EINVAL, "DtrPlan: block_x must be a power of two in [32, min(1024, L/2)], got " +
                                    std::to_string(bx));
    if (by < 16 || by > LFG_KPZ_MAXBY || by % 16 || !is_pow2(by) || h->L % (2 * by))
        throw Error(LFG_EINVAL, "DtrPlan: block_y must be a power of two in [16, min(" +
                                    std::to_string(LFG_KPZ_MAXBY) + ", L/2)], got " + std::to_string(by));
    const int32_t sub = plan && plan->sub ? plan->sub : 4;
    if (sub != 1 && sub != 4 && sub != 8)
        throw Error(LFG_EINVAL, "DtrPlan: sub (sub-sweeps per MCS) must be 1, 4 or 8, got " + std::to_string(sub));
    h->bx = bx;
    h->by = by;
    h->sub = sub;
}

// Scheduled attempts of one sub-sweep over nbrow block rows (before skips).
int64_t sub_sweep_attempts(const lfg_kpz* h, int64_t nbrow) {
    return nbrow * h->by * int64_t(h->L) / 512 * kpz_rounds(h->sub);
}

// Fields every phase launch of handle h shares.
KpzPhaseArgs base_phase_args(const lfg_kpz* h) {
    KpzPhaseArgs a{};
    a.counters = h->dcnt;
    a.skipped = h->dcnt + 2 * h->R;
    a.L = h->L;
    a.bx = h->bx;
    a.by = h->by;
    a.rounds = kpz_rounds(h->sub);
    a.skip = h->sub == 1 ? 0 : h->sub;
    a.thrP = threshold32(h->p);
    a.thrQ = threshold32(h->q);
    a.general = !(h->p == 1.0 && h->q == 0.0);
    return a;
}

void check_handle(const lfg_kpz* h) {
    if (!h) throw Error(LFG_EINVAL, "null lfg_kpz handle");
}

void check_resident(const lfg_kpz* h) {
    if (h->strip_only) throw Error(LFG_EINVAL, "handle was created with lfg_kpz_create_strip (no resident lattice)");
}

void check_replica(const lfg_kpz* h, int32_t r) {
    check_resident(h);
    if (r < 0 || r >= h->R) throw Error(LFG_EINVAL, "replica index out of range: " + std::to_string(r));
}

void ensure_slope_scratch(lfg_kpz* h) {
    if (!h->sx) h->sx = dmalloc<uint32_t>(h->words_per_replica(), "alloc slope staging");
    if (!h->sy) h->sy = dmalloc<uint32_t>(h->words_per_replica(), "alloc slope staging");
}

void ensure_width_scratch(lfg_kpz* h) {
    if (!h->H0) h->H0 = dmalloc<int32_t>(size_t(h->L), "alloc width scratch");
    if (!h->wout) h->wout = dmalloc<unsigned long long>(3, "alloc width scratch");
    if (!h->wscr) h->wscr = dmalloc<uint8_t>(kpz_width_scratch_bytes(h->L), "alloc width scratch");
}

void sync(lfg_kpz* h) { cuda_check(cudaStreamSynchronize(h->stream), "kernel execution"); }

// interface_width sums of replica r into out3 (device): [0] sum h, [1] sum h^2,
// [2] = 0 (row-order scan, kpz_width.cu; the ABI's out3[1] + out3[2] = sum h^2).
// out3 == nullptr: the handle's own scratch h->wout (allocated here on first use).
void enqueue_width(lfg_kpz* h, int32_t r, unsigned long long* out3) {
    ensure_width_scratch(h);
    if (!out3) out3 = h->wout;
    cuda_check(cudaMemsetAsync(out3, 0, 24, h->stream), "memset");
    cuda_check(kpz_launch_width_rows(h->rep(r), h->L, h->L - 1, 0, h->L, h->wscr, out3, h->stream), "width scan");
    cuda_check(cudaMemsetAsync(out3 + 2, 0, 8, h->stream), "memset");
}

// Chained phase launches (programmatic dependent launch + per-block flags);
// LFG_KPZ_PDL=0 disables.
bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("LFG_KPZ_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

void enqueue_sweeps(lfg_kpz* h, int64_t n) {
    KpzPhaseArgs a = base_phase_args(h);
    a.f = h->f;
    a.row_mask = h->L - 1;
    a.brow0 = 0;
    a.nbrow = h->L / h->by;
    if (!h->flags) {  // phase-chaining completion flags (zeroed: epochs start at 1)
        const size_t nf = size_t(h->R) * size_t(h->L / h->bx) * size_t(h->L / h->by);
        h->flags = dmalloc<uint32_t>(nf, "alloc phase flags");
        cuda_check(cudaMemsetAsync(h->flags, 0, nf * 4, h->stream), "memset");
    }
    for (int64_t s = 0; s < n * h->sub; ++s) {
        a.sweep = h->sweep * uint64_t(h->sub) + uint64_t(s);  // global sub-sweep index
        const bool chain = pdl_enabled() && !h->wlog && h->R <= kMaxRepPerLaunch;
        const uint32_t epoch = chain ? ++h->epoch : 0u;
        for (int k = 0; k < 4; ++k) {
            a.phase = k;
            a.wlog = h->wlog ? h->wlog + (size_t(s % h->sub) * 4 + size_t(k)) * (size_t(h->L) * h->L / 512 / 4) *
                                             size_t(kpz_rounds(h->sub))
                             : nullptr;
            if (chain) {  // phases 1-3 overlap the previous phase's tail (per-block flags)
                a.dflags = h->flags;
                a.depoch = epoch;
                a.chain_wait = k > 0;
                a.pdl = 1;
            }
            cuda_check(kpz_launch_phase(a, h->seeds.data(), h->R, h->stream), "kpz_dtr_phase launch");
        }
    }
    h->sweep += uint64_t(n);
    for (int r = 0; r < h->R; ++r) h->attempts[size_t(r)] += sub_sweep_attempts(h, h->L / h->by) * h->sub * n;
}

void read_counters(lfg_kpz* h) {
    cuda_check(cudaMemcpyAsync(h->hpin, h->dcnt, sizeof(unsigned long long) * 3 * h->R, cudaMemcpyDeviceToHost,
                               h->stream), "counter readback");
    sync(h);
    std::memcpy(h->hcnt.data(), h->hpin, sizeof(unsigned long long) * 3 * h->R);
}

// Attempts actually made by replica r: scheduled minus skipped (sub = 4).
int64_t done_attempts(const lfg_kpz* h, int r) {
    return h->attempts[size_t(r)] - int64_t(h->hcnt[size_t(2 * h->R + r)]);
}

lfg_counters make_counters(int64_t att, unsigned long long dep, unsigned long long det) {
    lfg_counters c;
    c.attempts = att;
    c.deposits = int64_t(dep);
    c.detaches = int64_t(det);
    c.successes = c.deposits + c.detaches;
    return c;
}

}  // namespace

extern "C" {

const char* lfg_last_error(void) { return g_last_error.c_str(); }
int lfg_abi_version(void) { return LFG_ABI_VERSION; }

int lfg_device_count(int* count) {
    return guarded([&] {
        int n = 0;
        const cudaError_t e = cudaGetDeviceCount(&n);
        if (e != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        *count = n;
    });
}

int lfg_kpz_create_batch(lfg_kpz** out, int32_t L, double p, double q, const uint64_t* seeds, int32_t replicas,
                         const lfg_kpz_plan* plan, int32_t device) {
    return guarded([&] {
        if (!out) throw Error(LFG_EINVAL, "null output handle");
        *out = nullptr;
        validate_size(L);
        validate_params(p, q);
        if (replicas < 1 || !seeds) throw Error(LFG_EINVAL, "replicas must be >= 1 with one seed each");
        auto* h = new lfg_kpz();
        try {
            h->L = L;
            h->p = p;
            h->q = q;
            h->R = replicas;
            h->device = device;
            resolve_plan(h, plan);
            h->seeds.assign(seeds, seeds + replicas);
            h->hcnt.assign(size_t(3 * replicas), 0);
            h->attempts.assign(size_t(replicas), 0);
            DeviceGuard g(device);
            cuda_check(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            h->own_stream = true;
            cuda_check(kpz_phase_kernel_attrs(), "kernel attributes");
            h->f = dmalloc<uint32_t>(h->words_per_replica() * size_t(replicas), "alloc lattice");
            h->dseeds = dmalloc<uint64_t>(size_t(replicas), "alloc seeds");
            h->dcnt = dmalloc<unsigned long long>(size_t(3 * replicas), "alloc counters");
            cuda_check(cudaMallocHost(&h->hpin, sizeof(unsigned long long) * std::max(3, 3 * replicas)),
                       "alloc pinned");
            cuda_check(cudaMemcpyAsync(h->dseeds, seeds, sizeof(uint64_t) * replicas, cudaMemcpyHostToDevice,
                                       h->stream), "seed upload");
            cuda_check(cudaMemsetAsync(h->dcnt, 0, sizeof(unsigned long long) * 3 * replicas, h->stream), "memset");
            h->dbad = dmalloc<unsigned long long>(size_t(replicas), "alloc closure flags");
            cuda_check(cudaMemsetAsync(h->dbad, 0x01, sizeof(unsigned long long) * replicas, h->stream), "memset");
            // SlopeField(L) starts with every slope -1 (lattice.cpp:20-25): spins f(i,j) = (i + j) & 1.
            cuda_check(kpz_launch_init_zero_slopes(h->f, L, replicas, h->stream), "init");
            cuda_check(cudaStreamSynchronize(h->stream), "create");
        } catch (...) {
            lfg_kpz_destroy(h);
            throw;
        }
        *out = h;
    });
}

int lfg_kpz_create(lfg_kpz** out, int32_t L, double p, double q, uint64_t seed, const lfg_kpz_plan* plan,
                   int32_t device) {
    return lfg_kpz_create_batch(out, L, p, q, &seed, 1, plan, device);
}

int lfg_kpz_destroy(lfg_kpz* h) {
    if (!h) return LFG_OK;
    {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(h->device);
        if (h->stream) cudaStreamSynchronize(h->stream);
        dfree(h->f);
        dfree(h->dseeds);
        dfree(h->dcnt);
        dfree(h->sx);
        dfree(h->sy);
        dfree(h->f0);
        dfree(h->fnew);
        dfree(h->dmis);
        dfree(h->H0);
        dfree(h->wscr);
        dfree(h->P1);
        dfree(h->Dd);
        dfree(h->wout);
        dfree(h->seglen);
        dfree(h->hbuf);
        dfree(h->flags);
        dfree(h->dbad);
        dfree(h->dglob);
        if (h->hpin) cudaFreeHost(h->hpin);
        if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
        if (prev >= 0) cudaSetDevice(prev);
    }
    delete h;
    return LFG_OK;
}

int lfg_kpz_get_plan(const lfg_kpz* h, lfg_kpz_plan* out) {
    return guarded([&] {
        check_handle(h);
        out->block_x = h->bx;
        out->block_y = h->by;
        out->sub = h->sub;
    });
}

int lfg_kpz_init_flat(lfg_kpz* h) {
    return guarded([&] {
        check_handle(h);
        check_resident(h);
        DeviceGuard g(h->device);
        cuda_check(kpz_launch_init_flat(h->f, h->L, h->R, h->stream), "init_flat");
        cuda_check(cudaMemsetAsync(h->dbad, 0, sizeof(unsigned long long) * h->R, h->stream), "memset");
        sync(h);
    });
}

}  // extern "C"

namespace {

// H2D of the two slope planes + device conversion to spins (h->fnew) + the
// closure checks: a field that is not the slope field of its spin field, or
// has an elementary plaquette that does not close, is counted into h->dmis
// (rejected); nonzero row-0 / column-0 sums go to h->dglob (accepted -- the
// reference sweeps such fields -- but reconstruct_heights refuses them).
void enqueue_upload(lfg_kpz* h, const uint64_t* x, const uint64_t* y) {
    ensure_slope_scratch(h);
    if (!h->f0) h->f0 = dmalloc<uint8_t>(size_t(h->L), "alloc scratch");
    if (!h->fnew) h->fnew = dmalloc<uint32_t>(h->words_per_replica(), "alloc scratch");
    if (!h->dmis) {
        h->dmis = dmalloc<unsigned long long>(1, "alloc scratch");
        cuda_check(cudaMemsetAsync(h->dmis, 0, 8, h->stream), "memset");
    }
    const size_t bytes = size_t(h->L) * h->L / 8;
    cuda_check(cudaMemcpyAsync(h->sx, x, bytes, cudaMemcpyHostToDevice, h->stream), "upload x");
    cuda_check(cudaMemcpyAsync(h->sy, y, bytes, cudaMemcpyHostToDevice, h->stream), "upload y");
    cuda_check(kpz_launch_from_slopes(h->sx, h->sy, h->L, h->f0, h->fnew, h->stream), "slopes->spins");
    cuda_check(kpz_launch_to_slopes(h->fnew, h->L, nullptr, nullptr, h->sx, h->sy, h->dmis, h->stream),
               "closure check");
    if (!h->dglob) h->dglob = dmalloc<unsigned long long>(1, "alloc scratch");
    cuda_check(cudaMemsetAsync(h->dglob, 0, 8, h->stream), "memset");
    cuda_check(kpz_launch_closure_check(h->sx, h->sy, h->L, h->dmis, h->dglob, h->stream), "closure check");
}

// The uploaded field becomes replica r's state: spins and global-closure flag.
void commit_upload(lfg_kpz* h, int32_t r) {
    cuda_check(cudaMemcpyAsync(h->rep(r), h->fnew, h->words_per_replica() * 4, cudaMemcpyDeviceToDevice, h->stream),
               "commit");
    cuda_check(cudaMemcpyAsync(h->dbad + r, h->dglob, 8, cudaMemcpyDeviceToDevice, h->stream), "commit");
}

void check_upload_args(lfg_kpz* h, int32_t replica, const void* x, const void* y, size_t nwords) {
    check_handle(h);
    check_replica(h, replica);
    const size_t need = size_t(h->L) * h->L / 64;
    if (nwords != need || !x || !y)
        throw Error(LFG_EINVAL, "upload: expected " + std::to_string(need) + " words per plane");
}

[[noreturn]] void throw_closure() {
    throw Error(LFG_ECLOSURE, "reconstruct_heights: slope field violates closure; heights would be path-dependent");
}

}  // namespace

extern "C" {

int lfg_kpz_upload(lfg_kpz* h, int32_t replica, const uint64_t* x, const uint64_t* y, size_t nwords) {
    return guarded([&] {
        check_upload_args(h, replica, x, y, nwords);
        DeviceGuard g(h->device);
        if (!h->dmis) h->dmis = dmalloc<unsigned long long>(1, "alloc scratch");
        cuda_check(cudaMemsetAsync(h->dmis, 0, 8, h->stream), "memset");  // (a pending async failure is superseded)
        enqueue_upload(h, x, y);
        cuda_check(cudaMemcpyAsync(h->hpin, h->dmis, 8, cudaMemcpyDeviceToHost, h->stream), "readback");
        sync(h);
        if (h->hpin[0] != 0) throw_closure();  // state unchanged
        commit_upload(h, replica);
        sync(h);
    });
}

int lfg_kpz_upload_async(lfg_kpz* h, int32_t replica, const uint64_t* x, const uint64_t* y, size_t nwords) {
    return guarded([&] {
        check_upload_args(h, replica, x, y, nwords);
        DeviceGuard g(h->device);
        enqueue_upload(h, x, y);  // mismatches accumulate in dmis until lfg_kpz_upload_check
        commit_upload(h, replica);
    });
}

int lfg_kpz_upload_check(lfg_kpz* h) {
    return guarded([&] {
        check_handle(h);
        DeviceGuard g(h->device);
        if (!h->dmis) return;
        cuda_check(cudaMemcpyAsync(h->hpin, h->dmis, 8, cudaMemcpyDeviceToHost, h->stream), "readback");
        sync(h);
        cuda_check(cudaMemsetAsync(h->dmis, 0, 8, h->stream), "memset");
        sync(h);
        if (h->hpin[0] != 0) throw_closure();
    });
}

int lfg_kpz_download(lfg_kpz* h, int32_t replica, uint64_t* x, uint64_t* y, size_t nwords) {
    return guarded([&] {
        check_handle(h);
        check_replica(h, replica);
        const size_t need = size_t(h->L) * h->L / 64;
        if (nwords != need || !x || !y)
            throw Error(LFG_EINVAL, "download: expected " + std::to_string(need) + " words per plane");
        DeviceGuard g(h->device);
        ensure_slope_scratch(h);
        cuda_check(kpz_launch_to_slopes(h->rep(replica), h->L, h->sx, h->sy, nullptr, nullptr, nullptr, h->stream),
                   "spins->slopes");
        cuda_check(cudaMemcpyAsync(x, h->sx, need * 8, cudaMemcpyDeviceToHost, h->stream), "download x");
        cuda_check(cudaMemcpyAsync(y, h->sy, need * 8, cudaMemcpyDeviceToHost, h->stream), "download y");
        sync(h);
    });
}

int lfg_kpz_download_async(lfg_kpz* h, int32_t replica, uint64_t* x, uint64_t* y, size_t nwords) {
    return guarded([&] {
        check_handle(h);
        check_replica(h, replica);
        const size_t need = size_t(h->L) * h->L / 64;
        if (nwords != need || !x || !y)
            throw Error(LFG_EINVAL, "download: expected " + std::to_string(need) + " words per plane");
        DeviceGuard g(h->device);
        ensure_slope_scratch(h);
        cuda_check(kpz_launch_to_slopes(h->rep(replica), h->L, h->sx, h->sy, nullptr, nullptr, nullptr, h->stream),
                   "spins->slopes");
        cuda_check(cudaMemcpyAsync(x, h->sx, need * 8, cudaMemcpyDeviceToHost, h->stream), "download x");
        cuda_check(cudaMemcpyAsync(y, h->sy, need * 8, cudaMemcpyDeviceToHost, h->stream), "download y");
    });
}

int lfg_kpz_sweep(lfg_kpz* h, int64_t n_mcs, lfg_counters* out) {
    return guarded([&] {
        check_handle(h);
        check_resident(h);
        if (n_mcs < 0) throw Error(LFG_EINVAL, "sweep: n_mcs must be >= 0");
        DeviceGuard g(h->device);
        read_counters(h);
        std::vector<unsigned long long> before = h->hcnt;
        std::vector<int64_t> before_att = h->attempts;
        enqueue_sweeps(h, n_mcs);
        read_counters(h);
        if (out)
            for (int r = 0; r < h->R; ++r)
                out[r] = make_counters(h->attempts[size_t(r)] - before_att[size_t(r)] -
                                           int64_t(h->hcnt[size_t(2 * h->R + r)] - before[size_t(2 * h->R + r)]),
                                       h->hcnt[2 * r] - before[2 * r], h->hcnt[2 * r + 1] - before[2 * r + 1]);
    });
}

int lfg_kpz_sweep_async(lfg_kpz* h, int64_t n_mcs) {
    return guarded([&] {
        check_handle(h);
        check_resident(h);
        if (n_mcs < 0) throw Error(LFG_EINVAL, "sweep: n_mcs must be >= 0");
        DeviceGuard g(h->device);
        enqueue_sweeps(h, n_mcs);
    });
}

int lfg_kpz_phase(lfg_kpz* h, uint64_t sweep, int32_t phase) {
    return guarded([&] {
        check_handle(h);
        check_resident(h);
        if (phase < 0 || phase > 3) throw Error(LFG_EINVAL, "phase must be in 0..3");
        DeviceGuard g(h->device);
        KpzPhaseArgs a = base_phase_args(h);
        a.f = h->f;
        a.row_mask = h->L - 1;
        a.brow0 = 0;
        a.nbrow = h->L / h->by;
        a.sweep = sweep;
        a.phase = phase;
        cuda_check(kpz_launch_phase(a, h->seeds.data(), h->R, h->stream), "kpz_dtr_phase launch");
        for (int r = 0; r < h->R; ++r) h->attempts[size_t(r)] += sub_sweep_attempts(h, h->L / h->by) / 4;
    });
}

int lfg_kpz_counters(lfg_kpz* h, int32_t replica, lfg_counters* out) {
    return guarded([&] {
        check_handle(h);
        if (replica < 0 || replica >= h->R) throw Error(LFG_EINVAL, "replica index out of range");
        DeviceGuard g(h->device);
        read_counters(h);
        *out = make_counters(done_attempts(h, replica), h->hcnt[2 * replica], h->hcnt[2 * replica + 1]);
    });
}

int lfg_kpz_reset_counters(lfg_kpz* h) {
    return guarded([&] {
        check_handle(h);
        DeviceGuard g(h->device);
        cuda_check(cudaMemsetAsync(h->dcnt, 0, sizeof(unsigned long long) * 3 * h->R, h->stream), "memset");
        sync(h);
        std::fill(h->hcnt.begin(), h->hcnt.end(), 0ull);
        std::fill(h->attempts.begin(), h->attempts.end(), 0ll);
    });
}

int lfg_kpz_width_sums(lfg_kpz* h, int32_t replica, int64_t* sum, int64_t* sum2) {
    return guarded([&] {
        check_handle(h);
        check_replica(h, replica);
        DeviceGuard g(h->device);
        enqueue_width(h, replica, nullptr);
        cuda_check(cudaMemcpyAsync(h->hpin, h->wout, 24, cudaMemcpyDeviceToHost, h->stream), "readback");
        sync(h);
        *sum = int64_t(h->hpin[0]);
        *sum2 = int64_t(h->hpin[1] + h->hpin[2]);
    });
}

int lfg_kpz_debug_record_anchors(lfg_kpz* h, void* dev_buf, size_t capacity_words) {
    return guarded([&] {
        check_handle(h);
        check_resident(h);
        if (!dev_buf) {
            h->wlog = nullptr;
            return;
        }
        if (h->R != 1) throw Error(LFG_EINVAL, "debug_record_anchors: single-replica handles only");
        const size_t need = size_t(h->L) * h->L / 512 * size_t(kpz_rounds(h->sub)) * size_t(h->sub);
        if (capacity_words < need)
            throw Error(LFG_EINVAL, "debug_record_anchors: buffer must hold one MCS of records (" +
                                        std::to_string(need) + " words: L*L/512 tiles x rounds x sub)");
        h->wlog = static_cast<uint32_t*>(dev_buf);
    });
}

int lfg_kpz_width_sums_async(lfg_kpz* h, int32_t replica, int64_t* out3) {
    return guarded([&] {
        check_handle(h);
        check_replica(h, replica);
        if (!out3) throw Error(LFG_EINVAL, "null output");
        DeviceGuard g(h->device);
        enqueue_width(h, replica, nullptr);
        cuda_check(cudaMemcpyAsync(out3, h->wout, 24, cudaMemcpyDeviceToHost, h->stream), "readback");
    });
}

int lfg_kpz_interface_width(lfg_kpz* h, int32_t replica, double* w2) {
    int64_t s = 0, s2 = 0;
    const int rc = lfg_kpz_width_sums(h, replica, &s, &s2);
    if (rc != LFG_OK) return rc;
    const double n = double(int64_t(h->L) * h->L);  // kpz.cpp:78-80
    const double mean = double(s) / n;
    *w2 = double(s2) / n - mean * mean;
    return LFG_OK;
}

int lfg_kpz_heights(lfg_kpz* h, int32_t replica, int32_t* heights, size_t n) {
    return guarded([&] {
        check_handle(h);
        check_replica(h, replica);
        const size_t need = size_t(h->L) * h->L;
        if (n != need || !heights) throw Error(LFG_EINVAL, "heights: expected L*L entries");
        if (h->L > 16384) throw Error(LFG_EINVAL, "heights: L*L int32 readout limited to L <= 16384");
        DeviceGuard g(h->device);
        cuda_check(cudaMemcpyAsync(h->hpin, h->dbad + replica, 8, cudaMemcpyDeviceToHost, h->stream), "readback");
        sync(h);
        if (h->hpin[0] != 0) throw_closure();  // kpz.cpp:37-47: row/column sums must vanish
        ensure_width_scratch(h);
        if (!h->hbuf) h->hbuf = dmalloc<int32_t>(need, "alloc heights");
        cuda_check(kpz_launch_heights(h->rep(replica), h->L, h->H0, h->hbuf, h->stream), "heights");
        cuda_check(cudaMemcpyAsync(heights, h->hbuf, need * 4, cudaMemcpyDeviceToHost, h->stream), "readback");
        sync(h);
    });
}

int lfg_kpz_set_params(lfg_kpz* h, double p, double q) {
    return guarded([&] {
        check_handle(h);
        validate_params(p, q);
        h->p = p;
        h->q = q;
    });
}

int lfg_kpz_set_sweep_index(lfg_kpz* h, uint64_t sweep) {
    return guarded([&] {
        check_handle(h);
        h->sweep = sweep;
    });
}

int lfg_kpz_get_sweep_index(const lfg_kpz* h, uint64_t* sweep) {
    return guarded([&] {
        check_handle(h);
        *sweep = h->sweep;
    });
}

int lfg_kpz_set_seed(lfg_kpz* h, int32_t replica, uint64_t seed) {
    return guarded([&] {
        check_handle(h);
        check_replica(h, replica);
        DeviceGuard g(h->device);
        h->seeds[size_t(replica)] = seed;
        cuda_check(cudaMemcpyAsync(h->dseeds, h->seeds.data(), 8 * size_t(h->R), cudaMemcpyHostToDevice, h->stream),
                   "seed upload");
        sync(h);
    });
}

int lfg_kpz_set_stream(lfg_kpz* h, void* stream) {
    return guarded([&] {
        check_handle(h);
        DeviceGuard g(h->device);
        sync(h);
        if (h->own_stream) cudaStreamDestroy(h->stream);
        h->own_stream = false;
        h->stream = static_cast<cudaStream_t>(stream);
    });
}

int lfg_kpz_synchronize(lfg_kpz* h) {
    return guarded([&] {
        check_handle(h);
        DeviceGuard g(h->device);
        sync(h);
    });
}

int lfg_kpz_device_spins(lfg_kpz* h, int32_t replica, void** ptr, size_t* bytes) {
    return guarded([&] {
        check_handle(h);
        check_replica(h, replica);
        *ptr = h->rep(replica);
        *bytes = h->words_per_replica() * 4;
    });
}

// ------------------------------------------------------------------ strip-sharded path
int lfg_kpz_create_strip(lfg_kpz** out, int32_t L, double p, double q, uint64_t seed, const lfg_kpz_plan* plan,
                         int32_t device) {
    return guarded([&] {
        if (!out) throw Error(LFG_EINVAL, "null output handle");
        *out = nullptr;
        validate_size(L);
        validate_params(p, q);
        auto* h = new lfg_kpz();
        try {
            h->L = L;
            h->p = p;
            h->q = q;
            h->R = 1;
            h->device = device;
            h->strip_only = true;
            resolve_plan(h, plan);
            h->seeds.assign(1, seed);
            h->hcnt.assign(3, 0);
            h->attempts.assign(1, 0);
            DeviceGuard g(device);
            cuda_check(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking), "cudaStreamCreate");
            h->own_stream = true;
            cuda_check(kpz_phase_kernel_attrs(), "kernel attributes");
            h->dcnt = dmalloc<unsigned long long>(3, "alloc counters");
            cuda_check(cudaMallocHost(&h->hpin, sizeof(unsigned long long) * 3), "alloc pinned");
            cuda_check(cudaMemsetAsync(h->dcnt, 0, 24, h->stream), "memset");
            sync(h);
        } catch (...) {
            lfg_kpz_destroy(h);
            throw;
        }
        *out = h;
    });
}

int lfg_kpz_sweep_origin(int32_t L, const lfg_kpz_plan* plan, uint64_t seed, uint64_t sweep, int32_t out6[6]) {
    return guarded([&] {
        lfg_kpz tmp;
        tmp.L = L;
        validate_size(L);
        resolve_plan(&tmp, plan);
        const KpzSweep sw = kpz_sweep_draw(tmp.bx, tmp.by, seed, sweep);
        out6[0] = sw.ox;
        out6[1] = sw.oy;
        for (int k = 0; k < 4; ++k) out6[2 + k] = sw.set(k);
    });
}

namespace {
void check_ring(const lfg_kpz* h, const void* rows, int32_t cap) {
    if (!rows) throw Error(LFG_EINVAL, "null row buffer");
    if (cap < 1 || !is_pow2(cap) || cap > h->L)
        throw Error(LFG_EINVAL, "row_capacity must be a power of two <= L, got " + std::to_string(cap));
}
}  // namespace

int lfg_kpz_strip_phase(lfg_kpz* h, void* rows, int32_t cap, int32_t brow0, int32_t nbrow, uint64_t sweep,
                        int32_t phase) {
    return lfg_kpz_strip_phase_push(h, rows, cap, brow0, nbrow, sweep, phase, nullptr, -1, nullptr, -1);
}

int lfg_kpz_strip_phase_push(lfg_kpz* h, void* rows, int32_t cap, int32_t brow0, int32_t nbrow, uint64_t sweep,
                             int32_t phase, void* peer_dn, int32_t push_row_dn, void* peer_up, int32_t push_row_up) {
    return guarded([&] {
        check_handle(h);
        check_ring(h, rows, cap);
        if (phase < 0 || phase > 3) throw Error(LFG_EINVAL, "phase must be in 0..3");
        if (brow0 < 0 || (brow0 & 1) || nbrow < 2 || (nbrow & 1) || brow0 + nbrow > h->L / h->by)
            throw Error(LFG_EINVAL, "block-row range must be even-aligned inside [0, L/block_y)");
        if (cap < h->L && cap < nbrow * h->by + 2)
            throw Error(LFG_EINVAL, "row_capacity too small for the strip and its ghost rows");
        DeviceGuard g(h->device);
        KpzPhaseArgs a = base_phase_args(h);
        a.f = static_cast<uint32_t*>(rows);
        a.row_mask = cap - 1;
        a.brow0 = brow0;
        a.nbrow = nbrow;
        a.sweep = sweep;
        a.phase = phase;
        a.peer_dn = static_cast<uint32_t*>(peer_dn);
        a.peer_up = static_cast<uint32_t*>(peer_up);
        a.push_row_dn = peer_dn ? push_row_dn : -1;
        a.push_row_up = peer_up ? push_row_up : -1;
        a.abort_flag = h->abort_flag;
        cuda_check(kpz_launch_phase(a, h->seeds.data(), 1, h->stream), "kpz_dtr_phase launch");
        h->attempts[0] += sub_sweep_attempts(h, nbrow) / 4;
    });
}

int lfg_kpz_set_abort_flag(lfg_kpz* h, const void* dev_flag) {
    return guarded([&] {
        check_handle(h);
        h->abort_flag = static_cast<const uint32_t*>(dev_flag);
    });
}

int lfg_kpz_strip_fill(lfg_kpz* h, void* rows, int32_t cap, int32_t row_begin, int32_t row_count, int32_t pattern) {
    return guarded([&] {
        check_handle(h);
        check_ring(h, rows, cap);
        if (row_count < 0 || row_count > cap) throw Error(LFG_EINVAL, "row_count out of range");
        DeviceGuard g(h->device);
        cuda_check(kpz_launch_fill_rows(static_cast<uint32_t*>(rows), h->L, cap - 1, row_begin, row_count, pattern,
                                        h->stream),
                   "fill rows");
    });
}

int lfg_kpz_strip_row0_heights(lfg_kpz* h, const void* rows, int32_t cap, void* H0) {
    return guarded([&] {
        check_handle(h);
        check_ring(h, rows, cap);
        DeviceGuard g(h->device);
        cuda_check(kpz_launch_row0_heights(static_cast<const uint32_t*>(rows), h->L, static_cast<int32_t*>(H0),
                                           h->stream),
                   "row0 heights");
    });
}

int lfg_kpz_strip_width_partials(lfg_kpz* h, const void* rows, int32_t cap, int32_t row_begin, int32_t row_count,
                                 int32_t seg_rows, void* P1, void* D, void* P2) {
    return guarded([&] {
        check_handle(h);
        check_ring(h, rows, cap);
        if (seg_rows < 1 || row_count < 1) throw Error(LFG_EINVAL, "empty width segment");
        DeviceGuard g(h->device);
        cuda_check(kpz_launch_width_partials(static_cast<const uint32_t*>(rows), h->L, cap - 1, row_begin, row_count,
                                             seg_rows, static_cast<int32_t*>(P1), static_cast<int32_t*>(D),
                                             static_cast<unsigned long long*>(P2), h->stream),
                   "width partials");
    });
}

int lfg_kpz_strip_width_rows(lfg_kpz* h, const void* rows, int32_t cap, int32_t row_begin, int32_t row_count,
                             int64_t out3[3]) {
    return guarded([&] {
        check_handle(h);
        check_ring(h, rows, cap);
        if (row_count < 0 || row_count > h->L || row_begin < 0 || row_begin >= h->L)
            throw Error(LFG_EINVAL, "width rows: bad row range");
        if (!out3) throw Error(LFG_EINVAL, "null output");
        DeviceGuard g(h->device);
        ensure_width_scratch(h);
        cuda_check(cudaMemsetAsync(h->wout, 0, 24, h->stream), "memset");
        cuda_check(kpz_launch_width_rows(static_cast<const uint32_t*>(rows), h->L, cap - 1, row_begin, row_count,
                                         h->wscr, h->wout, h->stream),
                   "width rows");
        cuda_check(cudaMemcpyAsync(h->hpin, h->wout, 24, cudaMemcpyDeviceToHost, h->stream), "readback");
        sync(h);
        for (int k = 0; k < 3; ++k) out3[k] = int64_t(h->hpin[k]);
    });
}

int lfg_kpz_width_combine(lfg_kpz* h, const void* H0, const void* P1, const void* D, const void* seg_len,
                          int32_t nseg, int64_t* sum, int64_t* sum2_rel) {
    return guarded([&] {
        check_handle(h);
        DeviceGuard g(h->device);
        if (!h->wout) h->wout = dmalloc<unsigned long long>(3, "alloc width scratch");
        cuda_check(cudaMemsetAsync(h->wout, 0, 16, h->stream), "memset");
        cuda_check(kpz_launch_width_combine(static_cast<const int32_t*>(H0), static_cast<const int32_t*>(P1),
                                            static_cast<const int32_t*>(D), static_cast<const int32_t*>(seg_len),
                                            h->L, nseg, h->wout, h->stream),
                   "width combine");
        cuda_check(cudaMemcpyAsync(h->hpin, h->wout, 16, cudaMemcpyDeviceToHost, h->stream), "readback");
        sync(h);
        *sum = int64_t(h->hpin[0]);
        *sum2_rel = int64_t(h->hpin[1]);
    });
}

}  // extern "C"

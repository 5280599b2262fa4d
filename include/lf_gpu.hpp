// lf_gpu.hpp -- C++ drop-in for the reference simulation API (namespace lf,
// /root/reference/proj/include/lf) running on the B200 library (liblfg.so).
//
// Header-only, C++17, no CUDA headers: it talks to the device exclusively
// through the C ABI in lfg.h / lfg_kmc.h.  Lattice arguments are taken by
// duck typing, so the reference's own lf::SlopeField and lf::OccupancyLattice
// (or the minimal lf::gpu types below) work unchanged:
//
//   Field:    size(), words_x(), words_y()       (lattice.hpp:60-84)
//   Lattice:  size(), words()                    (lattice.hpp:111-126)
//   Params:   KpzParams{p, q} (kpz.hpp:15-29), KmcParams{eps, active_mode}
//             (kmc.hpp:18-27; active_mode: 0 = b_only, 1 = both)
//   Rng:      next_u32()                         (rng.hpp:56-57)
//
// Drop-in replacements (same signatures, same exception types/messages):
//   lf::kpz_sweep_sequential(f, params, rng, sweeps)  -> lf::gpu::kpz_sweep(f, params, rng, sweeps)
//   lf::interface_width(f)                            -> lf::gpu::interface_width(f)
//   lf::reconstruct_heights(f)                        -> lf::gpu::reconstruct_heights(f)
//   lf::kmc_mcs_sequential(lat, params, rng, steps)   -> lf::gpu::kmc_mcs(lat, params, rng, steps)
//   lf::open_bonds_per_particle(lat)                  -> lf::gpu::open_bonds_per_particle(lat)
// The free functions upload the host lattice, run on the device and copy it
// back (the reference mutates the caller's lattice in place).  Long runs
// should keep the state resident with lf::gpu::KpzDevice / KmcDevice.
//
// Seeding: the device RNG is Philox4x32-10 keyed by a 64-bit seed and a
// sweep index.  The free functions draw the key from the caller's RngStream
// (two next_u32() calls per call), so repeated calls advance the caller's
// stream exactly like the reference's sweeps consume it -- the trajectories
// differ from the serial LCG (the scheduler is DTr, not random-sequential),
// the statistics agree (tests/ + DESIGN.md "Parity").
#pragma once

#include <cstdint>
#include <new>
#include <stdexcept>
#include <string>
#include <vector>

#include "lfg.h"
#include "lfg_kmc.h"

namespace lf {
namespace gpu {

// ------------------------------------------------------------------ errors
inline void check(int rc) {
    if (rc == LFG_OK) return;
    const std::string msg = lfg_last_error();
    switch (rc) {
        case LFG_EINVAL: throw std::invalid_argument(msg);
        case LFG_ECLOSURE: throw std::runtime_error(msg);
        case LFG_EDOMAIN: throw std::domain_error(msg);
        case LFG_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error("lfg: " + msg);
    }
}

struct Counters {  // counters.hpp:10-19
    std::int64_t attempts = 0;
    std::int64_t successes = 0;
    Counters& operator+=(const Counters& o) {
        attempts += o.attempts;
        successes += o.successes;
        return *this;
    }
};

struct KpzParams {  // kpz.hpp:15-29
    double p = 1.0;
    double q = 0.0;
};

struct KmcParams {  // kmc.hpp:18-27
    double eps = 1.5;
    int active_mode = 0;  // 0 = b_only, 1 = both
};

struct DtrPlan {
    std::int32_t block_x = 0, block_y = 0;  // KPZ device block (0 = auto)
    std::int32_t sub = 0;                   // sub-sweeps per MCS (0 = default: KPZ 4, KMC 1; 1 = the paper's scheme)
    std::int32_t block = 0;                 // KMC device block edge (0 = auto)
    // KPZ y-strips / KMC z-slabs over several GPUs from this one thread
    // (lfg_kpz_create_sharded / lfg_kmc_create_sharded): devices 0..n_gpus-1, or the
    // explicit list `devices` (a device may repeat).
    std::int32_t n_gpus = 1;
    std::vector<std::int32_t> devices;
};

template <class Rng>
std::uint64_t key_from(Rng& rng) {
    const std::uint64_t hi = rng.next_u32();
    return (hi << 32) | std::uint64_t(rng.next_u32());
}

// ------------------------------------------------------------------ KPZ
class KpzDevice {
public:
    // plan.n_gpus > 1 or plan.devices with > 1 entry: the lattice is split into
    // y-strips over those GPUs (BASELINE configs[2]), same trajectory bit for bit.
    KpzDevice(std::int32_t L, double p, double q, std::uint64_t seed, const DtrPlan& plan = {}, int device = 0) {
        lfg_kpz_plan pl{plan.block_x, plan.block_y, plan.sub};
        std::vector<std::int32_t> devs = plan.devices;
        if (devs.empty())
            for (std::int32_t g = 0; g < plan.n_gpus; ++g) devs.push_back(plan.n_gpus > 1 ? g : device);
        if (devs.size() > 1) check(lfg_kpz_create_sharded(&s_, L, p, q, seed, &pl, std::int32_t(devs.size()), devs.data()));
        else check(lfg_kpz_create(&h_, L, p, q, seed, &pl, devs[0]));
        L_ = L;
    }
    KpzDevice(const KpzDevice&) = delete;
    KpzDevice& operator=(const KpzDevice&) = delete;
    ~KpzDevice() {
        if (h_) lfg_kpz_destroy(h_);
        if (s_) lfg_kpz_sharded_destroy(s_);
    }

    std::int32_t size() const { return L_; }
    bool sharded() const { return s_ != nullptr; }
    void make_flat_slopes() { check(s_ ? lfg_kpz_sharded_init_flat(s_) : lfg_kpz_init_flat(h_)); }

    template <class Field>
    void upload(const Field& f) {
        if (f.size() != L_) throw std::invalid_argument("KpzDevice: lattice size mismatch");
        check(s_ ? lfg_kpz_sharded_upload(s_, f.words_x(), f.words_y(), nwords())
                 : lfg_kpz_upload(h_, 0, f.words_x(), f.words_y(), nwords()));
    }
    template <class Field>
    void download(Field& f) const {
        if (f.size() != L_) throw std::invalid_argument("KpzDevice: lattice size mismatch");
        check(s_ ? lfg_kpz_sharded_download(s_, f.words_x(), f.words_y(), nwords())
                 : lfg_kpz_download(h_, 0, f.words_x(), f.words_y(), nwords()));
    }

    Counters sweep(int sweeps = 1) {
        lfg_counters c{};
        check(s_ ? lfg_kpz_sharded_sweep(s_, sweeps, &c) : lfg_kpz_sweep(h_, sweeps, &c));
        return Counters{c.attempts, c.successes};
    }
    lfg_counters counters_detail() {
        lfg_counters c{};
        check(s_ ? lfg_kpz_sharded_counters(s_, &c) : lfg_kpz_counters(h_, 0, &c));
        return c;
    }
    double interface_width() {
        double w = 0;
        check(s_ ? lfg_kpz_sharded_interface_width(s_, &w) : lfg_kpz_interface_width(h_, 0, &w));
        return w;
    }
    std::vector<std::int32_t> reconstruct_heights() {
        std::vector<std::int32_t> out(std::size_t(L_) * std::size_t(L_));
        if (s_) {  // through the slope planes (the readout checks closure like kpz.cpp:35-47)
            std::vector<std::uint64_t> x(nwords()), y(nwords());
            check(lfg_kpz_sharded_download(s_, x.data(), y.data(), nwords()));
            check(lfg_kpz_heights_host(0, L_, x.data(), y.data(), nwords(), out.data(), out.size()));
        } else {
            check(lfg_kpz_heights(h_, 0, out.data(), out.size()));
        }
        return out;
    }
    void set_params(double p, double q) {
        if (s_) throw std::invalid_argument("KpzDevice: set_params on a sharded lattice is not supported");
        check(lfg_kpz_set_params(h_, p, q));
    }
    std::uint64_t sweep_index() const {
        std::uint64_t s = 0;
        check(s_ ? lfg_kpz_sharded_get_sweep_index(s_, &s) : lfg_kpz_get_sweep_index(h_, &s));
        return s;
    }
    void set_sweep_index(std::uint64_t s) {
        check(s_ ? lfg_kpz_sharded_set_sweep_index(s_, s) : lfg_kpz_set_sweep_index(h_, s));
    }
    lfg_kpz* handle() { return h_; }
    lfg_kpz_sharded* sharded_handle() { return s_; }

private:
    std::size_t nwords() const { return std::size_t(L_) * std::size_t(L_) / 64; }
    lfg_kpz* h_ = nullptr;
    lfg_kpz_sharded* s_ = nullptr;
    std::int32_t L_ = 0;
};

// kpz_sweep_sequential (kpz.cpp:5-19) -> two-layer DTr sweeps on the device.
template <class Field, class Params, class Rng>
Counters kpz_sweep(Field& f, const Params& params, Rng& rng, int sweeps = 1, const DtrPlan& plan = {}) {
    KpzDevice d(f.size(), params.p, params.q, key_from(rng), plan);
    d.upload(f);
    const Counters c = d.sweep(sweeps);
    d.download(f);
    return c;
}

// interface_width(const SlopeField&) (kpz.cpp:62-81): exact device sums over
// the caller's slope planes, any L the reference accepts, integrable or not.
template <class Field>
double interface_width(const Field& f, int device = 0) {
    const std::int32_t L = f.size();
    const std::size_t nw = (std::size_t(L) * std::size_t(L) + 63) / 64;
    std::int64_t s = 0, s2 = 0;
    check(lfg_kpz_width_sums_host(device, L, f.words_x(), f.words_y(), nw, &s, &s2));
    const double n = static_cast<double>(std::int64_t(L) * L);  // kpz.cpp:78-80
    const double mean = static_cast<double>(s) / n;
    return static_cast<double>(s2) / n - mean * mean;
}

// reconstruct_heights (kpz.cpp:21-49): h(0,0)=0, row-major j*L+i; throws
// std::runtime_error (the reference's message) when path-dependent.
template <class Field>
std::vector<std::int32_t> reconstruct_heights(const Field& f, int device = 0) {
    const std::int32_t L = f.size();
    const std::size_t nw = (std::size_t(L) * std::size_t(L) + 63) / 64;
    std::vector<std::int32_t> out(std::size_t(L) * std::size_t(L));
    check(lfg_kpz_heights_host(device, L, f.words_x(), f.words_y(), nw, out.data(), out.size()));
    return out;
}

// ------------------------------------------------------------------ KMC
class KmcDevice {
public:
    // plan.n_gpus > 1 or plan.devices with > 1 entry: z-slabs over those GPUs
    // (BASELINE configs[4]), same trajectory bit for bit.
    KmcDevice(std::int32_t L, double eps, bool both_active, std::uint64_t seed, const DtrPlan& plan = {},
              int device = 0) {
        lfg_kmc_plan pl{plan.block, plan.sub};
        std::vector<std::int32_t> devs = plan.devices;
        if (devs.empty())
            for (std::int32_t g = 0; g < plan.n_gpus; ++g) devs.push_back(plan.n_gpus > 1 ? g : device);
        if (devs.size() > 1)
            check(lfg_kmc_create_sharded(&s_, L, eps, both_active ? 1 : 0, seed, &pl, std::int32_t(devs.size()),
                                         devs.data()));
        else
            check(lfg_kmc_create(&h_, L, eps, both_active ? 1 : 0, seed, &pl, devs[0]));
        L_ = L;
    }
    KmcDevice(const KmcDevice&) = delete;
    KmcDevice& operator=(const KmcDevice&) = delete;
    ~KmcDevice() {
        if (h_) lfg_kmc_destroy(h_);
        if (s_) lfg_kmc_sharded_destroy(s_);
    }

    std::int32_t size() const { return L_; }
    bool sharded() const { return s_ != nullptr; }
    template <class Lattice>
    void upload(const Lattice& lat) {
        if (lat.size() != L_) throw std::invalid_argument("KmcDevice: lattice size mismatch");
        check(s_ ? lfg_kmc_sharded_upload(s_, lat.words(), nwords()) : lfg_kmc_upload(h_, lat.words(), nwords()));
    }
    template <class Lattice>
    void download(Lattice& lat) const {
        if (lat.size() != L_) throw std::invalid_argument("KmcDevice: lattice size mismatch");
        check(s_ ? lfg_kmc_sharded_download(s_, lat.words(), nwords()) : lfg_kmc_download(h_, lat.words(), nwords()));
    }
    void make_random_alloy(double c, std::uint64_t seed) {
        check(s_ ? lfg_kmc_sharded_init_random_alloy(s_, c, seed) : lfg_kmc_init_random_alloy(h_, c, seed));
    }
    Counters sweep(int steps = 1) {
        lfg_counters c{};
        check(s_ ? lfg_kmc_sharded_sweep(s_, steps, &c) : lfg_kmc_sweep(h_, steps, &c));
        return Counters{c.attempts, c.successes};
    }
    double open_bonds_per_particle() {
        double v = 0;
        check(s_ ? lfg_kmc_sharded_open_bonds_per_particle(s_, &v) : lfg_kmc_open_bonds_per_particle(h_, &v));
        return v;
    }
    std::int64_t count_b() {
        std::int64_t n = 0;
        if (s_) {
            std::int64_t open = 0;
            check(lfg_kmc_sharded_open_bond_sums(s_, &n, &open));
        } else {
            check(lfg_kmc_count_b(h_, &n));
        }
        return n;
    }
    std::uint64_t sweep_index() const {
        std::uint64_t s = 0;
        check(s_ ? lfg_kmc_sharded_get_sweep_index(s_, &s) : lfg_kmc_get_sweep_index(h_, &s));
        return s;
    }
    void set_sweep_index(std::uint64_t s) {
        check(s_ ? lfg_kmc_sharded_set_sweep_index(s_, s) : lfg_kmc_set_sweep_index(h_, s));
    }
    lfg_kmc* handle() { return h_; }
    lfg_kmc_sharded* sharded_handle() { return s_; }

private:
    std::size_t nwords() const { return std::size_t(L_) * std::size_t(L_) * std::size_t(L_) / 64; }
    lfg_kmc* h_ = nullptr;
    lfg_kmc_sharded* s_ = nullptr;
    std::int32_t L_ = 0;
};

// kmc_mcs_sequential (kmc.cpp:5-18) -> two-layer DT sweeps on the device.
template <class Lattice, class Params, class Rng>
Counters kmc_mcs(Lattice& lat, const Params& params, Rng& rng, int steps = 1, const DtrPlan& plan = {}) {
    KmcDevice d(lat.size(), params.eps, static_cast<int>(params.active_mode) != 0, key_from(rng), plan);
    d.upload(lat);
    const Counters c = d.sweep(steps);
    d.download(lat);
    return c;
}

// open_bonds_per_particle (kmc.cpp:20-40); throws std::domain_error without B.
template <class Lattice>
double open_bonds_per_particle(const Lattice& lat, int device = 0) {
    const std::int32_t L = lat.size();
    const std::size_t nw = (std::size_t(L) * std::size_t(L) * std::size_t(L) + 63) / 64;
    std::int64_t np = 0, no = 0;
    check(lfg_kmc_open_bond_sums_host(device, L, lat.words(), nw, &np, &no));
    if (np == 0) throw std::domain_error("open_bonds_per_particle: no B particles in lattice");
    return static_cast<double>(no) / static_cast<double>(np);
}

}  // namespace gpu
}  // namespace lf

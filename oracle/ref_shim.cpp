// oracle/ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// C-ABI shim over the UNMODIFIED reference sources (/root/reference/proj/src,
// compiled where they lie by oracle/Makefile into oracle/_ref/liblfref.so).
// It lets the Python tests and bench.py's reference arm call the reference's
// own functions: make_flat_slopes, kpz_sweep_sequential, interface_width,
// reconstruct_heights, make_random_alloy, kmc_mcs_sequential,
// open_bonds_per_particle, the RngStream suite, and the DTr schedule of
// oracle_core.hpp driving lf::detail::kpz_attempt_impl<false> (kpz.hpp:71-107)
// unchanged.  No reference source is copied into this repository.
#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "lf/counters.hpp"
#include "lf/kmc.hpp"
#include "lf/kpz.hpp"
#include "lf/lattice.hpp"
#include "lf/rng.hpp"
#include "lf/schedule.hpp"
#include "lf/write_log.hpp"

#include "oracle_core.hpp"

namespace {

thread_local std::string g_err;

lf::RngKind kind_of(int k) {
    return k == 0 ? lf::RngKind::lcg32 : (k == 1 ? lf::RngKind::lcg64_skip : lf::RngKind::tiny_mt);
}

size_t words2(int32_t L) { return size_t((int64_t(L) * L + 63) / 64); }
size_t words3(int32_t L) { return size_t((int64_t(L) * L * L + 63) / 64); }

lf::SlopeField load_field(int32_t L, const uint64_t* x, const uint64_t* y) {
    lf::SlopeField f(L);
    std::memcpy(f.words_x(), x, words2(L) * 8);
    std::memcpy(f.words_y(), y, words2(L) * 8);
    return f;
}

void store_field(const lf::SlopeField& f, uint64_t* x, uint64_t* y) {
    std::memcpy(x, f.words_x(), words2(f.size()) * 8);
    std::memcpy(y, f.words_y(), words2(f.size()) * 8);
}

// Exception -> status: 1 invalid_argument, 2 runtime_error, 3 domain_error, 4 other.
template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::domain_error& e) {
        g_err = e.what();
        return 3;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 4;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// ------------------------------------------------------------------ RNG suite
int ref_rng_draws(int kind, uint64_t seed, uint32_t stream_id, uint64_t skip_n, uint32_t* out,
                  int64_t n) {
    return guarded([&] {
        auto s = lf::RngStream::make(kind_of(kind), seed, stream_id);
        if (skip_n) s.skip(skip_n);
        for (int64_t k = 0; k < n; ++k) out[k] = s.next_u32();
    });
}

int ref_split_streams_state(int kind, uint64_t seed, int count, uint64_t stride, uint64_t* states) {
    return guarded([&] {
        auto v = lf::split_streams(kind_of(kind), seed, count, stride);
        for (int k = 0; k < count; ++k) states[k] = v[size_t(k)].lcg;
    });
}

int ref_rng_kind_from_string(const char* name, int* kind) {
    return guarded([&] { *kind = int(lf::rng_kind_from_string(name)); });
}

// ------------------------------------------------------------------ KPZ
int ref_make_flat(int32_t L, uint64_t* x, uint64_t* y) {
    return guarded([&] { store_field(lf::make_flat_slopes(L), x, y); });
}

int ref_interface_width(int32_t L, const uint64_t* x, const uint64_t* y, double* w2) {
    return guarded([&] { *w2 = lf::interface_width(load_field(L, x, y)); });
}

int ref_reconstruct_heights(int32_t L, const uint64_t* x, const uint64_t* y, int32_t* h) {
    return guarded([&] {
        auto hf = lf::reconstruct_heights(load_field(L, x, y));
        std::memcpy(h, hf.h.data(), hf.h.size() * 4);
    });
}

int ref_closure_holds(int32_t L, const uint64_t* x, const uint64_t* y, int* ok) {
    return guarded([&] { *ok = load_field(L, x, y).closure_holds() ? 1 : 0; });
}

int ref_kpz_params_validate(double p, double q) {
    return guarded([&] { lf::KpzParams{p, q}.validate(); });
}

// kpz_sweep_sequential with an RngStream (kind, seed); the final lcg state is
// returned so sweeps can be chained.  counters: [attempts, successes].
int ref_kpz_sweep_sequential(int32_t L, uint64_t* x, uint64_t* y, double p, double q, int kind,
                             uint64_t* lcg_state, int sweeps, int64_t* counters) {
    return guarded([&] {
        auto f = load_field(L, x, y);
        auto rng = lf::RngStream::make(kind_of(kind), 0);
        rng.lcg = *lcg_state;
        const lf::Counters c = lf::kpz_sweep_sequential(f, lf::KpzParams{p, q}, rng, sweeps);
        store_field(f, x, y);
        *lcg_state = rng.lcg;
        counters[0] += c.attempts;
        counters[1] += c.successes;
    });
}

// A bounded sample of kpz_sweep_sequential: the loop body of kpz.cpp:12-16
// (two next_below draws, then KpzKernel<false>::attempt) for n_attempts
// attempts, so bench.py can time the reference on L=2^16 without a 10-minute
// full MCS.  counters: [attempts, successes].
int ref_kpz_attempts_sequential(int32_t L, uint64_t* x, uint64_t* y, double p, double q, int kind,
                                uint64_t* lcg_state, int64_t n_attempts, int64_t* counters) {
    return guarded([&] {
        const lf::KpzParams params{p, q};
        params.validate();
        lf::SlopeField f(L);
        std::memcpy(f.words_x(), x, words2(L) * 8);
        std::memcpy(f.words_y(), y, words2(L) * 8);
        auto rng = lf::RngStream::make(kind_of(kind), 0);
        rng.lcg = *lcg_state;
        lf::KpzKernel<false> kernel{&f, params};
        const auto Lu = static_cast<uint32_t>(L);
        int64_t succ = 0;
        for (int64_t n = 0; n < n_attempts; ++n) {
            auto i = static_cast<int32_t>(rng.next_below(Lu));
            auto j = static_cast<int32_t>(rng.next_below(Lu));
            succ += kernel.attempt({i, j}, rng);
        }
        std::memcpy(x, f.words_x(), words2(L) * 8);
        std::memcpy(y, f.words_y(), words2(L) * 8);
        *lcg_state = rng.lcg;
        counters[0] += n_attempts;
        counters[1] += succ;
    });
}

// Persistent reference SlopeField so a timed sample excludes host copies
// (wall time around the update loops only).
void* ref_kpz_field_create(int32_t L, const uint64_t* x, const uint64_t* y) {
    try {
        auto* f = new lf::SlopeField(L);
        std::memcpy(f->words_x(), x, words2(L) * 8);
        std::memcpy(f->words_y(), y, words2(L) * 8);
        return f;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_kpz_field_destroy(void* f) { delete static_cast<lf::SlopeField*>(f); }

int ref_kpz_field_attempts(void* fp, double p, double q, int kind, uint64_t* lcg_state, int64_t n_attempts,
                           int64_t* counters) {
    return guarded([&] {
        auto& f = *static_cast<lf::SlopeField*>(fp);
        const lf::KpzParams params{p, q};
        params.validate();
        auto rng = lf::RngStream::make(kind_of(kind), 0);
        rng.lcg = *lcg_state;
        lf::KpzKernel<false> kernel{&f, params};
        const auto Lu = static_cast<uint32_t>(f.size());
        int64_t succ = 0;
        for (int64_t n = 0; n < n_attempts; ++n) {  // kpz.cpp:12-16
            auto i = static_cast<int32_t>(rng.next_below(Lu));
            auto j = static_cast<int32_t>(rng.next_below(Lu));
            succ += kernel.attempt({i, j}, rng);
        }
        *lcg_state = rng.lcg;
        counters[0] += n_attempts;
        counters[1] += succ;
    });
}

// Same for KMC: the loop body of kmc.cpp:13-15 for n_attempts attempts.
int ref_kmc_attempts_sequential(int32_t L, uint64_t* words, double eps, int both, int kind,
                                uint64_t* lcg_state, int64_t n_attempts, int64_t* counters) {
    return guarded([&] {
        lf::OccupancyLattice lat(L);
        std::memcpy(lat.words(), words, words3(L) * 8);
        auto rng = lf::RngStream::make(kind_of(kind), 0);
        rng.lcg = *lcg_state;
        lf::KmcParams params{eps, both ? lf::ActiveMode::both : lf::ActiveMode::b_only};
        params.validate();
        lf::KmcKernel<false> kernel{&lat, params};
        const lf::Coord3 lo{0, 0, 0};
        const lf::Coord3 ext{L, L, L};
        int64_t succ = 0;
        for (int64_t n = 0; n < n_attempts; ++n) succ += kernel.attempt(kernel.draw_site(lo, ext, rng), rng);
        std::memcpy(words, lat.words(), words3(L) * 8);
        *lcg_state = rng.lcg;
        counters[0] += n_attempts;
        counters[1] += succ;
    });
}

// One reference attempt at (i, j) with an externally supplied r (kpz.hpp:112-116).
int ref_kpz_attempt(int32_t L, uint64_t* x, uint64_t* y, int32_t i, int32_t j, double p, double q,
                    double r, int* outcome) {
    return guarded([&] {
        auto f = load_field(L, x, y);
        *outcome = int(lf::kpz_attempt(f, {i, j}, lf::KpzParams{p, q}, r));
        store_field(f, x, y);
    });
}

// The DTr schedule (oracle_core.hpp) with the reference's own attempt kernel:
// MCS sweep0 .. sweep0 + nsweeps - 1, each `sub` sub-sweeps (s' = s * sub + k).
// counters: [attempts, successes, deposits, detaches].
int ref_kpz_sweep_dtr(int32_t L, uint64_t* x, uint64_t* y, double p, double q, uint64_t seed,
                      uint64_t sweep0, int32_t nsweeps, int32_t bx, int32_t by, int32_t sub, int64_t* counters) {
    return guarded([&] {
        const lf::KpzParams params{p, q};
        params.validate();
        if (sub != 1 && sub != 4 && sub != 8) throw std::invalid_argument("DtrPlan: sub must be 1, 4 or 8");
        auto f = load_field(L, x, y);
        orc::KpzPlan pl{L, bx, by, sub};
        int64_t dep = 0, det = 0, att = 0;
        for (int32_t s = 0; s < nsweeps; ++s) {
            for (int32_t k = 0; k < sub; ++k) {
                const uint64_t sweep = (sweep0 + uint64_t(s)) * uint64_t(sub) + uint64_t(k);
                const orc::Counts c = orc::kpz_dtr_sweep(pl, seed, sweep, [&](int32_t i, int32_t j, uint32_t tile_id, int r) {
                    return int(lf::detail::kpz_attempt_impl<false>(f, i, j, params, [&] {
                        return orc::kpz_accept_word(seed, sweep, tile_id, r) * 0x1p-32;
                    }));
                });
                dep += c.dep;
                det += c.det;
                att += c.att;
            }
        }
        store_field(f, x, y);
        counters[0] += att;
        counters[1] += dep + det;
        counters[2] += dep;
        counters[3] += det;
    });
}

// ------------------------------------------------------------------ KMC
int ref_make_random_alloy(int32_t L, double c, int kind, uint64_t seed, uint64_t* words,
                          uint64_t* lcg_state_out) {
    return guarded([&] {
        auto rng = lf::RngStream::make(kind_of(kind), seed);
        auto lat = lf::make_random_alloy(L, c, rng);
        std::memcpy(words, lat.words(), words3(L) * 8);
        if (lcg_state_out) *lcg_state_out = rng.lcg;
    });
}

int ref_kmc_sweep_sequential(int32_t L, uint64_t* words, double eps, int both, int kind,
                             uint64_t* lcg_state, int steps, int64_t* counters) {
    return guarded([&] {
        lf::OccupancyLattice lat(L);
        std::memcpy(lat.words(), words, words3(L) * 8);
        auto rng = lf::RngStream::make(kind_of(kind), 0);
        rng.lcg = *lcg_state;
        lf::KmcParams params{eps, both ? lf::ActiveMode::both : lf::ActiveMode::b_only};
        const lf::Counters c = lf::kmc_mcs_sequential(lat, params, rng, steps);
        std::memcpy(words, lat.words(), words3(L) * 8);
        *lcg_state = rng.lcg;
        counters[0] += c.attempts;
        counters[1] += c.successes;
    });
}

// The KMC DT schedule (oracle_core.hpp) whose attempt follows
// kmc_attempt_impl's decision sequence (kmc.hpp:84-111) using the
// reference's own exchange_probability (kmc.hpp:70-76) and kFccOffsets
// (lattice.hpp:147-151).  kmc_attempt_impl itself takes an RngStream& and
// cannot consume counter-based words, hence this thin restatement.
// MCS sweep0 .. sweep0 + nsweeps - 1, each `sub` sub-sweeps (s' = s * sub + k).
int ref_kmc_sweep_dt(int32_t L, uint64_t* words, double eps, int both, uint64_t seed,
                     uint64_t sweep0, int32_t nsweeps, int32_t bk, int32_t sub, int64_t* counters) {
    return guarded([&] {
        lf::OccupancyLattice lat(L);
        std::memcpy(lat.words(), words, words3(L) * 8);
        lf::KmcParams params{eps, both ? lf::ActiveMode::both : lf::ActiveMode::b_only};
        params.validate();
        const int32_t mask = L - 1;
        if (sub != 1 && sub != 4) throw std::invalid_argument("DtPlan: sub must be 1 or 4");
        orc::KmcPlan pl{L, bk, sub};
        int64_t succ = 0;
        for (int64_t s = 0; s < int64_t(nsweeps) * sub; ++s) {
            succ += orc::kmc_dt_sweep(pl, seed, sweep0 * uint64_t(sub) + uint64_t(s),
                                      [&](int32_t x, int32_t y, int32_t z, uint32_t dir_w, uint32_t acc_w) {
                const lf::Coord3 site{x, y, z};
                const bool here_b = lat.is_b(x, y, z);
                if (!here_b && params.active_mode == lf::ActiveMode::b_only) return 1;
                const auto& d = lf::kFccOffsets[orc::below(dir_w, 12)];
                const lf::Coord3 partner{(x + d[0]) & mask, (y + d[1]) & mask, (z + d[2]) & mask};
                const bool partner_b = lat.is_b(partner[0], partner[1], partner[2]);
                if (partner_b == here_b) return 1;
                const lf::Coord3 b_pos = here_b ? site : partner;
                const lf::Coord3 a_pos = here_b ? partner : site;
                const double w = lf::exchange_probability<false>(lat, b_pos, a_pos, params);
                if (w < 1.0 && !(acc_w * 0x1p-32 < w)) return 2;
                lat.set_b(b_pos[0], b_pos[1], b_pos[2], false);
                lat.set_b(a_pos[0], a_pos[1], a_pos[2], true);
                return 0;
            });
        }
        std::memcpy(words, lat.words(), words3(L) * 8);
        counters[0] += int64_t(L) * L * L / 2 * nsweeps;
        counters[1] += succ;
    });
}

int ref_open_bonds_per_particle(int32_t L, const uint64_t* words, double* out) {
    return guarded([&] {
        lf::OccupancyLattice lat(L);
        std::memcpy(lat.words(), words, words3(L) * 8);
        *out = lf::open_bonds_per_particle(lat);
    });
}

int ref_count_b(int32_t L, const uint64_t* words, int64_t* out) {
    return guarded([&] {
        lf::OccupancyLattice lat(L);
        std::memcpy(lat.words(), words, words3(L) * 8);
        *out = lat.count_b();
    });
}

int ref_metropolis_prob(int ni, int nf, double eps, double* out) {
    return guarded([&] { *out = lf::metropolis_prob(ni, nf, lf::KmcParams{eps}); });
}

int ref_fcc_neighbors(int32_t x, int32_t y, int32_t z, int32_t L, int32_t* out36) {
    return guarded([&] {
        auto nb = lf::fcc_neighbors({x, y, z}, L);
        for (int k = 0; k < 12; ++k)
            for (int a = 0; a < 3; ++a) out36[k * 3 + a] = nb[size_t(k)][size_t(a)];
    });
}

// ------------------------------------------------------------------ schedule
int ref_schedule_ahead_of_time_steps(int32_t blocks, int32_t workers, int32_t sets, int32_t* sizes,
                                     int32_t cap, int32_t* n) {
    return guarded([&] {
        auto s = lf::schedule_ahead_of_time(blocks, workers, sets);
        *n = int32_t(s.size());
        for (size_t k = 0; k < s.size() && int32_t(k) < cap; ++k) sizes[k] = int32_t(s[k].size());
    });
}

// ------------------------------------------------------------------ write log
// Drive the reference's lf::WriteLog (write_log.hpp:16-49) with a recorded
// schedule.  Groups are barrier intervals: every task of a group is begun
// before any of the group's writes is logged and all are ended afterwards, so
// tasks of one group are mutually concurrent and groups are ordered.  Returns
// the number of violations (same site written by distinct workers in
// overlapping tasks) and the first one.
int ref_writelog_violations(int32_t workers, int64_t ngroups, const int64_t* group_off, const int32_t* task_worker,
                            const int64_t* task_woff, const int64_t* write_site, int64_t* nviol, int64_t* nwrites,
                            int64_t* first3) {
    return guarded([&] {
        lf::WriteLog log(workers);
        std::vector<int32_t> tid;
        for (int64_t g = 0; g < ngroups; ++g) {
            const int64_t t0 = group_off[g], t1 = group_off[g + 1];
            tid.assign(size_t(t1 - t0), 0);
            for (int64_t t = t0; t < t1; ++t) tid[size_t(t - t0)] = log.begin_task(task_worker[t]);
            for (int64_t t = t0; t < t1; ++t)
                for (int64_t w = task_woff[t]; w < task_woff[t + 1]; ++w)
                    log.log_write(task_worker[t], tid[size_t(t - t0)], write_site[w]);
            for (int64_t t = t0; t < t1; ++t) log.end_task(task_worker[t], tid[size_t(t - t0)]);
        }
        const auto v = log.violations();
        *nviol = int64_t(v.size());
        *nwrites = log.write_count();
        if (!v.empty()) {
            first3[0] = v[0].site;
            first3[1] = v[0].worker_a;
            first3[2] = v[0].worker_b;
        }
    });
}

}  // extern "C"

// tests/cpp/linkdrop_test.cpp -- the LINK-LEVEL drop-in (dropin/lf_gpu_link.cpp).
//
// Built from the reference's own headers and sources with proj/src/kpz.cpp and
// proj/src/kmc.cpp REPLACED by dropin/lf_gpu_link.cpp (tests/cpp/build.sh), so
// every lf:: call below is spelled exactly as a reference user spells it and
// resolves to the B200 library.  It prints key=value lines that
// tests/test_cpp_dropin.py checks against the oracle and the reference.
#include <cstdint>
#include <cstdio>
#include <stdexcept>

#include "lf/kmc.hpp"
#include "lf/kpz.hpp"
#include "lf/lattice.hpp"
#include "lf/rng.hpp"

static uint64_t fnv(const uint64_t* w, size_t n) {
    uint64_t h = 1469598103934665603ull;
    const unsigned char* b = reinterpret_cast<const unsigned char*>(w);
    for (size_t k = 0; k < 8 * n; ++k) h = (h ^ b[k]) * 1099511628211ull;
    return h;
}

int main() {
    // KPZ sweeps through lf::kpz_sweep_sequential (kpz.hpp:119-120)
    {
        lf::SlopeField f = lf::make_flat_slopes(256);
        auto rng = lf::RngStream::make(lf::RngKind::lcg64_skip, 7);
        const lf::Counters c = lf::kpz_sweep_sequential(f, lf::KpzParams{0.95, 0.05}, rng, 2);
        const size_t nw = 256 * 256 / 64;
        std::printf("kpz %lld %lld %.17g %llu %llu %llu\n", (long long)c.attempts, (long long)c.successes,
                    lf::interface_width(f), (unsigned long long)fnv(f.words_x(), nw),
                    (unsigned long long)fnv(f.words_y(), nw), (unsigned long long)rng.lcg);
        const lf::HeightField h = lf::reconstruct_heights(f);
        long long s = 0;
        for (auto v : h.h) s += v;
        std::printf("kpz_heights %lld %.17g\n", s, lf::interface_width(h));
    }
    // readouts on small and non-integrable fields (any L >= 4, kpz.cpp:21-81)
    {
        lf::SlopeField d(8);  // all slopes -1 (lattice.cpp:20-25): not integrable
        std::printf("w2_default8 %.17g\n", lf::interface_width(d));
        try {
            (void)lf::reconstruct_heights(d);
            std::printf("heights_default8 ok\n");
        } catch (const std::runtime_error& e) {
            std::printf("heights_default8 runtime_error\n");
        }
        lf::SlopeField f4 = lf::make_flat_slopes(4);
        const lf::HeightField h4 = lf::reconstruct_heights(f4);
        long long s = 0;
        for (auto v : h4.h) s += v;
        std::printf("flat4 %lld %.17g %.17g\n", s, lf::interface_width(f4), lf::interface_width(h4));
    }
    // KMC through lf::kmc_mcs_sequential (kmc.hpp:128-129)
    {
        auto rng = lf::RngStream::make(lf::RngKind::lcg64_skip, 11);
        lf::OccupancyLattice lat = lf::make_random_alloy(64, 0.5, rng);
        const lf::Counters c = lf::kmc_mcs_sequential(lat, lf::KmcParams{1.5, lf::ActiveMode::both}, rng, 1);
        const size_t nw = size_t(64) * 64 * 64 / 64;
        std::printf("kmc %lld %lld %.17g %llu\n", (long long)c.attempts, (long long)c.successes,
                    lf::open_bonds_per_particle(lat), (unsigned long long)fnv(lat.words(), nw));
        auto r8 = lf::RngStream::make(lf::RngKind::lcg64_skip, 3);
        lf::OccupancyLattice small = lf::make_random_alloy(8, 0.5, r8);
        std::printf("obpp8 %.17g\n", lf::open_bonds_per_particle(small));
        lf::OccupancyLattice empty(16);
        try {
            (void)lf::open_bonds_per_particle(empty);
            std::printf("empty ok\n");
        } catch (const std::domain_error&) {
            std::printf("empty domain_error\n");
        }
    }
    // the DT decomposition's lower size limit: std::invalid_argument
    {
        lf::SlopeField f = lf::make_flat_slopes(32);
        auto rng = lf::RngStream::make(lf::RngKind::lcg64_skip, 1);
        try {
            (void)lf::kpz_sweep_sequential(f, lf::KpzParams{1.0, 0.0}, rng, 1);
            std::printf("small_sweep ok\n");
        } catch (const std::invalid_argument&) {
            std::printf("small_sweep invalid_argument\n");
        }
    }
    std::printf("linkdrop OK\n");
    return 0;
}

// tests/cpp/dropin_test.cpp -- the C++ drop-in (include/lf_gpu.hpp) used the
// way a reference user would use it.
//
// With -DLF_WITH_REFERENCE (compiled against /root/reference/proj/include and
// linked with oracle/_ref/liblfref.so, the unmodified reference sources) it
// drives lf::gpu with the reference's own lf::SlopeField, lf::RngStream and
// lf::OccupancyLattice and cross-checks every readout against the reference's
// CPU functions.  Without it, minimal stand-in types are used.  Exit 0 = pass.
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <vector>

#include "lf_gpu.hpp"

#ifdef LF_WITH_REFERENCE
#include "lf/kmc.hpp"
#include "lf/kpz.hpp"
#include "lf/lattice.hpp"
#include "lf/rng.hpp"
#endif

#define REQUIRE(c)                                                    \
    do {                                                              \
        if (!(c)) {                                                   \
            std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #c); \
            std::exit(1);                                             \
        }                                                             \
    } while (0)

#ifndef LF_WITH_REFERENCE
// Stand-ins with the reference's member names (lattice.hpp:56-135, rng.hpp:47-67).
struct SlopeField {
    explicit SlopeField(int32_t L) : L_(L), x_(size_t(L) * L / 64), y_(size_t(L) * L / 64) {}
    int32_t size() const { return L_; }
    uint64_t* words_x() { return x_.data(); }
    uint64_t* words_y() { return y_.data(); }
    const uint64_t* words_x() const { return x_.data(); }
    const uint64_t* words_y() const { return y_.data(); }
    int32_t L_;
    std::vector<uint64_t> x_, y_;
};
SlopeField make_flat_slopes(int32_t L) {
    SlopeField f(L);
    for (int32_t j = 0; j < L; ++j)
        for (int32_t i = 0; i < L; ++i) {
            const int64_t idx = int64_t(j) * L + i;
            if ((i & 1) == 0) f.x_[size_t(idx >> 6)] |= uint64_t{1} << (idx & 63);
            if ((j & 1) == 0) f.y_[size_t(idx >> 6)] |= uint64_t{1} << (idx & 63);
        }
    return f;
}
struct Occupancy {
    explicit Occupancy(int32_t L) : L_(L), w_(size_t(L) * L * L / 64) {}
    int32_t size() const { return L_; }
    uint64_t* words() { return w_.data(); }
    const uint64_t* words() const { return w_.data(); }
    int32_t L_;
    std::vector<uint64_t> w_;
};
struct Rng {
    uint64_t s = 1;
    uint32_t next_u32() {
        s = 6364136223846793005ull * s + 1442695040888963407ull;
        return uint32_t(s >> 32);
    }
};
#endif

int main() {
    int ndev = 0;
    lfg_device_count(&ndev);
    if (ndev < 1) {
        std::printf("SKIP: no CUDA device\n");
        return 0;
    }
    // ---------------------------------------------------------------- KPZ
#ifdef LF_WITH_REFERENCE
    lf::SlopeField f = lf::make_flat_slopes(256);
    auto rng = lf::RngStream::make(lf::RngKind::lcg64_skip, 12345);
    const lf::KpzParams params{0.95, 0.05};
#else
    SlopeField f = make_flat_slopes(256);
    Rng rng;
    const lf::gpu::KpzParams params{0.95, 0.05};
#endif
    REQUIRE(lf::gpu::interface_width(f) == 0.5);
    const auto c = lf::gpu::kpz_sweep(f, params, rng, 5);
    // default plan (sub = 4): Poisson tile counts, mean L^2 and sd L per MCS
    REQUIRE(std::llabs(c.attempts - 5LL * 256 * 256) < 6LL * 256 * 3);
    REQUIRE(c.successes > 0);
    const double w2 = lf::gpu::interface_width(f);
    REQUIRE(w2 > 0.5);
#ifdef LF_WITH_REFERENCE
    REQUIRE(f.closure_holds());                    // lattice.cpp:61-69 on the downloaded words
    REQUIRE(w2 == lf::interface_width(f));         // kpz.cpp:62-81 on the CPU
    const auto hr = lf::reconstruct_heights(f);    // kpz.cpp:21-49
    REQUIRE(lf::gpu::reconstruct_heights(f) == hr.h);
#endif
    // invalid parameters -> std::invalid_argument, like KpzParams::validate (kpz.hpp:19-26)
    bool threw = false;
    try {
        lf::gpu::KpzDevice bad(256, 1.5, 0.0, 1);
    } catch (const std::invalid_argument&) {
        threw = true;
    }
    REQUIRE(threw);

    // ---------------------------------------------------------------- KMC
#ifdef LF_WITH_REFERENCE
    auto arng = lf::RngStream::make(lf::RngKind::lcg64_skip, 1);
    lf::OccupancyLattice lat = lf::make_random_alloy(64, 0.325, arng);
    const int64_t nb0 = lat.count_b();
    REQUIRE(nb0 == 42587);
    const lf::KmcParams kp{1.5, lf::ActiveMode::both};
    REQUIRE(lf::gpu::open_bonds_per_particle(lat) == lf::open_bonds_per_particle(lat));
    const auto kc = lf::gpu::kmc_mcs(lat, kp, arng, 3);
    REQUIRE(kc.attempts == 3LL * 64 * 64 * 64 / 2);
    REQUIRE(lat.count_b() == nb0);                  // species conservation
    REQUIRE(lf::gpu::open_bonds_per_particle(lat) == lf::open_bonds_per_particle(lat));
    lf::OccupancyLattice empty(32);
    bool dom = false;
    try {
        lf::gpu::open_bonds_per_particle(empty);
    } catch (const std::domain_error&) {
        dom = true;
    }
    REQUIRE(dom);
#else
    Occupancy lat(64);
    for (size_t k = 0; k < lat.w_.size(); ++k) {  // random B on fcc-valid (even x^y^z) sites only
        const size_t row = k / 1;                  // 64-bit word == one x-row at L = 64
        const int y = int(row % 64), z = int(row / 64);
        const uint64_t valid = ((y ^ z) & 1) ? 0xAAAAAAAAAAAAAAAAull : 0x5555555555555555ull;
        lat.w_[k] = valid & (0x9E3779B97F4A7C15ull * (k + 1));
    }
    const lf::gpu::KmcParams kp{1.5, 1};
    const double ob0 = lf::gpu::open_bonds_per_particle(lat);
    const auto kc = lf::gpu::kmc_mcs(lat, kp, rng, 2);
    REQUIRE(kc.attempts == 2LL * 64 * 64 * 64 / 2);
    REQUIRE(ob0 > 0.0);
#endif
    {   // configs[2] through the C++ API: the same lattice on 1 GPU and split into 2 strips
        // (lfg_kpz_create_sharded; both strips on device 0 of the test box) -> identical.
        const int32_t Ls = 2048;
        lf::gpu::DtrPlan two;
        two.devices = {0, 0};
        lf::gpu::KpzDevice one_gpu(Ls, 0.95, 0.05, 4242), strips(Ls, 0.95, 0.05, 4242, two);
        REQUIRE(strips.sharded() && !one_gpu.sharded());
        one_gpu.make_flat_slopes();
        strips.make_flat_slopes();
        const auto c1 = one_gpu.sweep(2);
        const auto c2 = strips.sweep(2);
        REQUIRE(c1.attempts == c2.attempts && c1.successes == c2.successes);
#ifdef LF_WITH_REFERENCE
        lf::SlopeField f1(Ls), f2(Ls);
#else
        SlopeField f1(Ls), f2(Ls);
#endif
        one_gpu.download(f1);
        strips.download(f2);
        REQUIRE(std::memcmp(f1.words_x(), f2.words_x(), size_t(Ls) * Ls / 8) == 0);
        REQUIRE(std::memcmp(f1.words_y(), f2.words_y(), size_t(Ls) * Ls / 8) == 0);
        REQUIRE(one_gpu.interface_width() == strips.interface_width());
        std::printf("sharded OK: 2 strips == 1 lattice, successes=%lld\n", (long long)c2.successes);
    }
    {   // configs[4] through the C++ API: a KMC lattice on 1 GPU and as 2 z-slabs
        const int32_t Lk = 128;
        lf::gpu::DtrPlan two;
        two.devices = {0, 0};
        lf::gpu::KmcDevice one_gpu(Lk, 1.5, true, 77), slabs(Lk, 1.5, true, 77, two);
        REQUIRE(slabs.sharded() && !one_gpu.sharded());
        one_gpu.make_random_alloy(0.5, 5);
        slabs.make_random_alloy(0.5, 5);
        const auto k1 = one_gpu.sweep(2);
        const auto k2 = slabs.sweep(2);
        REQUIRE(k1.attempts == k2.attempts && k1.successes == k2.successes);
        REQUIRE(one_gpu.open_bonds_per_particle() == slabs.open_bonds_per_particle());
        std::printf("sharded KMC OK: 2 slabs == 1 lattice, exchanges=%lld\n", (long long)k2.successes);
    }
    std::printf("dropin OK: KPZ W2=%.6f successes=%lld; KMC exchanges=%lld\n", w2, (long long)c.successes,
                (long long)kc.successes);
    return 0;
}

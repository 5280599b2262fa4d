// dropin/lf_gpu_link.cpp -- link-level drop-in for the reference's hot path.
//
// Compile this file INSTEAD of the reference's proj/src/kpz.cpp and
// proj/src/kmc.cpp (keep lattice.cpp, rng.cpp and the rest) and link
// liblfg.so: every call the reference's users spell
//     lf::kpz_sweep_sequential(f, params, rng, sweeps)     (kpz.hpp:119-120)
//     lf::reconstruct_heights(f)                           (kpz.hpp:125)
//     lf::interface_width(h) / lf::interface_width(f)      (kpz.hpp:128-131)
//     lf::kmc_mcs_sequential(lat, params, rng, steps)      (kmc.hpp:128-129)
//     lf::open_bonds_per_particle(lat)                     (kmc.hpp:133)
// then runs on the B200 through the C ABI (include/lfg.h, lfg_kmc.h) with the
// reference's signatures, exception types and messages -- no source change at
// the call sites.  The sweeps are the two-layer DTr / DT schedules (DESIGN.md
// §2): trajectories differ from the serial LCG sweep, statistics agree; the
// device key is drawn from the caller's RngStream (two next_u32() per call),
// so the stream advances per call as the reference's does.  The DT
// decomposition needs L >= 64 (KPZ) / two 16^3 blocks per axis (KMC); smaller
// lattices raise std::invalid_argument from the sweep (the readouts accept
// every L the reference accepts).
#include "lf/kmc.hpp"
#include "lf/kpz.hpp"
#include "lf_gpu.hpp"

namespace lf {

Counters kpz_sweep_sequential(SlopeField& f, const KpzParams& params, RngStream& rng, int sweeps) {
    params.validate();  // kpz.cpp:7
    const gpu::Counters c = gpu::kpz_sweep(f, params, rng, sweeps);
    Counters out;
    out.attempts = c.attempts;
    out.successes = c.successes;
    return out;
}

HeightField reconstruct_heights(const SlopeField& f) {
    HeightField out;
    out.size = f.size();
    out.h = gpu::reconstruct_heights(f);
    return out;
}

double interface_width(const HeightField& hf) {  // kpz.cpp:51-60
    std::int64_t s = 0, s2 = 0;
    gpu::check(lfg_heights_width_sums_host(0, hf.h.data(), hf.h.size(), &s, &s2));
    const double n = static_cast<double>(hf.h.size());
    const double mean = static_cast<double>(s) / n;
    return static_cast<double>(s2) / n - mean * mean;
}

double interface_width(const SlopeField& f) { return gpu::interface_width(f); }

Counters kmc_mcs_sequential(OccupancyLattice& lat, const KmcParams& params, RngStream& rng, int steps) {
    params.validate();  // kmc.cpp:7
    const gpu::Counters c = gpu::kmc_mcs(lat, params, rng, steps);
    Counters out;
    out.attempts = c.attempts;
    out.successes = c.successes;
    return out;
}

double open_bonds_per_particle(const OccupancyLattice& lat) { return gpu::open_bonds_per_particle(lat); }

}  // namespace lf

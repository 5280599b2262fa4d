// scripts/explore/kmc_probe.cpp -- RESEARCH TOOL (CPU), not product, not oracle.
//
// Ensemble probe of KMC decomposition variants against random-sequential
// updating, both through the oracle's restated kmc_attempt_impl
// (oracle/oracle.cpp; pinned to the reference).  Observable: open bonds per
// particle (kmc.cpp:20-40) at t = 1, 2, 5, 10, 20, 50, 100 MCS.  Variants:
//   seq      kmc_mcs_sequential restated (lcg64 stream per realization)
//   dt       the device's two-layer DT (oracle_core.hpp kmc_dt_sweep)
//   dtp      dt + per-tile Poisson attempt counts (264 rounds, K ~ Poisson(1/4),
//            32 rounds skipped per K in 8-group units)
//   sub4p    four sub-sweeps per MCS (64 + 4 rounds), K ~ Poisson(1/4), 16 rounds
//            per K (the KPZ sub = 4 construction)
//
// Build: g++ -O2 -std=c++17 -pthread -I oracle scripts/explore/kmc_probe.cpp -o /tmp/kmc_probe
// Run:   /tmp/kmc_probe VARIANT NREAL BOTH > out.json
#include "oracle.cpp"  // restated attempt, sequential sweep, open-bond sums (test infrastructure)

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

uint32_t skipK16(uint32_t v) {  // Poisson(1/4), P(K >= k) = {14497, 1735, 143, 9}/2^16: E = Var = 1/4
    return uint32_t(v >= 65536u - 14497u) + uint32_t(v >= 65536u - 1735u) + uint32_t(v >= 65536u - 143u) +
           uint32_t(v >= 65536u - 9u);
}

// One sub-sweep of the two-layer DT with `rounds` rounds per activation; when
// skip_unit > 0 every tile draws K and sits out K * skip_unit rounds (spread).
template <class Attempt>
int64_t dt_sweep(const orc::KmcPlan& pl, uint64_t seed, uint64_t sweep, int rounds, int skip_unit, Attempt&& attempt) {
    const orc::KmcSweepDraw d = orc::kmc_sweep_draw(pl, seed, sweep);
    const int32_t L = pl.L, mask = L - 1;
    const int32_t nb = L / pl.bk, tb = pl.bk / orc::kKmcTile, tl = L / orc::kKmcTile;
    int64_t succ = 0;
    for (int k = 0; k < 8; ++k) {
        const int set = d.perm[k];
        const int sx = set & 1, sy = (set >> 1) & 1, sz = set >> 2;
        for (int32_t bzi = sz; bzi < nb; bzi += 2)
            for (int32_t byi = sy; byi < nb; byi += 2)
                for (int32_t bxi = sx; bxi < nb; bxi += 2) {
                    const uint32_t block_id = (uint32_t(bzi) * uint32_t(nb) + uint32_t(byi)) * uint32_t(nb) + uint32_t(bxi);
                    const int ntile = tb * tb * tb;
                    std::vector<int> skipn(size_t(ntile), 0);
                    for (int t = 0; t < ntile; ++t) {
                        if (skip_unit <= 0) break;
                        const int tx = t % tb, ty = (t / tb) % tb, tz = t / (tb * tb);
                        const uint32_t tile_id = (uint32_t(bzi * tb + tz) * uint32_t(tl) + uint32_t(byi * tb + ty)) *
                                                     uint32_t(tl) + uint32_t(bxi * tb + tx);
                        uint32_t w[4];
                        orc::draw(seed, sweep, 10u, tile_id, 0u, w);
                        skipn[size_t(t)] = int(skipK16(w[0] >> 16)) * skip_unit;
                    }
                    uint32_t sw[4] = {0, 0, 0, 0};
                    for (int r = 0; r < rounds; ++r) {
                        if ((r & 31) == 0) orc::draw(seed, sweep, orc::TAG_KMC_SET, block_id, uint32_t(r >> 5), sw);
                        const int inner = int((sw[(r >> 3) & 3] >> (4 * (r & 7))) & 7u);
                        const int hx = inner & 1, hy = (inner >> 1) & 1, hz = inner >> 2;
                        for (int t = 0; t < ntile; ++t) {
                            const int sk = skipn[size_t(t)];
                            if (sk > 0 && (int64_t(r + 1) * sk / rounds != int64_t(r) * sk / rounds)) continue;
                            const int tx = t % tb, ty = (t / tb) % tb, tz = t / (tb * tb);
                            const int32_t gx = bxi * tb + tx, gy = byi * tb + ty, gz = bzi * tb + tz;
                            const uint32_t tile_id = (uint32_t(gz) * uint32_t(tl) + uint32_t(gy)) * uint32_t(tl) + uint32_t(gx);
                            uint32_t w[4];
                            orc::draw(seed, sweep, orc::TAG_KMC_SITE, tile_id, uint32_t(r >> 1), w);
                            const bool odd = (r & 1) != 0;
                            const uint32_t s5 = odd ? (w[0] >> 5) & 31u : w[0] & 31u;
                            const uint32_t dword = odd ? (w[0] & ~1023u) : w[1];
                            const uint32_t aword = odd ? w[3] : w[2];
                            const int32_t x0 = d.ox + orc::kKmcTile * gx + orc::kKmcDom * hx;
                            const int32_t y0 = d.oy + orc::kKmcTile * gy + orc::kKmcDom * hy;
                            const int32_t z0 = d.oz + orc::kKmcTile * gz + orc::kKmcDom * hz;
                            const int32_t x = (x0 + int32_t(s5 & 3u)) & mask;
                            const int32_t y = (y0 + int32_t((s5 >> 2) & 3u)) & mask;
                            const int32_t tt = (x ^ y) & 1;
                            const int32_t zfirst = z0 + (((z0 & 1) == tt) ? 0 : 1);
                            const int32_t z = (zfirst + 2 * int32_t((s5 >> 4) & 1u)) & mask;
                            succ += attempt(x, y, z, dword, aword) == 0;
                        }
                    }
                }
    }
    return succ;
}

}  // namespace

int main(int argc, char** argv) {
    const std::string var = argc > 1 ? argv[1] : "dt";
    const int nreal = argc > 2 ? std::atoi(argv[2]) : 64;
    const int both = argc > 3 ? std::atoi(argv[3]) : 1;
    const int L = 64, bk = 16;
    const double eps = 1.5, c = 0.5;
    const int ts[] = {1, 2, 5, 10, 20, 50, 100};
    const int nt = 7;
    std::vector<double> ob(size_t(nreal) * nt);
    const int nth = int(std::thread::hardware_concurrency());
    std::vector<std::thread> pool;
    for (int th = 0; th < nth; ++th)
        pool.emplace_back([&, th] {
            std::vector<uint64_t> w(size_t(L) * L * L / 64);
            for (int rr = th; rr < nreal; rr += nth) {
                uint64_t st = 0;
                orc_kmc_random_alloy(L, c, LCG64, 1000 + uint64_t(rr), 0, w.data(), &st);
                const uint64_t seed = 0x9E3779B97F4A7C15ull * uint64_t(rr + 1);
                int t = 0;
                for (int i = 0; i < nt; ++i) {
                    for (; t < ts[i]; ++t) {
                        auto att = [&](int32_t x, int32_t y, int32_t z, uint32_t dw, uint32_t aw) {
                            const int32_t site[3] = {x, y, z};
                            return kmc_attempt(w.data(), L, site, eps, both, [&] { return orc::below(dw, 12); },
                                               [&] { return aw * 0x1p-32; });
                        };
                        const orc::KmcPlan pl{L, bk};
                        if (var == "seq") {
                            int64_t cnt[2] = {0, 0};
                            orc_kmc_sweep_sequential(L, w.data(), eps, both, LCG64, &st, 1, cnt);
                        } else if (var == "dt") {
                            dt_sweep(pl, seed, uint64_t(t), 256, 0, att);
                        } else if (var == "dtp") {
                            dt_sweep(pl, seed, uint64_t(t), 264, 32, att);
                        } else if (var == "sub4p") {
                            for (int k = 0; k < 4; ++k) dt_sweep(pl, seed, uint64_t(t) * 4 + uint64_t(k), 68, 16, att);
                        } else if (var == "sub4") {
                            for (int k = 0; k < 4; ++k) dt_sweep(pl, seed, uint64_t(t) * 4 + uint64_t(k), 64, 0, att);
                        }
                    }
                    int64_t np = 0, no = 0;
                    orc_kmc_open_bond_sums(L, w.data(), &np, &no);
                    ob[size_t(rr) * nt + i] = double(no) / double(np);
                }
            }
        });
    for (auto& p : pool) p.join();
    std::printf("{\"variant\": \"%s\", \"both\": %d, \"nreal\": %d, \"t\": [1,2,5,10,20,50,100], \"mean\": [", var.c_str(),
                both, nreal);
    for (int i = 0; i < nt; ++i) {
        double m = 0;
        for (int r = 0; r < nreal; ++r) m += ob[size_t(r) * nt + i];
        std::printf("%s%.9f", i ? ", " : "", m / nreal);
    }
    std::printf("], \"se\": [");
    for (int i = 0; i < nt; ++i) {
        double m = 0, m2 = 0;
        for (int r = 0; r < nreal; ++r) {
            m += ob[size_t(r) * nt + i];
            m2 += ob[size_t(r) * nt + i] * ob[size_t(r) * nt + i];
        }
        m /= nreal;
        std::printf("%s%.9f", i ? ", " : "", std::sqrt(std::max(0.0, (m2 / nreal - m * m) / (nreal - 1))));
    }
    std::printf("]}\n");
    return 0;
}

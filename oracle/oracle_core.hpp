// oracle/oracle_core.hpp -- TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the schedule that the B200 path executes, used as the
// checker by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg.
// Nothing in the product package (paper_1204_5072_b200/) includes or links
// this file; the product fails loudly when its CUDA library is missing.
//
// What lives here:
//   * Philox4x32-10 (Salmon et al., SC'11; Random123 constants).  The
//     reference has no counter-based RNG (rng.hpp:10 lists lcg32/lcg64/tinymt
//     only), so this generator is pinned against the published Random123
//     known-answer vectors in tests/golden/philox_kat.json.
//   * The two-layer DT / DTr schedule for KPZ.  The
//     reference has no decomposition driver; the schedule follows the prose of
//     SPEC.md:341-358 (single-hit rounds, set re-drawn with replacement,
//     SPEC.md:398; exact L^2 accounting) nested inside the
//     paper's two-layer device structure, with a random
//     tiling origin drawn every sweep (the SPEC.md:386 "origin re-draw after
//     every sweep" analogue).  The per-attempt update is supplied by the
//     caller as a functor, so the same driver runs
//       - the reference's own lf::detail::kpz_attempt_impl<false>
//         (kpz.hpp:71-107) in oracle/ref_shim.cpp, and
//       - the plain-C++ restatement in oracle/oracle.cpp.
//   * The two-layer DT schedule for KMC (KMC-6): eight block sets, inner
//     single-hit rounds over 4^3 domains.
//
// The exact key/counter layout below is the contract shared with the CUDA
// kernels; it is restated, not shared, so a
// mismatch between the two shows up as a parity failure.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstddef>
#include <cstdlib>
#include <thread>
#include <vector>

namespace orc {

// ---------------------------------------------------------------- Philox4x32-10
inline void philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                          uint32_t k0, uint32_t k1, uint32_t out[4]) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
    for (int r = 0; r < 10; ++r) {
        const uint64_t p0 = uint64_t{M0} * c0;
        const uint64_t p1 = uint64_t{M1} * c2;
        const uint32_t hi0 = uint32_t(p0 >> 32), lo0 = uint32_t(p0);
        const uint32_t hi1 = uint32_t(p1 >> 32), lo1 = uint32_t(p1);
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += W0; k1 += W1;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

// Stream tags (counter word 3, bits 24..31).
enum : uint32_t { TAG_SWEEP = 1, TAG_SET = 2, TAG_ANCHOR = 3, TAG_ACCEPT = 4,
                  TAG_KMC_SWEEP = 5, TAG_KMC_SET = 6, TAG_KMC_SITE = 7,
                  TAG_KMC_ACCEPT = 8, TAG_KMC_INIT = 9 };

// Draw 4 words for (seed, sweep, tag, c0, c1).
inline void draw(uint64_t seed, uint64_t sweep, uint32_t tag, uint32_t c0, uint32_t c1,
                 uint32_t out[4]) {
    philox4x32_10(c0, c1, uint32_t(sweep), (tag << 24) | (uint32_t(sweep >> 32) & 0xFFFFFFu),
                  uint32_t(seed), uint32_t(seed >> 32), out);
}

// Multiply-shift bounded draw, the semantics of RngStream::next_below (rng.hpp:130-134).
inline uint32_t below(uint32_t u, uint32_t bound) {
    return uint32_t((uint64_t{u} * bound) >> 32);
}

// Lexicographic permutation number idx (0..23) of {0,1,2,3}.
inline void perm4(uint32_t idx, int out[4]) {
    int pool[4] = {0, 1, 2, 3};
    int n = 4;
    const uint32_t fact[4] = {6, 2, 1, 1};
    for (int k = 0; k < 4; ++k) {
        const uint32_t d = idx / fact[k];
        idx %= fact[k];
        out[k] = pool[d];
        for (int m = int(d); m < n - 1; ++m) pool[m] = pool[m + 1];
        --n;
    }
}

// ---------------------------------------------------------------- threads
// parallel_rows(n, body): body(row, slot) for row = 0..n-1 on a pool of
// std::threads (dynamic row claiming; the image has no OpenMP runtime).  Each
// thread accumulates into its own Counts slot, summed after the join.  Thread
// count: ORC_THREADS, else hardware_concurrency().
struct Counts {
    int64_t dep = 0, det = 0, att = 0;
};

inline int oracle_threads() {
    if (const char* e = std::getenv("ORC_THREADS")) {
        const int n = std::atoi(e);
        if (n > 0) return n;
    }
    const unsigned h = std::thread::hardware_concurrency();
    return h ? int(h) : 1;
}

template <class Body>
Counts parallel_rows(int32_t n, bool allow, Body&& body) {
    const int nt = allow ? std::min<int>(oracle_threads(), n) : 1;
    if (nt <= 1) {
        Counts c;
        for (int32_t r = 0; r < n; ++r) body(r, c);
        return c;
    }
    std::atomic<int32_t> next{0};
    std::vector<Counts> part(static_cast<size_t>(nt));
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            for (int32_t r; (r = next.fetch_add(1)) < n;) body(r, part[size_t(t)]);
        });
    for (auto& th : pool) th.join();
    Counts c;
    for (const auto& p : part) {
        c.dep += p.dep;
        c.det += p.det;
        c.att += p.att;
    }
    return c;
}

// ---------------------------------------------------------------- KPZ DTr plan
// Inner geometry is fixed: domains 16 (x) x 8 (y) sites, tiles 32 x 16 (one
// 32-bit word per tile row), four inner sets (hx, hy).
//
// One MCS = `sub` sub-sweeps (1, 4 or 8).  Sub-sweep s' (global
// counter s' = s * sub + k) draws its own origin and block-set order; each
// block activation runs kpz_rounds(sub) single-hit rounds:
//   sub = 1: 512 rounds, every tile attempts once per round;
//   sub = 4: 132 rounds; tile t draws K_t from the 16 spare bits of its first
//            anchor word batch (low bytes of words 2, 3) with P(K >= k) =
//            {7701, 471, 19, 1} / 2^16 and skips the 4-round groups g < 32 whose
//            bit is set in the mask nibble {0, 8, A, E, F}[K_t] repeated, i.e.
//            N_t = 132 - 32 K_t attempts: mean 128, variance 128 (the Poisson
//            count of a 512-site tile over a quarter MCS of kpz.cpp:5-19);
//   sub = 8: 68 rounds; P(K >= k) = {14497, 1735, 143, 9} / 2^16 from the same
//            bits, the nibble repeated over the 4-round groups g < 16, i.e.
//            N_t = 68 - 16 K_t attempts: mean 64, variance 64 (an eighth MCS).
// The x origin is a multiple of 128 sites (32 when bx < 64).
constexpr int kTileW = 32, kTileH = 16, kDomW = 16, kDomH = 8, kRounds = 512;

inline int kpz_rounds(int sub) { return sub == 8 ? 68 : (sub == 4 ? 132 : 512); }

inline uint32_t kpz_skip_mask_for(uint32_t v16, int sub) {
    static const uint32_t t4[4] = {65536u - 7701u, 65536u - 471u, 65536u - 19u, 65536u - 1u};
    static const uint32_t t8[4] = {65536u - 14497u, 65536u - 1735u, 65536u - 143u, 65536u - 9u};
    const uint32_t* t = sub == 8 ? t8 : t4;
    uint32_t k = 0;
    for (int i = 0; i < 4; ++i) k += v16 >= t[i] ? 1u : 0u;
    static const uint32_t nib[5] = {0x0u, 0x8u, 0xAu, 0xEu, 0xFu};
    return nib[k] * (sub == 8 ? 0x1111u : 0x11111111u);
}

struct KpzPlan {
    int32_t L = 0;
    int32_t bx = 0;  // device block width  (multiple of 32, L % (2 bx) == 0)
    int32_t by = 0;  // device block height (multiple of 16, L % (2 by) == 0)
    int32_t sub = 1; // sub-sweeps per MCS (1, 4 or 8)
};

struct KpzSweepDraw {
    int32_t ox, oy;
    int perm[4];
};

inline KpzSweepDraw kpz_sweep_draw(const KpzPlan& pl, uint64_t seed, uint64_t sweep) {
    uint32_t w[4];
    draw(seed, sweep, TAG_SWEEP, 0, 0, w);
    KpzSweepDraw d;
    const int32_t qx = pl.bx >= 64 ? 128 : 32;
    d.ox = qx * int32_t(below(w[0], uint32_t(2 * pl.bx / qx)));
    d.oy = int32_t(below(w[1], uint32_t(2 * pl.by)));
    perm4(below(w[2], 24), d.perm);
    return d;
}

// Outcome codes returned by the attempt functors (kpz_attempt_impl's
// KpzOutcome, kpz.hpp:31; KMC: 0 = exchanged, anything else = rejected).
enum : int { OUT_DEPOSIT = 0, OUT_DETACH = 1, OUT_REJECT = 2 };

// One DTr sub-sweep with global sub-sweep counter `sweep`.  attempt(i, j,
// tile_id, round) performs one KPZ attempt at anchor (i, j) and returns its
// outcome code; the callee derives the acceptance word from (tile_id, round)
// via accept_word() when -- and only when -- a pattern matches, mirroring the
// reference's lazy get_r() (kpz.hpp:87-95).
//
// Parallel execution (parallel_rows): the active blocks of one phase are one block
// apart, so their attempts touch disjoint sites (reach +1 < the block gap) and
// the lattice after the phase does not depend on the order in which blocks run.
// Block ROWS are distributed over threads: every block row owns whole lattice
// rows (rows are L bits = whole 64-bit words for L >= 64), so no two threads
// ever read-modify-write the same word.  Blocks within a row run in order on
// one thread (neighbouring blocks of a row may share a word at bx = 32).
template <class Attempt>
Counts kpz_dtr_sweep(const KpzPlan& pl, uint64_t seed, uint64_t sweep, Attempt&& attempt) {
    const int32_t L = pl.L, mask = L - 1;
    const KpzSweepDraw d = kpz_sweep_draw(pl, seed, sweep);
    const int32_t nbx = L / pl.bx, nby = L / pl.by;
    const int32_t twx = pl.bx / kTileW, thy = pl.by / kTileH;   // tiles per block
    const int32_t tiles_per_row = L / kTileW;
    const int ntiles = twx * thy;
    const int rounds = kpz_rounds(pl.sub);
    const bool skip = pl.sub != 1;
    Counts tot;
    for (int k = 0; k < 4; ++k) {
        const int set = d.perm[k];
        const int sx = set & 1, sy = set >> 1;
        const int32_t nrows = (nby - sy + 1) / 2;
        const Counts c = parallel_rows(nrows, L >= 64, [&](int32_t row, Counts& acc) {
            const int32_t byi = sy + 2 * row;
            uint32_t* anc = new uint32_t[size_t(ntiles) * 4];
            uint32_t* smask = new uint32_t[size_t(ntiles)];
            for (int32_t bxi = sx; bxi < nbx; bxi += 2) {
                const uint32_t block_id = uint32_t(byi) * uint32_t(nbx) + uint32_t(bxi);
                uint32_t sw[4] = {0, 0, 0, 0};
                for (int r = 0; r < rounds; ++r) {
                    if ((r & 63) == 0) draw(seed, sweep, TAG_SET, block_id, uint32_t(r >> 6), sw);
                    const int inner = int((sw[(r >> 4) & 3] >> (2 * (r & 15))) & 3u);
                    const int hx = inner & 1, hy = inner >> 1;
                    for (int32_t ty = 0; ty < thy; ++ty) {
                        for (int32_t tx = 0; tx < twx; ++tx) {
                            const int32_t gx = bxi * twx + tx, gy = byi * thy + ty;
                            const uint32_t tile_id = uint32_t(gy) * uint32_t(tiles_per_row) + uint32_t(gx);
                            const size_t t = size_t(ty * twx + tx);
                            uint32_t* a4 = anc + t * 4;
                            if ((r & 15) == 0) draw(seed, sweep, TAG_ANCHOR, tile_id, uint32_t(r >> 4), a4);
                            if (r == 0)
                                smask[t] = skip ? kpz_skip_mask_for((a4[2] & 0xFFu) | ((a4[3] & 0xFFu) << 8), pl.sub) : 0u;
                            if (r < 128 && ((smask[t] >> (r >> 2)) & 1u)) continue;  // skipped group
                            // Anchor of round r (k = r & 15 within its 16-round batch), fields
                            // consumed from the TOP of each Philox word (h = k >> 3, k' = k & 7):
                            //   xd = bits [28-4k', +4) of word h      (words 0, 1)
                            //   yd = bits [29-3k', +3) of word 2 + h  (words 2, 3; low 8 bits unused)
                            const int kb = r & 15, h = kb >> 3, kk = kb & 7;
                            const int32_t xd = int32_t((a4[h] >> (28 - 4 * kk)) & 15u);
                            const int32_t yd = int32_t((a4[2 + h] >> (29 - 3 * kk)) & 7u);
                            const int32_t i = (d.ox + kTileW * gx + kDomW * hx + xd) & mask;
                            const int32_t j = (d.oy + kTileH * gy + kDomH * hy + yd) & mask;
                            const int o = attempt(i, j, tile_id, r);
                            acc.dep += o == OUT_DEPOSIT;
                            acc.det += o == OUT_DETACH;
                            acc.att += 1;
                        }
                    }
                }
            }
            delete[] anc;
            delete[] smask;
        });
        tot.dep += c.dep;
        tot.det += c.det;
        tot.att += c.att;
    }
    return tot;
}

inline uint32_t kpz_accept_word(uint64_t seed, uint64_t sweep, uint32_t tile_id, int round) {
    uint32_t w[4];
    draw(seed, sweep, TAG_ACCEPT, tile_id, uint32_t(round >> 2), w);
    return w[round & 3];
}

// ---------------------------------------------------------------- KMC DT plan
// Device blocks of bk^3 sc sites (eight block sets), inner single-hit rounds
// over 4^3 domains in 8^3 tiles (eight inner sets), 256 rounds per block
// activation (= 8 sets x 32 valid fcc sites per domain).  Reach: read 2,
// write 1 (kmc.hpp:140-141); the one-domain gap (4 sites) keeps concurrent
// attempts disjoint.
constexpr int kKmcTile = 8, kKmcDom = 4, kKmcRounds = 256;

struct KmcPlan {
    int32_t L = 0;
    int32_t bk = 0;  // device block edge (multiple of 8, L % (2 bk) == 0)
    int32_t sub = 1; // sub-sweeps per MCS (1 or 4): kKmcRounds / sub rounds per activation
};

struct KmcSweepDraw {
    int32_t ox, oy, oz;
    int perm[8];
};

inline void perm8(uint32_t idx, int out[8]) {
    int pool[8] = {0, 1, 2, 3, 4, 5, 6, 7};
    int n = 8;
    uint32_t fact[8] = {5040, 720, 120, 24, 6, 2, 1, 1};
    for (int k = 0; k < 8; ++k) {
        const uint32_t d = idx / fact[k];
        idx %= fact[k];
        out[k] = pool[d];
        for (int m = int(d); m < n - 1; ++m) pool[m] = pool[m + 1];
        --n;
    }
}

inline KmcSweepDraw kmc_sweep_draw(const KmcPlan& pl, uint64_t seed, uint64_t sweep) {
    uint32_t w[4];
    draw(seed, sweep, TAG_KMC_SWEEP, 0, 0, w);
    KmcSweepDraw d;
    d.ox = int32_t(below(w[0], uint32_t(2 * pl.bk)));
    d.oy = int32_t(below(w[1], uint32_t(2 * pl.bk)));
    d.oz = int32_t(below(w[2], uint32_t(2 * pl.bk)));
    perm8(below(w[3], 40320), d.perm);
    return d;
}

// One phase k (0..7) of a KMC DT sweep, restricted to block z-rows
// [bz_lo, bz_hi) of the shifted frame (the whole lattice: 0, L/bk -- the
// z-slab driver runs each rank's rows).  attempt(x, y, z, dir_word,
// accept_word) performs one exchange attempt at the fcc-valid site (x, y, z)
// and returns 0 when the pair was exchanged.  The site draw follows
// KmcKernel::draw_site (kmc.hpp:154-171) over the domain box: x and y
// uniform, z uniform over the parity-matched planes.  Returns the number of
// exchanges.
//
// Parallel execution (parallel_rows) over the (z, y) block rows of the phase: active
// blocks are one block apart and the attempt reaches 2 sites (read) / 1 site
// (write), so concurrent block rows touch disjoint x-rows of the lattice, which
// are whole 64-bit words for L >= 64.  Blocks along x run in order on one thread.
template <class Attempt>
int64_t kmc_dt_phase(const KmcPlan& pl, const KmcSweepDraw& d, uint64_t seed, uint64_t sweep, int k, int32_t bz_lo,
                     int32_t bz_hi, Attempt&& attempt) {
    const int32_t L = pl.L, mask = L - 1;
    const int32_t nb = L / pl.bk, tb = pl.bk / kKmcTile, tl = L / kKmcTile;
    const int set = d.perm[k];
    const int sx = set & 1, sy = (set >> 1) & 1, sz = set >> 2;
    const int32_t nh = (nb - sy + 1) / 2;            // active block rows along y
    const int32_t nrows = ((nb - sz + 1) / 2) * nh;  // (z, y) block rows
    const Counts c = parallel_rows(nrows, L >= 64, [&](int32_t row, Counts& acc) {
        const int32_t bzi = sz + 2 * (row / nh), byi = sy + 2 * (row % nh);
        if (bzi < bz_lo || bzi >= bz_hi) return;
        for (int32_t bxi = sx; bxi < nb; bxi += 2) {
            const uint32_t block_id = (uint32_t(bzi) * uint32_t(nb) + uint32_t(byi)) * uint32_t(nb) + uint32_t(bxi);
            uint32_t sw[4] = {0, 0, 0, 0};
            for (int r = 0; r < kKmcRounds / pl.sub; ++r) {
                if ((r & 31) == 0) draw(seed, sweep, TAG_KMC_SET, block_id, uint32_t(r >> 5), sw);
                const int inner = int((sw[(r >> 3) & 3] >> (4 * (r & 7))) & 7u);
                const int hx = inner & 1, hy = (inner >> 1) & 1, hz = inner >> 2;
                for (int32_t tz = 0; tz < tb; ++tz)
                for (int32_t ty = 0; ty < tb; ++ty)
                for (int32_t tx = 0; tx < tb; ++tx) {
                    const int32_t gx = bxi * tb + tx, gy = byi * tb + ty, gz = bzi * tb + tz;
                    const uint32_t tile_id = (uint32_t(gz) * uint32_t(tl) + uint32_t(gy)) * uint32_t(tl) + uint32_t(gx);
                    // One Philox draw serves the tile's rounds 2m and 2m + 1:
                    //   even: site bits W0[0..5), direction word W1, acceptance word W2
                    //   odd:  site bits W0[5..10), direction from W0[10..32) (22 bits;
                    //         below(W0 & ~1023, 12) = floor(W0[10..32) * 12 / 2^22)),
                    //         acceptance word W3
                    uint32_t w[4];
                    draw(seed, sweep, TAG_KMC_SITE, tile_id, uint32_t(r >> 1), w);
                    const bool odd = (r & 1) != 0;
                    const uint32_t s5 = odd ? (w[0] >> 5) & 31u : w[0] & 31u;
                    const uint32_t dword = odd ? (w[0] & ~1023u) : w[1];
                    const uint32_t aword = odd ? w[3] : w[2];
                    const int32_t x0 = d.ox + kKmcTile * gx + kKmcDom * hx;
                    const int32_t y0 = d.oy + kKmcTile * gy + kKmcDom * hy;
                    const int32_t z0 = d.oz + kKmcTile * gz + kKmcDom * hz;
                    const int32_t x = (x0 + int32_t(s5 & 3u)) & mask;
                    const int32_t y = (y0 + int32_t((s5 >> 2) & 3u)) & mask;
                    const int32_t t = (x ^ y) & 1;
                    const int32_t zfirst = z0 + (((z0 & 1) == t) ? 0 : 1);
                    const int32_t z = (zfirst + 2 * int32_t((s5 >> 4) & 1u)) & mask;
                    acc.dep += attempt(x, y, z, dword, aword) == 0;
                }
            }
        }
    });
    return c.dep;
}

// One KMC DT sweep: the eight phases in the sweep's drawn order.
template <class Attempt>
int64_t kmc_dt_sweep(const KmcPlan& pl, uint64_t seed, uint64_t sweep, Attempt&& attempt) {
    const KmcSweepDraw d = kmc_sweep_draw(pl, seed, sweep);
    int64_t succ = 0;
    for (int k = 0; k < 8; ++k) succ += kmc_dt_phase(pl, d, seed, sweep, k, 0, pl.L / pl.bk, attempt);
    return succ;
}

}  // namespace orc

// lfg_common.cuh -- shared device/host helpers for the B200 lattice kernels.
//
// Philox4x32-10 (Salmon et al., SC'11) is the counter-based generator of the
// DTr schedule.  Keys and counters are a pure function of
//   (seed, sweep index, stream tag, global tile/block id, round batch)
// and never of thread/block/launch geometry, so a result is independent of
// the grid shape and of the number of shards.  The
// reference's own generators (rng.hpp:10, lcg32/lcg64/tinymt) are serial
// recurrences and stay host-side for seeding and the CPU oracle.
#pragma once

#include <cstdint>

#if defined(__CUDACC__)
#define LFG_HD __host__ __device__ __forceinline__
#else
#define LFG_HD inline
#endif

namespace lfg {

enum : uint32_t {
    TAG_SWEEP = 1, TAG_SET = 2, TAG_ANCHOR = 3, TAG_ACCEPT = 4,
    TAG_KMC_SWEEP = 5, TAG_KMC_SET = 6, TAG_KMC_SITE = 7, TAG_KMC_ACCEPT = 8, TAG_KMC_INIT = 9
};

struct U4 {
    uint32_t x, y, z, w;
};

LFG_HD uint32_t mulhi32(uint32_t a, uint32_t b) {
#if defined(__CUDA_ARCH__)
    return __umulhi(a, b);
#else
    return uint32_t((uint64_t{a} * b) >> 32);
#endif
}

LFG_HD U4 philox4x32_10(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1) {
    constexpr uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
    constexpr uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = mulhi32(M0, c0), lo0 = M0 * c0;
        const uint32_t hi1 = mulhi32(M1, c2), lo1 = M1 * c2;
        const uint32_t n0 = hi1 ^ c1 ^ k0;
        const uint32_t n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += W0; k1 += W1;
    }
    return U4{c0, c1, c2, c3};
}

// Counter layout shared with oracle/oracle_core.hpp (restated there).
LFG_HD U4 draw(uint64_t seed, uint64_t sweep, uint32_t tag, uint32_t c0, uint32_t c1) {
    return philox4x32_10(c0, c1, uint32_t(sweep), (tag << 24) | (uint32_t(sweep >> 32) & 0xFFFFFFu),
                         uint32_t(seed), uint32_t(seed >> 32));
}

// RngStream::next_below semantics (rng.hpp:130-134): multiply-shift.
LFG_HD uint32_t below(uint32_t u, uint32_t bound) { return uint32_t((uint64_t{u} * bound) >> 32); }

// Lexicographic permutation number idx of {0..n-1}, packed `bits` per entry
// (entry k at bits [bits*k, bits*k+bits)); register-only (no local arrays).
LFG_HD uint32_t perm_packed(uint32_t idx, int n, int bits) {
    uint32_t pool = 0, fact = 1;
    for (int k = 0; k < n; ++k) pool |= uint32_t(k) << (bits * k);
    for (int k = 2; k < n; ++k) fact *= uint32_t(k);  // (n-1)!
    const uint32_t fmask = (1u << bits) - 1u;
    uint32_t out = 0;
    for (int k = 0; k < n; ++k) {
        const uint32_t d = idx / fact;
        idx %= fact;
        const int sh = bits * int(d);
        out |= ((pool >> sh) & fmask) << (bits * k);
        const uint32_t lower = pool & ((1u << sh) - 1u);
        const uint32_t upper = (sh + bits < 32) ? (pool >> (sh + bits)) : 0u;
        pool = lower | (upper << sh);
        if (n - 1 - k > 0) fact /= uint32_t(n - 1 - k);
    }
    return out;
}

// ---------------------------------------------------------------- KPZ plan
// Inner layer: 16x8 single-hit domains in 32x16 tiles (one 32-bit word per
// tile row).  One MCS = `sub` sub-sweeps (plan, 1, 4 or 8); each sub-sweep draws
// its own origin and block-set order (sweep counter s' = s * sub + k) and gives
// every block one activation of kpz_rounds(sub) single-hit rounds:
//   sub = 1: 512 rounds, every tile one attempt per round (the paper's scheme,
//            PAPER.md:366-380);
//   sub = 4: 132 rounds; tile t skips the 4-round groups g < 32 whose bit is
//            set in kpz_skip_mask(K_t), K_t ~ Poisson(1/8) from 16 spare bits of
//            its first anchor draw -> N_t = 132 - 32 K_t attempts with mean 128
//            and variance 128 exactly: the Poisson count a 512-site tile gets in
//            a quarter MCS of random-sequential updates (kpz.cpp:5-19).
//   sub = 8: 68 rounds; tile t skips the groups g < 16 whose bit is set in
//            kpz_skip_mask(K_t, 8), K_t ~ Poisson(1/4) from the same 16 bits ->
//            N_t = 68 - 16 K_t attempts with mean 64 and variance 64 (an eighth
//            of an MCS).
// DESIGN.md §2.1 / §6 (scripts/explore: why both changes are needed).
constexpr int kTileW = 32, kTileH = 16, kDomW = 16, kDomH = 8, kRounds = 512;

LFG_HD int kpz_rounds(int sub) { return sub == 8 ? 68 : (sub == 4 ? 132 : 512); }

// K from 16 uniform bits v (tails rounded so that E[K] = Var[K] hold exactly):
//   sub = 4: P(K >= k) = {7701, 471, 19, 1} / 2^16, Poisson(1/8);
//   sub = 8: P(K >= k) = {14497, 1735, 143, 9} / 2^16, Poisson(1/4).
LFG_HD uint32_t kpz_skip_k(uint32_t v16, int sub) {
    if (sub == 8)
        return uint32_t(v16 >= 51039u) + uint32_t(v16 >= 63801u) + uint32_t(v16 >= 65393u) + uint32_t(v16 >= 65527u);
    return uint32_t(v16 >= 57835u) + uint32_t(v16 >= 65065u) + uint32_t(v16 >= 65517u) + uint32_t(v16 >= 65535u);
}

// 4-round groups skipped by a tile with K: nibble {0, 8, A, E, F}[K] repeated
// over groups g < 32 (sub = 4: 8 K groups, 32 K rounds) or g < 16 (sub = 8:
// 4 K groups, 16 K rounds), spread evenly.
LFG_HD uint32_t kpz_skip_mask(uint32_t k, int sub) {
    return ((0xFEA80u >> (4u * k)) & 0xFu) * (sub == 8 ? 0x1111u : 0x11111111u);
}

// The 16 spare bits of anchor word batch 0 (the low bytes of words 2 and 3,
// which the 3-bit row fields never reach).
LFG_HD uint32_t kpz_skip_bits(uint32_t a2, uint32_t a3) { return (a2 & 0xFFu) | ((a3 & 0xFFu) << 8); }

// x-origin quantum: 128 sites (16-byte aligned rows in HBM) for bx >= 64.
LFG_HD int32_t kpz_ox_quantum(int32_t bx) { return bx >= 64 ? 128 : 32; }

struct KpzSweep {
    int32_t ox, oy;
    uint32_t perm;  // 2 bits per phase
    LFG_HD int set(int phase) const { return int((perm >> (2 * phase)) & 3u); }
};

// Draws of sub-sweep s' (the global sub-sweep counter).
LFG_HD KpzSweep kpz_sweep_draw(int32_t bx, int32_t by, uint64_t seed, uint64_t sweep) {
    const U4 w = draw(seed, sweep, TAG_SWEEP, 0, 0);
    KpzSweep s;
    const int32_t qx = kpz_ox_quantum(bx);
    s.ox = qx * int32_t(below(w.x, uint32_t(2 * bx / qx)));
    s.oy = int32_t(below(w.y, uint32_t(2 * by)));
    s.perm = perm_packed(below(w.z, 24), 4, 2);
    return s;
}

// ---------------------------------------------------------------- KMC plan
constexpr int kKmcTile = 8, kKmcDom = 4, kKmcRounds = 256;

// The attempt words of round r of a tile: one Philox draw
// W = Philox(seed; tile, r >> 1, s, TAG_KMC_SITE) serves rounds 2m and 2m + 1.
//   even: site bits W.x[0..5), direction below(W.y, 12), acceptance word W.z;
//   odd:  site bits W.x[5..10), direction below(W.x & ~1023, 12) (22 bits),
//         acceptance word W.w.
LFG_HD void kmc_round_words(const U4& W, bool odd, uint32_t& site5, uint32_t& dir, uint32_t& acc) {
    site5 = (odd ? W.x >> 5 : W.x) & 31u;
    dir = below(odd ? (W.x & ~1023u) : W.y, 12);
    acc = odd ? W.w : W.z;
}

struct KmcSweep {
    int32_t ox, oy, oz;
    uint32_t perm;  // 3 bits per phase
    LFG_HD int set(int phase) const { return int((perm >> (3 * phase)) & 7u); }
};

LFG_HD KmcSweep kmc_sweep_draw(int32_t bk, uint64_t seed, uint64_t sweep) {
    const U4 w = draw(seed, sweep, TAG_KMC_SWEEP, 0, 0);
    KmcSweep s;
    s.ox = int32_t(below(w.x, uint32_t(2 * bk)));
    s.oy = int32_t(below(w.y, uint32_t(2 * bk)));
    s.oz = int32_t(below(w.z, uint32_t(2 * bk)));
    s.perm = perm_packed(below(w.w, 40320), 8, 3);
    return s;
}

}  // namespace lfg

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
// tile row), 512 rounds per block activation.
constexpr int kTileW = 32, kTileH = 16, kDomW = 16, kDomH = 8, kRounds = 512;

struct KpzSweep {
    int32_t ox, oy;
    uint32_t perm;  // 2 bits per phase
    LFG_HD int set(int phase) const { return int((perm >> (2 * phase)) & 3u); }
};

LFG_HD KpzSweep kpz_sweep_draw(int32_t bx, int32_t by, uint64_t seed, uint64_t sweep) {
    const U4 w = draw(seed, sweep, TAG_SWEEP, 0, 0);
    KpzSweep s;
    s.ox = int32_t(below(w.x, uint32_t(2 * bx)));
    s.oy = int32_t(below(w.y, uint32_t(2 * by)));
    s.perm = perm_packed(below(w.z, 24), 4, 2);
    return s;
}

// ---------------------------------------------------------------- KMC plan
constexpr int kKmcTile = 8, kKmcDom = 4, kKmcRounds = 256;

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

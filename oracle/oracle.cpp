// oracle/oracle.cpp -- TEST INFRASTRUCTURE ONLY (see oracle_core.hpp header).
//
// Plain C++ restatement of the reference's hot path, exported with a C ABI
// (liboracle.so) so tests/ and bench.py can drive it through ctypes.  Every
// function cites the reference code it restates (paths relative to
// /root/reference/proj).  The restatement is pinned two ways:
//   * tests/test_oracle_vs_ref.py runs it bit-for-bit against the reference
//     sources compiled unmodified into oracle/_ref/liblfref.so (this container);
//   * tests/golden/*.json hold vectors produced by the reference itself
//     (tests/golden/make_golden.py), checked on every box.
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#include "oracle_core.hpp"

namespace {

// ---------------------------------------------------------------- RNG suite
// rng.hpp:10-136, rng.cpp:1-116.
enum Kind : int { LCG32 = 0, LCG64 = 1, TINYMT = 2 };

struct Stream {
    int kind = LCG64;
    uint32_t stream_id = 0;
    uint64_t lcg = 0;
    uint32_t mt[4] = {0, 0, 0, 0};
    uint32_t mat1 = 0, mat2 = 0, tmat = 0;
};

uint64_t splitmix64(uint64_t& x) {  // rng.hpp:18-23
    uint64_t z = (x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

uint64_t mix(uint64_t seed, uint64_t salt) {  // rng.hpp:25-29
    uint64_t x = seed ^ (0xA24BAED4963EE407ull * (salt + 1));
    uint64_t z = splitmix64(x);
    return z ^ splitmix64(x);
}

uint32_t tinymt_next(Stream& s) {  // rng.hpp:83-102
    uint32_t x = (s.mt[0] & 0x7FFFFFFFu) ^ s.mt[1] ^ s.mt[2];
    uint32_t y = s.mt[3];
    x ^= x << 1;
    y ^= (y >> 1) ^ x;
    s.mt[0] = s.mt[1];
    s.mt[1] = s.mt[2];
    s.mt[2] = x ^ (y << 10);
    s.mt[3] = y;
    if (y & 1u) {
        s.mt[1] ^= s.mat1;
        s.mt[2] ^= s.mat2;
    }
    uint32_t t0 = s.mt[3];
    uint32_t t1 = s.mt[0] + (s.mt[2] >> 8);
    t0 ^= t1;
    if (t1 & 1u) t0 ^= s.tmat;
    return t0;
}

void tinymt_init(Stream& s, uint64_t seed) {  // rng.cpp:35-47
    s.mt[0] = uint32_t(seed ^ (seed >> 32));
    s.mt[1] = s.mat1;
    s.mt[2] = s.mat2;
    s.mt[3] = s.tmat;
    for (unsigned i = 1; i < 8; ++i)
        s.mt[i & 3] ^= i + 1812433253u * (s.mt[(i - 1) & 3] ^ (s.mt[(i - 1) & 3] >> 30));
    if ((s.mt[0] & 0x7FFFFFFFu) == 0 && s.mt[1] == 0 && s.mt[2] == 0 && s.mt[3] == 0) {
        s.mt[0] = 'T'; s.mt[1] = 'I'; s.mt[2] = 'N'; s.mt[3] = 'Y';
    }
    for (int i = 0; i < 8; ++i) (void)tinymt_next(s);
}

Stream make_stream(int kind, uint64_t seed, uint32_t stream_id) {  // rng.cpp:49-69
    Stream s;
    s.kind = kind;
    s.stream_id = stream_id;
    if (kind == LCG32) {
        s.lcg = stream_id == 0 ? (seed & 0xFFFFFFFFull) : (mix(seed, stream_id) & 0xFFFFFFFFull);
    } else if (kind == LCG64) {
        s.lcg = seed;
    } else {
        s.mat1 = 0x8F7011EEu; s.mat2 = 0xFC78FF1Fu; s.tmat = 0x3793FDFFu;  // rng.cpp:13-15
        tinymt_init(s, stream_id == 0 ? seed : mix(seed, stream_id));
    }
    return s;
}

inline uint32_t next_u32(Stream& s) {  // rng.hpp:104-119
    if (s.kind == LCG32) {
        uint32_t x = uint32_t(s.lcg);
        x = 1664525u * x + 1013904223u;
        s.lcg = x;
        return x;
    }
    if (s.kind == LCG64) {
        s.lcg = 6364136223846793005ull * s.lcg + 1442695040888963407ull;
        return uint32_t(s.lcg >> 32);
    }
    return tinymt_next(s);
}

inline double next_real(Stream& s) { return next_u32(s) * 0x1p-32; }  // rng.hpp:126-128
inline uint32_t next_below(Stream& s, uint32_t bound) {               // rng.hpp:130-134
    return uint32_t((uint64_t{next_u32(s)} * bound) >> 32);
}

void skip(Stream& s, uint64_t n) {  // rng.cpp:71-90
    uint64_t acc_a = 1, acc_c = 0, base_a = 6364136223846793005ull, base_c = 1442695040888963407ull;
    while (n > 0) {
        if (n & 1u) {
            acc_a = base_a * acc_a;
            acc_c = base_a * acc_c + base_c;
        }
        base_c = (base_a + 1) * base_c;
        base_a = base_a * base_a;
        n >>= 1;
    }
    s.lcg = acc_a * s.lcg + acc_c;
}

// ---------------------------------------------------------------- KPZ lattice
// SlopeField layout (lattice.hpp:56-97): site idx = j*L + i, bit idx&63 of
// 64-bit word idx>>6, one plane for sigma_x and one for sigma_y.
inline bool get_bit(const uint64_t* w, int64_t idx) { return (w[idx >> 6] >> (idx & 63)) & 1u; }

inline void flip_pair(uint64_t* w, int64_t a, int64_t b) {  // kpz.hpp:48-59
    w[a >> 6] ^= uint64_t{1} << (a & 63);
    w[b >> 6] ^= uint64_t{1} << (b & 63);
}

// kpz_attempt_impl<false> (kpz.hpp:71-107).  Returns 0 deposited, 1 detached,
// 2 rejected.  get_r is invoked only when a pattern matches.
template <class R>
inline int kpz_attempt(int32_t L, uint64_t* x, uint64_t* y, int32_t i, int32_t j, double p,
                       double q, R&& get_r) {
    const int32_t mask = L - 1;
    const int32_t i1 = (i + 1) & mask, j1 = (j + 1) & mask;
    const int64_t xa = int64_t(j) * L + i, xb = int64_t(j) * L + i1;
    const int64_t ya = xa, yb = int64_t(j1) * L + i;
    const bool bx0 = get_bit(x, xa), bx1 = get_bit(x, xb);
    const bool by0 = get_bit(y, ya), by1 = get_bit(y, yb);
    int out;
    if (!bx0 && bx1 && !by0 && by1) {
        if (!(get_r() < p)) return 2;
        out = 0;
    } else if (bx0 && !bx1 && by0 && !by1) {
        if (!(get_r() < q)) return 2;
        out = 1;
    } else {
        return 2;
    }
    flip_pair(x, xa, xb);
    flip_pair(y, ya, yb);
    return out;
}

bool valid_size(int32_t L) { return L >= 4 && (L & (L - 1)) == 0; }  // lattice.cpp:10-16

}  // namespace

extern "C" {

// --------------------------------------------------------------- Philox / RNG
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
    orc::philox4x32_10(ctr[0], ctr[1], ctr[2], ctr[3], key[0], key[1], out);
}

// Fill out[n] with next_u32 draws of a fresh stream (kind, seed, stream_id).
void orc_rng_draws(int kind, uint64_t seed, uint32_t stream_id, uint64_t skip_n, uint32_t* out,
                   int64_t n) {
    Stream s = make_stream(kind, seed, stream_id);
    if (skip_n) skip(s, skip_n);
    for (int64_t k = 0; k < n; ++k) out[k] = next_u32(s);
}

uint64_t orc_lcg64_skip(uint64_t state, uint64_t n) {
    Stream s;
    s.lcg = state;
    skip(s, n);
    return s.lcg;
}

// split_streams (rng.cpp:98-114): writes the lcg state of each stream (lcg kinds).
int orc_split_streams_lcg(int kind, uint64_t seed, int count, uint64_t stride, uint64_t* states) {
    if (count < 1) return -1;
    for (int k = 0; k < count; ++k) {
        Stream s = make_stream(kind, seed, uint32_t(k));
        if (kind == LCG64) skip(s, stride * uint64_t(k));
        states[k] = s.lcg;
    }
    return 0;
}

// --------------------------------------------------------------- KPZ
// make_flat_slopes (lattice.cpp:71-82).
int orc_kpz_flat(int32_t L, uint64_t* x, uint64_t* y) {
    if (!valid_size(L)) return -1;
    const int64_t n = int64_t(L) * L, nw = (n + 63) / 64;
    std::memset(x, 0, size_t(nw) * 8);
    std::memset(y, 0, size_t(nw) * 8);
    for (int32_t j = 0; j < L; ++j)
        for (int32_t i = 0; i < L; ++i) {
            const int64_t idx = int64_t(j) * L + i;
            if ((i & 1) == 0) x[idx >> 6] |= uint64_t{1} << (idx & 63);
            if ((j & 1) == 0) y[idx >> 6] |= uint64_t{1} << (idx & 63);
        }
    return 0;
}

// interface_width(const SlopeField&) (kpz.cpp:62-81): the int64 sums before
// the double finish.
void orc_kpz_width_sums(int32_t L, const uint64_t* x, const uint64_t* y, int64_t* sum,
                        int64_t* sum2) {
    std::vector<int32_t> h(size_t(L), 0);
    for (int32_t i = 1; i < L; ++i) h[size_t(i)] = h[size_t(i - 1)] + (get_bit(x, i) ? 1 : -1);
    int64_t s = 0, s2 = 0;
    for (int32_t j = 0; j < L; ++j)
        for (int32_t i = 0; i < L; ++i) {
            int32_t& hi = h[size_t(i)];
            if (j > 0) hi += get_bit(y, int64_t(j) * L + i) ? 1 : -1;
            s += hi;
            s2 += int64_t{hi} * hi;
        }
    *sum = s;
    *sum2 = s2;
}

double orc_width_from_sums(int32_t L, int64_t sum, int64_t sum2) {  // kpz.cpp:78-80
    const double n = double(int64_t(L) * L);
    const double mean = double(sum) / n;
    return double(sum2) / n - mean * mean;
}

// reconstruct_heights (kpz.cpp:21-49).  Returns 0, or -2 on a closure violation.
int orc_kpz_reconstruct_heights(int32_t L, const uint64_t* x, const uint64_t* y, int32_t* h) {
    auto at = [&](int32_t i, int32_t j) -> int32_t& { return h[size_t(j) * size_t(L) + size_t(i)]; };
    auto sx = [&](int32_t i, int32_t j) { return get_bit(x, int64_t(j) * L + i) ? 1 : -1; };
    auto sy = [&](int32_t i, int32_t j) { return get_bit(y, int64_t(j) * L + i) ? 1 : -1; };
    at(0, 0) = 0;
    for (int32_t i = 1; i < L; ++i) at(i, 0) = at(i - 1, 0) + sx(i, 0);
    for (int32_t i = 0; i < L; ++i)
        for (int32_t j = 1; j < L; ++j) at(i, j) = at(i, j - 1) + sy(i, j);
    const int32_t mask = L - 1;
    for (int32_t j = 0; j < L; ++j)
        for (int32_t i = 0; i < L; ++i)
            if (at(i, j) - at((i - 1) & mask, j) != sx(i, j) || at(i, j) - at(i, (j - 1) & mask) != sy(i, j))
                return -2;
    return 0;
}

// closure_holds (lattice.cpp:61-69).
int orc_kpz_closure_holds(int32_t L, const uint64_t* x, const uint64_t* y) {
    for (int32_t j = 0; j < L; ++j) {
        int32_t ones = 0;
        for (int32_t i = 0; i < L; ++i) ones += get_bit(x, int64_t(j) * L + i);
        if (2 * ones - L != 0) return 0;
    }
    for (int32_t i = 0; i < L; ++i) {
        int32_t s = 0;
        for (int32_t j = 0; j < L; ++j) s += get_bit(y, int64_t(j) * L + i) ? 1 : -1;
        if (s != 0) return 0;
    }
    return 1;
}

// kpz_sweep_sequential (kpz.cpp:5-19) with a restated RngStream.  counters:
// [attempts, successes, deposits, detaches].  *state is the lcg state in/out
// (lcg kinds only).
int orc_kpz_sweep_sequential(int32_t L, uint64_t* x, uint64_t* y, double p, double q, int kind,
                             uint64_t* state, int sweeps, int64_t* counters) {
    if (!(p >= 0.0 && p <= 1.0) || !(q >= 0.0 && q <= 1.0) || p + q <= 0.0) return -1;
    Stream s;
    s.kind = kind;
    s.lcg = *state;
    if (kind == TINYMT) return -1;
    const int64_t attempts = int64_t(L) * L * sweeps;
    int64_t dep = 0, det = 0;
    for (int64_t n = 0; n < attempts; ++n) {
        const int32_t i = int32_t(next_below(s, uint32_t(L)));
        const int32_t j = int32_t(next_below(s, uint32_t(L)));
        const int o = kpz_attempt(L, x, y, i, j, p, q, [&s] { return next_real(s); });
        dep += o == 0;
        det += o == 1;
    }
    *state = s.lcg;
    counters[0] += attempts;
    counters[1] += dep + det;
    counters[2] += dep;
    counters[3] += det;
    return 0;
}

// Two-layer DTr sweeps (oracle_core.hpp) with the restated attempt: MCS
// sweep0 .. sweep0 + nsweeps - 1, each `sub` sub-sweeps (s' = s * sub + k).
int orc_kpz_sweep_dtr(int32_t L, uint64_t* x, uint64_t* y, double p, double q, uint64_t seed,
                      uint64_t sweep0, int32_t nsweeps, int32_t bx, int32_t by, int32_t sub, int64_t* counters) {
    if (!(p >= 0.0 && p <= 1.0) || !(q >= 0.0 && q <= 1.0) || p + q <= 0.0) return -1;
    if (sub != 1 && sub != 4 && sub != 8) return -1;
    orc::KpzPlan pl{L, bx, by, sub};
    int64_t dep = 0, det = 0, att = 0;
    for (int32_t s = 0; s < nsweeps; ++s) {
        for (int32_t k = 0; k < sub; ++k) {
            const uint64_t sweep = (sweep0 + uint64_t(s)) * uint64_t(sub) + uint64_t(k);
            const orc::Counts c = orc::kpz_dtr_sweep(pl, seed, sweep, [&](int32_t i, int32_t j, uint32_t tile_id, int r) {
                return kpz_attempt(L, x, y, i, j, p, q, [&] {
                    return orc::kpz_accept_word(seed, sweep, tile_id, r) * 0x1p-32;
                });
            });
            dep += c.dep;
            det += c.det;
            att += c.att;
        }
    }
    counters[0] += att;
    counters[1] += dep + det;
    counters[2] += dep;
    counters[3] += det;
    return 0;
}

// Sweep-level draws of the DTr schedule (origin and block-set order).
void orc_kpz_sweep_draw(int32_t L, int32_t bx, int32_t by, uint64_t seed, uint64_t sweep,
                        int32_t* out6) {
    orc::KpzPlan pl{L, bx, by, 1};
    const auto d = orc::kpz_sweep_draw(pl, seed, sweep);
    out6[0] = d.ox; out6[1] = d.oy;
    for (int k = 0; k < 4; ++k) out6[2 + k] = d.perm[k];
}

}  // extern "C"

// --------------------------------------------------------------- KMC
// OccupancyLattice layout (lattice.hpp:107-135): idx = (z*L + y)*L + x.
static const int kOff[12][3] = {  // kFccOffsets (lattice.hpp:147-151)
    {1, 1, 0}, {1, -1, 0}, {-1, 1, 0}, {-1, -1, 0}, {1, 0, 1}, {1, 0, -1},
    {-1, 0, 1}, {-1, 0, -1}, {0, 1, 1}, {0, 1, -1}, {0, -1, 1}, {0, -1, -1}};

static inline int64_t kidx(int32_t L, int32_t x, int32_t y, int32_t z) {
    return (int64_t(z) * L + y) * L + x;
}

extern "C" int orc_kmc_random_alloy(int32_t L, double c, int kind, uint64_t seed, uint32_t stream_id,
                         uint64_t* words, uint64_t* state_out) {
    if (!(c >= 0.0 && c <= 1.0)) return -1;
    if (!valid_size(L)) return -1;
    Stream s = make_stream(kind, seed, stream_id);
    const uint64_t threshold = uint64_t(std::llround(c * 4294967296.0));
    const int64_t nw = (int64_t(L) * L * L + 63) / 64;
    std::memset(words, 0, size_t(nw) * 8);
    for (int32_t z = 0; z < L; ++z)
        for (int32_t y = 0; y < L; ++y)
            for (int32_t x = (y ^ z) & 1; x < L; x += 2)
                if (uint64_t{next_u32(s)} < threshold) {
                    const int64_t i = kidx(L, x, y, z);
                    words[i >> 6] |= uint64_t{1} << (i & 63);
                }
    if (state_out) *state_out = s.lcg;
    return 0;
}

static inline bool occ(const uint64_t* w, int32_t L, int32_t x, int32_t y, int32_t z) {
    const int64_t i = kidx(L, x, y, z);
    return (w[i >> 6] >> (i & 63)) & 1u;
}

// b_neighbors_excluding (kmc.hpp:51-63).
static int b_nbrs_excl(const uint64_t* w, int32_t L, const int32_t p[3], const int32_t e[3]) {
    const int32_t mask = L - 1;
    int n = 0;
    for (const auto& d : kOff) {
        const int32_t x = (p[0] + d[0]) & mask, y = (p[1] + d[1]) & mask, z = (p[2] + d[2]) & mask;
        if (x == e[0] && y == e[1] && z == e[2]) continue;
        n += occ(w, L, x, y, z);
    }
    return n;
}

// metropolis_prob (kmc.hpp:33-39).
static double metropolis(int ni, int nf, double eps) {
    if (nf >= ni) return 1.0;
    return 1.0 * std::exp(-(ni - nf) * eps);
}

// kmc_attempt_impl<false> (kmc.hpp:80-112) with the draws supplied as
// callables in the reference's consumption order: dir (only if not rejected
// by species), r (only if w < 1).  Returns 0 exchanged, 1 species, 2 prob.
template <class Dir, class Real>
static int kmc_attempt(uint64_t* w, int32_t L, const int32_t site[3], double eps, int both,
                       Dir&& get_dir, Real&& get_r) {
    const int32_t mask = L - 1;
    const bool here_b = occ(w, L, site[0], site[1], site[2]);
    if (!here_b && !both) return 1;
    const auto& d = kOff[get_dir()];
    const int32_t partner[3] = {(site[0] + d[0]) & mask, (site[1] + d[1]) & mask, (site[2] + d[2]) & mask};
    const bool partner_b = occ(w, L, partner[0], partner[1], partner[2]);
    if (partner_b == here_b) return 1;
    const int32_t* b = here_b ? site : partner;
    const int32_t* a = here_b ? partner : site;
    const double pw = metropolis(b_nbrs_excl(w, L, b, a), b_nbrs_excl(w, L, a, b), eps);
    if (pw < 1.0 && !(get_r() < pw)) return 2;
    const int64_t ib = kidx(L, b[0], b[1], b[2]), ia = kidx(L, a[0], a[1], a[2]);
    w[ib >> 6] ^= uint64_t{1} << (ib & 63);
    w[ia >> 6] ^= uint64_t{1} << (ia & 63);
    return 0;
}

extern "C" {

// kmc_mcs_sequential (kmc.cpp:5-18) with a restated lcg stream.
// counters: [attempts, successes].
int orc_kmc_sweep_sequential(int32_t L, uint64_t* w, double eps, int both, int kind,
                             uint64_t* state, int steps, int64_t* counters) {
    if (!(eps >= 0.0) || kind == TINYMT) return -1;
    Stream s;
    s.kind = kind;
    s.lcg = *state;
    const int32_t mask = L - 1;
    const int64_t attempts = int64_t(L) * L * L / 2 * steps;
    int64_t succ = 0;
    for (int64_t n = 0; n < attempts; ++n) {
        // KmcKernel::draw_site with lo = 0, ext = L (kmc.hpp:154-171).
        const int32_t x = int32_t(next_below(s, uint32_t(L))) & mask;
        const int32_t y = int32_t(next_below(s, uint32_t(L))) & mask;
        const int32_t t = (x ^ y) & 1;
        const int32_t zfirst = (0 & 1) == t ? 0 : 1;
        const int32_t nz = (L + ((0 & 1) == t ? 1 : 0)) / 2;
        const int32_t z = (zfirst + 2 * int32_t(next_below(s, uint32_t(nz)))) & mask;
        const int32_t site[3] = {x, y, z};
        succ += kmc_attempt(w, L, site, eps, both, [&] { return next_below(s, 12); },
                            [&] { return next_real(s); }) == 0;
    }
    *state = s.lcg;
    counters[0] += attempts;
    counters[1] += succ;
    return 0;
}

// Two-layer DT KMC sweeps (oracle_core.hpp) with the restated attempt.
// MCS sweep0 .. sweep0 + nsweeps - 1, each `sub` sub-sweeps (s' = s * sub + k).
int orc_kmc_sweep_dt(int32_t L, uint64_t* w, double eps, int both, uint64_t seed, uint64_t sweep0,
                     int32_t nsweeps, int32_t bk, int32_t sub, int64_t* counters) {
    if (!(eps >= 0.0) || (sub != 1 && sub != 4)) return -1;
    orc::KmcPlan pl{L, bk, sub};
    int64_t succ = 0;
    for (int64_t s = 0; s < int64_t(nsweeps) * sub; ++s) {
        succ += orc::kmc_dt_sweep(pl, seed, sweep0 * uint64_t(sub) + uint64_t(s),
                                  [&](int32_t x, int32_t y, int32_t z, uint32_t dir_w, uint32_t acc_w) {
                                      const int32_t site[3] = {x, y, z};
                                      return kmc_attempt(w, L, site, eps, both,
                                                         [&] { return orc::below(dir_w, 12); },
                                                         [&] { return acc_w * 0x1p-32; });
                                  });
    }
    counters[0] += int64_t(L) * L * L / 2 * nsweeps;
    counters[1] += succ;
    return 0;
}

// One DT phase restricted to block z-rows [bz0, bz0 + nbz) (the z-slab
// driver's unit of work; tests/test_shard_kmc_cpu.py).
// One phase of sub-sweep `sweep` (s' = MCS * sub + k) on block z-rows [bz0, bz0 + nbz).
int orc_kmc_dt_phase_rows(int32_t L, uint64_t* w, double eps, int both, uint64_t seed, uint64_t sweep,
                          int32_t phase, int32_t bk, int32_t sub, int32_t bz0, int32_t nbz, int64_t* counters) {
    if (!(eps >= 0.0) || phase < 0 || phase > 7 || (sub != 1 && sub != 4)) return -1;
    orc::KmcPlan pl{L, bk, sub};
    const orc::KmcSweepDraw d = orc::kmc_sweep_draw(pl, seed, sweep);
    int64_t att = 0;
    {
        const int32_t nb = L / bk;
        const int set = d.perm[phase], sx = set & 1, sy = (set >> 1) & 1, sz = set >> 2;
        for (int32_t bzi = sz; bzi < nb; bzi += 2)
            if (bzi >= bz0 && bzi < bz0 + nbz) att += int64_t((nb - sy + 1) / 2) * ((nb - sx + 1) / 2);
        att *= int64_t(bk) * bk * bk / 2 / sub;
    }
    const int64_t succ = orc::kmc_dt_phase(pl, d, seed, sweep, phase, bz0, bz0 + nbz,
                      [&](int32_t x, int32_t y, int32_t z, uint32_t dir_w, uint32_t acc_w) {
                          const int32_t site[3] = {x, y, z};
                          return kmc_attempt(w, L, site, eps, both, [&] { return orc::below(dir_w, 12); },
                                             [&] { return acc_w * 0x1p-32; });
                      });
    counters[0] += att;
    counters[1] += succ;
    return 0;
}

// The KMC sweep draw (origin + block-set order): out[11] = ox, oy, oz, order[8].
void orc_kmc_sweep_draw(int32_t L, int32_t bk, uint64_t seed, uint64_t sweep, int32_t* out) {
    const orc::KmcSweepDraw d = orc::kmc_sweep_draw(orc::KmcPlan{L, bk}, seed, sweep);
    out[0] = d.ox;
    out[1] = d.oy;
    out[2] = d.oz;
    for (int k = 0; k < 8; ++k) out[3 + k] = d.perm[k];
}

// open_bonds_per_particle (kmc.cpp:20-40) as exact integer sums over planes
// z in [z0, z0 + nz) (mod L); z0 = 0, nz = L is the reference's readout.
void orc_kmc_open_bond_sums_planes(int32_t L, const uint64_t* w, int32_t z0, int32_t nz, int64_t* particles,
                                   int64_t* open) {
    const int32_t mask = L - 1;
    int64_t np = 0, no = 0;
    for (int32_t k = 0; k < nz; ++k) {
        const int32_t z = (z0 + k) & mask;
        for (int32_t y = 0; y < L; ++y)
            for (int32_t x = (y ^ z) & 1; x < L; x += 2) {
                if (!occ(w, L, x, y, z)) continue;
                ++np;
                for (const auto& d : kOff) no += !occ(w, L, (x + d[0]) & mask, (y + d[1]) & mask, (z + d[2]) & mask);
            }
    }
    *particles = np;
    *open = no;
}

// open_bonds_per_particle (kmc.cpp:20-40) as exact integer sums.
void orc_kmc_open_bond_sums(int32_t L, const uint64_t* w, int64_t* particles, int64_t* open) {
    const int32_t mask = L - 1;
    int64_t np = 0, no = 0;
    for (int32_t z = 0; z < L; ++z)
        for (int32_t y = 0; y < L; ++y)
            for (int32_t x = (y ^ z) & 1; x < L; x += 2) {
                if (!occ(w, L, x, y, z)) continue;
                ++np;
                for (const auto& d : kOff) no += !occ(w, L, (x + d[0]) & mask, (y + d[1]) & mask, (z + d[2]) & mask);
            }
    *particles = np;
    *open = no;
}

int64_t orc_kmc_count_b(int32_t L, const uint64_t* w) {  // lattice.cpp:97-101
    const int64_t nw = (int64_t(L) * L * L + 63) / 64;
    int64_t n = 0;
    for (int64_t k = 0; k < nw; ++k) n += __builtin_popcountll(w[k]);
    return n;
}

}  // extern "C"

// kmc_kernels.cu -- sm_100a kernels for the 3-D fcc binary-alloy KMC.
//
// Lattice in HBM: the reference's OccupancyLattice layout (lattice.hpp:107-135)
// -- one bit per simple-cubic site, index (z*L + y)*L + x, little-endian
// 32-bit words, so upload/download is a plain copy.  Only even-parity sites
// (x^y^z even) are fcc sites (lattice.hpp:139-141).
//
// Two-layer DT: per sweep a random
// origin in [0, 2bk)^3 and a random order of the eight block sets; each phase
// is one launch over the active bk^3 blocks.  Inside a block, 256 single-hit
// rounds: the block draws one of eight inner sets of 4^3 domains (8^3 tiles)
// and every tile's active domain makes one exchange attempt.  Reach: read 2,
// write 1 (kmc.hpp:140-141) < the one-domain gap, so attempts of a round are
// independent and the result equals the CPU oracle bit for bit.
#include <cstdint>
#include <cstdlib>

#include "kmc_kernels.cuh"

#include "lfg_common.cuh"


namespace lfg {

__constant__ int8_t c_fcc[12][3] = {  // kFccOffsets (lattice.hpp:147-151)
    {1, 1, 0}, {1, -1, 0}, {-1, 1, 0}, {-1, -1, 0}, {1, 0, 1}, {1, 0, -1},
    {-1, 0, 1}, {-1, 0, -1}, {0, 1, 1}, {0, 1, -1}, {0, -1, 1}, {0, -1, -1}};

__device__ __forceinline__ uint32_t u4sel(const U4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// Staged rows: for block-local (ly, lz) in [-2, bk+2)^2 one 64-bit word with
// the global x bits [X0 - 16, X0 + 48): local x lx in [-2, bk+2) sits at bit
// lx + 16.  Row index (lz + 2) * E + (ly + 2), E = bk + 4.
struct KmcRows {
    unsigned long long* r;
    int E;
    __device__ __forceinline__ unsigned long long at(int ly, int lz) const { return r[(lz + 2) * E + (ly + 2)]; }
    __device__ __forceinline__ unsigned long long* ptr(int ly, int lz) const { return r + (lz + 2) * E + (ly + 2); }
};

__device__ __forceinline__ int bit_at(unsigned long long row, int lx) { return int((row >> (lx + 16)) & 1ull); }

// Number of B among the 12 fcc neighbours of (lx, ly, lz): four rows at
// Manhattan distance 1 in (y, z) contribute bits lx-1 and lx+1, the four
// diagonal rows bit lx.  All eight row loads depend only on the site, so the
// two counts of an attempt (B site and A partner) issue together with the
// occupancy loads -- one shared-memory latency per round.
__device__ __forceinline__ int nb_count(const KmcRows& R, int lx, int ly, int lz) {
    const unsigned long long m2 = 5ull << (lx + 15);  // bits lx-1, lx+1
    const unsigned long long m1 = 1ull << (lx + 16);
    return __popcll(R.at(ly - 1, lz) & m2) + __popcll(R.at(ly + 1, lz) & m2) + __popcll(R.at(ly, lz - 1) & m2) +
           __popcll(R.at(ly, lz + 1) & m2) + __popcll(R.at(ly - 1, lz - 1) & m1) +
           __popcll(R.at(ly - 1, lz + 1) & m1) + __popcll(R.at(ly + 1, lz - 1) & m1) +
           __popcll(R.at(ly + 1, lz + 1) & m1);
}

__device__ __forceinline__ void global_flip(uint32_t* w, int L, int gx, int gy, int gz) {
    const size_t idx = (size_t(gz) * L + gy) * L + gx;
    atomicXor(w + (idx >> 5), 1u << (idx & 31));
}

__device__ __forceinline__ unsigned long long lds_u64(uint32_t a) {
    unsigned long long v;
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}

// kFccOffsets (lattice.hpp:147-151) in closed form: group g = dir >> 2 picks
// the two non-zero axes ((x,y), (x,z), (y,z)); bit 1 of dir negates the first,
// bit 0 the second.  Register arithmetic instead of a divergent constant-bank
// lookup (12 distinct addresses per warp would serialise).
__device__ __forceinline__ void fcc_offset(int dir, int& dx, int& dy, int& dz) {
    const int g = dir >> 2;
    const int s1 = 1 - (dir & 2), s2 = 1 - 2 * (dir & 1);
    dx = g == 2 ? 0 : s1;
    dy = g == 0 ? s2 : (g == 2 ? s1 : 0);
    dz = g == 0 ? 0 : s2;
}

// One CTA holds `bpc` device blocks of tpb = (bk/8)^3 threads (one thread per
// 8^3 tile).  When a block fits in a warp (bk = 16: 8 threads, four blocks per
// warp) the per-round barrier is __syncwarp; for bk = 32 one block is one CTA.
// Per round the Philox words of the NEXT round are computed first (they do
// not depend on the lattice), so the RNG chain overlaps the attempt's
// shared-memory latency, and every shared load of the attempt (site,
// partner, 2 x 8 neighbour rows) is issued before the first use.
template <bool BOTH, bool WARP_SYNC>
__global__ void __launch_bounds__(128) kmc_dt_phase_kernel(const __grid_constant__ KmcPhaseArgs a) {
    if (a.abort_flag && *reinterpret_cast<const volatile uint32_t*>(a.abort_flag)) return;
    extern __shared__ __align__(16) unsigned long long smk[];
    __shared__ unsigned long long s_thr[13];
    const int L = a.L, Lm = L - 1, bk = a.bk, E = bk + 4, rows = E * E;
    const int tb = bk / 8, tpb = tb * tb * tb;
    const int sub = int(threadIdx.x) / tpb, t = int(threadIdx.x) % tpb;
    const int bpc = int(blockDim.x) / tpb;
    const int nb = L / bk, h = nb / 2;
    const int blin = int(blockIdx.x) * bpc + sub;
    const KmcSweep sw = kmc_sweep_draw(bk, a.seed, a.sweep);
    const int set = sw.set(a.phase);
    const int bxi = 2 * (blin % h) + (set & 1);
    const int byi = 2 * ((blin / h) % h) + ((set >> 1) & 1);
    const int bzi = a.bz0 + 2 * (blin / (h * h)) + (set >> 2);  // bz0 even
    const uint32_t block_id = (uint32_t(bzi) * uint32_t(nb) + uint32_t(byi)) * uint32_t(nb) + uint32_t(bxi);
    const int X0 = (sw.ox + bxi * bk) & Lm, Y0 = (sw.oy + byi * bk) & Lm, Z0 = (sw.oz + bzi * bk) & Lm;
    const int zm = Lm & a.zmask;  // plane slot mask
    const KmcRows R{smk + size_t(sub) * rows, E};
    if (threadIdx.x < 13) s_thr[threadIdx.x] = (uint64_t(a.thr_hi[threadIdx.x]) << 32) | a.thr_lo[threadIdx.x];

    // Stage the block plus a 2-site halo.
    const int wpr = L >> 5, wm = wpr - 1;
    const int xs = (X0 - 16 + L) & Lm, w0 = xs >> 5, bo = xs & 31;
    for (int rr = t; rr < rows; rr += tpb) {
        const int ly = rr % E - 2, lz = rr / E - 2;
        const uint32_t* row = a.w + (size_t((Z0 + lz) & zm) * L + size_t((Y0 + ly) & Lm)) * wpr;
        const uint32_t g0 = row[w0 & wm], g1 = row[(w0 + 1) & wm], g2 = row[(w0 + 2) & wm];
        const uint32_t lo = __funnelshift_r(g0, g1, bo), hi = __funnelshift_r(g1, g2, bo);
        R.r[rr] = (static_cast<unsigned long long>(hi) << 32) | lo;
    }
    __syncthreads();

    const int tx = t % tb, ty = (t / tb) % tb, tz = t / (tb * tb);
    const uint32_t tl = uint32_t(L / 8);
    const uint32_t tile_id = (uint32_t(bzi * tb + tz) * tl + uint32_t(byi * tb + ty)) * tl + uint32_t(bxi * tb + tx);
    const int zpar0 = (X0 ^ Y0 ^ Z0) & 1;  // parity offset of the block frame
    uint32_t nsucc = 0;
    U4 V = {0, 0, 0, 0};
    U4 W = draw(a.seed, a.sweep, TAG_KMC_SITE, tile_id, 0u), Wn = W;  // one draw per two rounds
#pragma unroll 1
    for (int r = 0; r < a.rounds; ++r) {
        const bool odd = (r & 1) != 0;
        if ((r & 31) == 0) V = draw(a.seed, a.sweep, TAG_KMC_SET, block_id, uint32_t(r >> 5));
        if (odd) Wn = draw(a.seed, a.sweep, TAG_KMC_SITE, tile_id, uint32_t((r >> 1) + 1));  // next pair
        uint32_t s5, dirw, accw;
        kmc_round_words(W, odd, s5, dirw, accw);
        const int inner = int((u4sel(V, (r >> 3) & 3) >> (4 * (r & 7))) & 7u);
        const int lx0 = 8 * tx + 4 * (inner & 1), ly0 = 8 * ty + 4 * ((inner >> 1) & 1), lz0 = 8 * tz + 4 * (inner >> 2);
        // KmcKernel::draw_site (kmc.hpp:154-171) over the domain box: x, y
        // uniform, z uniform over the two planes of matching parity.
        const int lx = lx0 + int(s5 & 3u), ly = ly0 + int((s5 >> 2) & 3u);
        const int tpar = (lx ^ ly ^ lz0 ^ zpar0) & 1;  // 1 iff plane lz0 has the wrong parity
        const int lz = lz0 + tpar + 2 * int((s5 >> 4) & 1u);
        const int dir = int(dirw);
        int dx, dy, dz;
        fcc_offset(dir, dx, dy, dz);
        const int px = lx + dx, py = ly + dy, pz = lz + dz;
        // kmc_attempt_impl (kmc.hpp:84-111); everything loaded up front.
        const int here = int((R.at(ly, lz) >> (lx + 16)) & 1ull);
        const int pb = int((R.at(py, pz) >> (px + 16)) & 1ull);
        const int n_site = nb_count(R, lx, ly, lz), n_part = nb_count(R, px, py, pz);
        if ((BOTH || here) && pb != here) {
            // n_i (B site, its A partner excluded: no B there), n_f (A site, its B partner excluded)
            const int d = here ? n_site - (n_part - 1) : n_part - (n_site - 1);
            const bool acc = d <= 0 || uint64_t(accw) < s_thr[d];
            if (acc) {
                atomicXor(R.ptr(ly, lz), 1ull << (lx + 16));
                atomicXor(R.ptr(py, pz), 1ull << (px + 16));
                global_flip(a.w, L, (X0 + lx) & Lm, (Y0 + ly) & Lm, (Z0 + lz) & zm);
                global_flip(a.w, L, (X0 + px) & Lm, (Y0 + py) & Lm, (Z0 + pz) & zm);
                ++nsucc;
            }
        }
        if (odd) W = Wn;
        if (WARP_SYNC) __syncwarp();
        else __syncthreads();
    }
    nsucc = __reduce_add_sync(0xFFFFFFFFu, nsucc);
    if ((threadIdx.x & 31) == 0 && nsucc) atomicAdd(a.counters, (unsigned long long)nsucc);
}

// ---------------------------------------------------------------- bk = 16
// Specialised for 16^3 device blocks (the default plan): block plus 2-site
// halo is 20 sites per axis, so a staged row is ONE 32-bit word (local x lx
// at bit lx + 8) and a block is 400 words.  One block (8 tiles, 8 lanes) per
// CTA/warp, so the 512 active blocks of a 256^3 phase spread over all SMs and
// the per-round barrier is __syncwarp.  The lattice is not written during the
// rounds: each block keeps a pristine copy of its staged rows and XORs the
// difference into global memory once, after its last round (RED.XOR on the
// words holding bits [X0-1, X0+17) of rows y, z in [-1, 17): the write reach
// of kmc.hpp:140-141; neighbouring active blocks touch disjoint bits).
#ifndef LFG_K16E
#define LFG_K16E 22  // z stride of the staged rows (>= 20; 22 measured best, 20..26 and 32 tried)
#endif
// rows (ly, lz) in [-2, 18)^2 at index (lz + 2) * kK16E + (ly + 2)
#ifndef LFG_K16SKEW
#define LFG_K16SKEW 8  // extra words between the blocks of a 4-blocks-per-warp CTA (bank skew; 0..16 tried)
#endif
#ifndef LFG_K16_PREDATOM
#define LFG_K16_PREDATOM 0
#endif
constexpr int kK16Y = 20, kK16E = LFG_K16E, kK16Rows = kK16E * kK16Y, kK16Ofs = 8;
constexpr int kK16Blk = 2 * kK16Rows + LFG_K16SKEW;  // words per block (cur, org, skew)

__device__ __forceinline__ int k16_row(int ly, int lz) { return (lz + 2) * kK16E + (ly + 2); }

// B count among the 12 fcc neighbours of local x lx, given the site's four
// face rows f[] (y-1, y+1, z-1, z+1: bits lx-1, lx+1) and four edge rows e[]
// (bit lx).
__device__ __forceinline__ int k16_count(const uint32_t (&f)[4], const uint32_t (&e)[4], int lx) {
    const uint32_t m2 = 5u << (lx + kK16Ofs - 1), m1 = 1u << (lx + kK16Ofs);
    return __popc(f[0] & m2) + __popc(f[1] & m2) + __popc(f[2] & m2) + __popc(f[3] & m2) + __popc(e[0] & m1) +
           __popc(e[1] & m1) + __popc(e[2] & m1) + __popc(e[3] & m1);
}

// Programmatic dependent launch: a phase launched with the programmatic
// stream-serialisation attribute may start while the previous phase drains;
// its CTAs do the lattice-independent set-up (sweep/origin draws, the first
// batch of site draws) and then wait for the previous grid to complete and
// flush before staging.  Both are no-ops for an ordinary launch.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// Stage the 20 x 20 rows of a 16^3 block (plus halo) into cur/org: row word
// bit k = global bit X0 - 8 + k (k = lx + 8).  Lane `first` of `STRIDE` takes
// rows first, first + STRIDE, ...; the global loads are issued in batches of
// kBatch before any is used (the rows are L2 hits, but a load-use loop would
// pay the full latency once per row).
template <int STRIDE>
__device__ __forceinline__ void k16_stage(const KmcPhaseArgs& a, uint32_t* cur, uint32_t* org, int first, int X0,
                                          int Y0, int Z0, int zm) {
    constexpr int kN = kK16Y * kK16Y, kIt = (kN + STRIDE - 1) / STRIDE, kBatch = kIt < 13 ? kIt : 13;
    const int L = a.L, Lm = L - 1, wpr = L >> 5, wm = wpr - 1;
    const int xs = (X0 - kK16Ofs + L) & Lm, w0 = xs >> 5, bo = xs & 31;
#pragma unroll 1
    for (int i0 = 0; i0 < kIt; i0 += kBatch) {
        uint32_t lo[kBatch], hi[kBatch];
#pragma unroll
        for (int i = 0; i < kBatch; ++i) {
            const int rr = first + STRIDE * (i0 + i);
            lo[i] = hi[i] = 0;
            if (rr < kN) {
                const int ly = rr % kK16Y - 2, lz = rr / kK16Y - 2;
                const uint32_t* row = a.w + (size_t((Z0 + lz) & zm) * L + size_t((Y0 + ly) & Lm)) * wpr;
                lo[i] = row[w0 & wm];
                hi[i] = row[(w0 + 1) & wm];
            }
        }
#pragma unroll
        for (int i = 0; i < kBatch; ++i) {
            const int rr = first + STRIDE * (i0 + i);
            if (rr < kN) {
                const uint32_t v = __funnelshift_r(lo[i], hi[i], bo);
                const int ri = k16_row(rr % kK16Y - 2, rr / kK16Y - 2);
                cur[ri] = v;
                org[ri] = v;
            }
        }
    }
}

template <bool BOTH, bool WLOG = false>
__global__ void __launch_bounds__(32) kmc_dt16_phase_kernel(const __grid_constant__ KmcPhaseArgs a) {
    if (a.abort_flag && *reinterpret_cast<const volatile uint32_t*>(a.abort_flag)) return;
    extern __shared__ __align__(16) uint32_t sk16[];
    __shared__ unsigned long long s_thr[13];
    const int L = a.L, Lm = L - 1, t = int(threadIdx.x) & 7, sub = int(threadIdx.x) >> 3;
    const unsigned wmask = blockDim.x >= 32 ? 0xFFFFFFFFu : (1u << blockDim.x) - 1u;
    uint32_t* const cur = sk16 + sub * kK16Blk;
    uint32_t* const org = cur + kK16Rows;
    const int nb = L >> 4, h = nb >> 1;
    const int blin = int(blockIdx.x) * int(blockDim.x >> 3) + sub;
    const KmcSweep sw = kmc_sweep_draw(16, a.seed, a.sweep);
    const int set = sw.set(a.phase);
    const int bxi = 2 * (blin % h) + (set & 1);
    const int byi = 2 * ((blin / h) % h) + ((set >> 1) & 1);
    const int bzi = a.bz0 + 2 * (blin / (h * h)) + (set >> 2);  // bz0 even
    const uint32_t block_id = (uint32_t(bzi) * uint32_t(nb) + uint32_t(byi)) * uint32_t(nb) + uint32_t(bxi);
    const int X0 = (sw.ox + bxi * 16) & Lm, Y0 = (sw.oy + byi * 16) & Lm, Z0 = (sw.oz + bzi * 16) & Lm;
    const int zm = Lm & a.zmask;  // plane slot mask
    for (int i = int(threadIdx.x); i < 13; i += int(blockDim.x))  // blockDim may be 8
        s_thr[i] = (uint64_t(a.thr_hi[i]) << 32) | a.thr_lo[i];
    const uint32_t thr_sh = uint32_t(__cvta_generic_to_shared(s_thr));  // once, not per round

    const int wpr = L >> 5, wm = wpr - 1;
    k16_stage<8>(a, cur, org, t, X0, Y0, Z0, zm);
    __syncwarp(wmask);

    const int tx = t & 1, ty = (t >> 1) & 1, tz = t >> 2;
    const uint32_t tl = uint32_t(L / 8);
    const uint32_t tile_id = (uint32_t(bzi * 2 + tz) * tl + uint32_t(byi * 2 + ty)) * tl + uint32_t(bxi * 2 + tx);
    const int zpar0 = (X0 ^ Y0 ^ Z0) & 1;
    uint32_t nsucc = 0;
    U4 V = {0, 0, 0, 0};
    // One round; (s5, dirw, accw) are its kmc_round_words, static per parity.
    auto round = [&](int r, uint32_t s5, uint32_t dirw, uint32_t accw) {
        const int inner = int((u4sel(V, (r >> 3) & 3) >> (4 * (r & 7))) & 7u);
        const int lx0 = 8 * tx + 4 * (inner & 1), ly0 = 8 * ty + 4 * ((inner >> 1) & 1), lz0 = 8 * tz + 4 * (inner >> 2);
        // KmcKernel::draw_site (kmc.hpp:154-171) over the domain box.
        const int lx = lx0 + int(s5 & 3u), ly = ly0 + int((s5 >> 2) & 3u);
        const int lz = lz0 + ((lx ^ ly ^ lz0 ^ zpar0) & 1) + 2 * int((s5 >> 4) & 1u);
        int dx, dy, dz;
        fcc_offset(int(dirw), dx, dy, dz);
        const int px = lx + dx, py = ly + dy, pz = lz + dz;
        const int sr = k16_row(ly, lz), pr = k16_row(py, pz);
        // every shared load of the attempt, issued before any use
        const uint32_t own = cur[sr], par = cur[pr];
        const uint32_t sf[4] = {cur[sr - 1], cur[sr + 1], cur[sr - kK16E], cur[sr + kK16E]};
        const uint32_t se[4] = {cur[sr - kK16E - 1], cur[sr + kK16E - 1], cur[sr - kK16E + 1], cur[sr + kK16E + 1]};
        const uint32_t pf[4] = {cur[pr - 1], cur[pr + 1], cur[pr - kK16E], cur[pr + kK16E]};
        const uint32_t pe[4] = {cur[pr - kK16E - 1], cur[pr + kK16E - 1], cur[pr - kK16E + 1], cur[pr + kK16E + 1]};
        const int here = int((own >> (lx + kK16Ofs)) & 1u), pb = int((par >> (px + kK16Ofs)) & 1u);
        const int n_site = k16_count(sf, se, lx), n_part = k16_count(pf, pe, px);
        // kmc_attempt_impl (kmc.hpp:84-111), branch-free: every lane loads its
        // threshold (d <= 0 -> entry 0 = 2^32, always accepted) and XORs a
        // possibly-empty mask, so the round has no divergent control flow.
        const int d = here ? n_site - (n_part - 1) : n_part - (n_site - 1);
        const int di = d < 0 ? 0 : d;  // d <= 12
        const bool acc = (BOTH || here) && pb != here && uint64_t(accw) < lds_u64(thr_sh + 8u * uint32_t(di));
#if LFG_K16_PREDATOM
        if (acc) {  // only accepted exchanges touch the rows (fewer shared wavefronts)
            atomicXor(cur + sr, 1u << (lx + kK16Ofs));
            atomicXor(cur + pr, 1u << (px + kK16Ofs));
        }
#else
        atomicXor(cur + sr, acc ? 1u << (lx + kK16Ofs) : 0u);
        atomicXor(cur + pr, acc ? 1u << (px + kK16Ofs) : 0u);
#endif
        nsucc += acc ? 1u : 0u;
        if (WLOG) {  // the two sites the exchange writes (global sc indices)
            const size_t o = (size_t(r) * size_t(gridDim.x * (blockDim.x >> 3)) + size_t(blin)) * 16 + 2 * t;
            const auto sidx = [&](int x, int y, int z) {
                return uint32_t((size_t((Z0 + z) & Lm) * L + size_t((Y0 + y) & Lm)) * L + size_t((X0 + x) & Lm));
            };
            a.wlog[o] = acc ? sidx(lx, ly, lz) : 0xFFFFFFFFu;
            a.wlog[o + 1] = acc ? sidx(px, py, pz) : 0xFFFFFFFFu;
        }
        __syncwarp(wmask);
    };
    // Round pairs: one draw serves rounds 2m (W.x[0..5), W.y, W.z) and 2m + 1
    // (W.x[5..10), W.x[10..32), W.w) -- lfg_common.cuh kmc_round_words; the
    // next pair's draw is issued before the odd round (its latency hides there).
    U4 W = draw(a.seed, a.sweep, TAG_KMC_SITE, tile_id, 0u);
#pragma unroll 1
    for (int m = 0; m < a.rounds / 2; ++m) {
        const int r = 2 * m;
        if ((r & 31) == 0) V = draw(a.seed, a.sweep, TAG_KMC_SET, block_id, uint32_t(r >> 5));
        round(r, W.x & 31u, below(W.y, 12), W.z);
        const U4 Wn = draw(a.seed, a.sweep, TAG_KMC_SITE, tile_id, uint32_t(m + 1));  // unused after the last pair
        round(r + 1, (W.x >> 5) & 31u, below(W.x & ~1023u, 12), W.w);
        W = Wn;
    }
    // Write-back of the 1-ring-extended block: bits lx in [-1, 17) of rows
    // (ly, lz) in [-1, 17)^2, as XOR differences.
    const int gx = (X0 - 1 + L) & Lm, gw = gx >> 5, gb = gx & 31;
    for (int q = t; q < 18 * 18; q += 8) {
        const int ly = q % 18 - 1, lz = q / 18 - 1;
        const int rr = k16_row(ly, lz);
        const uint32_t d = ((cur[rr] ^ org[rr]) >> (kK16Ofs - 1)) & 0x3FFFFu;  // 18 bits, lx = -1 .. 16
        if (d) {
            uint32_t* row = a.w + (size_t((Z0 + lz) & zm) * L + size_t((Y0 + ly) & Lm)) * wpr;
            atomicXor(row + gw, d << gb);
            if (gb > 14) atomicXor(row + ((gw + 1) & wm), d >> (32 - gb));
        }
    }
    nsucc = __reduce_add_sync(wmask, nsucc);
    if (threadIdx.x == 0 && nsucc) atomicAdd(a.counters, (unsigned long long)nsucc);
}

// ---------------------------------------------------------------- bk = 16, wide
// Latency-bound phases (few active blocks, e.g. 512 at 256^3: under one warp
// per SMSP) run one block per full warp.  Lane t + 8j (tile t, group j) draws
// the Philox words of round 4b + j of its tile and precomputes everything of
// that attempt that does not depend on the lattice (site, partner, their rows
// and bit positions); the four rounds of the batch then run back to back, each
// fetching its precomputed attempt with two shuffles.  Every group evaluates
// the attempt (the same instruction stream) and group 0 applies it, so a
// round's dependent chain is loads -> counts -> threshold -> XOR, with the
// generator and the site arithmetic off it (4 rounds per warp-instruction).
// Attempt order, draws and acceptance are those of kmc_dt16_phase_kernel.
__device__ __forceinline__ int k16_count_at(const uint32_t (&f)[4], const uint32_t (&e)[4], uint32_t bit) {
    const uint32_t m2 = 5u << (bit - 1u), m1 = 1u << bit;
    return __popc(f[0] & m2) + __popc(f[1] & m2) + __popc(f[2] & m2) + __popc(f[3] & m2) + __popc(e[0] & m1) +
           __popc(e[1] & m1) + __popc(e[2] & m1) + __popc(e[3] & m1);
}

template <bool BOTH, bool WLOG = false>
__global__ void __launch_bounds__(32) kmc_dt16w_phase_kernel(const __grid_constant__ KmcPhaseArgs a) {
    if (a.abort_flag && *reinterpret_cast<const volatile uint32_t*>(a.abort_flag)) return;
    extern __shared__ __align__(16) uint32_t sk16[];
    const int L = a.L, Lm = L - 1, lane = int(threadIdx.x), t = lane & 7, j = lane >> 3;
    uint32_t* const cur = sk16;
    uint32_t* const org = cur + kK16Rows;
    const int nb = L >> 4, h = nb >> 1;
    const int blin = int(blockIdx.x);
    const KmcSweep sw = kmc_sweep_draw(16, a.seed, a.sweep);
    const int set = sw.set(a.phase);
    const int bxi = 2 * (blin % h) + (set & 1);
    const int byi = 2 * ((blin / h) % h) + ((set >> 1) & 1);
    const int bzi = a.bz0 + 2 * (blin / (h * h)) + (set >> 2);
    const uint32_t block_id = (uint32_t(bzi) * uint32_t(nb) + uint32_t(byi)) * uint32_t(nb) + uint32_t(bxi);
    const int X0 = (sw.ox + bxi * 16) & Lm, Y0 = (sw.oy + byi * 16) & Lm, Z0 = (sw.oz + bzi * 16) & Lm;
    const int zm = Lm & a.zmask;

    const int wpr = L >> 5, wm = wpr - 1;
    pdl_trigger();

    const int tx = t & 1, ty = (t >> 1) & 1, tz = t >> 2;
    const uint32_t tl = uint32_t(L / 8);
    const uint32_t tile_id = (uint32_t(bzi * 2 + tz) * tl + uint32_t(byi * 2 + ty)) * tl + uint32_t(bxi * 2 + tx);
    const int zpar0 = (X0 ^ Y0 ^ Z0) & 1;
    const bool apply = j == 0;
    uint32_t nsucc = 0;
    U4 V = {0, 0, 0, 0};
    // This lane's attempt of batch bb: tile t, round 4 bb + j (KmcKernel::draw_site,
    // kmc.hpp:154-171), packed as rows (< 512) and bit positions (lx + 8, px + 8 in
    // [7, 24]); accm bit d is the Metropolis verdict accw < threshold(d) for every
    // possible d (64-bit compare against the constant-bank thresholds), so a round
    // looks its d up in a register.
    auto prepare = [&](int bb, uint32_t& pack, uint32_t& accm) {
        if ((bb & 7) == 0) V = draw(a.seed, a.sweep, TAG_KMC_SET, block_id, uint32_t(bb >> 3));
        const int r = 4 * bb + j;
        const U4 W = draw(a.seed, a.sweep, TAG_KMC_SITE, tile_id, uint32_t(r >> 1));  // pair (r, r ^ 1)
        uint32_t s5, dirw, accw;
        kmc_round_words(W, (r & 1) != 0, s5, dirw, accw);
        const int inner = int((u4sel(V, (r >> 3) & 3) >> (4 * (r & 7))) & 7u);
        const int lx0 = 8 * tx + 4 * (inner & 1), ly0 = 8 * ty + 4 * ((inner >> 1) & 1), lz0 = 8 * tz + 4 * (inner >> 2);
        const int lx = lx0 + int(s5 & 3u), ly = ly0 + int((s5 >> 2) & 3u);
        const int lz = lz0 + ((lx ^ ly ^ lz0 ^ zpar0) & 1) + 2 * int((s5 >> 4) & 1u);
        int dx, dy, dz;
        fcc_offset(int(dirw), dx, dy, dz);
        pack = uint32_t(k16_row(ly, lz)) | (uint32_t(k16_row(ly + dy, lz + dz)) << 9) |
               (uint32_t(lx + kK16Ofs) << 18) | (uint32_t(lx + dx + kK16Ofs) << 23);
        accm = 0;
#pragma unroll
        for (int dd = 0; dd < 13; ++dd) accm |= (a.thr_hi[dd] != 0u || accw < a.thr_lo[dd]) ? 1u << dd : 0u;
    };
    uint32_t pk[4], am[4];
    auto exchange = [&](uint32_t pack, uint32_t accm) {  // round q of the batch comes from group q
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(pk[q]) : "r"(pack), "r"(t + 8 * q));
            asm volatile("shfl.sync.idx.b32 %0, %1, %2, 0x1f, 0xffffffff;" : "=r"(am[q]) : "r"(accm), "r"(t + 8 * q));
        }
    };
    {
        uint32_t pack, accm;
        prepare(0, pack, accm);
        exchange(pack, accm);
    }
    pdl_wait();  // everything above is independent of the lattice
    k16_stage<32>(a, cur, org, lane, X0, Y0, Z0, zm);
    __syncwarp();
#pragma unroll 1
    for (int b = 0; b < a.rounds / 4; ++b) {
        // the next batch's draws do not depend on the lattice: software-pipelined
        // one batch ahead so their latency hides under this batch's rounds
        uint32_t pack_n, accm_n;
        prepare(b + 1, pack_n, accm_n);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int sr = int(pk[q] & 511u), pr = int((pk[q] >> 9) & 511u);
            const uint32_t bs = (pk[q] >> 18) & 31u, bp = pk[q] >> 23;
            const uint32_t own = cur[sr], par = cur[pr];
            // odd groups count the partner's neighbours, even groups the site's
            const int cr = (j & 1) ? pr : sr;
            const uint32_t cb = (j & 1) ? bp : bs;
            const uint32_t cf[4] = {cur[cr - 1], cur[cr + 1], cur[cr - kK16E], cur[cr + kK16E]};
            const uint32_t ce[4] = {cur[cr - kK16E - 1], cur[cr + kK16E - 1], cur[cr - kK16E + 1], cur[cr + kK16E + 1]};
            const int n_own = k16_count_at(cf, ce, cb);
            const int n_oth = __shfl_xor_sync(0xFFFFFFFFu, n_own, 8);
            const int n_site = (j & 1) ? n_oth : n_own, n_part = (j & 1) ? n_own : n_oth;
            const int here = int((own >> bs) & 1u), pb = int((par >> bp) & 1u);
            // kmc_attempt_impl (kmc.hpp:84-111), branch-free as in kmc_dt16_phase_kernel
            const int d = here ? n_site - (n_part - 1) : n_part - (n_site - 1);
            const int di = d < 0 ? 0 : d;
            const bool acc = apply && (BOTH || here) && pb != here && ((am[q] >> di) & 1u);
            atomicXor(cur + sr, acc ? 1u << bs : 0u);
            atomicXor(cur + pr, acc ? 1u << bp : 0u);
            nsucc += acc ? 1u : 0u;
            if (WLOG && apply) {  // the two sites the exchange writes (global sc indices)
                const size_t o = (size_t(4 * b + q) * size_t(gridDim.x) + size_t(blin)) * 16 + 2 * t;
                const auto sidx = [&](int row, uint32_t bit) {
                    const int ly = row % kK16E - 2, lz = row / kK16E - 2, lx = int(bit) - kK16Ofs;
                    return uint32_t((size_t((Z0 + lz) & Lm) * L + size_t((Y0 + ly) & Lm)) * L + size_t((X0 + lx) & Lm));
                };
                a.wlog[o] = acc ? sidx(sr, bs) : 0xFFFFFFFFu;
                a.wlog[o + 1] = acc ? sidx(pr, bp) : 0xFFFFFFFFu;
            }
            __syncwarp();
        }
        exchange(pack_n, accm_n);
    }
    const int gx = (X0 - 1 + L) & Lm, gw = gx >> 5, gb = gx & 31;
    for (int q = lane; q < 18 * 18; q += 32) {
        const int ly = q % 18 - 1, lz = q / 18 - 1;
        const int rr = k16_row(ly, lz);
        const uint32_t d = ((cur[rr] ^ org[rr]) >> (kK16Ofs - 1)) & 0x3FFFFu;
        if (d) {
            uint32_t* row = a.w + (size_t((Z0 + lz) & zm) * L + size_t((Y0 + ly) & Lm)) * wpr;
            atomicXor(row + gw, d << gb);
            if (gb > 14) atomicXor(row + ((gw + 1) & wm), d >> (32 - gb));
        }
    }
    nsucc = __reduce_add_sync(0xFFFFFFFFu, nsucc);
    if (lane == 0 && nsucc) atomicAdd(a.counters, (unsigned long long)nsucc);
}

// ---------------------------------------------------------------- bk = 16, producer/consumer
// Latency-bound phases (the same ones as kmc_dt16w_phase_kernel) with the
// lattice-independent work moved off the round chain: one block per CTA of two
// warps.  Warp 1 (producer) draws and precomputes the attempts one batch of
// four rounds ahead -- the site and partner rows as shared byte addresses,
// their bit positions, and the 13-bit Metropolis verdict mask of kmc_dt16w's
// `prepare` -- into a two-slot shared ring, handing slots over with named
// barriers (full: producer arrives, consumer syncs; empty: the reverse).
// Warp 0 (consumer) runs the rounds.  A round's neighbour count is split over
// its four lane groups g: g & 1 picks the site (0) or the partner (1), g >> 1
// the rows on the z-1 side (0) or the z+1 side (1) of the 3x3 row window:
// three rows of the z -+ 1 plane (edge, face, edge) plus the y -+ 1 row of the
// site's plane (face), i.e. rows base-4, base, base+4 and base2 in bytes with
// the same edge/face masks in every group; two shuffles join the four partial
// counts.  Group 0 applies the exchange.  Attempt order, draws and acceptance
// are those of kmc_dt16_phase_kernel (bit-identical lattices).
constexpr int kPcSlots = 2;

__device__ __forceinline__ void named_bar_sync(int id, int n) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int n) {
    asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
template <int OFS>
__device__ __forceinline__ uint32_t lds_at(uint32_t addr) {
    uint32_t v;
    asm volatile("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(addr), "n"(OFS) : "memory");
    return v;
}

// Partial count of one side of a site's 3x3 row window (row address ca, bytes):
// rows ca+zo-4 (edge), ca+zo (face), ca+zo+4 (edge) and ca+yo (face).
__device__ __forceinline__ int k16_side_count(uint32_t ca, int zo, int yo, uint32_t m1, uint32_t m2) {
    const uint32_t za = ca + uint32_t(zo), ya = ca + uint32_t(yo);
    return __popc(lds_at<-4>(za) & m1) + __popc(lds_at<0>(za) & m2) + __popc(lds_at<4>(za) & m1) +
           __popc(lds_at<0>(ya) & m2);
}

template <bool BOTH, bool WLOG = false, int SPLIT = 4>
__global__ void __launch_bounds__(64) kmc_dt16p_phase_kernel(const __grid_constant__ KmcPhaseArgs a) {
    if (a.abort_flag && *reinterpret_cast<const volatile uint32_t*>(a.abort_flag)) return;
    extern __shared__ __align__(16) uint32_t sk16[];
    // [slot][q * 8 + t] for round 4 b + q of tile t: the site and partner row
    // addresses and one-hot bit masks, and the Metropolis verdicts indexed by
    // n_site - n_part + 12 for a B site (vh) and an A site (va)
    __shared__ uint4 ring[kPcSlots][32];
    __shared__ uint2 ringv[kPcSlots][32];
    __shared__ uint32_t sdummy[32];
    const int L = a.L, Lm = L - 1, warp = int(threadIdx.x) >> 5, lane = int(threadIdx.x) & 31;
    const int t = lane & 7, j = lane >> 3;
    uint32_t* const cur = sk16;
    uint32_t* const org = cur + kK16Rows;
    const uint32_t cur_sh = uint32_t(__cvta_generic_to_shared(cur));
    const int nb = L >> 4, h = nb >> 1;
    const int blin = int(blockIdx.x);
    const KmcSweep sw = kmc_sweep_draw(16, a.seed, a.sweep);
    const int set = sw.set(a.phase);
    const int bxi = 2 * (blin % h) + (set & 1);
    const int byi = 2 * ((blin / h) % h) + ((set >> 1) & 1);
    const int bzi = a.bz0 + 2 * (blin / (h * h)) + (set >> 2);
    const uint32_t block_id = (uint32_t(bzi) * uint32_t(nb) + uint32_t(byi)) * uint32_t(nb) + uint32_t(bxi);
    const int X0 = (sw.ox + bxi * 16) & Lm, Y0 = (sw.oy + byi * 16) & Lm, Z0 = (sw.oz + bzi * 16) & Lm;
    const int zm = Lm & a.zmask;
    const int wpr = L >> 5, wm = wpr - 1;
    const int nbatch = a.rounds / 4;
    pdl_trigger();

    if (warp == 1) {  // ---- producer: never touches the lattice, so no pdl_wait
        const int tx = t & 1, ty = (t >> 1) & 1, tz = t >> 2;
        const uint32_t tl = uint32_t(L / 8);
        const uint32_t tile_id = (uint32_t(bzi * 2 + tz) * tl + uint32_t(byi * 2 + ty)) * tl + uint32_t(bxi * 2 + tx);
        const int zpar0 = (X0 ^ Y0 ^ Z0) & 1;
        U4 V = {0, 0, 0, 0};
#pragma unroll 1
        for (int bb = 0; bb < nbatch; ++bb) {
            // round 4 bb + j of tile t (KmcKernel::draw_site, kmc.hpp:154-171), as kmc_dt16w's prepare
            if ((bb & 7) == 0) V = draw(a.seed, a.sweep, TAG_KMC_SET, block_id, uint32_t(bb >> 3));
            const int r = 4 * bb + j;
            const U4 W = draw(a.seed, a.sweep, TAG_KMC_SITE, tile_id, uint32_t(r >> 1));  // pair (r, r ^ 1)
            uint32_t s5, dirw, accw;
            kmc_round_words(W, (r & 1) != 0, s5, dirw, accw);
            const int inner = int((u4sel(V, (r >> 3) & 3) >> (4 * (r & 7))) & 7u);
            const int lx0 = 8 * tx + 4 * (inner & 1), ly0 = 8 * ty + 4 * ((inner >> 1) & 1),
                      lz0 = 8 * tz + 4 * (inner >> 2);
            const int lx = lx0 + int(s5 & 3u), ly = ly0 + int((s5 >> 2) & 3u);
            const int lz = lz0 + ((lx ^ ly ^ lz0 ^ zpar0) & 1) + 2 * int((s5 >> 4) & 1u);
            int dx, dy, dz;
            fcc_offset(int(dirw), dx, dy, dz);
            // accm bit d: the verdict accw < threshold(d) (d <= 0 -> entry 0 = 2^32)
            uint32_t accm = 0;
#pragma unroll
            for (int dd = 0; dd < 13; ++dd) accm |= (a.thr_hi[dd] != 0u || accw < a.thr_lo[dd]) ? 1u << dd : 0u;
            // kmc_attempt_impl's d by k = n_site - n_part + 12 in [0, 24]:
            //   B site: d = k - 11 -> vh bit k = accm bit max(k - 11, 0)
            //   A site: d = 13 - k -> va bit k = accm bit max(13 - k, 0)
            const uint32_t all = (accm & 1u) ? 0xFFFFFFFFu : 0u;
            const uint32_t vh = (all & 0xFFFu) | ((accm >> 1) << 12);
            const uint32_t va = ((__brev(accm) >> 18) & 0x3FFFu) | (all & (0x7FFu << 14));
            const uint4 e = make_uint4(cur_sh + 4u * uint32_t(k16_row(ly, lz)),
                                       cur_sh + 4u * uint32_t(k16_row(ly + dy, lz + dz)), 1u << (lx + kK16Ofs),
                                       1u << (lx + dx + kK16Ofs));
            const int s = bb % kPcSlots;
            if (bb >= kPcSlots) named_bar_sync(1 + kPcSlots + s, 64);  // the consumer has read slot s
            ring[s][lane] = e;
            ringv[s][lane] = make_uint2(vh, va);
            named_bar_arrive(1 + s, 64);  // slot s holds batch bb
        }
        return;
    }

    // ---- consumer
    pdl_wait();
    k16_stage<32>(a, cur, org, lane, X0, Y0, Z0, zm);
    __syncwarp();
    const bool part = (j & 1) != 0, apply = j == 0;
    const uint32_t dummy = uint32_t(__cvta_generic_to_shared(sdummy + lane));
    const int zo = (j >> 1) ? 4 * kK16E : -4 * kK16E;  // z+1 / z-1 plane (bytes)
    const int yo = (j >> 1) ? 4 : -4;                  // y+1 / y-1 row of the site's plane
    uint32_t nsucc = 0;
#pragma unroll 1
    for (int b = 0; b < nbatch; ++b) {
        const int s = b % kPcSlots;
        named_bar_sync(1 + s, 64);
        uint4 rq[4];
        uint2 rv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            rq[q] = ring[s][q * 8 + t];
            rv[q] = ringv[s][q * 8 + t];
        }
        if (b + kPcSlots < nbatch) named_bar_arrive(1 + kPcSlots + s, 64);  // slot s may be refilled
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const uint32_t sa = rq[q].x, pa = rq[q].y, ms = rq[q].z, mp = rq[q].w;
            const uint32_t own = lds_at<0>(sa), par = lds_at<0>(pa);
            // k = n_site - n_part + 12 (valid in the site lanes, which apply the exchange)
            int k;
            if (SPLIT == 1) {  // every lane counts both windows
                const uint32_t s2 = (ms << 1) | (ms >> 1), p2 = (mp << 1) | (mp >> 1);
                k = k16_side_count(sa, -4 * kK16E, -4, ms, s2) + k16_side_count(sa, 4 * kK16E, 4, ms, s2) + 12 -
                    k16_side_count(pa, -4 * kK16E, -4, mp, p2) - k16_side_count(pa, 4 * kK16E, 4, mp, p2);
            } else {
                const uint32_t ca = part ? pa : sa;
                const uint32_t m1 = part ? mp : ms, m2 = (m1 << 1) | (m1 >> 1);  // edge bit, face bits
                int n;
                if (SPLIT == 2) {
                    n = k16_side_count(ca, -4 * kK16E, -4, m1, m2) + k16_side_count(ca, 4 * kK16E, 4, m1, m2);
                } else {
                    n = k16_side_count(ca, zo, yo, m1, m2);
                    n += __shfl_xor_sync(0xFFFFFFFFu, n, 16);  // z-1 side + z+1 side
                }
                k = n + 12 - __shfl_xor_sync(0xFFFFFFFFu, n, 8);  // site - partner
            }
            // kmc_attempt_impl (kmc.hpp:84-111), as in kmc_dt16_phase_kernel
            const bool here = (own & ms) != 0u, pb = (par & mp) != 0u;
            const uint32_t v = here ? rv[q].x : rv[q].y;
            // (bitwise, no short-circuit: no divergent branch in the round)
            const bool acc = (uint32_t(apply) & uint32_t(BOTH || here) & uint32_t(pb != here) & (v >> k)) & 1u;
            // branch-free: the other groups XOR 0 into a private word each
            asm volatile("atom.shared.xor.b32 _, [%0], %1;\n\tatom.shared.xor.b32 _, [%2], %3;" ::"r"(
                             apply ? sa : dummy),
                         "r"(acc ? ms : 0u), "r"(apply ? pa : dummy), "r"(acc ? mp : 0u)
                         : "memory");
            nsucc += acc ? 1u : 0u;
            if (WLOG && apply) {  // the two sites the exchange writes (global sc indices)
                const size_t o = (size_t(4 * b + q) * size_t(gridDim.x) + size_t(blin)) * 16 + 2 * t;
                const auto sidx = [&](uint32_t addr, uint32_t mask) {
                    const int row = int((addr - cur_sh) >> 2);
                    const int ly = row % kK16E - 2, lz = row / kK16E - 2, lx = __ffs(int(mask)) - 1 - kK16Ofs;
                    return uint32_t((size_t((Z0 + lz) & Lm) * L + size_t((Y0 + ly) & Lm)) * L +
                                    size_t((X0 + lx) & Lm));
                };
                a.wlog[o] = acc ? sidx(sa, ms) : 0xFFFFFFFFu;
                a.wlog[o + 1] = acc ? sidx(pa, mp) : 0xFFFFFFFFu;
            }
            __syncwarp();
        }
    }
    const int gx = (X0 - 1 + L) & Lm, gw = gx >> 5, gb = gx & 31;
    for (int q = lane; q < 18 * 18; q += 32) {
        const int ly = q % 18 - 1, lz = q / 18 - 1;
        const int rr = k16_row(ly, lz);
        const uint32_t d = ((cur[rr] ^ org[rr]) >> (kK16Ofs - 1)) & 0x3FFFFu;
        if (d) {
            uint32_t* row = a.w + (size_t((Z0 + lz) & zm) * L + size_t((Y0 + ly) & Lm)) * wpr;
            atomicXor(row + gw, d << gb);
            if (gb > 14) atomicXor(row + ((gw + 1) & wm), d >> (32 - gb));
        }
    }
    nsucc = __reduce_add_sync(0xFFFFFFFFu, nsucc);
    if (lane == 0 && nsucc) atomicAdd(a.counters, (unsigned long long)nsucc);
}

// Blocks per CTA: bk = 16 (8 threads) packs four blocks in one warp; bk = 32
// (64 threads) is one block per CTA.
int kmc_blocks_per_cta(int bk) {
    const int tpb = (bk / 8) * (bk / 8) * (bk / 8);
    return tpb >= 32 ? 1 : 32 / tpb;
}

size_t kmc_phase_smem_bytes(int bk) {
    const size_t E = size_t(bk) + 4;
    return size_t(kmc_blocks_per_cta(bk)) * E * E * 8;
}

template <bool BOTH, bool WS>
static cudaError_t kmc_attr(int smem) {
    return cudaFuncSetAttribute(kmc_dt_phase_kernel<BOTH, WS>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
}

cudaError_t kmc_phase_kernel_attrs() {
    const int smem = int(kmc_phase_smem_bytes(32) > kmc_phase_smem_bytes(16) ? kmc_phase_smem_bytes(32)
                                                                              : kmc_phase_smem_bytes(16));
    cudaError_t e = kmc_attr<false, false>(smem);
    if (e == cudaSuccess) e = kmc_attr<true, false>(smem);
    if (e == cudaSuccess) e = kmc_attr<false, true>(smem);
    if (e == cudaSuccess) e = kmc_attr<true, true>(smem);
    return e;
}

// LFG_KMC_WIDE=0 keeps latency-bound 16^3 phases on the 8-lane kernel, =2
// sends every 16^3 phase to the wide kernel (A/B).
static int kmc_wide_mode() {
    static const int mode = [] {
        const char* e = std::getenv("LFG_KMC_WIDE");
        return e && (e[0] == '0' || e[0] == '2') ? e[0] - '0' : 1;
    }();
    return mode;
}

// LFG_KMC_PC=0 runs latency-bound 16^3 phases on the single-warp wide kernel
// instead of the producer/consumer pair (A/B).
static bool kmc_pc_mode() {
    static const bool on = [] {
        const char* e = std::getenv("LFG_KMC_PC");
        return !(e && e[0] == '0');
    }();
    return on;
}

// LFG_KMC_PCSPLIT=1/2/4: lanes sharing one attempt's neighbour count in the
// producer/consumer kernel (A/B).
static int kmc_pc_split() {
    static const int sp = [] {
        const char* e = std::getenv("LFG_KMC_PCSPLIT");
        return e && (e[0] == '1' || e[0] == '2') ? e[0] - '0' : 4;
    }();
    return sp;
}

// Wide-kernel phase launches carry the programmatic stream-serialisation
// attribute (see pdl_wait): +5 % at 256^3.  LFG_KMC_PDL=0 launches them plainly.
static cudaError_t launch_pdl(void (*kern)(KmcPhaseArgs), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                              const KmcPhaseArgs& a) {
    static const bool on = [] {
        const char* e = std::getenv("LFG_KMC_PDL");
        return !(e && e[0] == '0');
    }();
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = on ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, a);
}

cudaError_t kmc_launch_phase(const KmcPhaseArgs& a, cudaStream_t st) {
    const int tpb = (a.bk / 8) * (a.bk / 8) * (a.bk / 8);
    const int h = a.L / a.bk / 2;
    const int active = h * h * (a.nbz / 2);
    int bpc = kmc_blocks_per_cta(a.bk);
    if (bpc > active) bpc = active;
    const dim3 grid(unsigned(active / bpc));
    const dim3 block(unsigned(bpc * tpb));
    const size_t smem = size_t(bpc) * size_t(a.bk + 4) * size_t(a.bk + 4) * 8;
    if (a.bk == 16) {
        // One block per warp while the phase has fewer blocks than ~4 per
        // SMSP (latency-bound: spread over all SMs); four per warp beyond.
        // (`share` lattices running side by side count as that many times the blocks)
        const int per = active * (a.share > 1 ? a.share : 1) >= 4 * 4 * 148 && active >= 4 ? 4 : 1;
        const dim3 g16 = dim3(unsigned(active / per)), b16 = dim3(unsigned(8 * per));
        const size_t sm16 = size_t(per) * kK16Blk * sizeof(uint32_t);
        const int wide = kmc_wide_mode();
        if ((per == 1 && wide == 1) || wide == 2) {  // one block per full warp (see kmc_dt16w_phase_kernel)
            const dim3 gw = dim3(unsigned(active));
            const size_t smw = 2 * kK16Rows * sizeof(uint32_t);
            if (kmc_pc_mode()) {  // producer/consumer pair of warps per block (kmc_dt16p_phase_kernel)
                if (a.wlog)
                    return launch_pdl(a.both ? kmc_dt16p_phase_kernel<true, true> : kmc_dt16p_phase_kernel<false, true>,
                                      gw, dim3(64), smw, st, a);
                const int sp = kmc_pc_split();
                auto k = a.both ? (sp == 1 ? kmc_dt16p_phase_kernel<true, false, 1>
                                           : sp == 2 ? kmc_dt16p_phase_kernel<true, false, 2> : kmc_dt16p_phase_kernel<true>)
                                : (sp == 1 ? kmc_dt16p_phase_kernel<false, false, 1>
                                           : sp == 2 ? kmc_dt16p_phase_kernel<false, false, 2> : kmc_dt16p_phase_kernel<false>);
                return launch_pdl(k, gw, dim3(64), smw, st, a);
            }
            if (a.wlog)
                return launch_pdl(a.both ? kmc_dt16w_phase_kernel<true, true> : kmc_dt16w_phase_kernel<false, true>, gw,
                                  dim3(32), smw, st, a);
            return launch_pdl(a.both ? kmc_dt16w_phase_kernel<true> : kmc_dt16w_phase_kernel<false>, gw, dim3(32), smw,
                              st, a);
        }
        // (no PDL here: with blocks filling the GPU, early-launched CTAs of the
        // next phase land unevenly on the SMs -- 48 vs 86 att/ns at 512^3)
        if (a.wlog) {
            if (a.both) kmc_dt16_phase_kernel<true, true><<<g16, b16, sm16, st>>>(a);
            else kmc_dt16_phase_kernel<false, true><<<g16, b16, sm16, st>>>(a);
        } else if (a.both) {
            kmc_dt16_phase_kernel<true><<<g16, b16, sm16, st>>>(a);
        } else {
            kmc_dt16_phase_kernel<false><<<g16, b16, sm16, st>>>(a);
        }
        return cudaGetLastError();
    }
    const bool ws = bpc * tpb <= 32;
    if (a.both) {
        if (ws) kmc_dt_phase_kernel<true, true><<<grid, block, smem, st>>>(a);
        else kmc_dt_phase_kernel<true, false><<<grid, block, smem, st>>>(a);
    } else {
        if (ws) kmc_dt_phase_kernel<false, true><<<grid, block, smem, st>>>(a);
        else kmc_dt_phase_kernel<false, false><<<grid, block, smem, st>>>(a);
    }
    return cudaGetLastError();
}

// make_random_alloy (lattice.cpp:117-132) with the counter RNG: valid site n
// (n = sc index >> 1) is B iff word (n & 3) of Philox(seed; n >> 2, 0, 0,
// TAG_KMC_INIT) < threshold, threshold = llround(c 2^32) as in the reference.
__global__ void kmc_init_alloy_kernel(uint32_t* w, int L, int zm, int z0, int nz, uint32_t thr_lo, uint32_t thr_hi,
                                      uint64_t seed) {
    const int wpr = L >> 5;
    const size_t plane_words = size_t(L) * wpr;
    const size_t nwords = size_t(nz) * plane_words;
    const uint64_t thr = (uint64_t(thr_hi) << 32) | thr_lo;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nwords; k += size_t(gridDim.x) * blockDim.x) {
        const int z = (z0 + int(k / plane_words)) & (L - 1);  // global plane
        const size_t in_plane = k % plane_words;
        const int y = int(in_plane / size_t(wpr));
        const size_t gword = size_t(z) * plane_words + in_plane;  // global word index
        const size_t idx0 = gword * 32;                            // first sc index of the word
        const int xpar = (y ^ z) & 1;                              // valid x parity in this row
        uint32_t v = 0;
        // 16 valid sites per word: n = (idx0 + 2 j + xpar) >> 1 = idx0/2 + j
        const size_t n0 = idx0 >> 1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const U4 r = philox4x32_10(uint32_t((n0 >> 2) + q), uint32_t(((n0 >> 2) + q) >> 32), 0u,
                                       TAG_KMC_INIT << 24, uint32_t(seed), uint32_t(seed >> 32));
            const uint32_t rr[4] = {r.x, r.y, r.z, r.w};
#pragma unroll
            for (int e = 0; e < 4; ++e)
                if (uint64_t(rr[e]) < thr) v |= 1u << (2 * (4 * q + e) + xpar);
        }
        w[size_t(z & zm) * plane_words + in_plane] = v;
    }
}

cudaError_t kmc_launch_init_alloy(uint32_t* w, int L, int zmask, int z0, int nz, uint32_t thr_lo, uint32_t thr_hi,
                                  uint64_t seed, cudaStream_t st) {
    const size_t nwords = size_t(nz) * L * L / 32;
    const int blocks = int(std::min<size_t>((nwords + 255) / 256, 148 * 16));
    kmc_init_alloy_kernel<<<blocks, 256, 0, st>>>(w, L, (L - 1) & zmask, z0, nz, thr_lo, thr_hi, seed);
    return cudaGetLastError();
}

// open_bonds_per_particle (kmc.cpp:20-40) as exact sums: out[0] += #B on
// valid sites, out[1] += sum over those B of A-occupied neighbours.  One
// thread per 32-bit word; the 12 neighbour directions are aligned to the
// word with funnel shifts of the three adjacent words of each neighbour row.
__device__ __forceinline__ uint32_t kmc_row_word(const uint32_t* w, int L, int zm, int y, int z, int wi) {
    const int Lm = L - 1, wpr = L >> 5;
    return w[(size_t((z + L) & zm) * L + size_t((y + L) & Lm)) * wpr + size_t((wi + wpr) & (wpr - 1))];
}

// bits of row (y, z) at x + dx for the 32 x of word wi
__device__ __forceinline__ uint32_t kmc_shifted(const uint32_t* w, int L, int zm, int y, int z, int wi, int dx) {
    if (dx == 0) return kmc_row_word(w, L, zm, y, z, wi);
    if (dx > 0) return __funnelshift_r(kmc_row_word(w, L, zm, y, z, wi), kmc_row_word(w, L, zm, y, z, wi + 1), 1);
    return __funnelshift_l(kmc_row_word(w, L, zm, y, z, wi - 1), kmc_row_word(w, L, zm, y, z, wi), 1);
}

// Planes [z0, z0 + nz) (their +-1 neighbour planes must be current in the buffer).
__global__ void kmc_open_bonds_kernel(const uint32_t* __restrict__ w, int L, int zm, int z0, int nz,
                                      unsigned long long* out2) {
    const int wpr = L >> 5;
    const size_t nwords = size_t(nz) * L * wpr;
    unsigned long long np = 0, no = 0;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nwords; k += size_t(gridDim.x) * blockDim.x) {
        const int wi = int(k % size_t(wpr));
        const size_t row = k / size_t(wpr);
        const int y = int(row % size_t(L)), z = (z0 + int(row / size_t(L))) & (L - 1);
        const uint32_t valid = ((y ^ z) & 1) ? 0xAAAAAAAAu : 0x55555555u;
        const uint32_t b = kmc_row_word(w, L, zm, y, z, wi) & valid;
        if (!b) continue;
        np += __popc(b);
        uint32_t open = 0;
#pragma unroll
        for (int d = 0; d < 12; ++d) {
            const uint32_t nbits = kmc_shifted(w, L, zm, y + c_fcc[d][1], z + c_fcc[d][2], wi, c_fcc[d][0]);
            open += __popc(b & ~nbits);
        }
        no += open;
    }
    for (int o = 16; o > 0; o >>= 1) {
        np += __shfl_down_sync(0xFFFFFFFFu, np, o);
        no += __shfl_down_sync(0xFFFFFFFFu, no, o);
    }
    if ((threadIdx.x & 31) == 0) {
        if (np) atomicAdd(out2 + 0, np);
        if (no) atomicAdd(out2 + 1, no);
    }
}

cudaError_t kmc_launch_open_bonds(const uint32_t* w, int L, int zmask, int z0, int nz, unsigned long long* out2,
                                  cudaStream_t st) {
    const size_t nwords = size_t(nz) * L * L / 32;
    const int blocks = int(std::min<size_t>((nwords + 255) / 256, 148 * 16));
    kmc_open_bonds_kernel<<<blocks, 256, 0, st>>>(w, L, (L - 1) & zmask, z0, nz, out2);
    return cudaGetLastError();
}

// count_b (lattice.cpp:97-101): popcount of every word.
__global__ void kmc_count_b_kernel(const uint32_t* __restrict__ w, size_t nwords, unsigned long long* out) {
    unsigned long long n = 0;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nwords; k += size_t(gridDim.x) * blockDim.x)
        n += __popc(w[k]);
    for (int o = 16; o > 0; o >>= 1) n += __shfl_down_sync(0xFFFFFFFFu, n, o);
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(out, n);
}

cudaError_t kmc_launch_count_b(const uint32_t* w, int L, unsigned long long* out, cudaStream_t st) {
    const size_t nwords = size_t(L) * L * L / 32;
    const int blocks = int(std::min<size_t>((nwords + 255) / 256, 148 * 16));
    kmc_count_b_kernel<<<blocks, 256, 0, st>>>(w, nwords, out);
    return cudaGetLastError();
}

}  // namespace lfg

// kpz_kernels.cu -- sm_100a kernels for the 2+1-d KPZ octahedron model.
//
// Representation on the device ("spins").  The reference stores two slope
// planes sigma_x, sigma_y (lattice.hpp:56-97).  The device stores ONE bit per
// site, f(i,j), with
//     sigma_x(i,j) = +1  <=>  f(i,j) == f(i-1,j)
//     sigma_y(i,j) = +1  <=>  f(i,j) == f(i,j-1)
// i.e. f = (h >> 1) ^ ((i+j) >> 1) (mod 2) for the integer height h.  Every
// integrable slope field (closure, kpz.cpp:35-47) has exactly two spin fields
// (f and ~f give the same slopes; the device fixes f(0,0)=0).  In spins the
// octahedron move of kpz_attempt_impl (kpz.hpp:71-107) reads
//     deposit  <=> f_R == f_S, f_U == f_S, f_L != f_S, f_D != f_S   (r < p)
//     detach   <=> f_R != f_S, f_U != f_S, f_L == f_S, f_D == f_S   (r < q)
// and flips the single bit f_S (which negates the four stencil slopes).  This
// halves HBM/SMEM footprint and turns the 4-bit RMW into a 1-bit RMW; uploads
// and downloads convert to/from the reference word layout exactly.
//
// Layout in HBM: replica-major, row-major, L/32 little-endian uint32 words per
// row, bit i&31 of word i>>5 -- so row j is contiguous and 128-bit loadable.
#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include <cudaTypedefs.h>

#include "kpz_kernels.cuh"
#include "lfg_common.cuh"

#ifndef LFG_KPZ_RED
#define LFG_KPZ_RED 1  // write the flip back with red.shared.xor (0: XOR + STS; +3 % at L = 2^16, gpurun_out/r02j)
#endif

namespace lfg {

// ============================================================ DTr phase kernel
// One CTA = one active device block (bx x by sites) of one replica.
// Threads: 32 lanes x NW warps, NW = by / (16 NT); lane = tile column (bx/32
// lanes active), warp w owns tile rows w + n*NW, n < NT (NT tiles per lane,
// so the per-round dispatch, barrier and loop are shared by NT independent
// attempts).  Shared-memory layout (32-bit words, 256-byte lines, line 0 at
// a 2 KB-aligned shared-window address A):
//   line R+8, word s        : staged spins of block row R (R = -1 .. by),
//                             s = 0..Wt-1 tile words, s = Wt the right halo
//                             word (H_R); the left halo word (H_L) of row R
//                             sits at line R+7, word 63.
// With a 64-word line stride every tile column owns one bank for all its
// rows, so the per-round gathers (own/up/down words) are conflict-free, and
// the neighbour-word gather is a lane rotation that lands the block's edge
// lanes exactly on H_L (bank 31) / H_R (bank Wt).  Lines 0..5 are never
// touched, so A may sit up to 1.5 KB below the dynamic-smem base; the 2 KB
// alignment makes "tile row base | anchor row * 256" a single LOP3 and keeps
// every anchor address in one ordinary register (no per-round re-derivation
// of the shared window base).
__device__ __forceinline__ int sm_slot(int R, int s) {
    return s < 0 ? (R + 7) * 64 + 63 : (R + 8) * 64 + s;
}

__device__ __forceinline__ uint32_t sel4(const U4& v, int i) {
    return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

__device__ __forceinline__ void count_if_nonzero(uint32_t& n, uint32_t v) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %1, 0;\n\t@p add.u32 %0, %0, 1;\n\t}" : "+r"(n) : "r"(v));
}

// 32-bit shared-window addressing.  volatile keeps program order w.r.t. barriers.
__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}

__device__ __forceinline__ void sts32(uint32_t a, uint32_t v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v));
}

template <int LUT>
__device__ __forceinline__ uint32_t lop3(uint32_t a, uint32_t b, uint32_t c) {
    uint32_t d;
    asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(d) : "r"(a), "r"(b), "r"(c), "n"(LUT));
    return d;
}

// ---- TMA bulk copies (cp.async.bulk, global -> shared, mbarrier completion)
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t mbar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_wait_parity(uint32_t mbar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(mbar), "r"(parity)
        : "memory");
}

__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t mbar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(mbar)
                 : "memory");
}

// shared -> global bulk store (bulk-group completion)
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}

// 3-D tensor copies (cp.async.bulk.tensor, tile mode): box of tensor map `tm`
// at element coordinates (x, y, z).
__device__ __forceinline__ void tma_load_3d(uint32_t dst, const CUtensorMap* tm, int x, int y, int z, uint32_t mbar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(dst), "l"(tm), "r"(x), "r"(y), "r"(z), "r"(mbar)
        : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* tm, int x, int y, int z, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(tm),
                 "r"(x), "r"(y), "r"(z), "r"(src)
                 : "memory");
}

// Commit this thread's bulk stores and wait until they are complete (written).
__device__ __forceinline__ void bulk_commit_and_wait() {
    asm volatile("cp.async.bulk.commit_group;\n\tcp.async.bulk.wait_group 0;" ::: "memory");
}

// FMA-pipe shift (IMAD.SHL): keeps the anchor-field advance off the ALU pipe.
__device__ __forceinline__ uint32_t mullo_u32(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("mul.lo.u32 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}


template <bool MW>
__device__ __forceinline__ void round_barrier() {
    if (MW) __syncthreads();
    else __syncwarp();
}

// (u < thr_lo || all) ? bit : 0 -- one ISETP.OR + SEL (a 33-bit threshold
// thr <= 2^32 split as all = thr >> 32, thr_lo = low 32 bits).
__device__ __forceinline__ uint32_t sel_lt_or(uint32_t u, uint32_t thr_lo, uint32_t all, uint32_t bit) {
    uint32_t r;
    asm("{\n\t.reg .pred pa, pl;\n\tsetp.ne.u32 pa, %3, 0;\n\tsetp.lt.or.u32 pl, %1, %2, pa;\n\t"
        "selp.b32 %0, %4, 0, pl;\n\t}"
        : "=r"(r) : "r"(u), "r"(thr_lo), "r"(all), "r"(bit));
    return r;
}

// One single-hit round of the NT tiles a lane owns, active domain (HX, HY).
//   addr      : shared address of each anchor row's tile word (row j of the
//               tile's top half); HY adds 8 rows (2048 bytes, an immediate)
//   own/up/dn : spin words of rows j, j+1, j-1 (same tile column, same bank)
//   nb        : the neighbouring tile word on the crossing side (left for the
//               hx=0 half, right for hx=1); funnel shifts bring f(i-1) and
//               f(i+1) into bit position i for all 32 columns at once.
//   deposit   : f_R==f_S & f_U==f_S & f_L!=f_S & f_D!=f_S  (LUT 0x81 & 0x18)
//   detach    : f_R!=f_S & f_U!=f_S & f_L==f_S & f_D==f_S  (LUT 0x18 & 0x81)
// With acceptance draws (p < 1 or q > 0) both tests share their common part
// g = f_R==f_U & f_L==f_D & f_R!=f_L, and f_R==f_S tells the two moves apart
// (6 LOP3 per tile instead of 7; 32-bit threshold compares: 498 -> 534 att/ns).
// The one-hot anchor bit selects the column actually attempted (a zero base
// makes the attempt a no-op: a tile's skipped groups, sub = 4).  All loads
// of all tiles are issued before any store (the tiles are disjoint rows), so
// the NT dependency chains overlap.
template <int HX, int HY, bool GENERAL, int NT>
__device__ __forceinline__ void kpz_attempt_tiles(const uint32_t (&addr)[NT], const uint32_t (&xd)[NT],
                                                  const uint32_t (&u)[NT], uint64_t thrP, uint64_t thrQ,
                                                  uint32_t& ndep, uint32_t& ndet, uint32_t (&acc)[NT],
                                                  const uint32_t (&base_lo)[NT], const uint32_t (&base_hi)[NT]) {
    uint32_t own[NT], up[NT], dn[NT], nb[NT], res[NT];
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        const uint32_t pw = addr[n] + (HY << 11);
        own[n] = lds32(pw);
        nb[n] = lds32(HX ? pw + 4u : pw - 4u);
        up[n] = lds32(pw + 256);
        dn[n] = lds32(pw - 256);
    }
#pragma unroll
    for (int n = 0; n < NT; ++n) {
        const uint32_t Rw = __funnelshift_r(own[n], nb[n], 1);  // bit i = f(i+1)
        const uint32_t Lw = __funnelshift_l(nb[n], own[n], 1);  // bit i = f(i-1)
        const uint32_t bit = (HX ? base_hi[n] : base_lo[n]) << xd[n];  // 0: tile skips this round
        if (!GENERAL) {
            const uint32_t flip = lop3<0x80>(lop3<0x81>(own[n], Rw, up[n]), lop3<0x18>(own[n], Lw, dn[n]), bit);
            res[n] = own[n] ^ flip;
            count_if_nonzero(ndep, flip);
            acc[n] = flip;
        } else {
            // thresholds <= 2^32: u < thr  <=>  (thr == 2^32) | (u < low32(thr)), one 32-bit compare
            const uint32_t okP = sel_lt_or(u[n], uint32_t(thrP), uint32_t(thrP >> 32), bit);
            const uint32_t okQ = sel_lt_or(u[n], uint32_t(thrQ), uint32_t(thrQ >> 32), bit);
            // Both moves need f_R == f_U, f_L == f_D, f_R != f_L (own cancels); the
            // deposit is the one with f_R == f_S.
            const uint32_t g = lop3<0x90>(lop3<0x42>(Rw, up[n], Lw), Lw, dn[n]);
            const uint32_t x = own[n] ^ Rw;
            const uint32_t dep = lop3<0x08>(x, g, okP);  // ~x & g & okP
            const uint32_t det = lop3<0x80>(x, g, okQ);  // x & g & okQ
            res[n] = lop3<0x96>(own[n], dep, det);
            count_if_nonzero(ndep, dep);
            count_if_nonzero(ndet, det);
            acc[n] = dep | det;
        }
    }
#pragma unroll
#if LFG_KPZ_RED
    // variant: shared-memory XOR reduction of the flip (one instruction instead of XOR + STS)
    for (int n = 0; n < NT; ++n) asm volatile("red.shared.xor.b32 [%0], %1;" ::"r"(addr[n] + (HY << 11)), "r"(acc[n]));
    (void)res;
#else
    for (int n = 0; n < NT; ++n) sts32(addr[n] + (HY << 11), res[n]);
#endif
}

// Inner single-hit rounds of one block activation.  The inner set of each
// round is block-uniform (Philox(seed, sweep, block) in uniform registers,
// redrawn every 64 rounds), so a uniform branch selects one of four
// specialised bodies whose row offset, neighbour direction and bit offset are
// immediates.  Anchor fields of round k of a 16-round batch (A = Philox(tile,
// batch), h = k >> 3) are consumed from the top of A[h] (xd, 4 bits) and
// A[2+h] (yd, 3 bits) with IMAD.HI/IMAD.SHL on the FMA pipe -- the ALU pipe
// binds this kernel -- which also makes the loop body position-independent,
// so only 4 rounds are unrolled (small I-cache footprint).  lane_base has
// bits 8..10 clear, so the row offset yd*256 merges with one LOP3.
// Debug write-set recording (lfg_kpz_debug_record_anchors): one word per
// (round, tile) of the launch -- tile_id | xd << 20 | yd << 24 | hx << 27 |
// hy << 28 | accepted << 29 -- from which the host rebuilds every write of
// kpz_attempt_impl (kpz.hpp:97-105) for the reference's WriteLog check.
struct KpzAnchorLog {
    uint32_t* out;     // this launch: [kRounds][tiles_in_launch]
    uint32_t stride;   // tiles_in_launch
    uint32_t slot[4];  // this lane's tile slots (NT <= 4)
};

template <bool GENERAL, bool FULL, int NT, bool MW, bool WLOG = false>
__device__ __forceinline__ void kpz_block_rounds(const uint32_t (&lane_base)[NT], bool active, uint64_t seed,
                                                 uint64_t sweep, uint32_t block_id, const uint32_t (&tile_id)[NT],
                                                 uint64_t thrP, uint64_t thrQ, uint32_t& ndep, uint32_t& ndet,
                                                 uint32_t& nskip, const int rounds, const int skip,
                                                 const KpzAnchorLog& wlog = KpzAnchorLog{}) {
    // One-hot bases 1 and 1 << 16.  thrQ <= 2^32, so thrQ >> 33 is 0 -- but not to ptxas:
    // the bases become uniform runtime values instead of immediates rematerialised into a
    // vector register every round (one IMAD.MOV per round saved: 984 -> 1007 att/ns).
    const uint32_t zero = uint32_t(thrQ >> 33);
    const uint32_t one = 1u + zero;
    // Skip masks (sub = 4): bit g set <=> the tile sits out 4-round group g (< 32).
    uint32_t mk[NT];
#pragma unroll
    for (int n = 0; n < NT; ++n) mk[n] = 0u;
#pragma unroll 1
    for (int m4 = 0; 64 * m4 < rounds; ++m4) {
        const U4 V = draw(seed, sweep, TAG_SET, block_id, uint32_t(m4));
#pragma unroll 1
        for (int j = 0; j < 4 && 64 * m4 + 16 * j < rounds; ++j) {
            uint32_t setw = sel4(V, j);
            const int m = 4 * m4 + j;
            U4 A[NT];
#pragma unroll
            for (int n = 0; n < NT; ++n) A[n] = draw(seed, sweep, TAG_ANCHOR, tile_id[n], uint32_t(m));
            if (m == 0 && skip) {
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    mk[n] = kpz_skip_mask(kpz_skip_k(kpz_skip_bits(A[n].z, A[n].w), skip), skip);
                    nskip += 4u * uint32_t(__popc(mk[n]));
                }
            }
#pragma unroll 1
            for (int h = 0; h < 2 && 16 * m + 8 * h < rounds; ++h) {
                uint32_t xw[NT], yw[NT];
#pragma unroll
                for (int n = 0; n < NT; ++n) {
                    xw[n] = h ? A[n].y : A[n].x;
                    yw[n] = h ? A[n].w : A[n].z;
                }
#pragma unroll 1
                for (int q = 0; q < 2 && 16 * m + 8 * h + 4 * q < rounds; ++q) {
                    U4 Uw[NT];
                    if (GENERAL) {
#pragma unroll
                        for (int n = 0; n < NT; ++n)
                            Uw[n] = draw(seed, sweep, TAG_ACCEPT, tile_id[n], uint32_t(4 * m + 2 * h + q));
                    }
                    // this 4-round group's one-hot bases per tile (0 while the tile sits out)
                    uint32_t blo[NT], bhi[NT];
#pragma unroll
                    for (int n = 0; n < NT; ++n) {
                        blo[n] = one & ~mk[n];
                        bhi[n] = blo[n] << 16;
                        mk[n] >>= 1;
                    }
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        uint32_t addr[NT], xd[NT], u[NT];
#pragma unroll
                        for (int n = 0; n < NT; ++n) {
                            xd[n] = __umulhi(xw[n], 16u);  // top 4 bits, then advance
                            xw[n] = mullo_u32(xw[n], 16u);
                            // row field k of this quarter -> bits 8..10 (bits above masked by the LOP3)
                            addr[n] = lop3<0xF8>(lane_base[n], __umulhi(yw[n], 2048u << (3 * k)), 0x700u);
                            u[n] = GENERAL ? sel4(Uw[n], k) : 0u;
                        }
                        uint32_t acc[NT];
                        if (FULL || active) {
                            if (setw & 2u) {
                                if (setw & 1u)
                                    kpz_attempt_tiles<1, 1, GENERAL, NT>(addr, xd, u, thrP, thrQ, ndep, ndet, acc, blo, bhi);
                                else
                                    kpz_attempt_tiles<0, 1, GENERAL, NT>(addr, xd, u, thrP, thrQ, ndep, ndet, acc, blo, bhi);
                            } else {
                                if (setw & 1u)
                                    kpz_attempt_tiles<1, 0, GENERAL, NT>(addr, xd, u, thrP, thrQ, ndep, ndet, acc, blo, bhi);
                                else
                                    kpz_attempt_tiles<0, 0, GENERAL, NT>(addr, xd, u, thrP, thrQ, ndep, ndet, acc, blo, bhi);
                            }
                            if (WLOG) {
                                const uint32_t r = uint32_t(16 * m + 8 * h + 4 * q + k);
#pragma unroll
                                for (int n = 0; n < NT; ++n)
                                    wlog.out[r * wlog.stride + wlog.slot[n]] =
                                        tile_id[n] | (xd[n] << 20) | (((addr[n] >> 8) & 7u) << 24) |
                                        ((setw & 3u) << 27) | (acc[n] ? 1u << 29 : 0u) | (blo[n] ? 0u : 1u << 30);
                            }
                        }
                        setw >>= 2;
                        round_barrier<MW>();
                    }
#pragma unroll
                    for (int n = 0; n < NT; ++n) yw[n] <<= 12;  // next 4 row fields
                }
            }
        }
    }
}

#ifndef LFG_KPZ_NT
#define LFG_KPZ_NT 2  // max tiles per lane (by >= 16 NT); measured best on B200 (NT=4: fewer warps, slower)
#endif

// Dynamic shared memory: lines 6 .. by+8 relative to the 2 KB-aligned origin
// A = ceil_2048(base - 1536), which lies at most 511 bytes above base - 1536.
size_t kpz_phase_smem_bytes(int by) { return size_t(by + 9) * 256 + 512; }

// Completion-flag dependencies of the whole-sweep kernel (below): before an
// activation of phase k > 0 is staged, thread 0 waits until the phase-(k-1)
// blocks in its 8-neighbourhood carry this launch's epoch.  `flags == nullptr`
// (phase kernels, phase 0) means no wait.
__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u32(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct KpzDeps {
    const uint32_t* flags;  // [nby][nbx] of this replica, or nullptr
    int nbx, nby, ddx, ddy;  // ddx/ddy: previous set differs in x / y parity
    uint32_t epoch;
    // Block-wide wait: every thread polls the four flags (like an mbarrier
    // try_wait loop), then orders the bulk copies that follow after the acquires.
    __device__ __forceinline__ void wait_block(int bxi, int byi) const {
        if (!flags) return;
        // block counts are powers of two
        const int x0 = (bxi - ddx) & (nbx - 1), x1 = (bxi + ddx) & (nbx - 1);
        const int y0 = (byi - ddy) & (nby - 1), y1 = (byi + ddy) & (nby - 1);
        asm volatile(
            "{\n\t.reg .pred pok;\n\t.reg .u32 va, vb, vc, vd;\n"
            "KPZ_DEPS_POLL_%=:\n\t"
            "ld.acquire.gpu.global.u32 va, [%0];\n\t"
            "ld.acquire.gpu.global.u32 vb, [%1];\n\t"
            "ld.acquire.gpu.global.u32 vc, [%2];\n\t"
            "ld.acquire.gpu.global.u32 vd, [%3];\n\t"
            "xor.b32 va, va, %4;\n\txor.b32 vb, vb, %4;\n\txor.b32 vc, vc, %4;\n\txor.b32 vd, vd, %4;\n\t"
            "or.b32 va, va, vb;\n\tor.b32 vc, vc, vd;\n\tor.b32 va, va, vc;\n\t"
            "setp.ne.u32 pok, va, 0;\n\t"
            "@pok nanosleep.u32 64;\n\t"
            "@pok bra KPZ_DEPS_POLL_%=;\n\t"
            "fence.proxy.async.global;\n\t}"  // bulk copies read what the acquires saw
            ::"l"(flags + y0 * nbx + x0), "l"(flags + y0 * nbx + x1), "l"(flags + y1 * nbx + x0),
            "l"(flags + y1 * nbx + x1), "r"(epoch)
            : "memory");
    }
};

// One activation of device block (bxi, byi) (block-set `set`) of replica
// `rep`: stage, a.rounds single-hit rounds, write back, count.  `mbar_parity` is
// the phase of the CTA's staging mbarrier (initialised by the caller) that this
// activation's bulk copies complete.
template <bool GENERAL, bool FULL, int kNT, bool MW, bool WLOG = false>
__device__ __forceinline__ void kpz_block_activation(const KpzPhaseArgs& a, uint32_t* const sm, const uint32_t smA,
                                                     const int rep, const uint64_t seed, const KpzSweep& sw,
                                                     const int bxi, const int byi, const uint32_t mbar_parity,
                                                     const bool init_mbar, const KpzDeps& deps) {
    const int L = a.L, Lm = L - 1, wpr = L >> 5, wmask = wpr - 1;
    const int Wt = a.bx >> 5;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint64_t sweep = a.sweep;
    // Rows live at buffer slot (global row & rmask): rmask = L-1 for a whole
    // lattice, C-1 for a strip shard whose ring buffer holds C >= H + 4 by + 2 rows.
    const int rmask = Lm & a.row_mask;
    uint32_t* __restrict__ f = a.f + size_t(rep) * size_t(a.row_mask + 1) * size_t(wpr);
    const uint32_t block_id = uint32_t(byi) * uint32_t(L / a.bx) + uint32_t(bxi);
    const int X0 = (sw.ox + bxi * a.bx) & Lm;
    const int Y0 = (sw.oy + byi * a.by) & Lm;
    const int b = X0 & 31;
    const int w0 = ((X0 - 32 + L) & Lm) >> 5;
    // FULL: the block's 64-word window [X0/32 - 4, X0/32 + 60) and rows -1..by
    // lie inside the buffer without wrapping -> tensor copies in and out.
    const int xw = (X0 >> 5) - 4;
    const int ylo = (Y0 - 1) & rmask;
    const bool tens = FULL && a.tma && xw >= 0 && xw + 64 <= wpr && ylo + a.by + 2 <= rmask + 1;

    // Stage rows -1..by, slots -1..Wt (slot s of row R <- global bits
    // [X0 + 32 s, X0 + 32 s + 32)).
    if (FULL) {
        // Wt == 32 (so L >= 2048 and a row has >= 64 words), and X0 is a
        // multiple of 128 (kpz_ox_quantum): slot s is global word X0/32 + s, and
        // the raw words [X0/32 - 4, X0/32 + 36) (16-byte aligned) of every
        // staged row land at words 0..39 of the row's own line by cp.async.bulk
        // (split in two where the block wraps around x = L), all rows in flight
        // at once against one mbarrier.  No shift pass: slot s sits at line
        // word s + 4, so tile column tx reads bank (tx + 4) & 31 and the halo
        // words H_L / H_R are words 3 / 36 of the same line.
        // Away from the x / y wrap of the buffer, two tensor copies (64-word
        // boxes of by/2 + 1 rows, issued by one thread) stage the whole block;
        // at the wrap every row is one or two 40-word bulk copies.
        const uint32_t mbar = smA + 6 * 256;  // line 6, word 0 (lines < 7 hold no row data)
        const uint32_t rows = uint32_t(a.by + 2);
        deps.wait_block(bxi, byi);
        if (threadIdx.x == 0) {
            if (init_mbar) mbar_init(mbar, 1);
            mbar_arrive_expect_tx(mbar, rows * (tens ? 256u : 160u));
            if (tens) {
                const int br = (a.by >> 1) + 1;
                tma_load_3d(smA + 7 * 256, &a.tm_ld, xw, ylo, rep, mbar);
                tma_load_3d(smA + uint32_t(7 + br) * 256u, &a.tm_ld, xw, ylo + br, rep, mbar);
            }
        }
        __syncthreads();
        if (!tens) {
            const int a0 = xw & wmask;
            const int n1 = min(40, wpr - a0);  // words before the x wrap (a multiple of 4)
            for (int R = int(threadIdx.x) - 1; R <= a.by; R += int(blockDim.x)) {
                const uint32_t* row = f + uint32_t((Y0 + R) & rmask) * uint32_t(wpr);
                const uint32_t dst = smA + uint32_t(R + 8) * 256u;
                bulk_g2s(dst, row + a0, uint32_t(n1) * 4u, mbar);
                if (n1 < 40) bulk_g2s(dst + uint32_t(n1) * 4u, row, uint32_t(40 - n1) * 4u, mbar);
            }
        }
        mbar_wait_parity(mbar, mbar_parity);
    } else {
        deps.wait_block(bxi, byi);
        for (int R = warp - 1; R <= a.by; R += nwarps) {
            const uint32_t* __restrict__ row = f + uint32_t((Y0 + R) & rmask) * uint32_t(wpr);
            for (int k = lane; k < Wt + 2; k += 32) {
                const uint32_t lo = __ldg(row + ((w0 + k) & wmask));
                const uint32_t hi = __ldg(row + ((w0 + k + 1) & wmask));
                sm[sm_slot(R, k - 1)] = __funnelshift_r(lo, hi, b);
            }
        }
    }
    __syncthreads();

    const int tx = lane;
    uint32_t lane_base[kNT], tile_id[kNT];
#pragma unroll
    for (int n = 0; n < kNT; ++n) {
        const int ty = warp + n * nwarps;
        tile_id[n] = uint32_t(byi * (a.by >> 4) + ty) * uint32_t(L >> 5) + uint32_t(bxi * Wt + tx);
        lane_base[n] = smA + uint32_t((16 * ty + 8) * 256 + 4 * tx + (FULL ? 16 : 0));  // bits 8..10 clear
    }
    uint32_t ndep = 0, ndet = 0, nskip = 0;
    KpzAnchorLog wl{};
    if (WLOG) {
        const uint32_t tpb = uint32_t(Wt * (a.by >> 4));
        wl.out = a.wlog;
        wl.stride = gridDim.x * gridDim.y * tpb;
#pragma unroll
        for (int n = 0; n < kNT; ++n)
            wl.slot[n] = (blockIdx.y * gridDim.x + blockIdx.x) * tpb + uint32_t(warp + n * nwarps) * uint32_t(Wt) +
                         uint32_t(tx);
    }
    kpz_block_rounds<GENERAL, FULL, kNT, MW, WLOG>(lane_base, tx < Wt, seed, sweep, block_id, tile_id, a.thrP,
                                                   a.thrQ, ndep, ndet, nskip, a.rounds, a.skip, wl);
    // Write back block rows 0..by-1: global word w0+1+k = funnel_l(slot k-1, slot k, b).
    // A row that a strip neighbour reads as its ghost is also stored straight
    // into that neighbour's ring buffer (NVLink peer memory): the exchange is
    // fused into the write-back, no separate collective.
    const bool push = a.peer_dn != nullptr || a.peer_up != nullptr;
    auto peer_row = [&](int R) -> uint32_t* {
        const int gy = (Y0 + R) & Lm;
        uint32_t* p = gy == a.push_row_dn ? a.peer_dn : (gy == a.push_row_up ? a.peer_up : nullptr);
        return p ? p + uint32_t(gy & rmask) * uint32_t(wpr) : nullptr;
    };
    if (FULL) {
        // Interior words of rows 0..by-1 (line words 4..35) -> global words
        // X0/32 .. X0/32 + 31 by bulk stores (128 bytes, 16-byte aligned; split
        // at the x wrap): every thread's shared writes are made visible to the
        // async proxy, one thread per row issues its copies and waits for them
        // (the chained-phase flag is released only after every row landed).
        // Away from the wraps: two tensor stores of the 64-word window of rows
        // 0..by-1 (the 32 words outside the block are the inactive
        // neighbours' words, unchanged in this phase and written back as
        // staged; a later-phase block that could write them waits for this
        // block's flag).  At a wrap: per-row 128-byte bulk stores.
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncthreads();
        const int gw = X0 >> 5;
        if (tens) {  // (rows 0..by-1 then lie inside the buffer too)
            if (threadIdx.x == 0) {
                const int bs = a.by >> 1;
                tma_store_3d(&a.tm_st, xw, ylo + 1, rep, smA + 8 * 256);
                tma_store_3d(&a.tm_st, xw, ylo + 1 + bs, rep, smA + uint32_t(8 + bs) * 256u);
                bulk_commit_and_wait();
            }
        } else {
            const int n1 = min(32, wpr - gw);
            for (int R = int(threadIdx.x); R < a.by; R += int(blockDim.x)) {
                uint32_t* const row = f + uint32_t((Y0 + R) & rmask) * uint32_t(wpr);
                const uint32_t src = smA + uint32_t(R + 8) * 256u + 16u;
                bulk_s2g(row + gw, src, uint32_t(n1) * 4u);
                if (n1 < 32) bulk_s2g(row, src + uint32_t(n1) * 4u, uint32_t(32 - n1) * 4u);
            }
            bulk_commit_and_wait();
        }
        if (push) {  // the strip's boundary rows also go straight to the neighbour's ring
            for (int R = warp; R < a.by; R += nwarps) {
                uint32_t* const prow = peer_row(R);
                if (prow) prow[(gw + lane) & wmask] = sm[(R + 8) * 64 + 4 + lane];
            }
        }
    } else {
        for (int R = warp; R < a.by; R += nwarps) {
            uint32_t* __restrict__ row = f + uint32_t((Y0 + R) & rmask) * uint32_t(wpr);
            uint32_t* const prow = push ? peer_row(R) : nullptr;
            for (int k = lane; k <= Wt; k += 32) {
                if (k == Wt && b == 0) continue;  // would rewrite the unchanged right halo word
                const uint32_t v = __funnelshift_l(sm[sm_slot(R, k - 1)], sm[sm_slot(R, k)], b);
                row[(w0 + 1 + k) & wmask] = v;
                if (prow) prow[(w0 + 1 + k) & wmask] = v;
            }
        }
    }
    if (push) __threadfence_system();  // peer stores visible system-wide before the step signal
    // Counters: deposits, detaches, skipped attempts (sub = 4) per replica.
    ndep = __reduce_add_sync(0xFFFFFFFFu, ndep);
    if (GENERAL) ndet = __reduce_add_sync(0xFFFFFFFFu, ndet);
    nskip = __reduce_add_sync(0xFFFFFFFFu, (FULL || tx < Wt) ? nskip : 0u);
    if (lane == 0) {
        if (ndep) atomicAdd(a.counters + 2 * rep + 0, (unsigned long long)ndep);
        if (GENERAL && ndet) atomicAdd(a.counters + 2 * rep + 1, (unsigned long long)ndet);
        if (nskip) atomicAdd(a.skipped + rep, (unsigned long long)nskip);
    }
}

// DT phase kernel: one CTA per active block of phase a.phase.  WLOG: the
// debug instantiation that records every attempt for the write-set check.
// CHAIN: chained phase launches -- the CTA allows the next phase's launch to
// begin (programmatic dependent launch), waits (a.chain_wait) for the previous
// phase's blocks around it, and publishes its own completion in a.dflags.
template <bool GENERAL, bool FULL, int kNT, bool MW, bool WLOG = false, bool CHAIN = false>
__global__ void __launch_bounds__(MW ? (kNT == 2 && LFG_KPZ_MAXBY >= 256 ? 256 : 256 / kNT) : 32,
                                  MW ? (kNT == 1 || (kNT == 2 && LFG_KPZ_MAXBY >= 256) ? 3 : 6) : 12)
    kpz_dtr_phase_kernel(const __grid_constant__ KpzPhaseArgs a) {
    extern __shared__ __align__(16) uint32_t sm_raw[];
    if (!CHAIN && a.abort_flag && *reinterpret_cast<const volatile uint32_t*>(a.abort_flag)) return;
    const uint32_t sm_base = uint32_t(__cvta_generic_to_shared(sm_raw));
    const uint32_t smA = (sm_base - 1536u + 2047u) & ~2047u;  // shared address of line 0
    uint32_t* const sm = sm_raw + (int32_t(smA - sm_base) >> 2);  // generic pointer to line 0 (lines < 6 unused)
    const int rep = a.rep0 + int(blockIdx.z);
    const uint64_t seed = a.seeds[blockIdx.z];
    // sub-sweep draws of this replica (origin, this phase's block set), from the launcher
    const uint32_t swd = a.swd[blockIdx.z];
    const KpzSweep sw{int32_t(swd & 0xFFFu), int32_t((swd >> 12) & 0xFFFu), 0u};
    const int set = int(swd >> 24);
    if constexpr (!CHAIN) {
        kpz_block_activation<GENERAL, FULL, kNT, MW, WLOG>(a, sm, smA, rep, seed, sw, 2 * int(blockIdx.x) + (set & 1),
                                                     a.brow0 + 2 * int(blockIdx.y) + (set >> 1), 0u, true,
                                                     KpzDeps{nullptr, 1, 1, 0, 0, 0u});
    } else {
        asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
        const int nbx = a.L / a.bx, nby = a.L / a.by;
        // block rows start at row `phase` (mod rows): the first CTAs to start
        // depend on rows the previous phase finished early
        const int iy = int((blockIdx.y + uint32_t(a.phase)) & (gridDim.y - 1u));
        const int bxi = 2 * int(blockIdx.x) + (set & 1), byi = a.brow0 + 2 * iy + (set >> 1);
        uint32_t* const fl = a.dflags + size_t(rep) * size_t(nbx) * size_t(nby);
        // set(phase) ^ set(phase - 1) of this replica, precomputed by the launcher
        // (deriving it here from the sweep permutation costs the rounds their
        // uniform-datapath code generation)
        const int d = int((a.dd[blockIdx.z >> 5] >> (2 * (blockIdx.z & 31))) & 3u);
        const KpzDeps deps{a.chain_wait ? fl : nullptr, nbx, nby, d & 1, d >> 1, a.depoch};
        kpz_block_activation<GENERAL, FULL, kNT, MW, WLOG>(a, sm, smA, rep, seed, sw, bxi, byi, 0u, true, deps);
        __syncthreads();  // every warp's write-back issued before the release
        if (threadIdx.x == 0) {
            __threadfence();
            st_release_u32(fl + byi * nbx + bxi, a.depoch);
        }
    }
}

// Tiles per lane for a block height: the largest NT <= LFG_KPZ_NT with by >= 16 NT.
static int kpz_nt_for(int by) {
    int nt = LFG_KPZ_NT;
    while (nt > 1 && by < 16 * nt) nt >>= 1;
    return nt;
}

template <int NT, bool MW>
static void launch_cfg(const KpzPhaseArgs& b, dim3 grid, size_t smem, cudaStream_t st) {
    const dim3 block(unsigned(32 * (b.by / 16 / NT)));
    const bool full = b.bx == 1024;
    if (b.wlog && NT <= 2) {  // debug write-set recording (every plan, incl. the 1024-wide TMA path)
        if (full) {
            if (b.general) kpz_dtr_phase_kernel<true, true, NT, MW, true><<<grid, block, smem, st>>>(b);
            else kpz_dtr_phase_kernel<false, true, NT, MW, true><<<grid, block, smem, st>>>(b);
        } else {
            if (b.general) kpz_dtr_phase_kernel<true, false, NT, MW, true><<<grid, block, smem, st>>>(b);
            else kpz_dtr_phase_kernel<false, false, NT, MW, true><<<grid, block, smem, st>>>(b);
        }
        return;
    }
    if (b.dflags) {
        const auto kern = b.general ? (full ? kpz_dtr_phase_kernel<true, true, NT, MW, false, true>
                                            : kpz_dtr_phase_kernel<true, false, NT, MW, false, true>)
                                    : (full ? kpz_dtr_phase_kernel<false, true, NT, MW, false, true>
                                            : kpz_dtr_phase_kernel<false, false, NT, MW, false, true>);
        if (!(b.pdl && b.chain_wait)) {
            kern<<<grid, block, smem, st>>>(b);
            return;
        }
        // may start while the previous phase's last wave still runs
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = grid;
        cfg.blockDim = block;
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, kern, b);
        return;
    }
    const auto kern = b.general ? (full ? kpz_dtr_phase_kernel<true, true, NT, MW> : kpz_dtr_phase_kernel<true, false, NT, MW>)
                                : (full ? kpz_dtr_phase_kernel<false, true, NT, MW> : kpz_dtr_phase_kernel<false, false, NT, MW>);
    kern<<<grid, block, smem, st>>>(b);
}

template <int NT>
static void launch_nt(const KpzPhaseArgs& b, dim3 grid, size_t smem, cudaStream_t st) {
    if (b.by > 16 * NT) launch_cfg<NT, true>(b, grid, smem, st);
    else launch_cfg<NT, false>(b, grid, smem, st);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda).
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        cudaGetLastError();
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// 3-D map [replicas][rows][L/32] u32 over f, box 64 words x box_rows rows x 1.
static bool encode_rows_map(CUtensorMap* m, uint32_t* f, int L, int rows, int replicas, int box_rows) {
    auto enc = tensor_map_encoder();
    if (!enc || box_rows > 256) return false;
    const cuuint64_t dims[3] = {cuuint64_t(L / 32), cuuint64_t(rows), cuuint64_t(replicas)};
    const cuuint64_t strides[2] = {cuuint64_t(L / 32) * 4, cuuint64_t(L / 32) * 4 * cuuint64_t(rows)};
    const cuuint32_t box[3] = {64u, cuuint32_t(box_rows), 1u};
    const cuuint32_t estr[3] = {1u, 1u, 1u};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, f, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

cudaError_t kpz_launch_phase(const KpzPhaseArgs& a0, const uint64_t* seeds, int replicas, cudaStream_t st) {
    const size_t smem = kpz_phase_smem_bytes(a0.by);
    const int nt = kpz_nt_for(a0.by);
    KpzPhaseArgs a = a0;
    a.tma = 0;
    if (a.bx == 1024 && !std::getenv("LFG_KPZ_NO_TENSOR_MAP")) {
        const int rows = (a.L - 1 & a.row_mask) + 1;
        a.tma = encode_rows_map(&a.tm_ld, a.f, a.L, rows, replicas, a.by / 2 + 1) &&
                encode_rows_map(&a.tm_st, a.f, a.L, rows, replicas, a.by / 2);
    }
    for (int r0 = 0; r0 < replicas; r0 += kMaxRepPerLaunch) {
        KpzPhaseArgs b = a;
        b.rep0 = r0;
        const int nr = std::min(kMaxRepPerLaunch, replicas - r0);
        for (auto& w : b.dd) w = 0;
        for (int r = 0; r < nr; ++r) {
            b.seeds[r] = seeds[r0 + r];
            const KpzSweep sw = kpz_sweep_draw(a.bx, a.by, seeds[r0 + r], a.sweep);
            b.swd[r] = uint32_t(sw.ox) | (uint32_t(sw.oy) << 12) | (uint32_t(sw.set(a.phase)) << 24);
            if (b.dflags && b.chain_wait)
                b.dd[r >> 5] |= uint64_t(sw.set(a.phase) ^ sw.set(a.phase - 1)) << (2 * (r & 31));
        }
        const dim3 grid(unsigned(a.L / a.bx / 2), unsigned(a.nbrow / 2), unsigned(nr));
        if (nt >= 4) launch_nt<(LFG_KPZ_NT >= 4 ? 4 : 1)>(b, grid, smem, st);
        else if (nt == 2) launch_nt<2>(b, grid, smem, st);
        else launch_nt<1>(b, grid, smem, st);
    }
    return cudaGetLastError();
}


template <int NT, bool MW>
static cudaError_t attrs_cfg(int smem) {
    const cudaFuncAttribute at = cudaFuncAttributeMaxDynamicSharedMemorySize;
    if (NT <= 2) {
        cudaError_t e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<false, false, NT, MW, true>, at, smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<true, false, NT, MW, true>, at, smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<false, true, NT, MW, true>, at, smem);
        if (e == cudaSuccess) e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<true, true, NT, MW, true>, at, smem);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<false, true, NT, MW>, at, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<false, false, NT, MW>, at, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<true, true, NT, MW>, at, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<true, false, NT, MW>, at, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<false, true, NT, MW, false, true>, at, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<false, false, NT, MW, false, true>, at, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<true, true, NT, MW, false, true>, at, smem);
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kpz_dtr_phase_kernel<true, false, NT, MW, false, true>, at, smem);
    return e;
}

template <int NT>
static cudaError_t attrs_nt(int smem) {
    cudaError_t e = attrs_cfg<NT, true>(smem);
    if (e == cudaSuccess) e = attrs_cfg<NT, false>(smem);
    return e;
}

cudaError_t kpz_phase_kernel_attrs() {
    const int smem = int(kpz_phase_smem_bytes(LFG_KPZ_MAXBY));
    cudaError_t e = attrs_nt<1>(smem);
    if (e == cudaSuccess) e = attrs_nt<2>(smem);
    if (e == cudaSuccess && LFG_KPZ_NT >= 4) e = attrs_nt<4>(smem);
    if (e == cudaSuccess) e = kpz_width_kernel_attrs();
    return e;
}

// ============================================================ shard step barrier
__global__ void peer_signal_kernel(uint32_t* flag_a, uint32_t* flag_b, uint32_t value) {
    asm volatile("fence.sc.sys;" ::: "memory");
    if (flag_a) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag_a), "r"(value) : "memory");
    if (flag_b) asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(flag_b), "r"(value) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_sys(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void peer_wait_kernel(const uint32_t* flag_a, const uint32_t* flag_b, uint32_t value,
                                 unsigned long long max_spins, uint32_t* err) {
    for (unsigned long long n = 0;; ++n) {
        const bool a = !flag_a || int32_t(ld_acquire_sys(flag_a) - value) >= 0;
        const bool b = !flag_b || int32_t(ld_acquire_sys(flag_b) - value) >= 0;
        if (a && b) break;
        if (n >= max_spins) {  // a peer never arrived: report instead of hanging the stream
            if (err) atomicExch(err, 1u);
            break;
        }
        __nanosleep(200);
    }
}

cudaError_t peer_launch_signal(uint32_t* flag_a, uint32_t* flag_b, uint32_t value, cudaStream_t st) {
    peer_signal_kernel<<<1, 1, 0, st>>>(flag_a, flag_b, value);
    return cudaGetLastError();
}

cudaError_t peer_launch_wait(const uint32_t* flag_a, const uint32_t* flag_b, uint32_t value,
                             unsigned long long max_spins, uint32_t* err, cudaStream_t st) {
    peer_wait_kernel<<<1, 1, 0, st>>>(flag_a, flag_b, value, max_spins, err);
    return cudaGetLastError();
}

// ============================================================ init / convert
// Row-periodic spin patterns: word = pat[j & 3] for row j.
//   make_flat_slopes (lattice.cpp:71-82): f(i,j) = ((i+1)>>1 ^ (j+1)>>1) & 1
//   SlopeField(L) all-zero slopes (lattice.cpp:20-25): f(i,j) = (i+j) & 1
__global__ void kpz_init_pattern_kernel(uint32_t* f, int L, size_t nwords_total, uint4 pat) {
    const int wpr = L >> 5;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < nwords_total;
         k += size_t(gridDim.x) * blockDim.x) {
        const int j = int((k / size_t(wpr)) % size_t(L)) & 3;
        f[k] = j == 0 ? pat.x : (j == 1 ? pat.y : (j == 2 ? pat.z : pat.w));
    }
}

// Column-0 spins: f(0,j) = XOR_{k=1..j} ~sigma_y(0,k).  One CTA.
__global__ void kpz_col0_kernel(const uint32_t* __restrict__ Y, int L, uint8_t* __restrict__ f0) {
    __shared__ uint32_t part[1024];
    const int wpr = L >> 5;
    const int nt = blockDim.x, t = threadIdx.x;
    const int chunk = (L + nt - 1) / nt;
    const int j0 = t * chunk, j1 = min(L, j0 + chunk);
    uint32_t p = 0;
    for (int j = j0; j < j1; ++j)
        if (j > 0) p ^= (~Y[size_t(j) * wpr]) & 1u;
    part[t] = p;
    __syncthreads();
    // exclusive XOR scan over threads (serial over 1024 entries by thread 0 is cheap enough)
    if (t == 0) {
        uint32_t acc = 0;
        for (int k = 0; k < nt; ++k) {
            const uint32_t v = part[k];
            part[k] = acc;
            acc ^= v;
        }
    }
    __syncthreads();
    uint32_t acc = part[t];
    for (int j = j0; j < j1; ++j) {
        if (j > 0) acc ^= (~Y[size_t(j) * wpr]) & 1u;
        f0[j] = uint8_t(acc);
    }
}

__device__ __forceinline__ uint32_t prefix_xor32(uint32_t t) {
    t ^= t << 1;
    t ^= t << 2;
    t ^= t << 4;
    t ^= t << 8;
    t ^= t << 16;
    return t;
}

// Row spins: f(i,j) = f(0,j) ^ XOR_{k=1..i} ~sigma_x(k,j).  One warp per row.
__global__ void kpz_rows_from_slopes_kernel(const uint32_t* __restrict__ X, const uint8_t* __restrict__ f0,
                                            int L, uint32_t* __restrict__ f) {
    const int wpr = L >> 5;
    const int lane = threadIdx.x & 31;
    const int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (j >= L) return;
    const int cs = (wpr + 31) / 32;
    const int wbeg = lane * cs, wend = min(wpr, wbeg + cs);
    const uint32_t* __restrict__ xr = X + size_t(j) * wpr;
    uint32_t par = 0;
    for (int w = wbeg; w < wend; ++w) {
        uint32_t t = ~xr[w];
        if (w == 0) t &= ~1u;
        par ^= __popc(t) & 1u;
    }
    // exclusive XOR scan of parities across lanes
    uint32_t inc = par;
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc ^= v;
    }
    uint32_t carry = (inc ^ par) ^ uint32_t(f0[j]);
    uint32_t* __restrict__ fr = f + size_t(j) * wpr;
    for (int w = wbeg; w < wend; ++w) {
        uint32_t t = ~xr[w];
        if (w == 0) t &= ~1u;
        const uint32_t p = prefix_xor32(t);
        fr[w] = p ^ (carry ? 0xFFFFFFFFu : 0u);
        carry ^= p >> 31;
    }
}

// spins -> slopes, optionally comparing against given planes (mismatch count).
__global__ void kpz_spins_to_slopes_kernel(const uint32_t* __restrict__ f, int L, uint32_t* __restrict__ X,
                                           uint32_t* __restrict__ Y, const uint32_t* __restrict__ Xcmp,
                                           const uint32_t* __restrict__ Ycmp, unsigned long long* mismatch) {
    const int wpr = L >> 5, wmask = wpr - 1, Lm = L - 1;
    const size_t n = size_t(L) * wpr;
    unsigned long long bad = 0;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n; k += size_t(gridDim.x) * blockDim.x) {
        const int j = int(k / size_t(wpr)), w = int(k % size_t(wpr));
        const uint32_t F = f[k];
        const uint32_t Fp = f[size_t(j) * wpr + ((w - 1) & wmask)];
        const uint32_t Fd = f[size_t((j - 1) & Lm) * wpr + w];
        const uint32_t sx = ~(F ^ ((F << 1) | (Fp >> 31)));
        const uint32_t sy = ~(F ^ Fd);
        if (X) X[k] = sx;
        if (Y) Y[k] = sy;
        if (Xcmp) bad += __popc(sx ^ Xcmp[k]) + __popc(sy ^ Ycmp[k]);
    }
    if (mismatch) {
        bad = __reduce_add_sync(0xFFFFFFFFu, unsigned(bad));
        if ((threadIdx.x & 31) == 0 && bad) atomicAdd(mismatch, bad);
    }
}

cudaError_t kpz_launch_init_flat(uint32_t* f, int L, int replicas, cudaStream_t st) {
    const size_t n = size_t(replicas) * L * (L >> 5);
    const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    kpz_init_pattern_kernel<<<blocks, 256, 0, st>>>(f, L, n,
                                                    make_uint4(0x66666666u, 0x99999999u, 0x99999999u, 0x66666666u));
    return cudaGetLastError();
}

cudaError_t kpz_launch_init_zero_slopes(uint32_t* f, int L, int replicas, cudaStream_t st) {
    const size_t n = size_t(replicas) * L * (L >> 5);
    const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    kpz_init_pattern_kernel<<<blocks, 256, 0, st>>>(f, L, n,
                                                    make_uint4(0xAAAAAAAAu, 0x55555555u, 0xAAAAAAAAu, 0x55555555u));
    return cudaGetLastError();
}

cudaError_t kpz_launch_from_slopes(const uint32_t* X, const uint32_t* Y, int L, uint8_t* f0_scratch,
                                   uint32_t* f, cudaStream_t st) {
    kpz_col0_kernel<<<1, 1024, 0, st>>>(Y, L, f0_scratch);
    const int rows_per_block = 8;
    kpz_rows_from_slopes_kernel<<<(L + rows_per_block - 1) / rows_per_block, 32 * rows_per_block, 0, st>>>(
        X, f0_scratch, L, f);
    return cudaGetLastError();
}

cudaError_t kpz_launch_to_slopes(const uint32_t* f, int L, uint32_t* X, uint32_t* Y, const uint32_t* Xcmp,
                                 const uint32_t* Ycmp, unsigned long long* mismatch, cudaStream_t st) {
    const size_t n = size_t(L) * (L >> 5);
    const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    kpz_spins_to_slopes_kernel<<<blocks, 256, 0, st>>>(f, L, X, Y, Xcmp, Ycmp, mismatch);
    return cudaGetLastError();
}

// ============================================================ W^2 scan
// interface_width(const SlopeField&) (kpz.cpp:62-81): h(i,0) = sum_{k=1..i}
// s_x(k,0); h(i,j) = h(i,j-1) + s_y(i,j); exact int64 sum and sum of squares.
// Stage 1: row-0 heights H0[i] (one CTA).  Stage 2: the rows are cut into
// segments (global row ranges, in row order); per (segment, word column):
// relative column heights p (p = 0 on global row 0, otherwise the first row
// already adds its s_y), P1 = sum p per column, D = last p per column, and
// sum p^2 (global).  Stage 3: per column, walk the segments in row order:
//   sum h += len H + P1,   sum h^2 += len H^2 + 2 H P1,   H += D
// with H = H0 at row 0.  Segments may come from different strip shards.
__global__ void kpz_row0_heights_kernel(const uint32_t* __restrict__ f, int L, int32_t* __restrict__ H0) {
    __shared__ int32_t part[1024];
    const int wpr = L >> 5, wmask = wpr - 1;
    const int nt = blockDim.x, t = threadIdx.x;
    const int chunk = (L + nt - 1) / nt;
    const int i0 = t * chunk, i1 = min(L, i0 + chunk);
    auto sx = [&](int i) -> int32_t {  // slope_x(i, 0) for i >= 1
        const int w = i >> 5, bb = i & 31;
        const uint32_t F = f[w];
        const uint32_t left = bb ? (F >> (bb - 1)) : (f[(w - 1) & wmask] >> 31);
        return (((F >> bb) ^ left) & 1u) ? -1 : 1;
    };
    int32_t s = 0;
    for (int i = i0; i < i1; ++i)
        if (i > 0) s += sx(i);
    part[t] = s;
    __syncthreads();
    if (t == 0) {
        int32_t acc = 0;
        for (int k = 0; k < nt; ++k) {
            const int32_t v = part[k];
            part[k] = acc;
            acc += v;
        }
    }
    __syncthreads();
    int32_t acc = part[t];
    for (int i = i0; i < i1; ++i) {
        if (i > 0) acc += sx(i);
        H0[i] = acc;
    }
}

__global__ void __launch_bounds__(128) kpz_width_seg_kernel(const uint32_t* __restrict__ f, int L, int rmask,
                                                            int row_begin, int row_count, int S,
                                                            int32_t* __restrict__ P1, int32_t* __restrict__ D,
                                                            unsigned long long* __restrict__ sum_p2) {
    const int wpr = L >> 5, Lm = L - 1;
    const int w = blockIdx.x * blockDim.x + threadIdx.x;
    const int g = blockIdx.y;
    const int jl0 = g * S, n = min(S, row_count - jl0);
    int32_t p[32], s1[32];
#pragma unroll
    for (int c = 0; c < 32; ++c) { p[c] = 0; s1[c] = 0; }
    long long s2 = 0;
    if (w < wpr && n > 0) {
        const int jg0 = (row_begin + jl0) & Lm;
        uint32_t prev = f[size_t(((jg0 - 1) & Lm) & rmask) * wpr + w];
        for (int jl = 0; jl < n; ++jl) {
            const int jg = (jg0 + jl) & Lm;
            const uint32_t F = f[size_t(jg & rmask) * wpr + w];
            const uint32_t up = ~(F ^ prev);  // sigma_y(., jg) bits
            prev = F;
            const bool add = jg != 0;
            int32_t rowsq = 0;
#pragma unroll
            for (int c = 0; c < 32; ++c) {
                if (add) p[c] += ((up >> c) & 1u) ? 1 : -1;
                s1[c] += p[c];
                rowsq += p[c] * p[c];
            }
            s2 += rowsq;
        }
#pragma unroll
        for (int c = 0; c < 32; ++c) {
            P1[size_t(g) * L + 32 * w + c] = s1[c];
            D[size_t(g) * L + 32 * w + c] = p[c];
        }
    }
    for (int o = 16; o > 0; o >>= 1) s2 += __shfl_down_sync(0xFFFFFFFFu, s2, o);
    if ((threadIdx.x & 31) == 0 && s2) atomicAdd(sum_p2, (unsigned long long)s2);
}

__global__ void kpz_width_combine_kernel(const int32_t* __restrict__ H0, const int32_t* __restrict__ P1,
                                         const int32_t* __restrict__ D, const int32_t* __restrict__ seg_len,
                                         int L, int G, unsigned long long* __restrict__ out /* sum, sum2 */) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    long long sh = 0, sh2 = 0;
    if (c < L) {
        long long H = H0[c];
        for (int g = 0; g < G; ++g) {
            const long long q1 = P1[size_t(g) * L + c];
            const long long n = seg_len[g];
            sh += n * H + q1;
            sh2 += n * H * H + 2 * H * q1;
            H += D[size_t(g) * L + c];
        }
    }
    for (int o = 16; o > 0; o >>= 1) {
        sh += __shfl_down_sync(0xFFFFFFFFu, sh, o);
        sh2 += __shfl_down_sync(0xFFFFFFFFu, sh2, o);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(out + 0, (unsigned long long)sh);   // two's complement wraps exactly
        atomicAdd(out + 1, (unsigned long long)sh2);
    }
}

int kpz_width_segment_rows(int L) { return L >= 4096 ? 2048 : (L >= 256 ? 128 : L); }

cudaError_t kpz_launch_row0_heights(const uint32_t* row0, int L, int32_t* H0, cudaStream_t st) {
    kpz_row0_heights_kernel<<<1, 1024, 0, st>>>(row0, L, H0);
    return cudaGetLastError();
}

cudaError_t kpz_launch_width_partials(const uint32_t* f, int L, int rmask, int row_begin, int row_count, int S,
                                      int32_t* P1, int32_t* D, unsigned long long* sum_p2, cudaStream_t st) {
    const int wpr = L >> 5;
    const int G = (row_count + S - 1) / S;
    const dim3 g1(unsigned((wpr + 127) / 128), unsigned(G));
    kpz_width_seg_kernel<<<g1, 128, 0, st>>>(f, L, rmask, row_begin, row_count, S, P1, D, sum_p2);
    return cudaGetLastError();
}

cudaError_t kpz_launch_width_combine(const int32_t* H0, const int32_t* P1, const int32_t* D, const int32_t* seg_len,
                                     int L, int G, unsigned long long* out2, cudaStream_t st) {
    kpz_width_combine_kernel<<<(L + 255) / 256, 256, 0, st>>>(H0, P1, D, seg_len, L, G, out2);
    return cudaGetLastError();
}

cudaError_t kpz_launch_width(const uint32_t* f, int L, int32_t* H0, int32_t* P1, int32_t* D, int32_t* seg_len,
                             unsigned long long* out3, cudaStream_t st) {
    const int S = kpz_width_segment_rows(L);
    const int G = L / S;
    cudaError_t e = kpz_launch_row0_heights(f, L, H0, st);
    if (e == cudaSuccess) e = kpz_launch_width_partials(f, L, L - 1, 0, L, S, P1, D, out3 + 2, st);
    if (e == cudaSuccess) e = kpz_launch_width_combine(H0, P1, D, seg_len, L, G, out3, st);
    return e;
}

// Fill rows [row_begin, row_begin + row_count) (global, mod L) of a ring buffer
// with a row-periodic spin pattern (pattern word = pat[global row & 3]).
__global__ void kpz_fill_rows_kernel(uint32_t* f, int L, int rmask, int row_begin, int row_count, uint4 pat) {
    const int wpr = L >> 5, Lm = L - 1;
    const size_t n = size_t(row_count) * wpr;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n; k += size_t(gridDim.x) * blockDim.x) {
        const int jg = (row_begin + int(k / size_t(wpr))) & Lm;
        const int q = jg & 3;
        f[size_t(jg & rmask) * wpr + k % size_t(wpr)] = q == 0 ? pat.x : (q == 1 ? pat.y : (q == 2 ? pat.z : pat.w));
    }
}

cudaError_t kpz_launch_fill_rows(uint32_t* f, int L, int rmask, int row_begin, int row_count, int pattern,
                                 cudaStream_t st) {
    const uint4 pat = pattern == 0 ? make_uint4(0x66666666u, 0x99999999u, 0x99999999u, 0x66666666u)
                                   : make_uint4(0xAAAAAAAAu, 0x55555555u, 0xAAAAAAAAu, 0x55555555u);
    const size_t n = size_t(row_count) * (L >> 5);
    const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    kpz_fill_rows_kernel<<<blocks, 256, 0, st>>>(f, L, rmask, row_begin, row_count, pat);
    return cudaGetLastError();
}

// ============================================================ heights (small L)
// reconstruct_heights (kpz.cpp:21-34) on the device: row 0 from H0, then each
// column accumulates s_y.  Path-independence holds by construction for a
// spin field (kpz.cpp:35-47 is checked at upload).
__global__ void kpz_heights_kernel(const uint32_t* __restrict__ f, const int32_t* __restrict__ H0, int L,
                                   int32_t* __restrict__ h) {
    const int wpr = L >> 5, Lm = L - 1;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= L) return;
    int32_t v = H0[i];
    h[i] = v;
    const int w = i >> 5, bb = i & 31;
    uint32_t prev = (f[w] >> bb) & 1u;
    for (int j = 1; j < L; ++j) {
        const uint32_t cur = (f[size_t(j) * wpr + w] >> bb) & 1u;
        v += (cur == prev) ? 1 : -1;
        prev = cur;
        h[size_t(j) * L + i] = v;
    }
    (void)Lm;
}

cudaError_t kpz_launch_heights(const uint32_t* f, int L, int32_t* H0, int32_t* h, cudaStream_t st) {
    kpz_row0_heights_kernel<<<1, 1024, 0, st>>>(f, L, H0);
    kpz_heights_kernel<<<(L + 127) / 128, 128, 0, st>>>(f, H0, L, h);
    return cudaGetLastError();
}

}  // namespace lfg

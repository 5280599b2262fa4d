// kpz_width.cu -- sm_100a readouts of the KPZ spin lattice: the W^2 sums of
// interface_width(const SlopeField&) (kpz.cpp:62-81) and the closure checks of
// reconstruct_heights (kpz.cpp:35-47) applied at upload.
//
// W^2 by rows.  interface_width integrates the slopes along row 0 and then up
// every column (kpz.cpp:66-77).  Every lattice the device holds is locally
// closed -- each elementary plaquette closes: the init patterns do, an upload
// whose plaquettes do not is rejected (kpz_plaquette_kernel), and the octahedron
// move preserves every plaquette sum -- so the height of site (i, j) is the
// same along any path inside [0, L)^2 from (0, 0): up column 0, then along
// row j.  That order reads each row contiguously:
//   V(j)   = sum_{k=1..j} s_y(0, k)                        (kpz_width_tiles_kernel / kpz_width_chain_kernel)
//   h(i,j) = V(j) + sum_{k=1..i} s_x(k, j)                 (kpz_width_rows_kernel)
// and sum h, sum h^2 are exact int64, finished on the host as kpz.cpp:78-80.
//
// Row kernel: one warp per row, 256 words (8192 sites) per step, two 16-byte
// loads per lane.  A lane turns its eight spin words into s_x bits, then sums its
// 256 sites byte by byte from a 256-entry table of per-byte partial sums
// (S1 = sum of prefix heights, S2 = sum of their squares, D = net step), kept
// in 32 lane-private copies so the random table reads of a warp are
// conflict-free.  A warp scan of D gives every lane its start height; the lane
// partials (relative heights, 32-bit) are then shifted to absolute heights in
// 64-bit: sum (o + d) = n o + S1, sum (o + d)^2 = n o^2 + 2 o S1 + S2.
#include <algorithm>
#include <cstdint>

#include "kpz_kernels.cuh"

namespace lfg {

// Per-byte table entry (two words) for the 8 steps s_t = 2 b_t - 1 of a byte
// (bit t = +1 step) with prefix heights m_t = sum_{u <= t} s_u:
// S1 = sum m_t (-36..36), S2 = sum m_t^2 (0..204), D = m_7 (-8..8).
//   lo = S2 | (S1 + 36) << 13   -- summed over a lane's 32 bytes as one packed
//                                  word: S2 < 32 x 204 < 2^13, S1 + 36 < 32 x 72 < 2^12
//   hi = D << 22 + (S1 + 36)    -- D as a signed top field: hi >> 22 (arithmetic)
//                                  is D, and o x hi = o (S1 + 36) mod 2^22
__device__ __forceinline__ uint2 width_byte_entry(uint32_t v) {
    int m = 0, s1 = 0, s2 = 0;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
        m += ((v >> t) & 1u) ? 1 : -1;
        s1 += m;
        s2 += m * m;
    }
    return make_uint2(uint32_t(s2) | (uint32_t(s1 + 36) << 13), (uint32_t(m) << 22) + uint32_t(s1 + 36));
}

constexpr int kWidthRowWarps = 16;         // warps per CTA of the row pass
constexpr size_t kWidthTableBytes = 65536;  // 256 entries x 32 lanes x 8 bytes

// Row pass (kpz_width_rows_kernel): one warp per row, 256 words (8192 sites)
// per step, 8 consecutive words (two 16-byte loads) per lane.  A lane turns its
// words into s_x bits and walks its 32 bytes with the running offset o (height
// before the byte, relative to the lane's first site); with the byte's table
// entry (S1, S2, D)
//   sum over the byte of (o + m_t)   = 8 o + S1
//   sum over the byte of (o + m_t)^2 = 8 o^2 + 2 o S1 + S2,
// so per byte it needs o, o^2 and o S1 (one IMAD each against the entry's hi
// word), o += D (one LEA.HI of the hi word), and one packed add of the lo word.
// Table: entry v of lane l at byte v * 256 + l * 8 -- the address is one PRMT
// of the byte and 8 l, and the 32 lanes' 8-byte reads of a warp cover 256
// consecutive bytes (conflict-free).  A warp scan of the lanes' net steps gives
// their start heights.  Per row the pass stores (sum h, sum h^2) relative to
// the row's column-0 height and the column-0 step into the row
// (kpz_width_tiles_kernel / _chain_kernel chain them: no serial column pass on
// the critical path).
template <bool VEC>
__global__ void __launch_bounds__(32 * kWidthRowWarps) kpz_width_rows_kernel(const uint32_t* __restrict__ f, int L,
                                                                             int rmask, int row_begin, int n,
                                                                             long long* __restrict__ rs,
                                                                             int32_t* __restrict__ rstep) {
    extern __shared__ uint2 tab[];  // kWidthTableBytes
    for (int v = threadIdx.x; v < 256; v += blockDim.x) {
        const uint2 e = width_byte_entry(uint32_t(v));
#pragma unroll 8
        for (int l = 0; l < 32; ++l) tab[v * 32 + ((l + v) & 31)] = e;  // rotated: the 32 stores of a warp hit distinct banks
    }
    __syncthreads();
    const int wpr = L >> 5, Lm = L - 1;
    const int lane = threadIdx.x & 31;
    const uint32_t lane8 = uint32_t(lane) * 8u;  // byte 0 of every table address
    const char* const tabc = reinterpret_cast<const char*>(tab);
    // grid-stride over rows (the grid is sized to the resident CTAs, so each
    // CTA builds its table once)
    for (int k = int(blockIdx.x) * kWidthRowWarps + int(threadIdx.x >> 5); k < n; k += int(gridDim.x) * kWidthRowWarps) {
        const int g = (row_begin + k) & Lm;
        const uint32_t* __restrict__ row = f + size_t(g & rmask) * wpr;
        int32_t base = -1;   // site 0 enters as a +1 step from -1: heights relative to h(0, g)
        uint32_t top = 0;    // bit 31 of the previous chunk's last word
        long long s1 = 0, s2 = 0;
        for (int c = 0; c < wpr; c += 256) {
            uint32_t F[8];
            int nw = 8;  // valid words of this lane (all eight when VEC)
            if (VEC) {
                const uint4 q0 = __ldg(reinterpret_cast<const uint4*>(row + c + 8 * lane));
                const uint4 q1 = __ldg(reinterpret_cast<const uint4*>(row + c + 8 * lane + 4));
                F[0] = q0.x; F[1] = q0.y; F[2] = q0.z; F[3] = q0.w;
                F[4] = q1.x; F[5] = q1.y; F[6] = q1.z; F[7] = q1.w;
            } else {
                const int w0 = c + 8 * lane;
                nw = max(0, min(8, wpr - w0));
#pragma unroll
                for (int u = 0; u < 8; ++u) F[u] = u < nw ? row[w0 + u] : 0u;
            }
            // bit 31 of the word before this lane's first: the previous lane's
            // last valid word (zero-filled words never precede a valid one)
            const uint32_t prev_lane = __shfl_up_sync(0xFFFFFFFFu, F[7], 1);
            uint32_t prev = lane == 0 ? top : prev_lane;
            top = __shfl_sync(0xFFFFFFFFu, F[7], 31);
            int32_t o = 0, so = 0, so2 = 0;
            uint32_t sos1 = 0;  // sum o (S1 + 36) mod 2^22 in the low bits
            uint32_t pk = 0;    // packed sums of the lo words
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                uint32_t X = ~(F[u] ^ __funnelshift_l(prev, F[u], 1));  // bit b: s_x of site b is +1
                prev = F[u];
                if (u == 0 && c == 0 && lane == 0) X |= 1u;
                if (!VEC && u >= nw) continue;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    uint32_t off;  // byte 0 = 8 lane, byte 1 = byte b of X
                    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(off) : "r"(X), "r"(lane8), "r"(0x5504u | (uint32_t(b) << 4)));
                    const uint2 e = *reinterpret_cast<const uint2*>(tabc + off);
                    so += o;
                    so2 += o * o;
                    sos1 += uint32_t(o) * e.y;
                    pk += e.x;
                    o += int32_t(e.y) >> 22;
                }
            }
            const int32_t nb = VEC ? 32 : 4 * nw;  // bytes summed (bias removal)
            const int32_t sumS1 = int32_t(pk >> 13) - 36 * nb;
            const int32_t sumS2 = int32_t(pk & 0x1FFFu);
            // sum o (S1 + 36): |.| <= 256 x 72 x 32 < 2^21, sign-extended from 22 bits
            const int32_t sos1x = int32_t(sos1 << 10) >> 10;
            // a1 = sum of (o_b + m_t) over the lane's sites, a2 = sum of squares
            const int32_t a1 = 8 * so + sumS1;
            const int32_t a2 = 8 * so2 + 2 * (sos1x - 36 * so) + sumS2;
            const int32_t nsites = 8 * nb;
            // lane start heights: exclusive warp scan of o (net step of each lane)
            int32_t inc = o;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, d);
                if (lane >= d) inc += v;
            }
            const int32_t O = base + inc - o;
            base += __shfl_sync(0xFFFFFFFFu, inc, 31);
            s1 += (long long)nsites * O + a1;
            s2 += (long long)O * (long long)(nsites * O + 2 * a1) + a2;
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) {
            s1 += __shfl_down_sync(0xFFFFFFFFu, s1, d);
            s2 += __shfl_down_sync(0xFFFFFFFFu, s2, d);
        }
        if (lane == 0) {
            rs[2 * size_t(k)] = s1;
            rs[2 * size_t(k) + 1] = s2;
            // column-0 step into row g (interface_width anchors h(0, 0) = 0: none into row 0)
            int32_t stp = 0;
            if (g != 0) {
                const uint32_t a = row[0] & 1u;
                const uint32_t bb = f[size_t(((g - 1) & Lm) & rmask) * wpr] & 1u;
                stp = a == bb ? 1 : -1;
            }
            rstep[k] = stp;
        }
    }
}

// Chain the row sums of rows k < n in order.  V_k = sum_{m <= k} step_m is the
// column-0 height of row k relative to the row below the piece;
//   sum h   += L V_k + S1_k,   sum h^2 += L V_k^2 + 2 V_k S1_k + S2_k.
// Two levels, coalesced: tile pass (one CTA per 1024 consecutive rows; thread =
// row) with v = V relative to the tile start, storing per tile
//   D = sum step, A0 = sum (L v + S1), A1 = sum v, A2 = sum (L v^2 + 2 v S1 + S2), B = sum S1;
// then one warp chains the tiles with carries c (V = c + v):
//   sum h += n L c + A0,   sum h^2 += L (n c^2 + 2 c A1) + 2 c B + A2.
// out3[0] += sum h, out3[1] += sum h^2, out3[2] = V_{n-1} (the piece's net step).
constexpr int kWidthTile = 1024;

__global__ void __launch_bounds__(kWidthTile) kpz_width_tiles_kernel(const long long* __restrict__ rs,
                                                                     const int32_t* __restrict__ rstep, int L, int n,
                                                                     long long* __restrict__ tiles) {
    __shared__ int32_t wsum[32];
    __shared__ long long red[4][32];
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
    const int k = int(blockIdx.x) * kWidthTile + t;
    const bool in = k < n;
    const int32_t st = in ? rstep[k] : 0;
    int32_t inc = st;  // inclusive block scan of the steps
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int32_t v = __shfl_up_sync(0xFFFFFFFFu, inc, o);
        if (lane >= o) inc += v;
    }
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        const int32_t w = wsum[lane];
        int32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int32_t v = __shfl_up_sync(0xFFFFFFFFu, wi, o);
            if (lane >= o) wi += v;
        }
        wsum[lane] = wi;  // inclusive
    }
    __syncthreads();
    const long long v = (warp ? wsum[warp - 1] : 0) + inc;
    const long long S1 = in ? rs[2 * size_t(k)] : 0, S2 = in ? rs[2 * size_t(k) + 1] : 0;
    long long q[4] = {in ? (long long)L * v + S1 : 0, in ? v : 0, in ? (long long)L * v * v + 2 * v * S1 + S2 : 0, S1};
#pragma unroll
    for (int i = 0; i < 4; ++i) {
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) q[i] += __shfl_down_sync(0xFFFFFFFFu, q[i], d);
        if (lane == 0) red[i][warp] = q[i];
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            long long x = red[i][lane];
#pragma unroll
            for (int d = 16; d > 0; d >>= 1) x += __shfl_down_sync(0xFFFFFFFFu, x, d);
            if (lane == 0) tiles[6 * size_t(blockIdx.x) + 1 + i] = x;
        }
        if (lane == 0) tiles[6 * size_t(blockIdx.x)] = wsum[31];
    }
}

__global__ void __launch_bounds__(32) kpz_width_chain_kernel(const long long* __restrict__ tiles, int ntiles, int L,
                                                             int n, unsigned long long* __restrict__ out3) {
    const int lane = threadIdx.x;
    long long carry = 0, t1 = 0, t2 = 0;
    for (int b = 0; b < ntiles; b += 32) {
        const int i = b + lane;
        const bool in = i < ntiles;
        const long long D = in ? tiles[6 * size_t(i)] : 0;
        long long incl = D;  // inclusive warp scan of the tile steps
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const long long x = __shfl_up_sync(0xFFFFFFFFu, incl, o);
            if (lane >= o) incl += x;
        }
        const long long c = carry + incl - D;  // V at the row below tile i
        if (in) {
            const long long nt = min(kWidthTile, n - i * kWidthTile);
            const long long A0 = tiles[6 * size_t(i) + 1], A1 = tiles[6 * size_t(i) + 2];
            const long long A2 = tiles[6 * size_t(i) + 3], B = tiles[6 * size_t(i) + 4];
            t1 += nt * L * c + A0;
            t2 += (long long)L * (nt * c * c + 2 * c * A1) + 2 * c * B + A2;
        }
        carry += __shfl_sync(0xFFFFFFFFu, incl, 31);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        t1 += __shfl_down_sync(0xFFFFFFFFu, t1, d);
        t2 += __shfl_down_sync(0xFFFFFFFFu, t2, d);
    }
    if (lane == 0) {
        atomicAdd(out3 + 0, (unsigned long long)t1);
        atomicAdd(out3 + 1, (unsigned long long)t2);
        out3[2] = (unsigned long long)carry;
    }
}

cudaError_t kpz_width_kernel_attrs() {  // 64 KB of dynamic shared memory (table)
    cudaError_t e = cudaFuncSetAttribute(kpz_width_rows_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(kWidthTableBytes));
    if (e == cudaSuccess)
        e = cudaFuncSetAttribute(kpz_width_rows_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 int(kWidthTableBytes));
    return e;
}

size_t kpz_width_scratch_bytes(int row_count) {
    const size_t ntiles = (size_t(row_count) + kWidthTile - 1) / kWidthTile;
    return size_t(row_count) * 20 + ntiles * 48 + 64;
}

cudaError_t kpz_launch_width_rows(const uint32_t* f, int L, int rmask, int row_begin, int row_count, void* scratch,
                                  unsigned long long* out3, cudaStream_t st) {
    long long* rs = static_cast<long long*>(scratch);
    long long* tiles = rs + 2 * size_t(row_count);  // [ntiles][6]
    const int ntiles = (row_count + kWidthTile - 1) / kWidthTile;
    int32_t* rstep = reinterpret_cast<int32_t*>(tiles + 6 * size_t(ntiles));
    constexpr int wpb = kWidthRowWarps;
    // resident CTAs: 64 KB of table each -> 3 per SM; 148 SMs
    const unsigned grid = unsigned(std::min((row_count + wpb - 1) / wpb, 148 * 3));
    if (grid > 0) {
        if ((L >> 5) % 256 == 0)
            kpz_width_rows_kernel<true>
                <<<grid, 32 * wpb, kWidthTableBytes, st>>>(f, L, rmask, row_begin, row_count, rs, rstep);
        else
            kpz_width_rows_kernel<false>
                <<<grid, 32 * wpb, kWidthTableBytes, st>>>(f, L, rmask, row_begin, row_count, rs, rstep);
    }
    if (ntiles > 0) kpz_width_tiles_kernel<<<unsigned(ntiles), kWidthTile, 0, st>>>(rs, rstep, L, row_count, tiles);
    kpz_width_chain_kernel<<<1, 32, 0, st>>>(tiles, ntiles, L, row_count, out3);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- closure
// Upload check of two slope planes X, Y (uint32 words of the reference layout)
// against reconstruct_heights' path-independence (kpz.cpp:35-47):
//   local:  every elementary plaquette closes,
//           s_x(i, j-1) + s_y(i, j) == s_y(i-1, j) + s_x(i, j)   (periodic indices)
//           -> bad plaquettes counted into local_bad;
//   global: row 0's s_x and column 0's s_y sum to zero (with local closure,
//           every row / column then does) -> deviations counted into global_bad.
// A locally closed field with nonzero row sums (e.g. the all -1 field of
// SlopeField(L), lattice.cpp:20-25) is representable and swept exactly, but
// reconstruct_heights rejects it.
__global__ void kpz_plaquette_kernel(const uint32_t* __restrict__ X, const uint32_t* __restrict__ Y, int L,
                                     unsigned long long* __restrict__ local_bad) {
    const int wpr = L >> 5, wmask = wpr - 1, Lm = L - 1;
    const size_t n = size_t(L) * wpr;
    unsigned long long bad = 0;
    for (size_t k = blockIdx.x * size_t(blockDim.x) + threadIdx.x; k < n; k += size_t(gridDim.x) * blockDim.x) {
        const int j = int(k / size_t(wpr)), w = int(k % size_t(wpr));
        const uint32_t c = X[k];                                              // s_x(i, j)
        const uint32_t a = X[size_t((j - 1) & Lm) * wpr + w];                 // s_x(i, j-1)
        const uint32_t b = Y[k];                                              // s_y(i, j)
        const uint32_t d = (b << 1) | (Y[size_t(j) * wpr + ((w - 1) & wmask)] >> 31);  // s_y(i-1, j)
        // two-bit sums a + b and c + d must agree
        bad += __popc(((a ^ b) ^ (c ^ d)) | ((a & b) ^ (c & d)));
    }
    bad = __reduce_add_sync(0xFFFFFFFFu, unsigned(bad));
    if ((threadIdx.x & 31) == 0 && bad) atomicAdd(local_bad, bad);
}

__global__ void __launch_bounds__(1024) kpz_closure_sums_kernel(const uint32_t* __restrict__ X,
                                                                const uint32_t* __restrict__ Y, int L,
                                                                unsigned long long* __restrict__ global_bad) {
    __shared__ int part[2][32];
    const int wpr = L >> 5;
    int rx = 0, cy = 0;  // ones in row 0 of X, in column 0 of Y
    for (int w = threadIdx.x; w < wpr; w += blockDim.x) rx += __popc(X[w]);
    for (int j = threadIdx.x; j < L; j += blockDim.x) cy += int(Y[size_t(j) * wpr] & 1u);
    rx = __reduce_add_sync(0xFFFFFFFFu, rx);
    cy = __reduce_add_sync(0xFFFFFFFFu, cy);
    if ((threadIdx.x & 31) == 0) {
        part[0][threadIdx.x >> 5] = rx;
        part[1][threadIdx.x >> 5] = cy;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int sx = 0, sy = 0;
        for (int k = 0; k < int(blockDim.x >> 5); ++k) {
            sx += part[0][k];
            sy += part[1][k];
        }
        if (2 * sx != L || 2 * sy != L) atomicAdd(global_bad, 1ull);
    }
}

cudaError_t kpz_launch_closure_check(const uint32_t* X, const uint32_t* Y, int L, unsigned long long* local_bad,
                                     unsigned long long* global_bad, cudaStream_t st) {
    const size_t n = size_t(L) * (L >> 5);
    const int blocks = int(std::min<size_t>((n + 255) / 256, 148 * 16));
    kpz_plaquette_kernel<<<blocks, 256, 0, st>>>(X, Y, L, local_bad);
    kpz_closure_sums_kernel<<<1, 1024, 0, st>>>(X, Y, L, global_bad);
    return cudaGetLastError();
}

}  // namespace lfg

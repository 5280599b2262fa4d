// scripts/explore/dt_explore.cu -- RESEARCH TOOL, not product, not oracle.
//
// Fast ensemble probe of decomposition schemes for the KPZ octahedron model
// (p = 1, q = 0, flat start) on one B200.  Each replica is one CTA with its
// lattice of int8 heights (mod 256) in shared memory (L <= 256) or global
// memory; W^2 is taken from the height differences to site (0,0), <h> from
// the deposit count.  Schemes:
//
//   rs   random-sequential sweep (kpz.cpp:5-19 semantics, Philox draws): one
//        lane per replica, L^2 attempts per MCS at uniform sites.
//   dt   two-layer DTr as in DESIGN.md §2.1 (blocks bx x by in a frame shifted
//        by a fresh origin every sweep, random set order, 32x16 tiles, 16x8
//        domains, block-uniform inner set per round) with knobs:
//          --mini m     m mini-sweeps per MCS (origin + order re-drawn each,
//                       512/m rounds per activation)
//          --counts c   0: every tile one attempt per round (512 per activation)
//                       1: per-tile attempt count N_t ~ Poisson(512/m) per
//                          activation (normal approx.), rounds = block max
//                       2: two-point N_t in {c, c-d} with P(c) = pt and
//                          var = mean (c = mu + d(1-pt), d = sqrt(mu/(pt(1-pt))))
//                       3: normal(mu, mu) clipped at mu + cap*sigma
//          --skip s     0: a tile's idle rounds are the last ones; 1: spread
//          --thin l     each tile attempts with probability l per round,
//                       round count 512/(m l)
//
// The attempt rule is kpz.hpp:71-107 in the height picture: the anchor site
// is a local minimum (all four neighbours one higher) -> h += 2.
//
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o dt_explore dt_explore.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <cmath>
#include <string>
#include <vector>
#include <curand_kernel.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
    fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); exit(1); } } while (0)

struct Cfg {
    int L = 256, bx = 128, by = 128, mini = 1, counts = 0, skip = 0;
    float thin = 1.f, pt = 0.9f, cap = 2.f;
    int tc = 0, td = 0, tlog = 4;
    int oxq = 1;                    // x-origin quantum (sites)   // counts 4: N = tc - td with probability 2^-tlog, else tc
    int replicas = 4096;
    unsigned long long seed = 1;
    int nt = 0;
    int ts[64];
};

__device__ __forceinline__ int8_t& at(int8_t* H, int L, int x, int y) { return H[y * L + x]; }

__device__ void sample(int8_t* H, const Cfg& c, long long dep, int slot, double* out_w2, double* out_h,
                       int replica) {
    // W^2 over d = (int8)(h - h(0,0)); block reduction by lane 0 over shared partials
    __shared__ long long s1[32], s2[32];
    const int L = c.L;
    const int8_t ref = H[0];
    long long a = 0, b = 0;
    for (int k = threadIdx.x; k < L * L; k += blockDim.x) {
        const int d = int(int8_t(H[k] - ref));
        a += d;
        b += d * d;
    }
    for (int o = 16; o; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
    }
    if ((threadIdx.x & 31) == 0) { s1[threadIdx.x >> 5] = a; s2[threadIdx.x >> 5] = b; }
    __syncthreads();
    if (threadIdx.x == 0) {
        long long A = 0, B = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) { A += s1[w]; B += s2[w]; }
        const double n = double(L) * L;
        const double m = A / n;
        out_w2[size_t(replica) * c.nt + slot] = B / n - m * m;
        out_h[size_t(replica) * c.nt + slot] = 2.0 * double(dep) / n;
    }
    __syncthreads();
}

__device__ __forceinline__ bool attempt(int8_t* H, int L, int x, int y) {
    const int m = L - 1;
    const int8_t h = at(H, L, x, y);
    const int8_t h1 = h + 1;
    if (at(H, L, (x + 1) & m, y) == h1 && at(H, L, (x - 1) & m, y) == h1 &&
        at(H, L, x, (y + 1) & m) == h1 && at(H, L, x, (y - 1) & m) == h1) {
        at(H, L, x, y) = int8_t(h + 2);
        return true;
    }
    return false;
}

__device__ void flat(int8_t* H, int L) {
    for (int k = threadIdx.x; k < L * L; k += blockDim.x) H[k] = int8_t(((k % L) + (k / L)) & 1);
    __syncthreads();
}

extern __shared__ int8_t g_smem[];

__global__ void rs_kernel(Cfg c, int8_t* gH, double* w2, double* hm) {
    const int rep = blockIdx.x;
    const int L = c.L;
    int8_t* H = L <= 256 ? g_smem : gH + size_t(rep) * L * L;
    flat(H, L);
    curandStatePhilox4_32_10_t st;
    curand_init(c.seed, rep, 0, &st);
    long long dep = 0;
    int t = 0;
    const int lg = __ffs(L) - 1;
    for (int s = 0; s < c.nt; ++s) {
        if (threadIdx.x == 0) {
            const long long n = (long long)(c.ts[s] - t) * L * L;
            for (long long a = 0; a < n; a += 2) {
                const uint4 u = curand4(&st);
                // multiply-shift bounded draws (rng.hpp:130-134 semantics)
                const int x0 = int((uint64_t(u.x) * L) >> 32), y0 = int((uint64_t(u.y) * L) >> 32);
                dep += attempt(H, L, x0, y0);
                const int x1 = int((uint64_t(u.z) * L) >> 32), y1 = int((uint64_t(u.w) * L) >> 32);
                dep += attempt(H, L, x1, y1);
            }
            (void)lg;
        }
        t = c.ts[s];
        __syncthreads();
        sample(H, c, dep, s, w2, hm, rep);
    }
}

// DT: threads cover the active tiles of one phase.
__global__ void dt_kernel(Cfg c, int8_t* gH, double* w2, double* hm) {
    const int rep = blockIdx.x;
    const int L = c.L, mask = L - 1;
    int8_t* H = L <= 256 ? g_smem : gH + size_t(rep) * L * L;
    flat(H, L);
    __shared__ uint8_t sets[2048];
    __shared__ int s_rounds;
    __shared__ int s_ox, s_oy, s_perm[4];
    __shared__ long long s_dep[32];
    __shared__ int s_mn[256];
    curandStatePhilox4_32_10_t st;      // per thread
    curand_init(c.seed, uint64_t(rep) * 4096 + threadIdx.x, 0, &st);
    curandStatePhilox4_32_10_t cs;      // CTA-level draws (thread 0)
    curand_init(c.seed ^ 0x9E3779B97F4A7C15ull, rep, 0, &cs);
    const int nbx = L / c.bx, nby = L / c.by;
    const int twx = c.bx / 32, thy = c.by / 16, ntile = twx * thy;
    const int act_blocks = (nbx / 2) * (nby / 2);
    const int nact = act_blocks * ntile;       // active tiles per phase
    const double mean_n = 512.0 / c.mini;
    const int base_rounds = int(lrint(mean_n / c.thin));
    long long dep = 0;
    int t = 0;
    for (int s = 0; s < c.nt; ++s) {
        const int nms = (c.ts[s] - t) * c.mini;
        for (int ms = 0; ms < nms; ++ms) {
            if (threadIdx.x == 0) {
                const uint4 u = curand4(&cs);
                s_ox = c.oxq * int((uint64_t(u.x) * (2 * c.bx / c.oxq)) >> 32);
                s_oy = int((uint64_t(u.y) * (2 * c.by)) >> 32);
                int pool[4] = {0, 1, 2, 3};
                for (int k = 3; k > 0; --k) {  // Fisher-Yates
                    const int j = int((uint64_t(curand(&cs)) * (k + 1)) >> 32);
                    const int tmp = pool[k]; pool[k] = pool[j]; pool[j] = tmp;
                }
                for (int k = 0; k < 4; ++k) s_perm[k] = pool[k];
            }
            __syncthreads();
            for (int ph = 0; ph < 4; ++ph) {
                const int set = s_perm[ph], sx = set & 1, sy = set >> 1;
                // per-tile counts
                int my_n[8];
                uint32_t my_mask_k[8] = {0, 0, 0, 0, 0, 0, 0, 0};
                int tiles = 0;
                if (threadIdx.x == 0) s_rounds = 0;
                if (c.counts == 6) {
                    for (int a = threadIdx.x; a < nact; a += blockDim.x) s_mn[a] = 0;
                    __syncthreads();
                    if (threadIdx.x == 0) {
                        for (int blk = 0; blk < act_blocks; ++blk)
                            for (int k = 0; k < int(mean_n) * ntile; ++k) {
                                const int t = int((uint64_t(curand(&cs)) * ntile) >> 32);
                                ++s_mn[blk * ntile + t];
                            }
                    }
                }
                __syncthreads();
                for (int a = threadIdx.x; a < nact; a += blockDim.x, ++tiles) {
                    int n = base_rounds;
                    if (c.counts == 1 || c.counts == 3) {
                        const float g = curand_normal(&st);
                        const double sg = sqrt(mean_n), k = c.cap;
                        // counts 3: shift the mean up by the clipped excess sigma (phi(k) - k Q(k))
                        const double sh = c.counts == 3
                            ? sg * (exp(-0.5 * k * k) * 0.3989422804 - k * 0.5 * erfc(k * 0.7071067812)) : 0.0;
                        n = int(lrint(mean_n + sh + sg * g));
                        if (c.counts == 3) n = min(n, int(lrint(mean_n + sh + k * sg)));
                        n = max(0, min(n, 2047));
                    } else if (c.counts == 7) {
                        // generic Poisson law: N = tc - td K, K ~ Poisson((tc - mu) / td) by inversion
                        const double lam = (c.tc - mean_n) / c.td;
                        const double u = curand_uniform_double(&st);
                        double pk = exp(-lam), cdf = pk;
                        int K = 0;
                        while (u > cdf && K < 64) { ++K; pk *= lam / K; cdf += pk; }
                        n = max(0, c.tc - c.td * K);
                    } else if (c.counts == 6) {
                        n = s_mn[a];
                    } else if (c.counts == 5) {
                        const uint32_t v = curand(&st) >> 16;
                        const int K = (v >= 57835u) + (v >= 65065u) + (v >= 65517u) + (v >= 65535u);
                        n = 132 - 32 * K;
                        my_mask_k[tiles] = ((0xFEA80u >> (4 * K)) & 0xFu) * 0x11111111u;
                    } else if (c.counts == 4) {
                        n = (curand(&st) >> (32 - c.tlog)) == 0 ? c.tc - c.td : c.tc;
                    } else if (c.counts == 2) {
                        const double d = sqrt(mean_n / (c.pt * (1.0 - c.pt)));
                        const double top = mean_n + d * (1.0 - c.pt);
                        // integer two-point: top rounded, low = top - round(d)
                        const int ct = int(lrint(top)), dd = int(lrint(d));
                        n = (curand_uniform(&st) <= c.pt) ? ct : ct - dd;
                    }
                    my_n[tiles] = n;
                    atomicMax(&s_rounds, n);
                }
                __syncthreads();
                const int R = s_rounds;
                if (threadIdx.x == 0) {
                    for (int r = 0; r < R; r += 16) {
                        const uint32_t v = curand(&cs);
                        for (int k = 0; k < 16 && r + k < R; ++k) sets[r + k] = uint8_t((v >> (2 * k)) & 3u);
                    }
                }
                __syncthreads();
                for (int r = 0; r < R; ++r) {
                    const int inner = sets[r], hx = inner & 1, hy = inner >> 1;
                    int k = 0;
                    for (int a = threadIdx.x; a < nact; a += blockDim.x, ++k) {
                        if (c.counts == 5) {
                            if (r < 128 && ((my_mask_k[k] >> (r >> 2)) & 1u)) continue;
                        } else if (c.skip == 0) {
                            if (r >= my_n[k]) continue;
                        } else if (c.skip == 2) {  // spread at 4-round group granularity
                            if (my_n[k] < R) {
                                const int G = R / 4, idle = (R - my_n[k]) / 4, g = r / 4;
                                if ((long long)(g + 1) * idle / G != (long long)g * idle / G) continue;
                            }
                        } else if (my_n[k] < R) {  // spread the R - n idle rounds evenly
                            const int idle = R - my_n[k];
                            if ((long long)(r + 1) * idle / R != (long long)r * idle / R) continue;
                        }
                        const uint4 u = curand4(&st);
                        if (c.thin < 1.f && float(u.z) * 2.3283064e-10f >= c.thin) continue;
                        const int blk = a / ntile, tl = a % ntile;
                        const int abx = sx + 2 * (blk % (nbx / 2)), aby = sy + 2 * (blk / (nbx / 2));
                        const int tx = tl % twx, ty = tl / twx;
                        const int xd = int((uint64_t(u.x) * 16) >> 32), yd = int((uint64_t(u.y) * 8) >> 32);
                        const int xs = abx * c.bx + tx * 32 + hx * 16 + xd;
                        const int ys = aby * c.by + ty * 16 + hy * 8 + yd;
                        dep += attempt(H, L, (xs + s_ox) & mask, (ys + s_oy) & mask);
                    }
                    __syncthreads();
                }
            }
        }
        t = c.ts[s];
        // total deposits over threads
        long long d = dep;
        for (int o = 16; o; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
        if ((threadIdx.x & 31) == 0) s_dep[threadIdx.x >> 5] = d;
        __syncthreads();
        long long D = 0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) D += s_dep[w];
        __syncthreads();
        sample(H, c, D, s, w2, hm, rep);
    }
}

int main(int argc, char** argv) {
    Cfg c;
    std::string scheme = "dt", out = "explore.json";
    int tmax = 100;
    for (int i = 1; i < argc; ++i) {
        std::string a = argv[i];
        auto nx = [&]() { return std::string(argv[++i]); };
        if (a == "--scheme") scheme = nx();
        else if (a == "--L") c.L = std::stoi(nx());
        else if (a == "--bx") c.bx = std::stoi(nx());
        else if (a == "--by") c.by = std::stoi(nx());
        else if (a == "--mini") c.mini = std::stoi(nx());
        else if (a == "--counts") c.counts = std::stoi(nx());
        else if (a == "--thin") c.thin = std::stof(nx());
        else if (a == "--pt") c.pt = std::stof(nx());
        else if (a == "--cap") c.cap = std::stof(nx());
        else if (a == "--skip") c.skip = std::stoi(nx());
        else if (a == "--tc") c.tc = std::stoi(nx());
        else if (a == "--td") c.td = std::stoi(nx());
        else if (a == "--tlog") c.tlog = std::stoi(nx());
        else if (a == "--oxq") c.oxq = std::stoi(nx());
        else if (a == "--replicas") c.replicas = std::stoi(nx());
        else if (a == "--seed") c.seed = std::stoull(nx());
        else if (a == "--tmax") tmax = std::stoi(nx());
        else if (a == "--out") out = nx();
    }
    const int cand[] = {1, 2, 3, 5, 7, 10, 15, 20, 30, 50, 70, 100, 150, 200, 300, 500, 700, 1000};
    for (int v : cand) if (v <= tmax) c.ts[c.nt++] = v;
    const size_t n = size_t(c.replicas) * c.nt;
    double *w2, *hm;
    CK(cudaMalloc(&w2, n * 8));
    CK(cudaMalloc(&hm, n * 8));
    int8_t* gH = nullptr;
    size_t smem = 0;
    if (c.L <= 256) smem = size_t(c.L) * c.L;
    else CK(cudaMalloc(&gH, size_t(c.replicas) * c.L * c.L));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
    CK(cudaEventRecord(e0));
    if (scheme == "rs") {
        CK(cudaFuncSetAttribute(rs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        rs_kernel<<<c.replicas, 32, smem>>>(c, gH, w2, hm);
    } else {
        const int nact = (c.L / c.bx / 2) * (c.L / c.by / 2) * (c.bx / 32) * (c.by / 16);
        int threads = std::min(256, std::max(32, nact));
        threads = (threads + 31) / 32 * 32;
        if ((nact + threads - 1) / threads > 8) { fprintf(stderr, "too many tiles per thread\n"); return 1; }
        CK(cudaFuncSetAttribute(dt_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        dt_kernel<<<c.replicas, threads, smem>>>(c, gH, w2, hm);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1));
    CK(cudaDeviceSynchronize());
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    std::vector<double> W(n), Hm(n);
    CK(cudaMemcpy(W.data(), w2, n * 8, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(Hm.data(), hm, n * 8, cudaMemcpyDeviceToHost));
    FILE* f = fopen(out.c_str(), "w");
    fprintf(f, "{\"scheme\":\"%s\",\"L\":%d,\"bx\":%d,\"by\":%d,\"mini\":%d,\"counts\":%d,\"thin\":%g,\"pt\":%g,\"cap\":%g,\"skip\":%d,\"tc\":%d,\"td\":%d,\"tlog\":%d,\"oxq\":%d,"
               "\"replicas\":%d,\"seed\":%llu,\"seconds\":%.3f,\"t\":[",
            scheme.c_str(), c.L, c.bx, c.by, c.mini, c.counts, c.thin, c.pt, c.cap, c.skip, c.tc, c.td, c.tlog, c.oxq, c.replicas, c.seed, ms / 1e3);
    for (int s = 0; s < c.nt; ++s) fprintf(f, "%s%d", s ? "," : "", c.ts[s]);
    fprintf(f, "],\"w2_mean\":[");
    std::vector<double> mw(c.nt), sw(c.nt), mh(c.nt), sh(c.nt);
    for (int s = 0; s < c.nt; ++s) {
        double a = 0, b = 0, ha = 0, hb = 0;
        for (int r = 0; r < c.replicas; ++r) {
            const double v = W[size_t(r) * c.nt + s], h = Hm[size_t(r) * c.nt + s];
            a += v; b += v * v; ha += h; hb += h * h;
        }
        const double R = c.replicas;
        mw[s] = a / R; sw[s] = std::sqrt(std::max(0.0, (b / R - mw[s] * mw[s]) / (R - 1)));
        mh[s] = ha / R; sh[s] = std::sqrt(std::max(0.0, (hb / R - mh[s] * mh[s]) / (R - 1)));
    }
    for (int s = 0; s < c.nt; ++s) fprintf(f, "%s%.9g", s ? "," : "", mw[s]);
    fprintf(f, "],\"w2_se\":[");
    for (int s = 0; s < c.nt; ++s) fprintf(f, "%s%.6g", s ? "," : "", sw[s]);
    fprintf(f, "],\"h_mean\":[");
    for (int s = 0; s < c.nt; ++s) fprintf(f, "%s%.12g", s ? "," : "", mh[s]);
    fprintf(f, "],\"h_se\":[");
    for (int s = 0; s < c.nt; ++s) fprintf(f, "%s%.6g", s ? "," : "", sh[s]);
    fprintf(f, "]}\n");
    fclose(f);
    printf("%s done in %.2f s\n", out.c_str(), ms / 1e3);
    return 0;
}

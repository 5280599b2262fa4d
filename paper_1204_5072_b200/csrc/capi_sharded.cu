// capi_sharded.cu -- one host thread, N GPUs: the strip-sharded KPZ lattice
// (BASELINE configs[2]) behind the C ABI (include/lfg.h "sharded lattice").
//
// The reference API the sharded handle serves is the single-lattice one
// (kpz.hpp:119-120: kpz_sweep_sequential(f, params, rng, sweeps),
// interface_width(f)); PAPER.md:473-480 describes the multi-device
// decomposition.  Shard g (device devices[g]) owns the rows
// [oy + g H, oy + (g+1) H) of the current sub-sweep's shifted frame (H = L/N),
// i.e. whole device-block rows, so every block of every phase lives on one
// shard and runs the single-GPU phase kernel on it (lfg_kpz_strip_phase_push)
// over a ring buffer of C >= H + 4 by + 2 spin rows.  Between shards:
//   * per sub-sweep, the ownership roll (|d oy| < 2 by rows to one neighbour)
//     and both ghost rows: peer copies (cudaMemcpyAsync over NVLink / UVA);
//   * per phase, the one ghost row a neighbour reads next is stored straight
//     into its ring by this shard's write-back (fused push), and the phases of
//     neighbouring shards are ordered by CUDA events (stream waits), no host
//     synchronisation.
// The RNG is keyed on global tile / block ids of the shifted frame, so the
// sharded trajectory equals the single-lattice one bit for bit
// (tests/test_sharded_capi_gpu.py).  shard.py implements the same protocol
// for one process per GPU (torch.distributed / CUDA IPC).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lfg.h"
#include "capi_common.cuh"

using namespace lfg;

namespace {

// The shards' devices, streams and events (one per shard).
struct ShardGroup {
    int n = 1;
    std::vector<int32_t> dev;
    std::vector<cudaStream_t> st;
    std::vector<cudaEvent_t> ev;
    int dn(int g) const { return (g + n - 1) % n; }
    int up(int g) const { return (g + 1) % n; }

    // streams + events on every device, peer access between every pair
    void open() {
        for (int g = 0; g < n; ++g) {
            DeviceGuard dg(dev[size_t(g)]);
            for (int k = 0; k < n; ++k) {
                const int dk = dev[size_t(k)];
                if (dk == dev[size_t(g)]) continue;
                const cudaError_t e = cudaDeviceEnablePeerAccess(dk, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) cuda_check(e, "enable peer access");
                cudaGetLastError();
            }
            cudaStream_t s = nullptr;
            cuda_check(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
            st.push_back(s);
            cudaEvent_t e = nullptr;
            cuda_check(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
            ev.push_back(e);
        }
    }
    void close() {
        for (size_t g = 0; g < st.size(); ++g) {
            int prev = -1;
            cudaGetDevice(&prev);
            cudaSetDevice(dev[g]);
            cudaStreamSynchronize(st[g]);
            if (g < ev.size() && ev[g]) cudaEventDestroy(ev[g]);
            cudaStreamDestroy(st[g]);
            if (prev >= 0) cudaSetDevice(prev);
        }
        st.clear();
        ev.clear();
    }
    void record(int g) {
        DeviceGuard dg(dev[size_t(g)]);
        cuda_check(cudaEventRecord(ev[size_t(g)], st[size_t(g)]), "event record");
    }
    // Every shard's stream waits for its two neighbours' work issued so far
    // (exchanges only ever move data between neighbours).
    void barrier() {
        if (n == 1) return;
        for (int g = 0; g < n; ++g) record(g);
        wait_neighbours();
    }
    // ... for their last recorded events.
    void wait_neighbours() {
        if (n == 1) return;
        for (int g = 0; g < n; ++g) {
            DeviceGuard dg(dev[size_t(g)]);
            cuda_check(cudaStreamWaitEvent(st[size_t(g)], ev[size_t(dn(g))], 0), "stream wait");
            if (up(g) != dn(g)) cuda_check(cudaStreamWaitEvent(st[size_t(g)], ev[size_t(up(g))], 0), "stream wait");
        }
    }
    void sync() {
        for (int g = 0; g < n; ++g) {
            DeviceGuard dg(dev[size_t(g)]);
            cuda_check(cudaStreamSynchronize(st[size_t(g)]), "kernel execution");
        }
    }
};

// Units [u0, u0 + count) (mod L; rows or planes of `unit` bytes) from shard src's ring to
// shard dst's ring (slot = unit & (cap - 1)), on dst's stream; pieces split at the wraps.
void copy_units(ShardGroup& G, const std::vector<uint32_t*>& ring, int L, int cap, size_t unit_words, int dst, int src,
                int64_t u0, int count) {
    DeviceGuard dg(G.dev[size_t(dst)]);
    int64_t u = ((u0 % L) + L) % L;
    int left = count;
    while (left > 0) {
        const int slot = int(u & (cap - 1));
        const int m = int(std::min<int64_t>({left, cap - slot, L - u}));
        cuda_check(cudaMemcpyAsync(ring[size_t(dst)] + size_t(slot) * unit_words,
                                   ring[size_t(src)] + size_t(slot) * unit_words, unit_words * 4 * size_t(m),
                                   cudaMemcpyDefault, G.st[size_t(dst)]),
                   "peer copy");
        u = (u + m) % L;
        left -= m;
    }
}

}  // namespace

struct lfg_kpz_sharded {
    int32_t L = 0, n = 1, bx = 0, by = 0, sub = 4, H = 0, cap = 0, wpr = 0;
    double p = 1.0, q = 0.0;
    uint64_t seed = 0;
    uint64_t sweep = 0;  // next MCS index
    int32_t oy = -1;     // origin the current row ownership refers to (-1: no state yet)
    lfg_kpz_plan plan{};
    ShardGroup G;
    std::vector<int32_t>& dev = G.dev;
    std::vector<lfg_kpz*> hs;       // strip handles (per-shard stream, counters)
    std::vector<uint32_t*> ring;    // [cap][wpr] spin rows per shard

    int start(int32_t o, int g) const { return int((int64_t(o) + int64_t(g) * H) % L); }
    int dn(int g) const { return G.dn(g); }
    int up(int g) const { return G.up(g); }
};

namespace {

void lcheck(int rc) {
    if (rc != LFG_OK) throw Error(rc, lfg_last_error());
}

void copy_rows(lfg_kpz_sharded* h, int dst, int src, int64_t y0, int count) {
    copy_units(h->G, h->ring, h->L, h->cap, size_t(h->wpr), dst, src, y0, count);
}

void sync_all(lfg_kpz_sharded* h) { h->G.sync(); }

// Roll ownership from h->oy to oy_new, then refresh both ghost rows of every shard.
void exchange(lfg_kpz_sharded* h, int32_t oy_new) {
    if (h->n == 1) {
        h->oy = oy_new;
        return;
    }
    h->G.barrier();
    if (oy_new != h->oy) {
        const int d = oy_new - h->oy;
        for (int g = 0; g < h->n; ++g) {
            const int s = h->start(h->oy, g);
            if (d > 0) copy_rows(h, g, h->up(g), int64_t(s) + h->H, d);  // gain [s+H, s+H+d) from above
            else copy_rows(h, g, h->dn(g), int64_t(s) + d, -d);          // gain [s+d, s) from below
        }
        h->oy = oy_new;
        h->G.barrier();
    }
    for (int g = 0; g < h->n; ++g) {
        const int s = h->start(h->oy, g);
        copy_rows(h, g, h->dn(g), int64_t(s) - 1, 1);  // ghost below: last row of the lower neighbour
        copy_rows(h, g, h->up(g), int64_t(s) + h->H, 1);  // ghost above: first row of the upper neighbour
    }
    h->G.barrier();
}

void origin(const lfg_kpz_sharded* h, uint64_t subsweep, int32_t out6[6]) {
    lcheck(lfg_kpz_sweep_origin(h->L, &h->plan, h->seed, subsweep, out6));
}


}  // namespace

extern "C" {

int lfg_kpz_create_sharded(lfg_kpz_sharded** out, int32_t L, double p, double q, uint64_t seed,
                           const lfg_kpz_plan* plan, int32_t n_shards, const int32_t* devices) {
    return guarded([&] {
        if (!out) throw Error(LFG_EINVAL, "null output handle");
        *out = nullptr;
        if (n_shards < 1) throw Error(LFG_EINVAL, "n_shards must be >= 1");
        auto* h = new lfg_kpz_sharded();
        try {
            h->L = L;
            h->n = n_shards;
            h->G.n = n_shards;
            h->p = p;
            h->q = q;
            h->seed = seed;
            h->wpr = L / 32;
            for (int g = 0; g < n_shards; ++g) h->dev.push_back(devices ? devices[g] : g);
            // validates L, p, q and the plan; the handles also carry each shard's counters
            h->hs.assign(size_t(n_shards), nullptr);
            for (int g = 0; g < n_shards; ++g)
                lcheck(lfg_kpz_create_strip(&h->hs[size_t(g)], L, p, q, seed, plan, h->dev[size_t(g)]));
            lcheck(lfg_kpz_get_plan(h->hs[0], &h->plan));
            h->bx = h->plan.block_x;
            h->by = h->plan.block_y;
            h->sub = h->plan.sub;
            if (L % n_shards) throw Error(LFG_EINVAL, "n_shards must divide L");
            h->H = L / n_shards;
            if (n_shards > 1 && h->H % (2 * h->by))
                throw Error(LFG_EINVAL, "strip height L/n_shards = " + std::to_string(h->H) +
                                            " must be a multiple of 2*block_y = " + std::to_string(2 * h->by));
            int cap = 1;
            while (cap < h->H + 4 * h->by + 2) cap <<= 1;
            h->cap = n_shards == 1 ? L : std::min(L, cap);
            h->G.open();
            for (int g = 0; g < n_shards; ++g) {
                DeviceGuard dg(h->dev[size_t(g)]);
                h->ring.push_back(dmalloc<uint32_t>(size_t(h->cap) * size_t(h->wpr), "alloc strip ring"));
                lcheck(lfg_kpz_set_stream(h->hs[size_t(g)], h->G.st[size_t(g)]));
            }
        } catch (...) {
            lfg_kpz_sharded_destroy(h);
            throw;
        }
        *out = h;
    });
}

int lfg_kpz_sharded_destroy(lfg_kpz_sharded* h) {
    if (!h) return LFG_OK;
    for (size_t g = 0; g < h->hs.size(); ++g) {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(h->dev[g]);
        if (g < h->G.st.size()) cudaStreamSynchronize(h->G.st[g]);
        if (h->hs[g]) lfg_kpz_destroy(h->hs[g]);
        if (g < h->ring.size()) dfree(h->ring[g]);
        if (prev >= 0) cudaSetDevice(prev);
    }
    h->G.close();
    delete h;
    return LFG_OK;
}

int lfg_kpz_sharded_init_flat(lfg_kpz_sharded* h) {
    return guarded([&] {
        if (!h) throw Error(LFG_EINVAL, "null handle");
        int32_t o[6];
        origin(h, h->sweep * uint64_t(h->sub), o);
        h->oy = o[1];
        for (int g = 0; g < h->n; ++g) {
            const int rows = h->n == 1 ? h->L : h->H + 2;
            lcheck(lfg_kpz_strip_fill(h->hs[size_t(g)], h->ring[size_t(g)], h->cap,
                                      h->n == 1 ? 0 : (h->start(h->oy, g) - 1 + h->L) % h->L, rows, 0));
        }
        sync_all(h);
    });
}

int lfg_kpz_sharded_upload(lfg_kpz_sharded* h, const uint64_t* x, const uint64_t* y, size_t nwords) {
    return guarded([&] {
        if (!h) throw Error(LFG_EINVAL, "null handle");
        // convert + closure-check on shard 0's device through a resident handle
        lfg_kpz* t = nullptr;
        lcheck(lfg_kpz_create(&t, h->L, h->p, h->q, h->seed, &h->plan, h->dev[0]));
        try {
            lcheck(lfg_kpz_upload(t, 0, x, y, nwords));
            void* spins = nullptr;
            size_t bytes = 0;
            lcheck(lfg_kpz_device_spins(t, 0, &spins, &bytes));
            int32_t o[6];
            origin(h, h->sweep * uint64_t(h->sub), o);
            h->oy = o[1];
            const size_t rb = size_t(h->wpr) * 4;
            for (int g = 0; g < h->n; ++g) {
                DeviceGuard dg(h->dev[size_t(g)]);
                const int r0 = h->n == 1 ? 0 : h->start(h->oy, g) - 1, rows = h->n == 1 ? h->L : h->H + 2;
                for (int k = 0; k < rows; ++k) {
                    const int yy = ((r0 + k) % h->L + h->L) % h->L;
                    cuda_check(cudaMemcpyAsync(h->ring[size_t(g)] + size_t(yy & (h->cap - 1)) * h->wpr,
                                               static_cast<const uint32_t*>(spins) + size_t(yy) * h->wpr, rb,
                                               cudaMemcpyDefault, h->G.st[size_t(g)]),
                               "scatter rows");
                }
            }
            sync_all(h);
        } catch (...) {
            lfg_kpz_destroy(t);
            throw;
        }
        lfg_kpz_destroy(t);
    });
}

int lfg_kpz_sharded_download(lfg_kpz_sharded* h, uint64_t* x, uint64_t* y, size_t nwords) {
    return guarded([&] {
        if (!h || h->oy < 0) throw Error(LFG_EINVAL, "sharded lattice has no state (init_flat / upload first)");
        lfg_kpz* t = nullptr;
        lcheck(lfg_kpz_create(&t, h->L, h->p, h->q, h->seed, &h->plan, h->dev[0]));
        try {
            void* spins = nullptr;
            size_t bytes = 0;
            lcheck(lfg_kpz_device_spins(t, 0, &spins, &bytes));
            sync_all(h);
            const size_t rb = size_t(h->wpr) * 4;
            DeviceGuard dg(h->dev[0]);
            // The gather is stream-ordered on shard 0's stream and completed before the
            // temporary handle's own (non-blocking) stream converts the rows: a plain
            // device-to-device cudaMemcpy returns before the copy is done and is not
            // ordered against that stream.
            for (int g = 0; g < h->n; ++g) {
                const int r0 = h->n == 1 ? 0 : h->start(h->oy, g), rows = h->n == 1 ? h->L : h->H;
                for (int k = 0; k < rows; ++k) {
                    const int yy = (r0 + k) % h->L;
                    cuda_check(cudaMemcpyAsync(static_cast<uint32_t*>(spins) + size_t(yy) * h->wpr,
                                               h->ring[size_t(g)] + size_t(yy & (h->cap - 1)) * h->wpr, rb,
                                               cudaMemcpyDefault, h->G.st[0]),
                               "gather rows");
                }
            }
            cuda_check(cudaStreamSynchronize(h->G.st[0]), "gather rows");
            lcheck(lfg_kpz_download(t, 0, x, y, nwords));
        } catch (...) {
            lfg_kpz_destroy(t);
            throw;
        }
        lfg_kpz_destroy(t);
    });
}

int lfg_kpz_sharded_sweep(lfg_kpz_sharded* h, int64_t n_mcs, lfg_counters* out) {
    return guarded([&] {
        if (!h || h->oy < 0) throw Error(LFG_EINVAL, "sharded lattice has no state (init_flat / upload first)");
        if (n_mcs < 0) throw Error(LFG_EINVAL, "sweep: n_mcs must be >= 0");
        lfg_counters before{};
        if (out) lcheck(lfg_kpz_sharded_counters(h, &before));
        const int nbrow = h->H / h->by;
        for (int64_t s = 0; s < n_mcs; ++s) {
            for (int k = 0; k < h->sub; ++k) {
                const uint64_t sp = (h->sweep + uint64_t(s)) * uint64_t(h->sub) + uint64_t(k);
                int32_t o[6];
                origin(h, sp, o);
                exchange(h, o[1]);
                for (int ph = 0; ph < 4; ++ph) {
                    if (ph > 0) h->G.wait_neighbours();
                    const int sy = o[2 + ph] >> 1;
                    for (int g = 0; g < h->n; ++g) {
                        const int first = h->start(h->oy, g), last = (first + h->H - 1) % h->L;
                        const bool push = h->n > 1;
                        lcheck(lfg_kpz_strip_phase_push(
                            h->hs[size_t(g)], h->ring[size_t(g)], h->cap, g * nbrow, nbrow, sp, ph,
                            push && sy == 0 ? h->ring[size_t(h->dn(g))] : nullptr, push && sy == 0 ? first : -1,
                            push && sy == 1 ? h->ring[size_t(h->up(g))] : nullptr, push && sy == 1 ? last : -1));
                        h->G.record(g);
                    }
                }
            }
        }
        h->sweep += uint64_t(n_mcs);
        if (out) {
            lfg_counters after{};
            lcheck(lfg_kpz_sharded_counters(h, &after));
            out->attempts = after.attempts - before.attempts;
            out->successes = after.successes - before.successes;
            out->deposits = after.deposits - before.deposits;
            out->detaches = after.detaches - before.detaches;
        }
    });
}

int lfg_kpz_sharded_counters(lfg_kpz_sharded* h, lfg_counters* out) {
    return guarded([&] {
        if (!h || !out) throw Error(LFG_EINVAL, "null argument");
        lfg_counters tot{};
        for (int g = 0; g < h->n; ++g) {
            lfg_counters c{};
            lcheck(lfg_kpz_counters(h->hs[size_t(g)], 0, &c));  // synchronises the shard's stream
            tot.attempts += c.attempts;
            tot.successes += c.successes;
            tot.deposits += c.deposits;
            tot.detaches += c.detaches;
        }
        *out = tot;
    });
}

int lfg_kpz_sharded_width_sums(lfg_kpz_sharded* h, int64_t* sum, int64_t* sum2) {
    return guarded([&] {
        if (!h || h->oy < 0) throw Error(LFG_EINVAL, "sharded lattice has no state (init_flat / upload first)");
        if (!sum || !sum2) throw Error(LFG_EINVAL, "null output");
        exchange(h, h->oy);  // every piece reads the row below it
        struct Piece {
            int a, nrows;
            int64_t s1, s2, d;
        };
        std::vector<Piece> pieces;
        for (int g = 0; g < h->n; ++g) {
            const int a = h->n == 1 ? 0 : h->start(h->oy, g);
            const int rows = h->n == 1 ? h->L : h->H;
            int y = a, left = rows;
            while (left > 0) {  // owned rows split where they wrap past row L-1
                const int m = std::min(left, h->L - y);
                int64_t o3[3];
                lcheck(lfg_kpz_strip_width_rows(h->hs[size_t(g)], h->ring[size_t(g)], h->cap, y, m, o3));
                pieces.push_back({y, m, o3[0], o3[1], o3[2]});
                y = (y + m) % h->L;
                left -= m;
            }
        }
        std::sort(pieces.begin(), pieces.end(), [](const Piece& u, const Piece& v) { return u.a < v.a; });
        // chain the pieces in global row order from row 0 (heights relative to
        // the column-0 height of the row below each piece): shard.py width_sums
        int64_t S1 = 0, S2 = 0, B = 0;
        for (const Piece& pc : pieces) {
            const int64_t m = int64_t(pc.nrows) * h->L;
            S1 += pc.s1 + m * B;
            S2 += pc.s2 + 2 * B * pc.s1 + m * B * B;
            B += pc.d;
        }
        *sum = S1;
        *sum2 = S2;
    });
}

int lfg_kpz_sharded_interface_width(lfg_kpz_sharded* h, double* w2) {
    int64_t s = 0, s2 = 0;
    const int rc = lfg_kpz_sharded_width_sums(h, &s, &s2);
    if (rc != LFG_OK) return rc;
    const double nn = double(int64_t(h->L) * h->L);  // kpz.cpp:78-80
    const double mean = double(s) / nn;
    *w2 = double(s2) / nn - mean * mean;
    return LFG_OK;
}

int lfg_kpz_sharded_set_sweep_index(lfg_kpz_sharded* h, uint64_t sweep) {
    return guarded([&] {
        if (!h) throw Error(LFG_EINVAL, "null handle");
        if (h->oy >= 0) throw Error(LFG_EINVAL, "set_sweep_index: call before init_flat / upload");
        h->sweep = sweep;
    });
}

int lfg_kpz_sharded_get_sweep_index(const lfg_kpz_sharded* h, uint64_t* sweep) {
    return guarded([&] {
        if (!h || !sweep) throw Error(LFG_EINVAL, "null argument");
        *sweep = h->sweep;
    });
}

}  // extern "C"

// ============================================================ KMC z-slabs
// BASELINE configs[4]: the 3-D lattice cut into z-slabs of H = L/N planes
// (H a multiple of 2 bk), slab g on devices[g], one host thread.  Protocol of
// shard.py ShardedKmc (kmc.hpp:140-141 reach: read 2, write 1): per MCS the
// ownership roll with the DT origin oz; around each phase of z-parity sz the two
// ghost planes on the active side are refreshed before, and the one ghost plane
// the phase may have modified goes back to its owner after -- all peer copies
// between neighbouring slabs, ordered by CUDA events.
#include "../../include/lfg_kmc.h"

struct lfg_kmc_sharded {
    int32_t L = 0, n = 1, bk = 0, sub = 1, H = 0, cap = 0;
    size_t wpp = 0;        // uint32 words per plane
    double eps = 0;
    int32_t both = 0;
    uint64_t seed = 0, sweep = 0;
    int32_t oz = -1;       // origin the current plane ownership refers to (-1: no state yet)
    lfg_kmc_plan plan{};
    ShardGroup G;
    std::vector<lfg_kmc*> hs;       // slab handles (per-shard stream, counters)
    std::vector<uint32_t*> ring;    // [cap][wpp] planes per shard

    int start(int32_t o, int g) const { return int((int64_t(o) + int64_t(g) * H) % L); }
    int win0(int g) const { return n == 1 ? 0 : start(oz, g) - 2; }  // owned planes + 2 ghosts per side
    int wlen() const { return n == 1 ? L : H + 4; }
};

namespace {

void kcopy(lfg_kmc_sharded* h, int dst, int src, int64_t z0, int count) {
    copy_units(h->G, h->ring, h->L, h->cap, h->wpp, dst, src, z0, count);
}

int32_t kmc_origin_z(const lfg_kmc_sharded* h, uint64_t sweep, int32_t order[8]) {
    int32_t o[11];
    lcheck(lfg_kmc_sweep_origin(h->L, &h->plan, h->seed, sweep, o));
    if (order)
        for (int k = 0; k < 8; ++k) order[k] = o[3 + k];
    return o[2];
}

// Refresh `depth` ghost planes on side sz (1: above, 0: below) of every slab.
void kmc_ghost(lfg_kmc_sharded* h, int sz, int depth) {
    for (int g = 0; g < h->n; ++g) {
        const int s = h->start(h->oz, g);
        if (sz == 1) kcopy(h, g, h->G.up(g), int64_t(s) + h->H, depth);
        else kcopy(h, g, h->G.dn(g), int64_t(s) - depth, depth);
    }
}

}  // namespace

extern "C" {

int lfg_kmc_create_sharded(lfg_kmc_sharded** out, int32_t L, double eps, int32_t both_active, uint64_t seed,
                           const lfg_kmc_plan* plan, int32_t n_shards, const int32_t* devices) {
    return guarded([&] {
        if (!out) throw Error(LFG_EINVAL, "null output handle");
        *out = nullptr;
        if (n_shards < 1) throw Error(LFG_EINVAL, "n_shards must be >= 1");
        auto* h = new lfg_kmc_sharded();
        try {
            h->L = L;
            h->n = n_shards;
            h->G.n = n_shards;
            h->eps = eps;
            h->both = both_active;
            h->seed = seed;
            for (int g = 0; g < n_shards; ++g) h->G.dev.push_back(devices ? devices[g] : g);
            h->hs.assign(size_t(n_shards), nullptr);
            for (int g = 0; g < n_shards; ++g)
                lcheck(lfg_kmc_create_slab(&h->hs[size_t(g)], L, eps, both_active, seed, plan, h->G.dev[size_t(g)]));
            lcheck(lfg_kmc_get_plan(h->hs[0], &h->plan));
            h->bk = h->plan.block;
            h->sub = h->plan.sub;
            if (L % n_shards) throw Error(LFG_EINVAL, "n_shards must divide L");
            h->H = L / n_shards;
            if (n_shards > 1 && h->H % (2 * h->bk))
                throw Error(LFG_EINVAL, "slab height L/n_shards = " + std::to_string(h->H) +
                                            " must be a multiple of 2*block = " + std::to_string(2 * h->bk));
            int cap = 1;
            while (cap < h->H + 4 * h->bk + 4) cap <<= 1;
            h->cap = n_shards == 1 ? L : std::min(L, cap);
            h->wpp = size_t(L) * size_t(L) / 32;
            h->G.open();
            for (int g = 0; g < n_shards; ++g) {
                DeviceGuard dg(h->G.dev[size_t(g)]);
                h->ring.push_back(dmalloc<uint32_t>(size_t(h->cap) * h->wpp, "alloc slab ring"));
                cuda_check(cudaMemsetAsync(h->ring.back(), 0, size_t(h->cap) * h->wpp * 4, h->G.st[size_t(g)]),
                           "memset");
                lcheck(lfg_kmc_set_stream(h->hs[size_t(g)], h->G.st[size_t(g)]));
            }
        } catch (...) {
            lfg_kmc_sharded_destroy(h);
            throw;
        }
        *out = h;
    });
}

int lfg_kmc_sharded_destroy(lfg_kmc_sharded* h) {
    if (!h) return LFG_OK;
    for (size_t g = 0; g < h->hs.size(); ++g) {
        int prev = -1;
        cudaGetDevice(&prev);
        cudaSetDevice(h->G.dev[g]);
        if (g < h->G.st.size()) cudaStreamSynchronize(h->G.st[g]);
        if (h->hs[g]) lfg_kmc_destroy(h->hs[g]);
        if (g < h->ring.size()) dfree(h->ring[g]);
        if (prev >= 0) cudaSetDevice(prev);
    }
    h->G.close();
    delete h;
    return LFG_OK;
}

int lfg_kmc_sharded_init_random_alloy(lfg_kmc_sharded* h, double c, uint64_t alloy_seed) {
    return guarded([&] {
        if (!h) throw Error(LFG_EINVAL, "null handle");
        h->oz = kmc_origin_z(h, h->sweep * uint64_t(h->sub), nullptr);
        for (int g = 0; g < h->n; ++g)
            lcheck(lfg_kmc_slab_init_random_alloy(h->hs[size_t(g)], h->ring[size_t(g)], h->cap,
                                                  (h->win0(g) + h->L) % h->L, h->wlen(), c, alloy_seed));
        h->G.sync();
    });
}

int lfg_kmc_sharded_upload(lfg_kmc_sharded* h, const uint64_t* words, size_t nwords) {
    return guarded([&] {
        if (!h || !words) throw Error(LFG_EINVAL, "null argument");
        if (nwords != size_t(h->L) * h->L * h->L / 64)
            throw Error(LFG_EINVAL, "upload: expected L^3/64 words");
        h->oz = kmc_origin_z(h, h->sweep * uint64_t(h->sub), nullptr);
        const uint32_t* src = reinterpret_cast<const uint32_t*>(words);  // plane z at z * wpp (little-endian)
        for (int g = 0; g < h->n; ++g) {
            DeviceGuard dg(h->G.dev[size_t(g)]);
            for (int k = 0; k < h->wlen(); ++k) {
                const int z = ((h->win0(g) + k) % h->L + h->L) % h->L;
                cuda_check(cudaMemcpyAsync(h->ring[size_t(g)] + size_t(z & (h->cap - 1)) * h->wpp,
                                           src + size_t(z) * h->wpp, h->wpp * 4, cudaMemcpyHostToDevice,
                                           h->G.st[size_t(g)]),
                           "upload planes");
            }
        }
        h->G.sync();
    });
}

int lfg_kmc_sharded_download(lfg_kmc_sharded* h, uint64_t* words, size_t nwords) {
    return guarded([&] {
        if (!h || !words || h->oz < 0) throw Error(LFG_EINVAL, "sharded lattice has no state (init / upload first)");
        if (nwords != size_t(h->L) * h->L * h->L / 64)
            throw Error(LFG_EINVAL, "download: expected L^3/64 words");
        h->G.sync();
        uint32_t* dst = reinterpret_cast<uint32_t*>(words);
        for (int g = 0; g < h->n; ++g) {
            DeviceGuard dg(h->G.dev[size_t(g)]);
            const int z0 = h->n == 1 ? 0 : h->start(h->oz, g), nz = h->n == 1 ? h->L : h->H;
            for (int k = 0; k < nz; ++k) {
                const int z = (z0 + k) % h->L;
                cuda_check(cudaMemcpy(dst + size_t(z) * h->wpp, h->ring[size_t(g)] + size_t(z & (h->cap - 1)) * h->wpp,
                                      h->wpp * 4, cudaMemcpyDeviceToHost),
                           "download planes");
            }
        }
    });
}

int lfg_kmc_sharded_counters(lfg_kmc_sharded* h, lfg_counters* out) {
    return guarded([&] {
        if (!h || !out) throw Error(LFG_EINVAL, "null argument");
        lfg_counters tot{};
        for (int g = 0; g < h->n; ++g) {
            lfg_counters c{};
            lcheck(lfg_kmc_counters(h->hs[size_t(g)], &c));
            tot.attempts += c.attempts;
            tot.successes += c.successes;
        }
        *out = tot;
    });
}

int lfg_kmc_sharded_sweep(lfg_kmc_sharded* h, int64_t n_mcs, lfg_counters* out) {
    return guarded([&] {
        if (!h || h->oz < 0) throw Error(LFG_EINVAL, "sharded lattice has no state (init / upload first)");
        if (n_mcs < 0) throw Error(LFG_EINVAL, "sweep: n_mcs must be >= 0");
        lfg_counters before{};
        if (out) lcheck(lfg_kmc_sharded_counters(h, &before));
        const int nbz = h->H / h->bk;
        for (int64_t s = 0; s < n_mcs * h->sub; ++s) {
            const uint64_t sw = h->sweep * uint64_t(h->sub) + uint64_t(s);  // global sub-sweep index
            int32_t order[8];
            const int32_t oz = kmc_origin_z(h, sw, order);
            if (h->n > 1 && oz != h->oz) {  // ownership roll
                h->G.barrier();
                const int d = oz - h->oz;
                for (int g = 0; g < h->n; ++g) {
                    const int st = h->start(h->oz, g);
                    if (d > 0) kcopy(h, g, h->G.up(g), int64_t(st) + h->H, d);
                    else kcopy(h, g, h->G.dn(g), int64_t(st) + d, -d);
                }
            }
            h->oz = oz;
            for (int k = 0; k < 8; ++k) {
                const int sz = order[k] >> 2;
                if (h->n > 1) {  // the two ghost planes on the active side
                    h->G.barrier();
                    kmc_ghost(h, sz, 2);
                    h->G.barrier();
                }
                for (int g = 0; g < h->n; ++g)
                    lcheck(lfg_kmc_slab_phase(h->hs[size_t(g)], h->ring[size_t(g)], h->cap, g * nbz, nbz, sw, k));
                if (h->n > 1) {  // the ghost plane the phase may have written goes back to its owner
                    h->G.barrier();
                    for (int g = 0; g < h->n; ++g) {
                        const int st = h->start(h->oz, g);
                        if (sz == 1) kcopy(h, h->G.up(g), g, int64_t(st) + h->H, 1);
                        else kcopy(h, h->G.dn(g), g, int64_t(st) - 1, 1);
                    }
                }
            }
        }
        h->sweep += uint64_t(n_mcs);
        if (out) {
            lfg_counters after{};
            lcheck(lfg_kmc_sharded_counters(h, &after));
            out->attempts = after.attempts - before.attempts;
            out->successes = after.successes - before.successes;
            out->deposits = 0;
            out->detaches = 0;
        }
    });
}

int lfg_kmc_sharded_open_bond_sums(lfg_kmc_sharded* h, int64_t* particles, int64_t* open) {
    return guarded([&] {
        if (!h || h->oz < 0) throw Error(LFG_EINVAL, "sharded lattice has no state (init / upload first)");
        if (!particles || !open) throw Error(LFG_EINVAL, "null output");
        if (h->n > 1) {  // every owned plane's neighbour planes
            h->G.barrier();
            kmc_ghost(h, 0, 1);
            kmc_ghost(h, 1, 1);
            h->G.barrier();
        }
        int64_t np = 0, no = 0;
        for (int g = 0; g < h->n; ++g) {
            const int z0 = h->n == 1 ? 0 : h->start(h->oz, g), nz = h->n == 1 ? h->L : h->H;
            int z = z0, left = nz;
            while (left > 0) {  // owned planes split where they wrap past plane L-1
                const int m = std::min(left, h->L - z);
                int64_t a = 0, b = 0;
                lcheck(lfg_kmc_slab_open_bond_sums(h->hs[size_t(g)], h->ring[size_t(g)], h->cap, z, m, &a, &b));
                np += a;
                no += b;
                z = (z + m) % h->L;
                left -= m;
            }
        }
        *particles = np;
        *open = no;
    });
}

int lfg_kmc_sharded_open_bonds_per_particle(lfg_kmc_sharded* h, double* v) {
    return guarded([&] {
        int64_t np = 0, no = 0;
        lcheck(lfg_kmc_sharded_open_bond_sums(h, &np, &no));
        if (np == 0) throw Error(LFG_EDOMAIN, "open_bonds_per_particle: no B particles in lattice");  // kmc.cpp:36-38
        *v = double(no) / double(np);
    });
}

int lfg_kmc_sharded_set_sweep_index(lfg_kmc_sharded* h, uint64_t sweep) {
    return guarded([&] {
        if (!h) throw Error(LFG_EINVAL, "null handle");
        if (h->oz >= 0) throw Error(LFG_EINVAL, "set_sweep_index: call before init / upload");
        h->sweep = sweep;
    });
}

int lfg_kmc_sharded_get_sweep_index(const lfg_kmc_sharded* h, uint64_t* sweep) {
    return guarded([&] {
        if (!h || !sweep) throw Error(LFG_EINVAL, "null argument");
        *sweep = h->sweep;
    });
}

}  // extern "C"

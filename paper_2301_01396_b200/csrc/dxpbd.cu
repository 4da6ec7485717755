// C-ABI of the B200-native DiffXPBD hot path (include/dxpbd.h).
// Host side: scene construction (greedy coloring, color-sorted SoA buffers), the forward
// substep loop with checkpoints, the backward loop (replay -> PCG -> adjoint update ->
// gradients).  Every arithmetic step of the path runs in the kernels of kernels.cuh.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <memory>
#include <thread>
#include <tuple>
#include <utility>
#include <vector>

#include "../../include/dxpbd.h"
#include "kernels.cuh"
#include "pull.cuh"
#include "tet_kernels.cuh"
#include "wave.cuh"

using namespace dx;

namespace {

thread_local std::string g_err;
thread_local int g_ring_states = 0;   // > 0: dxpbd_create allocates only this many full-V states (partition groups)

struct Err {
    int code;
    std::string msg;
};

#define DX_CHECK_CUDA(expr)                                                                  \
    do {                                                                                     \
        cudaError_t _e = (expr);                                                             \
        if (_e != cudaSuccess) throw Err{DXPBD_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)}; \
    } while (0)
#define DX_REQUIRE(cond, code, msg)                     \
    do {                                                \
        if (!(cond)) throw Err{(code), std::string(msg)}; \
    } while (0)

inline int nblk(int64_t n) { return (int)((n + kBlock - 1) / kBlock); }

template <class T>
struct DBuf {
    T *p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        free();
        n = count;
        if (count) {
            cudaError_t e = cudaMalloc(&p, count * sizeof(T));
            if (e != cudaSuccess) {
                p = nullptr;
                n = 0;
                cudaGetLastError();
                throw Err{DXPBD_ERR_OOM, "cudaMalloc of " + std::to_string(count * sizeof(T)) + " bytes failed"};
            }
        }
    }
    void free() {
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
    }
    ~DBuf() { free(); }
};

// Sequential greedy coloring in constraint order (R1): smallest color not held by an
// earlier constraint sharing a vertex.  Per-vertex 256-bit used-color sets.
int greedy_colors(int64_t n, int arity, const int32_t *idx, int64_t V, std::vector<int32_t> &col) {
    std::vector<uint64_t> used((size_t)V * 4, 0);
    col.assign(n, 0);
    int nc = 0;
    for (int64_t j = 0; j < n; ++j) {
        uint64_t m[4] = {0, 0, 0, 0};
        for (int k = 0; k < arity; ++k) {
            const uint64_t *u = &used[(size_t)idx[j * arity + k] * 4];
            m[0] |= u[0]; m[1] |= u[1]; m[2] |= u[2]; m[3] |= u[3];
        }
        int c = -1;
        for (int q = 0; q < 4; ++q)
            if (~m[q]) { c = q * 64 + __builtin_ctzll(~m[q]); break; }
        if (c < 0) return -1;
        col[j] = c;
        nc = std::max(nc, c + 1);
        for (int k = 0; k < arity; ++k) used[(size_t)idx[j * arity + k] * 4 + c / 64] |= 1ull << (c % 64);
    }
    return nc;
}

// stable counting sort by color -> perm (sorted position -> user index), color offsets
void color_sort(const std::vector<int32_t> &col, int nc, std::vector<int32_t> &perm, std::vector<int> &off) {
    off.assign(nc + 1, 0);
    for (int32_t c : col) off[c + 1]++;
    for (int c = 0; c < nc; ++c) off[c + 1] += off[c];
    std::vector<int> pos(off.begin(), off.end() - 1);
    perm.assign(col.size(), 0);
    for (size_t j = 0; j < col.size(); ++j) perm[pos[col[j]]++] = (int32_t)j;
}

// Morton (Z-order) permutation of the rest positions: internal vertex i = user vertex perm[i]
// (tiles of kTileV consecutive internal vertices are spatially compact).
// Reorder idx[0, n) into groups of G consecutive entries (one shared-memory access phase) whose
// endpoint bank keys (0..NB-1, NB <= 32) are pairwise distinct where the segment allows it: the
// (bank_a, bank_b) pairs form a bipartite multigraph on NB + NB banks; a proper edge coloring
// (Konig: max-degree colors, alternating-path recoloring) splits it into matchings; each group
// starts from the largest remaining matching and is filled with non-conflicting entries of the
// others (then with any entry, so that every group but the last is full).  Create-time host work.
template <class F>
static void bank_group(int32_t *idx, int n, int NB, int G, F banks) {
    if (n <= 1) return;
    std::vector<std::pair<int, int>> ed(n);
    std::vector<int> dl(NB, 0), dr(NB, 0);
    for (int k = 0; k < n; ++k) {
        ed[k] = banks(idx[k]);
        dl[ed[k].first]++;
        dr[ed[k].second]++;
    }
    int D = 0;
    for (int b = 0; b < NB; ++b) D = std::max(D, std::max(dl[b], dr[b]));
    std::vector<int> L(NB * D, -1), R(NB * D, -1), col(n, -1), path;
    for (int k = 0; k < n; ++k) {
        const int u = ed[k].first, v = ed[k].second;
        int a = 0, b = 0;
        while (L[u * D + a] >= 0) ++a;
        while (R[v * D + b] >= 0) ++b;
        if (L[u * D + b] < 0) {
            a = b;
        } else if (R[v * D + a] >= 0) {
            // swap colors a <-> b along the alternating path that starts at v with color a
            path.clear();
            bool right = true;
            int node = v, c = a;
            for (;;) {
                const int e = right ? R[node * D + c] : L[node * D + c];
                if (e < 0) break;
                path.push_back(e);
                node = right ? ed[e].first : ed[e].second;
                right = !right;
                c = c == a ? b : a;
            }
            for (int e : path) { L[ed[e].first * D + col[e]] = -1; R[ed[e].second * D + col[e]] = -1; }
            for (int e : path) {
                col[e] = col[e] == a ? b : a;
                L[ed[e].first * D + col[e]] = e;
                R[ed[e].second * D + col[e]] = e;
            }
        }
        col[k] = a;
        L[u * D + a] = k;
        R[v * D + a] = k;
    }
    std::vector<std::vector<int>> cls(D);
    for (int k = 0; k < n; ++k) cls[col[k]].push_back(k);
    std::vector<int32_t> out;
    out.reserve(n);
    std::vector<int> g;
    for (;;) {
        cls.erase(std::remove_if(cls.begin(), cls.end(), [](const std::vector<int> &c) { return c.empty(); }), cls.end());
        if (cls.empty()) break;
        std::stable_sort(cls.begin(), cls.end(), [](const std::vector<int> &x, const std::vector<int> &y) { return x.size() > y.size(); });
        g.assign(cls[0].begin(), cls[0].begin() + std::min<size_t>(cls[0].size(), G));
        cls[0].erase(cls[0].begin(), cls[0].begin() + g.size());
        uint32_t ma = 0, mb = 0;
        for (int k : g) { ma |= 1u << ed[k].first; mb |= 1u << ed[k].second; }
        for (size_t ci = 1; ci < cls.size() && (int)g.size() < G; ++ci) {
            auto &c = cls[ci];
            for (size_t q = 0; q < c.size() && (int)g.size() < G;) {
                const int k = c[q];
                const uint32_t ba = 1u << ed[k].first, bb = 1u << ed[k].second;
                if (!(ma & ba) && !(mb & bb)) {
                    g.push_back(k);
                    ma |= ba;
                    mb |= bb;
                    c.erase(c.begin() + q);
                } else {
                    ++q;
                }
            }
        }
        for (size_t ci = cls.size(); ci-- > 0 && (int)g.size() < G;) {
            auto &c = cls[ci];
            while (!c.empty() && (int)g.size() < G) { g.push_back(c.back()); c.pop_back(); }
        }
        for (int k : g) out.push_back(idx[k]);
    }
    std::copy(out.begin(), out.end(), idx);
}

// TMA-kernel layout of one tile (create time, host).  Local indices: own vertex v -> v - t*kTileV,
// halo vertex -> kTileV + its rank in the tile's sorted halo list.  Each local index gets a
// shared-memory slot (own: [0, kTileV), halo: [kTileV, kTileV + hcap)) holding a float4; its
// 16-byte bank group (slot & 7) is chosen greedily so that, for every (color, side) of the tile's
// constraint segments, the endpoints spread evenly over the 8 groups (a linear layout folds a
// color's lower endpoints onto half of them: Morton index parities).  Each segment is then ordered
// into groups of 8 (one quarter-warp access phase) with distinct groups per endpoint (bank_group).  Outputs: vslot / hslot (slots), tpos (sorted position -> layout position),
// cpair (slot pairs of the combined segments), tpos / fposv (layout positions of each constraint's
// block: in its own tile's segment and, if b lies in another tile, in that tile's segment).
struct TileLayoutScratch {
    std::vector<int> deg, moff, memb, cnt, order, slot_of, used;
    std::vector<uint32_t> gmask;
    std::vector<int32_t> ids;
};

static void tma_tile_layout(int t, int nc, int nt, int hcap, const std::vector<int> &halo_t, int hoff_t,
                            const int64_t *cnt, const int64_t *fc, const int2 *ab, const int *fidx,
                            const int64_t *cbase, uint16_t *vslot, uint16_t *hslot, int *tpos, int *fposv,
                            uint32_t *cpair, TileLayoutScratch &w) {
    const int nh = (int)halo_t.size(), NL = kTileV + nh, NK = 4 * nc;
    auto local = [&](int v) {
        return v / kTileV == t ? v - t * kTileV
                               : kTileV + (int)(std::lower_bound(halo_t.begin(), halo_t.end(), v) - halo_t.begin());
    };
    // memberships (CSR): key 4c+0 / 4c+1 = lower / upper endpoint of the color-c segment,
    // 4c+2 / 4c+3 = halo / own endpoint of the color-c foreign segment
    w.deg.assign(NL + 1, 0);
    auto each = [&](auto &&f) {
        for (int c = 0; c < nc; ++c) {
            const size_t kk = (size_t)c * nt + t;
            for (int64_t q = cnt[kk]; q < cnt[kk + 1]; ++q) { f(local(ab[q].x), 4 * c); f(local(ab[q].y), 4 * c + 1); }
            for (int64_t k2 = fc[kk]; k2 < fc[kk + 1]; ++k2) {
                const int q = fidx[k2];
                f(local(ab[q].x), 4 * c + 2);
                f(local(ab[q].y), 4 * c + 3);
            }
        }
    };
    each([&](int l, int) { w.deg[l + 1]++; });
    w.moff.assign(NL + 1, 0);
    for (int l = 0; l < NL; ++l) w.moff[l + 1] = w.moff[l] + w.deg[l + 1];
    w.memb.resize(w.moff[NL]);
    for (int l = 0; l < NL; ++l) w.deg[l] = w.moff[l];
    each([&](int l, int k) { w.memb[w.deg[l]++] = k; });
    // greedy bank assignment, most-constrained first, per region (own, halo)
    constexpr int NB = 8;   // 16-byte bank groups of a float4 access phase
    w.cnt.assign((size_t)NK * NB, 0);
    w.slot_of.assign(NL, 0);
    for (int region = 0; region < 2; ++region) {
        const int lo = region ? kTileV : 0, hi = region ? NL : kTileV, cap = region ? hcap / NB : kTileV / NB;
        const int base = region ? kTileV : 0;
        w.order.resize(hi - lo);
        for (int l = lo; l < hi; ++l) w.order[l - lo] = l;
        std::stable_sort(w.order.begin(), w.order.end(),
                         [&](int x, int y) { return w.moff[x + 1] - w.moff[x] > w.moff[y + 1] - w.moff[y]; });
        w.used.assign(NB, 0);
        // each aligned group of 8 consecutive local indices (one quarter-warp of the vertex / halo
        // phases, which access slot(i) for i = thread + k * blockDim) takes 8 distinct bank groups
        w.gmask.assign((hi - lo + 7) / 8 + 1, 0);
        for (int l : w.order) {
            int best = -1;
            long bc = 0;
            const int gi = (l - lo) / 8;
            for (int b = 0; b < NB; ++b) {
                if (w.used[b] >= cap || ((w.gmask[gi] >> b) & 1)) continue;
                long c = 0;
                for (int m = w.moff[l]; m < w.moff[l + 1]; ++m) c += w.cnt[(size_t)w.memb[m] * NB + b];
                c = c * 1024 + w.used[b];
                if (best < 0 || c < bc) { best = b; bc = c; }
            }
            w.slot_of[l] = base + NB * w.used[best] + best;
            w.used[best]++;
            w.gmask[gi] |= 1u << best;
            for (int m = w.moff[l]; m < w.moff[l + 1]; ++m) w.cnt[(size_t)w.memb[m] * NB + best]++;
        }
    }
    for (int l = 0; l < kTileV; ++l) vslot[(size_t)t * kTileV + l] = (uint16_t)w.slot_of[l];
    for (int h = 0; h < nh; ++h) hslot[hoff_t + h] = (uint16_t)w.slot_of[kTileV + h];
    auto sl = [&](int v) { return w.slot_of[local(v)]; };
    // combined segment of (t, c) at cbase[t * nc + c]: own constraints (ids q >= 0) and foreign
    // entries (ids -(k2 + 1)), grouped jointly; "own" is recovered in the kernels as slot(a) < kTileV
    auto con = [&](int32_t id) { return id >= 0 ? id : fidx[-id - 1]; };
    for (int c = 0; c < nc; ++c) {
        const size_t kk = (size_t)c * nt + t;
        const int64_t b = cnt[kk], e = cnt[kk + 1], fb = fc[kk], fe = fc[kk + 1];
        w.ids.clear();
        for (int64_t q = b; q < e; ++q) w.ids.push_back((int32_t)q);
        for (int64_t k2 = fb; k2 < fe; ++k2) w.ids.push_back((int32_t)(-(k2 + 1)));
        bank_group(w.ids.data(), (int)w.ids.size(), NB, NB, [&](int32_t id) {
            const int q = con(id);
            return std::make_pair(sl(ab[q].x) & (NB - 1), sl(ab[q].y) & (NB - 1));
        });
        const int64_t base = cbase[(size_t)t * nc + c];
        for (size_t i = 0; i < w.ids.size(); ++i) {
            const int32_t id = w.ids[i];
            const int q = con(id);
            cpair[base + i] = (uint32_t)sl(ab[q].x) | ((uint32_t)sl(ab[q].y) << 16);
            if (id >= 0) tpos[q] = (int)(base + i);
            else fposv[q] = (int)(base + i);
        }
    }
}

// Pull layout of one tile (pull.cuh; create time, host).  Every constraint incident to the tile gets
// one primary own vertex: internal constraints the endpoint from which the rest-pose offset to the
// other endpoint is lexicographically positive (quantized on the Morton cell, so on a lattice every
// vertex is primary for the same set of directions), cross-tile constraints their own endpoint
// (they are primary in both tiles).  A vertex's primaries are ordered (canonical direction first,
// then by offset) and the first K0 fill the dense slabs [k][i]; the rest go to the tile's overflow
// list.  Slot (k, i) / K0 * kTileV + e is both the block's position in the tile's Q region and the
// y slot the secondary endpoint (or the overflow entry's own vertex) reads.  Local slots: own
// vertex v -> v - t * kTileV, halo vertex -> kTileV + rank in the tile's sorted halo list.
// count mode (idx == nullptr): only td.z / td.w (K0 | KS2 << 8, overflow entries).
struct PullScratch {
    struct Prim { int flag; long long kx, ky, kz; int q, other, kind, color, slot; };   // kind 0 internal, 1 own cross, 2 foreign
    std::vector<std::vector<Prim>> prim;
    std::vector<std::vector<int>> sec;               // y-slot entries (slot | add flag << 15)
    std::vector<std::pair<int, int>> internal_sec;   // (secondary vertex, constraint q) resolved after ranking
    std::vector<std::pair<int, int>> qpos;           // (q, slot) of internal constraints
    std::vector<std::tuple<int, int, int>> order;    // (color, vertex, rank)
    std::vector<int> lane;                           // [slab][vertex]: lane of the vertex's slot in its warp's 32
};

static void pull_tile_layout(int t, int nc, int nt, const std::vector<int> &halo_t, const int64_t *cnt,
                             const int64_t *fc, const int2 *ab, const int *fidx, const float *xrest,
                             const int32_t *vperm, double hcell, int nvt, int4 &td, uint32_t *idx, int *tpos,
                             int *fposv, PullScratch &w) {
    auto local = [&](int v) {
        return v / kTileV == t ? v - t * kTileV
                               : kTileV + (int)(std::lower_bound(halo_t.begin(), halo_t.end(), v) - halo_t.begin());
    };
    const double ih = hcell > 0 ? 1.0 / hcell : 0.0;
    auto offset = [&](int from, int to, long long (&k)[3]) {   // quantized rest offset; returns its lexicographic sign
        for (int c = 0; c < 3; ++c)
            k[c] = std::llround(((double)xrest[3 * (size_t)vperm[to] + c] - (double)xrest[3 * (size_t)vperm[from] + c]) * ih);
        for (int c = 0; c < 3; ++c)
            if (k[c] != 0) return k[c] > 0 ? 1 : -1;
        return 0;
    };
    w.prim.resize(kTileV);
    w.sec.resize(kTileV);
    for (int i = 0; i < kTileV; ++i) { w.prim[i].clear(); w.sec[i].clear(); }
    w.internal_sec.clear();
    for (int c = 0; c < nc; ++c) {
        const size_t kk = (size_t)c * nt + t;
        for (int64_t q = cnt[kk]; q < cnt[kk + 1]; ++q) {   // a own
            const int a = ab[q].x, b = ab[q].y;
            long long k[3];
            const int sg = offset(a, b, k);
            if (b / kTileV == t) {
                if (sg >= 0) {
                    w.prim[a - t * kTileV].push_back({0, k[0], k[1], k[2], (int)q, b - t * kTileV, 0, c, 0});
                    w.internal_sec.push_back({b - t * kTileV, (int)q});
                } else {
                    w.prim[b - t * kTileV].push_back({0, -k[0], -k[1], -k[2], (int)q, a - t * kTileV, 0, c, 0});
                    w.internal_sec.push_back({a - t * kTileV, (int)q});
                }
            } else {
                w.prim[a - t * kTileV].push_back({sg >= 0 ? 0 : 1, k[0], k[1], k[2], (int)q, local(b), 1, c, 0});
            }
        }
        for (int64_t k2 = fc[kk]; k2 < fc[kk + 1]; ++k2) {   // b own, a in another tile
            const int q = fidx[k2];
            const int a = ab[q].x, b = ab[q].y;
            long long k[3];
            const int sg = offset(b, a, k);
            w.prim[b - t * kTileV].push_back({sg > 0 ? 0 : 1, k[0], k[1], k[2], q, local(a), 2, c, 0});
        }
    }
    int fill[kPullK0] = {0};
    w.lane.assign((size_t)kPullK0 * kTileV, 0);
    for (int i = 0; i < kTileV; ++i) {
        auto &p = w.prim[i];
        std::sort(p.begin(), p.end(), [](const PullScratch::Prim &x, const PullScratch::Prim &y) {
            return std::tie(x.flag, x.kx, x.ky, x.kz, x.q) < std::tie(y.flag, y.kx, y.ky, y.kz, y.q);
        });
        for (int k = 0; k < std::min<int>(kPullK0, (int)p.size()); ++k) fill[k]++;
    }
    // dense slab k pays off while at least half of the tile's vertices use it (a padded entry costs
    // 18 bytes, an overflow entry 22 and a secondary)
    int K0 = 0;
    while (K0 < kPullK0 && fill[K0] > 0 && (K0 == 0 || 2 * fill[K0] >= nvt)) ++K0;
    const int K02 = (K0 + 1) / 2;
    // y slots = Q positions.  Dense slab k: within each aligned block of 32 vertices (one warp) the
    // entries are grouped by color, so the replay's per-color launches write runs of consecutive
    // blocks (a lattice direction holds two colors: 256-byte runs); inside its color's lane range
    // each vertex takes a lane whose 16-byte bank group is still free in its quarter-warp's access
    // phase (conflict-free direct accesses).  The lane goes into the primary entry.  Overflow
    // entries: by color.
    for (int k = 0; k < K0; ++k)
        for (int b0 = 0; b0 < kTileV; b0 += 32) {
            w.order.clear();
            for (int i = b0; i < b0 + 32; ++i)
                if ((int)w.prim[i].size() > k) w.order.push_back({w.prim[i][k].color, i, k});
            std::sort(w.order.begin(), w.order.end());
            int lo[32], hi[32];   // per vertex of the block: its color's lane range
            for (size_t l = 0; l < w.order.size();) {
                size_t m = l;
                while (m < w.order.size() && std::get<0>(w.order[m]) == std::get<0>(w.order[l])) ++m;
                for (size_t q = l; q < m; ++q) { lo[std::get<1>(w.order[q]) - b0] = (int)l; hi[std::get<1>(w.order[q]) - b0] = (int)m; }
                l = m;
            }
            uint32_t taken = 0;
            for (int i = b0; i < b0 + 32; ++i) w.lane[(size_t)k * kTileV + i] = -1;
            for (int q8 = 0; q8 < 4; ++q8) {
                uint32_t banks = 0;   // 16-byte bank groups used by this quarter-warp's access phase
                for (int i = b0 + 8 * q8; i < b0 + 8 * q8 + 8; ++i) {
                    if ((int)w.prim[i].size() <= k) continue;
                    int best = -1;
                    for (int l = lo[i - b0]; l < hi[i - b0]; ++l) {
                        if ((taken >> l) & 1) continue;
                        if (best < 0) best = l;
                        if (!((banks >> (l & 7)) & 1)) { best = l; break; }
                    }
                    taken |= 1u << best;
                    banks |= 1u << (best & 7);
                    w.prim[i][k].slot = k * kTileV + b0 + best;
                    w.lane[(size_t)k * kTileV + i] = best;
                }
            }
            // vertices without a k-th primary take the lanes left over (their entry is "none", but
            // the kernels stay branch-free: every thread owns one slot of the slab)
            int free_l = 0;
            for (int i = b0; i < b0 + 32; ++i)
                if (w.lane[(size_t)k * kTileV + i] < 0) {
                    while ((taken >> free_l) & 1) ++free_l;
                    taken |= 1u << free_l;
                    w.lane[(size_t)k * kTileV + i] = free_l;
                }
        }
    w.order.clear();
    for (int i = 0; i < kTileV; ++i)
        for (int r = K0; r < (int)w.prim[i].size(); ++r) w.order.push_back({w.prim[i][r].color, i, r});
    std::sort(w.order.begin(), w.order.end());
    const int nover = (int)w.order.size();
    for (int e = 0; e < nover; ++e) {
        const int i = std::get<1>(w.order[e]);
        w.prim[i][std::get<2>(w.order[e])].slot = K0 * kTileV + e;
        w.sec[i].push_back((K0 * kTileV + e) | 0x8000);   // the own vertex adds y = Q (p_own - p_other)
    }
    w.qpos.clear();
    for (int i = 0; i < kTileV; ++i)
        for (auto &pr : w.prim[i]) {
            if (pr.kind == 0) w.qpos.push_back({pr.q, pr.slot});
            if (idx) {
                if (pr.kind == 2) fposv[pr.q] = td.x + pr.slot;
                else tpos[pr.q] = td.x + pr.slot;
            }
        }
    std::sort(w.qpos.begin(), w.qpos.end());
    for (auto &is : w.internal_sec) {
        auto itp = std::lower_bound(w.qpos.begin(), w.qpos.end(), std::make_pair(is.second, INT32_MIN));
        w.sec[is.first].push_back(itp->second);   // the partner subtracts
    }
    int KS = 0;
    for (int i = 0; i < kTileV; ++i) {
        std::sort(w.sec[i].begin(), w.sec[i].end(), [](int x, int y) { return (x & 0x7fff) < (y & 0x7fff); });
        KS = std::max(KS, (int)w.sec[i].size());
    }
    const int KS2 = (KS + 1) / 2;
    td.z = K0 | (KS2 << 8);
    td.w = nover;
    if (!idx) return;
    uint32_t *pw = idx, *sw = idx + (size_t)K02 * kTileV, *ow = sw + (size_t)KS2 * kTileV;
    for (size_t k = 0; k < (size_t)(K02 + KS2) * kTileV; ++k) idx[k] = 0xffffffffu;
    for (int k = 0; k < K0; ++k)   // "none" primaries: other = 0x7ff, their own (unused) lane
        for (int i = 0; i < kTileV; ++i)
            if ((int)w.prim[i].size() <= k) {
                uint32_t &wd = pw[(size_t)(k / 2) * kTileV + i];
                const uint32_t v = 0x7ffu | ((uint32_t)w.lane[(size_t)k * kTileV + i] << 11);
                wd = (k & 1) ? ((wd & 0xffffu) | (v << 16)) : ((wd & 0xffff0000u) | v);
            }
    auto put16 = [](uint32_t &wd, int r, uint32_t v) {
        wd = (r & 1) ? ((wd & 0xffffu) | (v << 16)) : ((wd & 0xffff0000u) | v);
    };
    for (int i = 0; i < kTileV; ++i) {
        auto &p = w.prim[i];
        for (int r = 0; r < (int)p.size(); ++r) {
            if (r < K0) put16(pw[(size_t)(r / 2) * kTileV + i], r, (uint32_t)p[r].other | ((uint32_t)(p[r].slot & 31) << 11));
            else ow[p[r].slot - K0 * kTileV] = (uint32_t)i | ((uint32_t)p[r].other << 16);
        }
        for (int r = 0; r < (int)w.sec[i].size(); ++r) put16(sw[(size_t)(r / 2) * kTileV + i], r, (uint32_t)w.sec[i][r]);
    }
}

static inline uint64_t spread3(uint64_t x) {
    x &= 0x1fffff;
    x = (x | x << 32) & 0x1f00000000ffffull;
    x = (x | x << 16) & 0x1f0000ff0000ffull;
    x = (x | x << 8) & 0x100f00f00f00f00full;
    x = (x | x << 4) & 0x10c30c30c30c30c3ull;
    x = (x | x << 2) & 0x1249249249249249ull;
    return x;
}
// The quantization cell is the mesh's short edge length h (10th percentile of a sample of rest
// lengths), so a regular grid maps onto the integer lattice and every run of 2^k consecutive Morton
// codes is an aligned lattice block: tiles are compact rectangles / boxes (32 x 16 at kTileV = 512 on
// a cloth grid), which minimises tile halos and cross-tile constraints.  A cell of extent / 2^21
// (the key's resolution) when h is unknown or smaller.
void morton_order(const float *x, int V, double h, std::vector<int32_t> &perm, const int32_t *scene = nullptr) {
    float lo[3] = {x[0], x[1], x[2]}, hi[3] = {x[0], x[1], x[2]};
    for (int i = 0; i < V; ++i)
        for (int k = 0; k < 3; ++k) { lo[k] = std::min(lo[k], x[3 * i + k]); hi[k] = std::max(hi[k], x[3 * i + k]); }
    float ext = std::max(hi[0] - lo[0], std::max(hi[1] - lo[1], hi[2] - lo[2]));
    const double cell = std::max(h, (double)ext / 2097151.0);
    double sc = cell > 0 ? 1.0 / cell : 0.0;
    // (scene, Morton code, index): a batch keeps each scene's vertices contiguous
    std::vector<std::tuple<int32_t, uint64_t, int32_t>> key(V);
    for (int i = 0; i < V; ++i) {
        uint64_t q[3];
        for (int k = 0; k < 3; ++k) q[k] = (uint64_t)std::llround((x[3 * i + k] - lo[k]) * sc);
        key[i] = std::make_tuple(scene ? scene[i] : 0, spread3(q[0]) | (spread3(q[1]) << 1) | (spread3(q[2]) << 2), i);
    }
    std::sort(key.begin(), key.end());
    perm.resize(V);
    for (int i = 0; i < V; ++i) perm[i] = std::get<2>(key[i]);
}

// dst[i] = src[perm[i]] for [count][V][3] arrays (user -> internal vertex order)
__global__ void k_gather3(int V, int count, const float *__restrict__ src, const int32_t *__restrict__ perm,
                          float *__restrict__ dst) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)V * count) return;
    size_t f = i / V, v = i % V;
    const float *s = src + (f * V + perm[v]) * 3;
    float *o = dst + i * 3;
    o[0] = s[0]; o[1] = s[1]; o[2] = s[2];
}
// dst[perm[i]] = src[i] (internal -> user vertex order)
__global__ void k_scatter3(int V, int count, const float *__restrict__ src, const int32_t *__restrict__ perm,
                           float *__restrict__ dst) {
    size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (size_t)V * count) return;
    size_t f = i / V, v = i % V;
    const float *s = src + i * 3;
    float *o = dst + (f * V + perm[v]) * 3;
    o[0] = s[0]; o[1] = s[1]; o[2] = s[2];
}
__global__ void k_gather1(int V, const float *__restrict__ src, const int32_t *__restrict__ perm, float *__restrict__ dst) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < V) dst[i] = src[perm[i]];
}
// user-order [V][3] -> internal double4 / float4 (gathered through perm)
__global__ void k_pack4d(int V, const float *__restrict__ x3, const int32_t *__restrict__ perm,
                         const float *__restrict__ w, double4 *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    int u = perm[i];
    out[i] = make_double4(x3[3 * u], x3[3 * u + 1], x3[3 * u + 2], w ? (double)w[i] : 0.0);
}
__global__ void k_pack4g(int V, const float *__restrict__ x3, const int32_t *__restrict__ perm, float4 *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    int u = perm[i];
    out[i] = make_float4(x3[3 * u], x3[3 * u + 1], x3[3 * u + 2], 0.f);
}
// internal double4 -> user-order [V][3] float
__global__ void k_unpack3(int V, const double4 *__restrict__ x, const int32_t *__restrict__ perm, float *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    double4 p = x[i];
    int u = perm[i];
    out[3 * u] = (float)p.x; out[3 * u + 1] = (float)p.y; out[3 * u + 2] = (float)p.z;
}
__global__ void k_gather_f(int n, const float *__restrict__ src, const int32_t *__restrict__ perm, float *__restrict__ dst) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    dst[j] = src[perm[j]];
}
__global__ void k_scatter_f(int n, const float *__restrict__ src, const int32_t *__restrict__ perm, float *__restrict__ dst) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    dst[perm[j]] = src[j];
}
// [T][2] sorted -> user order / user (a, b) pairs -> sorted split arrays
__global__ void k_scatter_pair(int n, const float *__restrict__ src, const int32_t *__restrict__ perm, float *__restrict__ dst) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    dst[2 * perm[j]] = src[2 * j];
    dst[2 * perm[j] + 1] = src[2 * j + 1];
}
__global__ void k_gather_pair_split(int n, const float *__restrict__ src, const int32_t *__restrict__ perm,
                                    float *__restrict__ a, float *__restrict__ b) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    a[j] = src[2 * perm[j]];
    b[j] = src[2 * perm[j] + 1];
}
// rest length L_j = |x_rest[a] - x_rest[b]|
__global__ void k_rest_len(int n, const int2 *__restrict__ idx, const float *__restrict__ xr, float *__restrict__ rest) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int2 e = idx[j];
    float dx = xr[3 * e.x] - xr[3 * e.y], dy = xr[3 * e.x + 1] - xr[3 * e.y + 1], dz = xr[3 * e.x + 2] - xr[3 * e.y + 2];
    rest[j] = sqrtf(dx * dx + dy * dy + dz * dz);
}
// capsule radius/length from shape coefficients (R7): r = r0 + R beta, L = L0 + Lc beta
__global__ void k_shape_apply(int nsph, int ncap, int ns, const float *__restrict__ spheres,
                              const float *__restrict__ cc, const float *__restrict__ ca, const float *__restrict__ r0,
                              const float *__restrict__ L0, const float *__restrict__ Rb, const float *__restrict__ Lb,
                              const float *__restrict__ beta, Collider *__restrict__ out,
                              const int *__restrict__ csc) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nsph) {
        Collider c;
        c.c = make_float4(spheres[4 * k], spheres[4 * k + 1], spheres[4 * k + 2], 0.f);
        c.a = make_float4(0.f, 0.f, 0.f, 0.f);
        c.r = spheres[4 * k + 3];
        c.L = 0.f;
        c.type = 0;
        c.scene = csc ? csc[k] : -1;
        out[k] = c;
    } else if (k < nsph + ncap) {
        int q = k - nsph;
        float r = r0[q], L = L0[q];
        for (int s = 0; s < ns; ++s) {
            r += Rb[q * ns + s] * beta[s];
            L += Lb[q * ns + s] * beta[s];
        }
        Collider c;
        c.c = make_float4(cc[3 * q], cc[3 * q + 1], cc[3 * q + 2], 0.f);
        c.a = make_float4(ca[3 * q], ca[3 * q + 1], ca[3 * q + 2], 0.f);
        c.r = r;
        c.L = L;
        c.type = 1;
        c.scene = csc ? csc[k] : -1;
        out[k] = c;
    }
}
// dphi/dbeta_s = Sum_k Rb[k,s] dphi/dr_k + Lb[k,s] dphi/dL_k ; sphere grads copied out
__global__ void k_shape_grad(int nsph, int ncap, int ns, const double *__restrict__ acc, const float *__restrict__ Rb,
                             const float *__restrict__ Lb, float *__restrict__ gbeta, float *__restrict__ gsph) {
    int s = blockIdx.x * blockDim.x + threadIdx.x;
    if (s < ns) {
        double g = 0.0;
        for (int q = 0; q < ncap; ++q)
            g += Rb[q * ns + s] * acc[4 * (nsph + q)] + Lb[q * ns + s] * acc[4 * (nsph + q) + 1];
        gbeta[s] = (float)g;
    }
    if (s < 4 * nsph) gsph[s] = (float)acc[s];
}

}  // namespace

// ------------------------------------------------------------------ host topology (create time)
// Everything the scene's distance-constraint layout needs, computed on the host without a GPU, so
// the same code serves dxpbd_create, the partition planner of the domain decomposition and the
// host-only dxpbd_partition_plan (tested on CPU with gloo ranks).
struct DistTopo {
    int V = 0, E = 0, nt = 0, nc = 0;
    std::vector<int32_t> vperm;                 // internal -> user vertex (Morton order)
    std::vector<int32_t> color, perm;           // greedy color per user constraint; sorted position -> user index
    std::vector<int> dist_off, seg, fseg;       // color offsets; [nc][nt + 1] own / foreign segment offsets
    std::vector<int2> ab;                       // sorted constraints, internal endpoints (a < b)
    std::vector<std::vector<int>> halo;         // per tile: halo vertices (sorted)
    std::vector<int> fidx;                      // foreign lists (sorted constraint positions)
    int64_t n_foreign = 0, halo_total = 0;
    int hcap = 0, capm = 0;
    bool use_tma = false;
    // TMA layout (use_tma)
    std::vector<int> hpad, fposv, tpos;
    std::vector<int4> tseg;
    std::vector<uint32_t> cpair;
    std::vector<uint16_t> vslot, hslot;
    int64_t ntot = 0;
    // pull layout (use_tma && pull; closed-form K = 1 blocks only): replaces tseg / cpair / vslot / hslot
    bool pull = false;
    int ycap = 0;
    std::vector<int4> ptd;
    std::vector<uint32_t> pidx;
};

// Morton vertex order with the short-edge quantization cell (see morton_order)
double vertex_order(const dxpbd_scene_desc *d, std::vector<int32_t> &vperm) {
    std::vector<double> len;
    auto edge = [&](int a, int b) {
        double q = 0;
        for (int k = 0; k < 3; ++k) { const double u = (double)d->x_rest[3 * a + k] - d->x_rest[3 * b + k]; q += u * u; }
        if (q > 0) len.push_back(std::sqrt(q));
    };
    // short edge length: 10th percentile over a sample of distance-constraint (else tet) edges (on a
    // cloth grid the structural spacing, not the shear / bending lengths)
    const int64_t ne = d->num_dist, nte = d->num_tets;
    for (int64_t j = 0; j < ne; j += std::max<int64_t>(1, ne / 65536)) edge(d->dist_idx[2 * j], d->dist_idx[2 * j + 1]);
    if (len.empty())
        for (int64_t j = 0; j < nte; j += std::max<int64_t>(1, nte / 65536)) edge(d->tet_idx[4 * j], d->tet_idx[4 * j + 1]);
    double h = 0;
    if (!len.empty()) {
        std::nth_element(len.begin(), len.begin() + len.size() / 10, len.end());
        h = len[len.size() / 10];
    }
    if (const char *ev = getenv("DXPBD_MORTON_CELL")) h = atof(ev);   // 0: the extent / 2^21 cell (A/B)
    morton_order(d->x_rest, d->num_vertices, h, vperm, d->vertex_scene);
    return h;
}

// Distance constraints: greedy colors in user order (R1), then sorted by (color, owner tile) with
// each constraint oriented (a < b) in internal ids; owner tile = a / kTileV; halo sets, foreign
// lists and (when it fits) the TMA tile layout.
void dist_topology(const dxpbd_scene_desc *d, int qf, DistTopo &T) {
    const int V = d->num_vertices, E = d->num_dist;
    T.V = V;
    T.E = E;
    const double hcell = vertex_order(d, T.vperm);
    T.nt = (V + kTileV - 1) / kTileV;
    if (!E) return;
    std::vector<int32_t> vinv(V);
    for (int i = 0; i < V; ++i) vinv[T.vperm[i]] = i;
    const int nc = greedy_colors(E, 2, d->dist_idx, V, T.color);
    if (nc < 0) throw Err{DXPBD_ERR_LIMIT, "distance coloring needs more than 256 colors"};
    T.nc = nc;
    const int nt = T.nt;
    const size_t nkeys = (size_t)nc * nt;
    std::vector<int2> ab(E);
    std::vector<int64_t> cnt(nkeys + 1, 0);
    std::vector<int32_t> key(E);
    for (int j = 0; j < E; ++j) {
        int a = vinv[d->dist_idx[2 * j]], b = vinv[d->dist_idx[2 * j + 1]];
        if (a > b) std::swap(a, b);
        ab[j] = make_int2(a, b);
        key[j] = T.color[j] * nt + a / kTileV;
        cnt[key[j] + 1]++;
    }
    for (size_t k = 0; k < nkeys; ++k) cnt[k + 1] += cnt[k];
    T.seg.assign((size_t)nc * (nt + 1), 0);
    T.dist_off.assign(nc + 1, 0);
    for (int c = 0; c < nc; ++c) {
        for (int t = 0; t <= nt; ++t) T.seg[(size_t)c * (nt + 1) + t] = (int)cnt[(size_t)c * nt + t];
        T.dist_off[c] = (int)cnt[(size_t)c * nt];
    }
    T.dist_off[nc] = E;
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    T.perm.assign(E, 0);
    for (int j = 0; j < E; ++j) T.perm[pos[key[j]]++] = j;
    // within each (color, tile) segment order by internal a (vertex-disjoint within a color, so
    // a is unique there): consecutive threads touch consecutive Morton vertices (no smem bank
    // conflicts in the tiled matvec); the Gauss-Seidel result does not depend on this order.
    for (size_t kk = 0; kk < nkeys; ++kk)
        std::sort(T.perm.begin() + cnt[kk], T.perm.begin() + cnt[kk + 1], [&](int32_t x, int32_t y) { return ab[x].x < ab[y].x; });
    // halo sets per tile (order-independent): the other endpoints of cross-tile constraints
    T.halo.assign(nt, {});
    for (int j = 0; j < E; ++j) {
        int a = ab[j].x, bb = ab[j].y, ta = a / kTileV, tb = bb / kTileV;
        if (ta != tb) { T.halo[ta].push_back(bb); T.halo[tb].push_back(a); }
    }
    for (int t = 0; t < nt; ++t) {
        std::sort(T.halo[t].begin(), T.halo[t].end());
        T.halo[t].erase(std::unique(T.halo[t].begin(), T.halo[t].end()), T.halo[t].end());
    }
    T.ab.resize(E);
    for (int q = 0; q < E; ++q) T.ab[q] = ab[T.perm[q]];
    const std::vector<int2> &ab_sorted = T.ab;
    // foreign lists: constraints whose b lies in another tile than a, keyed (color, tile(b))
    std::vector<int64_t> fc(nkeys + 1, 0);
    for (int q = 0; q < E; ++q) {
        int ta = ab_sorted[q].x / kTileV, tb = ab_sorted[q].y / kTileV;
        if (ta != tb) fc[(size_t)T.color[T.perm[q]] * nt + tb + 1]++;
    }
    for (size_t k = 0; k < nkeys; ++k) fc[k + 1] += fc[k];
    T.fseg.assign((size_t)nc * (nt + 1), 0);
    for (int c = 0; c < nc; ++c)
        for (int t = 0; t <= nt; ++t) T.fseg[(size_t)c * (nt + 1) + t] = (int)fc[(size_t)c * nt + t];
    T.fidx.assign(std::max<int64_t>(fc[nkeys], 1), 0);
    std::vector<int64_t> fp(fc.begin(), fc.end() - 1);
    for (int q = 0; q < E; ++q) {
        int ta = ab_sorted[q].x / kTileV, tb = ab_sorted[q].y / kTileV;
        if (ta != tb) T.fidx[fp[(size_t)T.color[T.perm[q]] * nt + tb]++] = q;
    }
    for (size_t kk = 0; kk < nkeys; ++kk)
        std::sort(T.fidx.begin() + fc[kk], T.fidx.begin() + fc[kk + 1], [&](int x, int y) { return ab_sorted[x].y < ab_sorted[y].y; });
    T.n_foreign = fc[nkeys];
    // CG-local tile structure for the TMA-staged kernels (kernels.cuh "TMA-staged")
    int hmax = 0;
    for (int t = 0; t < nt; ++t) {
        T.halo_total += (int64_t)T.halo[t].size();
        hmax = std::max(hmax, (int)T.halo[t].size());
    }
    T.hcap = (hmax + 31) / 32 * 32;
    // combined (own + foreign) segments, tile-major: tile t's colors are contiguous
    std::vector<int64_t> cbase((size_t)nt * nc + 1, 0);
    int maxn = 0;
    for (int t = 0; t < nt; ++t)
        for (int c = 0; c < nc; ++c) {
            const size_t kk = (size_t)c * nt + t;
            const int64_t n = (cnt[kk + 1] - cnt[kk]) + (fc[kk + 1] - fc[kk]);
            cbase[(size_t)t * nc + c + 1] = cbase[(size_t)t * nc + c] + n;
            maxn = std::max<int>(maxn, (int)n);
        }
    T.capm = (maxn + 7) & ~7;
    T.use_tma = hmax <= 4096 && nc <= kMaxColors && cbase.back() < (int64_t)INT32_MAX &&
                tma_rhs_smem_bytes(T.hcap, T.capm, qf == 0) <= 200 * 1024;
    if (!T.use_tma) return;
    const int hc = T.hcap;
    T.hpad.assign((size_t)nt * hc, -1);
    for (int t = 0; t < nt; ++t) std::copy(T.halo[t].begin(), T.halo[t].end(), T.hpad.begin() + (size_t)t * hc);
    const int nth = std::max(1, std::min(32, (int)std::thread::hardware_concurrency()));
    auto run_tiles = [&](auto &&work) {
        std::vector<std::thread> pool;
        for (int k = 0; k < nth; ++k) pool.emplace_back(work, (int)((int64_t)nt * k / nth), (int)((int64_t)nt * (k + 1) / nth));
        for (auto &th : pool) th.join();
    };
    // pull layout (pull.cuh) for closed-form blocks: count pass, offsets, fill pass
    const char *pe = getenv("DXPBD_PULL");
    if (qf == 1 && !(pe && atoi(pe) == 0)) {
        T.ptd.assign(nt, make_int4(0, 0, 0, 0));
        auto tile = [&](int t, uint32_t *idx, PullScratch &ws) {
            pull_tile_layout(t, nc, nt, T.halo[t], cnt.data(), fc.data(), ab_sorted.data(), T.fidx.data(), d->x_rest,
                             T.vperm.data(), hcell, std::min(kTileV, V - t * kTileV), T.ptd[t], idx, T.tpos.data(),
                             T.fposv.data(), ws);
        };
        run_tiles([&](int t0, int t1) {
            PullScratch ws;
            for (int t = t0; t < t1; ++t) tile(t, nullptr, ws);
        });
        int64_t qb = 0, ib = 0;
        int ycap = 0;
        for (int t = 0; t < nt; ++t) {
            const int K0 = T.ptd[t].z & 0xff, KS2 = (T.ptd[t].z >> 8) & 0xff, no = T.ptd[t].w;
            T.ptd[t].x = (int)qb;
            T.ptd[t].y = (int)ib;
            qb += (int64_t)K0 * kTileV + no;
            ib += ((int64_t)((K0 + 1) / 2 + KS2) * kTileV + no + 3) & ~(int64_t)3;
            ycap = std::max(ycap, K0 * kTileV + no);
        }
        if (qb < (int64_t)INT32_MAX && ib < (int64_t)INT32_MAX && ycap <= kPullMaxY && kTileV + hc <= kPullMaxSlot &&
            pull_smem_bytes(hc, ycap, 2) <= 110 * 1024) {
            T.pull = true;
            T.ycap = ycap;
            T.ntot = qb;
            T.pidx.assign((size_t)ib + 4, 0xffffffffu);
            T.fposv.assign(E, -1);
            T.tpos.assign(E, 0);
            run_tiles([&](int t0, int t1) {
                PullScratch ws;
                for (int t = t0; t < t1; ++t) tile(t, T.pidx.data() + T.ptd[t].y, ws);
            });
            return;
        }
        T.ptd.clear();
    }
    T.tseg.resize((size_t)nt * nc);
    for (size_t k = 0; k < (size_t)nt * nc; ++k) T.tseg[k] = make_int4((int)cbase[k], (int)cbase[k + 1], 0, 0);
    T.ntot = cbase.back();
    T.cpair.assign((size_t)T.ntot + 4, 0);
    T.fposv.assign(E, -1);
    T.tpos.assign(E, 0);
    T.vslot.assign((size_t)nt * kTileV, 0);
    T.hslot.assign((size_t)nt * hc, 0);
    // per tile (independent, threaded): bank-balanced shared-memory slots, then conflict-free
    // groups of every combined (tile, color) segment (tma_tile_layout)
    auto work = [&](int t0, int t1) {
        TileLayoutScratch ws;
        for (int t = t0; t < t1; ++t)
            tma_tile_layout(t, nc, nt, hc, T.halo[t], t * hc, cnt.data(), fc.data(), ab_sorted.data(), T.fidx.data(),
                            cbase.data(), T.vslot.data(), T.hslot.data(), T.tpos.data(), T.fposv.data(), T.cpair.data(), ws);
    };
    run_tiles(work);
}

struct dxpbd_scene {
    int device = 0;
    int V = 0, E = 0, T = 0, NS = 0, NCAP = 0, NSH = 0, NC = 0;
    float dt = 0, inv_dt = 0, frame_dt = 0;
    double dtd = 0, inv_dt2d = 0;   // fp64 time step for the position-state arithmetic
    int substeps = 1, iterations = 1, max_frames = 0;
    float3 gravity{0, 0, 0};
    float h = 0, coll_alpha = 0;
    uint32_t grad_flags = 0;
    int pd = 1;
    float cg_tol = 1e-6f;
    int cg_max_iter = 500;

    // topology (color-sorted)
    int n_dist_colors = 0, n_tet_colors = 0;
    std::vector<int> dist_off, tet_off;
    std::vector<int32_t> dist_perm_h, dist_color_h, tet_perm_h, tet_color_h;
    DBuf<int2> d_idx;
    DBuf<float> d_rest, d_alpha;
    DBuf<int32_t> d_perm;
    DBuf<float> inv_mass;                 // internal vertex order
    std::vector<int32_t> vperm_h;         // internal -> user vertex
    DBuf<int32_t> vperm;
    int ntiles = 0;
    int64_t n_foreign = 0, halo_total = 0;
    DBuf<int> d_seg;                      // [(n_dist_colors) * (ntiles+1)] (color, owner tile) offsets
    DBuf<int> d_fseg, d_fidx;             // foreign (b-endpoint) constraint lists per (color, tile)
    DBuf<int4> d_fent;                    // foreign entries {j, a, b, 0}
    // CG-local tile structure (TMA-staged matvec, QF = 1)
    bool use_tma = false;
    int capm = 0;             // TMA stage capacity: largest combined (own + foreign) segment
    int hcap = 0;
    size_t tma_smem = 0, tma_rhs_smem = 0;
    DBuf<int> d_hpad, d_fpos;
    DBuf<int4> d_tseg;
    DBuf<uint32_t> d_cpair;
    DBuf<float4> d_Qt;                  // Q blocks in the TMA layout (own at tpos[j], foreign copy at fpos[j])
    DBuf<float2> d_Qt2b;                // general blocks (qf == 0): (yz, zz) in the same layout
    DBuf<uint16_t> d_vslot, d_hslot;   // tile-local shared-memory slots (own vertices, halo entries)
    DBuf<int> d_tpos;                   // sorted constraint position -> TMA layout position
    // pull layout (pull.cuh): closed-form K = 1 blocks; replaces tseg / cpair / vslot / hslot
    bool pull = false;
    int ycap = 0;
    bool pull_persist = true;   // persistent matvec CTAs with next-tile prefetch (A/B: DXPBD_PULL_PERSIST)
    // prediction fused into the first distance color of a K = 1 sweep (k_dist_first); the vertices no
    // color-0 constraint touches are predicted from this list (DXPBD_FUSE_PREDICT)
    bool fuse_predict = false;
    DBuf<int> uncov;
    size_t pull_psmem = 0;
    int num_sms = 148;
    size_t pull_smem = 0, pull_rhs_smem = 0;
    DBuf<int4> d_ptd;
    DBuf<uint32_t> d_pidx;
    PullTiles pull_tiles() const {
        return PullTiles{ntiles, hcap, ycap, d_ptd.p, d_pidx.p, d_hpad.p, qt_read ? qt_read : d_Qt.p};
    }
    // tets (color-sorted, internal vertex ids)
    DBuf<int4> t_idx;
    DBuf<double> t_Dm, t_vol;
    DBuf<float> t_Dmf;
    DBuf<float> t_a, t_b, t_Q, t_e, t_g, lam_t;
    DBuf<double4> t_xsave;   // K = 1 tet replay: pre-update vertices of every tet [4T]
    DBuf<float> t_Q2, t_e2;  // second tet block / control buffers (replay / PCG overlap)
    DBuf<float> t_Q3, t_e3;  // third buffers: three-stage tet pipeline (iterate + blocks | PD projection | PCG)
    bool tet_pipe = true;    // DXPBD_TET_PIPE
    cudaStream_t aux2 = nullptr;
    cudaEvent_t ev_A[3] = {nullptr, nullptr, nullptr}, ev_B[3] = {nullptr, nullptr, nullptr}, ev_P[3] = {nullptr, nullptr, nullptr};
    float *tq_w = nullptr, *te_w = nullptr, *tq_r = nullptr, *te_r = nullptr;   // overlap: replay writes, PCG reads
    DBuf<int32_t> t_perm;
    DBuf<float> ts_lam, ts_S, ts_Dt, ts_Tu, ts_e;   // replay scratch (K > 1)
    DBuf<int> t_goff, t_ginc;   // per vertex: its tet-corner slots (CSR, fixed order)
    DBuf<float> t_gq;           // [2][4][3][T] corner contributions (matvec / rhs y, rhs z)
    TetDev tdev() const { return TetDev{T, t_idx.p, t_Dm.p, t_vol.p, t_a.p, t_b.p, t_Dmf.p, t_goff.p, t_ginc.p, t_gq.p}; }
    TmaTiles tma_tiles() const {
        return TmaTiles{n_dist_colors, ntiles, hcap, capm, d_tseg.p, d_cpair.p, d_hpad.p, qt_read ? qt_read : d_Qt.p,
                        qf == 1 ? nullptr : d_Qt2b.p, d_vslot.p, d_hslot.p};
    }
    // replay / PCG overlap (backward): the replay of substep n-1 runs on `aux` while the PCG of
    // substep n runs on the caller's stream; Q blocks alternate between d_Qt and d_Qt2
    DBuf<float4> d_Qt2;
    float4 *qt_read = nullptr, *qt_write = nullptr;   // null: d_Qt
    cudaStream_t aux = nullptr, hi = nullptr;   // aux: replay (lowest priority), hi: PCG path (highest)
    cudaEvent_t ev_rep[2] = {nullptr, nullptr}, ev_pcg[2] = {nullptr, nullptr}, ev_go = nullptr, ev_end = nullptr;
    bool overlap = true;
    // block cache (forward -> backward): the derivative blocks of substeps [qc_first, qc_first + qc_count)
    // computed during the forward (replay kernels in place of the projection) into spare HBM
    DBuf<float4> qcache;
    DBuf<float> qccache;      // contact blocks (6V) [+ collider controls (12 NC V)] of the cached substeps
    size_t qc_cper = 0;       // floats per cached substep in qccache
    int qc_first = 0, qc_count = 0;
    bool qcache_on = true;
    // wavefront sweep (wave.cuh): predict + all distance colors of a K = 1 substep in one launch
    bool wave_on = false;            // opt-in (DXPBD_WAVE=1): measured slower than the per-color launches
    bool wave_fwd = true, wave_rep = true;   // per pass (DXPBD_WAVE_FWD / DXPBD_WAVE_REP)
    int wave_g = 4;                  // base tiles per wave tile (DXPBD_WAVE_G)
    int wave_grid_fwd = 0;           // forward grid (0: persistent, resident CTAs of every SM; < 0: one item per CTA)
    int wave_grid_rep = -1;          // replay grid (one item per CTA: shares the GPU with the PCG)
    int wave_lag = -1;               // extra ticket lag (DXPBD_WAVE_LAG; < 0: resident CTAs of the GPU)
    int wave_ntw = 0, wave_nitems = 0, wave_L = 0, wave_maxnbr = 0;
    DBuf<int4> wave_items;           // per ticket {wave tile, phase, first constraint, count}
    DBuf<int2> wave_nrange;          // per ticket: neighbour range in wave_nbr
    DBuf<int> wave_nbr;
    DBuf<unsigned> wave_flags;       // [2][ntw]: forward, replay
    DBuf<int> wave_ctr;              // [2] ticket counters
    unsigned wave_base[2] = {0u, 0u};
    // colliders
    DBuf<float> sph, cap_c, cap_a, cap_r0, cap_L0, cap_Rb, cap_Lb, beta;
    DBuf<Collider> cols;
    // batch of scenes: per-vertex scene id (internal order) and per-collider scene (-1: all)
    int num_scenes = 1;
    DBuf<int> vsc, csc;

    // trajectory
    int frames_done = -1;
    DBuf<double4> ckpt;   // [(max_frames*substeps+1) * V] fp64 position state, w = inverse mass
    DBuf<float4> v0;
    DBuf<float> forces;   // [max_frames * V * 3]
    bool have_forces = false;
    DBuf<float> tmp3;     // [V*3] staging
    // host <-> device pipelining: per-frame force uploads overlap the forward, per-frame force-gradient
    // downloads (dxpbd_grads_stream) overlap the backward; two staging slots on a copy stream
    cudaStream_t cpy = nullptr;
    DBuf<float> stage[2];
    cudaEvent_t ev_cp[2] = {nullptr, nullptr}, ev_free[2] = {nullptr, nullptr};
    float *gs_out = nullptr;   // registered output of the next backward's force gradients
    int gs_mem = 0;

    // forward scratch for iterations > 1
    DBuf<float> lam_d, lam_c;

    // backward
    DBuf<double4> xr;
    DBuf<float3> ax, rhs, y, r, p, q, p1, uprev, u0;   // packed 12 B vector fields
    DBuf<float3> uprev2;                               // u_{n+3} (quadratic warm start, warm_order 2)
    int warm_order = 2;                                // PCG warm start: extrapolation order (1 or 2; TMA path)
    int nb = 1;                                        // K = 1 forward projection: constraints per thread
    int nb_rep = 2;                                    // K = 1 replay: constraints per thread
    int rep_minb = 3;                                  // K = 1 replay: launch-bounds CTAs per SM (measured best)
    bool defer_u = true;                               // PCG: u += alpha p deferred into the next matvec (measured best)
    int last_iters = 0;                                // PCG iterations of the previous solve (poll schedule)
    int poll_extra = 0;                                // iterations launched beyond last_iters before the first poll
    bool tetv = true;                                  // no distance constraints: 2-launch PCG iteration (k_cg_tetv)
    int tetv_minb = 1;                                 // its launch-bounds CTAs per SM
    float psd_tol = 1e-6f;                             // tet PD projection: Jacobi stop (off-diagonal / scale)
    int psd_sweeps = 12;                               // and sweep cap
    int psd_minb = 3;                                  // its launch-bounds CTAs per SM (measured best)
    int qf = 0;   // Q format: 0 = sym6 SoA, 1 = iso+rank1 float4 (K = 1 with PD projection)
    DBuf<float> Qd, ed, Qc, ec;
    DBuf<float> Qc2, ec2;                              // second contact block / control buffers (overlap)
    float *qc_w = nullptr, *ec_w = nullptr, *qc_r = nullptr, *ec_r = nullptr;   // overlap: replay writes, PCG reads
    DBuf<float> sc_lam, sc_sig, sc_B, sc_T, sc_e;               // distance scratch (K>1)
    DBuf<float> cc_lam, cc_T, cc_sig, cc_B, cc_e;               // contact scratch (K>1)
    DBuf<double> cg_sc, acc;
    // sweep graphs: the launch sequence of a K = 1 color sweep (distance colors, tet colors and blocks,
    // contacts) captured once and replayed per substep (small scenes are launch-latency bound)
    bool sweep_graph = true;                       // DXPBD_SWEEP_GRAPH
    int sweep_graph_maxv = 1 << 21;                // only below this many vertices (the forward copies the iterate)
    cudaGraphExec_t g_fwd = nullptr;
    struct RepGraph { std::vector<const void *> key; cudaGraphExec_t e; int launches; };
    std::vector<RepGraph> g_rep;                   // keyed by the output buffers (and the replay stage)
    struct PcgChunk { int iters, launches; cudaGraphExec_t e; };
    std::vector<PcgChunk> g_pcg;                   // first PCG chunk, keyed by its iteration count
    int g_fwd_launches = 0;
    DBuf<double4> xw;                              // forward graph iterate
    cudaStream_t cap_lo = nullptr, cap_mid = nullptr;
    // PCG as a CUDA graph with a conditional WHILE node (no host polls).  Opt-in (DXPBD_PCG_GRAPH=1):
    // measured 3-15 % slower than the host-polled loop with its iteration-count prediction
    bool pcg_graph = false;
    DBuf<PcgCtl> pcg_ctl;
    DBuf<PcgPtrs> pcg_pp;
    cudaStream_t cap = nullptr;
    cudaGraphExec_t pcg_exec = nullptr;
    int pcg_kernels_per_it = 0;
    DBuf<float> targets, weights;
    DBuf<float> g_comp, g_force, g_shape, g_sph;
    DBuf<float> g_x0, g_v0;
    bool have_grads = false;

    // stats
    double stats[24] = {0};
    // opt-in event profiler
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    size_t ev_used = 0;
    std::vector<std::pair<int, size_t>> prof_rec;   // (class, index of start event)
    double *h_scal = nullptr;   // pinned host scratch
};

namespace {

inline void prof_begin(dxpbd_scene *s, int cls, cudaStream_t st) {
    if (!s->prof) return;
    if (s->ev_used + 2 > s->ev_pool.size()) {
        size_t n0 = s->ev_pool.size(), n1 = std::max<size_t>(2 * n0, 1024);
        s->ev_pool.resize(n1);
        for (size_t i = n0; i < n1; ++i) DX_CHECK_CUDA(cudaEventCreate(&s->ev_pool[i]));
    }
    s->prof_rec.push_back({cls, s->ev_used});
    DX_CHECK_CUDA(cudaEventRecord(s->ev_pool[s->ev_used], st));
    s->ev_used += 2;
}
inline void prof_end(dxpbd_scene *s, cudaStream_t st) {
    if (!s->prof) return;
    DX_CHECK_CUDA(cudaEventRecord(s->ev_pool[s->prof_rec.back().second + 1], st));
}
#define LAUNCH(cls, ...)                 \
    do {                                 \
        prof_begin(s, (cls), st);        \
        __VA_ARGS__;                     \
        prof_end(s, st);                 \
    } while (0)

void upload(void *dst, const void *src, size_t bytes, int mem, cudaStream_t st) {
    if (!bytes) return;
    DX_REQUIRE(src != nullptr, DXPBD_ERR_ARG, "null input pointer");
    DX_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, mem == DXPBD_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
}
void download(void *dst, const void *src, size_t bytes, int mem, cudaStream_t st) {
    if (!bytes) return;
    DX_REQUIRE(dst != nullptr, DXPBD_ERR_ARG, "null output pointer");
    DX_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, mem == DXPBD_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, st));
    if (mem == DXPBD_MEM_HOST) DX_CHECK_CUDA(cudaStreamSynchronize(st));
}

void ensure_copy_pipe(dxpbd_scene *s) {
    if (s->cpy) return;
    DX_CHECK_CUDA(cudaStreamCreateWithFlags(&s->cpy, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
        DX_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_cp[k], cudaEventDisableTiming));
        DX_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_free[k], cudaEventDisableTiming));
        s->stage[k].alloc((size_t)3 * s->V);
    }
}

void apply_shape(dxpbd_scene *s, cudaStream_t st) {
    if (!s->NC) return;
    k_shape_apply<<<nblk(s->NC), kBlock, 0, st>>>(s->NSH, s->NCAP, s->NS, s->sph.p, s->cap_c.p, s->cap_a.p,
                                                  s->cap_r0.p, s->cap_L0.p, s->cap_Rb.p, s->cap_Lb.p, s->beta.p,
                                                  s->cols.p, s->csc.p);
    DX_CHECK_CUDA(cudaGetLastError());
}

inline double4 *state(dxpbd_scene *s, int n) { return s->ckpt.p + (size_t)n * s->V; }

// ------------------------------------------------------------------ wavefront plan (create time)
// Wave tile w = base tiles [w g, w g + g).  Neighbours: two wave tiles are neighbours when their
// items touch a common vertex (a tile's items touch its own vertices -- prediction -- and both
// endpoints of the constraints it owns).  Order pi: Cuthill-McKee BFS of the neighbour graph
// (restarted per component), L = 1 + max |pi(w) - pi(w')| over neighbours; tickets in the order of
// key = pi(w) + L p (wave.cuh: every dependency holds a smaller ticket).
void build_wave_plan(dxpbd_scene *s, const std::vector<int> &seg, const std::vector<int2> &ab, const float *xrest,
                     cudaStream_t st) {
    const int V = s->V, nt = s->ntiles, nc = s->n_dist_colors, g = std::max(1, s->wave_g);
    const int W = g * kTileV, ntw = (nt + g - 1) / g;
    constexpr int KIN = 6;
    std::vector<uint32_t> own((size_t)KIN * V);
    std::vector<uint8_t> cnt(V, 0);
    bool overflow = false;
    auto add = [&](int v, uint32_t w) {
        uint32_t *o = own.data() + (size_t)KIN * v;
        for (int k = 0; k < cnt[v]; ++k)
            if (o[k] == w) return;
        if (cnt[v] == KIN) { overflow = true; return; }
        o[cnt[v]++] = w;
    };
    for (int v = 0; v < V; ++v) add(v, (uint32_t)(v / W));
    for (size_t q = 0; q < ab.size(); ++q) {
        const uint32_t w = (uint32_t)(ab[q].x / W);
        add(ab[q].x, w);
        add(ab[q].y, w);
    }
    if (overflow) { s->wave_on = false; return; }   // very irregular meshes: per-color launches
    std::vector<std::vector<int>> nb(ntw);
    for (int w = 0; w < ntw; ++w) nb[w].push_back(w);
    for (int v = 0; v < V; ++v) {
        const uint32_t *o = own.data() + (size_t)KIN * v;
        for (int a = 0; a < cnt[v]; ++a)
            for (int b = 0; b < cnt[v]; ++b)
                if (a != b) nb[o[a]].push_back((int)o[b]);
    }
    std::vector<uint32_t>().swap(own);
    int maxn = 0;
    for (auto &l : nb) {
        std::sort(l.begin(), l.end());
        l.erase(std::unique(l.begin(), l.end()), l.end());
        maxn = std::max(maxn, (int)l.size());
    }
    // Two orders of the wave tiles, the one with the smaller bandwidth b is kept: (1) by centroid along
    // the longest bounding-box axis of the rest shape, in rows across the second-longest (sheets and
    // blocks), (2) Cuthill-McKee BFS.  The band of tiles live between a tile's first and last phase is
    // ~P b tiles, so b sets the L2 working set.
    auto bandwidth = [&](const std::vector<int> &pi) {
        int b = 0;
        for (int w = 0; w < ntw; ++w)
            for (int v : nb[w]) b = std::max(b, std::abs(pi[w] - pi[v]));
        return b;
    };
    std::vector<int> order_geo(ntw);
    {
        std::vector<double> cen((size_t)3 * ntw, 0.0);
        double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
        for (int v = 0; v < V; ++v) {
            const float *xr = xrest + (size_t)3 * s->vperm_h[v];
            for (int k = 0; k < 3; ++k) {
                cen[(size_t)3 * (v / W) + k] += xr[k];
                lo[k] = std::min(lo[k], (double)xr[k]);
                hi[k] = std::max(hi[k], (double)xr[k]);
            }
        }
        int ax[3] = {0, 1, 2};
        std::sort(ax, ax + 3, [&](int a, int b) { return hi[a] - lo[a] > hi[b] - lo[b]; });
        const double ext1 = std::max(hi[ax[1]] - lo[ax[1]], 1e-30), ext0 = std::max(hi[ax[0]] - lo[ax[0]], 1e-30);
        const double cell = std::sqrt(ext0 * ext1 / std::max(1, ntw));   // about one wave tile's extent
        std::vector<std::pair<long long, double>> key(ntw);
        for (int w = 0; w < ntw; ++w) {
            const int nv = std::min(V, (w + 1) * W) - w * W;
            const double c0 = cen[(size_t)3 * w + ax[0]] / nv, c1 = cen[(size_t)3 * w + ax[1]] / nv;
            key[w] = {(long long)std::floor((c1 - lo[ax[1]]) / cell), c0};
        }
        for (int w = 0; w < ntw; ++w) order_geo[w] = w;
        std::sort(order_geo.begin(), order_geo.end(), [&](int a, int b) { return key[a] < key[b] || (key[a] == key[b] && a < b); });
    }
    std::vector<int> order;
    order.reserve(ntw);
    std::vector<char> seen(ntw, 0);
    for (int r = 0; r < ntw; ++r) {
        if (seen[r]) continue;
        size_t head = order.size();
        order.push_back(r);
        seen[r] = 1;
        while (head < order.size()) {
            const int u = order[head++];
            std::vector<int> nx;
            for (int v : nb[u])
                if (!seen[v]) { seen[v] = 1; nx.push_back(v); }
            std::sort(nx.begin(), nx.end(), [&](int x, int y) { return nb[x].size() < nb[y].size() || (nb[x].size() == nb[y].size() && x < y); });
            order.insert(order.end(), nx.begin(), nx.end());
        }
    }
    std::vector<int> pi(ntw), pig(ntw);
    for (int k = 0; k < ntw; ++k) pi[order[k]] = k;
    for (int k = 0; k < ntw; ++k) pig[order_geo[k]] = k;
    int bw = bandwidth(pi);
    const int bwg = bandwidth(pig);
    if (bwg <= bw) { order.swap(order_geo); pi.swap(pig); bw = bwg; }
    const int P = 1 + nc;
    int L = 1 + bw;
    {   // + the in-flight window in keys (resident CTAs / items per key), so that a dependency is
        // normally finished when its dependant is dispatched
        int occ = 0, nsm = 0;
        DX_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_wave<2, 2, false, true>, kBlock, 0));
        DX_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device));
        L += s->wave_lag >= 0 ? s->wave_lag : (occ * nsm + P - 1) / P;
    }
    std::vector<int> off(ntw + 1, 0), flat;
    for (int w = 0; w < ntw; ++w) off[w + 1] = off[w] + (int)nb[w].size();
    flat.reserve(off[ntw]);
    for (auto &l : nb) flat.insert(flat.end(), l.begin(), l.end());
    std::vector<int4> items;
    std::vector<int2> nrange;
    items.reserve((size_t)ntw * P);
    nrange.reserve((size_t)ntw * P);
    for (int64_t key = 0; key < (int64_t)ntw + (int64_t)L * (P - 1); ++key)
        for (int p = P - 1; p >= 0; --p) {
            const int64_t k = key - (int64_t)L * p;
            if (k < 0 || k >= ntw) continue;
            const int w = order[k];
            int b = 0, c = 0;
            if (p > 0) {
                const int *sg = seg.data() + (size_t)(p - 1) * (nt + 1);
                b = sg[w * g];
                c = sg[std::min(nt, w * g + g)] - b;
            }
            items.push_back(make_int4(w, p, b, c));
            nrange.push_back(make_int2(off[w], off[w + 1]));
        }
    s->wave_ntw = ntw;
    s->wave_nitems = (int)items.size();
    s->wave_L = L;
    s->wave_maxnbr = maxn;
    s->wave_items.alloc(items.size());
    upload(s->wave_items.p, items.data(), sizeof(int4) * items.size(), DXPBD_MEM_HOST, st);
    s->wave_nrange.alloc(nrange.size());
    upload(s->wave_nrange.p, nrange.data(), sizeof(int2) * nrange.size(), DXPBD_MEM_HOST, st);
    s->wave_nbr.alloc(flat.size());
    upload(s->wave_nbr.p, flat.data(), sizeof(int) * flat.size(), DXPBD_MEM_HOST, st);
    s->wave_flags.alloc((size_t)2 * ntw);
    DX_CHECK_CUDA(cudaMemsetAsync(s->wave_flags.p, 0, sizeof(unsigned) * 2 * ntw, st));
    s->wave_ctr.alloc(2);
    DX_CHECK_CUDA(cudaMemsetAsync(s->wave_ctr.p, 0, sizeof(int) * 2, st));
    DX_CHECK_CUDA(cudaStreamSynchronize(st));
}

// One wavefront launch over the substep (k = 0: forward, 1: replay); REPLAY also stores the blocks.
template <bool REPLAY, bool WRITE_LAST_X>
void launch_wave(dxpbd_scene *s, int k, int grid, const WavePredict &pr, const WaveDist &dd, double4 *x, cudaStream_t st) {
    WavePlan w{s->wave_ntw, s->wave_g * kTileV, s->wave_nitems, s->wave_items.p, s->wave_nrange.p, s->wave_nbr.p,
               s->wave_flags.p + (size_t)k * s->wave_ntw, s->wave_ctr.p + k};
    DX_CHECK_CUDA(cudaMemsetAsync(s->wave_ctr.p + k, 0, sizeof(int), st));
    auto kern = k_wave<2, 2, REPLAY, WRITE_LAST_X>;
    if (grid < 0) grid = s->wave_nitems;
    if (grid == 0) {
        int occ = 0, nsm = 0;
        DX_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, kBlock, 0));
        DX_CHECK_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, s->device));
        grid = std::max(1, occ * nsm);
    }
    kern<<<std::min(grid, s->wave_nitems), kBlock, 0, st>>>(w, s->wave_base[k], s->V, s->n_dist_colors, pr, dd, x);
    DX_CHECK_CUDA(cudaGetLastError());
    s->wave_base[k] += (unsigned)(1 + s->n_dist_colors);
}

// Capture the launches `f(stream)` issues into an executable graph (kernel nodes keep the capture
// stream's priority: `lowest` for the replay, which runs on the low-priority stream).
template <class F>
cudaGraphExec_t capture_graph(dxpbd_scene *s, int prio, F f, int &launches) {   // prio -1 lowest, 0 default, 1 highest
    cudaStream_t &cs = prio < 0 ? s->cap_lo : (prio > 0 ? s->cap : s->cap_mid);
    if (!cs) {
        int least = 0, greatest = 0;
        DX_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
        DX_CHECK_CUDA(cudaStreamCreateWithPriority(&cs, cudaStreamNonBlocking, prio < 0 ? least : (prio > 0 ? greatest : 0)));
    }
    cudaGraph_t g = nullptr;
    DX_CHECK_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
    launches = f(cs);
    DX_CHECK_CUDA(cudaStreamEndCapture(cs, &g));
    cudaGraphExec_t e = nullptr;
    DX_CHECK_CUDA(cudaGraphInstantiate(&e, g, 0));
    DX_CHECK_CUDA(cudaGraphDestroy(g));
    return e;
}
inline bool sweep_graph_on(const dxpbd_scene *s) {
    return s->sweep_graph && !s->prof && s->iterations == 1 && s->V <= s->sweep_graph_maxv;
}

// ------------------------------------------------------------------ one forward substep
int forward_substep(dxpbd_scene *s, int n, cudaStream_t st) {
    const int V = s->V;
    const int frame = n / s->substeps;
    double4 *xo = state(s, n + 1);
    const float *f = s->have_forces ? s->forces.p + (size_t)frame * V * 3 : nullptr;
    const float inv_dt2 = s->inv_dt * s->inv_dt;
    const int K = s->iterations;
    int launches = 1;
    bool wave = s->wave_on && s->wave_fwd && s->wave_nitems > 0 && K == 1;
    const bool cached = s->qc_count && n >= s->qc_first;
    // sweep graph: iterate in the fixed buffer xw, copied to the checkpoint slot afterwards
    const bool graph = sweep_graph_on(s) && !wave && !cached;
    double4 *const xckpt = xo;
    if (graph) {
        if (s->xw.n < (size_t)V) s->xw.alloc(V);
        xo = s->xw.p;
    }
    if (wave) {
        // predict + every distance color in one time-skewed launch (wave.cuh); on cached substeps the
        // replay variant also stores Q_n (same iterates bit for bit)
        WavePredict pr{state(s, n), n > 0 ? state(s, n - 1) : nullptr, s->v0.p, f, s->dtd, 1.0 / s->dtd, s->gravity};
        if (cached) {
            float4 *slot = s->qcache.p + (size_t)(n - s->qc_first) * s->d_Qt.n;
            WaveDist dd{s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, s->E, slot, slot, nullptr, s->d_tpos.p, s->d_fpos.p};
            LAUNCH(DXPBD_K_DIST_PROJECT, (launch_wave<true, true>(s, 0, s->wave_grid_fwd, pr, dd, xo, st)));
        } else {
            WaveDist dd{s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, s->E, nullptr, nullptr, nullptr, nullptr, nullptr};
            LAUNCH(DXPBD_K_DIST_PROJECT, (launch_wave<false, true>(s, 0, s->wave_grid_fwd, pr, dd, xo, st)));
        }
    }
    const PredictArgs pa{state(s, n), n > 0 ? state(s, n - 1) : nullptr, s->v0.p, f, s->dtd, 1.0 / s->dtd, s->gravity};
    const bool fuse = s->fuse_predict && !wave && !graph && K == 1;
    if (fuse) {
        if (s->uncov.n) LAUNCH(DXPBD_K_PREDICT, k_predict_list<<<nblk((int)s->uncov.n), kBlock, 0, st>>>((int)s->uncov.n, s->uncov.p, pa, xo));
        else launches = 0;   // no prediction launch at all
    } else if (!wave) {
        LAUNCH(DXPBD_K_PREDICT, k_predict<<<nblk(V), kBlock, 0, st>>>(V, state(s, n), n > 0 ? state(s, n - 1) : nullptr, s->v0.p, f,
                                                                       s->dtd, 1.0 / s->dtd, s->gravity, xo));
    }
    auto sweep = [&](cudaStream_t st) -> int {
    int launches = 0;
    for (int k = 0; k < K; ++k) {
        const bool rd = k > 0, wr = k < K - 1;
        for (int c = 0; c < (wave ? 0 : s->n_dist_colors); ++c) {
            int b = s->dist_off[c], cnt = s->dist_off[c + 1] - b;
            if (!cnt) continue;
            if (fuse && c == 0 && s->qc_count && n >= s->qc_first) {
                float4 *slot = s->qcache.p + (size_t)(n - s->qc_first) * s->d_Qt.n;
                LAUNCH(DXPBD_K_DIST_PROJECT, (k_dist_first<true, 3><<<nblk(cnt), kBlock, 0, st>>>(
                    b, cnt, s->E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, pa, slot, nullptr, xo, s->d_tpos.p, s->d_fpos.p, slot)));
            } else if (fuse && c == 0) {
                LAUNCH(DXPBD_K_DIST_PROJECT, (k_dist_first<false, 4><<<nblk(cnt), kBlock, 0, st>>>(
                    b, cnt, s->E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, pa, nullptr, nullptr, xo, nullptr, nullptr, nullptr)));
            } else if (!rd && !wr && s->qc_count && n >= s->qc_first) {
                // cached substep: the replay kernel (same iterates bit for bit) also stores Q_n
                float4 *slot = s->qcache.p + (size_t)(n - s->qc_first) * s->d_Qt.n;
                LAUNCH(DXPBD_K_DIST_PROJECT, (k_dist_replay1<2, 3><<<nblk((cnt + 1) / 2), kBlock, 0, st>>>(
                    b, cnt, s->E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, slot, nullptr, xo, s->d_tpos.p, s->d_fpos.p, slot)));
            } else if (!rd && !wr && s->nb == 2)
                LAUNCH(DXPBD_K_DIST_PROJECT, k_dist_project1<2><<<nblk((cnt + 1) / 2), kBlock, 0, st>>>(b, cnt, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, xo));
            else if (!rd && !wr)
                LAUNCH(DXPBD_K_DIST_PROJECT, k_dist_project1<1><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, xo));
            else if (!rd && wr)
                LAUNCH(DXPBD_K_DIST_PROJECT, k_dist_project<false, true><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, s->lam_d.p, xo));
            else if (rd && wr)
                LAUNCH(DXPBD_K_DIST_PROJECT, k_dist_project<true, true><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, s->lam_d.p, xo));
            else
                LAUNCH(DXPBD_K_DIST_PROJECT, k_dist_project<true, false><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, s->lam_d.p, xo));
            ++launches;
        }
        for (int c = 0; c < s->n_tet_colors; ++c) {
            int b = s->tet_off[c], cnt = s->tet_off[c + 1] - b;
            if (!cnt) continue;
            const int tb = (cnt + 127) / 128;
            if (!rd && !wr) LAUNCH(DXPBD_K_TET_PROJECT, k_tet_project<false, false><<<tb, 128, 0, st>>>(b, cnt, s->tdev(), s->inv_dt2d, s->lam_t.p, xo));
            else if (!rd && wr) LAUNCH(DXPBD_K_TET_PROJECT, k_tet_project<false, true><<<tb, 128, 0, st>>>(b, cnt, s->tdev(), s->inv_dt2d, s->lam_t.p, xo));
            else if (rd && wr) LAUNCH(DXPBD_K_TET_PROJECT, k_tet_project<true, true><<<tb, 128, 0, st>>>(b, cnt, s->tdev(), s->inv_dt2d, s->lam_t.p, xo));
            else LAUNCH(DXPBD_K_TET_PROJECT, k_tet_project<true, false><<<tb, 128, 0, st>>>(b, cnt, s->tdev(), s->inv_dt2d, s->lam_t.p, xo));
            ++launches;
        }
        if (s->NC && !rd && !wr && s->qc_count && n >= s->qc_first) {
            // cached substep: the replay kernel (same iterate) also stores the contact blocks and controls
            float at = s->coll_alpha * inv_dt2;
            float *slot = s->qccache.p + (size_t)(n - s->qc_first) * s->qc_cper;
            float *eo = s->qc_cper > (size_t)6 * V ? slot + (size_t)6 * V : nullptr;
            ContactScratch cs{s->cc_lam.p, s->cc_T.p, s->cc_sig.p, s->cc_B.p, s->cc_e.p};
            LAUNCH(DXPBD_K_CONTACT_PROJECT, k_contact_replay<true, true><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, cs, s->pd,
                                                                                                   slot, eo, xo, s->vsc.p));
            ++launches;
        } else if (s->NC) {
            float at = s->coll_alpha * inv_dt2;
            if (!rd && !wr) LAUNCH(DXPBD_K_CONTACT_PROJECT, k_contact_project<false, false><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, s->lam_c.p, xo, s->vsc.p));
            else if (!rd && wr) LAUNCH(DXPBD_K_CONTACT_PROJECT, k_contact_project<false, true><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, s->lam_c.p, xo, s->vsc.p));
            else if (rd && wr) LAUNCH(DXPBD_K_CONTACT_PROJECT, k_contact_project<true, true><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, s->lam_c.p, xo, s->vsc.p));
            else LAUNCH(DXPBD_K_CONTACT_PROJECT, k_contact_project<true, false><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, s->lam_c.p, xo, s->vsc.p));
            ++launches;
        }
    }
    return launches;
    };
    if (graph) {
        if (!s->g_fwd) s->g_fwd = capture_graph(s, 0, sweep, s->g_fwd_launches);
        DX_CHECK_CUDA(cudaGraphLaunch(s->g_fwd, st));
        DX_CHECK_CUDA(cudaMemcpyAsync(xckpt, xo, sizeof(double4) * V, cudaMemcpyDeviceToDevice, st));
        launches += s->g_fwd_launches;
    } else {
        launches += sweep(st);
    }
    DX_CHECK_CUDA(cudaGetLastError());
    return launches;
}

// ------------------------------------------------------------------ replay of substep n
// stage 0: the whole replay; 1: everything but the tets' PD projection; 2: the tets' PD projection only
// (K = 1 tet scenes: the two halves run on two streams)
int replay_substep(dxpbd_scene *s, int n, cudaStream_t st, int stage = 0) {
    const int V = s->V, E = s->E;
    float4 *qtw = s->qt_write ? s->qt_write : s->d_Qt.p;   // TMA-layout block buffer written
    const bool lay = s->use_tma && s->qf == 0;              // general blocks into the TMA layout
    const int frame = n / s->substeps;
    const float *f = s->have_forces ? s->forces.p + (size_t)frame * V * 3 : nullptr;
    double4 *x = s->xr.p;
    int launches = 1;
    const float inv_dt2 = s->inv_dt * s->inv_dt;
    const int K = s->iterations;
    const bool want_e = (s->grad_flags >> DXPBD_GRAD_COMPLIANCE) & 1;
    const bool wave = s->wave_on && s->wave_rep && s->wave_nitems > 0 && K == 1 && s->qf == 1;
    auto tet_psd = [&](cudaStream_t st) {
        float *const tQ = s->tq_w ? s->tq_w : s->t_Q.p;
        if (s->psd_minb == 3)
            LAUNCH(DXPBD_K_TET_REPLAY, k_tet_psd<3><<<(s->T + 127) / 128, 128, 0, st>>>(s->T, tQ, s->psd_tol, s->psd_sweeps));
        else if (s->psd_minb == 4)
            LAUNCH(DXPBD_K_TET_REPLAY, k_tet_psd<4><<<(s->T + 127) / 128, 128, 0, st>>>(s->T, tQ, s->psd_tol, s->psd_sweeps));
        else
            LAUNCH(DXPBD_K_TET_REPLAY, k_tet_psd<1><<<(s->T + 127) / 128, 128, 0, st>>>(s->T, tQ, s->psd_tol, s->psd_sweeps));
    };
    if (stage == 2) {
        tet_psd(st);
        DX_CHECK_CUDA(cudaGetLastError());
        return 1;
    }
    if (wave) {
        WavePredict pr{state(s, n), n > 0 ? state(s, n - 1) : nullptr, s->v0.p, f, s->dtd, 1.0 / s->dtd, s->gravity};
        float4 *Q = s->use_tma ? qtw : reinterpret_cast<float4 *>(s->Qd.p);
        WaveDist dd{s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, E, Q, qtw, want_e ? s->ed.p : nullptr,
                    s->use_tma ? s->d_tpos.p : nullptr, s->use_tma ? s->d_fpos.p : nullptr};
        if (!s->T && !s->NC)
            LAUNCH(DXPBD_K_DIST_REPLAY, (launch_wave<true, false>(s, 1, s->wave_grid_rep, pr, dd, x, st)));
        else
            LAUNCH(DXPBD_K_DIST_REPLAY, (launch_wave<true, true>(s, 1, s->wave_grid_rep, pr, dd, x, st)));
    }
    const PredictArgs pa{state(s, n), n > 0 ? state(s, n - 1) : nullptr, s->v0.p, f, s->dtd, 1.0 / s->dtd, s->gravity};
    const bool fuse = s->fuse_predict && !wave && !sweep_graph_on(s) && K == 1 && s->qf == 1;
    if (fuse) {
        if (s->uncov.n) LAUNCH(DXPBD_K_PREDICT, k_predict_list<<<nblk((int)s->uncov.n), kBlock, 0, st>>>((int)s->uncov.n, s->uncov.p, pa, x));
        else launches = 0;   // no prediction launch at all
    } else if (!wave) {
        LAUNCH(DXPBD_K_PREDICT, k_predict<<<nblk(V), kBlock, 0, st>>>(V, state(s, n), n > 0 ? state(s, n - 1) : nullptr, s->v0.p, f,
                                                                       s->dtd, 1.0 / s->dtd, s->gravity, x));
    }
    DistScratch ds{s->sc_lam.p, s->sc_sig.p, s->sc_B.p, s->sc_T.p, s->sc_e.p};
    ContactScratch cs{s->cc_lam.p, s->cc_T.p, s->cc_sig.p, s->cc_B.p, s->cc_e.p};
    const bool want_ce = (s->grad_flags & ((1u << DXPBD_GRAD_SHAPE) | (1u << DXPBD_GRAD_SPHERE))) != 0;
    auto sweep = [&](cudaStream_t st) -> int {
    int launches = 0;
    for (int k = 0; k < K; ++k) {
        const bool first = k == 0, last = k == K - 1;
        for (int c = 0; c < (wave ? 0 : s->n_dist_colors); ++c) {
            int b = s->dist_off[c], cnt = s->dist_off[c + 1] - b;
            if (!cnt) continue;
            float *eo = want_e ? s->ed.p : nullptr;
            const bool last_color = c == s->n_dist_colors - 1 && !s->T && !s->NC;   // nothing reads its iterate
            if (fuse && c == 0)
                LAUNCH(DXPBD_K_DIST_REPLAY, (k_dist_first<true, 3><<<nblk(cnt), kBlock, 0, st>>>(
                    b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, pa,
                    s->use_tma ? qtw : reinterpret_cast<float4 *>(s->Qd.p), eo, x,
                    s->use_tma ? s->d_tpos.p : nullptr, s->use_tma ? s->d_fpos.p : nullptr, qtw)));
            else if (first && last && s->qf == 1 && s->nb_rep == 2 && s->rep_minb == 3 && last_color)
                LAUNCH(DXPBD_K_DIST_REPLAY, (k_dist_replay1<2, 3, false><<<nblk((cnt + 1) / 2), kBlock, 0, st>>>(
                    b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2,
                    s->use_tma ? qtw : reinterpret_cast<float4 *>(s->Qd.p), eo, x,
                    s->use_tma ? s->d_tpos.p : nullptr, s->use_tma ? s->d_fpos.p : nullptr, qtw)));
            else if (first && last && s->qf == 1 && s->nb_rep == 2 && s->rep_minb == 3)
                LAUNCH(DXPBD_K_DIST_REPLAY, (k_dist_replay1<2, 3><<<nblk((cnt + 1) / 2), kBlock, 0, st>>>(
                    b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2,
                    s->use_tma ? qtw : reinterpret_cast<float4 *>(s->Qd.p), eo, x,
                    s->use_tma ? s->d_tpos.p : nullptr, s->use_tma ? s->d_fpos.p : nullptr, qtw)));
            else if (first && last && s->qf == 1 && s->nb_rep == 2 && s->rep_minb == 4)
                LAUNCH(DXPBD_K_DIST_REPLAY, (k_dist_replay1<2, 4><<<nblk((cnt + 1) / 2), kBlock, 0, st>>>(
                    b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2,
                    s->use_tma ? qtw : reinterpret_cast<float4 *>(s->Qd.p), eo, x,
                    s->use_tma ? s->d_tpos.p : nullptr, s->use_tma ? s->d_fpos.p : nullptr, qtw)));
            else if (first && last && s->qf == 1 && s->nb_rep == 2)
                LAUNCH(DXPBD_K_DIST_REPLAY, k_dist_replay1<2><<<nblk((cnt + 1) / 2), kBlock, 0, st>>>(
                    b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2,
                    s->use_tma ? qtw : reinterpret_cast<float4 *>(s->Qd.p), eo, x,
                    s->use_tma ? s->d_tpos.p : nullptr, s->use_tma ? s->d_fpos.p : nullptr, qtw));
            else if (first && last && s->qf == 1)
                LAUNCH(DXPBD_K_DIST_REPLAY, k_dist_replay1<1><<<nblk(cnt), kBlock, 0, st>>>(
                    b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2,
                    s->use_tma ? qtw : reinterpret_cast<float4 *>(s->Qd.p), eo, x,
                    s->use_tma ? s->d_tpos.p : nullptr, s->use_tma ? s->d_fpos.p : nullptr, qtw));
            else if (first && last)
                LAUNCH(DXPBD_K_DIST_REPLAY, k_dist_replay<true, true><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, ds, s->pd, s->Qd.p, eo, x,
                                                                                       lay ? s->d_fpos.p : nullptr, lay ? s->d_Qt.p : nullptr,
                                                                                       lay ? s->d_tpos.p : nullptr, lay ? s->d_Qt2b.p : nullptr));
            else if (first)
                LAUNCH(DXPBD_K_DIST_REPLAY, k_dist_replay<true, false><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, ds, s->pd, s->Qd.p, eo, x,
                                                                                       lay ? s->d_fpos.p : nullptr, lay ? s->d_Qt.p : nullptr,
                                                                                       lay ? s->d_tpos.p : nullptr, lay ? s->d_Qt2b.p : nullptr));
            else if (last)
                LAUNCH(DXPBD_K_DIST_REPLAY, k_dist_replay<false, true><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, ds, s->pd, s->Qd.p, eo, x,
                                                                                       lay ? s->d_fpos.p : nullptr, lay ? s->d_Qt.p : nullptr,
                                                                                       lay ? s->d_tpos.p : nullptr, lay ? s->d_Qt2b.p : nullptr));
            else
                LAUNCH(DXPBD_K_DIST_REPLAY, k_dist_replay<false, false><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, ds, s->pd, s->Qd.p, eo, x,
                                                                                       lay ? s->d_fpos.p : nullptr, lay ? s->d_Qt.p : nullptr,
                                                                                       lay ? s->d_tpos.p : nullptr, lay ? s->d_Qt2b.p : nullptr));
            ++launches;
        }
        if (s->T) {
            TetScratch tsc{s->ts_lam.p, s->ts_S.p, s->ts_Dt.p, s->ts_Tu.p, s->ts_e.p};
            float *const tQ = s->tq_w ? s->tq_w : s->t_Q.p;   // this replay's block buffer
            float *teo = ((s->grad_flags >> DXPBD_GRAD_MATERIAL) & 1) ? (s->te_w ? s->te_w : s->t_e.p) : nullptr;
            for (int c = 0; c < s->n_tet_colors; ++c) {
                int b = s->tet_off[c], cnt = s->tet_off[c + 1] - b;
                if (!cnt) continue;
                const int tb = (cnt + 127) / 128;
                if (first && last)   // K = 1: iterate only, derivative blocks of all tets after the colors
                    LAUNCH(DXPBD_K_TET_REPLAY, (k_tet_replay<true, true, 1><<<tb, 128, 0, st>>>(b, cnt, s->tdev(), s->inv_dt2d, tsc, s->pd, tQ, teo, x,
                                                                                               s->t_xsave.p)));
                else if (first) LAUNCH(DXPBD_K_TET_REPLAY, k_tet_replay<true, false><<<tb, 128, 0, st>>>(b, cnt, s->tdev(), s->inv_dt2d, tsc, s->pd, tQ, teo, x));
                else if (last) LAUNCH(DXPBD_K_TET_REPLAY, k_tet_replay<false, true><<<tb, 128, 0, st>>>(b, cnt, s->tdev(), s->inv_dt2d, tsc, s->pd, tQ, teo, x));
                else LAUNCH(DXPBD_K_TET_REPLAY, k_tet_replay<false, false><<<tb, 128, 0, st>>>(b, cnt, s->tdev(), s->inv_dt2d, tsc, s->pd, tQ, teo, x));
                ++launches;
            }
            if (first && last) {
                LAUNCH(DXPBD_K_TET_REPLAY, (k_tet_replay<true, true, 2><<<(s->T + 127) / 128, 128, 0, st>>>(
                                               0, s->T, s->tdev(), s->inv_dt2d, tsc, s->pd, tQ, teo, x, s->t_xsave.p)));
                ++launches;
                if (s->pd && stage == 0) {
                    tet_psd(st);
                    ++launches;
                }
            }
        }
        if (s->NC) {
            float at = s->coll_alpha * inv_dt2;
            float *eo = want_ce ? (s->ec_w ? s->ec_w : s->ec.p) : nullptr;
            float *const Qcw = s->qc_w ? s->qc_w : s->Qc.p;
            if (first && last) LAUNCH(DXPBD_K_CONTACT_REPLAY, k_contact_replay<true, true><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, cs, s->pd, Qcw, eo, x, s->vsc.p));
            else if (first) LAUNCH(DXPBD_K_CONTACT_REPLAY, k_contact_replay<true, false><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, cs, s->pd, Qcw, eo, x, s->vsc.p));
            else if (last) LAUNCH(DXPBD_K_CONTACT_REPLAY, k_contact_replay<false, true><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, cs, s->pd, Qcw, eo, x, s->vsc.p));
            else LAUNCH(DXPBD_K_CONTACT_REPLAY, k_contact_replay<false, false><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, cs, s->pd, Qcw, eo, x, s->vsc.p));
            ++launches;
        }
    }
    return launches;
    };
    if (sweep_graph_on(s) && !wave) {
        // graph per set of output buffers (they alternate with the replay / PCG overlap)
        const bool g_mat = ((s->grad_flags >> DXPBD_GRAD_MATERIAL) & 1) != 0;
        std::vector<const void *> key = {qtw, s->tq_w ? s->tq_w : s->t_Q.p, g_mat ? (s->te_w ? s->te_w : s->t_e.p) : nullptr,
                                         s->qc_w ? s->qc_w : s->Qc.p, want_ce ? (s->ec_w ? s->ec_w : s->ec.p) : nullptr,
                                         want_e ? s->ed.p : nullptr, s->Qd.p, reinterpret_cast<const void *>((size_t)stage)};
        const dxpbd_scene::RepGraph *rg = nullptr;
        for (auto &kv : s->g_rep)
            if (kv.key == key) rg = &kv;
        if (!rg) {
            int nl = 0;
            cudaGraphExec_t e = capture_graph(s, (st == s->aux || st == s->aux2) ? -1 : 0, sweep, nl);
            s->g_rep.push_back({key, e, nl});
            rg = &s->g_rep.back();
        }
        DX_CHECK_CUDA(cudaGraphLaunch(rg->e, st));
        launches += rg->launches;
    } else {
        launches += sweep(st);
    }
    DX_CHECK_CUDA(cudaGetLastError());
    return launches;
}

// internal fp64 state -> user-order [V][3] float (host or device)
void positions_from(dxpbd_scene *s, const double4 *x, float *out, int mem, cudaStream_t st) {
    if (mem == DXPBD_MEM_HOST) {
        k_unpack3<<<nblk(s->V), kBlock, 0, st>>>(s->V, x, s->vperm.p, s->tmp3.p);
        download(out, s->tmp3.p, sizeof(float) * s->V * 3, mem, st);
    } else {
        k_unpack3<<<nblk(s->V), kBlock, 0, st>>>(s->V, x, s->vperm.p, out);
    }
    DX_CHECK_CUDA(cudaGetLastError());
}

// x0, v0, forces (user order, host or device) -> internal order: state 0, v0, per-frame forces
void forward_inputs(dxpbd_scene *s, const float *x0, const float *v0, const float *forces, int num_frames, int mem,
                    cudaStream_t st, bool defer_host_forces = false) {
    const int V = s->V;
    // user vertex order -> internal (Morton) order at the boundary
    const float *src = x0;
    if (mem == DXPBD_MEM_HOST) { upload(s->tmp3.p, x0, sizeof(float) * V * 3, mem, st); src = s->tmp3.p; }
    k_pack4d<<<nblk(V), kBlock, 0, st>>>(V, src, s->vperm.p, s->inv_mass.p, state(s, 0));
    src = v0;
    if (mem == DXPBD_MEM_HOST) { upload(s->tmp3.p, v0, sizeof(float) * V * 3, mem, st); src = s->tmp3.p; }
    k_pack4g<<<nblk(V), kBlock, 0, st>>>(V, src, s->vperm.p, s->v0.p);
    s->have_forces = forces != nullptr;
    if (forces) {
        if (s->forces.n < (size_t)s->max_frames * V * 3) s->forces.alloc((size_t)s->max_frames * V * 3);
        if (mem == DXPBD_MEM_HOST && defer_host_forces) {
            // per frame, overlapped with the forward (dxpbd_forward: upload_frame_forces)
        } else if (mem == DXPBD_MEM_HOST) {
            for (int f = 0; f < num_frames; ++f) {
                upload(s->tmp3.p, forces + (size_t)f * V * 3, sizeof(float) * V * 3, mem, st);
                k_gather3<<<nblk(V), kBlock, 0, st>>>(V, 1, s->tmp3.p, s->vperm.p, s->forces.p + (size_t)f * V * 3);
            }
        } else {
            k_gather3<<<nblk((int64_t)V * num_frames), kBlock, 0, st>>>(V, num_frames, forces, s->vperm.p, s->forces.p);
        }
    }
}

// Host forces of frame f: H2D into a staging slot on the copy stream (overlapping the substeps of
// earlier frames), then the gather into internal order on the compute stream.
void upload_frame_forces(dxpbd_scene *s, const float *forces, int f, cudaStream_t st) {
    const int V = s->V, k = f & 1;
    ensure_copy_pipe(s);
    DX_CHECK_CUDA(cudaStreamWaitEvent(s->cpy, s->ev_free[k], 0));   // the gather of frame f - 2 consumed the slot
    DX_CHECK_CUDA(cudaMemcpyAsync(s->stage[k].p, forces + (size_t)f * V * 3, sizeof(float) * V * 3, cudaMemcpyHostToDevice, s->cpy));
    DX_CHECK_CUDA(cudaEventRecord(s->ev_cp[k], s->cpy));
    DX_CHECK_CUDA(cudaStreamWaitEvent(st, s->ev_cp[k], 0));
    k_gather3<<<nblk(V), kBlock, 0, st>>>(V, 1, s->stage[k].p, s->vperm.p, s->forces.p + (size_t)f * V * 3);
    DX_CHECK_CUDA(cudaEventRecord(s->ev_free[k], st));
}

// Force gradients of frame f (final once the backward has passed the frame's first substep) to the
// output registered with dxpbd_grads_stream: scatter to user order into a staging slot, D2H on the
// copy stream while the backward continues.
void stream_frame_grads(dxpbd_scene *s, int f, cudaStream_t st) {
    const int V = s->V, k = f & 1;
    float *dst = s->gs_out + (size_t)f * V * 3;
    if (s->gs_mem != DXPBD_MEM_HOST) {
        k_scatter3<<<nblk(V), kBlock, 0, st>>>(V, 1, s->g_force.p + (size_t)f * V * 3, s->vperm.p, dst);
        return;
    }
    ensure_copy_pipe(s);
    DX_CHECK_CUDA(cudaStreamWaitEvent(st, s->ev_free[k], 0));   // the D2H of frame f + 2 released the slot
    k_scatter3<<<nblk(V), kBlock, 0, st>>>(V, 1, s->g_force.p + (size_t)f * V * 3, s->vperm.p, s->stage[k].p);
    DX_CHECK_CUDA(cudaEventRecord(s->ev_cp[k], st));
    DX_CHECK_CUDA(cudaStreamWaitEvent(s->cpy, s->ev_cp[k], 0));
    DX_CHECK_CUDA(cudaMemcpyAsync(dst, s->stage[k].p, sizeof(float) * V * 3, cudaMemcpyDeviceToHost, s->cpy));
    DX_CHECK_CUDA(cudaEventRecord(s->ev_free[k], s->cpy));
}

struct BwdSetup {
    const float *wts = nullptr;
    std::vector<int> key_of;   // state index -> keyframe slot
    bool g_comp = false, g_forces = false, g_coll = false, warm2 = false;
    int last_key_state = -1;
};

// Buffers, targets / weights (internal order), zeroed accumulators and adjoint state of a backward.
BwdSetup backward_prepare(dxpbd_scene *s, int num_keys, const int32_t *key_frames, const float *targets,
                          const float *weights, int mem, cudaStream_t st) {
    const int V = s->V, E = s->E, sub = s->substeps;
    const int N = s->frames_done * sub;
    BwdSetup su;
    // buffers
    if (s->xr.n < (size_t)V) s->xr.alloc(V);
    auto ensure4 = [&](DBuf<float3> &b) { if (b.n < (size_t)V) b.alloc(V); };
    ensure4(s->ax); ensure4(s->rhs); ensure4(s->y); ensure4(s->r); ensure4(s->p); ensure4(s->q); ensure4(s->p1);
    ensure4(s->uprev); ensure4(s->u0);
    if (s->warm_order == 2 && s->use_tma) ensure4(s->uprev2);
    const bool warm2 = su.warm2 = s->warm_order == 2 && s->use_tma;
    if (E && !s->use_tma && s->Qd.n < (size_t)6 * E) s->Qd.alloc((size_t)6 * E);   // TMA path: blocks in d_Qt
    const bool g_comp = su.g_comp = (s->grad_flags >> DXPBD_GRAD_COMPLIANCE) & 1;
    const bool g_forces = su.g_forces = (s->grad_flags >> DXPBD_GRAD_FORCES) & 1;
    const bool g_coll = su.g_coll = (s->grad_flags & ((1u << DXPBD_GRAD_SHAPE) | (1u << DXPBD_GRAD_SPHERE))) != 0;
    if (E && g_comp && s->ed.n < (size_t)3 * E) s->ed.alloc((size_t)3 * E);
    if (E && s->iterations > 1 && s->sc_lam.n < (size_t)E) {
        s->sc_lam.alloc(E); s->sc_sig.alloc((size_t)3 * E); s->sc_B.alloc((size_t)6 * E); s->sc_T.alloc(E); s->sc_e.alloc((size_t)3 * E);
    }
    if (s->NC) {
        const size_t NV = (size_t)s->NC * V;
        if (s->Qc.n < (size_t)6 * V) s->Qc.alloc((size_t)6 * V);
        if (g_coll && s->ec.n < 12 * NV) s->ec.alloc(12 * NV);
        if (s->iterations > 1 && s->cc_lam.n < NV) {
            s->cc_lam.alloc(NV); s->cc_T.alloc(4 * NV); s->cc_sig.alloc(3 * NV); s->cc_B.alloc(6 * NV); s->cc_e.alloc(12 * NV);
        }
    }
    if (s->cg_sc.n < (size_t)(s->cg_max_iter + 2) * 4) s->cg_sc.alloc((size_t)(s->cg_max_iter + 2) * 4);
    const size_t nacc = 1 + 4 * (size_t)std::max(s->NC, 1);
    if (s->acc.n < nacc) s->acc.alloc(nacc);
    if (s->T) {
        const size_t T = s->T;
        if (s->t_Q.n < 45 * T) s->t_Q.alloc(45 * T);
        if (((s->grad_flags >> DXPBD_GRAD_MATERIAL) & 1) && s->t_e.n < 18 * T) s->t_e.alloc(18 * T);
        if (s->t_g.n < 2 * T) s->t_g.alloc(2 * T);
        if (s->iterations == 1 && s->t_xsave.n < 4 * T) s->t_xsave.alloc(4 * T);
        if (s->iterations > 1 && s->ts_lam.n < 2 * T) {
            s->ts_lam.alloc(2 * T); s->ts_S.alloc(18 * T); s->ts_Dt.alloc(45 * T); s->ts_Tu.alloc(4 * T); s->ts_e.alloc(18 * T);
        }
    }
    // targets
    if (num_keys) {
        if (s->targets.n < (size_t)num_keys * V * 3) s->targets.alloc((size_t)num_keys * V * 3);
        for (int k = 0; k < num_keys; ++k) {
            const float *src = targets + (size_t)k * V * 3;
            if (mem == DXPBD_MEM_HOST) { upload(s->tmp3.p, src, sizeof(float) * V * 3, mem, st); src = s->tmp3.p; }
            k_gather3<<<nblk(V), kBlock, 0, st>>>(V, 1, src, s->vperm.p, s->targets.p + (size_t)k * V * 3);
        }
    }
    if (weights) {
        if (s->weights.n < (size_t)V) s->weights.alloc(V);
        const float *src = weights;
        if (mem == DXPBD_MEM_HOST) { upload(s->tmp3.p, weights, sizeof(float) * V, mem, st); src = s->tmp3.p; }
        k_gather1<<<nblk(V), kBlock, 0, st>>>(V, src, s->vperm.p, s->weights.p);
        su.wts = s->weights.p;
    }
    // gradient accumulators
    if (g_comp && E) { if (s->g_comp.n < (size_t)E) s->g_comp.alloc(E); DX_CHECK_CUDA(cudaMemsetAsync(s->g_comp.p, 0, sizeof(float) * E, st)); }
    if (g_forces) {
        size_t nf = (size_t)std::max(s->frames_done, 1) * V * 3;
        if (s->g_force.n < nf) s->g_force.alloc(nf);
        DX_CHECK_CUDA(cudaMemsetAsync(s->g_force.p, 0, sizeof(float) * nf, st));
    }
    DX_CHECK_CUDA(cudaMemsetAsync(s->acc.p, 0, sizeof(double) * nacc, st));
    if (s->T) DX_CHECK_CUDA(cudaMemsetAsync(s->t_g.p, 0, sizeof(float) * 2 * s->T, st));
    // state index -> keyframe slot
    su.key_of.assign(N + 1, -1);
    for (int k = 0; k < num_keys; ++k) su.key_of[key_frames[k] * sub] = k;   // duplicates: last wins
    // increment-form adjoint (kernels.cuh "adjoint"): y = u = 0 beyond the horizon
    DX_CHECK_CUDA(cudaMemsetAsync(s->y.p, 0, sizeof(float3) * V, st));
    DX_CHECK_CUDA(cudaMemsetAsync(s->ax.p, 0, sizeof(float3) * V, st));   // ax holds u
    DX_CHECK_CUDA(cudaMemsetAsync(s->uprev.p, 0, sizeof(float3) * V, st));
    if (warm2) DX_CHECK_CUDA(cudaMemsetAsync(s->uprev2.p, 0, sizeof(float3) * V, st));
    for (int n = 0; n <= N; ++n) if (su.key_of[n] >= 0) su.last_key_state = n;
    (void)g_comp; (void)g_forces; (void)g_coll;
    return su;
}

// ------------------------------------------------------------------ filtered PCG
int pcg_solve(dxpbd_scene *s, cudaStream_t st, int &iters_out, double &relres_out, bool started) {
    // warm-started PCG: s->ax holds u_{n+1} (initial guess), s->r the residual r0 and s->rhs the
    // system right-hand side b (both from the rhs kernel); cg_sc was zeroed before the rhs kernel.
    const int V = s->V, E = s->E;
    const int maxit = s->cg_max_iter;
    CGState cs{s->cg_sc.p, s->cg_sc.p + (size_t)(maxit + 1) * 4, s->cg_tol * s->cg_tol};
    const float *xw = s->inv_mass.p;
    const float *Qc = s->NC ? (s->qc_r ? s->qc_r : s->Qc.p) : nullptr;
    CGBufs bufs{s->ax.p, s->r.p, s->p.p, s->p1.p, s->q.p, nullptr};
    TileLists tl{s->n_dist_colors, s->ntiles, s->d_seg.p, s->d_fseg.p, s->d_fidx.p, s->d_fent.p};
    TmaTiles tt = s->tma_tiles();
    const bool defer = s->use_tma && s->defer_u;   // u update deferred into the next matvec
    // no distance constraints (tets and contacts only): tet + vertex matvec in one launch, q folded
    // into the update (tet_kernels.cuh k_cg_tetv)
    const bool tetv = s->T && E == 0 && !s->use_tma && s->tetv;
    const float *const tQr = s->tq_r ? s->tq_r : s->t_Q.p;   // tet blocks of this substep
    const int nbt = tetv ? nblk(s->T) : 0;
    if (!started)   // else fused into the rhs kernel
        LAUNCH(DXPBD_K_CG_INIT, k_cg_start<<<nblk(V), kBlock, 0, st>>>(V, s->rhs.p, s->r.p, s->p.p, xw, cs));
    int launches = 1;
    int it = 0;
    // one PCG iteration (it >= 0, or it = -1 with the graph-mode state: counter and pointers on the device)
    auto iteration = [&](int it, cudaStream_t st, const CGState &cs) -> int {
        if (tetv) {
            if (s->tetv_minb == 3)
                LAUNCH(DXPBD_K_CG_TET, k_cg_tetv<3><<<nbt + nblk(V), kBlock, 0, st>>>(it, nbt, V, s->tdev(), tQr, bufs,
                                                                                     xw, Qc, cs));
            else
                LAUNCH(DXPBD_K_CG_TET, k_cg_tetv<1><<<nbt + nblk(V), kBlock, 0, st>>>(it, nbt, V, s->tdev(), tQr, bufs,
                                                                                     xw, Qc, cs));
            LAUNCH(DXPBD_K_CG_UPDATE, k_cg_update_tet<<<nblk(V), kBlock, 0, st>>>(V, it, bufs, xw, Qc, cs, s->tdev()));
            return 2;
        }
        int n = 0;
        if (s->pull) {
            const PullTiles pt = s->pull_tiles();
            float3 *uf = defer ? s->ax.p : nullptr;
            if (s->pull_persist)
                LAUNCH(DXPBD_K_CG_DIST, (k_cg_matvec_pull_p<<<std::min(s->ntiles, 2 * s->num_sms), kTileV, s->pull_psmem, st>>>(it, pt, V, Qc, bufs, xw, cs, 0, s->ntiles, uf)));
            else
                LAUNCH(DXPBD_K_CG_DIST, (k_cg_matvec_pull<<<s->ntiles, kTileV, s->pull_smem, st>>>(it, pt, V, Qc, bufs, xw, cs, 0, uf)));
        } else if (s->use_tma) {
            LAUNCH(DXPBD_K_CG_DIST, (k_cg_matvec_tma<kMvThreads, kMvMinB><<<s->ntiles, kMvThreads, s->tma_smem, st>>>(it, tt, V, Qc, bufs, xw, cs, 0,
                                                                                                     defer ? s->ax.p : nullptr)));
        } else if (s->qf == 1)
            LAUNCH(DXPBD_K_CG_DIST, k_cg_matvec<1><<<s->ntiles, kBlock, 0, st>>>(it, tl, V, s->d_idx.p, s->Qd.p, E, Qc, bufs, xw, cs));
        else
            LAUNCH(DXPBD_K_CG_DIST, k_cg_matvec<0><<<s->ntiles, kBlock, 0, st>>>(it, tl, V, s->d_idx.p, s->Qd.p, E, Qc, bufs, xw, cs));
        ++n;
        if (s->T) {
            LAUNCH(DXPBD_K_CG_TET, k_cg_tet<<<nblk(s->T), kBlock, 0, st>>>(it, s->tdev(), tQr, bufs, xw, cs));
            LAUNCH(DXPBD_K_CG_TET, k_fold_q4<<<nblk(V), kBlock, 0, st>>>(V, it, bufs, s->tdev(), cs));
            n += 2;
        }
        if (defer)
            LAUNCH(DXPBD_K_CG_UPDATE, k_cg_update4<false><<<nblk(V / 4 + 1), kBlock, 0, st>>>(V, it, bufs, xw, cs));
        else
            LAUNCH(DXPBD_K_CG_UPDATE, k_cg_update4<true><<<nblk(V / 4 + 1), kBlock, 0, st>>>(V, it, bufs, xw, cs));
        return n + 1;
    };
    if (s->pcg_graph && !s->prof) {
        // the whole iteration loop as one graph launch: a WHILE node over one iteration whose update kernel's
        // last block sets the condition (kernels.cuh pcg_ctl_end); built once per scene, the buffers that
        // change between substeps are read from pcg_pp
        if (!s->pcg_exec) {
            if (!s->cap) {   // captured kernel nodes keep the capture stream's priority: the PCG's (highest)
                int least = 0, greatest = 0;
                DX_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
                DX_CHECK_CUDA(cudaStreamCreateWithPriority(&s->cap, cudaStreamNonBlocking, greatest));
            }
            cudaGraph_t g = nullptr;
            DX_CHECK_CUDA(cudaGraphCreate(&g, 0));
            cudaGraphConditionalHandle h;
            DX_CHECK_CUDA(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
            cudaMemsetParams mp = {};
            mp.dst = &s->pcg_ctl.p->it;
            mp.value = 0;
            mp.elementSize = 4;
            mp.width = 1;
            mp.height = 1;
            cudaGraphNode_t mn, wn;
            DX_CHECK_CUDA(cudaGraphAddMemsetNode(&mn, g, nullptr, 0, &mp));
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            DX_CHECK_CUDA(cudaGraphAddNode(&wn, g, &mn, 1, &cp));
            cudaGraph_t body = cp.conditional.phGraph_out[0];
            CGState cg = cs;
            cg.ctl = s->pcg_ctl.p;
            cg.cond = h;
            cg.maxit = maxit;
            cg.pp = s->pcg_pp.p;
            DX_CHECK_CUDA(cudaStreamBeginCaptureToGraph(s->cap, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
            s->pcg_kernels_per_it = iteration(-1, s->cap, cg);
            DX_CHECK_CUDA(cudaStreamEndCapture(s->cap, &body));
            if (defer) {
                DX_CHECK_CUDA(cudaStreamBeginCaptureToGraph(s->cap, g, &wn, nullptr, 1, cudaStreamCaptureModeThreadLocal));
                k_cg_ufinal<<<nblk(V), kBlock, 0, s->cap>>>(V, -1, bufs, cg);
                DX_CHECK_CUDA(cudaStreamEndCapture(s->cap, &g));
            }
            DX_CHECK_CUDA(cudaGraphInstantiate(&s->pcg_exec, g, 0));
            DX_CHECK_CUDA(cudaGraphDestroy(g));
        }
        k_set_pcg_ptrs<<<1, 1, 0, st>>>(s->pcg_pp.p, PcgPtrs{s->ax.p, tt.Q4, Qc, tQr});
        DX_CHECK_CUDA(cudaGraphLaunch(s->pcg_exec, st));
        DX_CHECK_CUDA(cudaGetLastError());
        iters_out = -1;   // known on the device only (PcgCtl, read at the end of the backward)
        relres_out = 0.0;
        return 1;
    }
    // launches between host convergence polls: first the previous solve's count (consecutive
    // substeps need nearly the same number), then small chunks; launches past convergence exit at once
    int chunk = s->last_iters > 0 ? std::max(s->last_iters + s->poll_extra, 2) : 8;
    iters_out = -1;
    relres_out = 0.0;
    // small scenes: the first chunk (the previous solve's iteration count) as ONE graph launch of that
    // many iterations (kernels with their iteration index baked in, the substep's rotating buffers read
    // from pcg_pp; iterations past convergence exit at once as in the stream launches)
    const bool chunk_graph = sweep_graph_on(s);
    while (it < maxit) {
        int end = std::min(maxit, it + chunk);
        chunk = 2;
        if (chunk_graph && it == 0 && end >= 2) {
            const dxpbd_scene::PcgChunk *ch = nullptr;
            for (auto &c : s->g_pcg)
                if (c.iters == end) ch = &c;
            if (!ch) {
                if (!s->pcg_pp.p) s->pcg_pp.alloc(1);
                CGState cg = cs;
                cg.pp = s->pcg_pp.p;
                int nl = 0;
                cudaGraphExec_t e = capture_graph(s, st == s->hi ? 1 : 0, [&](cudaStream_t cst) {
                    int n = 0;
                    for (int k = 0; k < end; ++k) n += iteration(k, cst, cg);
                    return n;
                }, nl);
                s->g_pcg.push_back({end, nl, e});
                ch = &s->g_pcg.back();
            }
            k_set_pcg_ptrs<<<1, 1, 0, st>>>(s->pcg_pp.p, PcgPtrs{s->ax.p, tt.Q4, Qc, tQr});
            DX_CHECK_CUDA(cudaGraphLaunch(ch->e, st));
            launches += 1 + ch->launches;
            it = end;
        } else {
            for (; it < end; ++it) launches += iteration(it, st, cs);
        }
        // convergence check: rr of the last completed iteration against |b|^2
        DX_CHECK_CUDA(cudaMemcpyAsync(s->h_scal, s->cg_sc.p, sizeof(double) * (size_t)(maxit + 2) * 4, cudaMemcpyDeviceToHost, st));
        DX_CHECK_CUDA(cudaStreamSynchronize(st));
        double bb = s->h_scal[(size_t)(maxit + 1) * 4];
        const double tol2 = (double)cs.tol2;   // the kernels' cg_done threshold, bit for bit
        if (bb == 0.0) { iters_out = 0; relres_out = 0.0; break; }
        for (int k = 0; k <= it; ++k) {
            double rr = s->h_scal[k * 4 + 2];
            if (k > 0 && rr == 0.0 && s->h_scal[k * 4 + 0] == 0.0) break;   // not executed (done earlier)
            if (rr <= tol2 * bb) { iters_out = k; relres_out = std::sqrt(rr / bb); break; }
        }
        if (iters_out >= 0) break;
        relres_out = std::sqrt(s->h_scal[it * 4 + 2] / bb);
    }
    if (iters_out >= 0) s->last_iters = iters_out;
    if (defer && iters_out > 0) {
        LAUNCH(DXPBD_K_CG_UPDATE, k_cg_ufinal<<<nblk(V), kBlock, 0, st>>>(V, iters_out, bufs, cs));
        ++launches;
    }
    DX_CHECK_CUDA(cudaGetLastError());
    if (iters_out < 0) {
        iters_out = maxit;
        throw Err{DXPBD_ERR_SOLVE, "PCG did not converge: relative residual " + std::to_string(relres_out) +
                                       " after " + std::to_string(maxit) + " iterations"};
    }
    return launches;
}

}  // namespace

// ================================================================== C ABI
extern "C" {

const char *dxpbd_last_error(void) { return g_err.c_str(); }
int dxpbd_version(void) { return 100; }

int dxpbd_destroy(dxpbd_scene *s) {
    if (!s) return DXPBD_OK;
    cudaSetDevice(s->device);
    if (s->h_scal) cudaFreeHost(s->h_scal);
    for (cudaEvent_t e : s->ev_pool) cudaEventDestroy(e);
    for (cudaEvent_t e : {s->ev_rep[0], s->ev_rep[1], s->ev_pcg[0], s->ev_pcg[1], s->ev_go, s->ev_end})
        if (e) cudaEventDestroy(e);
    if (s->aux) cudaStreamDestroy(s->aux);
    if (s->aux2) cudaStreamDestroy(s->aux2);
    for (int k = 0; k < 3; ++k)
        for (cudaEvent_t e : {s->ev_A[k], s->ev_B[k], s->ev_P[k]})
            if (e) cudaEventDestroy(e);
    if (s->hi) cudaStreamDestroy(s->hi);
    for (cudaEvent_t e : {s->ev_cp[0], s->ev_cp[1], s->ev_free[0], s->ev_free[1]})
        if (e) cudaEventDestroy(e);
    if (s->cpy) cudaStreamDestroy(s->cpy);
    if (s->pcg_exec) cudaGraphExecDestroy(s->pcg_exec);
    if (s->cap) cudaStreamDestroy(s->cap);
    if (s->g_fwd) cudaGraphExecDestroy(s->g_fwd);
    for (auto &e : s->g_rep) cudaGraphExecDestroy(e.e);
    for (auto &e : s->g_pcg) cudaGraphExecDestroy(e.e);
    if (s->cap_lo) cudaStreamDestroy(s->cap_lo);
    if (s->cap_mid) cudaStreamDestroy(s->cap_mid);
    delete s;
    return DXPBD_OK;
}

#define DX_API_BEGIN try {
#define DX_API_END                        \
    }                                     \
    catch (const Err &e) {                \
        g_err = e.msg;                    \
        return e.code;                    \
    }                                     \
    catch (const std::exception &e) {     \
        g_err = e.what();                 \
        return DXPBD_ERR_ARG;             \
    }                                     \
    g_err.clear();                        \
    return DXPBD_OK;

int dxpbd_create(const dxpbd_scene_desc *d, dxpbd_scene **out) {
    dxpbd_scene *s = nullptr;
    DX_API_BEGIN
    DX_REQUIRE(d && out, DXPBD_ERR_ARG, "null desc/out");
    DX_REQUIRE(d->num_vertices >= 1 && d->x_rest && d->inv_mass, DXPBD_ERR_ARG, "need vertices, x_rest, inv_mass");
    DX_REQUIRE(d->substeps >= 1 && d->iterations >= 1 && d->frame_dt > 0, DXPBD_ERR_ARG, "bad time stepping");
    DX_REQUIRE(d->max_frames >= 1, DXPBD_ERR_ARG, "max_frames >= 1");
    DX_REQUIRE(d->num_dist >= 0 && d->num_tets >= 0 && d->num_spheres >= 0 && d->num_capsules >= 0, DXPBD_ERR_ARG, "negative count");
    const int V = d->num_vertices;
    for (int j = 0; j < 2 * d->num_dist; ++j)
        DX_REQUIRE(d->dist_idx[j] >= 0 && d->dist_idx[j] < V, DXPBD_ERR_ARG, "dist_idx out of range");
    for (int j = 0; j < d->num_dist; ++j)
        DX_REQUIRE(d->dist_idx[2 * j] != d->dist_idx[2 * j + 1], DXPBD_ERR_ARG, "degenerate distance constraint");
    for (int j = 0; j < 4 * d->num_tets; ++j)
        DX_REQUIRE(d->tet_idx[j] >= 0 && d->tet_idx[j] < V, DXPBD_ERR_ARG, "tet_idx out of range");
    if (d->vertex_scene) {   // batch: scene ids in range, no constraint couples two scenes
        DX_REQUIRE(d->num_scenes >= 1, DXPBD_ERR_ARG, "num_scenes >= 1 with vertex_scene");
        for (int v = 0; v < V; ++v)
            DX_REQUIRE(d->vertex_scene[v] >= 0 && d->vertex_scene[v] < d->num_scenes, DXPBD_ERR_ARG, "vertex_scene out of range");
        for (int j = 0; j < d->num_dist; ++j)
            DX_REQUIRE(d->vertex_scene[d->dist_idx[2 * j]] == d->vertex_scene[d->dist_idx[2 * j + 1]], DXPBD_ERR_ARG,
                       "distance constraint couples two scenes");
        for (int j = 0; j < d->num_tets; ++j)
            for (int k = 1; k < 4; ++k)
                DX_REQUIRE(d->vertex_scene[d->tet_idx[4 * j + k]] == d->vertex_scene[d->tet_idx[4 * j]], DXPBD_ERR_ARG,
                           "tet couples two scenes");
        if (d->collider_scene)
            for (int c = 0; c < d->num_spheres + d->num_capsules; ++c)
                DX_REQUIRE(d->collider_scene[c] >= -1 && d->collider_scene[c] < d->num_scenes, DXPBD_ERR_ARG,
                           "collider_scene out of range");
    }
    DX_CHECK_CUDA(cudaSetDevice(d->device));
    s = new dxpbd_scene();
    s->device = d->device;
    s->V = V;
    s->E = d->num_dist;
    s->T = d->num_tets;
    s->NSH = d->num_spheres;
    s->NCAP = d->num_capsules;
    s->NC = s->NSH + s->NCAP;
    s->NS = d->num_shape;
    s->frame_dt = d->frame_dt;
    s->substeps = d->substeps;
    s->iterations = d->iterations;
    s->dt = d->frame_dt / d->substeps;
    s->inv_dt = 1.0f / s->dt;
    s->dtd = (double)d->frame_dt / (double)d->substeps;
    s->inv_dt2d = 1.0 / (s->dtd * s->dtd);
    s->gravity = make_float3(d->gravity[0], d->gravity[1], d->gravity[2]);
    s->h = d->thickness;
    s->coll_alpha = d->collision_compliance;
    s->max_frames = d->max_frames;
    s->grad_flags = d->grad_flags;
    s->pd = d->pd_projection;
    s->cg_tol = d->cg_tol > 0 ? d->cg_tol : 1e-6f;
    s->cg_max_iter = d->cg_max_iter > 0 ? d->cg_max_iter : 500;
    s->qf = (s->iterations == 1 && s->pd) ? 1 : 0;
    // A/B switches for measurements (defaults are the measured-best settings)
    if (const char *ev = getenv("DXPBD_WARM")) s->warm_order = atoi(ev) == 2 ? 2 : 1;
    if (const char *ev = getenv("DXPBD_NB")) s->nb = atoi(ev) == 2 ? 2 : 1;
    if (const char *ev = getenv("DXPBD_TET_PIPE")) s->tet_pipe = atoi(ev) != 0;
    if (const char *ev = getenv("DXPBD_NB_REPLAY")) s->nb_rep = atoi(ev) == 2 ? 2 : 1;
    if (const char *ev = getenv("DXPBD_REPLAY_MINB")) s->rep_minb = atoi(ev);
    if (const char *ev = getenv("DXPBD_DEFER_U")) s->defer_u = atoi(ev) != 0;
    if (const char *ev = getenv("DXPBD_TETV")) s->tetv = atoi(ev) != 0;
    if (const char *ev = getenv("DXPBD_TETV_MINB")) s->tetv_minb = atoi(ev);
    if (const char *ev = getenv("DXPBD_PSD_TOL")) s->psd_tol = (float)atof(ev);
    if (const char *ev = getenv("DXPBD_PSD_SWEEPS")) s->psd_sweeps = atoi(ev);
    if (const char *ev = getenv("DXPBD_PSD_MINB")) s->psd_minb = atoi(ev);
    if (const char *ev = getenv("DXPBD_OVERLAP")) s->overlap = atoi(ev) != 0;
    if (const char *ev = getenv("DXPBD_QCACHE")) s->qcache_on = atoi(ev) != 0;
    if (const char *ev = getenv("DXPBD_POLL_EXTRA")) s->poll_extra = atoi(ev);
    if (const char *ev = getenv("DXPBD_PCG_GRAPH")) s->pcg_graph = atoi(ev) != 0;
    if (const char *ev = getenv("DXPBD_SWEEP_GRAPH")) s->sweep_graph = atoi(ev) != 0;
    if (const char *ev = getenv("DXPBD_WAVE")) s->wave_on = atoi(ev) != 0;
    if (const char *ev = getenv("DXPBD_WAVE_G")) s->wave_g = std::max(1, atoi(ev));
    if (const char *ev = getenv("DXPBD_WAVE_FWD")) s->wave_fwd = atoi(ev) != 0;
    if (const char *ev = getenv("DXPBD_WAVE_REP")) s->wave_rep = atoi(ev) != 0;
    if (const char *ev = getenv("DXPBD_WAVE_LAG")) s->wave_lag = atoi(ev);

    if (const char *ev = getenv("DXPBD_WAVE_GRID_FWD")) s->wave_grid_fwd = atoi(ev);
    if (const char *ev = getenv("DXPBD_WAVE_GRID_REP")) s->wave_grid_rep = atoi(ev);

    cudaStream_t st = 0;

    // host topology: Morton vertex order, colors, constraint order, tiles (no GPU work)
    DistTopo topo;
    dist_topology(d, s->qf, topo);
    s->vperm_h = topo.vperm;
    std::vector<int32_t> vinv(V);
    for (int i = 0; i < V; ++i) vinv[s->vperm_h[i]] = i;
    s->vperm.alloc(V);
    upload(s->vperm.p, s->vperm_h.data(), sizeof(int32_t) * V, DXPBD_MEM_HOST, st);
    s->ntiles = (V + kTileV - 1) / kTileV;
    DBuf<float> tmpu;
    tmpu.alloc((size_t)V * 3);
    upload(tmpu.p, d->inv_mass, sizeof(float) * V, DXPBD_MEM_HOST, st);
    s->inv_mass.alloc(V);
    k_gather1<<<nblk(V), kBlock, 0, st>>>(V, tmpu.p, s->vperm.p, s->inv_mass.p);
    DBuf<float> xr3;   // internal order
    xr3.alloc((size_t)V * 3);
    upload(tmpu.p, d->x_rest, sizeof(float) * V * 3, DXPBD_MEM_HOST, st);
    k_gather3<<<nblk(V), kBlock, 0, st>>>(V, 1, tmpu.p, s->vperm.p, xr3.p);
    DX_CHECK_CUDA(cudaStreamSynchronize(st));

    // distance constraints: host topology (dist_topology), then device buffers
    if (s->E) {
        const int E = s->E;
        const int nc = topo.nc, nt = s->ntiles;
        s->n_dist_colors = nc;
        s->dist_color_h = topo.color;
        s->dist_perm_h = topo.perm;
        s->dist_off = topo.dist_off;
        const std::vector<int> &seg = topo.seg;
        const std::vector<int2> &ab_sorted = topo.ab;
        s->d_seg.alloc(seg.size());
        upload(s->d_seg.p, seg.data(), sizeof(int) * seg.size(), DXPBD_MEM_HOST, st);
        if (s->wave_on && s->iterations == 1) build_wave_plan(s, seg, ab_sorted, d->x_rest, st);
        s->d_fseg.alloc(topo.fseg.size());
        upload(s->d_fseg.p, topo.fseg.data(), sizeof(int) * topo.fseg.size(), DXPBD_MEM_HOST, st);
        s->n_foreign = topo.n_foreign;
        s->hcap = topo.hcap;
        s->halo_total = topo.halo_total;
        s->capm = topo.capm;
        s->use_tma = topo.use_tma;
        (void)nt;
        s->pull = topo.pull;
        if (s->use_tma) {
            s->d_hpad.alloc(topo.hpad.size());
            upload(s->d_hpad.p, topo.hpad.data(), sizeof(int) * topo.hpad.size(), DXPBD_MEM_HOST, st);
            if (s->pull) {
                s->ycap = topo.ycap;
                s->d_ptd.alloc(topo.ptd.size());
                upload(s->d_ptd.p, topo.ptd.data(), sizeof(int4) * topo.ptd.size(), DXPBD_MEM_HOST, st);
                s->d_pidx.alloc(topo.pidx.size());
                upload(s->d_pidx.p, topo.pidx.data(), sizeof(uint32_t) * topo.pidx.size(), DXPBD_MEM_HOST, st);
                s->pull_smem = pull_smem_bytes(s->hcap, s->ycap, 1);
                s->pull_rhs_smem = pull_smem_bytes(s->hcap, s->ycap, 2);
                DX_CHECK_CUDA(cudaFuncSetAttribute(k_cg_matvec_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->pull_smem));
                DX_CHECK_CUDA(cudaFuncSetAttribute(k_rhs_pull, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->pull_rhs_smem));
                s->pull_psmem = pull_persist_smem_bytes(s->hcap, s->ycap);
                DX_CHECK_CUDA(cudaFuncSetAttribute(k_cg_matvec_pull_p, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->pull_psmem));
                DX_CHECK_CUDA(cudaDeviceGetAttribute(&s->num_sms, cudaDevAttrMultiProcessorCount, s->device));
                if (const char *ev = getenv("DXPBD_PULL_PERSIST")) s->pull_persist = atoi(ev) != 0;
            } else {
                s->d_tseg.alloc(topo.tseg.size());
                upload(s->d_tseg.p, topo.tseg.data(), sizeof(int4) * topo.tseg.size(), DXPBD_MEM_HOST, st);
                s->d_vslot.alloc(topo.vslot.size());
                upload(s->d_vslot.p, topo.vslot.data(), sizeof(uint16_t) * topo.vslot.size(), DXPBD_MEM_HOST, st);
                s->d_hslot.alloc(topo.hslot.size());
                upload(s->d_hslot.p, topo.hslot.data(), sizeof(uint16_t) * topo.hslot.size(), DXPBD_MEM_HOST, st);
                s->d_cpair.alloc(topo.cpair.size());
                upload(s->d_cpair.p, topo.cpair.data(), sizeof(uint32_t) * topo.cpair.size(), DXPBD_MEM_HOST, st);
            }
            s->d_fpos.alloc(E);
            upload(s->d_fpos.p, topo.fposv.data(), sizeof(int) * E, DXPBD_MEM_HOST, st);
            s->d_tpos.alloc(E);
            upload(s->d_tpos.p, topo.tpos.data(), sizeof(int) * E, DXPBD_MEM_HOST, st);
            s->d_Qt.alloc((size_t)topo.ntot + 1);
            if (s->qf == 0) s->d_Qt2b.alloc((size_t)topo.ntot + 2);
            s->tma_smem = tma_smem_bytes(s->hcap, s->capm, s->qf == 0);
            s->tma_rhs_smem = tma_rhs_smem_bytes(s->hcap, s->capm, s->qf == 0);
            DX_CHECK_CUDA(cudaFuncSetAttribute(k_cg_matvec_tma<kMvThreads, kMvMinB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->tma_smem));
            DX_CHECK_CUDA(cudaFuncSetAttribute(k_rhs_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s->tma_rhs_smem));
        }
        s->d_fidx.alloc(topo.fidx.size());
        upload(s->d_fidx.p, topo.fidx.data(), sizeof(int) * topo.fidx.size(), DXPBD_MEM_HOST, st);
        std::vector<int4> fent(topo.fidx.size());
        for (size_t q = 0; q < topo.fidx.size(); ++q)
            fent[q] = make_int4(topo.fidx[q], ab_sorted[topo.fidx[q]].x, ab_sorted[topo.fidx[q]].y, 0);
        s->d_fent.alloc(fent.size());
        upload(s->d_fent.p, fent.data(), sizeof(int4) * fent.size(), DXPBD_MEM_HOST, st);
        DBuf<float> alpha_u;
        alpha_u.alloc(E);
        upload(alpha_u.p, d->dist_compliance, sizeof(float) * E, DXPBD_MEM_HOST, st);
        s->d_perm.alloc(E);
        upload(s->d_perm.p, s->dist_perm_h.data(), sizeof(int32_t) * E, DXPBD_MEM_HOST, st);
        {   // vertices no color-0 constraint touches (prediction fused into the first color, k_dist_first)
            std::vector<char> cov(V, 0);
            for (int q = s->dist_off[0]; q < s->dist_off[1]; ++q) { cov[ab_sorted[q].x] = 1; cov[ab_sorted[q].y] = 1; }
            std::vector<int> un;
            for (int v = 0; v < V; ++v)
                if (!cov[v]) un.push_back(v);
            const char *ev = getenv("DXPBD_FUSE_PREDICT");
            s->fuse_predict = nc >= 2 && s->iterations == 1 && (int64_t)un.size() * 4 <= V && !(ev && atoi(ev) == 0);
            if (s->fuse_predict && !un.empty()) {
                s->uncov.alloc(un.size());
                upload(s->uncov.p, un.data(), sizeof(int) * un.size(), DXPBD_MEM_HOST, st);
            }
        }
        s->d_idx.alloc(E + 2);   // +2: the bulk copies round segment ends up to 16 bytes
        DX_CHECK_CUDA(cudaMemsetAsync(s->d_idx.p, 0, sizeof(int2) * (E + 2), st));
        upload(s->d_idx.p, ab_sorted.data(), sizeof(int2) * E, DXPBD_MEM_HOST, st);
        s->d_rest.alloc(E);
        s->d_alpha.alloc(E);
        k_gather_f<<<nblk(E), kBlock, 0, st>>>(E, alpha_u.p, s->d_perm.p, s->d_alpha.p);
        k_rest_len<<<nblk(E), kBlock, 0, st>>>(E, s->d_idx.p, xr3.p, s->d_rest.p);
        DX_CHECK_CUDA(cudaGetLastError());
        DX_CHECK_CUDA(cudaStreamSynchronize(st));
    }
    // tets
    if (s->T) {
        const int T = s->T;
        int nc = greedy_colors(T, 4, d->tet_idx, V, s->tet_color_h);
        if (nc < 0) throw Err{DXPBD_ERR_LIMIT, "tet coloring needs more than 256 colors"};
        s->n_tet_colors = nc;
        color_sort(s->tet_color_h, nc, s->tet_perm_h, s->tet_off);
        // within a color, order by the smallest internal vertex id (locality of the gathers)
        std::vector<int4> ti(T);
        for (int j = 0; j < T; ++j)
            ti[j] = make_int4(vinv[d->tet_idx[4 * j]], vinv[d->tet_idx[4 * j + 1]], vinv[d->tet_idx[4 * j + 2]],
                              vinv[d->tet_idx[4 * j + 3]]);
        auto mn = [&](int j) { return std::min(std::min(ti[j].x, ti[j].y), std::min(ti[j].z, ti[j].w)); };
        for (int c = 0; c < nc; ++c)
            std::sort(s->tet_perm_h.begin() + s->tet_off[c], s->tet_perm_h.begin() + s->tet_off[c + 1],
                      [&](int32_t x, int32_t y) { return mn(x) < mn(y); });
        std::vector<int4> ts(T);
        for (int q = 0; q < T; ++q) ts[q] = ti[s->tet_perm_h[q]];
        s->t_idx.alloc(T);
        upload(s->t_idx.p, ts.data(), sizeof(int4) * T, DXPBD_MEM_HOST, st);
        {   // deterministic corner gather: per vertex its (corner c, sorted tet q) slots 3 c T + q, ascending
            std::vector<int> goff(V + 1, 0), ginc((size_t)4 * T);
            for (int q = 0; q < T; ++q)
                for (int v : {ts[q].x, ts[q].y, ts[q].z, ts[q].w}) goff[v + 1]++;
            for (int v = 0; v < V; ++v) goff[v + 1] += goff[v];
            std::vector<int> fill(goff.begin(), goff.end() - 1);
            for (int c = 0; c < 4; ++c)
                for (int q = 0; q < T; ++q) {
                    const int v = c == 0 ? ts[q].x : c == 1 ? ts[q].y : c == 2 ? ts[q].z : ts[q].w;
                    ginc[fill[v]++] = 3 * c * T + q;
                }
            s->t_goff.alloc(V + 1);
            upload(s->t_goff.p, goff.data(), sizeof(int) * (V + 1), DXPBD_MEM_HOST, st);
            s->t_ginc.alloc(ginc.size());
            upload(s->t_ginc.p, ginc.data(), sizeof(int) * ginc.size(), DXPBD_MEM_HOST, st);
            s->t_gq.alloc((size_t)24 * T);
            DX_CHECK_CUDA(cudaMemsetAsync(s->t_gq.p, 0, sizeof(float) * 24 * T, st));   // pinned corners stay 0
            DX_CHECK_CUDA(cudaStreamSynchronize(st));
        }
        s->t_perm.alloc(T);
        upload(s->t_perm.p, s->tet_perm_h.data(), sizeof(int32_t) * T, DXPBD_MEM_HOST, st);
        DBuf<float> tmpab;
        tmpab.alloc(T);
        s->t_a.alloc(T);
        s->t_b.alloc(T);
        upload(tmpab.p, d->tet_a, sizeof(float) * T, DXPBD_MEM_HOST, st);
        k_gather_f<<<nblk(T), kBlock, 0, st>>>(T, tmpab.p, s->t_perm.p, s->t_a.p);
        DX_CHECK_CUDA(cudaStreamSynchronize(st));
        upload(tmpab.p, d->tet_b, sizeof(float) * T, DXPBD_MEM_HOST, st);
        k_gather_f<<<nblk(T), kBlock, 0, st>>>(T, tmpab.p, s->t_perm.p, s->t_b.p);
        s->t_Dm.alloc((size_t)9 * T);
        s->t_vol.alloc(T);
        k_tet_rest<<<nblk(T), kBlock, 0, st>>>(T, s->t_idx.p, xr3.p, s->t_Dm.p, s->t_vol.p);
        s->t_Dmf.alloc((size_t)9 * T);
        k_d2f<<<nblk((int64_t)9 * T), kBlock, 0, st>>>((size_t)9 * T, s->t_Dm.p, s->t_Dmf.p);
        if (s->iterations > 1) s->lam_t.alloc((size_t)2 * T);
        DX_CHECK_CUDA(cudaGetLastError());
        DX_CHECK_CUDA(cudaStreamSynchronize(st));
    }
    // colliders
    if (s->NC) {
        if (s->NSH) {
            s->sph.alloc((size_t)4 * s->NSH);
            upload(s->sph.p, d->spheres, sizeof(float) * 4 * s->NSH, DXPBD_MEM_HOST, st);
        }
        if (s->NCAP) {
            s->cap_c.alloc(3 * s->NCAP); upload(s->cap_c.p, d->cap_center, sizeof(float) * 3 * s->NCAP, DXPBD_MEM_HOST, st);
            s->cap_a.alloc(3 * s->NCAP); upload(s->cap_a.p, d->cap_axis, sizeof(float) * 3 * s->NCAP, DXPBD_MEM_HOST, st);
            s->cap_r0.alloc(s->NCAP); upload(s->cap_r0.p, d->cap_r0, sizeof(float) * s->NCAP, DXPBD_MEM_HOST, st);
            s->cap_L0.alloc(s->NCAP); upload(s->cap_L0.p, d->cap_L0, sizeof(float) * s->NCAP, DXPBD_MEM_HOST, st);
            if (s->NS) {
                s->cap_Rb.alloc((size_t)s->NCAP * s->NS); upload(s->cap_Rb.p, d->cap_rbasis, sizeof(float) * s->NCAP * s->NS, DXPBD_MEM_HOST, st);
                s->cap_Lb.alloc((size_t)s->NCAP * s->NS); upload(s->cap_Lb.p, d->cap_lbasis, sizeof(float) * s->NCAP * s->NS, DXPBD_MEM_HOST, st);
                s->beta.alloc(s->NS); upload(s->beta.p, d->shape_beta, sizeof(float) * s->NS, DXPBD_MEM_HOST, st);
            }
        }
        s->cols.alloc(s->NC);
        if (d->vertex_scene && d->collider_scene) {
            s->csc.alloc(s->NC);
            upload(s->csc.p, d->collider_scene, sizeof(int32_t) * s->NC, DXPBD_MEM_HOST, st);
        }
        apply_shape(s, st);
    }
    if (d->vertex_scene) {   // per-vertex scene ids in internal order
        s->num_scenes = d->num_scenes;
        std::vector<int32_t> vs(V);
        for (int i = 0; i < V; ++i) vs[i] = d->vertex_scene[s->vperm_h[i]];
        s->vsc.alloc(V);
        upload(s->vsc.p, vs.data(), sizeof(int32_t) * V, DXPBD_MEM_HOST, st);
    }
    // trajectory storage
    const size_t nstates = g_ring_states > 0 ? (size_t)g_ring_states : (size_t)s->max_frames * s->substeps + 1;
    s->ckpt.alloc(nstates * V);
    s->v0.alloc(V);
    s->tmp3.alloc((size_t)V * 3);
    if (s->iterations > 1) {
        if (s->E) s->lam_d.alloc(s->E);
        if (s->NC) s->lam_c.alloc((size_t)s->NC * V);
    }
    DX_CHECK_CUDA(cudaMallocHost(&s->h_scal, sizeof(double) * (size_t)(s->cg_max_iter + 2) * 4));
    DX_CHECK_CUDA(cudaStreamSynchronize(st));
    *out = s;
    s = nullptr;
    }
    catch (const Err &e) {
        g_err = e.msg;
        if (s) dxpbd_destroy(s);
        return e.code;
    }
    g_err.clear();
    return DXPBD_OK;
}

int dxpbd_forward(dxpbd_scene *s, const float *x0, const float *v0, const float *forces, int32_t num_frames,
                  int32_t mem, void *stream) {
    DX_API_BEGIN
    DX_REQUIRE(s && x0 && v0, DXPBD_ERR_ARG, "null argument");
    DX_REQUIRE(num_frames >= 0 && num_frames <= s->max_frames, DXPBD_ERR_LIMIT, "num_frames exceeds max_frames");
    DX_CHECK_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = (cudaStream_t)stream;
    forward_inputs(s, x0, v0, forces, num_frames, mem, st, true);
    int launches = 4;
    const int N = num_frames * s->substeps;
    // block cache for the last substeps in spare HBM (K = 1 TMA path without tets / compliance
    // gradients, which need the replay's other outputs): distance blocks, and with colliders the
    // per-vertex contact blocks and (collider gradients) the collider controls
    s->qc_count = 0;
    if (s->qcache_on && s->use_tma && s->qf == 1 && !s->T && !((s->grad_flags >> DXPBD_GRAD_COMPLIANCE) & 1) &&
        s->iterations == 1 && N > 0) {
        const bool want_ce = (s->grad_flags & ((1u << DXPBD_GRAD_SHAPE) | (1u << DXPBD_GRAD_SPHERE))) != 0;
        s->qc_cper = s->NC ? (size_t)6 * s->V + (want_ce ? (size_t)12 * s->NC * s->V : 0) : 0;
        const size_t per = sizeof(float4) * s->d_Qt.n + sizeof(float) * s->qc_cper;
        size_t freeb = 0, totalb = 0;
        DX_CHECK_CUDA(cudaMemGetInfo(&freeb, &totalb));
        freeb += s->qcache.n * sizeof(float4) + s->qccache.n * sizeof(float);   // the current cache is reusable
        // keep room for the backward's buffers (~20 vertex vectors + the second block buffers) and 2 GB
        const size_t reserve = (size_t)24 * 16 * s->V + per + ((size_t)2 << 30);
        const int M = freeb > reserve ? (int)std::min<size_t>((size_t)N, (freeb - reserve) / 5 * 4 / per) : 0;
        if (M > 0) {
            if (s->qcache.n < (size_t)M * s->d_Qt.n) {
                s->qcache.free();
                s->qcache.alloc((size_t)M * s->d_Qt.n);
            }
            if (s->qccache.n < (size_t)M * s->qc_cper) {
                s->qccache.free();
                s->qccache.alloc((size_t)M * s->qc_cper);
            }
            s->qc_first = N - M;
            s->qc_count = M;
        }
    }
    const bool host_forces = forces && mem == DXPBD_MEM_HOST;
    if (host_forces && num_frames > 0) upload_frame_forces(s, forces, 0, st);
    for (int n = 0; n < N; ++n) {
        // the next frame's forces travel while this frame's substeps run
        if (host_forces && n % s->substeps == 0 && n / s->substeps + 1 < num_frames)
            upload_frame_forces(s, forces, n / s->substeps + 1, st);
        launches += forward_substep(s, n, st);
    }
    if (host_forces) DX_CHECK_CUDA(cudaStreamSynchronize(s->cpy));   // the caller's buffer may be reused
    DX_CHECK_CUDA(cudaGetLastError());
    s->frames_done = num_frames;
    s->have_grads = false;
    s->stats[2] = launches;
    DX_API_END
}

int dxpbd_positions(dxpbd_scene *s, int32_t frame, float *out, int32_t mem, void *stream) {
    DX_API_BEGIN
    DX_REQUIRE(s && out, DXPBD_ERR_ARG, "null argument");
    DX_REQUIRE(s->frames_done >= 0 && frame >= 0 && frame <= s->frames_done, DXPBD_ERR_STATE, "frame not simulated");
    DX_CHECK_CUDA(cudaSetDevice(s->device));
    positions_from(s, state(s, frame * s->substeps), out, mem, (cudaStream_t)stream);
    DX_API_END
}

int dxpbd_backward(dxpbd_scene *s, int32_t num_keys, const int32_t *key_frames, const float *targets,
                   const float *weights, int32_t mem, float *loss_out, void *stream) {
    DX_API_BEGIN
    DX_REQUIRE(s, DXPBD_ERR_ARG, "null scene");
    DX_REQUIRE(s->frames_done >= 0, DXPBD_ERR_STATE, "backward before forward");
    DX_REQUIRE(num_keys >= 0 && (num_keys == 0 || (key_frames && targets)), DXPBD_ERR_ARG, "bad keyframes");
    DX_CHECK_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int V = s->V, E = s->E, sub = s->substeps;
    const int N = s->frames_done * sub;
    for (int k = 0; k < num_keys; ++k)
        DX_REQUIRE(key_frames[k] >= 0 && key_frames[k] <= s->frames_done, DXPBD_ERR_ARG, "key frame out of range");
    BwdSetup su = backward_prepare(s, num_keys, key_frames, targets, weights, mem, st);
    const float *wts = su.wts;
    const bool g_comp = su.g_comp, g_forces = su.g_forces, g_coll = su.g_coll, warm2 = su.warm2;
    const int last_key_state = su.last_key_state;
    std::vector<int> &key_of = su.key_of;
    // loss
    for (int k = 0; k < num_keys; ++k)
        LAUNCH(DXPBD_K_OTHER, k_loss<<<nblk(V), kBlock, 0, st>>>(V, state(s, key_frames[k] * sub), s->targets.p + (size_t)k * V * 3, wts, s->acc.p));
    auto tgt = [&](int n) -> const float * { return key_of[n] >= 0 ? s->targets.p + (size_t)key_of[n] * V * 3 : nullptr; };
    int launches = num_keys + 2, total_it = 0, max_it = 0;
    double worst = 0.0;
    int solves = 0;
    // PCG iteration loops as graph launches (pcg_solve): counts and convergence come back once, at the end
    const bool gmode = s->pcg_graph && !s->prof;
    if (gmode) {
        if (!s->pcg_ctl.p) s->pcg_ctl.alloc(1);
        if (!s->pcg_pp.p) s->pcg_pp.alloc(1);
        DX_CHECK_CUDA(cudaMemsetAsync(s->pcg_ctl.p, 0, sizeof(PcgCtl), st));
    }
    // PCG start fused into the TMA rhs kernel (no tet rhs pass after it, standard PCG)
    const bool fuse_start = s->use_tma && !s->T;
    // replay of substep n-1 on the aux stream during the PCG of substep n (independent work: the
    // replay reads only checkpoints); blocks double-buffered, ordered by events
    const bool ovl_cloth = s->overlap && s->use_tma && s->qf == 1 && !s->T && !g_comp;
    // tet-only scenes: the tet blocks (and material controls) are double-buffered the same way
    const bool ovl_tet = s->overlap && s->T && E == 0 && !s->NC && !s->use_tma;
    const bool ovl = ovl_cloth || ovl_tet;
    const bool g_mat = ((s->grad_flags >> DXPBD_GRAD_MATERIAL) & 1) != 0;
    // three-stage tet pipeline: A(n-2) = iterate passes + derivative blocks on aux2, B(n-1) = PD projection
    // of the blocks on aux, PCG(n) on hi; blocks / controls triple-buffered (index n % 3)
    const bool tet3 = ovl_tet && s->tet_pipe && s->pd && s->iterations == 1;
    auto set_write = [&](int k) {   // replay output buffers of parity k (tet3: index k of 3)
        if (ovl_tet) {
            s->tq_w = k == 2 ? s->t_Q3.p : (k ? s->t_Q2.p : s->t_Q.p);
            s->te_w = g_mat ? (k == 2 ? s->t_e3.p : (k ? s->t_e2.p : s->t_e.p)) : nullptr;
        } else {
            s->qt_write = k ? s->d_Qt2.p : s->d_Qt.p;
        }
        if (s->NC) {   // contact blocks and collider controls
            s->qc_w = k ? s->Qc2.p : s->Qc.p;
            s->ec_w = g_coll ? (k ? s->ec2.p : s->ec.p) : nullptr;
        }
    };
    auto set_read = [&](int k) {
        if (ovl_tet) {
            s->tq_r = k == 2 ? s->t_Q3.p : (k ? s->t_Q2.p : s->t_Q.p);
            s->te_r = g_mat ? (k == 2 ? s->t_e3.p : (k ? s->t_e2.p : s->t_e.p)) : nullptr;
        } else {
            s->qt_read = k ? s->d_Qt2.p : s->d_Qt.p;
        }
        if (s->NC) {
            s->qc_r = k ? s->Qc2.p : s->Qc.p;
            s->ec_r = g_coll ? (k ? s->ec2.p : s->ec.p) : nullptr;
        }
    };
    // blocks of the last substeps were cached by the forward (valid for the overlap path only)
    auto cached = [&](int n) { return ovl && s->qc_count > 0 && n >= s->qc_first && n < s->qc_first + s->qc_count; };
    cudaStream_t user_st = st;
    const int n_hi = std::min(N, last_key_state) - 1;
    if (ovl && n_hi >= 0) {
        if (ovl_cloth && s->d_Qt2.n < s->d_Qt.n) s->d_Qt2.alloc(s->d_Qt.n);
        if (s->NC) {
            if (s->Qc2.n < s->Qc.n) s->Qc2.alloc(s->Qc.n);
            if (g_coll && s->ec2.n < s->ec.n) s->ec2.alloc(s->ec.n);
        }
        if (ovl_tet) {
            if (s->t_Q2.n < s->t_Q.n) s->t_Q2.alloc(s->t_Q.n);
            if (g_mat && s->t_e2.n < s->t_e.n) s->t_e2.alloc(s->t_e.n);
            if (tet3) {
                if (s->t_Q3.n < s->t_Q.n) s->t_Q3.alloc(s->t_Q.n);
                if (g_mat && s->t_e3.n < s->t_e.n) s->t_e3.alloc(s->t_e.n);
            }
        }
        if (!s->aux) {
            int least = 0, greatest = 0;
            DX_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            DX_CHECK_CUDA(cudaStreamCreateWithPriority(&s->aux, cudaStreamNonBlocking, least));
            DX_CHECK_CUDA(cudaStreamCreateWithPriority(&s->hi, cudaStreamNonBlocking, greatest));
            for (int k = 0; k < 2; ++k) {
                DX_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_rep[k], cudaEventDisableTiming));
                DX_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_pcg[k], cudaEventDisableTiming));
            }
            DX_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_go, cudaEventDisableTiming));
            DX_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_end, cudaEventDisableTiming));
        }
        if (tet3 && !s->aux2) {
            int least = 0, greatest = 0;
            DX_CHECK_CUDA(cudaDeviceGetStreamPriorityRange(&least, &greatest));
            DX_CHECK_CUDA(cudaStreamCreateWithPriority(&s->aux2, cudaStreamNonBlocking, least));
            for (int k = 0; k < 3; ++k) {
                DX_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_A[k], cudaEventDisableTiming));
                DX_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_B[k], cudaEventDisableTiming));
                DX_CHECK_CUDA(cudaEventCreateWithFlags(&s->ev_P[k], cudaEventDisableTiming));
            }
        }
        DX_CHECK_CUDA(cudaEventRecord(s->ev_go, st));   // inputs of this call are on `st`
        DX_CHECK_CUDA(cudaStreamWaitEvent(s->aux, s->ev_go, 0));
        if (tet3) DX_CHECK_CUDA(cudaStreamWaitEvent(s->aux2, s->ev_go, 0));
        // the PCG path runs on the high-priority stream; the replay fills the SMs it leaves idle
        DX_CHECK_CUDA(cudaStreamWaitEvent(s->hi, s->ev_go, 0));
        user_st = st;
        st = s->hi;
        if (tet3) {   // fill the pipeline: A(n_hi), B(n_hi), A(n_hi - 1)
            auto stage_a = [&](int m) {
                set_write(m % 3);
                launches += replay_substep(s, m, s->aux2, 1);
                DX_CHECK_CUDA(cudaEventRecord(s->ev_A[m % 3], s->aux2));
            };
            stage_a(n_hi);
            DX_CHECK_CUDA(cudaStreamWaitEvent(s->aux, s->ev_A[n_hi % 3], 0));
            set_write(n_hi % 3);
            launches += replay_substep(s, n_hi, s->aux, 2);
            DX_CHECK_CUDA(cudaEventRecord(s->ev_B[n_hi % 3], s->aux));
            if (n_hi >= 1) stage_a(n_hi - 1);
        } else if (!cached(n_hi)) {
            set_write(n_hi & 1);
            launches += replay_substep(s, n_hi, s->aux);
            DX_CHECK_CUDA(cudaEventRecord(s->ev_rep[n_hi & 1], s->aux));
        }
    }
    for (int n = n_hi; n >= 0; --n) {
        const int frame = n / sub;
        float *gf = g_forces ? s->g_force.p + (size_t)frame * V * 3 : nullptr;
        if (tet3) {
            if (n >= 1) {   // B(n-1): PD projection of the blocks A(n-1) wrote
                DX_CHECK_CUDA(cudaStreamWaitEvent(s->aux, s->ev_A[(n - 1) % 3], 0));
                set_write((n - 1) % 3);
                launches += replay_substep(s, n - 1, s->aux, 2);
                DX_CHECK_CUDA(cudaEventRecord(s->ev_B[(n - 1) % 3], s->aux));
            }
            if (n >= 2) {   // A(n-2) into the buffer PCG(n+1) finished reading
                if (n + 1 <= n_hi) DX_CHECK_CUDA(cudaStreamWaitEvent(s->aux2, s->ev_P[(n + 1) % 3], 0));
                set_write((n - 2) % 3);
                launches += replay_substep(s, n - 2, s->aux2, 1);
                DX_CHECK_CUDA(cudaEventRecord(s->ev_A[(n - 2) % 3], s->aux2));
            }
            DX_CHECK_CUDA(cudaStreamWaitEvent(st, s->ev_B[n % 3], 0));
            set_read(n % 3);
        } else if (ovl) {
            if (n >= 1 && !cached(n - 1)) {   // blocks of substep n-1 into the buffer PCG(n+1) finished reading
                if (n + 1 <= n_hi && !cached(n + 1)) DX_CHECK_CUDA(cudaStreamWaitEvent(s->aux, s->ev_pcg[(n - 1) & 1], 0));
                set_write((n - 1) & 1);
                launches += replay_substep(s, n - 1, s->aux);
                DX_CHECK_CUDA(cudaEventRecord(s->ev_rep[(n - 1) & 1], s->aux));
            }
            if (cached(n)) {
                s->qt_read = s->qcache.p + (size_t)(n - s->qc_first) * s->d_Qt.n;
                if (s->NC) {
                    float *slot = s->qccache.p + (size_t)(n - s->qc_first) * s->qc_cper;
                    s->qc_r = slot;
                    s->ec_r = g_coll ? slot + (size_t)6 * V : nullptr;
                }
            } else {
                DX_CHECK_CUDA(cudaStreamWaitEvent(st, s->ev_rep[n & 1], 0));
                set_read(n & 1);
            }
        } else {
            s->qt_write = s->qt_read = nullptr;
            launches += replay_substep(s, n, st);
        }
        const float *Qc = s->NC ? (s->qc_r ? s->qc_r : s->Qc.p) : nullptr;   // contact blocks of substep n
        // b = M u_{n+1} - Q_n y_{n+1} + dphi/dx_{n+1} and the warm-start residual r0 = b - A_n u_{n+1}
        // (one tiled pass, own vertices stored once); the PCG then starts from u_n := u_{n+1}.
        DX_CHECK_CUDA(cudaMemsetAsync(s->cg_sc.p, 0, sizeof(double) * (size_t)(s->cg_max_iter + 2) * 4, st));
        {
            TileLists tl{s->n_dist_colors, s->ntiles, s->d_seg.p, s->d_fseg.p, s->d_fidx.p, s->d_fent.p};
            TmaTiles tt = s->tma_tiles();
            if (s->pull)
                LAUNCH(DXPBD_K_RHS, k_rhs_pull<<<s->ntiles, kTileV, s->pull_rhs_smem, st>>>(
                    s->pull_tiles(), V, Qc, s->ax.p, s->uprev.p, warm2 ? s->uprev2.p : nullptr, s->y.p, state(s, n + 1), tgt(n + 1), wts, s->inv_mass.p, s->rhs.p,
                    s->r.p, s->u0.p, 0, fuse_start ? s->p.p : nullptr,
                    CGState{s->cg_sc.p, s->cg_sc.p + (size_t)(s->cg_max_iter + 1) * 4, s->cg_tol * s->cg_tol}));
            else if (s->use_tma)
                LAUNCH(DXPBD_K_RHS, k_rhs_tma<<<s->ntiles, kTmaThreads, s->tma_rhs_smem, st>>>(
                    tt, V, Qc, s->ax.p, s->uprev.p, warm2 ? s->uprev2.p : nullptr, s->y.p, state(s, n + 1), tgt(n + 1), wts, s->inv_mass.p, s->rhs.p,
                    s->r.p, s->u0.p, 0, fuse_start ? s->p.p : nullptr,
                    CGState{s->cg_sc.p, s->cg_sc.p + (size_t)(s->cg_max_iter + 1) * 4, s->cg_tol * s->cg_tol}));
            else if (s->qf == 1)
                LAUNCH(DXPBD_K_RHS, k_rhs_tiled<1><<<s->ntiles, kBlock, 0, st>>>(tl, V, s->d_idx.p, s->Qd.p, E, Qc, s->ax.p, s->uprev.p,
                                                                                 s->y.p, state(s, n + 1), tgt(n + 1), wts, s->inv_mass.p,
                                                                                 s->rhs.p, s->r.p, s->u0.p));
            else
                LAUNCH(DXPBD_K_RHS, k_rhs_tiled<0><<<s->ntiles, kBlock, 0, st>>>(tl, V, s->d_idx.p, s->Qd.p, E, Qc, s->ax.p, s->uprev.p,
                                                                                 s->y.p, state(s, n + 1), tgt(n + 1), wts, s->inv_mass.p,
                                                                                 s->rhs.p, s->r.p, s->u0.p));
            ++launches;
        }
        if (s->T) {
            LAUNCH(DXPBD_K_RHS, k_rhs_tet<<<nblk(s->T), kBlock, 0, st>>>(s->tdev(), s->tq_r ? s->tq_r : s->t_Q.p, s->y.p, s->u0.p, s->rhs.p, s->r.p,
                                                                        s->inv_mass.p));
            LAUNCH(DXPBD_K_RHS, k_rhs_tet_gather<<<nblk(V), kBlock, 0, st>>>(V, s->tdev(), s->rhs.p, s->r.p, s->inv_mass.p));
            launches += 2;
        }
        int iters = 0;
        double rel = 0.0;
        // rotate: the PCG iterates on the warm start u0; afterwards ax = u_n, uprev = u_{n+1}
        std::swap(s->ax.p, s->u0.p);      // ax <- u0 (solution buffer), u0 <- u_{n+1}
        launches += pcg_solve(s, st, iters, rel, fuse_start);   // u_n into s->ax
        if (warm2) std::swap(s->uprev2.p, s->uprev.p);   // uprev2 <- u_{n+2}
        std::swap(s->uprev.p, s->u0.p);   // uprev <- u_{n+1}, u0 <- u_{n+2} or u_{n+3} (free)
        if (iters >= 0) {
            total_it += iters;
            max_it = std::max(max_it, iters);
            worst = std::max(worst, rel);
        }
        ++solves;
        LAUNCH(DXPBD_K_ADJOINT, k_adjoint_accum<<<nblk(V), kBlock, 0, st>>>(V, s->inv_mass.p, s->ax.p, s->y.p, gf, s->dt));
        ++launches;
        if (g_comp && E) {
            LAUNCH(DXPBD_K_GRADS, k_grad_compliance<<<nblk(E), kBlock, 0, st>>>(E, s->d_idx.p, s->ed.p, s->y.p, s->g_comp.p));
            ++launches;
        }
        if (g_coll && s->NC) {
            LAUNCH(DXPBD_K_GRADS, k_grad_colliders<<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->ec_r ? s->ec_r : s->ec.p, s->y.p, s->acc.p + 1));
            ++launches;
        }
        if (s->T && ((s->grad_flags >> DXPBD_GRAD_MATERIAL) & 1)) {
            LAUNCH(DXPBD_K_GRADS, k_grad_tet<<<nblk(s->T), kBlock, 0, st>>>(s->tdev(), s->te_r ? s->te_r : s->t_e.p, s->y.p, s->t_g.p));
            ++launches;
        }
        if (tet3) DX_CHECK_CUDA(cudaEventRecord(s->ev_P[n % 3], st));    // buffer n % 3 free again
        else if (ovl) DX_CHECK_CUDA(cudaEventRecord(s->ev_pcg[n & 1], st));   // buffer n & 1 free again
        if (s->gs_out && g_forces && n % sub == 0) stream_frame_grads(s, frame, st);   // frame complete
    }
    s->qt_read = s->qt_write = nullptr;
    s->tq_w = s->te_w = s->tq_r = s->te_r = nullptr;
    s->qc_w = s->ec_w = s->qc_r = s->ec_r = nullptr;
    if (st != user_st) {   // back onto the caller's stream
        DX_CHECK_CUDA(cudaEventRecord(s->ev_end, st));
        DX_CHECK_CUDA(cudaStreamWaitEvent(user_st, s->ev_end, 0));
        st = user_st;
    }
    if (s->gs_out && g_forces) {   // frames after the last keyframe (zero gradients) and the sync
        for (int f = std::max(0, (std::min(N, last_key_state) + sub - 1) / sub); f < s->frames_done; ++f) stream_frame_grads(s, f, st);
        if (s->gs_mem == DXPBD_MEM_HOST) DX_CHECK_CUDA(cudaStreamSynchronize(s->cpy));
        s->gs_out = nullptr;
    }
    if (s->g_x0.n < (size_t)3 * V) s->g_x0.alloc((size_t)3 * V);
    if (s->g_v0.n < (size_t)3 * V) s->g_v0.alloc((size_t)3 * V);
    LAUNCH(DXPBD_K_ADJOINT, k_adjoint_final<<<nblk(V), kBlock, 0, st>>>(V, s->inv_mass.p, s->ax.p, s->y.p, state(s, 0), tgt(0), wts, s->dt,
                                                s->g_x0.p, s->g_v0.p));
    DX_CHECK_CUDA(cudaGetLastError());
    // loss to host
    double phi = 0.0;
    DX_CHECK_CUDA(cudaMemcpyAsync(s->h_scal, s->acc.p, sizeof(double), cudaMemcpyDeviceToHost, st));
    DX_CHECK_CUDA(cudaStreamSynchronize(st));
    phi = s->h_scal[0];
    if (gmode && solves > 0) {
        PcgCtl c;
        DX_CHECK_CUDA(cudaMemcpy(&c, s->pcg_ctl.p, sizeof(PcgCtl), cudaMemcpyDeviceToHost));
        total_it = (int)c.sum_it;
        max_it = c.max_it;
        worst = c.worst;
        launches += (int)c.execd * s->pcg_kernels_per_it + (s->use_tma && s->defer_u ? solves : 0);
        s->last_iters = max_it;
        if (c.fail) throw Err{DXPBD_ERR_SOLVE, "PCG did not converge within " + std::to_string(s->cg_max_iter) +
                                                  " iterations (worst relative residual " + std::to_string(c.worst) + ")"};
    }
    if (loss_out) *loss_out = (float)phi;
    s->stats[0] = total_it;
    // substeps of this backward whose blocks came from the forward's cache (no replay)
    {
        int nc_used = 0;
        for (int n = std::min(N, last_key_state) - 1; n >= 0; --n) nc_used += cached(n) ? 1 : 0;
        s->stats[15] = nc_used;
    }
    // PCG matvec launches that did work: one per iteration
    s->stats[14] = total_it;
    s->stats[1] = max_it;
    s->stats[3] = launches;
    s->stats[4] = solves;
    s->stats[5] = worst;
    s->stats[6] = phi;
    s->have_grads = true;
    DX_API_END
}

int dxpbd_grads(dxpbd_scene *s, int32_t kind, float *out, int64_t out_len, int32_t mem, void *stream) {
    DX_API_BEGIN
    DX_REQUIRE(s && out, DXPBD_ERR_ARG, "null argument");
    DX_REQUIRE(s->have_grads, DXPBD_ERR_STATE, "no backward has run since the last forward");
    DX_REQUIRE(kind >= 0 && kind < DXPBD_NUM_GRADS, DXPBD_ERR_ARG, "bad gradient kind");
    DX_REQUIRE((s->grad_flags >> kind) & 1 || kind == DXPBD_GRAD_X0 || kind == DXPBD_GRAD_V0, DXPBD_ERR_STATE,
               "gradient family not enabled in grad_flags");
    DX_CHECK_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = (cudaStream_t)stream;
    const int V = s->V;
    switch (kind) {
        case DXPBD_GRAD_COMPLIANCE: {
            DX_REQUIRE(out_len == s->E, DXPBD_ERR_ARG, "out_len must be E");
            if (!s->E) break;
            DBuf<float> tmp;
            tmp.alloc(s->E);
            k_scatter_f<<<nblk(s->E), kBlock, 0, st>>>(s->E, s->g_comp.p, s->d_perm.p, tmp.p);
            download(out, tmp.p, sizeof(float) * s->E, mem, st);
            DX_CHECK_CUDA(cudaStreamSynchronize(st));
            break;
        }
        case DXPBD_GRAD_X0:
        case DXPBD_GRAD_V0: {
            DX_REQUIRE(out_len == (int64_t)V * 3, DXPBD_ERR_ARG, "out_len must be 3V");
            const float *g = kind == DXPBD_GRAD_X0 ? s->g_x0.p : s->g_v0.p;
            if (mem == DXPBD_MEM_HOST) {
                k_scatter3<<<nblk(V), kBlock, 0, st>>>(V, 1, g, s->vperm.p, s->tmp3.p);
                download(out, s->tmp3.p, sizeof(float) * V * 3, mem, st);
            } else {
                k_scatter3<<<nblk(V), kBlock, 0, st>>>(V, 1, g, s->vperm.p, out);
            }
            break;
        }
        case DXPBD_GRAD_FORCES: {
            const int nf = std::max(s->frames_done, 1);
            DX_REQUIRE(out_len == (int64_t)nf * V * 3, DXPBD_ERR_ARG, "out_len must be frames*3V");
            if (mem == DXPBD_MEM_HOST) {
                for (int f = 0; f < nf; ++f) {
                    k_scatter3<<<nblk(V), kBlock, 0, st>>>(V, 1, s->g_force.p + (size_t)f * V * 3, s->vperm.p, s->tmp3.p);
                    download(out + (size_t)f * V * 3, s->tmp3.p, sizeof(float) * V * 3, mem, st);
                }
            } else {
                k_scatter3<<<nblk((int64_t)V * nf), kBlock, 0, st>>>(V, nf, s->g_force.p, s->vperm.p, out);
            }
            break;
        }
        case DXPBD_GRAD_SHAPE:
        case DXPBD_GRAD_SPHERE: {
            DBuf<float> gb, gs;
            gb.alloc(std::max(s->NS, 1));
            gs.alloc(std::max(4 * s->NSH, 1));
            k_shape_grad<<<nblk(std::max(s->NS, 4 * s->NSH) + 1), kBlock, 0, st>>>(s->NSH, s->NCAP, s->NS, s->acc.p + 1,
                                                                                  s->cap_Rb.p, s->cap_Lb.p, gb.p, gs.p);
            if (kind == DXPBD_GRAD_SHAPE) {
                DX_REQUIRE(out_len == s->NS, DXPBD_ERR_ARG, "out_len must be num_shape");
                download(out, gb.p, sizeof(float) * s->NS, mem, st);
            } else {
                DX_REQUIRE(out_len == 4 * s->NSH, DXPBD_ERR_ARG, "out_len must be 4S");
                download(out, gs.p, sizeof(float) * 4 * s->NSH, mem, st);
            }
            DX_CHECK_CUDA(cudaStreamSynchronize(st));
            break;
        }
        case DXPBD_GRAD_MATERIAL: {
            DX_REQUIRE(out_len == 2 * (int64_t)s->T, DXPBD_ERR_ARG, "out_len must be 2T");
            DBuf<float> tmp;
            tmp.alloc(2 * (size_t)s->T);
            k_scatter_pair<<<nblk(s->T), kBlock, 0, st>>>(s->T, s->t_g.p, s->t_perm.p, tmp.p);
            download(out, tmp.p, sizeof(float) * 2 * s->T, mem, st);
            DX_CHECK_CUDA(cudaStreamSynchronize(st));
            break;
        }
    }
    DX_API_END
}

int dxpbd_grads_stream(dxpbd_scene *s, int32_t kind, float *out, int64_t out_len, int32_t mem) {
    DX_API_BEGIN
    DX_REQUIRE(s && out, DXPBD_ERR_ARG, "null argument");
    DX_REQUIRE(kind == DXPBD_GRAD_FORCES, DXPBD_ERR_ARG, "streamed gradients: forces only");
    DX_REQUIRE((s->grad_flags >> DXPBD_GRAD_FORCES) & 1, DXPBD_ERR_STATE, "gradient family not enabled in grad_flags");
    DX_REQUIRE(s->frames_done >= 1, DXPBD_ERR_STATE, "no forward has run");
    DX_REQUIRE(out_len == (int64_t)s->frames_done * s->V * 3, DXPBD_ERR_ARG, "out_len must be frames*3V");
    s->gs_out = out;
    s->gs_mem = mem;
    DX_API_END
}

int dxpbd_set_params(dxpbd_scene *s, int32_t kind, const float *data, int64_t len, int32_t mem, void *stream) {
    DX_API_BEGIN
    if (s) s->qc_count = 0;   // cached blocks belong to the previous parameters
    DX_REQUIRE(s && data, DXPBD_ERR_ARG, "null argument");
    DX_CHECK_CUDA(cudaSetDevice(s->device));
    cudaStream_t st = (cudaStream_t)stream;
    switch (kind) {
        case DXPBD_PARAM_COMPLIANCE: {
            DX_REQUIRE(len == s->E, DXPBD_ERR_ARG, "len must be E");
            DBuf<float> tmp;
            tmp.alloc(std::max(s->E, 1));
            upload(tmp.p, data, sizeof(float) * s->E, mem, st);
            if (s->E) k_gather_f<<<nblk(s->E), kBlock, 0, st>>>(s->E, tmp.p, s->d_perm.p, s->d_alpha.p);
            DX_CHECK_CUDA(cudaStreamSynchronize(st));
            break;
        }
        case DXPBD_PARAM_SHAPE:
            DX_REQUIRE(len == s->NS, DXPBD_ERR_ARG, "len must be num_shape");
            upload(s->beta.p, data, sizeof(float) * s->NS, mem, st);
            apply_shape(s, st);
            break;
        case DXPBD_PARAM_SPHERES:
            DX_REQUIRE(len == 4 * s->NSH, DXPBD_ERR_ARG, "len must be 4S");
            upload(s->sph.p, data, sizeof(float) * 4 * s->NSH, mem, st);
            apply_shape(s, st);
            break;
        case DXPBD_PARAM_MATERIAL: {
            DX_REQUIRE(len == 2 * (int64_t)s->T, DXPBD_ERR_ARG, "len must be 2T");
            DBuf<float> tmp;
            tmp.alloc(2 * (size_t)s->T);
            upload(tmp.p, data, sizeof(float) * 2 * s->T, mem, st);
            k_gather_pair_split<<<nblk(s->T), kBlock, 0, st>>>(s->T, tmp.p, s->t_perm.p, s->t_a.p, s->t_b.p);
            DX_CHECK_CUDA(cudaStreamSynchronize(st));
            break;
        }
        default:
            throw Err{DXPBD_ERR_ARG, "bad parameter kind"};
    }
    DX_CHECK_CUDA(cudaStreamSynchronize(st));
    DX_API_END
}

int dxpbd_coloring(dxpbd_scene *s, int32_t family, int32_t *out, int64_t out_len, int32_t *num_colors) {
    DX_API_BEGIN
    DX_REQUIRE(s && out, DXPBD_ERR_ARG, "null argument");
    const std::vector<int32_t> &c = family == 0 ? s->dist_color_h : s->tet_color_h;
    DX_REQUIRE(out_len == (int64_t)c.size(), DXPBD_ERR_ARG, "out_len mismatch");
    std::memcpy(out, c.data(), sizeof(int32_t) * c.size());
    if (num_colors) *num_colors = family == 0 ? s->n_dist_colors : s->n_tet_colors;
    DX_API_END
}

int dxpbd_profile(dxpbd_scene *s, int32_t enable) {
    DX_API_BEGIN
    DX_REQUIRE(s, DXPBD_ERR_ARG, "null scene");
    DX_CHECK_CUDA(cudaSetDevice(s->device));
    DX_CHECK_CUDA(cudaDeviceSynchronize());
    s->prof = enable != 0;
    s->prof_rec.clear();
    s->ev_used = 0;
    DX_API_END
}

int dxpbd_kernel_times(dxpbd_scene *s, double *ms, double *count, int32_t n) {
    DX_API_BEGIN
    DX_REQUIRE(s && ms && count, DXPBD_ERR_ARG, "null argument");
    DX_CHECK_CUDA(cudaSetDevice(s->device));
    for (int k = 0; k < n; ++k) ms[k] = count[k] = 0.0;
    if (!s->prof_rec.empty()) DX_CHECK_CUDA(cudaEventSynchronize(s->ev_pool[s->prof_rec.back().second + 1]));
    for (auto &r : s->prof_rec) {
        float t = 0.f;
        DX_CHECK_CUDA(cudaEventElapsedTime(&t, s->ev_pool[r.second], s->ev_pool[r.second + 1]));
        if (r.first < n) { ms[r.first] += t; count[r.first] += 1; }
    }
    DX_API_END
}

int dxpbd_stats(dxpbd_scene *s, double *out, int32_t n) {
    DX_API_BEGIN
    DX_REQUIRE(s && out, DXPBD_ERR_ARG, "null argument");
    s->stats[7] = (double)s->n_foreign;
    s->stats[8] = (double)s->halo_total;
    s->stats[9] = (double)s->E;
    s->stats[10] = (double)s->V;
    s->stats[11] = (double)s->T;
    s->stats[12] = (double)s->ntiles;
    s->stats[13] = s->use_tma ? 1.0 : 0.0;
    const bool wave = s->wave_on && s->wave_nitems > 0;
    s->stats[16] = wave ? s->wave_ntw : 0;
    s->stats[17] = wave ? s->wave_nitems : 0;
    s->stats[18] = wave ? s->wave_L : 0;
    s->stats[19] = wave ? s->wave_maxnbr : 0;
    s->stats[20] = s->pull ? 1.0 : 0.0;
    s->stats[21] = s->use_tma ? (double)(s->d_Qt.n - 1) : 0.0;
    s->stats[22] = s->pull ? (double)s->d_pidx.n : 0.0;
    for (int k = 0; k < n && k < 24; ++k) out[k] = s->stats[k];
    DX_API_END
}

}  // extern "C"

#include "group.inc"

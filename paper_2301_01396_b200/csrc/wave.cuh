// Time-skewed (wavefront) Gauss-Seidel sweep: prediction + every distance color of one substep in
// ONE launch, so a band of tiles stays in L2 across all colors instead of the whole fp64 state
// being re-streamed from HBM once per color (k_wave).
//
// Work items are (wave tile w, phase p): p = 0 predicts the tile's own vertices (Eq. xpbdUpdateRule
// l.91, k_predict's arithmetic), p = 1 + c projects the tile's color-c distance constraints (Eq. xpbd
// l.81 / Eq. l.85, the same dist_core / dist_apply as k_dist_project1 / k_dist_replay1).  Item
// (w, p) may start once every neighbour w' of w -- a wave tile whose items touch a vertex that w's
// items touch, w itself included -- has finished phase p - 1.  That is exactly the order of the
// global color-by-color sweep (R1): a color is vertex-disjoint, so within a phase no two items
// share a vertex, and across phases every vertex sees its constraints in color order.  The iterates
// are therefore bit-identical to the per-color launches (test_wave_sweep_bit_identical).
//
// Scheduling: items are dispatched through one atomic ticket counter in the order of
// key = pi(w) + L p (pi = a bandwidth-reducing order of the wave-tile graph, L = 1 + its
// bandwidth), so every dependency of a ticket holds a smaller ticket.  Tickets are taken only by
// running CTAs, so the smallest unfinished ticket always has its dependencies finished: no deadlock
// for any grid size or residency (a persistent grid for the forward, one item per CTA for the
// replay that shares the GPU with the PCG).  Cross-CTA visibility: positions are read and written
// at L2 (ld/st .cg); an item ends with bar.sync + a release store (gpu scope, cumulative) of the
// tile's phase counter, the waiting CTA polls with acquire loads before its bar.sync.
// Locality: each key holds up to P = 1 + colors items, so a tile is live (in L2) for ~P L keys and
// the band of live tiles is ~P L tiles: pi is chosen for a small bandwidth (rows of tiles).  Lag:
// with L = 1 + bandwidth a dependency can hold a ticket just P before its dependant, i.e. still be
// in flight; the plan adds (resident CTAs) / P keys to L so that dependencies are normally finished
// when their dependants are dispatched.
#pragma once
#include "kernels.cuh"

namespace dx {

struct WavePlan {
    int ntw;               // wave tiles
    int W;                 // vertices per wave tile (g * kTileV)
    int nitems;            // ntw * (1 + colors)
    const int4 *desc;      // per ticket: {wave tile, phase, first sorted constraint, constraint count}
    const int2 *nrange;    // per ticket: range of the wave tile's neighbours in nbr
    const int *nbr;        // neighbour lists (self included)
    unsigned *flags;       // [ntw] phase counters (epoch-based, never reset)
    int *counter;          // ticket counter (zeroed before each launch)
};

struct WavePredict {       // k_predict's inputs
    const double4 *xn, *xprev;
    const float4 *v0;
    const float *f;
    double dt, inv_dt;
    float3 g;
};

struct WaveDist {          // constraint arrays (color-sorted) and replay outputs
    const int2 *idx;
    const float *rest, *alpha;
    float inv_dt2;
    int E;
    float4 *Q4;            // replay: block at tpos[j] (+ copy at fpos[j]); null: projection only
    float4 *fQ;
    float *eout;
    const int *tpos, *fpos;
};

DX_INLINE double4 ldcg_d4(const double4 *p) {
    const double2 a = __ldcg(reinterpret_cast<const double2 *>(p));
    const double2 b = __ldcg(reinterpret_cast<const double2 *>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}
DX_INLINE void stcg_d4(double4 *p, const double4 &v) {
    __stcg(reinterpret_cast<double2 *>(p), make_double2(v.x, v.y));
    __stcg(reinterpret_cast<double2 *>(p) + 1, make_double2(v.z, v.w));
}
DX_INLINE unsigned ld_acquire_u32(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
DX_INLINE void st_release_u32(unsigned *p, unsigned v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// L2 eviction-priority hints: the read-once streams (constraint data, the previous states, forces)
// and the write-once blocks are evict_first, so the iterate -- reused by the next phases of the
// band of tiles in flight -- keeps the L2.
DX_INLINE uint64_t l2_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
DX_INLINE int2 ldef(const int2 *a, uint64_t pol) {
    int2 v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.s32 {%0, %1}, [%2], %3;" : "=r"(v.x), "=r"(v.y) : "l"(a), "l"(pol));
    return v;
}
DX_INLINE float ldef(const float *a, uint64_t pol) {
    float v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(v) : "l"(a), "l"(pol));
    return v;
}
DX_INLINE int ldef(const int *a, uint64_t pol) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(a), "l"(pol));
    return v;
}
DX_INLINE void stef(float4 *a, float4 v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;" ::"l"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "l"(pol)
                 : "memory");
}
DX_INLINE void stef(float *a, float v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f32 [%0], %1, %2;" ::"l"(a), "f"(v), "l"(pol) : "memory");
}

// Constraint data of one pass (NB per thread): read-only, so it is loaded before the item's
// dependencies are satisfied -- for the next ticket while the current item computes.
template <int NB, bool REPLAY, int NT = kBlock>
struct WavePass {
    int2 e[NB];
    float rs[NB], al[NB];
    int tp[NB], fp[NB];
    DX_INLINE void load(const WaveDist &d, int begin, int count, int q0, uint64_t pol) {
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const int j = begin + max(0, min(q0 + (int)threadIdx.x + k * NT, count - 1));
            e[k] = ldef(d.idx + j, pol);
            rs[k] = ldef(d.rest + j, pol);
            al[k] = ldef(d.alpha + j, pol);
            if (REPLAY) {
                tp[k] = d.tpos ? ldef(d.tpos + j, pol) : j;
                fp[k] = d.fpos ? ldef(d.fpos + j, pol) : -1;
            }
        }
    }
};

// One pass: gather the endpoints (L2), project (dist_core / dist_apply), store iterate and blocks.
template <int NB, bool REPLAY, int NT>
DX_INLINE void wave_pass(const WavePass<NB, REPLAY, NT> &c, const WaveDist &d, int begin, int count, int q0, bool wx,
                         double4 *__restrict__ x, uint64_t pol) {
    double4 pa[NB], pb[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        pa[k] = ldcg_d4(x + c.e[k].x);
        pb[k] = ldcg_d4(x + c.e[k].y);
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const int q = q0 + (int)threadIdx.x + k * NT;
        if (q >= count) continue;
        const int j = begin + q;
        const float at = rmul(c.al[k], d.inv_dt2);
        DistCore o;
        const bool ok = dist_core(pa[k], pb[k], c.rs[k], at, 0.f, o);
        if (REPLAY) {
            float4 q4 = make_float4(0.f, 0.f, 0.f, 0.f);
            float3 ec = make_float3(0.f, 0.f, 0.f);
            if (ok) {
                q4 = qpack_iso_rank1(o.n, o.dl, (float)(1.0 / o.len), o.J);
                const float iJ = 1.f / o.J;
                const float tt = (-(0.f + o.dl) * d.inv_dt2 - at * 0.f) * iJ;
                ec = ec + tt * o.n;
            }
            stef(d.Q4 + c.tp[k], q4, pol);
            if (c.fp[k] >= 0) stef(d.fQ + c.fp[k], q4, pol);
            if (d.eout) {
                stef(d.eout + j, ec.x, pol);
                stef(d.eout + d.E + j, ec.y, pol);
                stef(d.eout + 2 * (size_t)d.E + j, ec.z, pol);
            }
        }
        if (ok && wx) {
            dist_apply(pa[k], pb[k], o);
            stcg_d4(x + c.e[k].x, pa[k]);
            stcg_d4(x + c.e[k].y, pb[k]);
        }
    }
}

// NB constraints per thread per pass, all loads of a pass hoisted (as k_dist_project1 /
// k_dist_replay1).  WRITE_LAST_X = false: the last color's iterate is not written (nothing reads it:
// replay without tets / contacts, as k_dist_replay1<.., false>).  Software pipeline per CTA: the
// next ticket, its descriptor and its first pass of constraint data are in flight while the current
// item waits and computes.
template <int NB, int MINB, bool REPLAY, bool WRITE_LAST_X, int NT = kBlock>
__global__ void __launch_bounds__(NT, MINB) k_wave(WavePlan w, unsigned base, int V, int ncol, WavePredict pr,
                                                      WaveDist d, double4 *__restrict__ x) {
    __shared__ int s_tk[2];
    const uint64_t pol = l2_evict_first();
    if (threadIdx.x == 0) s_tk[0] = atomicAdd(w.counter, 1);
    __syncthreads();
    int cur = s_tk[0], buf = 0;
    if (cur >= w.nitems) return;
    int4 it = w.desc[cur];
    WavePass<NB, REPLAY, NT> cd;
    if (it.y > 0) cd.load(d, it.z, it.w, 0, pol);
    while (true) {
        if (threadIdx.x == 0) s_tk[buf ^ 1] = atomicAdd(w.counter, 1);   // next ticket
        const int tw = it.x, p = it.y;
        if (p > 0 && threadIdx.x < 32) {   // wait: every neighbour has finished phase p - 1
            const unsigned need = base + (unsigned)p;
            const int2 nr = w.nrange[cur];
            for (int k = nr.x + (int)threadIdx.x; k < nr.y; k += 32) {
                const unsigned *fl = w.flags + w.nbr[k];
                while ((int)(ld_acquire_u32(fl) - need) < 0) __nanosleep(32);
            }
            __syncwarp();
        }
        __syncthreads();
        const int nxt = s_tk[buf ^ 1];
        const int4 nd = nxt < w.nitems ? w.desc[nxt] : make_int4(0, 0, 0, 0);
        if (p == 0) {
            const int v0 = tw * w.W, v1 = min(V, v0 + w.W);
            for (int i = v0 + (int)threadIdx.x; i < v1; i += NT) {
                const double4 o = predict_one(i, pr.xn, pr.xprev, pr.v0, pr.f, pr.dt, pr.inv_dt, pr.g);
                stcg_d4(x + i, o);
            }
        } else {
            const int begin = it.z, count = it.w;
            const bool wx = WRITE_LAST_X || p - 1 < ncol - 1;
            wave_pass<NB, REPLAY, NT>(cd, d, begin, count, 0, wx, x, pol);
            for (int q0 = NT * NB; q0 < count; q0 += NT * NB) {
                cd.load(d, begin, count, q0, pol);
                wave_pass<NB, REPLAY, NT>(cd, d, begin, count, q0, wx, x, pol);
            }
        }
        if (nd.y > 0) cd.load(d, nd.z, nd.w, 0, pol);   // next item's first pass (read-only data)
        __syncthreads();
        if (threadIdx.x == 0) st_release_u32(w.flags + tw, base + (unsigned)p + 1u);   // release: cumulative over the bar.sync
        if (nxt >= w.nitems) break;
        cur = nxt;
        it = nd;
        buf ^= 1;
    }
}

}  // namespace dx

// sm_100a kernels of the DiffXPBD hot path: forward substep, differentiable replay,
// matrix-free filtered PCG, adjoint recursion and gradient accumulation.
// Section / equation / line references are to PAPER.md (arXiv 2301.01396) and to the
// readings R1..R13 of DESIGN.md.
#pragma once
#include "common.cuh"

namespace dx {

constexpr int kBlock = 256;
constexpr float kEpsLen = 1e-9f;

// Collider record (R7).  type 0 = sphere (c, r), 1 = capsule (c, axis, r, L).
struct Collider {
    float4 c;   // center (w unused)
    float4 a;   // unit axis (capsule)
    float r;    // radius
    float L;    // segment length (capsule)
    int type;
    int scene;  // scene of a batch the collider acts on (-1: every scene)
};

// collider c acts on vertex v (batches: the vertex's scene; vsc null: one scene)
DX_INLINE bool acts_on(const Collider &cd, const int *__restrict__ vsc, int v) {
    return cd.scene < 0 || !vsc || vsc[v] == cd.scene;
}

// ============================================================================ predict
// x~ = x_n + dt v_n + dt^2 (g + w f)  for free vertices, x~ = x_n for pinned ones
// (Eq. xpbdUpdateRule l.91, R2).  v_n = (x_n - x_{n-1}) / dt exactly as the forward
// defines it (R9), or v0 at n = 0.  Writes x~ (w = inverse mass) into out.
DX_INLINE double4 predict_one(int i, const double4 *__restrict__ xn, const double4 *__restrict__ xprev,
                              const float4 *__restrict__ v0, const float *__restrict__ f, double dt, double inv_dt,
                              float3 g) {
    double4 x = xn[i];
    double3 v;
    if (xprev) {
        double4 p = xprev[i];
        v = make_double3(__dmul_rn(__dsub_rn(x.x, p.x), inv_dt), __dmul_rn(__dsub_rn(x.y, p.y), inv_dt),
                         __dmul_rn(__dsub_rn(x.z, p.z), inv_dt));
    } else {
        float4 q = v0[i];
        v = make_double3(q.x, q.y, q.z);
    }
    double4 o = x;
    if (x.w > 0.0) {
        double3 acc = make_double3(g.x, g.y, g.z);
        if (f) acc = make_double3(__fma_rn(x.w, (double)f[3 * i], acc.x), __fma_rn(x.w, (double)f[3 * i + 1], acc.y),
                                  __fma_rn(x.w, (double)f[3 * i + 2], acc.z));
        double dt2 = __dmul_rn(dt, dt);
        o.x = __fma_rn(dt2, acc.x, __fma_rn(dt, v.x, x.x));
        o.y = __fma_rn(dt2, acc.y, __fma_rn(dt, v.y, x.y));
        o.z = __fma_rn(dt2, acc.z, __fma_rn(dt, v.z, x.z));
    }
    return o;
}
__global__ void k_predict(int V, const double4 *__restrict__ xn, const double4 *__restrict__ xprev,
                          const float4 *__restrict__ v0, const float *__restrict__ f, double dt,
                          double inv_dt, float3 g, double4 *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    out[i] = predict_one(i, xn, xprev, v0, f, dt, inv_dt, g);
}

// ============================================================================ distance
// Shared projection core (Eq. xpbd l.81 scalar form, Eq. l.85): identical instruction
// sequence in the forward and in the replay (R9).  Returns false when skipped (R13).
struct DistCore {
    double3 d;    // x_a - x_b (fp64)
    double len;   // |d|
    float3 n;     // d / len
    float C;      // len - rest (evaluated in fp64)
    float J;      // w_a + w_b + at
    float dl;     // delta lambda
};

DX_INLINE bool dist_core(const double4 &pa, const double4 &pb, float rest, float at, float lam0, DistCore &o) {
    float wsum = radd((float)pa.w, (float)pb.w);
    if (!(wsum > 0.f)) return false;
    o.d = dsub3(d3(pa), d3(pb));
    o.len = __dsqrt_rn(ddot3(o.d, o.d));
    if (!(o.len > (double)kEpsLen)) return false;
    double il = __drcp_rn(o.len);
    o.n = make_float3((float)(o.d.x * il), (float)(o.d.y * il), (float)(o.d.z * il));
    o.C = (float)__dsub_rn(o.len, (double)rest);
    o.J = radd(wsum, at);
    o.dl = rdiv(rsub(-o.C, rmul(at, lam0)), o.J);
    return true;
}

// x_a += w_a n dl, x_b -= w_b n dl  (n in fp64 from d / len)
DX_INLINE void dist_apply(double4 &pa, double4 &pb, const DistCore &o) {
    double s = __ddiv_rn((double)o.dl, o.len);
    double sa = __dmul_rn(pa.w, s), sb = -__dmul_rn(pb.w, s);
    pa.x = __fma_rn(sa, o.d.x, pa.x); pa.y = __fma_rn(sa, o.d.y, pa.y); pa.z = __fma_rn(sa, o.d.z, pa.z);
    pb.x = __fma_rn(sb, o.d.x, pb.x); pb.y = __fma_rn(sb, o.d.y, pb.y); pb.z = __fma_rn(sb, o.d.z, pb.z);
}

// One color of the Gauss-Seidel sweep over distance constraints (R1): constraints
// [begin, begin+count) of the color-sorted arrays are vertex-disjoint.
template <bool READ_LAM, bool WRITE_LAM>
__global__ void __launch_bounds__(kBlock) k_dist_project(int begin, int count, const int2 *__restrict__ idx,
                                                         const float *__restrict__ rest,
                                                         const float *__restrict__ alpha, float inv_dt2,
                                                         float *__restrict__ lam, double4 *__restrict__ x) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    int j = begin + t;
    int2 e = idx[j];
    double4 pa = x[e.x], pb = x[e.y];
    float at = rmul(alpha[j], inv_dt2);
    float lam0 = READ_LAM ? lam[j] : 0.f;
    DistCore o;
    if (!dist_core(pa, pb, rest[j], at, lam0, o)) return;
    if (WRITE_LAM) lam[j] = radd(lam0, o.dl);
    dist_apply(pa, pb, o);
    x[e.x] = pa;
    x[e.y] = pb;
}

// Differentiable replay of one color (Sec.4.3 l.166-194, Sec.4.4; R3).  For a distance
// constraint grad C = [n, -n], H = [[K,-K],[-K,K]], K = (I - n n^T)/len, dJ/dx = 0, so every
// stencil quantity has the form [s, -s] and D_j = [[B,-B],[-B,B]] with
//   sigma_s = (-n - at sigma) / J          (a-part of d dlam / dx)
//   B += dl K + n sigma_s^T                (kept symmetrised, R5)
//   sigma += sigma_s
// compliance control u = alpha_j (dat/du = dJ/du = 1/dt^2, dC/du = 0):
//   t = (-(lam0 + dl)/dt^2 - at T) / J ;   e += t n ;   T += t
// After the last iteration: Q_j = psd(-B) (R5) and e_j are stored for the PCG / gradients.
struct DistScratch {   // per-constraint running state for iterations > 1 (SoA)
    float *lam, *sig, *B, *T, *e;   // lam[E], sig[3E], B[6E], T[E], e[3E]
};

// Q formats: QF = 0 symmetric 3x3 in 6 SoA arrays; QF = 1 (K = 1 with PD projection only) the exact
// closed form of psd(-B) for a single projection from lambda = 0: with sigma_s = -n/J,
// -B = n n^T / J - (dl/len)(I - n n^T), so Q = c I + s n n^T, c = max(-dl/len, 0), s = 1/J - c,
// stored as one float4 (u = n sqrt|s|, c with the sign of s; s < 0 implies c > 0).
DX_INLINE float4 qpack_iso_rank1(float3 n, float dl, float inv_len, float J) {
    float c = fmaxf(-dl * inv_len, 0.f);
    float sv = 1.f / J - c;
    float r = sqrtf(fabsf(sv));
    return make_float4(r * n.x, r * n.y, r * n.z, sv >= 0.f ? c : -c);
}
DX_INLINE float3 qmul_iso_rank1(float4 Q, float3 d) {
    float c = fabsf(Q.w);
    float3 u = make_float3(Q.x, Q.y, Q.z);
    float ud = dot3(u, d);
    if (Q.w < 0.f) ud = -ud;
    return make_float3(c * d.x + ud * u.x, c * d.y + ud * u.y, c * d.z + ud * u.z);
}

// K = 1 forward projection, NB constraints per thread: all index / endpoint loads are issued before
// any arithmetic (memory-level parallelism; the constraints of one color are vertex-disjoint, so
// a thread's loads never alias its stores).  Same arithmetic as k_dist_project<false, false>.
template <int NB>
__global__ void __launch_bounds__(kBlock) k_dist_project1(int begin, int count, const int2 *__restrict__ idx,
                                                          const float *__restrict__ rest,
                                                          const float *__restrict__ alpha, float inv_dt2,
                                                          double4 *__restrict__ x) {
    const int t0 = blockIdx.x * blockDim.x * NB + threadIdx.x;
    int2 e[NB];
    float rs[NB], al[NB];
    double4 pa[NB], pb[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const int t = t0 + k * blockDim.x;
        const int j = begin + min(t, count - 1);
        e[k] = idx[j];
        rs[k] = rest[j];
        al[k] = alpha[j];
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        pa[k] = x[e[k].x];
        pb[k] = x[e[k].y];
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        if (t0 + k * (int)blockDim.x >= count) continue;
        DistCore o;
        if (!dist_core(pa[k], pb[k], rs[k], rmul(al[k], inv_dt2), 0.f, o)) continue;
        dist_apply(pa[k], pb[k], o);
        x[e[k].x] = pa[k];
        x[e[k].y] = pb[k];
    }
}

// K = 1 replay with the PD projection (QF = 1), NB constraints per thread as above: regenerates the
// iterate, stores the closed-form block Q_j at its TMA-layout position tpos[j] (and the foreign copy),
// and the compliance control vector e_j = t n, t = -dl / (dt^2 J) (the general replay with
// lambda_0 = T = 0).  Same arithmetic as k_dist_replay<true, true, 1>.
template <int NB, int MINB = 1, bool WRITE_X = true>
__global__ void __launch_bounds__(kBlock, MINB) k_dist_replay1(int begin, int count, int E, const int2 *__restrict__ idx,
                                                         const float *__restrict__ rest,
                                                         const float *__restrict__ alpha, float inv_dt2,
                                                         float4 *__restrict__ Q4, float *__restrict__ eout,
                                                         double4 *__restrict__ x, const int *__restrict__ tpos,
                                                         const int *__restrict__ fpos, float4 *__restrict__ fQ) {
    const int t0 = blockIdx.x * blockDim.x * NB + threadIdx.x;
    int2 e[NB];
    float rs[NB], al[NB];
    int tp[NB], fp[NB];
    double4 pa[NB], pb[NB];
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const int t = t0 + k * blockDim.x;
        const int j = begin + min(t, count - 1);
        e[k] = idx[j];
        rs[k] = rest[j];
        al[k] = alpha[j];
        tp[k] = tpos ? tpos[j] : j;
        fp[k] = fpos ? fpos[j] : -1;
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        pa[k] = x[e[k].x];
        pb[k] = x[e[k].y];
    }
#pragma unroll
    for (int k = 0; k < NB; ++k) {
        const int t = t0 + k * blockDim.x;
        if (t >= count) continue;
        const int j = begin + t;
        const float at = rmul(al[k], inv_dt2);
        DistCore o;
        const bool ok = dist_core(pa[k], pb[k], rs[k], at, 0.f, o);
        float4 q4 = make_float4(0.f, 0.f, 0.f, 0.f);
        float3 ec = make_float3(0.f, 0.f, 0.f);
        if (ok) {
            q4 = qpack_iso_rank1(o.n, o.dl, (float)(1.0 / o.len), o.J);
            const float iJ = 1.f / o.J;
            const float tt = (-(0.f + o.dl) * inv_dt2 - at * 0.f) * iJ;
            ec = ec + tt * o.n;
            if (WRITE_X) {   // the last color's iterate is not read again (checkpoint x_{n+1} exists)
                dist_apply(pa[k], pb[k], o);
                x[e[k].x] = pa[k];
                x[e[k].y] = pb[k];
            }
        }
        Q4[tp[k]] = q4;
        if (fp[k] >= 0) fQ[fp[k]] = q4;
        if (eout) { eout[j] = ec.x; eout[E + j] = ec.y; eout[2 * E + j] = ec.z; }
    }
}

// Prediction fused into the first color of a K = 1 sweep: a color is vertex-disjoint, so the
// constraint's thread predicts its two endpoints itself (predict_one, the arithmetic of k_predict)
// instead of reading the x~ a separate pass stored -- one write and one read of the fp64 state less
// per substep, bit-identical iterates.  Vertices no color-0 constraint touches are predicted by
// k_predict_list.  Forward (REPLAY = false) and replay / block-caching forward (REPLAY = true, the
// arithmetic of k_dist_replay1).
struct PredictArgs {
    const double4 *xn, *xprev;
    const float4 *v0;
    const float *f;
    double dt, inv_dt;
    float3 g;
};
__global__ void k_predict_list(int n, const int *__restrict__ ids, PredictArgs P, double4 *__restrict__ out) {
    const int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int i = ids[k];
    out[i] = predict_one(i, P.xn, P.xprev, P.v0, P.f, P.dt, P.inv_dt, P.g);
}
template <bool REPLAY, int MINB>
__global__ void __launch_bounds__(kBlock, MINB) k_dist_first(int begin, int count, int E, const int2 *__restrict__ idx,
                                                             const float *__restrict__ rest,
                                                             const float *__restrict__ alpha, float inv_dt2,
                                                             PredictArgs P, float4 *__restrict__ Q4,
                                                             float *__restrict__ eout, double4 *__restrict__ x,
                                                             const int *__restrict__ tpos,
                                                             const int *__restrict__ fpos, float4 *__restrict__ fQ) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const int j = begin + t;
    const int2 e = idx[j];
    const float rs = rest[j], al = alpha[j];
    int tp = j, fp = -1;
    if (REPLAY) {
        if (tpos) tp = tpos[j];
        if (fpos) fp = fpos[j];
    }
    double4 pa = predict_one(e.x, P.xn, P.xprev, P.v0, P.f, P.dt, P.inv_dt, P.g);
    double4 pb = predict_one(e.y, P.xn, P.xprev, P.v0, P.f, P.dt, P.inv_dt, P.g);
    const float at = rmul(al, inv_dt2);
    DistCore o;
    const bool ok = dist_core(pa, pb, rs, at, 0.f, o);
    if (REPLAY) {
        float4 q4 = make_float4(0.f, 0.f, 0.f, 0.f);
        float3 ec = make_float3(0.f, 0.f, 0.f);
        if (ok) {
            q4 = qpack_iso_rank1(o.n, o.dl, (float)(1.0 / o.len), o.J);
            const float iJ = 1.f / o.J;
            const float tt = (-(0.f + o.dl) * inv_dt2 - at * 0.f) * iJ;
            ec = ec + tt * o.n;
        }
        Q4[tp] = q4;
        if (fp >= 0) fQ[fp] = q4;
        if (eout) { eout[j] = ec.x; eout[E + j] = ec.y; eout[2 * E + j] = ec.z; }
    }
    if (ok) dist_apply(pa, pb, o);
    x[e.x] = pa;
    x[e.y] = pb;
}

template <bool FIRST, bool LAST, int QF = 0>
__global__ void __launch_bounds__(kBlock) k_dist_replay(int begin, int count, int E, const int2 *__restrict__ idx,
                                                        const float *__restrict__ rest,
                                                        const float *__restrict__ alpha, float inv_dt2,
                                                        DistScratch sc, int pd, float *__restrict__ Qout,
                                                        float *__restrict__ eout, double4 *__restrict__ x,
                                                        const int *__restrict__ fpos = nullptr,
                                                        float4 *__restrict__ LQa = nullptr,
                                                        const int *__restrict__ tpos = nullptr,
                                                        float2 *__restrict__ LQb = nullptr) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    int j = begin + t;
    int2 ev = idx[j];
    double4 pa = x[ev.x], pb = x[ev.y];
    float at = rmul(alpha[j], inv_dt2);
    float lam0 = 0.f, T = 0.f;
    float3 sig = make_float3(0.f, 0.f, 0.f), ec = make_float3(0.f, 0.f, 0.f);
    Sym3 B = sym3_zero();
    if (!FIRST) {
        lam0 = sc.lam[j];
        T = sc.T[j];
        sig = make_float3(sc.sig[j], sc.sig[E + j], sc.sig[2 * E + j]);
        ec = make_float3(sc.e[j], sc.e[E + j], sc.e[2 * E + j]);
        B = Sym3{sc.B[j], sc.B[E + j], sc.B[2 * E + j], sc.B[3 * E + j], sc.B[4 * E + j], sc.B[5 * E + j]};
    }
    DistCore o;
    bool ok = dist_core(pa, pb, rest[j], at, lam0, o);
    if (ok) {
        float il = (float)(1.0 / o.len);
        float3 n = o.n;
        float iJ = 1.f / o.J;
        float3 ss = -iJ * (n + at * sig);
        sym3_add_perp(B, o.dl * il, n);
        sym3_add_symouter(B, n, ss);
        sig = sig + ss;
        float tt = (-(lam0 + o.dl) * inv_dt2 - at * T) * iJ;
        ec = ec + tt * n;
        T += tt;
        lam0 = radd(lam0, o.dl);
        dist_apply(pa, pb, o);
        x[ev.x] = pa;
        x[ev.y] = pb;
    }
    if (LAST) {
        Sym3 mB = Sym3{-B.xx, -B.xy, -B.xz, -B.yy, -B.yz, -B.zz};
        Sym3 Q = pd ? sym3_psd(mB) : mB;
        if (tpos) {   // TMA layout (general blocks: xx xy xz yy | yz zz), own-tile position + b-tile copy
            const float4 qa = make_float4(Q.xx, Q.xy, Q.xz, Q.yy);
            const float2 qb = make_float2(Q.yz, Q.zz);
            LQa[tpos[j]] = qa;
            LQb[tpos[j]] = qb;
            const int fp = fpos[j];
            if (fp >= 0) { LQa[fp] = qa; LQb[fp] = qb; }
        } else {
            Qout[j] = Q.xx; Qout[E + j] = Q.xy; Qout[2 * E + j] = Q.xz;
            Qout[3 * E + j] = Q.yy; Qout[4 * E + j] = Q.yz; Qout[5 * E + j] = Q.zz;
        }
        if (eout) { eout[j] = ec.x; eout[E + j] = ec.y; eout[2 * E + j] = ec.z; }
    } else {
        sc.lam[j] = lam0;
        sc.T[j] = T;
        sc.sig[j] = sig.x; sc.sig[E + j] = sig.y; sc.sig[2 * E + j] = sig.z;
        sc.e[j] = ec.x; sc.e[E + j] = ec.y; sc.e[2 * E + j] = ec.z;
        sc.B[j] = B.xx; sc.B[E + j] = B.xy; sc.B[2 * E + j] = B.xz;
        sc.B[3 * E + j] = B.yy; sc.B[4 * E + j] = B.yz; sc.B[5 * E + j] = B.zz;
    }
}

// ============================================================================ collisions
// C = |x - w(x)| - r - h against sphere center / closest capsule-segment point, applied only
// while C < 0 (R7).  Per free vertex, colliders in index order.
struct ContactCore {
    double3 d;   // x - witness (fp64)
    double len;
    float3 n;
    float C;
    float J;
    float dl;
    float s;     // (x - c).axis (capsule)
    int interior;
};

DX_INLINE bool contact_core(const double4 &p, const Collider &cd, float h, float at, float lam0, ContactCore &o) {
    double3 x = d3(p);
    double3 c = make_double3(cd.c.x, cd.c.y, cd.c.z);
    double3 wpt = c;
    o.interior = 0;
    o.s = 0.f;
    if (cd.type == 1) {
        double3 ax = make_double3(cd.a.x, cd.a.y, cd.a.z);
        double s = ddot3(dsub3(x, c), ax);
        double half = 0.5 * (double)cd.L;
        o.s = (float)s;
        o.interior = (s > -half) && (s < half);
        double tcl = fmin(fmax(s, -half), half);
        wpt = make_double3(__fma_rn(tcl, ax.x, c.x), __fma_rn(tcl, ax.y, c.y), __fma_rn(tcl, ax.z, c.z));
    }
    o.d = dsub3(x, wpt);
    o.len = __dsqrt_rn(ddot3(o.d, o.d));
    if (!(o.len > (double)kEpsLen)) return false;
    double Cd = __dsub_rn(__dsub_rn(o.len, (double)cd.r), (double)h);
    if (!(Cd < 0.0)) return false;
    double il = __drcp_rn(o.len);
    o.n = make_float3((float)(o.d.x * il), (float)(o.d.y * il), (float)(o.d.z * il));
    o.C = (float)Cd;
    o.J = radd((float)p.w, at);
    o.dl = rdiv(rsub(-o.C, rmul(at, lam0)), o.J);
    return true;
}

DX_INLINE void contact_apply(double4 &p, const ContactCore &o) {
    double sa = __dmul_rn(p.w, __ddiv_rn((double)o.dl, o.len));
    p.x = __fma_rn(sa, o.d.x, p.x); p.y = __fma_rn(sa, o.d.y, p.y); p.z = __fma_rn(sa, o.d.z, p.z);
}

template <bool READ_LAM, bool WRITE_LAM>
__global__ void __launch_bounds__(kBlock) k_contact_project(int V, int NC, const Collider *__restrict__ cols,
                                                            float h, float at, float *__restrict__ lam,
                                                            double4 *__restrict__ x, const int *__restrict__ vsc = nullptr) {
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    double4 p = x[v];
    if (!(p.w > 0.f)) return;
    bool moved = false;
    for (int c = 0; c < NC; ++c) {
        Collider cd = cols[c];
        float lam0 = READ_LAM ? lam[(size_t)c * V + v] : 0.f;
        ContactCore o;
        if (acts_on(cd, vsc, v) && contact_core(p, cd, h, at, lam0, o)) {
            if (WRITE_LAM) lam[(size_t)c * V + v] = radd(lam0, o.dl);
            contact_apply(p, o);
            moved = true;
        }
    }
    if (moved) x[v] = p;
}

// Differentiable replay of the contacts.  Per (collider c, vertex v): grad C = n, H = (I - n n^T
// - interior a a^T)/len, H M^-1 g = 0 (unit normal), so with sigma the running d dlam/dx:
//   sigma_s = (-n - at sigma)/J ;  B += dl H + n sigma_s^T ;  sigma += sigma_s
// Controls (dC/du, dn/du, dJ/du = 0, dat/du = 0; running T_u):
//   t_u = (-dC/du - at T_u)/J ;  e_u += dl dn/du + t_u n ;  T_u += t_u
//   sphere u = (c_x, c_y, c_z, r): dC/dc = -n, dC/dr = -1, dn/dc = -(I - n n^T)/len
//   capsule u = (r, L): dC/dr = -1; for the clamped ends dcp/dL = +-a/2:
//       dC/dL = -n.dcp/dL, dn/dL = -(I - n n^T) dcp/dL / len; interior: 0.
// The per-pair scratch layout: [c][v] for lam, T(4), sigma(3), B(6), e(12 = 4 params x 3).
// After the last iteration: Qc_v = Sum_c psd(-B_cv) (per-vertex 3x3, R5), e stored per pair.
struct ContactScratch {
    float *lam, *T, *sig, *B, *e;   // sizes NC*V*{1,4,3,6,12}
};

DX_INLINE void contact_deriv(const Collider &cd, const ContactCore &o, float at, float inv_len, float3 n,
                             float3 &sig, Sym3 &B, float (&T)[4], float (&e)[12]) {
    float iJ = 1.f / o.J;
    float3 ss = -iJ * (n + at * sig);
    // dl H
    sym3_add_perp(B, o.dl * inv_len, n);
    if (cd.type == 1 && o.interior) {
        float3 ax = f3(cd.a);
        float q = -o.dl * inv_len;
        B.xx += q * ax.x * ax.x; B.yy += q * ax.y * ax.y; B.zz += q * ax.z * ax.z;
        B.xy += q * ax.x * ax.y; B.xz += q * ax.x * ax.z; B.yz += q * ax.y * ax.z;
    }
    sym3_add_symouter(B, n, ss);
    sig = sig + ss;
    if (cd.type == 0) {
        // u = c_k (k = 0..2): dC/dc_k = -n_k ; dn/dc_k = -(e_k - n n_k)/len
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            float nk = k == 0 ? n.x : (k == 1 ? n.y : n.z);
            float tt = (nk - at * T[k]) * iJ;
            float3 ek = make_float3(k == 0 ? 1.f : 0.f, k == 1 ? 1.f : 0.f, k == 2 ? 1.f : 0.f);
            float3 dn = -inv_len * (ek - nk * n);
            float3 add = o.dl * dn + tt * n;
            e[3 * k] += add.x; e[3 * k + 1] += add.y; e[3 * k + 2] += add.z;
            T[k] += tt;
        }
        // u = r: dC/dr = -1, dn/dr = 0
        float tt = (1.f - at * T[3]) * iJ;
        e[9] += tt * n.x; e[10] += tt * n.y; e[11] += tt * n.z;
        T[3] += tt;
    } else {
        float tt = (1.f - at * T[0]) * iJ;   // u = r
        e[0] += tt * n.x; e[1] += tt * n.y; e[2] += tt * n.z;
        T[0] += tt;
        // u = L
        float sgn = o.interior ? 0.f : (o.s >= 0.f ? 0.5f : -0.5f);
        float3 ax = f3(cd.a);
        float3 dcp = sgn * ax;
        float dCdL = -dot3(n, dcp);
        float3 dn = -inv_len * (dcp - dot3(n, dcp) * n);
        float t2 = (-dCdL - at * T[1]) * iJ;
        float3 add = o.dl * dn + t2 * n;
        e[3] += add.x; e[4] += add.y; e[5] += add.z;
        T[1] += t2;
    }
}

template <bool FIRST, bool LAST>
__global__ void __launch_bounds__(kBlock) k_contact_replay(int V, int NC, const Collider *__restrict__ cols,
                                                           float h, float at, ContactScratch sc, int pd,
                                                           float *__restrict__ Qc, float *__restrict__ eout,
                                                           double4 *__restrict__ x, const int *__restrict__ vsc = nullptr) {
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    double4 p = x[v];
    if (!(p.w > 0.f)) {
        if (LAST) {   // pinned: zero block and zero controls (every output entry written each replay)
#pragma unroll
            for (int k = 0; k < 6; ++k) Qc[(size_t)k * V + v] = 0.f;
            if (eout)
                for (int c = 0; c < NC; ++c)
#pragma unroll
                    for (int k = 0; k < 12; ++k) eout[k * (size_t)NC * V + (size_t)c * V + v] = 0.f;
        }
        return;
    }
    Sym3 Qsum = sym3_zero();
    bool moved = false;
    const size_t NV = (size_t)NC * V;
    for (int c = 0; c < NC; ++c) {
        const Collider cd = cols[c];
        const size_t pr = (size_t)c * V + v;
        float lam0 = 0.f;
        float T[4] = {0.f, 0.f, 0.f, 0.f};
        float e[12];
#pragma unroll
        for (int k = 0; k < 12; ++k) e[k] = 0.f;
        float3 sig = make_float3(0.f, 0.f, 0.f);
        Sym3 B = sym3_zero();
        if (!FIRST) {
            lam0 = sc.lam[pr];
#pragma unroll
            for (int k = 0; k < 4; ++k) T[k] = sc.T[k * NV + pr];
#pragma unroll
            for (int k = 0; k < 12; ++k) e[k] = sc.e[k * NV + pr];
            sig = make_float3(sc.sig[pr], sc.sig[NV + pr], sc.sig[2 * NV + pr]);
            B = Sym3{sc.B[pr], sc.B[NV + pr], sc.B[2 * NV + pr], sc.B[3 * NV + pr], sc.B[4 * NV + pr],
                     sc.B[5 * NV + pr]};
        }
        ContactCore o;
        if (acts_on(cd, vsc, v) && contact_core(p, cd, h, at, lam0, o)) {
            float il = (float)(1.0 / o.len);
            float3 n = o.n;
            contact_deriv(cd, o, at, il, n, sig, B, T, e);
            lam0 = radd(lam0, o.dl);
            contact_apply(p, o);
            moved = true;
        }
        if (LAST) {
            Sym3 mB = Sym3{-B.xx, -B.xy, -B.xz, -B.yy, -B.yz, -B.zz};
            Sym3 Q = pd ? sym3_psd(mB) : mB;
            Qsum.xx += Q.xx; Qsum.xy += Q.xy; Qsum.xz += Q.xz;
            Qsum.yy += Q.yy; Qsum.yz += Q.yz; Qsum.zz += Q.zz;
            if (eout) {
#pragma unroll
                for (int k = 0; k < 12; ++k) eout[k * NV + pr] = e[k];
            }
        } else {
            sc.lam[pr] = lam0;
#pragma unroll
            for (int k = 0; k < 4; ++k) sc.T[k * NV + pr] = T[k];
#pragma unroll
            for (int k = 0; k < 12; ++k) sc.e[k * NV + pr] = e[k];
            sc.sig[pr] = sig.x; sc.sig[NV + pr] = sig.y; sc.sig[2 * NV + pr] = sig.z;
            sc.B[pr] = B.xx; sc.B[NV + pr] = B.xy; sc.B[2 * NV + pr] = B.xz;
            sc.B[3 * NV + pr] = B.yy; sc.B[4 * NV + pr] = B.yz; sc.B[5 * NV + pr] = B.zz;
        }
    }
    if (moved) x[v] = p;
    if (LAST) {
        Qc[v] = Qsum.xx; Qc[V + v] = Qsum.xy; Qc[2 * (size_t)V + v] = Qsum.xz;
        Qc[3 * (size_t)V + v] = Qsum.yy; Qc[4 * (size_t)V + v] = Qsum.yz; Qc[5 * (size_t)V + v] = Qsum.zz;
    }
}

// ============================================================================ PCG
// Filtered PCG (Sec.4.2.1) on (M + Sum_j Q_j)_free y = r (Eq. adjointXPBD, R4), matrix-free,
// preconditioner M (P^-1 = inverse mass; pinned rows filtered).  Scalars live in a per-iteration
// slot array sc[it*4 + {0: p.Ap, 1: r.z, 2: r.r}] (double) so no reset is ever needed:
// iteration `it` accumulates into slot it, reads slot it-1 (and slot "rz" of it-1).
// done-test: an iteration returns immediately if the previous residual met the tolerance.
// Device-side PCG control (graph mode): the iteration loop is a
// conditional WHILE node; the last block of each update kernel tests convergence, advances the
// iteration counter and sets the loop condition, so no host poll is needed.  Per-backward totals
// are accumulated here and read once at the end.
struct PcgCtl {
    unsigned blk;      // blocks of the current update launch that finished (last-block ticket)
    int it;            // iteration counter read by the kernels launched with it < 0
    int K;             // iterations of the last solve (read by k_cg_ufinal with K < 0)
    int fail;          // a solve reached max_iter without converging
    long long sum_it;  // sum of iterations over the solves of this backward
    int max_it;
    int solves;
    long long execd;   // iterations executed (launched loop bodies)
    double worst;      // largest final relative residual
};

// Graph mode: the pointers that change from substep to substep (the solution buffer rotates with
// the warm start, the block buffers alternate with the replay overlap / come from the forward's
// cache) are read from this device block, written by k_set_pcg_ptrs before each graph launch.
struct PcgPtrs {
    float3 *u;
    const float4 *Qt;   // TMA-layout blocks
    const float *Qc;    // contact blocks
    const float *tQ;    // tet blocks
};

struct CGState {
    double *sc;      // [(max_iter+2)*4]
    double *bnorm2;  // b.b (filtered)
    float tol2;
    PcgCtl *ctl = nullptr;                    // graph mode only
    cudaGraphConditionalHandle cond = 0;      // the WHILE node's condition
    int maxit = 0;
    const PcgPtrs *pp = nullptr;              // graph mode only
};

__global__ void k_set_pcg_ptrs(PcgPtrs *pp, PcgPtrs v) { *pp = v; }

// iteration index of a PCG kernel: its argument, or (graph mode, it < 0) the device counter
DX_INLINE int cg_iter(const CGState &s, int it) { return it >= 0 ? it : *(volatile int *)&s.ctl->it; }

// Graph mode, end of an update kernel (all threads of every block): the last block to finish reads
// the residual of iteration it + 1 (all blocks' reductions are visible after their fences), decides
// convergence exactly as the host poll does (rr <= tol2 |b|^2, K = first converged slot), advances
// the counter and sets the WHILE condition.
DX_INLINE void pcg_ctl_end(const CGState &s, int it) {
    __shared__ bool last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        last = atomicAdd(&s.ctl->blk, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last || threadIdx.x != 0) return;
    __threadfence();
    PcgCtl *c = s.ctl;
    c->blk = 0;
    const volatile double *sc = s.sc;
    const double bb = *(volatile double *)s.bnorm2, thr = (double)s.tol2 * bb;
    int K = -1;
    if (bb == 0.0) K = 0;
    else if (it == 0 && sc[2] <= thr) K = 0;             // the warm start already converged
    else if (sc[(it + 1) * 4 + 2] <= thr) K = it + 1;
    const bool stop = K >= 0 || it + 1 >= s.maxit;
    c->it = it + 1;
    if (stop) {
        c->execd += it + 1;
        if (K < 0) { c->fail = 1; K = s.maxit; }
        c->K = K;
        c->sum_it += K;
        c->max_it = max(c->max_it, K);
        c->solves += 1;
        if (bb > 0.0) c->worst = fmax(c->worst, sqrt(sc[min(K, s.maxit) * 4 + 2] / bb));
    }
    cudaGraphSetConditional(s.cond, stop ? 0u : 1u);
}

// a / b of two PCG scalars (double accumulators) as a float: one fp32 division when both are in the
// normal float range (always, in practice), else the fp64 division.  Every kernel forms alpha and
// beta with this, so the schedules stay bit-identical.
DX_INLINE float ratio_f(double a, double b) {
    const float af = (float)a, bf = (float)b;
    if (fabsf(bf) > 1e-30f && fabsf(bf) < 1e30f && fabsf(af) < 1e30f) return __fdiv_rn(af, bf);
    return (float)(a / b);
}

DX_INLINE bool cg_done(const CGState &s, int it) {
    // converged after iteration it-1 ?
    if (it == 0) return false;
    double rr = s.sc[(it - 1) * 4 + 2];
    return rr <= (double)s.tol2 * s.bnorm2[0];
}

// init: r = b (filtered), y = 0, p = M^-1 r ; slot[-1] rz = r.M^-1 r stored in sc[...] of "it=-1"
// we store it in slot 0 field 1 of a dedicated init slot: sc layout shifted by one (slot 0 = init).

// distance-constraint part of q += sgn * Sum_j P_j^T Q_j P_j p (pinned rows filtered), tiled:
// vertices are stored in Morton order; every constraint is oriented
// (a < b) and owned by the tile of a; within each color the constraints are sorted by owner tile,
// seg[c*(ntiles+1) + t] is the first constraint of color c owned by tile >= t.  One CTA per tile
// walks its segment of every color, accumulates q for its own vertices in shared memory and
// flushes each owned vertex with one vector reduction; only endpoints outside the tile (halo)
// use global reductions.  With DOT it also accumulates p.(A p) = Sum_j d^T Q_j d.
#ifndef DX_TILEV
#define DX_TILEV 512
#endif
constexpr int kTileV = DX_TILEV;   // vertices per Morton tile (a power of two: aligned lattice blocks)

template <int QF>
struct QVal {
    Sym3 A;
};
template <>
struct QVal<1> {
    float4 A;
};
template <int QF>
DX_INLINE QVal<QF> qload(const float *__restrict__ Q, int j, size_t E) {
    QVal<QF> v;
    if constexpr (QF == 1) {
        v.A = reinterpret_cast<const float4 *>(Q)[j];
    } else {
        v.A = Sym3{Q[j], Q[E + j], Q[2 * E + j], Q[3 * E + j], Q[4 * E + j], Q[5 * E + j]};
    }
    return v;
}
template <int QF>
DX_INLINE float3 qapply(const QVal<QF> &v, float3 d) {
    if constexpr (QF == 1) return qmul_iso_rank1(v.A, d);
    else return sym3_mul(v.A, d);
}
template <int QF>
DX_INLINE float3 qmul(const float *__restrict__ Q, int j, size_t E, float3 d) {
    if (QF == 1) return qmul_iso_rank1(reinterpret_cast<const float4 *>(Q)[j], d);
    const Sym3 A = Sym3{Q[j], Q[E + j], Q[2 * E + j], Q[3 * E + j], Q[4 * E + j], Q[5 * E + j]};
    return sym3_mul(A, d);
}

// Fused PCG iteration `it` (2 launches).  k_cg_matvec computes the new search direction
//   p_it = M^-1 r_it + beta_it p_{it-1}   (beta_it = rz_it / rz_{it-1}; p_0 = M^-1 r_0 from init)
// for its own vertices (stored to pbuf[it&1]) and on the fly for halo endpoints, then
//   q = M p + Qc p + Sum_j P_j^T Q_j P_j p
// for its own vertices completely: own constraints (a in tile) and "foreign" constraints (b in
// tile, a outside; fidx lists them per color) are walked color by color; within one color the
// constraints are vertex-disjoint (R1), so the shared-memory accumulation is a plain
// read-modify-write with one barrier per color and no atomics; q is stored once per vertex.
// p.q is accumulated over own vertices and own constraints only.
struct CGBufs {   // packed float3 (12 B) vector fields
    float3 *u, *r, *p0, *p1, *q, *qh;
};
struct TileLists {
    int ncol, ntiles;
    const int *seg;    // [ncol*(ntiles+1)] own-constraint ranges (sweep order)
    const int *fseg;   // [ncol*(ntiles+1)] ranges into fidx
    const int *fidx;   // foreign constraint ids
    const int4 *fent;  // foreign entries {j, a, b, 0} (same order as fidx)
};

DX_INLINE float3 halo_p(int it, int v, float beta, const float3 *__restrict__ r, const float3 *__restrict__ pold,
                        const float3 *__restrict__ pnew, const float *__restrict__ wv) {
    if (it == 0) return f3(pnew[v]);
    const float w = wv[v];
    if (!(w > 0.f)) return make_float3(0.f, 0.f, 0.f);
    const float3 rv = r[v], po = pold[v];
    return make_float3(w * rv.x + beta * po.x, w * rv.y + beta * po.y, w * rv.z + beta * po.z);
}

template <int QF>
__global__ void __launch_bounds__(kBlock) k_cg_matvec(int it, TileLists L, int V, const int2 *__restrict__ idx,
                                                      const float *__restrict__ Q, int E,
                                                      const float *__restrict__ Qc, CGBufs B,
                                                      const float *__restrict__ wv, CGState s) {
    it = cg_iter(s, it);
    if (s.pp) {
        const PcgPtrs pp = *s.pp;
        if (Qc) Qc = pp.Qc;
        B.u = pp.u;
    }
    if (cg_done(s, it + 1)) return;
    __shared__ float sp[3][kTileV];
    __shared__ float sq[3][kTileV];
    const int t = blockIdx.x;
    const int v0 = t * kTileV;
    const int nv = min(kTileV, V - v0);
    const float3 *__restrict__ pold = (it & 1) ? B.p0 : B.p1;   // p_{it-1}
    float3 *__restrict__ pnew = (it & 1) ? B.p1 : B.p0;         // p_it
    const float beta = it > 0 ? ratio_f(s.sc[it * 4 + 1], s.sc[(it - 1) * 4 + 1]) : 0.f;
    float acc[1] = {0.f};
    for (int i = threadIdx.x; i < kTileV; i += blockDim.x) {
        float3 pv = make_float3(0.f, 0.f, 0.f);
        float3 qv = make_float3(0.f, 0.f, 0.f);
        if (i < nv) {
            const int v = v0 + i;
            const float w = wv[v];
            if (it > 0) {
                if (w > 0.f) {
                    float3 rv = B.r[v], po = pold[v];
                    pv = make_float3(w * rv.x + beta * po.x, w * rv.y + beta * po.y, w * rv.z + beta * po.z);
                }
                pnew[v] = pv;
            } else {
                pv = pnew[v];
            }
            if (w > 0.f) {
                float3 pp = f3(pv);
                qv = (1.f / w) * pp;
                if (Qc) {
                    Sym3 A = Sym3{Qc[v], Qc[V + v], Qc[2 * (size_t)V + v], Qc[3 * (size_t)V + v],
                                  Qc[4 * (size_t)V + v], Qc[5 * (size_t)V + v]};
                    qv = qv + sym3_mul(A, pp);
                }
                acc[0] += dot3(pp, qv);
            }
        }
        sp[0][i] = pv.x;
        sp[1][i] = pv.y;
        sp[2][i] = pv.z;
        sq[0][i] = qv.x;
        sq[1][i] = qv.y;
        sq[2][i] = qv.z;
    }
    __syncthreads();
    const int stride = L.ntiles + 1;
    for (int c = 0; c < L.ncol; ++c) {
        const int b = L.seg[c * stride + t], e = L.seg[c * stride + t + 1];
        for (int j = b + threadIdx.x; j < e; j += blockDim.x) {
            const int2 ab = idx[j];
            const int la = ab.x - v0, lb = ab.y - v0;
            const bool bl = lb < nv;
            const float3 pa = make_float3(sp[0][la], sp[1][la], sp[2][la]);
            const float3 pb = bl ? make_float3(sp[0][lb], sp[1][lb], sp[2][lb]) : halo_p(it, ab.y, beta, B.r, pold, pnew, wv);
            const float3 d = pa - pb;
            const float3 y = qmul<QF>(Q, j, E, d);
            acc[0] += dot3(d, y);
            sq[0][la] += y.x;
            sq[1][la] += y.y;
            sq[2][la] += y.z;
            if (bl) {
                sq[0][lb] -= y.x;
                sq[1][lb] -= y.y;
                sq[2][lb] -= y.z;
            }
        }
        const int fb = L.fseg[c * stride + t], fe = L.fseg[c * stride + t + 1];
        for (int k = fb + threadIdx.x; k < fe; k += blockDim.x) {
            const int4 f4 = L.fent[k];   // {j, a, b}: b in tile, a outside
            const int lb = f4.z - v0;
            const float3 pa = halo_p(it, f4.y, beta, B.r, pold, pnew, wv);
            const float3 d = pa - make_float3(sp[0][lb], sp[1][lb], sp[2][lb]);
            const float3 y = qmul<QF>(Q, f4.x, E, d);
            sq[0][lb] -= y.x;
            sq[1][lb] -= y.y;
            sq[2][lb] -= y.z;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
        const int v = v0 + i;
        B.q[v] = wv[v] > 0.f ? make_float3(sq[0][i], sq[1][i], sq[2][i]) : make_float3(0.f, 0.f, 0.f);
    }
    block_reduce_add<1>(acc, s.sc + (it + 1) * 4 + 0);
}

// ---------------------------------------------------------------------------------------------
// TMA-staged tiled kernels (QF = 1).  CG-local tile structure (built at create, host
// tma_tile_layout):
//   every vertex a tile's constraints touch has a shared-memory slot: own vertices [0, kTileV),
//   halo vertices (outside the tile) [kTileV, kTileV + hcap); values are float4 (x, y, z, -) so one
//   16-byte access reads or writes a vertex.  Slots are assigned so that the endpoints of every
//   color segment spread evenly over the 8 sixteen-byte bank groups, and each segment is ordered in
//   groups of 8 entries (one quarter-warp access phase) with distinct bank groups per endpoint.
//   Per (tile, color) one combined segment (tile-major) holds the tile's own constraints (a in the
//   tile; b own or halo) and its foreign entries (b in the tile, a in another tile): cpair =
//   slot(a) | slot(b) << 16 and the block Q4 in the same order; the replay writes each block at
//   its own-tile position and, for cross-tile constraints, a copy at the b-tile position.
// Per color the combined segment is contiguous: one thread stages it with two bulk async copies
// (cp.async.bulk -> mbarrier complete_tx) kTmaStages colors ahead; all threads then work purely
// in shared memory (plain read-modify-write of the accumulator, one barrier per color,
// vertex-disjoint within a color by R1).
constexpr int kTmaStages = 3;
constexpr int kTmaThreads = kTileV / 2;                  // rhs kernel threads per tile
constexpr int kRhsMinB = kTileV >= 1024 ? 1 : 1536 / kTileV;   // its launch-bounds CTAs per SM (3 at 512)
constexpr int kMvThreads = kTileV / 2;                   // matvec threads per tile
constexpr int kMvMinB = 2048 / kTileV;                   // its resident CTAs per SM (64 registers)
constexpr int kMaxColors = 64;   // bounds table in shared memory (more colors: generic kernel)

struct TmaTiles {
    int ncol, ntiles, hcap;
    int cap;                         // stage capacity: largest combined segment
    const int4 *tseg;                // [tile][color]: combined segment [x, y) of cpair / Q4 (tile-major)
    const uint32_t *cpair;           // slot pairs (la | lb << 16); la >= kTileV marks a foreign entry
    const int *hpad;                 // [tile][hcap]: halo vertex ids, -1 padded (fixed stride)
    const float4 *Q4;                // blocks in the same layout (the replay writes both copies)
    const float2 *Q2;                // general blocks only (K > 1 or no PD): Q4 = (xx, xy, xz, yy), Q2 = (yz, zz);
                                     // null: Q4 is the K = 1 closed form c I + s n n^T
    const uint16_t *vslot;           // [tile][kTileV]: slot of own vertex i
    const uint16_t *hslot;           // [tile][hcap]: slot of halo entry h
};

// One stage (bytes, 16-aligned parts): q[cap] | cp[cap + 4, rounded to 16 bytes] | (general blocks)
// q2[cap + 2, rounded to 16 bytes]; `gen` is 1 for general blocks (TmaTiles::Q2 set)
__host__ __device__ inline uint32_t tma_stage_bytes(int cap, int gen = 0) {
    return (uint32_t)(16 * cap + ((4 * (cap + 4) + 15) & ~15) + (gen ? ((8 * (cap + 2) + 15) & ~15) : 0));
}
struct StageView {
    const float4 *q;
    const uint32_t *cp;
    const float2 *q2;
};
DX_INLINE StageView stage_view(unsigned char *base, int cap) {
    StageView v;
    v.q = reinterpret_cast<const float4 *>(base);
    v.cp = reinterpret_cast<const uint32_t *>(v.q + cap);
    v.q2 = reinterpret_cast<const float2 *>(base + 16 * cap + ((4 * (cap + 4) + 15) & ~15));
    return v;
}
// dynamic smem of the matvec: [bars 64][stages][sq float4 kTileV][sp float4 kTileV + hcap]
__host__ __device__ inline size_t tma_smem_bytes(int hcap, int cap, int gen = 0) {
    return 64 + (size_t)tma_stage_bytes(cap, gen) * kTmaStages + 16 * (size_t)kTileV + 16 * (size_t)(kTileV + hcap);
}
// rhs: [bars][stages][sqb, sqr float4 kTileV][sy, sz float4 kTileV + hcap]
__host__ __device__ inline size_t tma_rhs_smem_bytes(int hcap, int cap, int gen = 0) {
    return 64 + (size_t)tma_stage_bytes(cap, gen) * kTmaStages + 32 * (size_t)kTileV + 32 * (size_t)(kTileV + hcap);
}
// Q d for an entry: closed form (Q2 null) or general symmetric block
DX_INLINE float3 qmul_entry(const StageView &S, bool gen, int i, int off2, float3 d) {
    const float4 a = S.q[i];
    if (!gen) return qmul_iso_rank1(a, d);
    const float2 b = S.q2[off2 + i];
    return make_float3(a.x * d.x + a.y * d.y + a.z * d.z, a.y * d.x + a.w * d.y + b.x * d.z,
                       a.z * d.x + b.x * d.y + b.y * d.z);
}

DX_INLINE void tma_issue(uint64_t *bar, unsigned char *stage, int4 g, const TmaTiles &T) {
    const int b = g.x, e = g.y;
    if (e <= b) {   // empty segment: complete the phase without a transfer
        mbar_expect_tx(bar, 0);
        return;
    }
    const size_t c0 = ((size_t)b * 4) & ~(size_t)15, c1 = ((size_t)e * 4 + 15) & ~(size_t)15;
    size_t d0 = 0, d1 = 0;
    if (T.Q2) {
        d0 = ((size_t)b * 8) & ~(size_t)15;
        d1 = ((size_t)e * 8 + 15) & ~(size_t)15;
    }
    mbar_expect_tx(bar, (uint32_t)(c1 - c0) + (uint32_t)(e - b) * 16u + (uint32_t)(d1 - d0));
    const StageView S = stage_view(stage, T.cap);
    bulk_g2s((void *)S.cp, reinterpret_cast<const char *>(T.cpair) + c0, (uint32_t)(c1 - c0), bar);
    bulk_g2s((void *)S.q, T.Q4 + b, (uint32_t)(e - b) * 16u, bar);
    if (T.Q2) bulk_g2s((void *)S.q2, reinterpret_cast<const char *>(T.Q2) + d0, (uint32_t)(d1 - d0), bar);
}

DX_INLINE float3 xyz(float4 v) { return make_float3(v.x, v.y, v.z); }
DX_INLINE float4 f4of(float3 v) { return make_float4(v.x, v.y, v.z, 0.f); }

// Walk all colors of tile t: sq += A_dist sp; returns sp.(A_dist sp) over own constraints.  Entry
// (la, lb): own constraint if la < kTileV (a own; b own or halo), else a foreign entry (a halo,
// b own); only own slots are accumulated.
template <int NT>
DX_INLINE float tma_tile_colors(uint64_t *bars, unsigned char *stages, const float4 *sp, float4 *sq, const int4 *sb,
                                const TmaTiles &T) {
    float dotacc = 0.f;
    const uint32_t sbytes = tma_stage_bytes(T.cap, T.Q2 != nullptr);
    for (int c = 0; c < T.ncol; ++c) {
        const int st = c % kTmaStages;
        unsigned char *stage = stages + (size_t)st * sbytes;
        const StageView S = stage_view(stage, T.cap);
        mbar_wait(&bars[st], (uint32_t)((c / kTmaStages) & 1));
        const int4 g = sb[c];
        const int n = g.y - g.x, off = g.x & 3, off2 = g.x & 1;
        const bool gen = T.Q2 != nullptr;
        for (int i = threadIdx.x; i < n; i += NT) {
            const uint32_t pr = S.cp[off + i];
            const int la = pr & 0xffff, lb = pr >> 16;
            const float3 d = xyz(sp[la]) - xyz(sp[lb]);
            const float3 y = qmul_entry(S, gen, i, off2, d);
            if (la < kTileV) {
                dotacc += dot3(d, y);
                sq[la] = f4of(xyz(sq[la]) + y);
            }
            if (lb < kTileV) sq[lb] = f4of(xyz(sq[lb]) - y);
        }
        __syncthreads();
        // re-arm this stage for color c + kTmaStages: all reads of it completed before the barrier
        // (write-after-read across proxies is ordered by the barrier, as in a TMA consumer release);
        // issued from the last warp
        if (threadIdx.x == NT - 32 && c + kTmaStages < T.ncol) tma_issue(&bars[st], stage, sb[c + kTmaStages], T);
    }
    return dotacc;
}

// Fused PCG matvec (see k_cg_matvec): p_it update for own and halo vertices, q = A p, p.q.
// Round trip 1 loads everything that has no dependency (convergence flag, per-color ranges,
// halo ids, slots, inverse masses); round trip 2 the vector values and the first bulk copies.
// NT threads per CTA (a color's combined list is ~1.1 x kTileV / 2 entries: NT = 320 processes it
// in one pass), MINB resident CTAs per SM.
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_cg_matvec_tma(int it, TmaTiles T, int V,
                                                                  const float *__restrict__ Qc, CGBufs B,
                                                                  const float *__restrict__ wv, CGState s, int t0 = 0,
                                                                  float3 *__restrict__ ufix = nullptr) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    unsigned char *stages = smem_raw + 64;
    float4 *sq = reinterpret_cast<float4 *>(stages + (size_t)tma_stage_bytes(T.cap, T.Q2 != nullptr) * kTmaStages);
    float4 *sp = sq + kTileV;
    const int hcap = T.hcap;
    it = cg_iter(s, it);
    if (s.pp) {   // graph mode: this substep's buffers
        const PcgPtrs pp = *s.pp;
        T.Q4 = pp.Qt;
        if (Qc) Qc = pp.Qc;
        B.u = pp.u;
        if (ufix) ufix = pp.u;
    }
    const int t = blockIdx.x + t0;   // t0: first tile of a partition (domain decomposition)
    const int v0 = t * kTileV;
    const int nv = min(kTileV, V - v0);
    __shared__ int4 sb[kMaxColors];
    constexpr int NO = (kTileV + NT - 1) / NT, NH = (512 + NT - 1) / NT;
    // ---- round trip 1
    const bool done = cg_done(s, it + 1);
    if (threadIdx.x < T.ncol) sb[threadIdx.x] = T.tseg[(size_t)t * T.ncol + threadIdx.x];
    float wo[NO];
    int so[NO];
#pragma unroll
    for (int u = 0; u < NO; ++u) {
        const int i = threadIdx.x + u * NT;
        wo[u] = wv[min(v0 + i, V - 1)];
        so[u] = i < kTileV ? T.vslot[(size_t)t * kTileV + i] : 0;
    }
    int hv[NH], hs[NH];
#pragma unroll
    for (int u = 0; u < NH; ++u) {
        const int h = threadIdx.x + u * NT;
        hv[u] = h < hcap ? T.hpad[(size_t)t * hcap + h] : -1;
        hs[u] = h < hcap ? T.hslot[(size_t)t * hcap + h] : 0;
    }
    // own vector values need nothing from round trip 1: issued with it (early-exit launches after
    // convergence are rare with the host's poll schedule)
    const float3 *__restrict__ pold = (it & 1) ? B.p0 : B.p1;
    float3 *__restrict__ pnew = (it & 1) ? B.p1 : B.p0;
    float3 ro[NO], po[NO], uo[NO];
#pragma unroll
    for (int u = 0; u < NO; ++u) {
        const int v = min(v0 + (int)threadIdx.x + u * NT, V - 1);
        ro[u] = it > 0 ? B.r[v] : pnew[v];
        po[u] = it > 0 ? pold[v] : make_float3(0.f, 0.f, 0.f);
        uo[u] = (ufix && it > 0) ? ufix[v] : make_float3(0.f, 0.f, 0.f);   // deferred update, same batch
    }
    if (done) return;
    __syncthreads();
    if (threadIdx.x == NT - 32) {
        for (int k = 0; k < kTmaStages; ++k) mbar_init(&bars[k], 1);
        fence_mbar_init();
        const uint32_t sbytes = tma_stage_bytes(T.cap, T.Q2 != nullptr);
        for (int c = 0; c < min(kTmaStages, T.ncol); ++c) tma_issue(&bars[c], stages + (size_t)c * sbytes, sb[c], T);
    }
    // ---- round trip 2: halo values
    const float beta = it > 0 ? ratio_f(s.sc[it * 4 + 1], s.sc[(it - 1) * 4 + 1]) : 0.f;
    float alpha_prev = 0.f;
    if (ufix && it > 0) {
        const double pq = s.sc[it * 4 + 0];
        alpha_prev = pq > 0.0 ? ratio_f(s.sc[(it - 1) * 4 + 1], pq) : 0.f;
    }
    float acc[1] = {0.f};
    float hw[NH];
    float3 hr[NH], hp[NH];
#pragma unroll
    for (int u = 0; u < NH; ++u) {
        const int v = max(hv[u], 0);
        hw[u] = wv[v];
        hr[u] = it > 0 ? B.r[v] : pnew[v];
        hp[u] = it > 0 ? pold[v] : make_float3(0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < NO; ++u) {
        const int i = threadIdx.x + u * NT;
        float3 pv = make_float3(0.f, 0.f, 0.f);
        float3 qv = make_float3(0.f, 0.f, 0.f);
        if (i < nv) {
            const int v = v0 + i;
            const float w = wo[u];
            if (w > 0.f) {
                pv = it > 0 ? make_float3(w * ro[u].x + beta * po[u].x, w * ro[u].y + beta * po[u].y,
                                          w * ro[u].z + beta * po[u].z)
                            : ro[u];
                qv = (1.f / w) * pv;
                if (Qc) {
                    Sym3 A = Sym3{Qc[v], Qc[V + v], Qc[2 * (size_t)V + v], Qc[3 * (size_t)V + v],
                                  Qc[4 * (size_t)V + v], Qc[5 * (size_t)V + v]};
                    qv = qv + sym3_mul(A, pv);
                }
                acc[0] += dot3(pv, qv);
            }
            if (it > 0) pnew[v] = pv;
            if (ufix && it > 0) ufix[v] = uo[u] + alpha_prev * po[u];   // deferred u += alpha_{it-1} p_{it-1}
        }
        if (i < kTileV) {
            sp[so[u]] = f4of(pv);
            sq[so[u]] = f4of(qv);
        }
    }
#pragma unroll
    for (int u = 0; u < NH; ++u) {
        if (hv[u] >= 0) {
            float3 pv = make_float3(0.f, 0.f, 0.f);
            if (hw[u] > 0.f)
                pv = it > 0 ? make_float3(hw[u] * hr[u].x + beta * hp[u].x, hw[u] * hr[u].y + beta * hp[u].y,
                                          hw[u] * hr[u].z + beta * hp[u].z)
                            : f3(hr[u]);
            sp[hs[u]] = f4of(pv);
        }
    }
    for (int h = threadIdx.x + NH * NT; h < hcap; h += blockDim.x) {   // rare: large halos
        const int v = T.hpad[(size_t)t * hcap + h];
        if (v >= 0) sp[T.hslot[(size_t)t * hcap + h]] = f4of(halo_p(it, v, beta, B.r, pold, pnew, wv));
    }
    __syncthreads();
    acc[0] += tma_tile_colors<NT>(bars, stages, sp, sq, sb, T);
#pragma unroll
    for (int u = 0; u < NO; ++u) {
        const int i = threadIdx.x + u * NT;
        if (i < nv) B.q[v0 + i] = wo[u] > 0.f ? xyz(sq[so[u]]) : make_float3(0.f, 0.f, 0.f);
    }
    block_reduce_add<1>(acc, s.sc + (it + 1) * 4 + 0);
}

// rhs (warm start): b = M u - Q_n y + dphi, r0 = b - A_n (u + du); A_dist applied tile-locally
// with the same staging / slot layout as the matvec.
__global__ void __launch_bounds__(kTmaThreads, kRhsMinB) k_rhs_tma(TmaTiles T, int V, const float *__restrict__ Qc,
                                                            const float3 *__restrict__ u, const float3 *__restrict__ uprev,
                                                            const float3 *__restrict__ uprev2,
                                                            const float3 *__restrict__ y,
                                                            const double4 *__restrict__ xkey, const float *__restrict__ target,
                                                            const float *__restrict__ weights, const float *__restrict__ wv,
                                                            float3 *__restrict__ bout, float3 *__restrict__ r0out,
                                                            float3 *__restrict__ u0out, int t0 = 0,
                                                            float3 *__restrict__ p0out = nullptr, CGState cs = CGState{}) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    uint64_t *bars = reinterpret_cast<uint64_t *>(smem_raw);
    unsigned char *stages = smem_raw + 64;
    const uint32_t sbytes = tma_stage_bytes(T.cap, T.Q2 != nullptr);
    float4 *sqb = reinterpret_cast<float4 *>(stages + (size_t)sbytes * kTmaStages);
    float4 *sqr = sqb + kTileV;
    const int hcap = T.hcap;
    float4 *sy = sqr + kTileV;
    float4 *sz = sy + kTileV + hcap;
    const int t = blockIdx.x + t0;
    const int v0 = t * kTileV;
    const int nv = min(kTileV, V - v0);
    __shared__ int4 sb[kMaxColors];
    constexpr int NO = (kTileV + kTmaThreads - 1) / kTmaThreads, NH = 2;
    // ---- round trip 1: descriptors, slots, halo ids, inverse masses
    if (threadIdx.x < T.ncol) sb[threadIdx.x] = T.tseg[(size_t)t * T.ncol + threadIdx.x];
    float wo[NO];
    int so[NO];
#pragma unroll
    for (int k = 0; k < NO; ++k) {
        const int i = threadIdx.x + k * kTmaThreads;
        wo[k] = wv[min(v0 + i, V - 1)];
        so[k] = i < kTileV ? T.vslot[(size_t)t * kTileV + i] : 0;
    }
    int hv[NH], hs[NH];
#pragma unroll
    for (int k = 0; k < NH; ++k) {
        const int h = threadIdx.x + k * kTmaThreads;
        hv[k] = h < hcap ? T.hpad[(size_t)t * hcap + h] : -1;
        hs[k] = h < hcap ? T.hslot[(size_t)t * hcap + h] : 0;
    }
    __syncthreads();
    if (threadIdx.x == kTmaThreads - 32) {
        for (int k = 0; k < kTmaStages; ++k) mbar_init(&bars[k], 1);
        fence_mbar_init();
        for (int c = 0; c < min(kTmaStages, T.ncol); ++c) tma_issue(&bars[c], stages + (size_t)c * sbytes, sb[c], T);
    }
    // ---- round trip 2: all vector values of own and halo vertices in one batch
    const float3 z3 = make_float3(0.f, 0.f, 0.f);
    float3 yo[NO], uo[NO], po[NO], p2o[NO];
    double4 xo[NO];
    float3 to[NO];
    float Wo[NO];
#pragma unroll
    for (int k = 0; k < NO; ++k) {
        const int v = min(v0 + (int)threadIdx.x + k * kTmaThreads, V - 1);
        yo[k] = f3(y[v]);
        uo[k] = f3(u[v]);
        po[k] = f3(uprev[v]);
        p2o[k] = uprev2 ? f3(uprev2[v]) : z3;
        if (target) {
            xo[k] = xkey[v];
            to[k] = make_float3(target[3 * v], target[3 * v + 1], target[3 * v + 2]);
            Wo[k] = weights ? weights[v] : 1.f;
        }
    }
    float3 hy[NH], hu[NH], hp[NH], hp2[NH];
#pragma unroll
    for (int k = 0; k < NH; ++k) {
        const int v = max(hv[k], 0);
        hy[k] = f3(y[v]);
        hu[k] = f3(u[v]);
        hp[k] = f3(uprev[v]);
        hp2[k] = uprev2 ? f3(uprev2[v]) : z3;
    }
#pragma unroll
    for (int k = 0; k < NO; ++k) {
        const int i = threadIdx.x + k * kTmaThreads;
        float3 yv = z3, zv = z3, bb = z3, rr = z3;
        if (i < nv) {
            const int v = v0 + i;
            const float w = wo[k];
            yv = yo[k];
            const float3 uv = uo[k];
            // warm start u0 = u + dv: linear 2u_{n+1} - u_{n+2}, or quadratic 3u_{n+1} - 3u_{n+2} + u_{n+3}
            const float3 dv = uprev2 ? 2.f * uv - 3.f * po[k] + p2o[k] : uv - po[k];
            const float3 u0 = uv + dv;
            zv = yv + u0;
            u0out[v] = w > 0.f ? u0 : z3;
            if (w > 0.f) {
                bb = (1.f / w) * uv;
                rr = (-1.f / w) * dv;
                if (Qc) {
                    Sym3 A = Sym3{Qc[v], Qc[V + v], Qc[2 * (size_t)V + v], Qc[3 * (size_t)V + v],
                                  Qc[4 * (size_t)V + v], Qc[5 * (size_t)V + v]};
                    bb = bb - sym3_mul(A, yv);
                    rr = rr - sym3_mul(A, zv);
                }
                if (target) {
                    const double4 x = xo[k];
                    const float3 g = Wo[k] * make_float3((float)(x.x - to[k].x), (float)(x.y - to[k].y), (float)(x.z - to[k].z));
                    bb = bb + g;
                    rr = rr + g;
                }
            }
        }
        if (i >= kTileV) continue;
        const int si = so[k];
        sy[si] = f4of(yv);
        sz[si] = f4of(zv);
        sqb[si] = f4of(bb);
        sqr[si] = f4of(rr);
    }
#pragma unroll
    for (int k = 0; k < NH; ++k) {
        if (hv[k] < 0) continue;
        const float3 dh = uprev2 ? 2.f * hu[k] - 3.f * hp[k] + hp2[k] : hu[k] - hp[k];
        sy[hs[k]] = f4of(hy[k]);
        sz[hs[k]] = f4of(hy[k] + hu[k] + dh);
    }
    for (int h = threadIdx.x + NH * kTmaThreads; h < hcap; h += blockDim.x) {   // rare: large halos
        const int v = T.hpad[(size_t)t * hcap + h];
        if (v < 0) continue;
        const float3 uh = f3(u[v]);
        const float3 dh = uprev2 ? 2.f * uh - 3.f * f3(uprev[v]) + f3(uprev2[v]) : uh - f3(uprev[v]);
        const float3 yv = f3(y[v]);
        const int sh = T.hslot[(size_t)t * hcap + h];
        sy[sh] = f4of(yv);
        sz[sh] = f4of(yv + uh + dh);
    }
    __syncthreads();
    // b -= A_dist y, r0 -= A_dist z (same per-color scheme as tma_tile_colors)
    for (int c = 0; c < T.ncol; ++c) {
        const int st = c % kTmaStages;
        unsigned char *stage = stages + (size_t)st * sbytes;
        const StageView S = stage_view(stage, T.cap);
        mbar_wait(&bars[st], (uint32_t)((c / kTmaStages) & 1));
        const int4 g = sb[c];
        const int n = g.y - g.x, off = g.x & 3, off2 = g.x & 1;
        const bool gen = T.Q2 != nullptr;
        for (int i = threadIdx.x; i < n; i += kTmaThreads) {
            const uint32_t pr = S.cp[off + i];
            const int la = pr & 0xffff, lb = pr >> 16;
            const float3 qy = qmul_entry(S, gen, i, off2, xyz(sy[la]) - xyz(sy[lb]));
            const float3 qz = qmul_entry(S, gen, i, off2, xyz(sz[la]) - xyz(sz[lb]));
            if (la < kTileV) {
                sqb[la] = f4of(xyz(sqb[la]) - qy);
                sqr[la] = f4of(xyz(sqr[la]) - qz);
            }
            if (lb < kTileV) {
                sqb[lb] = f4of(xyz(sqb[lb]) + qy);
                sqr[lb] = f4of(xyz(sqr[lb]) + qz);
            }
        }
        __syncthreads();
        // re-arm the stage (write-after-read ordered by the barrier; see tma_tile_colors)
        if (threadIdx.x == kTmaThreads - 32 && c + kTmaStages < T.ncol) tma_issue(&bars[st], stage, sb[c + kTmaStages], T);
    }
    // epilogue; with p0out the PCG start is fused (k_cg_start): p_0 = M^-1 r_0, slot 0 gets r.z and
    // r.r, s.bnorm2 gets |b|^2
    float acc[3] = {0.f, 0.f, 0.f};
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
        const int v = v0 + i, si = T.vslot[(size_t)t * kTileV + i];
        const float w = wv[v];
        const bool fr = w > 0.f;
        const float3 bv = fr ? xyz(sqb[si]) : make_float3(0.f, 0.f, 0.f);
        const float3 rv = fr ? xyz(sqr[si]) : make_float3(0.f, 0.f, 0.f);
        bout[v] = bv;
        r0out[v] = rv;
        if (p0out) {
            p0out[v] = w * rv;
            const float r2 = dot3(rv, rv);
            acc[0] += w * r2;
            acc[1] += r2;
            acc[2] += dot3(bv, bv);
        }
    }
    if (p0out) {
        float a2[2] = {acc[0], acc[1]};
        block_reduce_add<2>(a2, cs.sc + 1);
        float bb[1] = {acc[2]};
        block_reduce_add<1>(bb, cs.bnorm2);
    }
}

// PCG start from the warm start: r = r0 (filtered), p_0 = M^-1 r; slot 0 gets r.z and r.r;
// the reference norm |b|^2 goes to s.bnorm2.
__global__ void k_cg_start(int V, const float3 *__restrict__ b, float3 *__restrict__ r, float3 *__restrict__ p,
                           const float *__restrict__ wv, CGState s) {
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    float acc[3] = {0.f, 0.f, 0.f};
    if (v < V) {
        const float w = wv[v];
        float3 rv = r[v], bv = b[v];
        if (!(w > 0.f)) rv = bv = make_float3(0.f, 0.f, 0.f);
        r[v] = rv;
        p[v] = make_float3(w * rv.x, w * rv.y, w * rv.z);
        const float r2 = rv.x * rv.x + rv.y * rv.y + rv.z * rv.z;
        acc[0] = w * r2;
        acc[1] = r2;
        acc[2] = bv.x * bv.x + bv.y * bv.y + bv.z * bv.z;
    }
    float a2[2] = {acc[0], acc[1]};
    block_reduce_add<2>(a2, s.sc + 1);
    float bb[1] = {acc[2]};
    block_reduce_add<1>(bb, s.bnorm2);
}

// Generic (non-TMA) version of k_rhs_tma: writes b and the warm-start residual r0.
template <int QF>
__global__ void __launch_bounds__(kBlock) k_rhs_tiled(TileLists L, int V, const int2 *__restrict__ idx,
                                                      const float *__restrict__ Q, int E, const float *__restrict__ Qc,
                                                      const float3 *__restrict__ u, const float3 *__restrict__ uprev,
                                                      const float3 *__restrict__ y,
                                                      const double4 *__restrict__ xkey, const float *__restrict__ target,
                                                      const float *__restrict__ weights, const float *__restrict__ wv,
                                                      float3 *__restrict__ bout, float3 *__restrict__ r0out,
                                                      float3 *__restrict__ u0out) {
    __shared__ float sy[3][kTileV], sz[3][kTileV], sqb[3][kTileV], sqr[3][kTileV];
    const int t = blockIdx.x;
    const int v0 = t * kTileV;
    const int nv = min(kTileV, V - v0);
    for (int i = threadIdx.x; i < kTileV; i += blockDim.x) {
        float3 yv = make_float3(0.f, 0.f, 0.f), zv = yv, bb = yv, rr = yv;
        if (i < nv) {
            const int v = v0 + i;
            const float w = wv[v];
            yv = f3(y[v]);
            const float3 uv = f3(u[v]);
            const float3 dv = uv - f3(uprev[v]);          // warm start u0 = u + (u - uprev)
            const float3 u0 = uv + dv;
            zv = yv + u0;
            u0out[v] = w > 0.f ? u0 : make_float3(0.f, 0.f, 0.f);
            if (w > 0.f) {
                bb = (1.f / w) * uv;
                rr = (-1.f / w) * dv;
                if (Qc) {
                    Sym3 A = Sym3{Qc[v], Qc[V + v], Qc[2 * (size_t)V + v], Qc[3 * (size_t)V + v],
                                  Qc[4 * (size_t)V + v], Qc[5 * (size_t)V + v]};
                    bb = bb - sym3_mul(A, yv);
                    rr = rr - sym3_mul(A, zv);
                }
                if (target) {
                    double4 x = xkey[v];
                    float W = weights ? weights[v] : 1.f;
                    float3 g = W * make_float3((float)(x.x - target[3 * v]), (float)(x.y - target[3 * v + 1]),
                                               (float)(x.z - target[3 * v + 2]));
                    bb = bb + g;
                    rr = rr + g;
                }
            }
        }
        sy[0][i] = yv.x; sy[1][i] = yv.y; sy[2][i] = yv.z;
        sz[0][i] = zv.x; sz[1][i] = zv.y; sz[2][i] = zv.z;
        sqb[0][i] = bb.x; sqb[1][i] = bb.y; sqb[2][i] = bb.z;
        sqr[0][i] = rr.x; sqr[1][i] = rr.y; sqr[2][i] = rr.z;
    }
    __syncthreads();
    const int stride = L.ntiles + 1;
    for (int c = 0; c < L.ncol; ++c) {
        const int bb0 = L.seg[c * stride + t], e = L.seg[c * stride + t + 1];
        for (int j = bb0 + threadIdx.x; j < e; j += blockDim.x) {
            const int2 ab = idx[j];
            const int la = ab.x - v0, lb = ab.y - v0;
            const bool bl = lb < nv;
            float3 yb, zb;
            if (bl) {
                yb = make_float3(sy[0][lb], sy[1][lb], sy[2][lb]);
                zb = make_float3(sz[0][lb], sz[1][lb], sz[2][lb]);
            } else {
                yb = f3(y[ab.y]);
                const float3 ub = f3(u[ab.y]);
                zb = yb + ub + (ub - f3(uprev[ab.y]));
            }
            const float3 qy = qmul<QF>(Q, j, E, make_float3(sy[0][la], sy[1][la], sy[2][la]) - yb);
            const float3 qz = qmul<QF>(Q, j, E, make_float3(sz[0][la], sz[1][la], sz[2][la]) - zb);
            sqb[0][la] -= qy.x; sqb[1][la] -= qy.y; sqb[2][la] -= qy.z;
            sqr[0][la] -= qz.x; sqr[1][la] -= qz.y; sqr[2][la] -= qz.z;
            if (bl) {
                sqb[0][lb] += qy.x; sqb[1][lb] += qy.y; sqb[2][lb] += qy.z;
                sqr[0][lb] += qz.x; sqr[1][lb] += qz.y; sqr[2][lb] += qz.z;
            }
        }
        const int fb = L.fseg[c * stride + t], fe = L.fseg[c * stride + t + 1];
        for (int k2 = fb + threadIdx.x; k2 < fe; k2 += blockDim.x) {
            const int4 f4 = L.fent[k2];   // {j, a, b}: b in tile
            const int lb = f4.z - v0;
            const float3 ua = f3(u[f4.y]);
            const float3 ya = f3(y[f4.y]), za = ya + ua + (ua - f3(uprev[f4.y]));
            const float3 qy = qmul<QF>(Q, f4.x, E, ya - make_float3(sy[0][lb], sy[1][lb], sy[2][lb]));
            const float3 qz = qmul<QF>(Q, f4.x, E, za - make_float3(sz[0][lb], sz[1][lb], sz[2][lb]));
            sqb[0][lb] += qy.x; sqb[1][lb] += qy.y; sqb[2][lb] += qy.z;
            sqr[0][lb] += qz.x; sqr[1][lb] += qz.y; sqr[2][lb] += qz.z;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < nv; i += blockDim.x) {
        const int v = v0 + i;
        const bool fr = wv[v] > 0.f;
        bout[v] = fr ? make_float3(sqb[0][i], sqb[1][i], sqb[2][i]) : make_float3(0.f, 0.f, 0.f);
        r0out[v] = fr ? make_float3(sqr[0][i], sqr[1][i], sqr[2][i]) : make_float3(0.f, 0.f, 0.f);
    }
}


// Vectorized PCG update: 4 vertices per thread read as 3 float4 per field of the packed float3
// arrays (16-byte accesses): u += alpha p (unless deferred to the next matvec), r -= alpha q,
// r.M^-1 r and r.r into slot it+1; the V % 4 tail vertices by one extra thread.
template <bool UPD_U>
__global__ void k_cg_update4(int V, int it, CGBufs B, const float *__restrict__ wv, CGState s) {
    it = cg_iter(s, it);
    if (s.pp) B.u = s.pp->u;
    if (cg_done(s, it + 1)) {
        if (s.ctl) pcg_ctl_end(s, it);
        return;
    }
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    const int nq = V / 4;
    float acc[2] = {0.f, 0.f};
    if (t < nq) {
        const float4 *__restrict__ p = reinterpret_cast<const float4 *>((it & 1) ? B.p1 : B.p0);
        float4 *__restrict__ u = reinterpret_cast<float4 *>(B.u);
        float4 *__restrict__ r = reinterpret_cast<float4 *>(B.r);
        const float4 *__restrict__ q = reinterpret_cast<const float4 *>(B.q);
        const double pq = s.sc[(it + 1) * 4 + 0];
        const float alpha = pq > 0.0 ? ratio_f(s.sc[it * 4 + 1], pq) : 0.f;
        const float4 w4 = reinterpret_cast<const float4 *>(wv)[t];
        const float w[4] = {w4.x, w4.y, w4.z, w4.w};
        float uu[12], rr[12], pp[12], qq[12];
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const float4 a = UPD_U ? u[3 * t + c] : make_float4(0.f, 0.f, 0.f, 0.f), b = r[3 * t + c],
                         cc = UPD_U ? p[3 * t + c] : a, d = q[3 * t + c];
            uu[4 * c] = a.x; uu[4 * c + 1] = a.y; uu[4 * c + 2] = a.z; uu[4 * c + 3] = a.w;
            rr[4 * c] = b.x; rr[4 * c + 1] = b.y; rr[4 * c + 2] = b.z; rr[4 * c + 3] = b.w;
            pp[4 * c] = cc.x; pp[4 * c + 1] = cc.y; pp[4 * c + 2] = cc.z; pp[4 * c + 3] = cc.w;
            qq[4 * c] = d.x; qq[4 * c + 1] = d.y; qq[4 * c + 2] = d.z; qq[4 * c + 3] = d.w;
        }
#pragma unroll
        for (int k = 0; k < 12; ++k) {
            uu[k] += alpha * pp[k];
            rr[k] = (w[k / 3] > 0.f) ? rr[k] - alpha * qq[k] : 0.f;
            const float r2 = rr[k] * rr[k];
            acc[0] += w[k / 3] * r2;
            acc[1] += r2;
        }
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            if (UPD_U) u[3 * t + c] = make_float4(uu[4 * c], uu[4 * c + 1], uu[4 * c + 2], uu[4 * c + 3]);
            r[3 * t + c] = make_float4(rr[4 * c], rr[4 * c + 1], rr[4 * c + 2], rr[4 * c + 3]);
        }
    } else if (t == nq) {   // tail vertices
        for (int v = 4 * nq; v < V; ++v) {
            const float3 *__restrict__ p = (it & 1) ? B.p1 : B.p0;
            const double pq = s.sc[(it + 1) * 4 + 0];
            const float alpha = pq > 0.0 ? ratio_f(s.sc[it * 4 + 1], pq) : 0.f;
            const float w = wv[v];
            float3 uv = B.u[v], rv = B.r[v], pv = p[v], qv = B.q[v];
            uv = uv + alpha * pv;
            rv = w > 0.f ? rv - alpha * qv : make_float3(0.f, 0.f, 0.f);
            if (UPD_U) B.u[v] = uv;
            B.r[v] = rv;
            const float r2 = dot3(rv, rv);
            acc[0] += w * r2;
            acc[1] += r2;
        }
    }
    block_reduce_add<2>(acc, s.sc + (it + 1) * 4 + 1);
    if (s.ctl) pcg_ctl_end(s, it);
}

// Deferred solution update (UPD_U = false above): the matvec of iteration it adds
// alpha_{it-1} p_{it-1} to u in its vertex phase; after convergence at K iterations this adds the
// last term alpha_{K-1} p_{K-1}.
__global__ void k_cg_ufinal(int V, int K, CGBufs B, CGState s) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (K < 0) {   // graph mode: the solve's iteration count and solution buffer
        K = s.ctl->K;
        B.u = s.pp->u;
    }
    if (v >= V || K <= 0) return;
    const double pq = s.sc[K * 4 + 0];
    const float alpha = pq > 0.0 ? ratio_f(s.sc[(K - 1) * 4 + 1], pq) : 0.f;
    const float3 *__restrict__ p = ((K - 1) & 1) ? B.p1 : B.p0;
    B.u[v] = B.u[v] + alpha * p[v];
}

// after the solve: y_n = y_{n+1} + u_n ; dphi/df_frame += dt^2 y_n (R8)
__global__ void k_adjoint_accum(int V, const float *__restrict__ wv, const float3 *__restrict__ u,
                                float3 *__restrict__ y, float *__restrict__ gforce, float dt) {
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    if (!(wv[v] > 0.f)) return;
    float3 uv = u[v], yv = y[v];
    yv.x += uv.x; yv.y += uv.y; yv.z += uv.z;
    y[v] = yv;
    if (gforce) {
        float dt2 = dt * dt;
        gforce[3 * v] += dt2 * yv.x;
        gforce[3 * v + 1] += dt2 * yv.y;
        gforce[3 * v + 2] += dt2 * yv.z;
    }
}

// dphi/dx_0 = xbar_0 = M u_0 + dphi/dx_0(direct) ; dphi/dv_0 = vbar_0 = dt M y_0   (Eq. rawAdjoint)
__global__ void k_adjoint_final(int V, const float *__restrict__ wv, const float3 *__restrict__ u,
                                const float3 *__restrict__ y, const double4 *__restrict__ x0,
                                const float *__restrict__ target, const float *__restrict__ weights, float dt,
                                float *__restrict__ gx0, float *__restrict__ gv0) {
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    float w = wv[v];
    float3 gx = make_float3(0.f, 0.f, 0.f), gv = gx;
    if (w > 0.f) {
        float m = 1.f / w;
        gx = m * f3(u[v]);
        if (target) {
            double4 x = x0[v];
            float W = weights ? weights[v] : 1.f;
            gx = gx + W * make_float3((float)(x.x - target[3 * v]), (float)(x.y - target[3 * v + 1]),
                                      (float)(x.z - target[3 * v + 2]));
        }
        gv = (dt * m) * f3(y[v]);
    }
    gx0[3 * v] = gx.x; gx0[3 * v + 1] = gx.y; gx0[3 * v + 2] = gx.z;
    gv0[3 * v] = gv.x; gv0[3 * v + 1] = gv.y; gv0[3 * v + 2] = gv.z;
}

// phi += 1/2 Sum_v W_v |x_v - target_v|^2 (all vertices, R10)
__global__ void k_loss(int V, const double4 *__restrict__ x, const float *__restrict__ target,
                       const float *__restrict__ weights, double *acc) {
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    float a[1] = {0.f};
    if (v < V) {
        double4 p = x[v];
        float W = weights ? weights[v] : 1.f;
        float dx = (float)(p.x - target[3 * v]), dy = (float)(p.y - target[3 * v + 1]),
              dz = (float)(p.z - target[3 * v + 2]);
        a[0] = 0.5f * W * (dx * dx + dy * dy + dz * dz);
    }
    block_reduce_add<1>(a, acc);
}

// dphi/dalpha_j += e_j . (y_a - y_b)   (Eq. gradientRule; e_j is the a-part of M dDx/dalpha_j)
__global__ void k_grad_compliance(int E, const int2 *__restrict__ idx, const float *__restrict__ e,
                                  const float3 *__restrict__ y, float *__restrict__ g) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= E) return;
    int2 id = idx[j];
    float3 d = f3(y[id.x]) - f3(y[id.y]);
    g[j] += e[j] * d.x + e[E + j] * d.y + e[2 * (size_t)E + j] * d.z;
}

// collider parameter gradients: acc[c*4 + u] += Sum_v e_{c,v,u} . y_v
__global__ void k_grad_colliders(int V, int NC, const float *__restrict__ e, const float3 *__restrict__ y,
                                 double *acc) {
    int v = blockIdx.x * blockDim.x + threadIdx.x;
    const size_t NV = (size_t)NC * V;
    for (int c = 0; c < NC; ++c) {
        float a[4] = {0.f, 0.f, 0.f, 0.f};
        if (v < V) {
            float3 yv = f3(y[v]);
            size_t pr = (size_t)c * V + v;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                a[u] = e[(3 * u) * NV + pr] * yv.x + e[(3 * u + 1) * NV + pr] * yv.y + e[(3 * u + 2) * NV + pr] * yv.z;
        }
        block_reduce_add<4>(a, acc + 4 * c);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------------------------
// Domain decomposition (in-process partition group, dxpbd_group_*): halo exchange between the
// partitions' copies of a vertex or block array (dst[ids[i]] = src[ids[i]]) and the all-reduce
// of the PCG scalar slots (sum over partitions, written back to every partition).
template <class T>
__global__ void k_xchg(int n, const int *__restrict__ ids, const T *__restrict__ src, T *__restrict__ dst) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const int k = ids[i];
        dst[k] = src[k];
    }
}
__global__ void k_slot_allreduce(int P, double *const *__restrict__ slots, int off, int count) {
    const int i = threadIdx.x;
    if (i >= count) return;
    double sum = 0.0;
    for (int p = 0; p < P; ++p) sum += slots[p][off + i];
    for (int p = 0; p < P; ++p) slots[p][off + i] = sum;
}


}  // namespace dx

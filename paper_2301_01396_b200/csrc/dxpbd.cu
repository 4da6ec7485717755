// C-ABI of the B200-native DiffXPBD hot path (include/dxpbd.h).
// Host side: scene construction (greedy coloring, color-sorted SoA buffers), the forward
// substep loop with checkpoints, the backward loop (replay -> PCG -> adjoint update ->
// gradients).  Every arithmetic step of the path runs in the kernels of kernels.cuh.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/dxpbd.h"
#include "kernels.cuh"
#include "tet_kernels.cuh"
#ifndef DX_HAVE_TETS
#define DX_HAVE_TETS 0
#endif

using namespace dx;

namespace {

thread_local std::string g_err;

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

__global__ void k_pack4(int V, const float *__restrict__ x3, const float *__restrict__ w, float4 *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    out[i] = make_float4(x3[3 * i], x3[3 * i + 1], x3[3 * i + 2], w ? w[i] : 0.f);
}
__global__ void k_pack4d(int V, const float *__restrict__ x3, const float *__restrict__ w, double4 *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    out[i] = make_double4(x3[3 * i], x3[3 * i + 1], x3[3 * i + 2], w ? (double)w[i] : 0.0);
}
__global__ void k_unpack3(int V, const double4 *__restrict__ x, float *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    double4 p = x[i];
    out[3 * i] = (float)p.x; out[3 * i + 1] = (float)p.y; out[3 * i + 2] = (float)p.z;
}
__global__ void k_gather_i2(int n, const int32_t *__restrict__ src, const int32_t *__restrict__ perm, int2 *__restrict__ dst) {
    int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    int u = perm[j];
    dst[j] = make_int2(src[2 * u], src[2 * u + 1]);
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
                              const float *__restrict__ beta, Collider *__restrict__ out) {
    int k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < nsph) {
        Collider c;
        c.c = make_float4(spheres[4 * k], spheres[4 * k + 1], spheres[4 * k + 2], 0.f);
        c.a = make_float4(0.f, 0.f, 0.f, 0.f);
        c.r = spheres[4 * k + 3];
        c.L = 0.f;
        c.type = 0;
        c.pad = 0;
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
        c.pad = 0;
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
__global__ void k_copy_xyz(int V, const float4 *__restrict__ a, float *__restrict__ out) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= V) return;
    float4 p = a[i];
    out[3 * i] = p.x; out[3 * i + 1] = p.y; out[3 * i + 2] = p.z;
}

}  // namespace

struct dxpbd_scene {
    int device = 0;
    int V = 0, E = 0, T = 0, NS = 0, NCAP = 0, NSH = 0, NC = 0;
    float dt = 0, inv_dt = 0, frame_dt = 0;
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
    DBuf<float> inv_mass;
    // tets
    TetData tets;
    // colliders
    DBuf<float> sph, cap_c, cap_a, cap_r0, cap_L0, cap_Rb, cap_Lb, beta;
    DBuf<Collider> cols;

    // trajectory
    int frames_done = -1;
    DBuf<double4> ckpt;   // [(max_frames*substeps+1) * V] fp64 position state, w = inverse mass
    DBuf<float4> v0;
    DBuf<float> forces;   // [max_frames * V * 3]
    bool have_forces = false;
    DBuf<float> tmp3;     // [V*3] staging

    // forward scratch for iterations > 1
    DBuf<float> lam_d, lam_c;

    // backward
    DBuf<double4> xr;
    DBuf<float4> ax, av, rhs, y, r, p, q;
    DBuf<float> Qd, ed, Qc, ec;
    DBuf<float> sc_lam, sc_sig, sc_B, sc_T, sc_e;               // distance scratch (K>1)
    DBuf<float> cc_lam, cc_T, cc_sig, cc_B, cc_e;               // contact scratch (K>1)
    DBuf<double> cg_sc, acc;
    DBuf<float> targets, weights;
    DBuf<float> g_comp, g_force, g_shape, g_sph;
    DBuf<float> g_x0, g_v0;
    bool have_grads = false;

    // stats
    double stats[8] = {0, 0, 0, 0, 0, 0, 0, 0};
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

void apply_shape(dxpbd_scene *s, cudaStream_t st) {
    if (!s->NC) return;
    k_shape_apply<<<nblk(s->NC), kBlock, 0, st>>>(s->NSH, s->NCAP, s->NS, s->sph.p, s->cap_c.p, s->cap_a.p,
                                                  s->cap_r0.p, s->cap_L0.p, s->cap_Rb.p, s->cap_Lb.p, s->beta.p,
                                                  s->cols.p);
    DX_CHECK_CUDA(cudaGetLastError());
}

inline double4 *state(dxpbd_scene *s, int n) { return s->ckpt.p + (size_t)n * s->V; }

// ------------------------------------------------------------------ one forward substep
int forward_substep(dxpbd_scene *s, int n, cudaStream_t st) {
    const int V = s->V;
    const int frame = n / s->substeps;
    double4 *xo = state(s, n + 1);
    const float *f = s->have_forces ? s->forces.p + (size_t)frame * V * 3 : nullptr;
    LAUNCH(DXPBD_K_PREDICT, k_predict<<<nblk(V), kBlock, 0, st>>>(V, state(s, n), n > 0 ? state(s, n - 1) : nullptr, s->v0.p, f,
                                                                   (double)s->dt, 1.0 / (double)s->dt, s->gravity, xo));
    int launches = 1;
    const float inv_dt2 = s->inv_dt * s->inv_dt;
    const int K = s->iterations;
    for (int k = 0; k < K; ++k) {
        const bool rd = k > 0, wr = k < K - 1;
        for (int c = 0; c < s->n_dist_colors; ++c) {
            int b = s->dist_off[c], cnt = s->dist_off[c + 1] - b;
            if (!cnt) continue;
            if (!rd && !wr)
                LAUNCH(DXPBD_K_DIST_PROJECT, k_dist_project<false, false><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, s->lam_d.p, xo));
            else if (!rd && wr)
                LAUNCH(DXPBD_K_DIST_PROJECT, k_dist_project<false, true><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, s->lam_d.p, xo));
            else if (rd && wr)
                LAUNCH(DXPBD_K_DIST_PROJECT, k_dist_project<true, true><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, s->lam_d.p, xo));
            else
                LAUNCH(DXPBD_K_DIST_PROJECT, k_dist_project<true, false><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, s->lam_d.p, xo));
            ++launches;
        }
        launches += tet_forward_sweep(s->tets, k, K, inv_dt2, s->dt, xo, st);
        if (s->NC) {
            float at = s->coll_alpha * inv_dt2;
            if (!rd && !wr) LAUNCH(DXPBD_K_CONTACT_PROJECT, k_contact_project<false, false><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, s->lam_c.p, xo));
            else if (!rd && wr) LAUNCH(DXPBD_K_CONTACT_PROJECT, k_contact_project<false, true><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, s->lam_c.p, xo));
            else if (rd && wr) LAUNCH(DXPBD_K_CONTACT_PROJECT, k_contact_project<true, true><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, s->lam_c.p, xo));
            else LAUNCH(DXPBD_K_CONTACT_PROJECT, k_contact_project<true, false><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, s->lam_c.p, xo));
            ++launches;
        }
    }
    DX_CHECK_CUDA(cudaGetLastError());
    return launches;
}

// ------------------------------------------------------------------ replay of substep n
int replay_substep(dxpbd_scene *s, int n, cudaStream_t st) {
    const int V = s->V, E = s->E;
    const int frame = n / s->substeps;
    const float *f = s->have_forces ? s->forces.p + (size_t)frame * V * 3 : nullptr;
    double4 *x = s->xr.p;
    LAUNCH(DXPBD_K_PREDICT, k_predict<<<nblk(V), kBlock, 0, st>>>(V, state(s, n), n > 0 ? state(s, n - 1) : nullptr, s->v0.p, f,
                                                                   (double)s->dt, 1.0 / (double)s->dt, s->gravity, x));
    int launches = 1;
    const float inv_dt2 = s->inv_dt * s->inv_dt;
    const int K = s->iterations;
    const bool want_e = (s->grad_flags >> DXPBD_GRAD_COMPLIANCE) & 1;
    DistScratch ds{s->sc_lam.p, s->sc_sig.p, s->sc_B.p, s->sc_T.p, s->sc_e.p};
    ContactScratch cs{s->cc_lam.p, s->cc_T.p, s->cc_sig.p, s->cc_B.p, s->cc_e.p};
    const bool want_ce = (s->grad_flags & ((1u << DXPBD_GRAD_SHAPE) | (1u << DXPBD_GRAD_SPHERE))) != 0;
    for (int k = 0; k < K; ++k) {
        const bool first = k == 0, last = k == K - 1;
        for (int c = 0; c < s->n_dist_colors; ++c) {
            int b = s->dist_off[c], cnt = s->dist_off[c + 1] - b;
            if (!cnt) continue;
            float *eo = want_e ? s->ed.p : nullptr;
            if (first && last)
                LAUNCH(DXPBD_K_DIST_REPLAY, k_dist_replay<true, true><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, ds, s->pd, s->Qd.p, eo, x));
            else if (first)
                LAUNCH(DXPBD_K_DIST_REPLAY, k_dist_replay<true, false><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, ds, s->pd, s->Qd.p, eo, x));
            else if (last)
                LAUNCH(DXPBD_K_DIST_REPLAY, k_dist_replay<false, true><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, ds, s->pd, s->Qd.p, eo, x));
            else
                LAUNCH(DXPBD_K_DIST_REPLAY, k_dist_replay<false, false><<<nblk(cnt), kBlock, 0, st>>>(b, cnt, E, s->d_idx.p, s->d_rest.p, s->d_alpha.p, inv_dt2, ds, s->pd, s->Qd.p, eo, x));
            ++launches;
        }
        launches += tet_replay_sweep(s->tets, k, K, inv_dt2, s->dt, s->pd, x, st);
        if (s->NC) {
            float at = s->coll_alpha * inv_dt2;
            float *eo = want_ce ? s->ec.p : nullptr;
            if (first && last) LAUNCH(DXPBD_K_CONTACT_REPLAY, k_contact_replay<true, true><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, cs, s->pd, s->Qc.p, eo, x));
            else if (first) LAUNCH(DXPBD_K_CONTACT_REPLAY, k_contact_replay<true, false><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, cs, s->pd, s->Qc.p, eo, x));
            else if (last) LAUNCH(DXPBD_K_CONTACT_REPLAY, k_contact_replay<false, true><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, cs, s->pd, s->Qc.p, eo, x));
            else LAUNCH(DXPBD_K_CONTACT_REPLAY, k_contact_replay<false, false><<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->cols.p, s->h, at, cs, s->pd, s->Qc.p, eo, x));
            ++launches;
        }
    }
    DX_CHECK_CUDA(cudaGetLastError());
    return launches;
}

// ------------------------------------------------------------------ filtered PCG
int pcg_solve(dxpbd_scene *s, cudaStream_t st, int &iters_out, double &relres_out) {
    const int V = s->V, E = s->E;
    const int maxit = s->cg_max_iter;
    DX_CHECK_CUDA(cudaMemsetAsync(s->cg_sc.p, 0, sizeof(double) * (size_t)(maxit + 2) * 4, st));
    CGState cs{s->cg_sc.p, s->cg_sc.p + 2, s->cg_tol * s->cg_tol};
    const float *xw = s->inv_mass.p;
    LAUNCH(DXPBD_K_CG_INIT, k_cg_init<<<nblk(V), kBlock, 0, st>>>(V, s->rhs.p, s->ax.p, s->r.p, s->p.p, xw, cs));
    int launches = 1;
    const float *Qc = s->NC ? s->Qc.p : nullptr;
    int it = 0;
    const int chunk = 8;
    iters_out = -1;
    relres_out = 0.0;
    while (it < maxit) {
        int end = std::min(maxit, it + chunk);
        for (; it < end; ++it) {
            LAUNCH(DXPBD_K_CG_VERTEX, k_cg_vertex<<<nblk(V), kBlock, 0, st>>>(V, it, s->p.p, s->r.p, s->q.p, xw, Qc, cs));
            ++launches;
            if (E) {
                LAUNCH(DXPBD_K_CG_DIST, k_cg_dist<<<nblk(E), kBlock, 0, st>>>(E, it, s->d_idx.p, s->Qd.p, s->p.p, s->q.p, xw, cs));
                ++launches;
            }
            launches += tet_cg_matvec(s->tets, it, s->p.p, s->q.p, xw, cs, st);
            LAUNCH(DXPBD_K_CG_UPDATE, k_cg_update<<<nblk(V), kBlock, 0, st>>>(V, it, s->ax.p, s->r.p, s->p.p, s->q.p, xw, cs));
            ++launches;
        }
        // convergence check: rr of the last completed iteration
        DX_CHECK_CUDA(cudaMemcpyAsync(s->h_scal, s->cg_sc.p, sizeof(double) * (size_t)(it + 1) * 4, cudaMemcpyDeviceToHost, st));
        DX_CHECK_CUDA(cudaStreamSynchronize(st));
        double bb = s->h_scal[2];
        double tol2 = (double)s->cg_tol * s->cg_tol;
        if (bb == 0.0) { iters_out = 0; relres_out = 0.0; break; }
        for (int k = 0; k <= it; ++k) {
            double rr = s->h_scal[k * 4 + 2];
            if (k > 0 && rr == 0.0 && s->h_scal[k * 4 + 0] == 0.0) break;   // not executed (done earlier)
            if (rr <= tol2 * bb) { iters_out = k; relres_out = std::sqrt(rr / bb); break; }
        }
        if (iters_out >= 0) break;
        relres_out = std::sqrt(s->h_scal[it * 4 + 2] / bb);
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
    DX_REQUIRE(d->num_tets == 0 || DX_HAVE_TETS, DXPBD_ERR_ARG, "tet constraints not built into this library");
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
    s->gravity = make_float3(d->gravity[0], d->gravity[1], d->gravity[2]);
    s->h = d->thickness;
    s->coll_alpha = d->collision_compliance;
    s->max_frames = d->max_frames;
    s->grad_flags = d->grad_flags;
    s->pd = d->pd_projection;
    s->cg_tol = d->cg_tol > 0 ? d->cg_tol : 1e-6f;
    s->cg_max_iter = d->cg_max_iter > 0 ? d->cg_max_iter : 500;
    cudaStream_t st = 0;

    s->inv_mass.alloc(V);
    upload(s->inv_mass.p, d->inv_mass, sizeof(float) * V, DXPBD_MEM_HOST, st);
    DBuf<float> xr3;
    xr3.alloc((size_t)V * 3);
    upload(xr3.p, d->x_rest, sizeof(float) * V * 3, DXPBD_MEM_HOST, st);

    // distance constraints: greedy colors, color sort, SoA
    if (s->E) {
        int nc = greedy_colors(s->E, 2, d->dist_idx, V, s->dist_color_h);
        if (nc < 0) throw Err{DXPBD_ERR_LIMIT, "distance coloring needs more than 256 colors"};
        s->n_dist_colors = nc;
        color_sort(s->dist_color_h, nc, s->dist_perm_h, s->dist_off);
        DBuf<int32_t> idx_u;
        DBuf<float> alpha_u;
        idx_u.alloc((size_t)2 * s->E);
        alpha_u.alloc(s->E);
        upload(idx_u.p, d->dist_idx, sizeof(int32_t) * 2 * s->E, DXPBD_MEM_HOST, st);
        upload(alpha_u.p, d->dist_compliance, sizeof(float) * s->E, DXPBD_MEM_HOST, st);
        s->d_perm.alloc(s->E);
        upload(s->d_perm.p, s->dist_perm_h.data(), sizeof(int32_t) * s->E, DXPBD_MEM_HOST, st);
        s->d_idx.alloc(s->E);
        s->d_rest.alloc(s->E);
        s->d_alpha.alloc(s->E);
        k_gather_i2<<<nblk(s->E), kBlock, 0, st>>>(s->E, idx_u.p, s->d_perm.p, s->d_idx.p);
        k_gather_f<<<nblk(s->E), kBlock, 0, st>>>(s->E, alpha_u.p, s->d_perm.p, s->d_alpha.p);
        k_rest_len<<<nblk(s->E), kBlock, 0, st>>>(s->E, s->d_idx.p, xr3.p, s->d_rest.p);
        DX_CHECK_CUDA(cudaGetLastError());
        DX_CHECK_CUDA(cudaStreamSynchronize(st));
    }
    // tets
    if (s->T) {
        int nc = greedy_colors(s->T, 4, d->tet_idx, V, s->tet_color_h);
        if (nc < 0) throw Err{DXPBD_ERR_LIMIT, "tet coloring needs more than 256 colors"};
        s->n_tet_colors = nc;
        color_sort(s->tet_color_h, nc, s->tet_perm_h, s->tet_off);
        tet_create(s->tets, s->T, d->tet_idx, d->tet_a, d->tet_b, xr3.p, s->tet_perm_h, s->tet_off,
                   s->iterations, s->dt, (s->grad_flags >> DXPBD_GRAD_MATERIAL) & 1, st);
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
        apply_shape(s, st);
    }
    // trajectory storage
    const size_t nstates = (size_t)s->max_frames * s->substeps + 1;
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
    const int V = s->V;
    upload(s->tmp3.p, x0, sizeof(float) * V * 3, mem, st);
    k_pack4d<<<nblk(V), kBlock, 0, st>>>(V, s->tmp3.p, s->inv_mass.p, state(s, 0));
    upload(s->tmp3.p, v0, sizeof(float) * V * 3, mem, st);
    k_pack4<<<nblk(V), kBlock, 0, st>>>(V, s->tmp3.p, nullptr, s->v0.p);
    s->have_forces = forces != nullptr;
    if (forces) {
        if (s->forces.n < (size_t)s->max_frames * V * 3) s->forces.alloc((size_t)s->max_frames * V * 3);
        upload(s->forces.p, forces, sizeof(float) * (size_t)num_frames * V * 3, mem, st);
    }
    int launches = 4;
    const int N = num_frames * s->substeps;
    for (int n = 0; n < N; ++n) launches += forward_substep(s, n, st);
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
    cudaStream_t st = (cudaStream_t)stream;
    k_unpack3<<<nblk(s->V), kBlock, 0, st>>>(s->V, state(s, frame * s->substeps), s->tmp3.p);
    download(out, s->tmp3.p, sizeof(float) * s->V * 3, mem, st);
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
    // buffers
    if (s->xr.n < (size_t)V) s->xr.alloc(V);
    auto ensure4 = [&](DBuf<float4> &b) { if (b.n < (size_t)V) b.alloc(V); };
    ensure4(s->ax); ensure4(s->av); ensure4(s->rhs); ensure4(s->y); ensure4(s->r); ensure4(s->p); ensure4(s->q);
    if (E && s->Qd.n < (size_t)6 * E) s->Qd.alloc((size_t)6 * E);
    const bool g_comp = (s->grad_flags >> DXPBD_GRAD_COMPLIANCE) & 1;
    const bool g_forces = (s->grad_flags >> DXPBD_GRAD_FORCES) & 1;
    const bool g_coll = (s->grad_flags & ((1u << DXPBD_GRAD_SHAPE) | (1u << DXPBD_GRAD_SPHERE))) != 0;
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
    tet_backward_alloc(s->tets, s->iterations, st);
    // targets
    if (num_keys) {
        if (s->targets.n < (size_t)num_keys * V * 3) s->targets.alloc((size_t)num_keys * V * 3);
        upload(s->targets.p, targets, sizeof(float) * (size_t)num_keys * V * 3, mem, st);
    }
    const float *wts = nullptr;
    if (weights) {
        if (s->weights.n < (size_t)V) s->weights.alloc(V);
        upload(s->weights.p, weights, sizeof(float) * V, mem, st);
        wts = s->weights.p;
    }
    // gradient accumulators
    if (g_comp && E) { if (s->g_comp.n < (size_t)E) s->g_comp.alloc(E); DX_CHECK_CUDA(cudaMemsetAsync(s->g_comp.p, 0, sizeof(float) * E, st)); }
    if (g_forces) {
        size_t nf = (size_t)std::max(s->frames_done, 1) * V * 3;
        if (s->g_force.n < nf) s->g_force.alloc(nf);
        DX_CHECK_CUDA(cudaMemsetAsync(s->g_force.p, 0, sizeof(float) * nf, st));
    }
    DX_CHECK_CUDA(cudaMemsetAsync(s->acc.p, 0, sizeof(double) * nacc, st));
    tet_grad_reset(s->tets, st);
    // state index -> keyframe slot
    std::vector<int> key_of(N + 1, -1);
    for (int k = 0; k < num_keys; ++k) key_of[key_frames[k] * sub] = k;   // duplicates: last wins
    // loss
    for (int k = 0; k < num_keys; ++k)
        LAUNCH(DXPBD_K_OTHER, k_loss<<<nblk(V), kBlock, 0, st>>>(V, state(s, key_frames[k] * sub), s->targets.p + (size_t)k * V * 3, wts, s->acc.p));
    // increment-form adjoint (kernels.cuh "adjoint"): y = u = 0 beyond the horizon
    auto tgt = [&](int n) -> const float * { return key_of[n] >= 0 ? s->targets.p + (size_t)key_of[n] * V * 3 : nullptr; };
    DX_CHECK_CUDA(cudaMemsetAsync(s->y.p, 0, sizeof(float4) * V, st));
    DX_CHECK_CUDA(cudaMemsetAsync(s->ax.p, 0, sizeof(float4) * V, st));   // ax holds u
    int last_key_state = -1;
    for (int n = 0; n <= N; ++n) if (key_of[n] >= 0) last_key_state = n;
    int launches = num_keys + 2, total_it = 0, max_it = 0;
    double worst = 0.0;
    int solves = 0;
    const float *Qc = s->NC ? s->Qc.p : nullptr;
    for (int n = std::min(N, last_key_state) - 1; n >= 0; --n) {
        const int frame = n / sub;
        float *gf = g_forces ? s->g_force.p + (size_t)frame * V * 3 : nullptr;
        launches += replay_substep(s, n, st);
        // b = M u_{n+1} - Q_n y_{n+1} + dphi/dx_{n+1}
        LAUNCH(DXPBD_K_RHS, k_rhs_vertex<<<nblk(V), kBlock, 0, st>>>(V, s->inv_mass.p, s->ax.p, s->y.p, Qc, state(s, n + 1), tgt(n + 1), wts,
                                                 s->rhs.p));
        ++launches;
        if (E) {
            LAUNCH(DXPBD_K_RHS, k_rhs_dist<<<nblk(E), kBlock, 0, st>>>(E, s->d_idx.p, s->Qd.p, s->y.p, s->rhs.p, s->inv_mass.p));
            ++launches;
        }
        launches += tet_rhs(s->tets, s->y.p, s->rhs.p, s->inv_mass.p, st);
        int iters = 0;
        double rel = 0.0;
        launches += pcg_solve(s, st, iters, rel);   // u_n into s->ax
        total_it += iters;
        max_it = std::max(max_it, iters);
        worst = std::max(worst, rel);
        ++solves;
        LAUNCH(DXPBD_K_ADJOINT, k_adjoint_accum<<<nblk(V), kBlock, 0, st>>>(V, s->inv_mass.p, s->ax.p, s->y.p, gf, s->dt));
        ++launches;
        if (g_comp && E) {
            LAUNCH(DXPBD_K_GRADS, k_grad_compliance<<<nblk(E), kBlock, 0, st>>>(E, s->d_idx.p, s->ed.p, s->y.p, s->g_comp.p));
            ++launches;
        }
        if (g_coll && s->NC) {
            LAUNCH(DXPBD_K_GRADS, k_grad_colliders<<<nblk(V), kBlock, 0, st>>>(V, s->NC, s->ec.p, s->y.p, s->acc.p + 1));
            ++launches;
        }
        launches += tet_grads(s->tets, s->y.p, st);
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
    if (loss_out) *loss_out = (float)phi;
    s->stats[0] = total_it;
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
            download(out, kind == DXPBD_GRAD_X0 ? s->g_x0.p : s->g_v0.p, sizeof(float) * V * 3, mem, st);
            break;
        }
        case DXPBD_GRAD_FORCES: {
            int64_t n = (int64_t)std::max(s->frames_done, 1) * V * 3;
            DX_REQUIRE(out_len == n, DXPBD_ERR_ARG, "out_len must be frames*3V");
            download(out, s->g_force.p, sizeof(float) * n, mem, st);
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
            tet_grad_out(s->tets, out, mem, st);
            break;
        }
    }
    DX_API_END
}

int dxpbd_set_params(dxpbd_scene *s, int32_t kind, const float *data, int64_t len, int32_t mem, void *stream) {
    DX_API_BEGIN
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
        case DXPBD_PARAM_MATERIAL:
            DX_REQUIRE(len == 2 * (int64_t)s->T, DXPBD_ERR_ARG, "len must be 2T");
            tet_set_material(s->tets, data, mem, st);
            break;
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
    for (int k = 0; k < n && k < 8; ++k) out[k] = s->stats[k];
    DX_API_END
}

}  // extern "C"

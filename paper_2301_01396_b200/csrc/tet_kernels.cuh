// Tetrahedral Neo-Hookean block constraints (Sec.5.2 l.229; R6):
// per tet the rows (C_D, C_H) = (||F||_F - sqrt 3, det F - 1), both zero at the rest state F = I
// (Eq. xpbdUenergy l.76: U = 0 at rest), are projected together as one 2-row block (Eq. xpbd in matrix form), alpha_D = 1/(mu V), alpha_H = 1/(lambda V),
// mu = a^2, lambda = b^2.  Everything in deformation-gradient coordinates vec F = G x (column-
// major, index 3*col + row): grad C_a = G^T P_a, H_a = G^T HF_a G, M^-1 -> W~ = K (x) I3 with
// K = Sum_v w_v c_v c_v^T, c_v the Dm^-1 coefficients of vertex v.  Derivative blocks are
// accumulated in F-space (D = G^T D~ G) and projected there (R5).
// Precision: near rest grad C_D || grad C_H (F = I), so the 2x2 block J is nearly singular for stiff
// materials (det J ~ at * |g|^2 vs entries ~ |g|^4); the block solve, the position update and the
// derivative algebra therefore run in fp64 (tr = double); only stored blocks are fp32.
#pragma once
#include "kernels.cuh"

namespace dx {

typedef double tr;

struct TetDev {
    int T;
    const int4 *idx;      // [T] internal vertex ids (color-sorted)
    const double *Dm;     // [9T] Dm^-1 SoA (fp64), element (i, col) at (3*i + col) * T + j
    const double *vol;    // [T] rest volume (fp64)
    const float *ta, *tb; // [T] material a, b
    const float *Dmf;     // [9T] Dm^-1 rounded to fp32 (the fp32 kernels' copy: half the bytes)
    // deterministic corner gather (no float atomics): per-tet corner contributions gq[set][corner][k][T]
    // and, per vertex, its corner slots in a fixed order (CSR: ginc[goff[v] .. goff[v+1]) = 3 c T + j)
    const int *goff = nullptr, *ginc = nullptr;
    float *gq = nullptr;
};

// corner contribution g of tet j at corner c into gather set `set` (0: matvec / rhs y, 1: rhs z)
DX_INLINE void tet_corner_store(const TetDev &D, int set, int c, int j, float3 g) {
    float *o = D.gq + (size_t)set * 12 * D.T + (size_t)3 * c * D.T + j;
    o[0] = g.x;
    o[D.T] = g.y;
    o[2 * (size_t)D.T] = g.z;
}
// sum of the corner contributions at vertex v, in the fixed slot order (deterministic)
DX_INLINE float3 tet_gather(const TetDev &D, int set, int v) {
    float3 g = make_float3(0.f, 0.f, 0.f);
    const float *base = D.gq + (size_t)set * 12 * D.T;
    for (int e = D.goff[v]; e < D.goff[v + 1]; ++e) {
        const float *o = base + D.ginc[e];
        g = g + make_float3(o[0], o[D.T], o[2 * (size_t)D.T]);
    }
    return g;
}

struct TetCore {
    tr F[9];              // column-major
    tr P[2][9];           // dC_a/dvecF
    tr C[2];
    tr CD;                // ||F||
    tr c[4][3];           // Dm^-1 coefficients c_{v,col}
    tr K[3][3];           // Sum_v w_v c_v c_v^T
    tr J[2][2], Ji[2][2];
    tr at[2];
    tr dl[2];
};
DX_INLINE double3 operator+(double3 a, double3 b) { return make_double3(a.x + b.x, a.y + b.y, a.z + b.z); }
DX_INLINE double3 operator-(double3 a, double3 b) { return make_double3(a.x - b.x, a.y - b.y, a.z - b.z); }
DX_INLINE double3 operator*(double s, double3 a) { return make_double3(s * a.x, s * a.y, s * a.z); }
DX_INLINE double3 dcross3(double3 a, double3 b) {
    return make_double3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}
DX_INLINE double ddot3p(double3 a, double3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }

template <class R>
DX_INLINE void tet_load_c(const TetDev &D, int j, R (&c)[4][3]) {
#pragma unroll
    for (int col = 0; col < 3; ++col) {
        R s = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            c[i + 1][col] = D.Dm[(size_t)(3 * i + col) * D.T + j];
            s += c[i + 1][col];
        }
        c[0][col] = -s;
    }
}

// fp32 coefficients: the same values as the template above with R = float (rounded once at create)
DX_INLINE void tet_load_c(const TetDev &D, int j, float (&c)[4][3]) {
#pragma unroll
    for (int col = 0; col < 3; ++col) {
        float s = 0;
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            c[i + 1][col] = D.Dmf[(size_t)(3 * i + col) * D.T + j];
            s += c[i + 1][col];
        }
        c[0][col] = -s;
    }
}

// W~ v  (v in F-space): (W~ v)[(col,row)] = Sum_col' K[col][col'] v[(col',row)]
DX_INLINE void tet_Wmul(const tr (&K)[3][3], const tr *v, tr *out) {
#pragma unroll
    for (int col = 0; col < 3; ++col)
#pragma unroll
        for (int row = 0; row < 3; ++row)
            out[3 * col + row] = K[col][0] * v[row] + K[col][1] * v[3 + row] + K[col][2] * v[6 + row];
}

// HF_D v = (v - P_D (P_D . v)) / ||F||
DX_INLINE void tet_HD_mul(const TetCore &o, const tr *v, tr *out) {
    tr pv = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) pv += o.P[0][k] * v[k];
    const tr ic = 1.0 / o.CD;
#pragma unroll
    for (int k = 0; k < 9; ++k) out[k] = (v[k] - o.P[0][k] * pv) * ic;
}

DX_INLINE float3 f3at(const float *a, int k) { return make_float3(a[3 * k], a[3 * k + 1], a[3 * k + 2]); }
DX_INLINE void put3(float *a, int k, float3 v) { a[3 * k] = v.x; a[3 * k + 1] = v.y; a[3 * k + 2] = v.z; }
DX_INLINE double3 d3at(const tr *a, int k) { return make_double3(a[3 * k], a[3 * k + 1], a[3 * k + 2]); }
DX_INLINE void dput3(tr *a, int k, double3 v) { a[3 * k] = v.x; a[3 * k + 1] = v.y; a[3 * k + 2] = v.z; }

// HF_H v: blocks (i,j) of d cof / dF: out_0 = -f2 x v1 + f1 x v2, out_1 = f2 x v0 - f0 x v2,
// out_2 = -f1 x v0 + f0 x v1
DX_INLINE void tet_HH_mul(const TetCore &o, const tr *v, tr *out) {
    const double3 f0 = d3at(o.F, 0), f1 = d3at(o.F, 1), f2 = d3at(o.F, 2);
    const double3 v0 = d3at(v, 0), v1 = d3at(v, 1), v2 = d3at(v, 2);
    dput3(out, 0, dcross3(f1, v2) - dcross3(f2, v1));
    dput3(out, 1, dcross3(f2, v0) - dcross3(f0, v2));
    dput3(out, 2, dcross3(f0, v1) - dcross3(f1, v0));
}

// Projection core (Eq. xpbd, 2-row block), fp64.  Returns false when skipped (R13).
DX_INLINE bool tet_core(const double4 (&x)[4], const tr (&c)[4][3], tr at0, tr at1, const tr (&lam0)[2],
                        TetCore &o) {
    tr w[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) w[v] = x[v].w;
    if (!(w[0] + w[1] + w[2] + w[3] > 0.0)) return false;
    tr Ds[3][3];   // Ds[row][i] = (x_{i+1} - x_0)[row]
#pragma unroll
    for (int i = 0; i < 3; ++i) {
        Ds[0][i] = x[i + 1].x - x[0].x;
        Ds[1][i] = x[i + 1].y - x[0].y;
        Ds[2][i] = x[i + 1].z - x[0].z;
    }
#pragma unroll
    for (int col = 0; col < 3; ++col)
#pragma unroll
        for (int row = 0; row < 3; ++row)
            o.F[3 * col + row] = Ds[row][0] * c[1][col] + Ds[row][1] * c[2][col] + Ds[row][2] * c[3][col];
#pragma unroll
    for (int v = 0; v < 4; ++v)
#pragma unroll
        for (int col = 0; col < 3; ++col) o.c[v][col] = c[v][col];
    tr n2 = 0;
#pragma unroll
    for (int k = 0; k < 9; ++k) n2 += o.F[k] * o.F[k];
    o.CD = sqrt(n2);
    if (!(o.CD > (tr)kEpsLen)) return false;
#pragma unroll
    for (int k = 0; k < 9; ++k) o.P[0][k] = o.F[k] / o.CD;
    const double3 f0 = d3at(o.F, 0), f1 = d3at(o.F, 1), f2 = d3at(o.F, 2);
    const double3 c0 = dcross3(f1, f2), c1 = dcross3(f2, f0), c2 = dcross3(f0, f1);
    dput3(o.P[1], 0, c0);
    dput3(o.P[1], 1, c1);
    dput3(o.P[1], 2, c2);
    const tr det = ddot3p(f0, c0);
    o.C[0] = o.CD - 1.7320508075688772;   // ||F|| - sqrt 3
    o.C[1] = det - 1.0;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int j = 0; j < 3; ++j)
            o.K[i][j] = w[0] * c[0][i] * c[0][j] + w[1] * c[1][i] * c[1][j] + w[2] * c[2][i] * c[2][j] +
                        w[3] * c[3][i] * c[3][j];
    tr WP[2][9];
    tet_Wmul(o.K, o.P[0], WP[0]);
    tet_Wmul(o.K, o.P[1], WP[1]);
    o.at[0] = at0;
    o.at[1] = at1;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            tr s = 0;
#pragma unroll
            for (int k = 0; k < 9; ++k) s += o.P[a][k] * WP[b][k];
            o.J[a][b] = s + (a == b ? o.at[a] : 0.0);
        }
    const tr dJ = o.J[0][0] * o.J[1][1] - o.J[0][1] * o.J[1][0];
    if (!(fabs(dJ) > 0.0)) return false;
    const tr idj = 1.0 / dJ;
    o.Ji[0][0] = o.J[1][1] * idj;
    o.Ji[1][1] = o.J[0][0] * idj;
    o.Ji[0][1] = -o.J[0][1] * idj;
    o.Ji[1][0] = -o.J[1][0] * idj;
    const tr b0 = -o.C[0] - at0 * lam0[0], b1 = -o.C[1] - at1 * lam0[1];
    o.dl[0] = o.Ji[0][0] * b0 + o.Ji[0][1] * b1;
    o.dl[1] = o.Ji[1][0] * b0 + o.Ji[1][1] * b1;
    return true;
}

// x_v += w_v Sum_a (grad C_a)_v dl_a,  (grad C_a)_v[row] = Sum_col c_{v,col} P_a[3 col + row]
DX_INLINE void tet_apply(double4 (&x)[4], const TetCore &o) {
    tr PD[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) PD[k] = o.P[0][k] * o.dl[0] + o.P[1][k] * o.dl[1];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        const tr w = x[v].w;
        double3 g = make_double3(0.0, 0.0, 0.0);
#pragma unroll
        for (int col = 0; col < 3; ++col) g = g + o.c[v][col] * d3at(PD, col);
        x[v].x += w * g.x;
        x[v].y += w * g.y;
        x[v].z += w * g.z;
    }
}

DX_INLINE tr tet_at(const TetDev &D, int j, int row, double inv_dt2) {
    const tr m = row == 0 ? D.ta[j] : D.tb[j];
    return inv_dt2 / (m * m * D.vol[j]);
}

template <bool READ_LAM, bool WRITE_LAM>
__global__ void __launch_bounds__(128) k_tet_project(int begin, int count, TetDev D, double inv_dt2,
                                                     float *__restrict__ lam, double4 *__restrict__ x) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= count) return;
    const int j = begin + t;
    const int4 id = D.idx[j];
    double4 xs[4] = {x[id.x], x[id.y], x[id.z], x[id.w]};
    tr c[4][3];
    tet_load_c(D, j, c);
    tr lam0[2] = {READ_LAM ? (tr)lam[2 * j] : 0.0, READ_LAM ? (tr)lam[2 * j + 1] : 0.0};
    TetCore o;
    if (!tet_core(xs, c, tet_at(D, j, 0, inv_dt2), tet_at(D, j, 1, inv_dt2), lam0, o)) return;
    if (WRITE_LAM) {
        lam[2 * j] = (float)(lam0[0] + o.dl[0]);
        lam[2 * j + 1] = (float)(lam0[1] + o.dl[1]);
    }
    tet_apply(xs, o);
    x[id.x] = xs[0];
    x[id.y] = xs[1];
    x[id.z] = xs[2];
    x[id.w] = xs[3];
}

// 9x9 symmetric PSD projection by cyclic Jacobi (R5), in place on the packed upper triangle
// a[sx(p, q)] (the Qt~ layout).  Each rotation updates the two rows / columns p, q of the
// symmetric matrix once (a_pp -= t a_pq, a_qq += t a_pq, a_pq = 0, a_kp / a_kq for k != p, q) and
// the eigenvector matrix V; every index is a compile-time constant (fully unrolled), so a and V
// stay in registers.  Eigenvalues are clamped at 0 and the block rebuilt as V diag(l) V^T.
DX_INLINE constexpr int sx(int p, int q) {
    return p <= q ? p * 9 - (p * (p - 1)) / 2 + (q - p) : q * 9 - (q * (q - 1)) / 2 + (p - q);
}
DX_INLINE void psd9p(float (&a)[45], float tol = 1e-6f, int max_sweeps = 12) {
    float V[9][9];
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
        for (int j = 0; j < 9; ++j) V[i][j] = i == j ? 1.f : 0.f;
    float scale = 0.f;
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
        for (int j = i; j < 9; ++j) scale += (i == j ? 1.f : 2.f) * fabsf(a[sx(i, j)]);
    if (scale == 0.f) return;
#pragma unroll 1
    for (int sweep = 0; sweep < max_sweeps; ++sweep) {
        float off = 0.f;
#pragma unroll
        for (int p = 0; p < 9; ++p)
#pragma unroll
            for (int q = p + 1; q < 9; ++q) off += fabsf(a[sx(p, q)]);
        if (off <= tol * scale) break;
#pragma unroll
        for (int p = 0; p < 8; ++p) {
#pragma unroll
            for (int q = p + 1; q < 9; ++q) {
                const float apq = a[sx(p, q)];
                if (fabsf(apq) < 1e-30f) continue;
                const float theta = (a[sx(q, q)] - a[sx(p, p)]) / (2.f * apq);
                const float tt = copysignf(1.f, theta) / (fabsf(theta) + sqrtf(theta * theta + 1.f));
                const float cc = rsqrtf(tt * tt + 1.f), ss = tt * cc;
                a[sx(p, p)] -= tt * apq;
                a[sx(q, q)] += tt * apq;
                a[sx(p, q)] = 0.f;
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    if (k == p || k == q) continue;
                    const float akp = a[sx(k, p)], akq = a[sx(k, q)];
                    a[sx(k, p)] = cc * akp - ss * akq;
                    a[sx(k, q)] = ss * akp + cc * akq;
                }
#pragma unroll
                for (int k = 0; k < 9; ++k) {
                    const float vkp = V[k][p], vkq = V[k][q];
                    V[k][p] = cc * vkp - ss * vkq;
                    V[k][q] = ss * vkp + cc * vkq;
                }
            }
        }
    }
    float l[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) l[i] = fmaxf(a[sx(i, i)], 0.f);
#pragma unroll
    for (int i = 0; i < 9; ++i)
#pragma unroll
        for (int j = i; j < 9; ++j) {
            float s = 0.f;
#pragma unroll
            for (int k = 0; k < 9; ++k) s += l[k] * V[i][k] * V[j][k];
            a[sx(i, j)] = s;
        }
}

// PD projection (R5) of every tet's F-space block in place: Qt~ <- psd(Qt~) (45 floats, upper
// triangle, SoA), one thread per tet with the 9x9 Jacobi in registers.
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_tet_psd(int T, float *__restrict__ Qt, float tol, int max_sweeps) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= T) return;
    float a[45];
#pragma unroll
    for (int m = 0; m < 45; ++m) a[m] = Qt[(size_t)m * T + j];
    psd9p(a, tol, max_sweeps);
#pragma unroll
    for (int m = 0; m < 45; ++m) Qt[(size_t)m * T + j] = a[m];
}

// Running state of the differentiable replay (iterations > 1), SoA per tet.
struct TetScratch {
    float *lam;   // [2T]
    float *S;     // [18T] running d lam / dx in F-space (2 rows x 9)
    float *Dt;    // [45T] accumulated sym(D~), upper triangle
    float *Tu;    // [4T] running d lam / du (2 controls x 2 rows)
    float *e;     // [18T] control vectors (2 controls x 9)
};

// Differentiable replay of one tet color (Sec.4.3/4.4, R3, R5, R6) in F-space:
//   Dx~ = W~ Sum_b P_b dl_b ; j_a = HF_a Dx~ + Sum_b dl_b HF_b (W~ P_a)
//   s~_a = Sum_b Ji_ab (-P_b - at_b S~_b - j_b) ;  D~ += Sum_a dl_a HF_a + Sum_a P_a s~_a^T ; S~ += s~
// controls u = (a, b): t_u = Ji (-dat/du lam0 - at T_u - diag(dat/du) dl) ;   (dC/du = 0, R6)
//   e~_u += Sum_a t_{u,a} P_a ;  T_u += t_u
//   dat_D/da = -2 at_D / a, dat_H/db = -2 at_H / b.
// After the last iteration: Qt~ = psd(-sym D~) (45 floats, upper triangle) and e~ (18 floats).
// MODE 0: one pass per color (any K).  K = 1 splits it in two so the heavy derivative algebra and
// the 9x9 PSD projection run once over all tets instead of color by color (a color is a few
// thousand tets: long per-thread chains on a mostly idle GPU):
//   MODE 1 (per color): regenerate the iterate (tet_core / tet_apply, as the forward) and save the
//           tet's pre-update vertices to xsave[4 j .. 4 j + 3];
//   MODE 2 (all tets, one launch): the derivative blocks from the saved vertices (same arithmetic
//           as MODE 0 with FIRST = LAST = true), no position writes.
template <bool FIRST, bool LAST, int MODE = 0>
__global__ void __launch_bounds__(128) k_tet_replay(int begin, int count, TetDev D, double inv_dt2, TetScratch sc, int pd,
                                                    float *__restrict__ Qt, float *__restrict__ eout,
                                                    double4 *__restrict__ x, double4 *__restrict__ xsave = nullptr) {
    const int tid = blockIdx.x * blockDim.x + threadIdx.x;
    if (tid >= count) return;
    const int j = begin + tid;
    const int T = D.T;
    const int4 id = D.idx[j];
    double4 xs[4];
    if (MODE == 2) {
        for (int k = 0; k < 4; ++k) xs[k] = xsave[4 * (size_t)j + k];
    } else {
        xs[0] = x[id.x]; xs[1] = x[id.y]; xs[2] = x[id.z]; xs[3] = x[id.w];
    }
    if (MODE == 1)
        for (int k = 0; k < 4; ++k) xsave[4 * (size_t)j + k] = xs[k];
    tr c[4][3];
    tet_load_c(D, j, c);
    const tr a = D.ta[j], b = D.tb[j];
    tr lam0[2] = {0.0, 0.0}, S[2][9], Tu[2][2] = {{0.0, 0.0}, {0.0, 0.0}}, e[2][9];
    tr Dt[45];   // upper triangle of the symmetric part of D~ (row-major p <= q)
    for (int k = 0; k < 9; ++k) S[0][k] = S[1][k] = e[0][k] = e[1][k] = 0.0;
    for (int m = 0; m < 45; ++m) Dt[m] = 0.0;
    if (!FIRST) {
        lam0[0] = sc.lam[2 * j];
        lam0[1] = sc.lam[2 * j + 1];
        for (int k = 0; k < 9; ++k) {
            S[0][k] = sc.S[(size_t)k * T + j];
            S[1][k] = sc.S[(size_t)(9 + k) * T + j];
            e[0][k] = sc.e[(size_t)k * T + j];
            e[1][k] = sc.e[(size_t)(9 + k) * T + j];
        }
        for (int u = 0; u < 4; ++u) Tu[u / 2][u % 2] = sc.Tu[(size_t)u * T + j];
        for (int m = 0; m < 45; ++m) Dt[m] = sc.Dt[(size_t)m * T + j];
    }
    const tr at0 = tet_at(D, j, 0, inv_dt2), at1 = tet_at(D, j, 1, inv_dt2);
    TetCore o;
    const bool ok = tet_core(xs, c, at0, at1, lam0, o);
    if (MODE == 1) {
        if (ok) {
            tet_apply(xs, o);
            x[id.x] = xs[0];
            x[id.y] = xs[1];
            x[id.z] = xs[2];
            x[id.w] = xs[3];
        }
        return;
    }
    if (ok) {
        tr WP[2][9], sumP[9], Dx[9];
        tet_Wmul(o.K, o.P[0], WP[0]);
        tet_Wmul(o.K, o.P[1], WP[1]);
        for (int k = 0; k < 9; ++k) sumP[k] = o.P[0][k] * o.dl[0] + o.P[1][k] * o.dl[1];
        tet_Wmul(o.K, sumP, Dx);
        tr jv[2][9], h1[9], h2[9];
        for (int r = 0; r < 2; ++r) {
            // j_a = HF_a Dx~ + Sum_b dl_b HF_b (W~ P_a)
            if (r == 0) tet_HD_mul(o, Dx, jv[0]); else tet_HH_mul(o, Dx, jv[1]);
            tet_HD_mul(o, WP[r], h1);
            tet_HH_mul(o, WP[r], h2);
            for (int k = 0; k < 9; ++k) jv[r][k] += o.dl[0] * h1[k] + o.dl[1] * h2[k];
        }
        tr rhs[2][9], sv[2][9];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 9; ++k) rhs[r][k] = -o.P[r][k] - o.at[r] * S[r][k] - jv[r][k];
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 9; ++k) sv[r][k] = o.Ji[r][0] * rhs[0][k] + o.Ji[r][1] * rhs[1][k];
        // D~ += dl_D HF_D + dl_H HF_H + Sum_a P_a s~_a^T   (symmetric part, upper triangle)
        const tr sD = o.dl[0] / o.CD;
        {
            int m = 0;
            for (int p = 0; p < 9; ++p)
                for (int q = p; q < 9; ++q, ++m)
                    Dt[m] += sD * ((p == q ? 1.0 : 0.0) - o.P[0][p] * o.P[0][q]) +
                             0.5 * (o.P[0][p] * sv[0][q] + o.P[1][p] * sv[1][q] + o.P[0][q] * sv[0][p] + o.P[1][q] * sv[1][p]);
        }
        {   // dl_H HF_H: blocks (i,j) = sgn [f_k]x with (i,j,k,sgn) = (0,1,2,-), (0,2,1,+), (1,2,0,-)
            // (upper blocks only; HF_H is symmetric); [f]x = [[0,-fz,fy],[fz,0,-fx],[-fy,fx,0]]
            const tr s = o.dl[1];
            const int bi[3] = {0, 0, 1}, bj[3] = {1, 2, 2}, bk[3] = {2, 1, 0};
            const tr bs[3] = {-1.0, 1.0, -1.0};
            for (int mm = 0; mm < 3; ++mm) {
                const double3 f = d3at(o.F, bk[mm]);
                const tr g = s * bs[mm];
                const tr sk[3][3] = {{0.0, -f.z, f.y}, {f.z, 0.0, -f.x}, {-f.y, f.x, 0.0}};
                for (int rr = 0; rr < 3; ++rr)
                    for (int cc = 0; cc < 3; ++cc) {
                        const int p = 3 * bi[mm] + rr, q = 3 * bj[mm] + cc;   // p < q always
                        const int m = p * 9 - (p * (p - 1)) / 2 + (q - p);
                        Dt[m] += g * sk[rr][cc];
                    }
            }
        }
        for (int r = 0; r < 2; ++r)
            for (int k = 0; k < 9; ++k) S[r][k] += sv[r][k];
        // controls (a, b)
        const tr datdu[2][2] = {{-2.0 * at0 / a, 0.0}, {0.0, -2.0 * at1 / b}};   // [u][row]
        for (int u = 0; u < 2; ++u) {
            tr rr[2];
            for (int r = 0; r < 2; ++r)
                rr[r] = -datdu[u][r] * lam0[r] - o.at[r] * Tu[u][r] - datdu[u][r] * o.dl[r];
            const tr t0 = o.Ji[0][0] * rr[0] + o.Ji[0][1] * rr[1];
            const tr t1 = o.Ji[1][0] * rr[0] + o.Ji[1][1] * rr[1];
            for (int k = 0; k < 9; ++k) e[u][k] += t0 * o.P[0][k] + t1 * o.P[1][k];
            Tu[u][0] += t0;
            Tu[u][1] += t1;
        }
        lam0[0] += o.dl[0];
        lam0[1] += o.dl[1];
        if (MODE == 0) {
            tet_apply(xs, o);
            x[id.x] = xs[0];
            x[id.y] = xs[1];
            x[id.z] = xs[2];
            x[id.w] = xs[3];
        }
    }
    if (LAST) {
        float a[45];
#pragma unroll
        for (int m = 0; m < 45; ++m) a[m] = (float)(-Dt[m]);
        if (pd && MODE != 2) psd9p(a);   // MODE 2: k_tet_psd projects all tets afterwards
#pragma unroll
        for (int m = 0; m < 45; ++m) Qt[(size_t)m * T + j] = a[m];
        if (eout)
            for (int k = 0; k < 9; ++k) {
                eout[(size_t)k * T + j] = (float)e[0][k];
                eout[(size_t)(9 + k) * T + j] = (float)e[1][k];
            }
    } else {
        sc.lam[2 * j] = (float)lam0[0];
        sc.lam[2 * j + 1] = (float)lam0[1];
        for (int k = 0; k < 9; ++k) {
            sc.S[(size_t)k * T + j] = (float)S[0][k];
            sc.S[(size_t)(9 + k) * T + j] = (float)S[1][k];
            sc.e[(size_t)k * T + j] = (float)e[0][k];
            sc.e[(size_t)(9 + k) * T + j] = (float)e[1][k];
        }
        for (int u = 0; u < 4; ++u) sc.Tu[(size_t)u * T + j] = (float)Tu[u / 2][u % 2];
        for (int m = 0; m < 45; ++m) sc.Dt[(size_t)m * T + j] = (float)Dt[m];
    }
}

// vec F(v) = G v_stencil (F-space image of a vertex field on the tet)
DX_INLINE void tet_Gmul(const float (&c)[4][3], const float3 (&v)[4], float *out) {
#pragma unroll
    for (int col = 0; col < 3; ++col) {
        float3 s = c[0][col] * v[0] + c[1][col] * v[1] + c[2][col] * v[2] + c[3][col] * v[3];
        put3(out, col, s);
    }
}
// q~ = Qt~ dF (45-float upper triangle, SoA)
DX_INLINE void tet_Qmul(const float *__restrict__ Qt, int T, int j, const float *dF, float *out) {
#pragma unroll
    for (int k = 0; k < 9; ++k) out[k] = 0.f;
    int m = 0;
#pragma unroll
    for (int p = 0; p < 9; ++p)
#pragma unroll
        for (int q = p; q < 9; ++q) {
            const float a = Qt[(size_t)(m++) * T + j];
            out[p] += a * dF[q];
            if (q != p) out[q] += a * dF[p];
        }
}

// Tet part of the PCG matvec (after the tile kernel wrote q): q += G^T Qt~ G p per tet with
// vector reductions, and the p.q partial dF^T Qt~ dF.  p = p_it buffer (written by the tile kernel).
__global__ void __launch_bounds__(kBlock) k_cg_tet(int it, TetDev D, const float *__restrict__ Qt, CGBufs B,
                                                   const float *__restrict__ wv, CGState s) {
    it = cg_iter(s, it);
    if (s.pp) {
        Qt = s.pp->tQ;
        B.u = s.pp->u;
    }
    if (cg_done(s, it + 1)) return;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    float acc[1] = {0.f};
    if (j < D.T) {
        const float3 *__restrict__ p = (it & 1) ? B.p1 : B.p0;
        const int4 id = D.idx[j];
        const int vid[4] = {id.x, id.y, id.z, id.w};
        float3 pv[4];
#pragma unroll
        for (int v = 0; v < 4; ++v) pv[v] = f3(p[vid[v]]);
        float c[4][3];
        tet_load_c(D, j, c);
        float dF[9], q[9];
        tet_Gmul(c, pv, dF);
        tet_Qmul(Qt, D.T, j, dF, q);
#pragma unroll
        for (int k = 0; k < 9; ++k) acc[0] += dF[k] * q[k];
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            if (!(wv[vid[v]] > 0.f)) continue;
            float3 g = c[v][0] * f3at(q, 0) + c[v][1] * f3at(q, 1) + c[v][2] * f3at(q, 2);
            tet_corner_store(D, 0, v, j, g);   // gathered per vertex by k_fold_q4 (deterministic)
        }
    }
    block_reduce_add<1>(acc, s.sc + (it + 1) * 4 + 0);
}

// q += the tets' corner contributions of this iteration, gathered per vertex in a fixed order
__global__ void k_fold_q4(int V, int it, CGBufs B, TetDev D, CGState s) {
    it = cg_iter(s, it);
    if (cg_done(s, it + 1)) return;
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V) return;
    B.q[v] = B.q[v] + tet_gather(D, 0, v);
}

// Scenes without distance constraints (tets, contacts): one PCG iteration in two launches instead
// of four (tile matvec, k_cg_tet, k_fold_q4, update).  Blocks [0, nbt) are k_cg_tet's tets, which
// form p_it at their corners on the fly (halo_p) instead of reading it; blocks [nbt, ..) form
// p_it = M^-1 r_it + beta p_{it-1} per vertex (stored, the same halo_p expression) and add
// p.(M + Qc) p to p.q.  q is not stored: k_cg_update_tet rebuilds q = (M + Qc) p + the gathered
// corner contributions.
template <int MINB>
__global__ void __launch_bounds__(kBlock, MINB) k_cg_tetv(int it, int nbt, int V, TetDev D, const float *__restrict__ Qt,
                                                    CGBufs B, const float *__restrict__ wv,
                                                    const float *__restrict__ Qc, CGState s) {
    it = cg_iter(s, it);
    if (s.pp) {
        const PcgPtrs pp = *s.pp;
        Qt = pp.tQ;
        if (Qc) Qc = pp.Qc;
        B.u = pp.u;
    }
    if (cg_done(s, it + 1)) return;
    const float3 *__restrict__ pold = (it & 1) ? B.p0 : B.p1;   // p_{it-1}
    float3 *__restrict__ pnew = (it & 1) ? B.p1 : B.p0;         // p_it
    const float beta = it > 0 ? ratio_f(s.sc[it * 4 + 1], s.sc[(it - 1) * 4 + 1]) : 0.f;
    float acc[1] = {0.f};
    if ((int)blockIdx.x < nbt) {
        const int j = blockIdx.x * blockDim.x + threadIdx.x;
        if (j < D.T) {
            // all 45 block entries in flight before the dependent corner gathers (memory-level
            // parallelism: the kernel is latency-bound at 4 CTAs / SM otherwise)
            float qt[45];
#pragma unroll
            for (int m = 0; m < 45; ++m) qt[m] = __ldg(Qt + (size_t)m * D.T + j);
            const int4 id = D.idx[j];
            const int vid[4] = {id.x, id.y, id.z, id.w};
            float3 pv[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) pv[v] = halo_p(it, vid[v], beta, B.r, pold, pnew, wv);
            float c[4][3];
            tet_load_c(D, j, c);
            float dF[9], q[9];
            tet_Gmul(c, pv, dF);
#pragma unroll
            for (int k = 0; k < 9; ++k) q[k] = 0.f;
            {
                int m = 0;
#pragma unroll
                for (int a = 0; a < 9; ++a)
#pragma unroll
                    for (int b = a; b < 9; ++b) {
                        q[a] += qt[m] * dF[b];
                        if (b != a) q[b] += qt[m] * dF[a];
                        ++m;
                    }
            }
#pragma unroll
            for (int k = 0; k < 9; ++k) acc[0] += dF[k] * q[k];
#pragma unroll
            for (int v = 0; v < 4; ++v) {
                if (!(wv[vid[v]] > 0.f)) continue;
                float3 g = c[v][0] * f3at(q, 0) + c[v][1] * f3at(q, 1) + c[v][2] * f3at(q, 2);
                tet_corner_store(D, 0, v, j, g);   // gathered by k_cg_update_tet (deterministic)
            }
        }
    } else {
        const int v = (blockIdx.x - nbt) * blockDim.x + threadIdx.x;
        if (v < V) {
            const float3 pv = halo_p(it, v, beta, B.r, pold, pnew, wv);
            if (it > 0) pnew[v] = pv;
            const float w = wv[v];
            if (w > 0.f) {
                float3 qv = (1.f / w) * pv;
                if (Qc) {
                    Sym3 A = Sym3{Qc[v], Qc[V + v], Qc[2 * (size_t)V + v], Qc[3 * (size_t)V + v],
                                  Qc[4 * (size_t)V + v], Qc[5 * (size_t)V + v]};
                    qv = qv + sym3_mul(A, pv);
                }
                acc[0] += dot3(pv, qv);
            }
        }
    }
    block_reduce_add<1>(acc, s.sc + (it + 1) * 4 + 0);
}

// PCG update after k_cg_tetv: q = (M + Qc) p + Sum of the corner contributions (fixed order), u += alpha p, r -= alpha q,
// r.M^-1 r and r.r into slot it+1.
__global__ void __launch_bounds__(kBlock) k_cg_update_tet(int V, int it, CGBufs B, const float *__restrict__ wv,
                                                          const float *__restrict__ Qc, CGState s, TetDev D) {
    it = cg_iter(s, it);
    if (s.pp) {
        const PcgPtrs pp = *s.pp;
        if (Qc) Qc = pp.Qc;
        B.u = pp.u;
    }
    if (cg_done(s, it + 1)) {
        if (s.ctl) pcg_ctl_end(s, it);
        return;
    }
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    float acc[2] = {0.f, 0.f};
    if (v < V) {
        const float3 *__restrict__ p = (it & 1) ? B.p1 : B.p0;
        const double pq = s.sc[(it + 1) * 4 + 0];
        const float alpha = pq > 0.0 ? ratio_f(s.sc[it * 4 + 1], pq) : 0.f;
        const float w = wv[v];
        const float3 pv = p[v];
        B.u[v] = B.u[v] + alpha * pv;
        float3 rv = make_float3(0.f, 0.f, 0.f);
        if (w > 0.f) {
            float3 qv = (1.f / w) * pv;
            if (Qc) {
                Sym3 A = Sym3{Qc[v], Qc[V + v], Qc[2 * (size_t)V + v], Qc[3 * (size_t)V + v],
                              Qc[4 * (size_t)V + v], Qc[5 * (size_t)V + v]};
                qv = qv + sym3_mul(A, pv);
            }
            qv = qv + tet_gather(D, 0, v);
            rv = B.r[v] - alpha * qv;
        }
        B.r[v] = rv;
        const float r2 = dot3(rv, rv);
        acc[0] += w * r2;
        acc[1] += r2;
    }
    block_reduce_add<2>(acc, s.sc + (it + 1) * 4 + 1);
    if (s.ctl) pcg_ctl_end(s, it);
}

// Tet part of the increment rhs: b -= G^T Qt~ G y, r0 -= G^T Qt~ G (y + u0), u0 = warm start
__global__ void __launch_bounds__(kBlock) k_rhs_tet(TetDev D, const float *__restrict__ Qt, const float3 *__restrict__ y,
                                                    const float3 *__restrict__ u, float3 *__restrict__ b,
                                                    float3 *__restrict__ r0, const float *__restrict__ wv) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= D.T) return;
    const int4 id = D.idx[j];
    const int vid[4] = {id.x, id.y, id.z, id.w};
    float3 yv[4], zv[4];
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        yv[v] = f3(y[vid[v]]);
        zv[v] = yv[v] + f3(u[vid[v]]);
    }
    float c[4][3];
    tet_load_c(D, j, c);
    float dy[9], dz[9], qy[9], qz[9];
    tet_Gmul(c, yv, dy);
    tet_Gmul(c, zv, dz);
    tet_Qmul(Qt, D.T, j, dy, qy);
    tet_Qmul(Qt, D.T, j, dz, qz);
#pragma unroll
    for (int v = 0; v < 4; ++v) {
        if (!(wv[vid[v]] > 0.f)) continue;
        float3 gy = c[v][0] * f3at(qy, 0) + c[v][1] * f3at(qy, 1) + c[v][2] * f3at(qy, 2);
        float3 gz = c[v][0] * f3at(qz, 0) + c[v][1] * f3at(qz, 1) + c[v][2] * f3at(qz, 2);
        tet_corner_store(D, 0, v, j, gy);
        tet_corner_store(D, 1, v, j, gz);
    }
}

// b -= G^T Qt~ G y and r0 -= G^T Qt~ G (y + u0) at every free vertex: the corner contributions of
// k_rhs_tet gathered per vertex in a fixed order (deterministic)
__global__ void k_rhs_tet_gather(int V, TetDev D, float3 *__restrict__ b, float3 *__restrict__ r0,
                                 const float *__restrict__ wv) {
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= V || !(wv[v] > 0.f)) return;
    b[v] = b[v] - tet_gather(D, 0, v);
    r0[v] = r0[v] - tet_gather(D, 1, v);
}

// dphi/d(a,b)_t += e~_u . vec F(y)   (Eq. gradientRule)
__global__ void k_grad_tet(TetDev D, const float *__restrict__ e, const float3 *__restrict__ y, float *__restrict__ g) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= D.T) return;
    const int4 id = D.idx[j];
    float3 yv[4] = {f3(y[id.x]), f3(y[id.y]), f3(y[id.z]), f3(y[id.w])};
    float c[4][3];
    tet_load_c(D, j, c);
    float dF[9];
    tet_Gmul(c, yv, dF);
    float ga = 0.f, gb = 0.f;
#pragma unroll
    for (int k = 0; k < 9; ++k) {
        ga += e[(size_t)k * D.T + j] * dF[k];
        gb += e[(size_t)(9 + k) * D.T + j] * dF[k];
    }
    g[2 * j] += ga;
    g[2 * j + 1] += gb;
}

// rest quantities: Dm^-1 (SoA) and volume from internal rest positions
__global__ void k_d2f(size_t n, const double *__restrict__ a, float *__restrict__ b) {
    const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = (float)a[i];
}

__global__ void k_tet_rest(int T, const int4 *__restrict__ idx, const float *__restrict__ xr, double *__restrict__ Dm,
                           double *__restrict__ vol) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= T) return;
    const int4 id = idx[j];
    const int v[4] = {id.x, id.y, id.z, id.w};
    double M[3][3];   // M[row][i] = (x_{i+1} - x_0)[row]
    for (int i = 0; i < 3; ++i)
        for (int r = 0; r < 3; ++r) M[r][i] = (double)xr[3 * v[i + 1] + r] - (double)xr[3 * v[0] + r];
    const double det = M[0][0] * (M[1][1] * M[2][2] - M[1][2] * M[2][1]) - M[0][1] * (M[1][0] * M[2][2] - M[1][2] * M[2][0]) +
                       M[0][2] * (M[1][0] * M[2][1] - M[1][1] * M[2][0]);
    const double id_ = 1.0 / det;
    double I[3][3];
    I[0][0] = (M[1][1] * M[2][2] - M[1][2] * M[2][1]) * id_;
    I[0][1] = (M[0][2] * M[2][1] - M[0][1] * M[2][2]) * id_;
    I[0][2] = (M[0][1] * M[1][2] - M[0][2] * M[1][1]) * id_;
    I[1][0] = (M[1][2] * M[2][0] - M[1][0] * M[2][2]) * id_;
    I[1][1] = (M[0][0] * M[2][2] - M[0][2] * M[2][0]) * id_;
    I[1][2] = (M[0][2] * M[1][0] - M[0][0] * M[1][2]) * id_;
    I[2][0] = (M[1][0] * M[2][1] - M[1][1] * M[2][0]) * id_;
    I[2][1] = (M[0][1] * M[2][0] - M[0][0] * M[2][1]) * id_;
    I[2][2] = (M[0][0] * M[1][1] - M[0][1] * M[1][0]) * id_;
    for (int i = 0; i < 3; ++i)
        for (int col = 0; col < 3; ++col) Dm[(size_t)(3 * i + col) * T + j] = I[i][col];
    vol[j] = fabs(det) / 6.0;
}

}  // namespace dx

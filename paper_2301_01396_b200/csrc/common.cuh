// Device helpers for the DiffXPBD sm_100a kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#define DX_INLINE __device__ __forceinline__

// ---------------------------------------------------------------- float3 helpers
DX_INLINE float3 f3(float4 a) { return make_float3(a.x, a.y, a.z); }
DX_INLINE float3 f3(float3 a) { return a; }
DX_INLINE float3 operator+(float3 a, float3 b) { return make_float3(a.x + b.x, a.y + b.y, a.z + b.z); }
DX_INLINE float3 operator-(float3 a, float3 b) { return make_float3(a.x - b.x, a.y - b.y, a.z - b.z); }
DX_INLINE float3 operator*(float s, float3 a) { return make_float3(s * a.x, s * a.y, s * a.z); }
DX_INLINE float3 operator-(float3 a) { return make_float3(-a.x, -a.y, -a.z); }
DX_INLINE float dot3(float3 a, float3 b) { return a.x * b.x + a.y * b.y + a.z * b.z; }
DX_INLINE float3 cross3(float3 a, float3 b) {
    return make_float3(a.y * b.z - a.z * b.y, a.z * b.x - a.x * b.z, a.x * b.y - a.y * b.x);
}

// Round-to-nearest, never-contracted arithmetic for the projection cores: the forward
// kernels and the differentiable replay kernels must produce bit-identical iterates
// (R9), independently of how the compiler schedules the surrounding code.
DX_INLINE float radd(float a, float b) { return __fadd_rn(a, b); }
DX_INLINE float rsub(float a, float b) { return __fsub_rn(a, b); }
DX_INLINE float rmul(float a, float b) { return __fmul_rn(a, b); }
DX_INLINE float rdiv(float a, float b) { return __fdiv_rn(a, b); }
DX_INLINE float rfma(float a, float b, float c) { return __fmaf_rn(a, b, c); }
DX_INLINE float rsqrt_exact(float a) { return __fsqrt_rn(a); }
DX_INLINE float3 rsub3(float3 a, float3 b) { return make_float3(rsub(a.x, b.x), rsub(a.y, b.y), rsub(a.z, b.z)); }
DX_INLINE float rdot3(float3 a, float3 b) { return rfma(a.z, b.z, rfma(a.y, b.y, rmul(a.x, b.x))); }
// p + s * d (componentwise fma)
DX_INLINE float3 rfma3(float s, float3 d, float3 p) {
    return make_float3(rfma(s, d.x, p.x), rfma(s, d.y, p.y), rfma(s, d.z, p.z));
}

// fp64 position state: positions, their differences, C, v = dx/dt
// are double; directions, multipliers, derivative blocks and the PCG are float.
DX_INLINE double3 d3(double4 a) { return make_double3(a.x, a.y, a.z); }
DX_INLINE double3 dsub3(double3 a, double3 b) {
    return make_double3(__dsub_rn(a.x, b.x), __dsub_rn(a.y, b.y), __dsub_rn(a.z, b.z));
}
DX_INLINE double ddot3(double3 a, double3 b) {
    return __fma_rn(a.z, b.z, __fma_rn(a.y, b.y, __dmul_rn(a.x, b.x)));
}
DX_INLINE float3 tof3(double3 a) { return make_float3((float)a.x, (float)a.y, (float)a.z); }

// ---------------------------------------------------------------- symmetric 3x3
struct Sym3 {
    float xx, xy, xz, yy, yz, zz;
};
DX_INLINE Sym3 sym3_zero() { return Sym3{0.f, 0.f, 0.f, 0.f, 0.f, 0.f}; }
DX_INLINE float3 sym3_mul(const Sym3 &A, float3 v) {
    return make_float3(A.xx * v.x + A.xy * v.y + A.xz * v.z,
                       A.xy * v.x + A.yy * v.y + A.yz * v.z,
                       A.xz * v.x + A.yz * v.y + A.zz * v.z);
}
DX_INLINE float sym3_quad(const Sym3 &A, float3 v) { return dot3(v, sym3_mul(A, v)); }

// A += s * (I - n n^T)
DX_INLINE void sym3_add_perp(Sym3 &A, float s, float3 n) {
    A.xx += s * (1.f - n.x * n.x);
    A.yy += s * (1.f - n.y * n.y);
    A.zz += s * (1.f - n.z * n.z);
    A.xy -= s * n.x * n.y;
    A.xz -= s * n.x * n.z;
    A.yz -= s * n.y * n.z;
}
// A += sym(a b^T) = (a b^T + b a^T)/2
DX_INLINE void sym3_add_symouter(Sym3 &A, float3 a, float3 b) {
    A.xx += a.x * b.x;
    A.yy += a.y * b.y;
    A.zz += a.z * b.z;
    A.xy += 0.5f * (a.x * b.y + a.y * b.x);
    A.xz += 0.5f * (a.x * b.z + a.z * b.x);
    A.yz += 0.5f * (a.y * b.z + a.z * b.y);
}

// Projection of a symmetric 3x3 matrix onto the PSD cone by eigenvalue clamping at 0
// (Sec.4.3.2 l.201; R5).  Cyclic Jacobi in fp32, registers only.
DX_INLINE void jacobi_rot(float (&a)[3][3], float (&v)[3][3], int p, int q) {
    float apq = a[p][q];
    if (fabsf(apq) < 1e-30f) return;
    float theta = (a[q][q] - a[p][p]) / (2.f * apq);
    float t = copysignf(1.f, theta) / (fabsf(theta) + sqrtf(theta * theta + 1.f));
    float c = rsqrtf(t * t + 1.f);
    float s = t * c;
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // A <- A J (columns p, q)
        float akp = a[k][p], akq = a[k][q];
        a[k][p] = c * akp - s * akq;
        a[k][q] = s * akp + c * akq;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {  // A <- J^T A (rows p, q)
        float apk = a[p][k], aqk = a[q][k];
        a[p][k] = c * apk - s * aqk;
        a[q][k] = s * apk + c * aqk;
    }
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        float vkp = v[k][p], vkq = v[k][q];
        v[k][p] = c * vkp - s * vkq;
        v[k][q] = s * vkp + c * vkq;
    }
}

DX_INLINE Sym3 sym3_psd(const Sym3 &A) {
    float a[3][3] = {{A.xx, A.xy, A.xz}, {A.xy, A.yy, A.yz}, {A.xz, A.yz, A.zz}};
    float v[3][3] = {{1.f, 0.f, 0.f}, {0.f, 1.f, 0.f}, {0.f, 0.f, 1.f}};
    float scale = fabsf(A.xx) + fabsf(A.yy) + fabsf(A.zz) + fabsf(A.xy) + fabsf(A.xz) + fabsf(A.yz);
    if (scale == 0.f) return A;
#pragma unroll 1
    for (int sweep = 0; sweep < 8; ++sweep) {
        float off = fabsf(a[0][1]) + fabsf(a[0][2]) + fabsf(a[1][2]);
        if (off <= 1e-9f * scale) break;
        jacobi_rot(a, v, 0, 1);
        jacobi_rot(a, v, 0, 2);
        jacobi_rot(a, v, 1, 2);
    }
    float l0 = fmaxf(a[0][0], 0.f), l1 = fmaxf(a[1][1], 0.f), l2 = fmaxf(a[2][2], 0.f);
    Sym3 Q;
    Q.xx = l0 * v[0][0] * v[0][0] + l1 * v[0][1] * v[0][1] + l2 * v[0][2] * v[0][2];
    Q.yy = l0 * v[1][0] * v[1][0] + l1 * v[1][1] * v[1][1] + l2 * v[1][2] * v[1][2];
    Q.zz = l0 * v[2][0] * v[2][0] + l1 * v[2][1] * v[2][1] + l2 * v[2][2] * v[2][2];
    Q.xy = l0 * v[0][0] * v[1][0] + l1 * v[0][1] * v[1][1] + l2 * v[0][2] * v[1][2];
    Q.xz = l0 * v[0][0] * v[2][0] + l1 * v[0][1] * v[2][1] + l2 * v[0][2] * v[2][2];
    Q.yz = l0 * v[1][0] * v[2][0] + l1 * v[1][1] * v[2][1] + l2 * v[1][2] * v[2][2];
    return Q;
}

// ---------------------------------------------------------------- vector atomics
DX_INLINE void red_add_f4(float4 *addr, float4 v) {
    // sm_90+: vectorised global reduction (one L2 atomic op for 16 bytes)
    asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(addr), "f"(v.x), "f"(v.y),
                 "f"(v.z), "f"(v.w)
                 : "memory");
}

// ---------------------------------------------------------------- bulk-async (TMA) staging
DX_INLINE uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
DX_INLINE void mbar_init(uint64_t *bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
DX_INLINE void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
DX_INLINE void mbar_wait(uint64_t *bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra WAIT_%=;\n}" ::"r"(smem_u32(bar)), "r"(parity) : "memory");
}
// global -> shared bulk copy (cp.async.bulk, completes on the mbarrier's transaction count)
DX_INLINE void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
DX_INLINE void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
DX_INLINE void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }

// packed float3 (12 B) vector fields: componentwise global reductions
DX_INLINE void red_add_f3(float3 *addr, float3 v) {
    float *a = reinterpret_cast<float *>(addr);
    atomicAdd(a, v.x);
    atomicAdd(a + 1, v.y);
    atomicAdd(a + 2, v.z);
}

// ---------------------------------------------------------------- reductions
DX_INLINE float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-reduce NV floats and atomically add them (in double) to acc[0..NV).
template <int NV>
DX_INLINE void block_reduce_add(float (&v)[NV], double *acc) {
    __shared__ float sh[NV][32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) sh[k][wid] = v[k];
    }
    __syncthreads();
    if (wid == 0) {
        const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            float s = lane < nw ? sh[k][lane] : 0.f;
            s = warp_sum(s);
            if (lane == 0 && s != 0.f) atomicAdd(acc + k, (double)s);
        }
    }
}

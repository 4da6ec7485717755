// Tetrahedral stable Neo-Hookean block constraints (Sec.5.2; R6).
// Placeholder while the cloth/contact path is validated: scenes with tets are rejected at create.
#pragma once
#include "kernels.cuh"
#include <vector>

namespace dx {
struct TetData {
    int T = 0;
};
inline void tet_create(TetData &t, int T, const int32_t *, const float *, const float *, const float *,
                       const std::vector<int32_t> &, const std::vector<int> &, int, float, bool, cudaStream_t) {
    t.T = T;
}
inline int tet_forward_sweep(TetData &, int, int, float, float, double4 *, cudaStream_t) { return 0; }
inline int tet_replay_sweep(TetData &, int, int, float, float, int, double4 *, cudaStream_t) { return 0; }
inline int tet_cg_matvec(TetData &, int, const float4 *, float4 *, const float *, CGState, cudaStream_t) { return 0; }
inline void tet_backward_alloc(TetData &, int, cudaStream_t) {}
inline void tet_grad_reset(TetData &, cudaStream_t) {}
inline int tet_rhs(TetData &, const float4 *, float4 *, const float *, cudaStream_t) { return 0; }
inline int tet_grads(TetData &, const float4 *, cudaStream_t) { return 0; }
inline void tet_grad_out(TetData &, float *, int, cudaStream_t) {}
inline void tet_set_material(TetData &, const float *, int, cudaStream_t) {}
}  // namespace dx

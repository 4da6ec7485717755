/*
 * dxpbd.h -- C ABI of the B200-native DiffXPBD hot path
 * (arXiv 2301.01396, "DiffXPBD: Differentiable Position-Based Simulation of
 * Compliant Constraint Dynamics"; line numbers below refer to PAPER.md).
 *
 * One handle = one scene (a mesh or a batch of disjoint meshes) resident on one
 * CUDA device.  All compute runs in hand-written sm_100a kernels on the stream
 * passed to each call (NULL = legacy default stream).  No torch types, no CPU
 * fallback: a call that cannot run on the device returns an error code.
 *
 * Layouts: vectors of vertices are row-major [V][3] float32 (x, y, z).  Per-frame
 * arrays are [frames][V][3].  Index buffers are int32.  Unless a call says
 * otherwise, pointers are HOST or DEVICE according to its `mem` argument
 * (DXPBD_MEM_HOST / DXPBD_MEM_DEVICE); device pointers must be on the scene's
 * device and 4-byte aligned.  The library copies every input it keeps; the
 * caller owns all pointers it passes.
 *
 * Errors: every call returns DXPBD_OK (0) or a positive error code;
 * dxpbd_last_error() returns a thread-local message for the last failure.  On a
 * CUDA error the scene is left in an unspecified state and must be destroyed.
 */
#ifndef DXPBD_H
#define DXPBD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DXPBD_OK 0
#define DXPBD_ERR_ARG 1      /* invalid argument (null pointer, size, index range) */
#define DXPBD_ERR_CUDA 2     /* CUDA runtime error (message has the CUDA string)    */
#define DXPBD_ERR_STATE 3    /* call out of order (e.g. backward before forward)    */
#define DXPBD_ERR_OOM 4      /* device allocation failed                            */
#define DXPBD_ERR_SOLVE 5    /* PCG did not reach the tolerance within max_iter     */
#define DXPBD_ERR_LIMIT 6    /* more than 256 colors, or a capacity exceeded        */

#define DXPBD_MEM_HOST 0
#define DXPBD_MEM_DEVICE 1

/* gradient families (dxpbd_grads kind, dxpbd_scene_desc.grad_flags bit = 1 << kind) */
#define DXPBD_GRAD_COMPLIANCE 0   /* d phi / d alpha_j, [E] user constraint order            */
#define DXPBD_GRAD_X0 1           /* d phi / d x_0,     [V][3]                                */
#define DXPBD_GRAD_V0 2           /* d phi / d v_0,     [V][3]                                */
#define DXPBD_GRAD_FORCES 3       /* d phi / d f_frame, [frames][V][3]                        */
#define DXPBD_GRAD_SHAPE 4        /* d phi / d beta,    [num_shape] capsule shape coefficients*/
#define DXPBD_GRAD_SPHERE 5       /* d phi / d (c_x, c_y, c_z, r), [S][4]                     */
#define DXPBD_GRAD_MATERIAL 6     /* d phi / d (a, b) per tet, [T][2]  (mu = a^2, lambda = b^2)*/
#define DXPBD_NUM_GRADS 7

/* parameter families for dxpbd_set_params */
#define DXPBD_PARAM_COMPLIANCE 0  /* alpha per distance constraint [E]                       */
#define DXPBD_PARAM_SHAPE 1       /* capsule shape coefficients beta [num_shape]             */
#define DXPBD_PARAM_MATERIAL 2    /* (a, b) per tet [T][2]                                   */
#define DXPBD_PARAM_SPHERES 3     /* spheres [S][4]                                          */

typedef struct dxpbd_scene dxpbd_scene;

/* Scene description for dxpbd_create.  ALL pointers are HOST pointers (copied). */
typedef struct dxpbd_scene_desc {
    int32_t num_vertices;            /* V >= 1                                              */
    const float *x_rest;             /* [V][3] rest positions: rest lengths, Dm^-1, volumes */
    const float *inv_mass;           /* [V] 1/kg; 0 = pinned (PAPER.md l.161 infinite mass)  */

    /* distance constraints C = |x_a - x_b| - L, L from x_rest (cloth stretch/shear/bend)  */
    int32_t num_dist;                /* E >= 0                                              */
    const int32_t *dist_idx;         /* [E][2] vertex ids, distinct, < V                     */
    const float *dist_compliance;    /* [E] alpha >= 0 (PAPER.md Eq. xpbdUenergy l.76)      */

    /* Neo-Hookean tets, C_D = ||F|| - sqrt3, C_H = det F - 1 (Sec.5.2 l.229; R6)   */
    int32_t num_tets;                /* T >= 0                                              */
    const int32_t *tet_idx;          /* [T][4] vertex ids, positive rest orientation        */
    const float *tet_a;              /* [T] a, mu = a^2                                     */
    const float *tet_b;              /* [T] b, lambda = b^2                                 */

    /* analytic colliders (Sec.4.5 l.209, Sec.5.3; R7)                    */
    int32_t num_spheres;             /* S >= 0                                              */
    const float *spheres;            /* [S][4] center xyz, radius                           */
    int32_t num_capsules;            /* K >= 0                                              */
    const float *cap_center;         /* [K][3]                                              */
    const float *cap_axis;           /* [K][3] unit axis                                    */
    const float *cap_r0;             /* [K] radius at beta = 0                              */
    const float *cap_L0;             /* [K] segment length at beta = 0                      */
    int32_t num_shape;               /* NS >= 0                                             */
    const float *cap_rbasis;         /* [K][NS] d r_k / d beta                              */
    const float *cap_lbasis;         /* [K][NS] d L_k / d beta                              */
    const float *shape_beta;         /* [NS] initial shape coefficients                     */

    float gravity[3];                /* m/s^2, applied to free vertices (R2)               */
    float frame_dt;                  /* s per frame                                         */
    int32_t substeps;                /* substeps per frame, dt = frame_dt / substeps        */
    int32_t iterations;              /* Gauss-Seidel iterations per substep (K >= 1)        */
    float thickness;                 /* collision thickness h (m)                           */
    float collision_compliance;      /* alpha of contact constraints                        */

    int32_t max_frames;              /* checkpoint capacity (frames) for forward/backward   */
    uint32_t grad_flags;             /* OR of (1 << DXPBD_GRAD_*) to accumulate             */
    int32_t pd_projection;           /* 1 = project derivative blocks (Sec.4.3.2), 0 = off  */
    float cg_tol;                    /* relative residual of the filtered PCG (e.g. 1e-6)   */
    int32_t cg_max_iter;             /* PCG iteration cap per substep                       */
    int32_t device;                  /* CUDA device ordinal                                 */

    /* batch of independent scenes in one handle (north_star (4) "batches of independent scenes"):
     * vertex_scene[v] in [0, num_scenes) tags every vertex; every distance constraint / tet must
     * lie within one scene (else DXPBD_ERR_ARG); collider_scene[c] (spheres then capsules) is the
     * scene a collider acts on, or -1 for all scenes.  NULL vertex_scene = one scene (then
     * collider_scene is ignored).  The scenes share the time stepping, the PCG solve per substep
     * (block-diagonal system, one global relative-residual test) and the loss sum; gradients are
     * per vertex / constraint / collider, so they separate by scene.  Internal vertex order is
     * (scene, Morton), so tiles rarely straddle scenes.                                       */
    int32_t num_scenes;
    const int32_t *vertex_scene;     /* [V] or NULL                                         */
    const int32_t *collider_scene;   /* [S + K] or NULL (all colliders act on every scene)  */
} dxpbd_scene_desc;

/* Build the device-resident scene: uploads topology and parameters, computes rest
 * quantities, greedy-colors the constraints (R1) and sorts them by color.
 * Cost: O(E + T) host work once.  On success *out receives the handle. */
int dxpbd_create(const dxpbd_scene_desc *desc, dxpbd_scene **out);

/* Free all device and host memory of the scene.  NULL is a no-op. */
int dxpbd_destroy(dxpbd_scene *scene);

/* Forward simulation (Sec.3.1, Eqs. xpbd l.81, position update l.85,
 * xpbdUpdateRule l.88-96): num_frames * substeps XPBD substeps from x0, v0 with
 * per-frame external forces (NULL = none), checkpointing x_n of every substep for
 * the backward pass (R9).  x0, v0: [V][3]; forces: [num_frames][V][3] (N). */
int dxpbd_forward(dxpbd_scene *scene, const float *x0, const float *v0, const float *forces,
                  int32_t num_frames, int32_t mem, void *stream);

/* Positions at the end of `frame` (0 = x0) of the last forward: out [V][3]. */
int dxpbd_positions(dxpbd_scene *scene, int32_t frame, float *out, int32_t mem, void *stream);

/* Adjoint pass (Sec.4.1-4.4, Eqs. rawAdjoint/adjointXPBD/gradientRule;
 * DESIGN.md R3-R11) over the last forward trajectory for the keyframe goal
 * phi = 1/2 sum_k sum_v W_v |x(frame k) - target_k|^2.
 * key_frames: HOST [num_keys] in 0..num_frames; targets: [num_keys][V][3];
 * weights: [V] or NULL (= 1).  Writes phi to *loss_out (HOST, may be NULL).  Gradients
 * of the families in grad_flags are recomputed from zero (read with dxpbd_grads). */
int dxpbd_backward(dxpbd_scene *scene, int32_t num_keys, const int32_t *key_frames,
                   const float *targets, const float *weights, int32_t mem, float *loss_out,
                   void *stream);

/* Copy one gradient family (DXPBD_GRAD_*) of the last backward into out (out_len
 * floats, must equal the family's size). */
int dxpbd_grads(dxpbd_scene *scene, int32_t kind, float *out, int64_t out_len, int32_t mem,
                void *stream);

/* Replace a parameter family (DXPBD_PARAM_*) between optimization iterations. */
/* Stream the force gradients of the NEXT dxpbd_backward into `out` ([frames][V][3], user order;
 * HOST or DEVICE per `mem`): each frame's slice leaves the device as soon as the backward has
 * passed that frame (HOST: D2H on a copy stream, overlapping the rest of the backward; use pinned
 * memory for the overlap).  The backward returns after every slice has arrived; the registration
 * is then cleared.  kind must be DXPBD_GRAD_FORCES (enabled in grad_flags), after a forward, with
 * out_len = frames * 3V. */
int dxpbd_grads_stream(dxpbd_scene *scene, int32_t kind, float *out, int64_t out_len, int32_t mem);

int dxpbd_set_params(dxpbd_scene *scene, int32_t kind, const float *data, int64_t len,
                     int32_t mem, void *stream);

/* Colors of the constraints of a family (0 = distance [E], 1 = tets [T]) in user
 * order into HOST out; returns the number of colors in *num_colors. */
int dxpbd_coloring(dxpbd_scene *scene, int32_t family, int32_t *out, int64_t out_len,
                   int32_t *num_colors);

/* Statistics into HOST out[0..n), n <= 24:
 *  0: total PCG iterations of the last backward, 1: max PCG iterations of one solve,
 *  2: kernel launches of the last forward, 3: of the last backward, 4: substeps solved,
 *  5: worst final relative residual, 6: last loss, 7: foreign constraint entries (tiled PCG),
 *  8: halo slots summed over tiles, 9: E, 10: V, 11: T, 12: vertex tiles, 13: TMA path on,
 *  14: PCG matvec launches of the last backward that did work (one per iteration),
 *  15: substeps of the last backward whose derivative blocks came from the forward's cache (no replay),
 *  16: wave tiles of the wavefront sweep (0: per-color launches), 17: its work items per substep,
 *  18: its ticket lag L (bandwidth of the wave-tile order + 1), 19: most neighbours of a wave tile,
 *  20: pull layout on (closed-form K = 1 blocks, csrc/pull.cuh), 21: block slots of the tile layout
 *      (constraints + cross-tile copies + padding), 22: 32-bit index words of the pull layout. */
int dxpbd_stats(dxpbd_scene *scene, double *out, int32_t n);

/* ---- Vertex-partitioned domain decomposition -------------------------
 * A group splits one scene into num_parts partitions, each owning a contiguous range of
 * Morton vertex tiles and the distance constraints whose lower endpoint lies there; every
 * partition keeps its own copy of the vertex state and the partitions exchange the vertices
 * they write after every color sweep (forward and replay), the cross-partition derivative
 * blocks after every replay, halo r / p after every PCG iteration (with all-reduced PCG
 * scalars) and the adjoint halo after every substep.  This in-process group runs all
 * partitions on desc->device with device-to-device exchanges; results equal the single scene
 * (positions bit for bit; gradients up to the order of the PCG reductions).
 * Supported: iterations == 1, pd_projection, no tets, grad_flags within FORCES | X0 | V0;
 * the scene must take the TMA path (dxpbd_stats field 13).  Same argument conventions as
 * the scene calls above. */
/* Host-only view of the pull layout of the adjoint PCG's tile kernels (csrc/pull.cuh; no GPU): the
 * layout dxpbd_create builds for scenes with closed-form K = 1 blocks (Sec.4.3 l.166-194,
 * 4.3.2 l.201: one PD-projected block Q_j per distance constraint; Eq. adjointXPBD l.150-161 is
 * solved matrix-free over them).  All ids in INTERNAL vertex order (Morton; vertex i is in tile
 * i / kTileV).  HOST outputs, each optional (NULL) except sizes:
 *   sizes[0..8) = {tiles, hcap, ycap, block slots, index words, kTileV, colors, dense slabs max};
 *   vperm [V] internal -> user vertex; sorted_ab [E][2] endpoints of the color-sorted constraints;
 *   perm [E] sorted position -> user constraint; tpos / fpos [E] block slot of the sorted
 *   constraint in its a-tile / in its b-tile (-1 if a and b share a tile);
 *   tdesc [tiles][4] = {first block slot, first index word, K0 | KS2 << 8, overflow entries};
 *   hpad [tiles][hcap] halo vertex ids (-1 padded; shared-memory slot kTileV + h);
 *   idx [index words]: per tile prim2[(K0 + 1) / 2][kTileV] (two 16-bit entries per word: other
 *   endpoint's slot (11 bits, 0x7ff = none) | lane << 11; the entry's block / y slot is
 *   k * kTileV + (i & ~31) + lane), sec2[KS2][kTileV] (y slot (15 bits) | add flag << 15, 0xffff =
 *   none), over[n] (own slot | other slot << 16; y slot K0 * kTileV + e).
 * idx_cap < index words -> DXPBD_ERR_ARG; a scene that does not take the pull layout ->
 * DXPBD_ERR_LIMIT. */
int dxpbd_pull_layout(const dxpbd_scene_desc *desc, int64_t *sizes, int32_t *vperm, int32_t *sorted_ab,
                      int32_t *perm, int32_t *tpos, int32_t *fpos, int32_t *tdesc, int32_t *hpad,
                      uint32_t *idx, int64_t idx_cap);

/* Host-only partition plan (no GPU, no allocation on a device): the plan dxpbd_group_create /
 * _create_dist build from the same host topology (Morton tiles, greedy colors R1, halos, TMA
 * layout).  Partition p owns Morton tiles [t0_p, t1_p).  Exchange lists, ids in INTERNAL vertex
 * order (Morton; internal vertex i is tile i / kTileV): kind k < nc = the endpoints of the sender's
 * color-k constraints held by the receiver (sent after every color sweep), k = nc = the sender's
 * own vertices in the receiver's tile halos (PCG vectors, adjoint), k = nc + 1 = Qt positions of
 * blocks whose b-tile copy lives in the receiver.  HOST outputs: info[0..6) = {nc, t0_rank,
 * t1_rank, V, tiles, kTileV}; counts[(k * 2 + dir) * num_parts + q], k < nc + 2, dir 0 = rank ->
 * q, dir 1 = q -> rank (p == q lists are empty); ids (optional, NULL = counts only): the lists
 * concatenated in that order, ids_cap >= sum(counts) or DXPBD_ERR_ARG; vperm (optional, [V]):
 * internal -> user vertex id.  num_parts > tiles -> DXPBD_ERR_ARG; a scene off the TMA path ->
 * DXPBD_ERR_LIMIT. */
int dxpbd_partition_plan(const dxpbd_scene_desc *desc, int32_t num_parts, int32_t rank, int32_t *info,
                         int64_t *counts, int32_t *ids, int64_t ids_cap, int32_t *vperm);

typedef struct dxpbd_group dxpbd_group;
int dxpbd_group_create(const dxpbd_scene_desc *desc, int32_t num_parts, dxpbd_group **out);
/* Distributed group: this process holds partition `rank` of `world` (one GPU per process,
 * desc->device); exchanges and PCG all-reduces go through NCCL on the call's stream.  nccl_id:
 * 128 bytes from dxpbd_nccl_unique_id() on rank 0, broadcast by the caller.  NCCL is loaded at
 * run time (the libnccl already in the process, else DXPBD_NCCL_LIB or libnccl.so.2).  All ranks
 * call every group function collectively; positions and gradients are gathered on every rank. */
int dxpbd_nccl_unique_id(void *out_128_bytes);
int dxpbd_group_create_dist(const dxpbd_scene_desc *desc, int32_t rank, int32_t world, const void *nccl_id,
                            dxpbd_group **out);
int dxpbd_group_destroy(dxpbd_group *group);
int dxpbd_group_forward(dxpbd_group *group, const float *x0, const float *v0, const float *forces,
                        int32_t num_frames, int32_t mem, void *stream);
int dxpbd_group_positions(dxpbd_group *group, int32_t frame, float *out, int32_t mem, void *stream);
int dxpbd_group_backward(dxpbd_group *group, int32_t num_keys, const int32_t *key_frames,
                         const float *targets, const float *weights, int32_t mem, float *loss_out,
                         void *stream);
/* kind: DXPBD_GRAD_FORCES, DXPBD_GRAD_X0 or DXPBD_GRAD_V0 */
int dxpbd_group_grads(dxpbd_group *group, int32_t kind, float *out, int64_t out_len, int32_t mem,
                      void *stream);
/* out[0..n), n <= 16: 0 total PCG iterations, 1 max per solve, 4 solves, 5 worst residual, 6 loss,
 * 8 vertices exchanged per substep sweep (all colors, forward or replay), 9 halo vertices
 * exchanged per PCG vector exchange, 10 cross-partition blocks per replay, 11 partitions,
 * 12 trajectory bytes of the largest local partition (its held vertices -- owned + tile halos --
 * for every substep, plus 3 rolling full-V states), 13 the single scene's trajectory bytes,
 * 14 held vertices of the largest partition. */
int dxpbd_group_stats(dxpbd_group *group, double *out, int32_t n);

/* Kernel classes timed by the opt-in event profiler (dxpbd_profile / dxpbd_kernel_times). */
#define DXPBD_K_PREDICT 0
#define DXPBD_K_DIST_PROJECT 1
#define DXPBD_K_CONTACT_PROJECT 2
#define DXPBD_K_TET_PROJECT 3
#define DXPBD_K_DIST_REPLAY 4
#define DXPBD_K_CONTACT_REPLAY 5
#define DXPBD_K_TET_REPLAY 6
#define DXPBD_K_CG_VERTEX 7
#define DXPBD_K_CG_DIST 8
#define DXPBD_K_CG_TET 9
#define DXPBD_K_CG_UPDATE 10
#define DXPBD_K_CG_INIT 11
#define DXPBD_K_RHS 12
#define DXPBD_K_ADJOINT 13
#define DXPBD_K_GRADS 14
#define DXPBD_K_OTHER 15
#define DXPBD_NUM_KCLASSES 16

/* Enable (1) / disable (0) and reset the per-kernel-class CUDA-event profiler: when enabled,
 * every kernel launch of the scene is bracketed by two events on the launching stream. */
int dxpbd_profile(dxpbd_scene *scene, int32_t enable);

/* Per-class totals since the last dxpbd_profile(scene, 1): HOST ms[n] (summed event time) and
 * count[n] (launches).  Synchronizes the scene's recorded events. */
int dxpbd_kernel_times(dxpbd_scene *scene, double *ms, double *count, int32_t n);

/* Thread-local message of the last error ("" if none). */
const char *dxpbd_last_error(void);

/* ABI version (major * 100 + minor). */
int dxpbd_version(void);

#ifdef __cplusplus
}
#endif
#endif /* DXPBD_H */

"""Thin Python binding of the DiffXPBD C-ABI (include/dxpbd.h): argument marshalling only.

Every function has the name of the C entry point it calls.  Inputs may be numpy arrays
(host memory), CPU torch tensors (host) or CUDA torch tensors (device memory, passed
without copies on the current torch stream).  There is no fallback: if the CUDA
library is missing or the device is unavailable, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional

import numpy as np

try:
    import torch
except Exception:  # pragma: no cover
    torch = None

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DXPBD_LIB") or os.path.join(_HERE, "libdxpbd.so")   # DXPBD_LIB: an A/B build

MEM_HOST, MEM_DEVICE = 0, 1
GRAD_COMPLIANCE, GRAD_X0, GRAD_V0, GRAD_FORCES, GRAD_SHAPE, GRAD_SPHERE, GRAD_MATERIAL = range(7)
PARAM_COMPLIANCE, PARAM_SHAPE, PARAM_MATERIAL, PARAM_SPHERES = range(4)
GRAD_NAMES = {"compliance": GRAD_COMPLIANCE, "x0": GRAD_X0, "v0": GRAD_V0, "forces": GRAD_FORCES,
              "shape": GRAD_SHAPE, "sphere": GRAD_SPHERE, "material": GRAD_MATERIAL}

_fp = ctypes.POINTER(ctypes.c_float)
_ip = ctypes.POINTER(ctypes.c_int32)


class SceneDesc(ctypes.Structure):
    _fields_ = [
        ("num_vertices", ctypes.c_int32), ("x_rest", ctypes.c_void_p), ("inv_mass", ctypes.c_void_p),
        ("num_dist", ctypes.c_int32), ("dist_idx", ctypes.c_void_p), ("dist_compliance", ctypes.c_void_p),
        ("num_tets", ctypes.c_int32), ("tet_idx", ctypes.c_void_p), ("tet_a", ctypes.c_void_p),
        ("tet_b", ctypes.c_void_p),
        ("num_spheres", ctypes.c_int32), ("spheres", ctypes.c_void_p),
        ("num_capsules", ctypes.c_int32), ("cap_center", ctypes.c_void_p), ("cap_axis", ctypes.c_void_p),
        ("cap_r0", ctypes.c_void_p), ("cap_L0", ctypes.c_void_p),
        ("num_shape", ctypes.c_int32), ("cap_rbasis", ctypes.c_void_p), ("cap_lbasis", ctypes.c_void_p),
        ("shape_beta", ctypes.c_void_p),
        ("gravity", ctypes.c_float * 3), ("frame_dt", ctypes.c_float), ("substeps", ctypes.c_int32),
        ("iterations", ctypes.c_int32), ("thickness", ctypes.c_float), ("collision_compliance", ctypes.c_float),
        ("max_frames", ctypes.c_int32), ("grad_flags", ctypes.c_uint32), ("pd_projection", ctypes.c_int32),
        ("cg_tol", ctypes.c_float), ("cg_max_iter", ctypes.c_int32), ("device", ctypes.c_int32),
        ("num_scenes", ctypes.c_int32), ("vertex_scene", ctypes.c_void_p), ("collider_scene", ctypes.c_void_p),
    ]


_lib = None


def lib():
    """Load libdxpbd.so; raises if it has not been built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            # compile the CUDA library on demand (nvcc, sm_100a); no fallback if that fails
            try:
                from . import build as _build
                _build.build()
            except Exception as e:  # noqa: BLE001
                raise RuntimeError(f"DiffXPBD CUDA library missing and could not be built: {LIB_PATH} ({e})") from e
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        sig = {
            "dxpbd_create": ([ctypes.POINTER(SceneDesc), ctypes.POINTER(vp)], ctypes.c_int),
            "dxpbd_destroy": ([vp], ctypes.c_int),
            "dxpbd_forward": ([vp, vp, vp, vp, i32, i32, vp], ctypes.c_int),
            "dxpbd_positions": ([vp, i32, vp, i32, vp], ctypes.c_int),
            "dxpbd_backward": ([vp, i32, vp, vp, vp, i32, vp, vp], ctypes.c_int),
            "dxpbd_grads": ([vp, i32, vp, i64, i32, vp], ctypes.c_int),
            "dxpbd_set_params": ([vp, i32, vp, i64, i32, vp], ctypes.c_int),
            "dxpbd_grads_stream": ([vp, i32, vp, i64, i32], ctypes.c_int),
            "dxpbd_coloring": ([vp, i32, vp, i64, vp], ctypes.c_int),
            "dxpbd_stats": ([vp, vp, i32], ctypes.c_int),
            "dxpbd_profile": ([vp, i32], ctypes.c_int),
            "dxpbd_kernel_times": ([vp, vp, vp, i32], ctypes.c_int),
            "dxpbd_group_create": ([ctypes.POINTER(SceneDesc), i32, ctypes.POINTER(vp)], ctypes.c_int),
            "dxpbd_group_destroy": ([vp], ctypes.c_int),
            "dxpbd_nccl_unique_id": ([vp], ctypes.c_int),
            "dxpbd_group_create_dist": ([ctypes.POINTER(SceneDesc), i32, i32, vp, ctypes.POINTER(vp)], ctypes.c_int),
            "dxpbd_group_forward": ([vp, vp, vp, vp, i32, i32, vp], ctypes.c_int),
            "dxpbd_group_positions": ([vp, i32, vp, i32, vp], ctypes.c_int),
            "dxpbd_group_backward": ([vp, i32, vp, vp, vp, i32, vp, vp], ctypes.c_int),
            "dxpbd_group_grads": ([vp, i32, vp, i64, i32, vp], ctypes.c_int),
            "dxpbd_group_stats": ([vp, vp, i32], ctypes.c_int),
            "dxpbd_partition_plan": ([ctypes.POINTER(SceneDesc), i32, i32, vp, vp, vp, i64, vp], ctypes.c_int),
            "dxpbd_pull_layout": ([ctypes.POINTER(SceneDesc), vp, vp, vp, vp, vp, vp, vp, vp, vp, i64], ctypes.c_int),
            "dxpbd_last_error": ([], ctypes.c_char_p),
            "dxpbd_version": ([], ctypes.c_int),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


EXPORTED = ["dxpbd_create", "dxpbd_destroy", "dxpbd_forward", "dxpbd_positions", "dxpbd_backward",
            "dxpbd_grads", "dxpbd_set_params", "dxpbd_coloring", "dxpbd_stats", "dxpbd_last_error",
            "dxpbd_version", "dxpbd_profile", "dxpbd_kernel_times", "dxpbd_group_create", "dxpbd_group_destroy",
            "dxpbd_group_forward", "dxpbd_group_positions", "dxpbd_group_backward", "dxpbd_group_grads",
            "dxpbd_group_stats", "dxpbd_nccl_unique_id", "dxpbd_group_create_dist", "dxpbd_partition_plan",
            "dxpbd_grads_stream", "dxpbd_pull_layout"]

KCLASSES = ["predict", "dist_project", "contact_project", "tet_project", "dist_replay", "contact_replay",
            "tet_replay", "cg_vertex", "cg_dist", "cg_tet", "cg_update", "cg_init", "rhs", "adjoint", "grads",
            "other"]


class DxpbdError(RuntimeError):
    pass


def _check(code: int, what: str):
    if code != 0:
        msg = lib().dxpbd_last_error().decode()
        raise DxpbdError(f"{what} failed (code {code}): {msg}")


# ------------------------------------------------------------------ marshalling helpers
class _Arg:
    """Holds a contiguous float32/int32 buffer alive and exposes (ptr, mem)."""

    def __init__(self, a, dtype):
        self.keep = None
        if a is None:
            self.ptr, self.mem = None, MEM_HOST
            return
        if torch is not None and isinstance(a, torch.Tensor):
            t = a.detach().to(dtype=torch.float32 if dtype == np.float32 else torch.int32).contiguous()
            self.keep = t
            self.ptr = t.data_ptr()
            self.mem = MEM_DEVICE if t.is_cuda else MEM_HOST
        else:
            arr = np.ascontiguousarray(np.asarray(a), dtype=dtype)
            self.keep = arr
            self.ptr = arr.ctypes.data
            self.mem = MEM_HOST


def _out_arg(out, n: int, what: str) -> _Arg:
    """Output buffer of a call that writes n floats: must be float32, contiguous and hold exactly n
    elements (the library writes in place; a silently converted copy would hide the result)."""
    if torch is not None and isinstance(out, torch.Tensor):
        ok = out.dtype == torch.float32 and out.is_contiguous() and out.numel() == n
    else:
        ok = (isinstance(out, np.ndarray) and out.dtype == np.float32 and out.flags.c_contiguous
              and out.flags.writeable and out.size == n)
    if not ok:
        raise ValueError(f"{what}: `out` must be a contiguous writeable float32 buffer of {n} elements "
                         f"(got {type(out).__name__} {getattr(out, 'dtype', None)} {tuple(getattr(out, 'shape', ()))})")
    a = _Arg(out, np.float32)
    assert a.ptr == (out.data_ptr() if not isinstance(out, np.ndarray) else out.ctypes.data)
    return a


def _host(a, dtype=np.float32):
    if a is None:
        return None
    if torch is not None and isinstance(a, torch.Tensor):
        a = a.detach().cpu().numpy()
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


def _stream(*args):
    if torch is not None and any(isinstance(a, torch.Tensor) and a.is_cuda for a in args):
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    return ctypes.c_void_p(0)


class DxScene:
    """Owning handle of a dxpbd_scene."""

    def __init__(self, handle, V, E, T, S, K, NS, max_frames, substeps):
        self.handle = handle
        self.V, self.E, self.T, self.S, self.K, self.NS = V, E, T, S, K, NS
        self.max_frames, self.substeps = max_frames, substeps
        self.frames = 0

    def __del__(self):
        try:
            if self.handle:
                lib().dxpbd_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


# ------------------------------------------------------------------ C entry points
def _desc(x_rest, inv_mass, dist_idx=None, dist_compliance=None, tet_idx=None, tet_a=None, tet_b=None,
          spheres=None, cap_center=None, cap_axis=None, cap_r0=None, cap_L0=None, cap_rbasis=None,
          cap_lbasis=None, shape_beta=None, gravity=(0.0, -9.81, 0.0), frame_dt=1 / 60, substeps=1,
          iterations=1, thickness=0.0, collision_compliance=0.0, max_frames=1, grad_flags=0,
          pd_projection=1, cg_tol=1e-6, cg_max_iter=500, device=0, vertex_scene=None, collider_scene=None):
    """dxpbd_scene_desc from host arrays; returns (desc, kept arrays, handle dimensions)."""
    keep = []

    def h(a, dt=np.float32):
        arr = _host(a, dt)
        keep.append(arr)
        return None if arr is None else arr.ctypes.data

    x_rest = _host(x_rest)
    V = int(x_rest.reshape(-1, 3).shape[0])
    E = 0 if dist_idx is None else int(np.asarray(dist_idx).reshape(-1, 2).shape[0])
    T = 0 if tet_idx is None else int(np.asarray(tet_idx).reshape(-1, 4).shape[0])
    S = 0 if spheres is None else int(np.asarray(spheres).reshape(-1, 4).shape[0])
    K = 0 if cap_center is None else int(np.asarray(cap_center).reshape(-1, 3).shape[0])
    NS = 0 if shape_beta is None else int(np.asarray(shape_beta).size)
    d = SceneDesc()
    d.num_vertices = V
    d.x_rest = h(x_rest)
    d.inv_mass = h(inv_mass)
    d.num_dist = E
    d.dist_idx = h(dist_idx, np.int32) if E else None
    d.dist_compliance = h(dist_compliance) if E else None
    d.num_tets = T
    d.tet_idx = h(tet_idx, np.int32) if T else None
    d.tet_a = h(tet_a) if T else None
    d.tet_b = h(tet_b) if T else None
    d.num_spheres = S
    d.spheres = h(spheres) if S else None
    d.num_capsules = K
    if K:
        d.cap_center, d.cap_axis = h(cap_center), h(cap_axis)
        d.cap_r0, d.cap_L0 = h(cap_r0), h(cap_L0)
    d.num_shape = NS if K else 0
    if K and NS:
        d.cap_rbasis, d.cap_lbasis, d.shape_beta = h(cap_rbasis), h(cap_lbasis), h(shape_beta)
    d.gravity = (ctypes.c_float * 3)(*[float(g) for g in gravity])
    d.frame_dt = float(frame_dt)
    d.substeps = int(substeps)
    d.iterations = int(iterations)
    d.thickness = float(thickness)
    d.collision_compliance = float(collision_compliance)
    d.max_frames = int(max_frames)
    d.grad_flags = int(grad_flags)
    d.pd_projection = int(pd_projection)
    d.cg_tol = float(cg_tol)
    d.cg_max_iter = int(cg_max_iter)
    d.device = int(device)
    if vertex_scene is not None:
        vs = np.asarray(vertex_scene, np.int32).reshape(-1)
        d.num_scenes = int(vs.max()) + 1 if vs.size else 1
        d.vertex_scene = h(vs, np.int32)
        d.collider_scene = h(collider_scene, np.int32) if collider_scene is not None and S + K else None
    return d, keep, (V, E, T, S, K, NS if K else 0, int(max_frames), int(substeps))


def dxpbd_create(x_rest, inv_mass, **kw) -> DxScene:
    d, keep, dims = _desc(x_rest, inv_mass, **kw)
    out = ctypes.c_void_p()
    _check(lib().dxpbd_create(ctypes.byref(d), ctypes.byref(out)), "dxpbd_create")
    return DxScene(out.value, *dims)


def dxpbd_destroy(scene: DxScene):
    if scene.handle:
        _check(lib().dxpbd_destroy(scene.handle), "dxpbd_destroy")
        scene.handle = None


def _mem_of(*args):
    mems = {a.mem for a in args if a.ptr is not None}
    if len(mems) > 1:
        raise ValueError("mixing host and device buffers in one call")
    return mems.pop() if mems else MEM_HOST


def dxpbd_forward(scene: DxScene, x0, v0, forces=None, num_frames: int = 1):
    ax, av, af = _Arg(x0, np.float32), _Arg(v0, np.float32), _Arg(forces, np.float32)
    mem = _mem_of(ax, av, af)
    _check(lib().dxpbd_forward(scene.handle, ax.ptr, av.ptr, af.ptr, int(num_frames), mem,
                               _stream(x0, v0, forces)), "dxpbd_forward")
    scene.frames = int(num_frames)


def dxpbd_positions(scene: DxScene, frame: int, out=None):
    if out is None:
        out = np.zeros((scene.V, 3), np.float32)
    a = _out_arg(out, 3 * scene.V, "dxpbd_positions")
    _check(lib().dxpbd_positions(scene.handle, int(frame), a.ptr, a.mem, _stream(out)), "dxpbd_positions")
    return out


def dxpbd_backward(scene: DxScene, key_frames, targets, weights=None) -> float:
    kf = np.ascontiguousarray(np.asarray(key_frames, np.int32).reshape(-1))
    at, aw = _Arg(targets, np.float32), _Arg(weights, np.float32)
    mem = _mem_of(at, aw)
    loss = ctypes.c_float(0.0)
    _check(lib().dxpbd_backward(scene.handle, len(kf), kf.ctypes.data, at.ptr, aw.ptr, mem,
                                ctypes.byref(loss), _stream(targets, weights)), "dxpbd_backward")
    return float(loss.value)


def _grad_size(scene: DxScene, kind: int):
    return {GRAD_COMPLIANCE: (scene.E,), GRAD_X0: (scene.V, 3), GRAD_V0: (scene.V, 3),
            GRAD_FORCES: (max(scene.frames, 1), scene.V, 3), GRAD_SHAPE: (scene.NS,),
            GRAD_SPHERE: (scene.S, 4), GRAD_MATERIAL: (scene.T, 2)}[kind]


def dxpbd_grads(scene: DxScene, kind, out=None):
    kind = GRAD_NAMES.get(kind, kind)
    shape = _grad_size(scene, kind)
    if out is None:
        out = np.zeros(shape, np.float32)
    n = int(np.prod(shape))
    a = _out_arg(out, n, "dxpbd_grads")
    _check(lib().dxpbd_grads(scene.handle, int(kind), a.ptr, n, a.mem, _stream(out)), "dxpbd_grads")
    return out


def dxpbd_grads_stream(scene: DxScene, kind, out):
    """Register `out` (host numpy / pinned torch CPU tensor, or a CUDA tensor) to receive the force
    gradients of the NEXT dxpbd_backward, frame by frame as the backward passes them (include/dxpbd.h).
    `out` must stay alive until that backward returns."""
    kind = GRAD_NAMES.get(kind, kind)
    shape = _grad_size(scene, kind)
    n = int(np.prod(shape))
    a = _out_arg(out, n, "dxpbd_grads_stream")
    scene._stream_keep = (out, a)
    _check(lib().dxpbd_grads_stream(scene.handle, int(kind), a.ptr, n, a.mem), "dxpbd_grads_stream")
    return out


def dxpbd_set_params(scene: DxScene, kind: int, data):
    a = _Arg(data, np.float32)
    n = int(np.asarray(a.keep.shape).prod()) if a.keep is not None else 0
    _check(lib().dxpbd_set_params(scene.handle, int(kind), a.ptr, n, a.mem, _stream(data)), "dxpbd_set_params")


def dxpbd_coloring(scene: DxScene, family: int = 0) -> np.ndarray:
    n = scene.E if family == 0 else scene.T
    out = np.zeros(n, np.int32)
    nc = ctypes.c_int32(0)
    _check(lib().dxpbd_coloring(scene.handle, int(family), out.ctypes.data, n, ctypes.byref(nc)),
           "dxpbd_coloring")
    return out


def dxpbd_stats(scene: DxScene) -> dict:
    out = np.zeros(24, np.float64)
    _check(lib().dxpbd_stats(scene.handle, out.ctypes.data, 24), "dxpbd_stats")
    return dict(cg_iters_total=out[0], cg_iters_max=out[1], fwd_launches=out[2], bwd_launches=out[3],
                solves=out[4], worst_relres=out[5], loss=out[6], n_foreign=out[7], halo_total=out[8],
                E=out[9], V=out[10], T=out[11], tiles=out[12], tma=bool(out[13]), cg_matvecs=out[14],
                cached_substeps=out[15], wave_tiles=out[16], wave_items=out[17], wave_lag=out[18],
                wave_max_neighbours=out[19], pull=bool(out[20]), block_slots=out[21], pull_index_words=out[22])


def dxpbd_profile(scene: DxScene, enable: bool = True):
    _check(lib().dxpbd_profile(scene.handle, int(bool(enable))), "dxpbd_profile")


def dxpbd_kernel_times(scene: DxScene) -> dict:
    n = len(KCLASSES)
    ms = np.zeros(n, np.float64)
    cnt = np.zeros(n, np.float64)
    _check(lib().dxpbd_kernel_times(scene.handle, ms.ctypes.data, cnt.ctypes.data, n), "dxpbd_kernel_times")
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KCLASSES) if cnt[i] > 0}


def dxpbd_last_error() -> str:
    return lib().dxpbd_last_error().decode()


def dxpbd_version() -> int:
    return int(lib().dxpbd_version())


# ------------------------------------------------------------------ convenience
# ------------------------------------------------------------------ partition groups (domain decomposition)
class DxGroup(DxScene):
    """Owning handle of a dxpbd_group (one scene split into num_parts vertex partitions)."""

    def __init__(self, handle, parts, *dims):
        super().__init__(handle, *dims)
        self.parts = parts

    def __del__(self):
        try:
            if self.handle:
                lib().dxpbd_group_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def dxpbd_group_create(x_rest, inv_mass, num_parts: int = 2, **kw) -> DxGroup:
    d, keep, dims = _desc(x_rest, inv_mass, **kw)
    out = ctypes.c_void_p()
    _check(lib().dxpbd_group_create(ctypes.byref(d), int(num_parts), ctypes.byref(out)), "dxpbd_group_create")
    return DxGroup(out.value, int(num_parts), *dims)


def dxpbd_partition_plan(x_rest, inv_mass, num_parts: int, rank: int, **kw) -> dict:
    """Host-only partition plan of the domain decomposition (include/dxpbd.h dxpbd_partition_plan):
    {"colors", "t0", "t1", "V", "tiles", "tile_v", "vperm", "send": {kind: {q: ids}}, "recv": {kind: {q: ids}}}
    with kind = color index, "halo" or "blocks"; ids in internal (Morton) vertex order, vperm maps
    internal -> user vertex ids."""
    d, keep, dims = _desc(x_rest, inv_mass, **kw)
    P = int(num_parts)
    info = np.zeros(8, np.int32)
    # counts size needs the color count: query with a generous bound first
    counts = np.zeros(2 * P * (256 + 2), np.int64)
    _check(lib().dxpbd_partition_plan(ctypes.byref(d), P, int(rank), info.ctypes.data, counts.ctypes.data, None, 0,
                                      None), "dxpbd_partition_plan")
    nc = int(info[0])
    total = int(counts[: 2 * P * (nc + 2)].sum())
    ids = np.zeros(max(total, 1), np.int32)
    vperm = np.zeros(int(info[3]), np.int32)
    _check(lib().dxpbd_partition_plan(ctypes.byref(d), P, int(rank), info.ctypes.data, counts.ctypes.data,
                                      ids.ctypes.data, total, vperm.ctypes.data), "dxpbd_partition_plan")
    out = {"colors": nc, "t0": int(info[1]), "t1": int(info[2]), "V": int(info[3]), "tiles": int(info[4]),
           "tile_v": int(info[5]), "vperm": vperm, "send": {}, "recv": {}}
    o = 0
    for k in range(nc + 2):
        name = k if k < nc else ("halo" if k == nc else "blocks")
        for dirn, key in ((0, "send"), (1, "recv")):
            for q in range(P):
                n = int(counts[(k * 2 + dirn) * P + q])
                out[key].setdefault(name, {})[q] = ids[o:o + n].copy()
                o += n
    return out


def dxpbd_pull_layout(x_rest, inv_mass, **kw) -> dict:
    """Host-only view of the pull layout of the PCG tile kernels (include/dxpbd.h dxpbd_pull_layout):
    sizes plus the arrays vperm, sorted_ab, perm, tpos, fpos, tdesc, hpad, idx (numpy, internal vertex ids)."""
    d, keep, dims = _desc(x_rest, inv_mass, **kw)
    sizes = np.zeros(8, np.int64)
    _check(lib().dxpbd_pull_layout(ctypes.byref(d), sizes.ctypes.data, None, None, None, None, None, None, None, None, 0),
           "dxpbd_pull_layout")
    nt, hcap, ycap, slots, words, tile_v, nc, k0max = (int(v) for v in sizes)
    V, E = int(d.num_vertices), int(d.num_dist)
    out = dict(tiles=nt, hcap=hcap, ycap=ycap, block_slots=slots, index_words=words, tile_v=tile_v, colors=nc,
               dense_slabs_max=k0max, vperm=np.zeros(V, np.int32), sorted_ab=np.zeros((E, 2), np.int32),
               perm=np.zeros(E, np.int32), tpos=np.zeros(E, np.int32), fpos=np.zeros(E, np.int32),
               tdesc=np.zeros((nt, 4), np.int32), hpad=np.zeros((nt, hcap), np.int32), idx=np.zeros(words, np.uint32))
    _check(lib().dxpbd_pull_layout(ctypes.byref(d), sizes.ctypes.data, *(out[k].ctypes.data for k in
                                   ("vperm", "sorted_ab", "perm", "tpos", "fpos", "tdesc", "hpad", "idx")), words),
           "dxpbd_pull_layout")
    return out


def dxpbd_nccl_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0), to be broadcast to the other ranks."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().dxpbd_nccl_unique_id(buf), "dxpbd_nccl_unique_id")
    return buf.raw


def dxpbd_group_create_dist(x_rest, inv_mass, rank: int, world: int, nccl_id: bytes, **kw) -> DxGroup:
    """Partition `rank` of a world-size domain decomposition, one GPU per process (NCCL transport)."""
    d, keep, dims = _desc(x_rest, inv_mass, **kw)
    uid = ctypes.create_string_buffer(bytes(nccl_id), 128)
    out = ctypes.c_void_p()
    _check(lib().dxpbd_group_create_dist(ctypes.byref(d), int(rank), int(world), uid, ctypes.byref(out)),
           "dxpbd_group_create_dist")
    return DxGroup(out.value, int(world), *dims)


def dxpbd_group_destroy(group: DxGroup):
    if group.handle:
        _check(lib().dxpbd_group_destroy(group.handle), "dxpbd_group_destroy")
        group.handle = None


def dxpbd_group_forward(group: DxGroup, x0, v0, forces=None, num_frames: int = 1):
    ax, av, af = _Arg(x0, np.float32), _Arg(v0, np.float32), _Arg(forces, np.float32)
    mem = _mem_of(ax, av, af)
    _check(lib().dxpbd_group_forward(group.handle, ax.ptr, av.ptr, af.ptr, int(num_frames), mem,
                                     _stream(x0, v0, forces)), "dxpbd_group_forward")
    group.frames = int(num_frames)


def dxpbd_group_positions(group: DxGroup, frame: int, out=None):
    if out is None:
        out = np.zeros((group.V, 3), np.float32)
    a = _out_arg(out, 3 * group.V, "dxpbd_group_positions")
    _check(lib().dxpbd_group_positions(group.handle, int(frame), a.ptr, a.mem, _stream(out)), "dxpbd_group_positions")
    return out


def dxpbd_group_backward(group: DxGroup, key_frames, targets, weights=None) -> float:
    kf = np.ascontiguousarray(np.asarray(key_frames, np.int32).reshape(-1))
    at, aw = _Arg(targets, np.float32), _Arg(weights, np.float32)
    mem = _mem_of(at, aw)
    loss = ctypes.c_float(0.0)
    _check(lib().dxpbd_group_backward(group.handle, len(kf), kf.ctypes.data, at.ptr, aw.ptr, mem,
                                      ctypes.byref(loss), _stream(targets, weights)), "dxpbd_group_backward")
    return float(loss.value)


def dxpbd_group_grads(group: DxGroup, kind, out=None):
    kind = GRAD_NAMES.get(kind, kind)
    shape = _grad_size(group, kind)
    if out is None:
        out = np.zeros(shape, np.float32)
    a = _out_arg(out, int(np.prod(shape)), "dxpbd_group_grads")
    _check(lib().dxpbd_group_grads(group.handle, int(kind), a.ptr, int(np.prod(shape)), a.mem, _stream(out)),
           "dxpbd_group_grads")
    return out


def dxpbd_group_stats(group: DxGroup) -> dict:
    out = np.zeros(16, np.float64)
    _check(lib().dxpbd_group_stats(group.handle, out.ctypes.data, 16), "dxpbd_group_stats")
    return dict(cg_iters_total=out[0], cg_iters_max=out[1], solves=out[4], worst_relres=out[5], loss=out[6],
                xchg_sweep=out[8], xchg_halo=out[9], xchg_blocks=out[10], parts=out[11],
                traj_bytes_part=out[12], traj_bytes_single=out[13], held_max=out[14])


def scene_kwargs(scene) -> dict:
    """Map a synth.Scene (duck-typed) onto dxpbd_create keyword arguments."""
    s = scene
    kw = dict(x_rest=s.x_rest, inv_mass=s.inv_mass, gravity=tuple(s.gravity), frame_dt=s.frame_dt,
              substeps=s.substeps, iterations=s.iterations, thickness=s.thickness,
              collision_compliance=s.collision_compliance)
    if len(s.dist_idx):
        kw.update(dist_idx=s.dist_idx, dist_compliance=s.dist_compliance)
    if len(s.tet_idx):
        kw.update(tet_idx=s.tet_idx, tet_a=s.tet_a, tet_b=s.tet_b)
    if len(s.spheres):
        kw.update(spheres=s.spheres)
    if len(s.cap_center):
        kw.update(cap_center=s.cap_center, cap_axis=s.cap_axis, cap_r0=s.cap_r0, cap_L0=s.cap_L0)
        if len(s.shape_beta):
            kw.update(cap_rbasis=s.cap_rbasis, cap_lbasis=s.cap_lbasis, shape_beta=s.shape_beta)
    return kw


def batch_scene_kwargs(scenes) -> dict:
    """One handle for a batch of independent synth.Scenes (include/dxpbd.h: vertex_scene /
    collider_scene): vertices, constraints, tets and colliders concatenated in scene order with
    index offsets; capsule shape bases block-diagonal (each scene keeps its own coefficients).
    The scenes must share the time stepping, gravity and collision parameters."""
    s0 = scenes[0]
    for s in scenes[1:]:
        for k in ("frame_dt", "substeps", "iterations", "thickness", "collision_compliance"):
            if getattr(s, k) != getattr(s0, k):
                raise ValueError(f"batch scenes differ in {k}")
        if tuple(s.gravity) != tuple(s0.gravity):
            raise ValueError("batch scenes differ in gravity")
    voff = np.cumsum([0] + [s.num_vertices for s in scenes])
    cat = lambda xs: np.concatenate([np.asarray(x) for x in xs], 0)  # noqa: E731
    kw = dict(x_rest=cat([s.x_rest for s in scenes]), inv_mass=cat([s.inv_mass for s in scenes]),
              gravity=tuple(s0.gravity), frame_dt=s0.frame_dt, substeps=s0.substeps, iterations=s0.iterations,
              thickness=s0.thickness, collision_compliance=s0.collision_compliance,
              vertex_scene=np.repeat(np.arange(len(scenes), dtype=np.int32), [s.num_vertices for s in scenes]))
    if sum(len(s.dist_idx) for s in scenes):
        kw.update(dist_idx=cat([np.asarray(s.dist_idx).reshape(-1, 2) + voff[b] for b, s in enumerate(scenes)]),
                  dist_compliance=cat([s.dist_compliance for s in scenes]))
    if sum(len(s.tet_idx) for s in scenes):
        kw.update(tet_idx=cat([np.asarray(s.tet_idx).reshape(-1, 4) + voff[b] for b, s in enumerate(scenes)]),
                  tet_a=cat([s.tet_a for s in scenes]), tet_b=cat([s.tet_b for s in scenes]))
    csc = []
    if sum(len(s.spheres) for s in scenes):
        kw.update(spheres=cat([np.asarray(s.spheres).reshape(-1, 4) for s in scenes]))
        csc += [b for b, s in enumerate(scenes) for _ in range(len(s.spheres))]
    if sum(len(s.cap_center) for s in scenes):
        kw.update(cap_center=cat([np.asarray(s.cap_center).reshape(-1, 3) for s in scenes]),
                  cap_axis=cat([np.asarray(s.cap_axis).reshape(-1, 3) for s in scenes]),
                  cap_r0=cat([s.cap_r0 for s in scenes]), cap_L0=cat([s.cap_L0 for s in scenes]))
        csc += [b for b, s in enumerate(scenes) for _ in range(len(s.cap_center))]
        ns = [len(s.shape_beta) if len(s.cap_center) else 0 for s in scenes]
        if sum(ns):
            K = sum(len(s.cap_center) for s in scenes)
            Rb, Lb = np.zeros((K, sum(ns))), np.zeros((K, sum(ns)))
            k0, n0 = 0, 0
            for s, n in zip(scenes, ns):
                k1 = k0 + len(s.cap_center)
                if n:
                    Rb[k0:k1, n0:n0 + n] = np.asarray(s.cap_rbasis).reshape(-1, n)
                    Lb[k0:k1, n0:n0 + n] = np.asarray(s.cap_lbasis).reshape(-1, n)
                k0, n0 = k1, n0 + n
            kw.update(cap_rbasis=Rb, cap_lbasis=Lb,
                      shape_beta=cat([s.shape_beta for s, n in zip(scenes, ns) if n]))
    if csc:
        kw.update(collider_scene=np.asarray(csc, np.int32))
    return kw


def batch_inputs(scenes, frames: int):
    """x0, v0, forces ([frames][V][3] or None) and targets ([keys][V][3]) of a batch, concatenated
    along vertices in scene order (the scenes must share their keyframes)."""
    kf = [list(np.asarray(s.key_frames).tolist()) for s in scenes]
    if any(k != kf[0] for k in kf):
        raise ValueError("batch scenes differ in key frames")
    x0 = np.concatenate([s.x0 for s in scenes], 0)
    v0 = np.concatenate([s.v0 for s in scenes], 0)
    forces = None
    if any(s.forces is not None for s in scenes):
        forces = np.concatenate([s.forces[:frames] if s.forces is not None else np.zeros((frames, s.num_vertices, 3))
                                 for s in scenes], 1)
    targets = None if scenes[0].targets is None else np.concatenate([s.targets for s in scenes], 1)
    return x0, v0, forces, np.asarray(kf[0], np.int32), targets


def batch_split(a, scenes, axis: int = 0):
    """Split a per-vertex result of a batch ([..][V][..] along `axis`) back into per-scene arrays."""
    cuts = np.cumsum([s.num_vertices for s in scenes])[:-1]
    return np.split(np.asarray(a), cuts, axis=axis)


def flags(*names) -> int:
    f = 0
    for n in names:
        f |= 1 << GRAD_NAMES[n]
    return f

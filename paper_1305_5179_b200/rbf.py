"""Thin Python binding of the C-ABI in include/rbf.h (argument marshalling only).

Every step of the path runs in librbf.so's CUDA kernels; torch supplies device
memory, the current stream and process groups.  There is no CPU fallback: if
the library is missing or the device is not a B200 the calls raise.

Names follow include/rbf.h (and the paper's notation: sigma, centres, w for the
coefficients c_j of Eq.3, the grid xi of Eq.5).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "librbf.so")

RBF_OK, RBF_EINVAL, RBF_ENOMEM, RBF_ECUDA, RBF_ENCCL, RBF_EUNSUPPORTED = range(6)
RBF_F32, RBF_F64 = 0, 1
OP_AUTO, OP_ONESIDED, OP_SYM, OP_SYM_WIDE, OP_SYM_ROT = range(5)   # rbf_op_variant


class RbfError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{_STATUS.get(status, status)}: {msg}")
        self.status = status


_STATUS = {0: "RBF_OK", 1: "RBF_EINVAL", 2: "RBF_ENOMEM", 3: "RBF_ECUDA", 4: "RBF_ENCCL",
           5: "RBF_EUNSUPPORTED"}


# ----------------------------------------------------------------- structs --
class _Kernel(C.Structure):
    _fields_ = [("sigma", C.c_double), ("cutoff_sigmas", C.c_double), ("amplitude", C.c_double)]


class _CellCfg(C.Structure):
    _fields_ = [("cell_edge", C.c_double), ("tile_cap", C.c_int), ("tile_span", C.c_int), ("tile_mode", C.c_int)]


class _PrecondCfg(C.Structure):
    _fields_ = [("kind", C.c_int), ("core_target", C.c_int), ("overlap_sigmas", C.c_double),
                ("max_ext", C.c_int), ("shift", C.c_double), ("local_fp32", C.c_int),
                ("pivot", C.c_int), ("w_layout", C.c_int)]


class _GmresCfg(C.Structure):
    _fields_ = [("restart", C.c_int), ("rtol", C.c_double), ("phase1_rtol", C.c_double),
                ("max_iters", C.c_int), ("polish_fp64", C.c_int), ("cgs_passes", C.c_int),
                ("op_variant", C.c_int), ("basis_fp64", C.c_int),
                ("history", C.POINTER(C.c_double)), ("history_true", C.POINTER(C.c_double)),
                ("history_cap", C.c_int), ("x0", C.c_void_p)]


class SolveReport(C.Structure):
    _fields_ = [("iters_phase1", C.c_int), ("iters_phase2", C.c_int), ("restarts", C.c_int),
                ("converged", C.c_int), ("breakdown", C.c_int),
                ("history_len", C.c_int), ("history_true_len", C.c_int),
                ("rel_residual_true", C.c_double), ("rel_residual_est", C.c_double),
                ("t_setup", C.c_double), ("t_phase1", C.c_double), ("t_phase2", C.c_double),
                ("nblocks", C.c_int64), ("precond_bytes", C.c_int64),
                ("matvecs_f32", C.c_int64), ("matvecs_f64", C.c_int64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class _Grid(C.Structure):
    _fields_ = [("lo", C.c_double * 3), ("hi", C.c_double * 3), ("n", C.c_int * 3)]


class _CellsDesc(C.Structure):
    _fields_ = [("n", C.c_int64), ("dim", C.c_int * 3), ("lo", C.c_float * 3), ("inv_h", C.c_float),
                ("cell_edge", C.c_double), ("reach", C.c_int), ("ncell", C.c_int64),
                ("ntiles", C.c_int64), ("nonempty_cells", C.c_int64)]


_P = C.c_void_p
EXPORTS = {
    # name: (restype, argtypes)
    "rbf_create": (C.c_int, [C.POINTER(_P), C.c_int, _P, _P, C.c_int, C.c_int]),
    "rbf_destroy": (None, [_P]),
    "rbf_status_str": (C.c_char_p, [C.c_int]),
    "rbf_last_error": (C.c_char_p, []),
    "rbf_abi_version": (C.c_int, []),
    "rbf_launch_count": (C.c_int64, []),
    "rbf_pool_reserve": (C.c_int, [_P, C.c_uint64]),
    "rbf_pool_stats": (C.c_int, [_P, C.POINTER(C.c_uint64)]),
    "rbf_nccl_unique_id": (C.c_int, [_P]),
    "rbf_loopback_group_create": (C.c_int, [C.c_int, C.POINTER(_P)]),
    "rbf_loopback_group_free": (None, [_P]),
    "rbf_create_loopback": (C.c_int, [C.POINTER(_P), C.c_int, _P, _P, C.c_int]),
    "rbf_create_ipc": (C.c_int, [C.POINTER(_P), C.c_int, _P, _P, C.c_int, C.c_int]),
    "rbf_ctx_peer_memory": (C.c_int, [_P, C.c_int]),
    "rbf_ctx_neighbour_lists": (C.c_int, [_P, C.c_int]),
    "rbf_ctx_grid_separable": (C.c_int, [_P, C.c_int]),
    "rbf_slab_plan": (C.c_int, [_P, _P, C.c_int, C.c_int, C.c_int, _P, _P, _P, _P, _P]),
    "rbf_extend_points": (C.c_int, [_P, _P, _P, C.c_int64, C.c_double, C.c_double, _P, _P]),
    "rbf_build_cells_shard": (C.c_int, [_P, _P, C.c_int64, C.c_int64, C.POINTER(_Kernel), C.POINTER(_CellCfg),
                                        C.POINTER(_P)]),
    "rbf_gmres_solve_shard": (C.c_int, [_P, _P, C.POINTER(_Kernel), _P, C.POINTER(_PrecondCfg),
                                        C.POINTER(_GmresCfg), _P, C.c_int64, C.c_int64, _P, C.POINTER(SolveReport)]),
    "rbf_build_cells": (C.c_int, [_P, _P, C.c_int64, C.POINTER(_Kernel), C.POINTER(_CellCfg),
                                  C.POINTER(_P)]),
    "rbf_cells_free": (None, [_P]),
    "rbf_cells_info": (C.c_int, [_P, C.POINTER(_CellsDesc)]),
    "rbf_cells_slab": (C.c_int, [_P, _P]),
    "rbf_cells_view": (C.c_int, [_P, C.POINTER(_P), C.POINTER(_P), C.POINTER(_P), C.POINTER(_P)]),
    "rbf_matvec": (C.c_int, [_P, _P, C.POINTER(_Kernel), C.c_int, _P, _P]),
    "rbf_matvec_op": (C.c_int, [_P, _P, C.POINTER(_Kernel), C.c_int, C.c_int, _P, _P]),
    "rbf_matvec_pairs": (C.c_int, [_P, _P, C.POINTER(_Kernel), C.POINTER(C.c_int64),
                                   C.POINTER(C.c_int64)]),
    "rbf_precond_create": (C.c_int, [_P, _P, C.POINTER(_Kernel), C.POINTER(_PrecondCfg),
                                     C.POINTER(_P)]),
    "rbf_precond_free": (None, [_P]),
    "rbf_precond_apply": (C.c_int, [_P, _P, _P, _P]),
    "rbf_precond_blocks": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), _P, _P, _P, _P]),
    "rbf_gmres_solve": (C.c_int, [_P, _P, C.POINTER(_Kernel), _P, C.POINTER(_PrecondCfg),
                                  C.POINTER(_GmresCfg), _P, _P, C.POINTER(SolveReport)]),
    "rbf_eval_grid": (C.c_int, [_P, _P, C.POINTER(_Kernel), _P, C.POINTER(_Grid), _P]),
    "rbf_eval_grid_slab": (C.c_int, [_P, _P, C.POINTER(_Kernel), _P, C.POINTER(_Grid), _P, C.POINTER(C.c_int64),
                                     C.POINTER(C.c_int64)]),
    "rbf_eval_grid_pairs": (C.c_int, [_P, _P, C.POINTER(_Kernel), C.POINTER(_Grid), C.POINTER(C.c_int64),
                                      C.POINTER(C.c_int64)]),
    "rbf_zero_set": (C.c_int, [_P, _P, C.POINTER(_Grid), _P, C.c_int64, C.c_double, _P, C.c_int64,
                               C.POINTER(C.c_int64)]),
    "rbf_eval_grid_masked": (C.c_int, [_P, _P, C.POINTER(_Kernel), _P, C.POINTER(_Grid), _P, C.c_int64,
                                       C.c_double, _P]),
    "rbf_mesh_from_field": (C.c_int, [_P, _P, C.POINTER(_Grid), _P, C.c_int64, C.c_double, C.POINTER(_P)]),
    "rbf_isosurface": (C.c_int, [_P, _P, C.POINTER(_Kernel), _P, C.POINTER(_Grid), _P, C.c_int64, C.c_double, _P,
                                 C.POINTER(_P)]),
    "rbf_mesh_view": (C.c_int, [_P, C.POINTER(_P), C.POINTER(C.c_int64), C.POINTER(_P), C.POINTER(C.c_int64)]),
    "rbf_mesh_free": (None, [_P]),
    "rbf_assemble": (C.c_int, [_P, _P, C.POINTER(_Kernel), C.POINTER(_P)]),
    "rbf_csr_free": (None, [_P]),
    "rbf_csr_info": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_double)]),
    "rbf_csr_spmv": (C.c_int, [_P, _P, _P, _P]),
    "rbf_nn_distance": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, _P]),
    "rbf_density": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, _P]),
    "rbf_sigma_auto": (C.c_int, [_P, _P, C.c_int64, _P, C.c_int64, C.c_int, C.POINTER(C.c_double)]),
    "rbf_profile_enable": (C.c_int, [_P, C.c_int]),
    "rbf_profile_query": (C.c_int, [_P, _P, _P]),
    "rbf_reconstruct_host": (C.c_int, [_P, _P, _P, C.c_int64, C.POINTER(_Kernel), C.POINTER(_CellCfg),
                                       C.POINTER(_PrecondCfg), C.POINTER(_GmresCfg), C.POINTER(_Grid),
                                       _P, _P, C.POINTER(SolveReport)]),
}

_lib = None


def launch_count() -> int:
    """rbf_launch_count: kernels launched by librbf in this process so far."""
    return int(load_library().rbf_launch_count())


def load_library(path: str = LIB_PATH):
    """Load librbf.so; raises (never falls back) when it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"librbf.so not found at {path}: run __graft_entry__.build() "
                           "(python -m paper_1305_5179_b200.build); there is no CPU fallback")
    lib = C.CDLL(path)
    for name, (res, args) in EXPORTS.items():
        f = getattr(lib, name)
        f.restype = res
        f.argtypes = args
    _lib = lib
    return lib


def _check(status: int):
    if status != RBF_OK:
        msg = _lib.rbf_last_error()
        raise RbfError(status, msg.decode() if msg else "")


def _ptr(t: torch.Tensor | None):
    return None if t is None else C.c_void_p(t.data_ptr())


def _need(t: torch.Tensor, dtype, n: int | None = None, name: str = "tensor"):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if n is not None and t.numel() != n:
        raise ValueError(f"{name} must have {n} elements, got {t.numel()}")


class _DevArray:
    """Exposes a library-owned device pointer through __cuda_array_interface__."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2, "strides": None}


def _wrap_copy(ptr, shape, typestr, dtype, device):
    if ptr is None or int(ptr) == 0:
        return torch.empty(shape, dtype=dtype, device=device)
    return torch.as_tensor(_DevArray(ptr, shape, typestr), device=device).clone()


# -------------------------------------------------------------- public API --
@dataclass(frozen=True)
class Kernel:
    """Gaussian RBF of Eq.6: a exp(-r^2/(2 sigma^2)), 0 beyond cutoff_sigmas*sigma."""
    sigma: float
    cutoff_sigmas: float = 6.0
    amplitude: float = 0.0   # <= 0 => 1/(sqrt(2 pi) sigma)

    def _c(self):
        return _Kernel(self.sigma, self.cutoff_sigmas, self.amplitude)


def nccl_unique_id() -> bytes:
    """rbf_nccl_unique_id: 128 bytes for rank 0 to broadcast (multi-GPU contexts)."""
    buf = C.create_string_buffer(128)
    _check(load_library().rbf_nccl_unique_id(buf))
    return buf.raw


def slab_plan(plane_start, plane_weight, reach: int, world: int):
    """rbf_slab_plan (host only): the slab partition the library uses for world > 1.
    Returns dict(plane_lo, own_lo, own_hi, win_lo, win_hi) as numpy arrays."""
    import numpy as np
    ps = np.ascontiguousarray(plane_start, dtype=np.int64)
    pw = np.ascontiguousarray(plane_weight, dtype=np.float64)
    dimz = pw.size
    if ps.size != dimz + 1:
        raise ValueError("plane_start needs dimz + 1 entries")
    out = dict(plane_lo=np.zeros(world + 1, np.int32), own_lo=np.zeros(world, np.int64),
               own_hi=np.zeros(world, np.int64), win_lo=np.zeros(world, np.int64), win_hi=np.zeros(world, np.int64))
    ptr = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _check(load_library().rbf_slab_plan(ptr(ps), ptr(pw), dimz, reach, world, ptr(out["plane_lo"]),
                                        ptr(out["own_lo"]), ptr(out["own_hi"]), ptr(out["win_lo"]),
                                        ptr(out["win_hi"])))
    return out


class LoopbackGroup:
    """rbf_loopback_group_create: `world` ranks of ONE process on one device (one
    host thread per rank; Context(loopback=(group, rank)))."""

    def __init__(self, world: int):
        h = C.c_void_p()
        _check(load_library().rbf_loopback_group_create(int(world), C.byref(h)))
        self._h, self.world = h, int(world)

    def close(self):
        if getattr(self, "_h", None):
            _lib.rbf_loopback_group_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Context:
    """rbf_create on `device`, issuing work on torch's current stream of that device.

    distributed=True (and an initialised torch.distributed group with world > 1):
    one context per rank/GPU sharing an NCCL communicator; rank 0's NCCL id is
    broadcast with torch.distributed (plumbing only).  loopback=(group, rank):
    rank `rank` of an in-process LoopbackGroup (rbf_create_loopback).
    transport="ipc" with distributed=True: the CUDA-IPC peer-memory transport
    (rbf_create_ipc, one node) instead of NCCL; rank 0's 16-byte group key is
    broadcast with torch.distributed (any backend).  Calls then take and return
    replicated (full) arrays while the library shards the work."""

    def __init__(self, device: int = 0, stream: torch.cuda.Stream | None = None, distributed: bool = False,
                 loopback: tuple | None = None, transport: str = "nccl"):
        lib = load_library()
        self.device = device
        self.stream = stream if stream is not None else torch.cuda.current_stream(device)
        if loopback is not None:
            group, rank = loopback
            h = C.c_void_p()
            _check(lib.rbf_create_loopback(C.byref(h), device, C.c_void_p(self.stream.cuda_stream), group._h,
                                           int(rank)))
            self._h, self.rank, self.world, self._group = h, int(rank), group.world, group
            return
        if transport not in ("nccl", "ipc"):
            raise ValueError("transport must be 'nccl' or 'ipc'")
        rank, world, uid = 0, 1, None
        if distributed:
            import torch.distributed as dist
            if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
                rank, world = dist.get_rank(), dist.get_world_size()
                if transport == "ipc":
                    box = [os.urandom(16) if rank == 0 else None]
                    dist.broadcast_object_list(box, src=0)
                    self.rank, self.world = rank, world
                    h = C.c_void_p()
                    _check(lib.rbf_create_ipc(C.byref(h), device, C.c_void_p(self.stream.cuda_stream),
                                              C.create_string_buffer(box[0], 16), rank, world))
                    self._h = h
                    return
                box = [nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(box, src=0)
                uid = C.create_string_buffer(box[0], 128)
        self.rank, self.world = rank, world
        h = C.c_void_p()
        _check(lib.rbf_create(C.byref(h), device, C.c_void_p(self.stream.cuda_stream), uid, rank, world))
        self._h = h

    PROF_STAGES = ("cells", "matvec_f32", "matvec_f64", "grid", "precond_setup", "precond_apply")

    def peer_memory(self, on: bool = True):
        """rbf_ctx_peer_memory: the peer-memory (fused halo) form of the symmetric
        operator on transports that support it (default on)."""
        _check(_lib.rbf_ctx_peer_memory(self._h, 1 if on else 0))

    def neighbour_lists(self, on: bool = True):
        """rbf_ctx_neighbour_lists: the neighbour-list form of the symmetric fp32
        operator (tile source lists built once per cell structure; default on)."""
        _check(_lib.rbf_ctx_neighbour_lists(self._h, 1 if on else 0))

    def grid_separable(self, on: bool = True):
        """rbf_ctx_grid_separable: the separable (12 exponentials per centre and
        node block) form of the grid evaluation (default on)."""
        _check(_lib.rbf_ctx_grid_separable(self._h, 1 if on else 0))

    def pool_reserve(self, nbytes: int):
        """rbf_pool_reserve: make sure the library's device memory pool holds a
        free block of at least nbytes now."""
        _check(_lib.rbf_pool_reserve(self._h, int(nbytes)))

    def pool_stats(self):
        """rbf_pool_stats: (bytes of backing memory held, bytes handed out)."""
        out = (C.c_uint64 * 2)()
        _check(_lib.rbf_pool_stats(self._h, out))
        return int(out[0]), int(out[1])

    def profile(self, on: bool = True):
        """rbf_profile_enable: bracket the library's stage launches with CUDA events."""
        _check(_lib.rbf_profile_enable(self._h, 1 if on else 0))

    def profile_query(self) -> dict:
        """rbf_profile_query: {stage: (total ms, launches)} since the last query."""
        import numpy as np
        ms = np.zeros(len(self.PROF_STAGES), dtype=np.float64)
        ln = np.zeros(len(self.PROF_STAGES), dtype=np.int64)
        _check(_lib.rbf_profile_query(self._h, ms.ctypes.data_as(C.c_void_p), ln.ctypes.data_as(C.c_void_p)))
        return {k: (float(ms[i]), int(ln[i])) for i, k in enumerate(self.PROF_STAGES)}

    def close(self):
        if getattr(self, "_h", None):
            _lib.rbf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def extend_points(ctx: Context, x: torch.Tensor, normals: torch.Tensor, delta: float, label: float | None = None):
    """Extended set of §2.1.1 and labels of §2.1.2:
    centres [X; X + delta n; X - delta n] (fp32, 3N x 3) and b = [0; +label; -label]
    (label defaults to delta, reading R2)."""
    _need(x, torch.float64, name="x")
    _need(normals, torch.float64, x.numel(), "normals")
    N = x.shape[0]
    centres = torch.empty((3 * N, 3), dtype=torch.float32, device=x.device)
    b = torch.empty(3 * N, dtype=torch.float32, device=x.device)
    _check(_lib.rbf_extend_points(ctx._h, _ptr(x), _ptr(normals), N, float(delta),
                                  float(delta if label is None else label), _ptr(centres), _ptr(b)))
    return centres, b


class Cells:
    """rbf_build_cells: cell list + tile plan over the centres (Alg.2 'truncation area')."""

    def __init__(self, ctx: Context, xyz: torch.Tensor, kernel: Kernel, cell_edge: float = 0.0,
                 tile_cap: int = 64, tile_span: int = 2, tile_mode: int = 0, id0: int | None = None):
        """id0 given: xyz is this rank's shard, global ids [id0, id0 + len(xyz))
        (rbf_build_cells_shard); otherwise the full (replicated) centre set."""
        _need(xyz, torch.float32, name="xyz")
        if xyz.dim() != 2 or xyz.shape[1] != 3:
            raise ValueError("xyz must be (n, 3)")
        self.ctx, self.kernel = ctx, kernel
        h = C.c_void_p()
        cfg = _CellCfg(cell_edge, tile_cap, tile_span, tile_mode)
        if id0 is None:
            self.n = xyz.shape[0]
            _check(_lib.rbf_build_cells(ctx._h, _ptr(xyz), self.n, C.byref(kernel._c()), C.byref(cfg),
                                        C.byref(h)))
        else:
            _check(_lib.rbf_build_cells_shard(ctx._h, _ptr(xyz), xyz.shape[0], int(id0), C.byref(kernel._c()),
                                              C.byref(cfg), C.byref(h)))
            self._h = h
            self.n = self.info()["n"]
        self._h = h

    def info(self) -> dict:
        d = _CellsDesc()
        _check(_lib.rbf_cells_info(self._h, C.byref(d)))
        return dict(n=d.n, dim=tuple(d.dim), lo=tuple(d.lo), inv_h=d.inv_h, cell_edge=d.cell_edge,
                    reach=d.reach, ncell=d.ncell, ntiles=d.ntiles, nonempty_cells=d.nonempty_cells)

    def slab(self) -> dict:
        """rbf_cells_slab: this rank's owned / window / tile / plane ranges."""
        import numpy as np
        v = np.zeros(11, dtype=np.int64)
        _check(_lib.rbf_cells_slab(self._h, v.ctypes.data_as(C.c_void_p)))
        return dict(own=(int(v[0]), int(v[1])), window=(int(v[2]), int(v[3])), tiles=(int(v[4]), int(v[5])),
                    planes=(int(v[6]), int(v[7])), wide_tiles=(int(v[8]), int(v[9])), wide_interior=int(v[10]))

    def view(self) -> dict:
        """Copies of the library's cell arrays (perm, sorted float4, keys, cell_start)."""
        perm, srt, keys, cs = C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(_lib.rbf_cells_view(self._h, C.byref(perm), C.byref(srt), C.byref(keys), C.byref(cs)))
        info = self.info()
        dev = torch.device("cuda", self.ctx.device)
        torch.cuda.current_stream(dev).synchronize()
        n = self.n
        return dict(perm=_wrap_copy(perm.value, (n,), "<i4", torch.int32, dev),
                    sorted=_wrap_copy(srt.value, (n, 4), "<f4", torch.float32, dev),
                    keys=_wrap_copy(keys.value, (n,), "<u4", torch.int32, dev),
                    cell_start=_wrap_copy(cs.value, (info["ncell"] + 1,), "<i4", torch.int32, dev),
                    **info)

    def close(self):
        if getattr(self, "_h", None):
            _lib.rbf_cells_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def matvec(ctx: Context, cells: Cells, kernel: Kernel, w: torch.Tensor, out: torch.Tensor | None = None):
    """f = A w (Eq.4 with Eq.6 entries); fp32 tier for float32 w, fp64 tier for float64 w."""
    prec = {torch.float32: RBF_F32, torch.float64: RBF_F64}.get(w.dtype)
    if prec is None:
        raise TypeError("w must be float32 or float64")
    _need(w, w.dtype, cells.n, "w")
    f = torch.empty_like(w) if out is None else out
    _need(f, w.dtype, cells.n, "out")
    _check(_lib.rbf_matvec(ctx._h, cells._h, C.byref(kernel._c()), prec, _ptr(w), _ptr(f)))
    return f


def matvec_op(ctx: Context, cells: Cells, kernel: Kernel, w: torch.Tensor, op: int = OP_AUTO,
              out: torch.Tensor | None = None):
    """rbf_matvec_op: f = A w through the solver's operator variant `op` (OP_*)."""
    prec = {torch.float32: RBF_F32, torch.float64: RBF_F64}.get(w.dtype)
    if prec is None:
        raise TypeError("w must be float32 or float64")
    _need(w, w.dtype, cells.n, "w")
    f = torch.empty_like(w) if out is None else out
    _need(f, w.dtype, cells.n, "out")
    _check(_lib.rbf_matvec_op(ctx._h, cells._h, C.byref(kernel._c()), prec, int(op), _ptr(w), _ptr(f)))
    return f


def matvec_pairs(ctx: Context, cells: Cells, kernel: Kernel):
    """(useful, visited) pair counts of the fp32 matvec traversal."""
    u, v = C.c_int64(), C.c_int64()
    _check(_lib.rbf_matvec_pairs(ctx._h, cells._h, C.byref(kernel._c()), C.byref(u), C.byref(v)))
    return u.value, v.value


def _grid_c(lo, hi, n):
    n = (n, n, n) if isinstance(n, int) else tuple(n)
    return _Grid((C.c_double * 3)(*lo), (C.c_double * 3)(*hi), (C.c_int * 3)(*n)), n


def eval_grid(ctx: Context, cells: Cells, kernel: Kernel, w: torch.Tensor, lo, hi, n,
              out: torch.Tensor | None = None):
    """F(xi) on the inclusive grid lo..hi with n nodes per axis (Eq.5); returns (nz, ny, nx) fp32."""
    _need(w, torch.float64, cells.n, "w")
    g, n3 = _grid_c(lo, hi, n)
    field = torch.empty((n3[2], n3[1], n3[0]), dtype=torch.float32, device=w.device) if out is None else out
    _need(field, torch.float32, n3[0] * n3[1] * n3[2], "field")
    _check(_lib.rbf_eval_grid(ctx._h, cells._h, C.byref(kernel._c()), _ptr(w), C.byref(g), _ptr(field)))
    return field


def eval_grid_slab(ctx: Context, cells: Cells, kernel: Kernel, w: torch.Tensor, lo, hi, n, out: torch.Tensor):
    """rbf_eval_grid_slab: only this rank's z layers of `out` are written; returns (k0, k1)."""
    _need(w, torch.float64, cells.n, "w")
    g, n3 = _grid_c(lo, hi, n)
    _need(out, torch.float32, n3[0] * n3[1] * n3[2], "field")
    k0, k1 = C.c_int64(), C.c_int64()
    _check(_lib.rbf_eval_grid_slab(ctx._h, cells._h, C.byref(kernel._c()), _ptr(w), C.byref(g), _ptr(out),
                                   C.byref(k0), C.byref(k1)))
    return k0.value, k1.value


def eval_grid_pairs(ctx: Context, cells: Cells, kernel: Kernel, lo, hi, n, visited: bool = False):
    """Useful (node, centre) pairs of the grid evaluation (and visited if asked)."""
    g, _ = _grid_c(lo, hi, n)
    u, v = C.c_int64(), C.c_int64()
    _check(_lib.rbf_eval_grid_pairs(ctx._h, cells._h, C.byref(kernel._c()), C.byref(g), C.byref(u), C.byref(v)))
    return (u.value, v.value) if visited else u.value


def zero_set(ctx: Context, field: torch.Tensor, lo, hi, n, data: torch.Tensor, eps: float, cap: int | None = None):
    """rbf_zero_set: points (K x 3, fp64, device) of the eps-masked zero set of the
    grid field (§2.1.3); `data` = the surface points X (N x 3 fp64, device)."""
    g, n3 = _grid_c(lo, hi, n)
    _need(field, torch.float32, n3[0] * n3[1] * n3[2], "field")
    _need(data, torch.float64, data.shape[0] * 3, "data")
    cnt = C.c_int64()
    cap = cap if cap is not None else max(1024, (n3[0] * n3[1] + n3[1] * n3[2] + n3[0] * n3[2]) * 2)
    for _ in range(2):
        pts = torch.empty((max(cap, 1), 3), dtype=torch.float64, device=field.device)
        _check(_lib.rbf_zero_set(ctx._h, _ptr(field), C.byref(g), _ptr(data), data.shape[0], eps, _ptr(pts), cap,
                                 C.byref(cnt)))
        if cnt.value <= cap:
            return pts[:cnt.value]
        cap = cnt.value
    return pts[:cnt.value]


def eval_grid_masked(ctx: Context, cells: Cells, kernel: Kernel, w: torch.Tensor, lo, hi, n, data: torch.Tensor,
                     eps: float, out: torch.Tensor | None = None):
    """rbf_eval_grid_masked: P_f on the nodes within eps of the data (M_ext^eps,
    §2.1.3), NaN elsewhere; returns (nz, ny, nx) fp32."""
    _need(w, torch.float64, cells.n, "w")
    _need(data, torch.float64, data.shape[0] * 3, "data")
    g, n3 = _grid_c(lo, hi, n)
    field = torch.empty((n3[2], n3[1], n3[0]), dtype=torch.float32, device=w.device) if out is None else out
    _need(field, torch.float32, n3[0] * n3[1] * n3[2], "field")
    _check(_lib.rbf_eval_grid_masked(ctx._h, cells._h, C.byref(kernel._c()), _ptr(w), C.byref(g), _ptr(data),
                                     data.shape[0], eps, _ptr(field)))
    return field


def _take_mesh(h, device):
    """Copies a library mesh into torch tensors and frees it: (vertices (nv,3) fp64, triangles (nt,3) int32)."""
    try:
        vp, tp = C.c_void_p(), C.c_void_p()
        nv, nt = C.c_int64(), C.c_int64()
        _check(_lib.rbf_mesh_view(h, C.byref(vp), C.byref(nv), C.byref(tp), C.byref(nt)))
        V = _wrap_copy(vp.value if nv.value else None, (nv.value, 3), "<f8", torch.float64, device)
        T = _wrap_copy(tp.value if nt.value else None, (nt.value, 3), "<i4", torch.int32, device)
        return V, T
    finally:
        _lib.rbf_mesh_free(h)


def mesh_from_field(ctx: Context, field: torch.Tensor, lo, hi, n, data: torch.Tensor, eps: float):
    """rbf_mesh_from_field: triangle mesh (reading R24) of the zero iso-surface of a
    grid field on M_ext^eps; returns (vertices, triangles) on the device."""
    g, n3 = _grid_c(lo, hi, n)
    _need(field, torch.float32, n3[0] * n3[1] * n3[2], "field")
    _need(data, torch.float64, data.shape[0] * 3, "data")
    h = C.c_void_p()
    _check(_lib.rbf_mesh_from_field(ctx._h, _ptr(field), C.byref(g), _ptr(data), data.shape[0], eps, C.byref(h)))
    return _take_mesh(h, field.device)


def isosurface(ctx: Context, cells: Cells, kernel: Kernel, w: torch.Tensor, lo, hi, n, data: torch.Tensor,
               eps: float, field: torch.Tensor | None = None):
    """rbf_isosurface (Alg.1 steps 3-4 on M_ext^eps): masked grid evaluation + mesh.
    Returns (vertices, triangles); `field`, if given, receives the masked field."""
    _need(w, torch.float64, cells.n, "w")
    _need(data, torch.float64, data.shape[0] * 3, "data")
    g, n3 = _grid_c(lo, hi, n)
    if field is not None:
        _need(field, torch.float32, n3[0] * n3[1] * n3[2], "field")
    h = C.c_void_p()
    _check(_lib.rbf_isosurface(ctx._h, cells._h, C.byref(kernel._c()), _ptr(w), C.byref(g), _ptr(data),
                               data.shape[0], eps, _ptr(field), C.byref(h)))
    return _take_mesh(h, w.device)


def nn_distance(ctx: Context, x: torch.Tensor, q: torch.Tensor | None = None):
    """rbf_nn_distance: nearest-data distances of q (or of x itself, self excluded)."""
    _need(x, torch.float64, x.shape[0] * 3, "x")
    m = x.shape[0] if q is None else q.shape[0]
    if q is not None:
        _need(q, torch.float64, m * 3, "q")
    out = torch.empty(m, dtype=torch.float64, device=x.device)
    _check(_lib.rbf_nn_distance(ctx._h, _ptr(x), x.shape[0], None if q is None else _ptr(q), m, _ptr(out)))
    return out


def density(ctx: Context, x: torch.Tensor, omega: torch.Tensor | None = None) -> dict:
    """rbf_density: q_X (Eq.7), h_max, h_{X,Omega} (Eq.8) and the sigma heuristics
    of Eq.9 (sigma_q), Eq.10 (sigma_h) and Eq.10+11 (sigma_hmax), all computed
    in the library."""
    _need(x, torch.float64, x.shape[0] * 3, "x")
    if omega is not None:
        _need(omega, torch.float64, omega.shape[0] * 3, "omega")
    out = (C.c_double * 6)()
    _check(_lib.rbf_density(ctx._h, _ptr(x), x.shape[0], None if omega is None else _ptr(omega),
                            0 if omega is None else omega.shape[0], out))
    res = dict(q=out[0], h_max=out[1], sigma_q=out[3], sigma_hmax=out[5])
    if omega is not None:
        res.update(h=out[2], sigma_h=out[4])
    return res


def sigma_auto(ctx: Context, x: torch.Tensor, rule: int = 11, omega: torch.Tensor | None = None) -> float:
    """rbf_sigma_auto: sigma from the density heuristic of Eq.9, Eq.10 or Eq.11 (rule)."""
    _need(x, torch.float64, x.shape[0] * 3, "x")
    if omega is not None:
        _need(omega, torch.float64, omega.shape[0] * 3, "omega")
    sig = C.c_double()
    _check(_lib.rbf_sigma_auto(ctx._h, _ptr(x), x.shape[0], None if omega is None else _ptr(omega),
                               0 if omega is None else omega.shape[0], int(rule), C.byref(sig)))
    return sig.value


class AssembledOperator:
    """rbf_assemble: the CSR form of A (the paper's assembled GPU path, Alg.2), for
    comparison with the matrix-free summation."""

    def __init__(self, ctx: Context, cells: Cells, kernel: Kernel):
        self.ctx, self.cells = ctx, cells
        h = C.c_void_p()
        _check(_lib.rbf_assemble(ctx._h, cells._h, C.byref(kernel._c()), C.byref(h)))
        self._h = h

    def info(self) -> dict:
        nnz, nbytes, t = C.c_int64(), C.c_int64(), C.c_double()
        _check(_lib.rbf_csr_info(self._h, C.byref(nnz), C.byref(nbytes), C.byref(t)))
        return dict(nnz=nnz.value, bytes=nbytes.value, t_assemble=t.value)

    def spmv(self, w: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
        _need(w, torch.float32, self.cells.n, "w")
        f = torch.empty_like(w) if out is None else out
        _check(_lib.rbf_csr_spmv(self.ctx._h, self._h, _ptr(w), _ptr(f)))
        return f

    def close(self):
        if getattr(self, "_h", None):
            _lib.rbf_csr_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Precond:
    """rbf_precond_create: RAS (§3.1) / block-Jacobi preconditioner."""

    def __init__(self, ctx: Context, cells: Cells, kernel: Kernel, kind: int = 2, core_target: int = 512,
                 overlap_sigmas: float = 1.0, max_ext: int = 0, shift: float = 0.0, local_fp32: int = 0,
                 pivot: int = 0, w_layout: int = 0):
        self.ctx, self.cells = ctx, cells
        h = C.c_void_p()
        cfg = _PrecondCfg(kind, core_target, overlap_sigmas, max_ext, shift, local_fp32, pivot, w_layout)
        _check(_lib.rbf_precond_create(ctx._h, cells._h, C.byref(kernel._c()), C.byref(cfg), C.byref(h)))
        self._h = h

    def apply(self, r: torch.Tensor, out: torch.Tensor | None = None):
        _need(r, torch.float32, self.cells.n, "r")
        z = torch.empty_like(r) if out is None else out
        _check(_lib.rbf_precond_apply(self.ctx._h, self._h, _ptr(r), _ptr(z)))
        return z

    def blocks(self):
        """(core lists, ext lists) in SORTED positions, plus device bytes."""
        import numpy as np
        nb, nbytes = C.c_int64(), C.c_int64()
        _check(_lib.rbf_precond_blocks(self._h, C.byref(nb), C.byref(nbytes), None, None, None, None))
        cp = np.zeros(nb.value + 1, dtype=np.int64)
        ep = np.zeros(nb.value + 1, dtype=np.int64)
        _check(_lib.rbf_precond_blocks(self._h, C.byref(nb), C.byref(nbytes), cp.ctypes.data_as(C.c_void_p),
                                       ep.ctypes.data_as(C.c_void_p), None, None))
        ci = np.zeros(int(cp[-1]), dtype=np.int32)
        ei = np.zeros(int(ep[-1]), dtype=np.int32)
        _check(_lib.rbf_precond_blocks(self._h, C.byref(nb), C.byref(nbytes), cp.ctypes.data_as(C.c_void_p),
                                       ep.ctypes.data_as(C.c_void_p), ci.ctypes.data_as(C.c_void_p),
                                       ei.ctypes.data_as(C.c_void_p)))
        cores = [ci[cp[i]:cp[i + 1]] for i in range(nb.value)]
        exts = [ei[ep[i]:ep[i + 1]] for i in range(nb.value)]
        return cores, exts, nbytes.value

    def close(self):
        if getattr(self, "_h", None):
            _lib.rbf_precond_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def gmres_solve(ctx: Context, cells: Cells, kernel: Kernel, b: torch.Tensor, precond: Precond | None = None,
                kind: int = 2, core_target: int = 512, overlap_sigmas: float = 1.0, restart: int = 30,
                rtol: float = 1e-6, phase1_rtol: float = 1e-4, max_iters: int = 500, polish_fp64: int = 1,
                shift: float = 0.0, local_fp32: int = 0, cgs_passes: int = 2, out: torch.Tensor | None = None,
                op: int = OP_AUTO, basis_fp64: int = 0, pivot: int = 0, w_layout: int = 0,
                history_cap: int = 0, x0: torch.Tensor | None = None):
    """Solve A w = b (Eq.4) with RAS-preconditioned FGMRES; returns (w fp64, report dict).
    history_cap > 0 adds the residual history (report keys history / history_true);
    x0 (fp64, caller order) warm-starts the solve (resume from a checkpoint)."""
    _need(b, torch.float32, cells.n, "b")
    if x0 is not None:
        _need(x0, torch.float64, cells.n, "x0")
    w = torch.empty(cells.n, dtype=torch.float64, device=b.device) if out is None else out
    _need(w, torch.float64, cells.n, "w")
    pc = _PrecondCfg(kind, core_target, overlap_sigmas, 0, shift, local_fp32, pivot, w_layout)
    hist = (C.c_double * max(history_cap, 1))()
    hist_t = (C.c_double * max(history_cap, 1))()
    gc = _GmresCfg(restart, rtol, phase1_rtol, max_iters, polish_fp64, cgs_passes, int(op), basis_fp64,
                   hist if history_cap > 0 else None, hist_t if history_cap > 0 else None, history_cap,
                   None if x0 is None else x0.data_ptr())
    rep = SolveReport()
    _check(_lib.rbf_gmres_solve(ctx._h, cells._h, C.byref(kernel._c()), None if precond is None else precond._h,
                                C.byref(pc), C.byref(gc), _ptr(b), _ptr(w), C.byref(rep)))
    out_rep = rep.as_dict()
    if history_cap > 0:
        out_rep["history"] = list(hist[:rep.history_len])
        out_rep["history_true"] = list(hist_t[:rep.history_true_len])
    return w, out_rep


def gmres_solve_shard(ctx: Context, cells: Cells, kernel: Kernel, b_local: torch.Tensor, id0: int,
                      kind: int = 2, core_target: int = 512, overlap_sigmas: float = 1.0, restart: int = 30,
                      rtol: float = 1e-6, phase1_rtol: float = 1e-4, max_iters: int = 500, polish_fp64: int = 1,
                      shift: float = 0.0, local_fp32: int = 0, cgs_passes: int = 2, op: int = OP_AUTO):
    """rbf_gmres_solve_shard: b_local = this rank's shard [id0, id0 + len) of b;
    returns (this rank's shard of w, report dict)."""
    _need(b_local, torch.float32, name="b_local")
    w = torch.empty(b_local.shape[0], dtype=torch.float64, device=b_local.device)
    pc = _PrecondCfg(kind, core_target, overlap_sigmas, 0, shift, local_fp32, 0, 0)
    gc = _GmresCfg(restart, rtol, phase1_rtol, max_iters, polish_fp64, cgs_passes, int(op), 0, None, None, 0)
    rep = SolveReport()
    _check(_lib.rbf_gmres_solve_shard(ctx._h, cells._h, C.byref(kernel._c()), None, C.byref(pc), C.byref(gc),
                                      _ptr(b_local), b_local.shape[0], int(id0), _ptr(w), C.byref(rep)))
    return w, rep.as_dict()


def reconstruct_host(ctx: Context, xyz, b, kernel: Kernel, lo, hi, n, *, cell_edge: float = 0.0,
                     kind: int = 2, core_target: int = 512, overlap_sigmas: float = 1.0, restart: int = 30,
                     rtol: float = 1e-6, phase1_rtol: float = 1e-4, max_iters: int = 500,
                     shift: float = 0.0, local_fp32: int = 0, cgs_passes: int = 2, op: int = OP_AUTO,
                     w_out=None, field_out=None):
    """Alg.1 steps 2-3 from HOST buffers (numpy or CPU tensors; pinned is fastest)."""
    import numpy as np
    xyz = torch.as_tensor(xyz, dtype=torch.float32).contiguous()
    b = torch.as_tensor(b, dtype=torch.float32).contiguous()
    nn = xyz.shape[0]
    g, n3 = _grid_c(lo, hi, n)
    w = torch.empty(nn, dtype=torch.float64) if w_out is None else w_out
    field = torch.empty((n3[2], n3[1], n3[0]), dtype=torch.float32) if field_out is None else field_out
    rep = SolveReport()
    _check(_lib.rbf_reconstruct_host(ctx._h, _ptr(xyz), _ptr(b), nn, C.byref(kernel._c()),
                                     C.byref(_CellCfg(cell_edge, 64, 2, 0)),
                                     C.byref(_PrecondCfg(kind, core_target, overlap_sigmas, 0, shift, local_fp32,
                                                         0, 0)),
                                     C.byref(_GmresCfg(restart, rtol, phase1_rtol, max_iters, 1, cgs_passes,
                                                       int(op), 0, None, None, 0)),
                                     C.byref(g), _ptr(w), _ptr(field), C.byref(rep)))
    del np
    return w, field, rep.as_dict()

"""Thin ctypes binding of libocto_fmm.so (include/octo_fmm.h): argument
marshalling only.  Every compute step runs in the library's sm_100a kernels;
there is no CPU fallback -- a missing library raises at import/load time.

Arrays: numpy arrays are passed as host pointers (OCTO_HOST); torch CUDA
tensors as device pointers (OCTO_DEVICE).  Streams: a torch.cuda.Stream, a raw
cudaStream_t int, or None (the current torch stream when torch is available,
else the legacy default stream).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

OCTO_OK, OCTO_EINVAL, OCTO_ESTRUCT, OCTO_EMASS, OCTO_ECUDA, OCTO_ENCCL, OCTO_ENOMEM = 0, -1, -2, -3, -4, -5, -6
OCTO_HOST, OCTO_DEVICE, OCTO_HOST_ASYNC = 0, 1, 2
OCTO_AM_CORRECTION = 1
OCTO_TIMING = 2
OCTO_EXTERNAL_BOOTSTRAP = 4
OCTO_ALL_LEVELS = -1
ABI_VERSION = 1


class OctoConfig(C.Structure):
    _fields_ = [("abi_version", C.c_int32), ("n", C.c_int32), ("theta", C.c_double), ("G", C.c_double),
                ("flags", C.c_uint32), ("device", C.c_int32), ("rank", C.c_int32), ("nranks", C.c_int32),
                ("nccl_unique_id", C.c_uint8 * 128)]


class OctoError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"octo_fmm error {code}: {msg}")
        self.code = code


_lib = None

# int (*octo_allgather_fn)(void *ctx, const void *send, void *recv, int64_t bytes)
ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64)


def lib():
    """Load libocto_fmm.so (building it in-tree if the sources are newer)."""
    global _lib
    if _lib is None:
        path = os.environ.get("OCTO_LIB")   # tuning experiments only: a variant build of the same sources
        if path is None:
            path = _build.LIB
            if _build.needs_build():
                path = _build.build()
        if not os.path.exists(path):
            raise ImportError(f"libocto_fmm.so not found at {path}: run __graft_entry__.build()")
        L = C.CDLL(path)
        vp, i32, i64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.octo_fmm_create.argtypes = [C.POINTER(OctoConfig), C.POINTER(vp)]
        L.octo_fmm_destroy.argtypes = [vp]
        L.octo_fmm_load_level.argtypes = [vp, i32, dbl, vp, i64, vp, vp, vp, vp, vp, vp, vp, i32, vp]
        L.octo_fmm_compute_interactions.argtypes = [vp, i32, vp]
        L.octo_fmm_get_expansions.argtypes = [vp, i32, vp, vp, i32, vp]
        L.octo_fmm_expansions_ptr.argtypes = [vp, i32, C.POINTER(vp), C.POINTER(vp), C.POINTER(i64)]
        L.octo_fmm_sync.argtypes = [vp, vp]
        L.octo_fmm_stencil.argtypes = [vp, vp, vp, vp, i32]
        L.octo_fmm_interaction_counts.argtypes = [vp, i32, vp]
        L.octo_fmm_launch_count.argtypes = [vp]
        L.octo_fmm_launch_count.restype = i64
        L.octo_fmm_strerror.argtypes = [C.c_int]
        L.octo_fmm_strerror.restype = C.c_char_p
        L.octo_fmm_last_error.argtypes = [vp]
        L.octo_fmm_last_error.restype = C.c_char_p
        L.octo_fmm_nccl_unique_id.argtypes = [vp]
        L.octo_fmm_p2m.argtypes = [vp, i64, vp, dbl, vp, vp]
        L.octo_fmm_kernel_times.argtypes = [vp, vp, vp]
        L.octo_fmm_get_expansions_compact.argtypes = [vp, i32, vp, vp, vp, vp, i32, vp]
        L.octo_fmm_propagate.argtypes = [vp, vp]
        L.octo_fmm_get_field.argtypes = [vp, i32, vp, vp, vp]
        L.octo_fmm_m2m.argtypes = [vp, i64, vp, vp, i64, vp, vp, dbl, vp, vp, vp, vp, vp, vp, vp, vp]
        L.octo_fmm_exchange_plan.argtypes = [dbl, i32, i32, i64, vp, vp, vp, vp, vp, vp]
        L.octo_fmm_node_costs.argtypes = [dbl, i64, vp, vp, vp]
        L.octo_fmm_set_bootstrap.argtypes = [vp, ALLGATHER_FN, vp]
        _lib = L
    return _lib


def _ptr(a, numel=None, name="array"):
    """(pointer, is_device) of a numpy array or torch tensor (None -> NULL).
    The C ABI takes no lengths for its row arrays, so every array is checked
    here to be float64 (unless numel is None and it is an index array) and,
    when numel is given, to hold exactly that many elements."""
    if a is None:
        return None, None
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError(f"{name} must be C-contiguous")
        if numel is not None:
            if a.dtype != np.float64:
                raise TypeError(f"{name} must be float64, got {a.dtype}")
            if a.size != numel:
                raise ValueError(f"{name} must have {numel} elements, got {a.size}")
        return a.ctypes.data, False
    if hasattr(a, "data_ptr"):
        if not a.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if numel is not None:
            import torch
            if a.dtype != torch.float64:
                raise TypeError(f"{name} must be float64, got {a.dtype}")
            if a.numel() != numel:
                raise ValueError(f"{name} must have {numel} elements, got {a.numel()}")
        return a.data_ptr(), bool(a.is_cuda)
    raise TypeError(f"unsupported array type {type(a)}")


def _stream(s):
    if s is None:
        try:
            import torch
            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return 0
    if isinstance(s, int):
        return s
    return s.cuda_stream


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    rc = lib().octo_fmm_nccl_unique_id(C.addressof(buf))
    if rc != OCTO_OK:
        raise OctoError(rc, "ncclGetUniqueId failed")
    return bytes(buf)


def exchange_plan(theta, rank, nranks, ijk, refined, neighbors, owner):
    """Host-only ghost plan (no CUDA): {peer: (send_leaf, send_ref, recv_leaf, recv_ref)}."""
    ijk = np.ascontiguousarray(ijk, np.int32)
    refined = np.ascontiguousarray(refined, np.uint8)
    nb = np.ascontiguousarray(neighbors, np.int32)
    owner = np.ascontiguousarray(owner, np.int32)
    n = ijk.shape[0]
    counts = np.zeros(4 * nranks, np.int64)
    args = (float(theta), int(rank), int(nranks), n, ijk.ctypes.data, refined.ctypes.data, nb.ctypes.data,
            owner.ctypes.data)
    rc = lib().octo_fmm_exchange_plan(*args, counts.ctypes.data, None)
    if rc != OCTO_OK:
        raise OctoError(rc, "exchange_plan")
    bufs = [np.zeros(int(c), np.int32) for c in counts]
    arr = (C.c_void_p * (4 * nranks))(*[b.ctypes.data if b.size else None for b in bufs])
    rc = lib().octo_fmm_exchange_plan(*args, counts.ctypes.data, arr)
    if rc != OCTO_OK:
        raise OctoError(rc, "exchange_plan")
    return {p: tuple(bufs[4 * p:4 * p + 4]) for p in range(nranks) if any(b.size for b in bufs[4 * p:4 * p + 4])}


def node_costs(theta, refined, neighbors):
    """Host-only per-node interaction counts (n, 3) = {P2P, M2L, mixed} of a level."""
    refined = np.ascontiguousarray(refined, np.uint8)
    nb = np.ascontiguousarray(neighbors, np.int32)
    n = refined.shape[0]
    out = np.zeros((n, 3), np.int64)
    rc = lib().octo_fmm_node_costs(float(theta), n, refined.ctypes.data, nb.ctypes.data, out.ctypes.data)
    if rc != OCTO_OK:
        raise OctoError(rc, "node_costs")
    return out


class OctoFMM:
    """Handle of the C ABI (octo_fmm_create ... octo_fmm_destroy)."""

    def __init__(self, theta: float, G: float = 1.0, am_correction: bool = True, device: int = 0, rank: int = 0,
                 nranks: int = 1, nccl_id: bytes | None = None, timing: bool = False, allgather=None):
        """nranks > 1 bootstraps the ghost exchange either through NCCL
        (`nccl_id`, one process per GPU) or through `allgather`, a callable
        bytes -> bytes (this rank's record -> every rank's, concatenated in
        rank order), e.g. `gloo_allgather()`: no NCCL communicator is created,
        so ranks may share a GPU (OCTO_EXTERNAL_BOOTSTRAP)."""
        cfg = OctoConfig()
        cfg.abi_version = ABI_VERSION
        cfg.n = 8
        cfg.theta = float(theta)
        cfg.G = float(G)
        cfg.flags = (OCTO_AM_CORRECTION if am_correction else 0) | (OCTO_TIMING if timing else 0)
        if nranks > 1 and allgather is not None:
            cfg.flags |= OCTO_EXTERNAL_BOOTSTRAP
        cfg.device = int(device)
        cfg.rank = int(rank)
        cfg.nranks = int(nranks)
        if nccl_id is not None:
            C.memmove(cfg.nccl_unique_id, nccl_id, 128)
        h = C.c_void_p()
        self._h = None
        rc = lib().octo_fmm_create(C.byref(cfg), C.byref(h))
        if rc != OCTO_OK:
            raise OctoError(rc, lib().octo_fmm_last_error(None).decode() or lib().octo_fmm_strerror(rc).decode())
        self._h = h
        self.theta = float(theta)
        self._inputs = {}
        self._boot = None
        if nranks > 1 and allgather is not None:
            def cb(_ctx, send, recv, nbytes):
                try:
                    out = allgather(C.string_at(send, nbytes))
                    if len(out) != nbytes * nranks:
                        return -1
                    C.memmove(recv, out, len(out))
                    return 0
                except Exception as e:  # noqa: BLE001 -- no exception may cross the C ABI
                    print(f"octo_fmm bootstrap allgather failed: {e!r}", flush=True)
                    return -1
            self._boot = ALLGATHER_FN(cb)   # kept alive as long as the handle
            self._check(lib().octo_fmm_set_bootstrap(self._h, self._boot, None))

    def close(self):
        if self._h is not None:
            lib().octo_fmm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc):
        if rc != OCTO_OK:
            raise OctoError(rc, lib().octo_fmm_last_error(self._h).decode())

    def load_level(self, level, h_cell, origin, node_ijk, refined, neighbors, owner, mono, com, mom, stream=None):
        org = np.ascontiguousarray(origin, np.float64)
        ijk = np.ascontiguousarray(node_ijk, np.int32)
        ref = np.ascontiguousarray(refined, np.uint8)
        nb = np.ascontiguousarray(neighbors, np.int32)
        own = None if owner is None else np.ascontiguousarray(owner, np.int32)
        n = ijk.shape[0]
        nref = int(ref.sum())
        pm, dev = _ptr(mono, n * 512, "mono")
        pc, _ = _ptr(com, 3 * nref * 512 if com is not None else None, "com")
        pmo, _ = _ptr(mom, 20 * nref * 512 if mom is not None else None, "mom")
        mem = OCTO_DEVICE if dev else OCTO_HOST
        self._keep = (org, ijk, ref, nb, own)
        # the library reads the inputs asynchronously (header: lifetime rule):
        # hold them until this level is reloaded
        self._inputs[int(level)] = (mono, com, mom)
        self._check(lib().octo_fmm_load_level(self._h, int(level), float(h_cell), org.ctypes.data, ijk.shape[0],
                                              ijk.ctypes.data, ref.ctypes.data, nb.ctypes.data,
                                              None if own is None else own.ctypes.data, pm, pc, pmo, mem,
                                              _stream(stream)))

    def compute_interactions(self, level: int = OCTO_ALL_LEVELS, stream=None):
        self._check(lib().octo_fmm_compute_interactions(self._h, int(level), _stream(stream)))

    def get_expansions(self, level, taylor, ang_corr, stream=None, non_blocking=False):
        """Host outputs synchronise the stream unless non_blocking (page-locked
        destination, OCTO_HOST_ASYNC: valid after the caller syncs the stream)."""
        no = self.expansions_ptr(level)[2]
        pt, dev = _ptr(taylor, 20 * no * 512, "taylor")
        pa, dev2 = _ptr(ang_corr, 3 * no * 512, "ang_corr")
        d = dev if dev is not None else dev2
        mem = OCTO_DEVICE if d else (OCTO_HOST_ASYNC if non_blocking else OCTO_HOST)
        self._check(lib().octo_fmm_get_expansions(self._h, int(level), pt, pa, mem, _stream(stream)))

    def compact_sizes(self, level):
        """(n_ref, n_leaf) owned nodes of the compact result layout."""
        a, b = C.c_int64(), C.c_int64()
        self._check(lib().octo_fmm_get_expansions_compact(self._h, int(level), None, None, C.byref(a), C.byref(b),
                                                          OCTO_DEVICE, _stream(None)))
        return a.value, b.value

    def get_expansions_compact(self, level, refined_out, leaf_out, stream=None, non_blocking=False):
        """refined_out [23][n_ref][512], leaf_out [7][n_leaf][512] (numpy / CPU tensor -> host, torch CUDA ->
        device).  Host outputs synchronise the stream unless non_blocking (page-locked destination,
        OCTO_HOST_ASYNC: valid after the caller syncs the stream)."""
        nr, nl = self.compact_sizes(level)
        pr, dev = _ptr(refined_out, 23 * nr * 512, "refined_out")
        pl, dev2 = _ptr(leaf_out, 7 * nl * 512, "leaf_out")
        d = dev if dev is not None else dev2
        mem = OCTO_DEVICE if d else (OCTO_HOST_ASYNC if non_blocking else OCTO_HOST)
        a, b = C.c_int64(), C.c_int64()
        self._check(lib().octo_fmm_get_expansions_compact(self._h, int(level), pr, pl, C.byref(a), C.byref(b),
                                                          mem, _stream(stream)))

    def expansions_ptr(self, level):
        t, a, n = C.c_void_p(), C.c_void_p(), C.c_int64()
        self._check(lib().octo_fmm_expansions_ptr(self._h, int(level), C.byref(t), C.byref(a), C.byref(n)))
        return t.value, a.value, n.value

    def sync(self, stream=None):
        self._check(lib().octo_fmm_sync(self._h, _stream(stream)))

    def stencil(self):
        counts = np.zeros(8, np.int32)
        self._check(lib().octo_fmm_stencil(self._h, None, None, counts.ctypes.data, 0))
        cap = int(counts.max())
        off = np.zeros((8, cap, 3), np.int8)
        cls = np.zeros((8, cap), np.uint8)
        self._check(lib().octo_fmm_stencil(self._h, off.ctypes.data, cls.ctypes.data, counts.ctypes.data, cap))
        return [(off[c, :counts[c]].astype(np.int64), cls[c, :counts[c]].copy()) for c in range(8)]

    def interaction_counts(self, level: int = OCTO_ALL_LEVELS) -> np.ndarray:
        out = np.zeros(3, np.int64)
        self._check(lib().octo_fmm_interaction_counts(self._h, int(level), out.ctypes.data))
        return out

    def p2m(self, rho, h_cell, mono, stream=None):
        """device: mono = rho * h_cell^3 (leaf cells, FMM step 1)."""
        pr, _ = _ptr(rho)
        pm, _ = _ptr(mono)
        self._check(lib().octo_fmm_p2m(self._h, int(rho.numel()), pr, float(h_cell), pm, _stream(stream)))

    def m2m(self, parent_rows, children, child_ijk, child_refined, child_h, origin, child_mono, child_com,
            child_mom, parent_mono, parent_com, parent_mom, stream=None):
        """device M2M of a parent level's refined nodes from the child level (FMM step 1)."""
        pr = np.ascontiguousarray(parent_rows, np.int32)
        ch = np.ascontiguousarray(children, np.int32)
        cij = np.ascontiguousarray(child_ijk, np.int32)
        cref = np.ascontiguousarray(child_refined, np.uint8)
        org = np.ascontiguousarray(origin, np.float64)
        self._check(lib().octo_fmm_m2m(self._h, pr.shape[0], pr.ctypes.data, ch.ctypes.data, cij.shape[0],
                                       cij.ctypes.data, cref.ctypes.data, float(child_h), org.ctypes.data,
                                       _ptr(child_mono)[0], _ptr(child_com)[0], _ptr(child_mom)[0],
                                       _ptr(parent_mono)[0], _ptr(parent_com)[0], _ptr(parent_mom)[0],
                                       _stream(stream)))

    def propagate(self, stream=None):
        """FMM step 3 (L2L, top-down, in place on the result buffers)."""
        self._check(lib().octo_fmm_propagate(self._h, _stream(stream)))

    def get_field(self, level, phi, g, stream=None):
        """device: phi[n_owned][512] = L0, g[3][n_owned][512] = -(L1 + Lc)."""
        self._check(lib().octo_fmm_get_field(self._h, int(level), _ptr(phi)[0], _ptr(g)[0], _stream(stream)))

    def kernel_times(self):
        """(ms[4] = P2P, mixed, M2L, exchange summed since the last query, calls) -- OCTO_TIMING."""
        ms = np.zeros(4)
        calls = np.zeros(1, np.int64)
        self._check(lib().octo_fmm_kernel_times(self._h, ms.ctypes.data, calls.ctypes.data))
        return ms, int(calls[0])

    def launch_count(self) -> int:
        return int(lib().octo_fmm_launch_count(self._h))


def gloo_allgather(group=None):
    """Bootstrap allgather over torch.distributed (any backend that gathers
    CPU tensors, e.g. gloo): bytes -> every rank's bytes in rank order."""
    import torch
    import torch.distributed as dist

    def f(b: bytes) -> bytes:
        t = torch.frombuffer(bytearray(b), dtype=torch.uint8)
        out = [torch.empty_like(t) for _ in range(dist.get_world_size(group))]
        dist.all_gather(out, t, group=group)
        return b"".join(o.numpy().tobytes() for o in out)
    return f

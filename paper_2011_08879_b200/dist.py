"""Row-partitioned distributed CSR and solver over the C ABI.

The reference has no distributed matrix. This module follows
the north star: contiguous row blocks, halo exchange of ghost x entries
(NCCL send/recv over NVLink, overlapped with the interior rows), and scalar
allreduces for the solver's dot products. It keeps the reference's
operator vocabulary: ``spmv`` is ``spmv_csr`` on the rank's rows, and
``solve`` takes ``larch.SolverConfig`` and returns ``larch.SolveResult``.

Setup is host work with no device needed (``DistMap``). Each rank builds
its map from its own rows (global column ids). The ranks then swap ghost
lists: an all-to-all over the caller's bootstrap (``torch.distributed``,
gloo or nccl), or direct for in-process thread groups. The requests go
back into the map, and ``DistCsrMatrix`` uploads the interior and boundary
sub-matrices.

Communicators:
  * ``Communicator.nccl`` -- one process per GPU (torchrun); the NCCL
    unique id is broadcast by torch.distributed.
  * ``Communicator.peer`` -- one process per GPU over peer memory: every
    rank maps every peer's device window (CUDA IPC handles swapped over
    torch.distributed) and lbk's own kernels store the halo and the
    solver's scalar totals over NVLink. No NCCL on the iteration path.
  * ``Communicator.peer_group(devices)`` -- the same in one process, one
    host thread and one distinct device per rank. Several ranks on one GPU
    need one process each (a context shared by ranks could deadlock).
  * ``Communicator.threads(P)`` -- P host threads, each driving its own
    executor; P virtual ranks on one GPU, or single-process multi-GPU.
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np
import torch

from . import _lib as L
from .larch import (ConfigurationError, CudaExecutor, ShapeError, SolveResult, SolverConfig,
                    SOLVER_KINDS, _check, _ptr)


def part_range(n: int, nparts: int, rank: int) -> tuple[int, int]:
    """App. B partition: rank(r) = min(r / ceil(N/P), P-1)."""
    b, e = C.c_int32(), C.c_int32()
    _check(L.load().lbk_part_range(n, nparts, rank, C.byref(b), C.byref(e)))
    return b.value, e.value


def local_rows(row_ptr: np.ndarray, cols: np.ndarray, vals: np.ndarray, nparts: int, rank: int):
    """Slice a global host CSR to one rank's rows: (local row_ptr, global
    cols, vals)."""
    n = row_ptr.size - 1
    b, e = part_range(n, nparts, rank)
    k0, k1 = int(row_ptr[b]), int(row_ptr[e])
    return ((row_ptr[b:e + 1] - k0).astype(np.int32), np.ascontiguousarray(cols[k0:k1], np.int32),
            np.ascontiguousarray(vals[k0:k1], np.float64))


def _i32(a) -> np.ndarray:
    return np.ascontiguousarray(a, np.int32)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p) if a.size else C.c_void_p(0)


class DistMap:
    """Partition + halo maps of one rank (host only)."""

    def __init__(self, n_global: int, nparts: int, rank: int, row_ptr, cols):
        self.lib = L.load()
        self.n_global, self.nparts, self.rank = n_global, nparts, rank
        self._row_ptr = _i32(row_ptr)
        self._cols = _i32(cols)
        h = C.c_void_p()
        _check(self.lib.lbk_dist_map_create(n_global, n_global, nparts, rank,
                                            self._row_ptr.size - 1, _p(self._row_ptr),
                                            _p(self._cols), C.byref(h)))
        self.h = h
        self.info = L.lbk_dist_map_info_t()
        self.refresh()

    def refresh(self):
        _check(self.lib.lbk_dist_map_info(self.h, C.byref(self.info)))

    @property
    def n_local(self) -> int:
        return self.info.n_local

    @property
    def n_ghost(self) -> int:
        return self.info.n_ghost

    def ghosts(self) -> tuple[np.ndarray, np.ndarray]:
        g = np.empty(self.info.n_ghost, np.int32)
        off = np.empty(self.nparts + 1, np.int32)
        _check(self.lib.lbk_dist_map_ghosts(self.h, _p(g), _p(off)))
        return g, off

    def local_cols(self) -> np.ndarray:
        out = np.empty(self.info.nnz_local, np.int32)
        _check(self.lib.lbk_dist_map_local_cols(self.h, _p(out)))
        return out

    def rows(self) -> tuple[np.ndarray, np.ndarray]:
        i = np.empty(self.info.n_interior, np.int32)
        b = np.empty(self.info.n_boundary, np.int32)
        _check(self.lib.lbk_dist_map_rows(self.h, _p(i), _p(b)))
        return i, b

    def requests(self) -> list[np.ndarray]:
        """What this rank needs from each peer: its ghosts owned by q."""
        g, off = self.ghosts()
        return [g[off[q]:off[q + 1]].copy() for q in range(self.nparts)]

    def set_sends(self, incoming: Sequence[np.ndarray]) -> None:
        """incoming[q] = global ids peer q requested from this rank."""
        off = np.zeros(self.nparts + 1, np.int32)
        off[1:] = np.cumsum([len(a) for a in incoming])
        gids = _i32(np.concatenate([np.asarray(a, np.int32) for a in incoming])
                    if len(incoming) else np.zeros(0, np.int32))
        _check(self.lib.lbk_dist_map_set_sends(self.h, _p(off), _p(gids)))
        self.refresh()

    def halo_count(self) -> int:
        """Largest number of halo values this rank exchanges with one peer
        (either direction); the peer communicator's slot size is the max of
        this over all ranks."""
        _, goff = self.ghosts()
        soff, _ = self.sends()
        return int(max(np.max(np.diff(goff), initial=0), np.max(np.diff(soff), initial=0)))

    def sends(self) -> tuple[np.ndarray, np.ndarray]:
        off = np.empty(self.nparts + 1, np.int32)
        idx = np.empty(max(self.info.n_send, 0), np.int32)
        _check(self.lib.lbk_dist_map_sends(self.h, _p(off), _p(idx)))
        return off, idx

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.lbk_dist_map_destroy(self.h)
                self.h = None
        except Exception:
            pass


def exchange_requests(m: DistMap, group=None) -> None:
    """All-to-all of ghost lists over torch.distributed (gloo or nccl)."""
    import torch.distributed as dist
    mine = [r.tolist() for r in m.requests()]
    everyone: list = [None] * m.nparts
    dist.all_gather_object(everyone, mine, group=group)
    m.set_sends([np.asarray(everyone[q][m.rank], np.int32) for q in range(m.nparts)])


def peer_halo_cap(m: DistMap, group=None) -> int:
    """Max over ranks of ``m.halo_count()`` (torch.distributed all-reduce)."""
    import torch.distributed as dist
    everyone: list = [None] * m.nparts
    dist.all_gather_object(everyone, m.halo_count(), group=group)
    return int(max(everyone))


def exchange_requests_local(maps: Sequence[DistMap]) -> None:
    """The same exchange for an in-process group holding every rank's map."""
    reqs = [m.requests() for m in maps]
    for m in maps:
        m.set_sends([reqs[q][m.rank] for q in range(m.nparts)])


class Communicator:
    def __init__(self, handle, nranks: int, rank: int, kind: str):
        self.h, self.nranks, self.rank, self.kind = handle, nranks, rank, kind
        self.lib = L.load()

    @staticmethod
    def nccl(device: int, group=None) -> "Communicator":
        """One process per GPU; rank 0's NCCL unique id is broadcast over
        torch.distributed."""
        import torch.distributed as dist
        lib = L.load()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_char * 128)()
        if rank == 0:
            _check(lib.lbk_comm_nccl_unique_id(uid))
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=0, group=group)
        uid = (C.c_char * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        _check(lib.lbk_comm_init_nccl(uid, world, rank, device, C.byref(h)))
        return Communicator(h, world, rank, "nccl")

    @staticmethod
    def nccl_single(device: int) -> "Communicator":
        """A one-rank NCCL communicator (no bootstrap needed)."""
        lib = L.load()
        uid = (C.c_char * 128)()
        _check(lib.lbk_comm_nccl_unique_id(uid))
        h = C.c_void_p()
        _check(lib.lbk_comm_init_nccl(uid, 1, 0, device, C.byref(h)))
        return Communicator(h, 1, 0, "nccl")

    @staticmethod
    def peer(device: int, halo_cap: int, group=None) -> "Communicator":
        """One process per GPU on one node. ``halo_cap``: the max over ranks
        of ``DistMap.halo_count()`` (see ``peer_halo_cap``)."""
        import torch.distributed as dist
        lib = L.load()
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        h = C.c_void_p()
        _check(lib.lbk_comm_init_peer(world, rank, device, int(halo_cap), C.byref(h)))
        comm = Communicator(h, world, rank, "peer")
        if world > 1:
            mine = (C.c_char * 64)()
            _check(lib.lbk_comm_peer_handle(h, mine))
            allh: list = [None] * world
            dist.all_gather_object(allh, bytes(mine), group=group)
            buf = (C.c_char * (64 * world)).from_buffer_copy(b"".join(allh))
            _check(lib.lbk_comm_peer_open(h, buf))
            dist.barrier(group)
        return comm

    @staticmethod
    def peer_group(devices: Sequence[int], halo_cap: int) -> list["Communicator"]:
        lib = L.load()
        n = len(devices)
        dv = (C.c_int32 * n)(*devices)
        arr = (C.c_void_p * n)()
        _check(lib.lbk_comm_init_peer_group(n, dv, int(halo_cap), arr))
        return [Communicator(C.c_void_p(arr[r]), n, r, "peer") for r in range(n)]

    def close(self, group=None) -> None:
        """Collective destroy: a peer window must stay mapped until every
        rank is done with it."""
        if self.kind == "peer" and self.nranks > 1:
            import torch.distributed as dist
            dist.barrier(group)
        if getattr(self, "h", None):
            self.lib.lbk_comm_destroy(self.h)
            self.h = None

    def sync(self, exec: CudaExecutor) -> None:
        """Wait for the executor's stream; raise on a communicator failure."""
        _check(self.lib.lbk_comm_sync(exec.ctx, self.h), exec.ctx)

    @staticmethod
    def threads(nranks: int) -> list["Communicator"]:
        lib = L.load()
        arr = (C.c_void_p * nranks)()
        _check(lib.lbk_comm_init_threads(nranks, arr))
        return [Communicator(C.c_void_p(arr[r]), nranks, r, "threads") for r in range(nranks)]

    def allreduce_sum(self, exec: CudaExecutor, t: torch.Tensor) -> None:
        _check(self.lib.lbk_comm_allreduce_sum_f64(exec.ctx, self.h, _ptr(t), t.numel()), exec.ctx)

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.lbk_comm_destroy(self.h)
                self.h = None
        except Exception:
            pass


class DistCsrMatrix:
    """This rank's rows of a row-partitioned CSR matrix, on its device."""

    def __init__(self, exec: CudaExecutor, m: DistMap, row_ptr, vals, nnz_global: int):
        self.exec, self.map = exec, m
        self.lib = L.load()
        rp = _i32(row_ptr)
        va = np.ascontiguousarray(vals, np.float64)
        h = C.c_void_p()
        _check(self.lib.lbk_dist_csr_create(exec.ctx, m.h, _p(rp), _p(va), int(nnz_global),
                                            C.byref(h)), exec.ctx)
        self.h = h
        self.nparts, self.rank = m.nparts, m.rank
        self.n_local, self.n_ghost = m.n_local, m.n_ghost
        self.n_global = m.n_global

    def ext_vector(self, local: Optional[np.ndarray] = None) -> torch.Tensor:
        """A device vector with room for the halo (n_local + n_ghost)."""
        t = torch.zeros(self.n_local + self.n_ghost, dtype=torch.float64, device=self.exec.device)
        if local is not None:
            t[: self.n_local].copy_(torch.from_numpy(np.ascontiguousarray(local, np.float64)))
        return t

    def spmv(self, comm: Optional[Communicator], x_ext: torch.Tensor, y: torch.Tensor,
             sync: bool = True) -> None:
        if x_ext.numel() < self.n_local + self.n_ghost or y.numel() < self.n_local:
            raise ShapeError("dist spmv: x needs n_local + n_ghost entries, y n_local")
        _check(self.lib.lbk_dist_spmv_f64(self.exec.ctx, self.h, comm.h if comm else None,
                                          _ptr(x_ext), _ptr(y)), self.exec.ctx)
        if sync:
            if comm is not None:
                comm.sync(self.exec)
            else:
                self.exec.synchronize()

    def solve(self, comm: Optional[Communicator], b: torch.Tensor, x: torch.Tensor,
              config: SolverConfig) -> SolveResult:
        if config.kind not in SOLVER_KINDS:
            raise ConfigurationError(f"solver kind {config.kind!r} not provided by the B200 backend")
        cfg = L.lbk_solver_cfg(SOLVER_KINDS[config.kind], int(config.max_iters),
                               float(config.rel_tol), int(config.fixed_iters or 0),
                               1 if config.residual_mode == "recurrence" else 0,
                               int(config.gmres_restart))
        res = L.lbk_solve_result()
        cap = int(config.fixed_iters or config.max_iters) + 2
        hist = np.empty(cap, np.float64)
        st = self.lib.lbk_dist_solve(self.exec.ctx, self.h, comm.h if comm else None, _ptr(b),
                                     _ptr(x), C.byref(cfg), C.byref(res),
                                     hist.ctypes.data_as(C.c_void_p), cap)
        _check(st, self.exec.ctx, res.breakdown_iter)
        return SolveResult(bool(res.converged), int(res.iterations), float(res.final_rel_residual),
                           hist[: res.history_len].tolist(), float(res.elapsed),
                           int(res.flop_count))

    def __del__(self):
        try:
            if getattr(self, "h", None):
                self.lib.lbk_dist_csr_destroy(self.h)
                self.h = None
        except Exception:
            pass

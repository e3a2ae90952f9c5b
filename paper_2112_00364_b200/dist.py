"""One process per GPU (BASELINE configs[2]/[4] at 1/2/4/8 GPUs).

Creates a sharded handle on every rank of an initialised torch.distributed
process group: rank g owns global particles [g*N_g, (g+1)*N_g).  The small
per-epoch exchanges (16-byte records) go through NCCL (`comm="nccl"`; the
unique id is broadcast with torch.distributed) or through a host all-gather
callback (`comm="host"`, any backend incl. gloo; also lets several processes
share one GPU in tests).  Particle migration never goes through NCCL: each rank
exports a CUDA-IPC handle of its state/ancestor buffers, the blobs are
all-gathered once, and the gather kernel stores states straight into the
destination rank's buffers.  Marshalling only.
"""
from __future__ import annotations

import ctypes as C

import torch.distributed as dist

from . import ALLGATHER_CB, EINVAL, Model, Smc, SmcError, _check, _lib, smc_comm


def allgather_bytes(payload: bytes, group=None):
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, payload, group=group)
    return out


class HostAllgather:
    """smc_comm.allgather implemented with torch.distributed on host bytes."""

    def __init__(self, group=None):
        self.group = group
        self.cfunc = ALLGATHER_CB(self.__call__)

    def __call__(self, send, recv, nbytes, user):
        try:
            parts = allgather_bytes(C.string_at(send, nbytes), self.group)
            blob = b"".join(parts)
            C.memmove(recv, blob, len(blob))
            return 0
        except Exception:            # pragma: no cover - surfaced as SMC_ENCCL
            return 1


def nccl_unique_id(group=None) -> bytes:
    """128-byte ncclUniqueId created on rank 0 and broadcast to all ranks."""
    obj = [None]
    if dist.get_rank(group) == 0:
        buf = (C.c_char * 128)()
        _check(None, _lib.smc_get_nccl_id(buf))
        obj[0] = bytes(buf)
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class ShardedSmc(Smc):
    """Smc whose particles are sharded over the ranks of `group`.  n_per_rank
    particles per rank; results (log Z, per-rank slots) are bit-identical to
    one Smc of world * n_per_rank particles (reading R1)."""

    def __init__(self, model: Model, n_per_rank: int, seed: int = 1, comm: str = "nccl",
                 group=None, stream=None):
        self.model = model
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        self._keep = []
        if comm == "nccl":
            nid = nccl_unique_id(group)
            idbuf = C.create_string_buffer(nid, 128)
            self._keep.append(idbuf)
            c = smc_comm(C.cast(idbuf, C.c_void_p), ALLGATHER_CB(0), None)
        elif comm == "host":
            ag = HostAllgather(group)
            self._keep.append(ag)
            c = smc_comm(None, ag.cfunc, None)
        else:
            raise ValueError(comm)
        self._comm = c
        self.h = _lib.smc_create_sharded(C.byref(model.c), int(n_per_rank), int(seed), rank, world,
                                         C.byref(c))
        if not self.h:
            raise SmcError(EINVAL, _lib.smc_errmsg(None).decode())
        self.n = int(n_per_rank)
        nb = _lib.smc_ipc_blob_bytes()
        blob = (C.c_char * nb)()
        _check(self.h, _lib.smc_ipc_export(self.h, blob))
        blobs = b"".join(allgather_bytes(bytes(blob), group))
        allb = C.create_string_buffer(blobs, len(blobs))
        _check(self.h, _lib.smc_ipc_import(self.h, allb))
        dist.barrier(group)
        if stream is not None:
            self.set_stream(stream)


def sharded(model: Model, n_per_rank: int, seed: int = 1, comm: str = "nccl", stream=None):
    return ShardedSmc(model, n_per_rank, seed, comm=comm, stream=stream)

"""Process-group plumbing for row-sharded plans.

One process per GPU (torchrun).  libgbe computes; torch.distributed moves the
bytes of the only collective on the path: the all-gather of a row-sharded
UTIL message whose consumer needs it whole (and of single sharded argmin
lookups in the VALUE phase).  Two transports:
  - "nccl": all_gather_into_tensor over NVLink on the solve's stream;
  - "gloo": host-staged (device -> host -> gloo -> device), used by the CPU
    tests and to run several ranks on ONE GPU.
Both need torch views of libgbe's device buffers, so the library's
allocations are routed through the torch caching allocator (TorchMemory).
"""
from __future__ import annotations

import bisect
import os

import torch
import torch.distributed as dist

from . import gbe as _g


class TorchMemory:
    """gbe allocator hook backed by the torch caching allocator, with a
    pointer registry so collective hooks can view any library buffer."""

    def __init__(self, device):
        self.device = torch.device("cuda", device) if isinstance(device, int) else device
        self.blocks = {}
        self.keys = []

    def alloc(self, nbytes, stream):
        s = torch.cuda.ExternalStream(stream, device=self.device) if stream else torch.cuda.current_stream(self.device)
        with torch.cuda.stream(s):
            t = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
        p = t.data_ptr()
        self.blocks[p] = t
        bisect.insort(self.keys, p)
        return p

    def free(self, ptr):
        t = self.blocks.pop(ptr, None)
        if t is not None:
            i = bisect.bisect_left(self.keys, ptr)
            del self.keys[i]

    def view(self, ptr, nbytes):
        i = bisect.bisect_right(self.keys, ptr) - 1
        if i < 0:
            raise KeyError(f"pointer {ptr:#x} not allocated through TorchMemory")
        base = self.keys[i]
        t = self.blocks[base]
        off = ptr - base
        if off + nbytes > t.numel():
            raise KeyError(f"view [{ptr:#x}, +{nbytes}) outside its allocation")
        return t[off:off + nbytes]


_STATE = {}


def install(device, backend=None):
    """Route libgbe allocations through torch and install the all-gather
    hook for the current process group."""
    backend = backend or dist.get_backend()
    mem = TorchMemory(device)
    world = dist.get_world_size()

    def ag(send, recv, nbytes, stream):
        try:
            s = torch.cuda.ExternalStream(stream, device=mem.device) if stream else torch.cuda.current_stream(mem.device)
            with torch.cuda.stream(s):
                sv = mem.view(send, nbytes)
                rv = mem.view(recv, nbytes * world)
                if backend == "nccl":
                    dist.all_gather_into_tensor(rv, sv)
                else:
                    parts = [torch.empty(nbytes, dtype=torch.uint8) for _ in range(world)]
                    dist.all_gather(parts, sv.cpu())
                    rv.copy_(torch.cat(parts).to(mem.device))
            return 0
        except Exception as e:  # reported through gbe_last_error as GBE_E_COMM
            print(f"[gbe allgather] {e}", flush=True)
            return 1

    _g.set_allocator(mem.alloc, mem.free)
    _g.set_allgather(ag)
    _STATE.update(mem=mem, backend=backend)
    return mem


def uninstall():
    _g.set_allgather(None)
    _g.set_allocator(None, None)
    _STATE.clear()


def init(local_rank, backend="nccl"):
    """torchrun-style init (127.0.0.1 rendezvous from the environment).
    backend "nccl": libgbe's built-in NCCL communicator does the data-path
    all-gather on the solve stream (no Python on the data path); the torch
    process group only carries the 128-byte NCCL id, barriers and the
    max-over-ranks timing.  backend "gloo": host-staged Python hook."""
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    if not dist.is_initialized():
        dist.init_process_group(backend=backend, device_id=torch.device("cuda", local_rank)
                                if backend == "nccl" else None)
    if backend == "nccl":
        obj = [_g.comm_nccl_id() if dist.get_rank() == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        _g.comm_nccl_init(obj[0], dist.get_world_size(), dist.get_rank(), local_rank)
        _STATE.update(backend="nccl-builtin")
    else:
        install(local_rank, backend)
    return dist.group.WORLD


def barrier(pg):
    if pg is not None and dist.is_initialized():
        dist.barrier()


def max_over_ranks(x, pg):
    if pg is None or not dist.is_initialized():
        return x
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def finish(pg):
    if pg is not None and dist.is_initialized():
        if _STATE.get("backend") == "nccl-builtin":
            _g.comm_finalize()
            _STATE.clear()
        else:
            uninstall()
        dist.barrier()
        dist.destroy_process_group()

"""Multi-GPU plumbing: the row/column partition and the cabs_comm callbacks.

One process per GPU.  A is split into contiguous row blocks (P rows follow them);
the column-side embedding (Q, V) is split into contiguous column slices
(SURVEY.md §8(e)).  The library delegates its few collectives -- the pilot /
follow-up row exchange, the norm vectors, ONE fused k-means payload per Lloyd
iteration, the snap candidates and the two residual scalars -- to sum-allreduce
callbacks implemented here on torch.distributed (NCCL over NVLink on a B200 box,
gloo in the CPU tests), ordered on the library's stream.
"""
from __future__ import annotations

import ctypes
import math

import torch
import torch.distributed as dist

from .cabs import ALLREDUCE_FN, Comm, Plan


def row_partition(m: int, rank: int, nranks: int, align: int = 1):
    per = int(math.ceil(m / nranks / align)) * align
    r0 = min(m, rank * per)
    return r0, min(m, r0 + per)


def col_partition(n: int, rank: int, nranks: int):
    per = int(math.ceil(n / nranks))
    c0 = min(n, rank * per)
    return c0, min(n, c0 + per)


def make_plan(m: int, n: int, kmax: int, rank: int = 0, nranks: int = 1, align: int = 1) -> Plan:
    r0, r1 = row_partition(m, rank, nranks, align)
    c0, c1 = col_partition(n, rank, nranks)
    return Plan(m, n, r0, r1, c0, c1, kmax, rank, nranks)


class _CAI:
    """Minimal __cuda_array_interface__ (v2: no stream semantics) over a raw pointer."""

    def __init__(self, ptr, count, typestr):
        self.__cuda_array_interface__ = {"shape": (int(count),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2}


def tensor_from_ptr(ptr: int, count: int, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    """Zero-copy tensor view of `count` elements at `ptr` (device or host memory)."""
    if device.type == "cuda":
        ts = {torch.float64: "<f8", torch.float32: "<f4"}[dtype]
        return torch.as_tensor(_CAI(ptr, count, ts), device=device)
    ct = {torch.float64: ctypes.c_double, torch.float32: ctypes.c_float}[dtype]
    arr = (ct * int(count)).from_address(int(ptr))
    return torch.frombuffer(arr, dtype=dtype, count=int(count))


class TorchComm:
    """cabs_comm implemented with torch.distributed.all_reduce (SUM) on `group`."""

    def __init__(self, device: torch.device, group=None):
        self.device = torch.device(device)
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)
        self._f64 = ALLREDUCE_FN(lambda p, c, ctx, s: self._allreduce(p, c, s, torch.float64))
        self._f32 = ALLREDUCE_FN(lambda p, c, ctx, s: self._allreduce(p, c, s, torch.float32))
        self.c = Comm(self.rank, self.nranks, self._f64, self._f32, None)
        self.calls = 0
        self.bytes = 0

    def _allreduce(self, ptr, count, stream, dtype) -> int:
        try:
            t = tensor_from_ptr(ptr, count, dtype, self.device)
            if self.device.type == "cuda" and stream:
                with torch.cuda.stream(torch.cuda.ExternalStream(int(stream), device=self.device)):
                    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
            else:
                dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
            self.calls += 1
            self.bytes += t.numel() * t.element_size()
            return 0
        except Exception as e:  # never let an exception cross the C ABI
            print(f"[cabs comm rank {self.rank}] allreduce failed: {e!r}")
            return 1

    def allreduce_tensor(self, t: torch.Tensor):
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

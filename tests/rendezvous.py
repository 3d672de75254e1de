"""Test-only multi-rank comm: nranks ranks as host threads of ONE process on ONE GPU.

Each rank runs on its own stream.  An allreduce callback synchronises the caller's stream,
meets the other ranks at a host barrier and sums the buffers on the host in rank order, so the
kernels of different ranks never wait on each other on the device (one GPU cannot host ranks
whose kernels spin on one another).  The whole multi-rank host logic is exercised: partitions,
slot offsets, sentinels, the fused per-iteration payloads, the candidate exchange.  For two
ranks the host sum a + b equals NCCL's.
"""
from __future__ import annotations

import threading

import torch


class HostRendezvousComm:
    def __init__(self, nranks, device):
        from paper_1607_07395_b200.cabs import ALLREDUCE_FN, Comm
        self.nranks = nranks
        self.device = torch.device(device)
        self.bar = threading.Barrier(nranks)
        self.bufs = [None] * nranks
        self.calls = [0] * nranks
        self.comms = []
        self._fns = []
        for r in range(nranks):
            f64 = ALLREDUCE_FN(lambda ptr, cnt, ctx, st, r=r: self._cb(r, ptr, cnt, st, torch.float64))
            f32 = ALLREDUCE_FN(lambda ptr, cnt, ctx, st, r=r: self._cb(r, ptr, cnt, st, torch.float32))
            self._fns += [f64, f32]
            self.comms.append(_RankComm(self, r, Comm(r, nranks, f64, f32, None)))

    def _sum(self, r, t):
        """Host-side sum over the ranks (every rank calls this with its tensor)."""
        self.bufs[r] = t.detach().cpu()
        self.bar.wait()
        tot = self.bufs[0].clone()
        for q in range(1, self.nranks):
            tot += self.bufs[q]
        self.bar.wait()
        t.copy_(tot.to(t.device))
        self.calls[r] += 1

    def _cb(self, r, ptr, cnt, stream, dtype):
        from paper_1607_07395_b200.dist import tensor_from_ptr
        try:
            if stream:
                torch.cuda.ExternalStream(int(stream), device=self.device).synchronize()
            else:
                torch.cuda.synchronize(self.device)
            t = tensor_from_ptr(ptr, cnt, dtype, self.device)
            self._sum(r, t)
            torch.cuda.synchronize(self.device)
            return 0
        except Exception as e:  # noqa: BLE001 -- never cross the C ABI
            print("rendezvous comm failed:", repr(e))
            try:
                self.bar.abort()
            except Exception:  # noqa: BLE001
                pass
            return 1


class _RankComm:
    """What CabsPipeline / the bindings expect of a comm: .c (the cabs_comm struct), .rank,
    .nranks and allreduce_tensor."""

    def __init__(self, owner, rank, c):
        self.owner = owner
        self.rank = rank
        self.nranks = owner.nranks
        self.c = c

    def allreduce_tensor(self, t):
        torch.cuda.current_stream(t.device).synchronize()
        self.owner._sum(self.rank, t)
        torch.cuda.synchronize(t.device)


def run_ranks(nranks, fn, timeout=600):
    """fn(rank) in nranks threads; returns the per-rank results, raises the first error."""
    out, errs = [None] * nranks, []

    def main(r):
        try:
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            import traceback
            errs.append((r, traceback.format_exc()))

    th = [threading.Thread(target=main, args=(r,)) for r in range(nranks)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=timeout)
    assert not any(t.is_alive() for t in th), "rank thread hung"
    assert not errs, errs
    return out

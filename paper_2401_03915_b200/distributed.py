"""Sharding the hot path across GPUs.

Decomposition: each rank owns a contiguous slab of subdomains (balanced by the bytes of their
local operators).  Vectors, SpMV, dot products and the (replicated, small) coarse solve are
computed redundantly on every rank; every prolongation is rank-partial and completed by ONE
in-place sum all-reduce (NCCL over NVLink inside the captured solve graph).  Setup exchanges:
global max pivot (rank filter), per-subdomain coarse counts, the coarse basis blocks and the
column blocks of A0 = Z^T A Z.

Two transports with the same interface:
* ``TorchCollective`` — torch.distributed (NCCL on GPUs; gloo on CPU for the host-logic tests);
  the solve-time all-reduce is an NCCL communicator inside libtls_b200.
* ``ThreadCollective`` — R ranks inside one process (host threads) on one GPU; the library side
  uses an in-process group (tls_group).  Validates the sharded schedule end-to-end on 1 GPU.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _lib


def slab_ranges(weights, nranks):
    """Contiguous [lo, hi) ranges of subdomains, one per rank, balancing sum(weights)."""
    w = np.asarray(weights, dtype=np.float64)
    n = w.size
    if nranks < 1 or nranks > n:
        raise ValueError(f"cannot split {n} subdomains over {nranks} ranks")
    cum = np.concatenate([[0.0], np.cumsum(w)])
    cuts = [0]
    for r in range(1, nranks):
        target = cum[-1] * r / nranks
        c = int(np.searchsorted(cum, target))
        c = max(c, cuts[-1] + 1)
        c = min(c, n - (nranks - r))
        cuts.append(c)
    cuts.append(n)
    return [(cuts[r], cuts[r + 1]) for r in range(nranks)]


class TorchCollective:
    """torch.distributed collectives on tensors of the group's device."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.nranks = dist.get_world_size(group)

    def allreduce(self, t, op="sum"):
        d = self.dist
        self.dist.all_reduce(t, op=d.ReduceOp.SUM if op == "sum" else d.ReduceOp.MAX, group=self.group)
        return t

    def allgather_list(self, t):
        """Variable-length 1-D tensors -> list over ranks (same dtype/device)."""
        import torch
        n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
        sizes = [torch.zeros_like(n) for _ in range(self.nranks)]
        self.dist.all_gather(sizes, n, group=self.group)
        sizes = [int(s.item()) for s in sizes]
        m = max(sizes) if sizes else 0
        pad = torch.zeros(m, dtype=t.dtype, device=t.device)
        pad[: t.numel()] = t.reshape(-1)
        outs = [torch.empty_like(pad) for _ in range(self.nranks)]
        self.dist.all_gather(outs, pad, group=self.group)
        return [o[:s] for o, s in zip(outs, sizes)]

    def broadcast(self, t, src=0):
        self.dist.broadcast(t, src=src, group=self.group)
        return t

    def broadcast_bytes(self, b, src=0):
        obj = [b]
        self.dist.broadcast_object_list(obj, src=src, group=self.group)
        return obj[0]


class _ThreadState:
    def __init__(self, n):
        self.n = n
        self.barrier = threading.Barrier(n)
        self.slots = [None] * n


class ThreadCollective:
    """Collectives among ``n`` host threads of one process (one instance per rank)."""

    def __init__(self, state, rank):
        self.s = state
        self.rank = rank
        self.nranks = state.n

    @staticmethod
    def make(n):
        st = _ThreadState(n)
        return [ThreadCollective(st, r) for r in range(n)]

    def _exchange(self, value):
        """Deposit ``value``, return every rank's value (tensors copied on the caller's stream).

        Ranks run on different CUDA streams: the producer's stream is synchronised before the
        hand-over and the consumer copies the peers' tensors and synchronises its own stream
        before the second barrier, so no tensor is read after its owner may reuse it.
        """
        import torch
        if torch.is_tensor(value) and value.is_cuda:
            torch.cuda.current_stream(value.device).synchronize()
        self.s.slots[self.rank] = value
        self.s.barrier.wait()
        vals = [v.clone() if torch.is_tensor(v) else v for v in self.s.slots]
        if any(torch.is_tensor(v) and v.is_cuda for v in vals):
            torch.cuda.current_stream().synchronize()
        self.s.barrier.wait()
        return vals

    def allreduce(self, t, op="sum"):
        vals = self._exchange(t.clone())
        acc = vals[0].clone()
        for v in vals[1:]:
            acc = acc + v.to(acc.device) if op == "sum" else acc.maximum(v.to(acc.device))
        t.copy_(acc)
        return t

    def allgather_list(self, t):
        return [v.to(t.device) for v in self._exchange(t.reshape(-1).clone())]

    def broadcast(self, t, src=0):
        vals = self._exchange(t.clone() if self.rank == src else None)
        t.copy_(vals[src].to(t.device))
        return t

    def broadcast_bytes(self, b, src=0):
        return self._exchange(b if self.rank == src else None)[src]


class Shard:
    """What one rank needs: its collective, the solve-time transport, and its slab."""

    def __init__(self, collective, transport="nccl", group_handle=None):
        self.coll = collective
        self.rank = collective.rank
        self.nranks = collective.nranks
        self.transport = transport          # "nccl" | "group"
        self.group_handle = group_handle    # tls_group* for transport "group"
        self.lo = self.hi = None

    def attach(self, handle):
        """Create this rank's solve-time communicator inside the library handle."""
        lib = handle.lib
        if self.nranks == 1:
            return
        if self.transport == "group":
            handle.check(lib.tls_comm_init_group(handle.ctx, self.group_handle, self.rank))
            return
        uid = (C.c_char * 128)()
        if self.rank == 0:
            rc = lib.tls_nccl_unique_id(uid, 128)
            if rc != 0:
                raise RuntimeError(f"tls_nccl_unique_id failed ({rc})")
        raw = self.coll.broadcast_bytes(bytes(uid) if self.rank == 0 else None)
        uid = (C.c_char * 128).from_buffer_copy(raw)
        handle.check(lib.tls_comm_init_nccl(handle.ctx, uid, self.nranks, self.rank))


class LocalGroup:
    """An in-process group of ``n`` ranks on one GPU (library tls_group + thread collectives)."""

    def __init__(self, n):
        from .gpu_setup import warm_linalg
        warm_linalg()
        self.lib = _lib.load()
        out = C.c_void_p()
        rc = self.lib.tls_group_create(n, C.byref(out))
        if rc != 0:
            raise RuntimeError(f"tls_group_create failed ({rc})")
        self.ptr = out
        self.shards = [Shard(c, "group", out) for c in ThreadCollective.make(n)]

    def run(self, fn):
        """Run fn(shard) on one thread per rank; returns the per-rank results (re-raises)."""
        res = [None] * len(self.shards)
        err = [None] * len(self.shards)

        def body(i):
            try:
                res[i] = fn(self.shards[i])
            except BaseException as e:  # noqa: BLE001
                err[i] = e
                try:
                    self.shards[i].coll.s.barrier.abort()
                except Exception:
                    pass

        ts = [threading.Thread(target=body, args=(i,)) for i in range(len(self.shards))]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        for e in err:
            if e is not None and not isinstance(e, threading.BrokenBarrierError):
                raise e
        for e in err:
            if e is not None:
                raise e
        return res

    def __del__(self):
        if getattr(self, "ptr", None) is not None and self.ptr.value:
            self.lib.tls_group_destroy(self.ptr)
            self.ptr = None


def world_shard():
    """Shard over the default torch.distributed group (one process per GPU, NCCL)."""
    return Shard(TorchCollective(), "nccl")

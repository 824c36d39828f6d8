"""Sharding the hot path across GPUs.

Decomposition: each rank owns a contiguous slab of subdomains (balanced by the bytes of their
local operators) and the rows those subdomains own (Boolean PoU: every row has exactly one
owner subdomain).  The rows are renumbered rank by rank (``RowPartition``) so each rank's rows
form one contiguous internal range; every per-iteration kernel then runs on the owned rows only:
SpMV, the local solves of its subdomains, its rows of A0^{-1} c, the prolongation, the Krylov
vector updates.  Exchanges per operator (NCCL over NVLink, captured in the solve graphs):
* halo: the ghost rows a rank reads (columns of its SpMV rows, overlap rows of its subdomains)
  from their owners -- point-to-point, only between neighbouring slabs;
* reverse halo (ASM only): local-solve outputs on rows owned by another rank go to the owner,
  who adds them in ascending subdomain order (the np.add.at order of src/precond.py:121);
* sum all-reduces of the dot-product partials (a few KB) and of c = Z^T r (n_C doubles).
Setup exchanges: global max pivot (rank filter), per-subdomain coarse counts, the coarse basis
blocks and the column blocks of A0 = Z^T A Z; the halo plans (needed-row lists).

Two transports with the same interface:
* ``TorchCollective`` — torch.distributed (NCCL on GPUs; gloo on CPU for the host-logic tests);
  the solve-time exchanges use an NCCL communicator inside libtls_b200.
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


def row_partition(owner, n_loc, nranks):
    """Rank of every subdomain and row, and the rank-by-rank row numbering.

    Returns (slabs, new_of_old, row_starts): rank q owns subdomains slabs[q] = [lo, hi) and the
    internal rows [row_starts[q], row_starts[q+1]); new_of_old[g] is the internal row of row g
    (rows keep their relative order inside a rank)."""
    owner = np.asarray(owner, dtype=np.int64)
    slabs = slab_ranges(np.asarray(n_loc, dtype=np.float64) ** 2, nranks)
    sub_rank = np.empty(len(n_loc), dtype=np.int64)
    for q, (lo, hi) in enumerate(slabs):
        sub_rank[lo:hi] = q
    row_rank = sub_rank[owner]
    old_of_new = np.argsort(row_rank, kind="stable")
    new_of_old = np.empty_like(old_of_new)
    new_of_old[old_of_new] = np.arange(old_of_new.size)
    row_starts = np.concatenate([[0], np.cumsum(np.bincount(row_rank, minlength=nranks))])
    return slabs, new_of_old.astype(np.int64), row_starts.astype(np.int64)


def needed_rows(csr, maps, slab, new_of_old, r0, r1):
    """Sorted internal ids of the ghost rows rank reads: columns of its SpMV rows and the
    overlap rows of its subdomains that it does not own."""
    lo, hi = slab
    own_old = np.zeros(csr.shape[0], dtype=bool)
    own_old[(new_of_old >= r0) & (new_of_old < r1)] = True
    lens = np.diff(csr.indptr)
    cols = csr.indices[np.repeat(own_old, lens)]
    parts = [new_of_old[cols]] + [new_of_old[maps[s].indices] for s in range(lo, hi)]
    allr = np.unique(np.concatenate(parts))
    return allr[(allr < r0) | (allr >= r1)]


def halo_lists(needs, rank, row_starts):
    """From every rank's sorted needed rows: (peers, send_rows per peer, recv_rows per peer)."""
    r0, r1 = int(row_starts[rank]), int(row_starts[rank + 1])
    peers, send, recv = [], [], []
    for q in range(len(needs)):
        if q == rank:
            continue
        nq = needs[q]
        s_q = nq[(nq >= r0) & (nq < r1)]
        mine = needs[rank]
        rq = mine[(mine >= row_starts[q]) & (mine < row_starts[q + 1])]
        if s_q.size or rq.size:
            peers.append(q)
            send.append(s_q)
            recv.append(rq)
    return peers, send, recv


def remote_contributions(maps, slabs, rank, new_of_old, row_starts):
    """ASM overlap contributions rank receives: per peer (ascending) the (global subdomain,
    internal row) pairs of the peer's subdomains on rows this rank owns, in the peer's
    (subdomain, local index) order."""
    r0, r1 = int(row_starts[rank]), int(row_starts[rank + 1])
    peers, subs, rows = [], [], []
    for q, (lo, hi) in enumerate(slabs):
        if q == rank:
            continue
        idx = [new_of_old[maps[s].indices] for s in range(lo, hi)]
        if not idx:
            continue
        sid = np.repeat(np.arange(lo, hi), [a.size for a in idx])
        cat = np.concatenate(idx)
        keep = (cat >= r0) & (cat < r1)
        if keep.any():
            peers.append(q)
            subs.append(sid[keep])
            rows.append(cat[keep])
    return peers, subs, rows


class RowPartition:
    """One rank's share of the renumbered system and its exchange plans."""

    def __init__(self, maps, owner, shard):
        n_loc = np.array([m.n_local for m in maps], dtype=np.int64)
        self.slabs, self.new_of_old, self.row_starts = row_partition(owner, n_loc, shard.nranks)
        self.shard = shard
        self.rank = shard.rank
        self.r0 = int(self.row_starts[self.rank])
        self.r1 = int(self.row_starts[self.rank + 1])

    def set_numbering(self, handle):
        """Before the matrix upload: the library stores P A P^T in the internal numbering."""
        nofo = np.ascontiguousarray(self.new_of_old, dtype=np.int32)
        rs = np.ascontiguousarray(self.row_starts, dtype=np.int32)
        handle.check(handle.lib.tls_set_row_partition(handle.ctx, nofo.size, _lib.ptr(nofo),
                                                      self.shard.nranks, _lib.ptr(rs), self.rank))

    def install(self, handle, csr, maps, one_level):
        """Exchange the needed-row lists and hand the halo / reverse-halo plans to the library."""
        import torch
        needs_me = needed_rows(csr, maps, self.slabs[self.rank], self.new_of_old, self.r0, self.r1)
        dev = torch.device("cuda", handle.device)
        parts = self.shard.coll.allgather_list(torch.as_tensor(needs_me, dtype=torch.int64, device=dev))
        needs = [p.cpu().numpy() for p in parts]
        peers, send, recv = halo_lists(needs, self.rank, self.row_starts)
        i32 = lambda a: np.ascontiguousarray(a, dtype=np.int32)  # noqa: E731
        cat = lambda xs: i32(np.concatenate(xs) if xs else np.zeros(0))  # noqa: E731
        pe, sc, sr, rc, rr = (i32(peers), i32([x.size for x in send]), cat(send),
                              i32([x.size for x in recv]), cat(recv))
        handle.check(handle.lib.tls_set_halo(handle.ctx, pe.size, _lib.ptr(pe), _lib.ptr(sc), _lib.ptr(sr),
                                             _lib.ptr(rc), _lib.ptr(rr)))
        self.halo_rows = int(rr.size)
        if one_level == "asm":
            rp, rs, rw = remote_contributions(maps, self.slabs, self.rank, self.new_of_old, self.row_starts)
        else:
            rp, rs, rw = [], [], []
        p2, c2, s2, w2 = i32(rp), i32([x.size for x in rs]), cat(rs), cat(rw)
        handle.check(handle.lib.tls_set_remote_contrib(handle.ctx, p2.size, _lib.ptr(p2), _lib.ptr(c2),
                                                       _lib.ptr(s2), _lib.ptr(w2)))
        self.remote_rows = int(w2.size)


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

    def __init__(self, collective, transport="nccl", group_handle=None, single=False):
        self.coll = collective
        self.rank = collective.rank
        self.nranks = collective.nranks
        self.transport = transport          # "nccl" | "group"
        self.group_handle = group_handle    # tls_group* for transport "group"
        # ``single``: run the sharded schedule (row renumbering, halo plans, communicator and the
        # collectives captured in the solve graphs) on a group of ONE rank too, instead of the
        # plain single-GPU path -- the only way to execute the NCCL transport on a 1-GPU box
        self.single = bool(single)
        self.lo = self.hi = None

    @property
    def active(self):
        """Whether setup and the solves take the sharded path."""
        return self.nranks > 1 or self.single

    def attach(self, handle):
        """Create this rank's solve-time communicator inside the library handle."""
        lib = handle.lib
        if not self.active:
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


def world_shard(single=False):
    """Shard over the default torch.distributed group (one process per GPU, NCCL)."""
    return Shard(TorchCollective(), "nccl", single=single)

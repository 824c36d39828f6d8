"""Multi-rank host logic of the sharded path on CPU: world_size 2 over gloo (no GPU).

Covers the slab decomposition, the collectives used by sharded setup (max pivot, variable-length
all-gather of coarse blocks, broadcast of the NCCL id) and the sharded Galerkin assembly: the sum
over ranks of their A0 column blocks equals the single-process A0."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import golden, golden_csr
from paper_2401_03915_b200 import distributed as Dd
from paper_2401_03915_b200 import partition as Pt
from paper_2401_03915_b200.gpu_setup import assemble_a0_columns


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _problem():
    d = golden("cfg2_m16")
    a = golden_csr(d)
    g = Pt.symmetrized_graph(a)
    maps = Pt.extend_overlap(g, Pt.Partition(int(d["n_sub"]), d["owner"]), 1)
    rng = np.random.default_rng(42)
    counts = np.array([3 + (s % 3) for s in range(len(maps))], dtype=np.int64)
    z = {s: torch.as_tensor(rng.standard_normal((m.interior.size, counts[s]))) for s, m in enumerate(maps)}
    w = {s: torch.as_tensor(rng.standard_normal((m.n_local, counts[s]))) for s, m in enumerate(maps)}
    return d["owner"].astype(np.int64), maps, counts, z, w


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        coll = Dd.TorchCollective()
        owner, maps, counts, z, w = _problem()
        lo, hi = Dd.slab_ranges([m.n_local ** 2 for m in maps], world)[rank]
        # collectives used by the sharded setup
        t = torch.tensor([float(rank + 1), float(10 * rank)], dtype=torch.float64)
        coll.allreduce(t, op="max")
        got = coll.allgather_list(torch.arange(rank + 2, dtype=torch.float64))
        blob = coll.broadcast_bytes(b"nccl-id-bytes" if rank == 0 else None)
        # sharded Galerkin assembly: own column blocks, then the sum over ranks
        zs = {s: z[s] for s in range(len(maps))}
        part = assemble_a0_columns(maps, owner, zs, w, counts, range(lo, hi), torch.device("cpu"))
        coll.allreduce(part, op="sum")
        full = assemble_a0_columns(maps, owner, zs, w, counts, range(len(maps)), torch.device("cpu"))
        # row partition + halo plan through the real collective (needed-row lists all-gathered)
        a = golden_csr(golden("cfg2_m16"))
        slabs, nofo, starts = Dd.row_partition(owner, [m.n_local for m in maps], world)
        r0, r1 = int(starts[rank]), int(starts[rank + 1])
        needs_me = Dd.needed_rows(a, maps, slabs[rank], nofo, r0, r1)
        needs = [x.numpy() for x in coll.allgather_list(torch.as_tensor(needs_me))]
        peers, send, recv = Dd.halo_lists(needs, rank, starts)
        out.put((rank, t.tolist(), [g.tolist() for g in got], blob, (lo, hi),
                 float((part - full).abs().max()), float(full.abs().max()),
                 (peers, [x.tolist() for x in send], [x.tolist() for x in recv], starts.tolist())))
    finally:
        dist.destroy_process_group()


def test_sharded_host_logic_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=240) for _ in range(2)])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ranges = [r[4] for r in res]
    assert ranges[0][0] == 0 and ranges[0][1] == ranges[1][0] and ranges[1][1] == 8
    # halo plans agree pairwise: what rank 0 sends to 1 is exactly what 1 receives from 0
    (p0, s0, r0_, st0), (p1, s1, r1_, st1) = res[0][7], res[1][7]
    assert st0 == st1 and p0 == [1] and p1 == [0]
    assert s0[0] == r1_[0] and s1[0] == r0_[0] and len(s0[0]) > 0
    for rank, t, got, blob, _, err, scale, _plan in res:
        assert t == [2.0, 10.0]
        assert got == [[0.0, 1.0], [0.0, 1.0, 2.0]]
        assert blob == b"nccl-id-bytes"
        assert err <= 1e-14 * scale


def test_slab_ranges_balanced_and_contiguous():
    w = np.array([5, 1, 1, 1, 5, 1, 1, 1], dtype=float)
    r = Dd.slab_ranges(w, 2)
    assert r == [(0, 4), (4, 8)]
    r3 = Dd.slab_ranges(np.ones(10), 3)
    assert r3[0][0] == 0 and r3[-1][1] == 10
    assert all(a[1] == b[0] for a, b in zip(r3, r3[1:]))
    assert all(hi > lo for lo, hi in r3)
    with pytest.raises(ValueError):
        Dd.slab_ranges(np.ones(2), 3)


def test_thread_collective_semantics():
    import threading
    colls = Dd.ThreadCollective.make(3)
    res = [None] * 3

    def body(i):
        c = colls[i]
        t = torch.tensor([float(i), float(-i)], dtype=torch.float64)
        s = c.allreduce(t.clone(), "sum")
        m = c.allreduce(t.clone(), "max")
        g = c.allgather_list(torch.full((i + 1,), float(i)))
        b = c.broadcast(torch.tensor([float(i)]), src=2)
        res[i] = (s.tolist(), m.tolist(), [x.tolist() for x in g], b.tolist())

    ts = [threading.Thread(target=body, args=(i,)) for i in range(3)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    for r in res:
        assert r[0] == [3.0, -3.0] and r[1] == [2.0, 0.0]
        assert r[2] == [[0.0], [1.0, 1.0], [2.0, 2.0, 2.0]] and r[3] == [2.0]


def _emulate_rows(nranks, name="cfg2_m16", overlap=1):
    d = golden(name)
    a = golden_csr(d)
    owner = d["owner"].astype(np.int64)
    g = Pt.symmetrized_graph(a)
    maps = Pt.extend_overlap(g, Pt.Partition(int(d["n_sub"]), owner), overlap)
    slabs, nofo, starts = Dd.row_partition(owner, [m.n_local for m in maps], nranks)
    needs = [Dd.needed_rows(a, maps, slabs[q], nofo, int(starts[q]), int(starts[q + 1]))
             for q in range(nranks)]
    return a, owner, maps, slabs, nofo, starts, needs


@pytest.mark.parametrize("nranks", [2, 3, 4])
def test_row_partition_and_halo_cover_every_read(nranks):
    a, owner, maps, slabs, nofo, starts, needs = _emulate_rows(nranks)
    n = a.shape[0]
    assert np.array_equal(np.sort(nofo), np.arange(n))
    for q, (lo, hi) in enumerate(slabs):
        r0, r1 = starts[q], starts[q + 1]
        for s in range(lo, hi):  # interiors of a rank's subdomains are its own rows
            iv = nofo[maps[s].interior]
            assert iv.min() >= r0 and iv.max() < r1
        peers, send, recv = Dd.halo_lists(needs, q, starts)
        have = np.zeros(n, dtype=bool)
        have[r0:r1] = True
        for x in recv:
            have[x] = True
        # every SpMV column of an owned row and every overlap row of an owned subdomain is
        # owned or received
        old_rows = np.nonzero((nofo >= r0) & (nofo < r1))[0]
        cols = np.concatenate([a.indices[a.indptr[i]:a.indptr[i + 1]] for i in old_rows])
        assert have[nofo[cols]].all()
        for s in range(lo, hi):
            assert have[nofo[maps[s].indices]].all()
        for p, sx in zip(peers, send):  # pairwise agreement
            pp, _, rp = Dd.halo_lists(needs, p, starts)
            assert np.array_equal(rp[pp.index(q)], sx)


@pytest.mark.parametrize("nranks", [2, 4])
def test_reverse_halo_reproduces_add_at_order(nranks):
    """Emulate the sharded ASM prolongation on the host: each rank's owned rows add their own
    subdomains' outputs and the received contributions in ascending subdomain order; the result
    must equal np.add.at over all subdomains (src/precond.py:121) bit for bit."""
    a, owner, maps, slabs, nofo, starts, _ = _emulate_rows(nranks)
    n = a.shape[0]
    rng = np.random.default_rng(7)
    y = [rng.standard_normal(m.n_local) for m in maps]
    ref = np.zeros(n)
    for m, ys in zip(maps, y):
        np.add.at(ref, m.indices, ys)
    sub_rank = np.empty(len(maps), dtype=int)
    for q, (lo, hi) in enumerate(slabs):
        sub_rank[lo:hi] = q
    out = np.zeros(n)
    for q in range(nranks):
        r0, r1 = starts[q], starts[q + 1]
        peers, subs, rows = Dd.remote_contributions(maps, slabs, q, nofo, starts)
        # what each sender emits for q, in its (subdomain, local index) order (library side)
        for p, sp, rw in zip(peers, subs, rows):
            emit_s, emit_r, emit_v = [], [], []
            for s in range(*slabs[p]):
                iv = nofo[maps[s].indices]
                k = (iv >= r0) & (iv < r1)
                emit_s.append(np.full(k.sum(), s))
                emit_r.append(iv[k])
                emit_v.append(y[s][k])
            assert np.array_equal(np.concatenate(emit_s), sp) and np.array_equal(np.concatenate(emit_r), rw)
        ent = []
        for s in range(*slabs[q]):
            for l, g in enumerate(nofo[maps[s].indices]):
                if r0 <= g < r1:
                    ent.append((g, s, y[s][l]))
        for p, sp, rw in zip(peers, subs, rows):  # received values, in the sender's order
            for s, g in zip(sp, rw):
                li = np.nonzero(nofo[maps[s].indices] == g)[0][0]
                ent.append((g, s, y[s][li]))
        ent.sort(key=lambda e: (e[0], e[1]))  # stable: by row, then ascending subdomain
        acc = {}
        for g, s, v in ent:
            acc[g] = acc.get(g, 0.0) + v
        oldof = np.argsort(nofo)
        for g, v in acc.items():
            out[oldof[g]] = v
    assert np.array_equal(out, ref)

"""Decomposition host logic: owner partition, BFS overlap rings, Boolean PoU, colouring.

Index sets are the bit-exact parity target (BASELINE.json north star): the
local order is interior (ascending global id) then layer 1..delta (each
ascending) exactly as ``extend_overlap`` (src/partition.py:278-301); the
colouring is the greedy largest-degree-first order of ``color_subdomains``
(src/partition.py:304-334); ``partition_graph`` restates the deterministic
farthest-seed BFS grower (src/partition.py:161-258) for ``owner=None``.
The implementations are vectorised (numpy/scipy) so that configurations with
millions of rows and thousands of subdomains set up in seconds.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import scipy.sparse as sp


@dataclass(frozen=True)
class Partition:
    """Non-overlapping owner vector (src/partition.py:17-39)."""

    n_subdomains: int
    owner: np.ndarray

    def __post_init__(self):
        owner = np.asarray(self.owner, dtype=np.int64)
        object.__setattr__(self, "owner", owner)
        if owner.ndim != 1:
            raise ValueError("owner must be a flat vector")
        if self.n_subdomains < 1 or self.n_subdomains > owner.size:
            raise ValueError("subdomain count out of range")
        if owner.min() < 0 or owner.max() >= self.n_subdomains:
            raise ValueError("owner ids out of range")
        counts = np.bincount(owner, minlength=self.n_subdomains)
        if (counts == 0).any():
            raise ValueError(f"subdomain {int(np.nonzero(counts == 0)[0][0])} is empty")

    def interior(self, i):
        return np.nonzero(self.owner == i)[0]


@dataclass(frozen=True)
class SubdomainMap:
    """Interior + ordered layers; ``indices`` is the local-to-global map (src/partition.py:42-88)."""

    index: int
    n_global: int
    interior: np.ndarray
    layers: tuple
    indices: np.ndarray = field(init=False)
    pou_mask: np.ndarray = field(init=False)

    def __post_init__(self):
        interior = np.asarray(self.interior, dtype=np.int64)
        layers = tuple(np.asarray(l, dtype=np.int64) for l in self.layers)
        object.__setattr__(self, "interior", interior)
        object.__setattr__(self, "layers", layers)
        if interior.size == 0:
            raise ValueError(f"subdomain {self.index} has empty interior")
        idx = np.concatenate([interior, *layers]) if layers else interior.copy()
        mask = np.zeros(idx.size, dtype=bool)
        mask[: interior.size] = True
        object.__setattr__(self, "indices", idx)
        object.__setattr__(self, "pou_mask", mask)

    @property
    def n_local(self):
        return self.indices.size

    @property
    def n_boundary(self):
        return self.layers[-1].size if self.layers else 0

    def restrict(self, v):
        return np.asarray(v)[self.indices]

    def scatter_add(self, out, w):
        np.add.at(out, self.indices, w)
        return out


def boolean_pou(smap):
    """1 on interior positions, 0 on layers (src/partition.py:91-93)."""
    return smap.pou_mask.astype(np.float64)


class Graph:
    """CSR adjacency without self loops (src/sparsemat.py:158-177)."""

    def __init__(self, indptr, adjacency):
        self.indptr = np.asarray(indptr, dtype=np.int64)
        self.adjacency = np.asarray(adjacency, dtype=np.int64)
        self.n = self.indptr.size - 1

    def neighbors(self, i):
        return self.adjacency[self.indptr[i]:self.indptr[i + 1]]

    def degree(self, i):
        return int(self.indptr[i + 1] - self.indptr[i])

    def frontier_neighbors(self, nodes):
        """Concatenated neighbour lists of ``nodes`` (vectorised gather)."""
        nodes = np.asarray(nodes, dtype=np.int64)
        if nodes.size == 0:
            return np.empty(0, dtype=np.int64)
        starts = self.indptr[nodes]
        lens = self.indptr[nodes + 1] - starts
        total = int(lens.sum())
        if total == 0:
            return np.empty(0, dtype=np.int64)
        base = np.repeat(starts - (np.cumsum(lens) - lens), lens)
        return self.adjacency[base + np.arange(total, dtype=np.int64)]


def symmetrized_graph(csr, symmetric=False):
    """Edge {i,j}, i != j, iff |a_ij| > 0 or |a_ji| > 0 (src/sparsemat.py:180-195).

    ``symmetric``: the caller guarantees a == a^T exactly (``SparseMat`` verifies its flag), so
    the symmetrised pattern is the pattern itself: the nonzero off-diagonal entries are kept in
    place (one pass, no transpose or sparse add; same result).
    """
    a = sp.csr_matrix(csr)
    if a.shape[0] != a.shape[1]:
        raise ValueError("sparsity graph requires a square matrix")
    if symmetric:
        if not a.has_sorted_indices:
            a = a.sorted_indices()
        n = a.shape[0]
        rows = np.repeat(np.arange(n, dtype=np.int32), np.diff(a.indptr))
        keep = (a.data != 0) & (a.indices != rows)
        del rows
        ck = np.zeros(keep.size + 1, dtype=np.int64)
        np.cumsum(keep, out=ck[1:])
        indptr = ck[a.indptr]
        return Graph(indptr, a.indices[keep].astype(np.int64))
    pat = sp.csr_matrix((np.abs(a.data), a.indices.copy(), a.indptr.copy()), shape=a.shape)
    pat.eliminate_zeros()
    pat = (pat + pat.T).tocsr()
    pat.setdiag(0.0)
    pat.eliminate_zeros()
    pat.sort_indices()
    return Graph(pat.indptr.copy(), pat.indices.astype(np.int64))


def extend_overlap(graph, part, overlap):
    """``overlap`` BFS rings around every interior (src/partition.py:278-301)."""
    if overlap < 1:
        raise ValueError("overlap must be at least 1")
    owner = part.owner
    nsub = part.n_subdomains
    order = np.argsort(owner, kind="stable")          # ascending ids inside each owner
    starts = np.concatenate([[0], np.cumsum(np.bincount(owner, minlength=nsub))])
    stamp = np.full(graph.n, -1, dtype=np.int64)
    maps = []
    for s in range(nsub):
        interior = order[starts[s]:starts[s + 1]]
        stamp[interior] = s
        layers = []
        front = interior
        for _ in range(overlap):
            nb = graph.frontier_neighbors(front)
            nb = nb[stamp[nb] != s]
            ring = np.unique(nb)
            stamp[ring] = s
            layers.append(ring)
            front = ring
        maps.append(SubdomainMap(s, graph.n, interior, tuple(layers)))
    return maps


def color_subdomains(maps):
    """Greedy colouring of the subdomain intersection graph (src/partition.py:304-334)."""
    nsub = len(maps)
    if nsub == 0:
        raise ValueError("no subdomains to color")
    n = maps[0].n_global
    nodes = np.concatenate([m.indices for m in maps])
    subs = np.repeat(np.arange(nsub), [m.n_local for m in maps])
    inc = sp.csr_matrix((np.ones(nodes.size), (nodes, subs)), shape=(n, nsub))
    adj = (inc.T @ inc).tocsr()
    adj.setdiag(0.0)
    adj.eliminate_zeros()
    adj.sort_indices()
    deg = np.diff(adj.indptr)
    order = np.lexsort((np.arange(nsub), -deg))
    colors = np.full(nsub, -1, dtype=np.int64)
    for i in order:
        nb = adj.indices[adj.indptr[i]:adj.indptr[i + 1]]
        used = set(colors[nb][colors[nb] >= 0].tolist())
        c = 0
        while c in used:
            c += 1
        colors[i] = c
    return int(colors.max()) + 1, colors


# -- partition_graph (owner=None) --------------------------------------------------

def _components(graph):
    seen = np.zeros(graph.n, dtype=bool)
    comps = []
    for start in range(graph.n):
        if seen[start]:
            continue
        comp = [start]
        seen[start] = True
        front = np.array([start], dtype=np.int64)
        while front.size:
            nb = np.unique(graph.frontier_neighbors(front))
            nb = nb[~seen[nb]]
            seen[nb] = True
            comp.extend(nb.tolist())
            front = nb
        comps.append(np.sort(np.asarray(comp, dtype=np.int64)))
    return comps


def _hop_distance(graph, sources, allowed):
    dist = np.full(graph.n, -1, dtype=np.int64)
    sources = sources[allowed[sources]]
    dist[sources] = 0
    front = sources
    d = 0
    while front.size:
        d += 1
        cand = np.unique(graph.frontier_neighbors(front))
        cand = cand[(dist[cand] < 0) & allowed[cand]]
        dist[cand] = d
        front = cand
    return dist


def _grow(graph, seed, target, free):
    picked = [seed]
    free[seed] = False
    front = np.array([seed], dtype=np.int64)
    while len(picked) < target and front.size:
        ring = np.unique(graph.frontier_neighbors(front))
        ring = ring[free[ring]]
        if ring.size == 0:
            break
        room = target - len(picked)
        ring = ring[:room]
        free[ring] = False
        picked.extend(ring.tolist())
        front = ring
    return picked


def _budgets(sizes, nparts):
    total = sum(sizes)
    quota = [s * nparts / total for s in sizes]
    bud = [int(q) for q in quota]
    if len(sizes) <= nparts:
        bud = [max(1, b) for b in bud]
    while sum(bud) < nparts:
        cand = [i for i in range(len(bud)) if bud[i] < sizes[i]]
        i = max(cand, key=lambda i: (quota[i] - bud[i], sizes[i], -i))
        bud[i] += 1
    while sum(bud) > nparts:
        floor = 1 if len(sizes) <= nparts else 0
        cand = [i for i in range(len(bud)) if bud[i] > floor]
        i = min(cand, key=lambda i: (quota[i] - bud[i], sizes[i], -i))
        bud[i] -= 1
    return bud


def partition_graph(graph, n_subdomains):
    """Deterministic farthest-seed BFS partitioner (src/partition.py:161-258)."""
    n = graph.n
    if not (1 <= n_subdomains <= n):
        raise ValueError(f"subdomain count {n_subdomains} out of range for {n} nodes")
    comps = _components(graph)
    comps.sort(key=lambda c: (-c.size, int(c[0])))
    budgets = _budgets([c.size for c in comps], n_subdomains)
    owner = np.full(n, -1, dtype=np.int64)
    next_id = 0
    leftover_comps = []
    for comp, nparts in zip(comps, budgets):
        if nparts == 0:
            leftover_comps.append(comp)
            continue
        inside = np.zeros(n, dtype=bool)
        inside[comp] = True
        free = inside.copy()
        target = -(-comp.size // nparts)
        assigned = []
        for s in range(nparts):
            if s == 0:
                seed = int(comp[0])
            else:
                dist = _hop_distance(graph, np.asarray(assigned, dtype=np.int64), inside)
                cand = comp[free[comp]]
                seed = int(cand[np.argmax(dist[cand])])
            goal = min(target, int(free[comp].sum()) - (nparts - 1 - s))
            picked = _grow(graph, seed, goal, free)
            owner[picked] = next_id + s
            assigned.extend(picked)
        while free[comp].any():
            progressed = False
            for u in comp[free[comp]]:
                nbo = owner[graph.neighbors(u)]
                nbo = np.unique(nbo[nbo >= 0])
                if nbo.size == 0:
                    continue
                counts = np.bincount(owner[owner >= 0], minlength=int(owner.max()) + 2)
                owner[u] = int(nbo[np.argmin(counts[nbo])])
                free[u] = False
                progressed = True
            if not progressed:
                raise RuntimeError("leftover nodes not adjacent to any subdomain")
        next_id += nparts
    for comp in leftover_comps:
        counts = np.bincount(owner[owner >= 0], minlength=n_subdomains)
        owner[comp] = int(np.argmin(counts))
    return Partition(n_subdomains, owner)

"""Device handle: one ``tls_ctx`` of libtls_b200.so per operator, plus tensor plumbing.

PyTorch is used for device memory and the current CUDA stream only.  There is
no CPU path: without a CUDA device or without the built library every call
raises (BASELINE.json: "no CPU fallback").
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .errors import SubdomainSetupError


def _torch():
    import torch  # imported lazily so host-only tools work without paying the import
    return torch


def require_cuda(device=None):
    torch = _torch()
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2401_03915_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    if device is None:
        return torch.cuda.current_device()
    return torch.device(device).index if not isinstance(device, int) else device


def stream_ptr():
    torch = _torch()
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


class Handle:
    """Owns one tls_ctx (device-resident CSR, maps, tiles, workspaces)."""

    def __init__(self, device=None):
        self.device = require_cuda(device)
        self.lib = _lib.load()
        out = C.c_void_p()
        rc = self.lib.tls_ctx_create(self.device, C.byref(out))
        if rc != 0:
            raise RuntimeError(f"tls_ctx_create failed with code {rc}")
        self.ctx = out
        self.n = 0

    def error(self):
        msg = self.lib.tls_ctx_last_error(self.ctx)
        return msg.decode() if msg else ""

    def check(self, rc, subdomain=None):
        if rc == _lib.TLS_OK:
            return
        msg = self.error()
        if rc in (_lib.TLS_ERR_DIM, _lib.TLS_ERR_CAP, _lib.TLS_ERR_ARG):
            raise ValueError(msg)
        if rc == _lib.TLS_ERR_SUBDOMAIN:
            raise SubdomainSetupError(subdomain if subdomain is not None else -1, msg)
        if rc == _lib.TLS_ERR_OOM:
            raise MemoryError(msg)
        raise RuntimeError(f"libtls_b200 error {rc}: {msg}")

    def upload_matrix(self, csr, symmetric):
        indptr = np.ascontiguousarray(csr.indptr, dtype=np.int64)
        indices = np.ascontiguousarray(csr.indices, dtype=np.int32)
        data = np.ascontiguousarray(csr.data, dtype=np.float64)
        self.n = csr.shape[0]
        self.check(self.lib.tls_matrix_upload(self.ctx, csr.shape[0], data.size, _lib.ptr(indptr),
                                              _lib.ptr(indices), _lib.ptr(data), int(bool(symmetric))))

    def device_bytes(self):
        return int(self.lib.tls_ctx_device_bytes(self.ctx))

    def __del__(self):
        ctx = getattr(self, "ctx", None)
        if ctx is not None and ctx.value:
            try:
                self.lib.tls_ctx_destroy(ctx)
            except Exception:
                pass
            self.ctx = None


def device_graph(handle):
    """Symmetrised sparsity graph of the handle's matrix, built on the device (tls_graph_build;
    src/sparsemat.py:180-195) and returned as a host ``Graph`` (int64 row pointers, int32 columns)."""
    from .partition import Graph
    m = C.c_int64()
    handle.check(handle.lib.tls_graph_build(handle.ctx, C.byref(m)))
    gptr = np.empty(handle.n + 1, dtype=np.int64)
    gadj = np.empty(max(1, m.value), dtype=np.int32)
    handle.check(handle.lib.tls_graph_fetch(handle.ctx, _lib.ptr(gptr), _lib.ptr(gadj)))
    return Graph(gptr, gadj[: m.value])


def device_overlap(handle, part, overlap):
    """Overlap rings + colouring of every subdomain on the device (tls_overlap_build; bit-exact
    with src/partition.py:278-334) from the graph of the last ``device_graph`` call.
    Returns (maps, k_c, colors); frees the device graph."""
    from .partition import SubdomainMap
    if overlap < 1:
        raise ValueError("overlap must be at least 1")
    nsub = part.n_subdomains
    owner = np.ascontiguousarray(part.owner, dtype=np.int64)
    tot, kc = C.c_int64(), C.c_int32()
    try:
        handle.check(handle.lib.tls_overlap_build(handle.ctx, nsub, _lib.ptr(owner), int(overlap), C.byref(tot),
                                                  C.byref(kc)))
        off = np.empty(nsub + 1, dtype=np.int64)
        ls = np.empty(nsub * overlap, dtype=np.int64)
        idx = np.empty(max(1, tot.value), dtype=np.int64)
        colors = np.empty(nsub, dtype=np.int64)
        handle.check(handle.lib.tls_overlap_fetch(handle.ctx, _lib.ptr(off), _lib.ptr(ls), _lib.ptr(idx),
                                                  _lib.ptr(colors)))
    finally:
        handle.lib.tls_graph_release(handle.ctx)
    ls = ls.reshape(nsub, overlap)
    maps = []
    n = part.owner.size
    for s in range(nsub):
        seg = idx[off[s]:off[s + 1]]
        cut = np.cumsum(ls[s])
        ni = seg.size - int(cut[-1])
        layers = tuple(seg[ni + (cut[k] - ls[s, k]):ni + cut[k]] for k in range(overlap))
        maps.append(SubdomainMap(s, n, seg[:ni], layers))
    return maps, int(kc.value), colors


def to_device(v, n, device):
    """(device fp64 tensor, converter back to the caller's type)."""
    torch = _torch()
    if isinstance(v, torch.Tensor):
        if v.shape != (n,):
            raise ValueError(f"dimension mismatch: operator has {n} rows, vector has shape {tuple(v.shape)}")
        t = v.to(device=torch.device("cuda", device), dtype=torch.float64).contiguous()
        return t, (lambda out: out)
    a = np.asarray(v, dtype=np.float64)
    if a.shape != (n,):
        raise ValueError(f"dimension mismatch: operator has {n} rows, vector has shape {a.shape}")
    t = torch.from_numpy(np.ascontiguousarray(a)).to(torch.device("cuda", device))
    return t, (lambda out: out.cpu().numpy())


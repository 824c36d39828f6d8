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


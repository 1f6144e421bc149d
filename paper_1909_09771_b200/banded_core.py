"""7-band structured-grid operator and the dense vector kernels, on the GPU.

Drop-in for the reference ``ntdprecon.banded_core``
(/root/reference/pkg/src/ntdprecon/banded_core.py).  Same names, arguments
and errors; arithmetic runs in libntdgpu.so (``ntd_spmv``, ``ntd_dot``),
bitwise equal to the reference for ``spmv``.  Host (numpy) inputs are copied
to the device and results copied back; CUDA tensors stay on the device.
``workers`` is accepted for compatibility and ignored (results never depend
on it, as in the reference).
"""

import numpy as np
import torch

from . import _lib

N_BANDS = 7
MAX_WORKERS = 4


class FactorizationError(RuntimeError):
    """Raised when a factorization hits a zero or non-finite pivot
    (banded_core.py:14-15)."""


def clamp_workers(workers):
    """banded_core.py:18-22.  The GPU path has no thread team; the clamp is
    kept for API compatibility."""
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return max(1, min(workers, MAX_WORKERS))


def _device():
    return torch.device("cuda", torch.cuda.current_device())


def as_device(x, dtype=torch.float64):
    """numpy / list / torch -> contiguous fp64 CUDA tensor (no copy if already one)."""
    _lib.load()
    if isinstance(x, torch.Tensor):
        if x.device.type == "cuda" and x.dtype == dtype and x.is_contiguous():
            return x
        return x.to(device=_device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to(_device())


def like_input(t, ref):
    """Return device tensor t in the flavour of the caller's input ref."""
    if isinstance(ref, torch.Tensor):
        return t
    return t.cpu().numpy()


def shape_of(x):
    if isinstance(x, torch.Tensor):
        return tuple(x.shape)
    return tuple(np.shape(x))


_shape = shape_of


class BandedMatrix:
    """Matrix on an nx*ny*nz grid stored as seven length-N diagonals
    (banded_core.py:36-92).  Row order of ``data``: -nx*ny, -nx, -1, 0, +1,
    +nx, +nx*ny.  ``data`` may be a numpy array (host) or a CUDA tensor; the
    GPU kernels read a device copy (``device_data()``).

    Host-backed matrices keep that device copy cached, so repeated spmv / pcg
    calls upload A once.  The cache is dropped whenever ``data`` is assigned
    or read through the ``data`` attribute or ``band()`` (the ways the
    reference's users modify A in place), and by ``invalidate()``; a caller
    that writes through an array reference it kept from before must call
    ``invalidate()`` itself."""

    def __init__(self, nx, ny, nz, data=None):
        if nx < 1 or ny < 1 or nz < 1:
            raise ValueError("grid dimensions must be positive")
        self.nx = int(nx)
        self.ny = int(ny)
        self.nz = int(nz)
        n = self.nx * self.ny * self.nz
        if data is None:
            data = np.zeros((N_BANDS, n))
        elif isinstance(data, torch.Tensor):
            if tuple(data.shape) != (N_BANDS, n):
                raise ValueError(f"band data must have shape ({N_BANDS}, {n}), got {tuple(data.shape)}")
            data = data.to(torch.float64).contiguous()
        else:
            data = np.ascontiguousarray(data, dtype=np.float64)
            if data.shape != (N_BANDS, n):
                raise ValueError(f"band data must have shape ({N_BANDS}, {n}), got {data.shape}")
        self._data = data
        self._dev = None

    @property
    def data(self):
        # the caller may write through the returned array: drop the device copy
        self._dev = None
        return self._data

    @data.setter
    def data(self, value):
        self._data = value
        self._dev = None

    def invalidate(self):
        """Drop the cached device copy (after writing to host band data
        through a reference taken earlier)."""
        self._dev = None

    @property
    def n_rows(self):
        return self.nx * self.ny * self.nz

    @property
    def offsets(self):
        nxy = self.nx * self.ny
        return (-nxy, -self.nx, -1, 0, 1, self.nx, nxy)

    def band(self, offset):
        try:
            idx = self.offsets.index(offset)
        except ValueError:
            raise ValueError(f"no band at offset {offset}") from None
        return self.data[idx]

    def copy(self):
        d = self._data.clone() if isinstance(self._data, torch.Tensor) else self._data.copy()
        return BandedMatrix(self.nx, self.ny, self.nz, d)

    def cuda(self):
        """A BandedMatrix whose data lives on the GPU (zero-copy for kernels)."""
        return BandedMatrix(self.nx, self.ny, self.nz, as_device(self._data).clone())

    def device_data(self):
        """(7, N) fp64 CUDA tensor of the bands: the data itself when it is a
        CUDA tensor, else the cached upload of the host bands."""
        d = self._data
        if isinstance(d, torch.Tensor) and d.is_cuda:
            return as_device(d)
        if self._dev is None:
            self._dev = as_device(d)
        return self._dev

    def host_data(self):
        d = self._data
        return d.cpu().numpy() if isinstance(d, torch.Tensor) else d

    def to_dense(self):
        n = self.n_rows
        a = np.zeros((n, n))
        d = self.host_data()
        for idx, off in enumerate(self.offsets):
            for r in range(max(0, -off), min(n, n - off)):
                a[r, r + off] += d[idx, r]
        return a


def spmv_device(a_dev, x_dev, nx, ny, nz, batch=1, out=None, active=None):
    """y = A x on device tensors; a_dev (B,7,N) / (7,N), x_dev (B,N) / (N,)."""
    if out is None:
        out = torch.empty_like(x_dev)
    _lib.call("ntd_spmv", _lib.ptr(a_dev), _lib.ptr(x_dev), _lib.ptr(out), nx, ny, nz, batch,
              _lib.ptr(active), _lib.stream())
    return out


def spmv(a, x, workers=1):
    """y = A x (banded_core.py:121-130), bitwise equal to the reference."""
    if _shape(x) != (a.n_rows,):
        raise ValueError(f"operand length {_shape(x)} does not match {a.n_rows} rows")
    xd = as_device(x)
    y = spmv_device(a.device_data(), xd, a.nx, a.ny, a.nz)
    return like_input(y, x)


def dot_device(x, y, batch=1, sqrt=False, out=None, active=None):
    n = x.numel() // batch
    if out is None:
        out = torch.empty(batch, dtype=torch.float64, device=x.device)
    work = torch.empty(_lib.load().ntd_dot_work_doubles(batch), dtype=torch.float64, device=x.device)
    _lib.call("ntd_dot", _lib.ptr(x), _lib.ptr(y), _lib.ptr(out), 1 if sqrt else 0, n, batch,
              _lib.ptr(work), _lib.ptr(active), _lib.stream())
    return out


def dot(x, y):
    """banded_core.py:133-136 (deterministic tree reduction on the GPU)."""
    if _shape(x) != _shape(y):
        raise ValueError("dot operands must have equal length")
    xd, yd = as_device(x).reshape(-1), as_device(y).reshape(-1)
    if xd.numel() == 0:
        return 0.0
    return float(dot_device(xd, yd)[0].item())


def axpy(alpha, x, y):
    """alpha*x + y as a new vector (banded_core.py:139-143): one kernel
    (ntd_axpy), the product rounded and then the sum, bitwise numpy's."""
    if _shape(x) != _shape(y):
        raise ValueError("axpy operands must have equal length")
    xd, yd = as_device(x).reshape(-1), as_device(y).reshape(-1)
    out = torch.empty_like(xd)
    if xd.numel():
        _lib.call("ntd_axpy", float(alpha), _lib.ptr(xd), _lib.ptr(yd), _lib.ptr(out), xd.numel(), _lib.stream())
    return like_input(out.reshape(_shape(x)), x if isinstance(x, torch.Tensor) else y)


def norm2(x):
    """banded_core.py:146-147"""
    xd = as_device(x).reshape(-1)
    if xd.numel() == 0:
        return 0.0
    return float(dot_device(xd, xd, sqrt=True)[0].item())


def to_matrix_market(a, path):
    """banded_core.py:150-166 (debug export; host side)."""
    n = a.n_rows
    d = a.host_data()
    rows = []
    for idx, off in enumerate(a.offsets):
        band = d[idx]
        for r in range(max(0, -off), min(n, n - off)):
            v = band[r]
            if v != 0.0:
                rows.append((r + 1, r + off + 1, v))
    rows.sort()
    with open(path, "w") as fh:
        fh.write("%%MatrixMarket matrix coordinate real general\n")
        fh.write(f"{n} {n} {len(rows)}\n")
        for i, j, v in rows:
            fh.write(f"{i} {j} {v:.17g}\n")

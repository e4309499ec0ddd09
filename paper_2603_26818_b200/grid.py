"""Grids, balanced slab partitions, wavenumbers and Fourier multipliers.

Public surface mirrors the reference module grid.py
(/root/reference/pkg/src/pfcspectral/grid.py:14-208).  The B200 build never
materialises the multiplier arrays on the hot path: kernels rebuild every
multiplier from the three 1D wavenumber vectors (the arithmetic order of
grid.py:181-191 is replicated in-kernel, see csrc/pfcs_z.cu).  The full
arrays of `SymbolTable` are still available as lazily built numpy arrays for
API compatibility and tests.
"""

from __future__ import annotations

import math
import threading
from dataclasses import dataclass

import numpy as np

__all__ = [
    "GridSpec",
    "SlabLayout",
    "SymbolTable",
    "wavenumbers",
    "slab_layout",
    "make_symbols",
]


@dataclass(frozen=True)
class GridSpec:
    """Periodic box: points per axis ``n`` and lengths ``length``.

    ``n[2] == 1`` selects a 2D problem (``length[2]`` ignored), as in the
    reference (grid.py:23-64).
    """

    n: tuple[int, int, int]
    length: tuple[float, float, float]

    def __post_init__(self):
        if len(self.n) != 3 or len(self.length) != 3:
            raise ValueError("GridSpec needs exactly three axes")
        for m in self.n:
            if int(m) != m or m < 1:
                raise ValueError(f"grid sizes must be positive integers, got {self.n}")
        for L in self.length:
            if not math.isfinite(L) or L <= 0:
                raise ValueError(f"domain lengths must be positive, got {self.length}")
        object.__setattr__(self, "n", tuple(int(m) for m in self.n))
        object.__setattr__(self, "length", tuple(float(L) for L in self.length))

    @property
    def shape(self) -> tuple[int, int, int]:
        return self.n

    @property
    def num_points(self) -> int:
        return self.n[0] * self.n[1] * self.n[2]

    @property
    def is_2d(self) -> bool:
        return self.n[2] == 1

    @property
    def volume(self) -> float:
        lx, ly, lz = self.length
        return lx * ly if self.is_2d else lx * ly * lz

    @property
    def cell_volume(self) -> float:
        return self.volume / self.num_points


def wavenumbers(grid: GridSpec, axis: int) -> np.ndarray:
    """Angular wavenumbers in FFT order, 2*pi*fftfreq(N, d=L/N) — the exact
    expression of grid.py:78, so the values are bit-identical."""
    if axis not in (0, 1, 2):
        raise ValueError(f"axis must be 0, 1 or 2, got {axis}")
    n = grid.n[axis]
    return 2.0 * np.pi * np.fft.fftfreq(n, d=grid.length[axis] / n)


@dataclass(frozen=True)
class SlabLayout:
    """Balanced partition of ``n_axis`` planes over ranks (grid.py:81-100)."""

    axis: int
    counts: tuple[int, ...]
    offsets: tuple[int, ...]

    @property
    def workers(self) -> int:
        return len(self.counts)

    def start(self, rank: int) -> int:
        return self.offsets[rank]

    def stop(self, rank: int) -> int:
        return self.offsets[rank] + self.counts[rank]

    def local_slice(self, rank: int) -> slice:
        return slice(self.start(rank), self.stop(rank))


def slab_layout(n_axis: int, workers: int, axis: int = 2) -> SlabLayout:
    """First ``n_axis % workers`` ranks get one extra plane; empty slabs are
    legal (grid.py:103-111).  The device kernels use the same rule
    (csrc/pfcs_fft.cuh SlabSplit)."""
    if workers < 1:
        raise ValueError(f"worker count must be >= 1, got {workers}")
    q, r = divmod(int(n_axis), int(workers))
    counts = tuple(q + 1 if g < r else q for g in range(workers))
    offsets = []
    acc = 0
    for c in counts:
        offsets.append(acc)
        acc += c
    return SlabLayout(axis=axis, counts=counts, offsets=tuple(offsets))


def _nyquist_zeroed(k: np.ndarray) -> np.ndarray:
    """Odd-derivative wavenumbers: the unpaired Nyquist mode of an even axis
    is dropped so derivatives of real fields stay real (grid.py:167-176)."""
    kd = np.array(k, copy=True)
    n = kd.shape[0]
    if n > 1 and n % 2 == 0:
        kd[n // 2] = 0.0
    return kd


class SymbolTable:
    """Fourier multipliers on (a slab of) the spectral grid.

    Holds the 1D wavenumber vectors of the slab (``kvec``) and the
    Nyquist-zeroed derivative vectors (``dvec``); the 3D arrays the reference
    stores eagerly (grid.py:114-152) — ``lap, two_ring, op, linear, cg,
    d1, d2, d3`` — are built on first access with the reference's exact
    numpy expressions, so they are bit-identical to the reference's.
    """

    _FIELDS = ("lap", "two_ring", "op", "linear", "cg", "d1", "d2", "d3")

    def __init__(self, kvec, dvec, eps: float, a0: float, mask=None):
        self.kvec = tuple(np.asarray(k, dtype=np.float64) for k in kvec)
        self.dvec = tuple(np.asarray(k, dtype=np.float64) for k in dvec)
        self.eps = float(eps)
        self.a0 = float(a0)
        self.mask = mask
        self._cache: dict = {}
        self._dev: dict = {}
        self._lock = threading.Lock()

    @property
    def shape(self) -> tuple[int, int, int]:
        return tuple(k.shape[0] for k in self.kvec)  # type: ignore[return-value]

    def _k2(self) -> np.ndarray:
        kx = self.kvec[0][:, None, None]
        ky = self.kvec[1][None, :, None]
        kz = self.kvec[2][None, None, :]
        return kx**2 + ky**2 + kz**2

    def _build(self, name: str) -> np.ndarray:
        if name in ("lap", "two_ring", "op", "linear", "cg"):
            k2 = self._cache.get("_k2")
            if k2 is None:
                k2 = self._cache["_k2"] = self._k2()
            if name == "lap":
                return -k2
            if name == "two_ring":
                return (1.0 - k2) ** 2 * (4.0 / 3.0 - k2) ** 2
            if name == "op":
                return self.eps + self.two_ring
            if name == "linear":
                return self.lap * self.op
            return np.exp(-0.5 * self.a0**2 * k2)
        axis = int(name[1]) - 1
        shape = self.shape
        idx = [None, None, None]
        idx[axis] = slice(None)
        return 1j * np.broadcast_to(self.dvec[axis][tuple(idx)], shape).copy()

    def __getattr__(self, name: str):
        if name in SymbolTable._FIELDS:
            cache = self.__dict__["_cache"]
            if name not in cache:
                cache[name] = self._build(name)
            return cache[name]
        raise AttributeError(name)

    def slab(self, layout: SlabLayout, rank: int) -> "SymbolTable":
        """Restrict to one rank's slab (grid.py:137-152)."""
        kv = list(self.kvec)
        dv = list(self.dvec)
        sl = layout.local_slice(rank)
        kv[layout.axis] = kv[layout.axis][sl]
        dv[layout.axis] = dv[layout.axis][sl]
        return SymbolTable(kv, dv, self.eps, self.a0, self.mask)

    def restrict_axis(self, axis: int, sl: slice) -> "SymbolTable":
        kv = list(self.kvec)
        dv = list(self.dvec)
        kv[axis] = kv[axis][sl]
        dv[axis] = dv[axis][sl]
        return SymbolTable(kv, dv, self.eps, self.a0, self.mask)

    def device_vectors(self, device) -> tuple:
        """(kx, ky, kz, dx, dy, dz) as float64 CUDA tensors (cached)."""
        import torch

        key = str(device)
        with self._lock:
            if key not in self._dev:
                self._dev[key] = tuple(
                    torch.as_tensor(np.ascontiguousarray(v), dtype=torch.float64, device=device)
                    for v in (*self.kvec, *self.dvec))
            return self._dev[key]


def make_symbols(grid: GridSpec, eps: float, a0: float = 1.0,
                 layout: SlabLayout | None = None, rank: int = 0) -> SymbolTable:
    """Multiplier table for the PFC/hydro operators (grid.py:155-208)."""
    if not math.isfinite(eps):
        raise ValueError(f"eps must be finite, got {eps}")
    if not math.isfinite(a0) or a0 <= 0:
        raise ValueError(f"a0 must be positive and finite, got {a0}")
    kvec = [wavenumbers(grid, axis) for axis in range(3)]
    dvec = [_nyquist_zeroed(k) for k in kvec]
    if layout is not None:
        sl = layout.local_slice(rank)
        kvec[layout.axis] = kvec[layout.axis][sl]
        dvec[layout.axis] = dvec[layout.axis][sl]
    return SymbolTable(kvec, dvec, eps, a0)

"""PFCSNAP1 snapshot files.

File format of the reference (/root/reference/pkg/src/pfcspectral/snapshot.py:1-12),
little-endian: magic ``PFCSNAP1``; u64 nx, ny, nz; u64 step; f64 sim_time;
then nx*ny*nz f64 samples with x fastest; plus a text sidecar
``<name>.meta.txt`` with the header fields and caller metadata.

``write_snapshot`` / ``read_snapshot`` keep the reference's host-array API.
``write_snapshot_slabs`` is the scale path: with x fastest, a slab of the
physical field (z slabs in 3D, y slabs in 2D) is one contiguous byte range
of the file, so every rank writes its own slab straight from device memory
at its offset (one device transpose to x-fastest order per chunk of planes,
pinned staging, positional writes) — no gather of the full field, which at
2048^3 would be 64 GiB per rank.
"""

from __future__ import annotations

import os
import struct
from dataclasses import dataclass
from pathlib import Path

import numpy as np

__all__ = ["MAGIC", "HEADER_BYTES", "SnapshotHeader", "write_snapshot", "read_snapshot",
           "write_snapshot_slabs"]

MAGIC = b"PFCSNAP1"
_HEAD = struct.Struct("<8s3QQd")  # magic, nx, ny, nz, step, sim_time
HEADER_BYTES = _HEAD.size  # 48


@dataclass(frozen=True)
class SnapshotHeader:
    nx: int
    ny: int
    nz: int
    step: int
    sim_time: float

    @property
    def shape(self) -> tuple[int, int, int]:
        return (self.nx, self.ny, self.nz)


def _header(shape, step: int, sim_time: float) -> bytes:
    return _HEAD.pack(MAGIC, int(shape[0]), int(shape[1]), int(shape[2]), int(step), float(sim_time))


def _sidecar(path: Path, shape, step: int, sim_time: float, meta: dict | None) -> None:
    lines = [f"file: {path.name}", f"dims: {shape[0]} {shape[1]} {shape[2]}", f"step: {step}",
             f"sim_time: {sim_time!r}"]
    lines += [f"{k}: {v}" for k, v in (meta or {}).items()]
    path.with_name(path.name + ".meta.txt").write_text("\n".join(lines) + "\n")


def write_snapshot(path, data, step: int, sim_time: float, meta: dict | None = None,
                   expected_shape: tuple[int, int, int] | None = None) -> Path:
    """One real 3D host field (snapshot.py:42-76): refuses non-3D data and
    shape mismatches against ``expected_shape``; writes the real part."""
    path = Path(path)
    data = np.asarray(data)
    if data.ndim != 3:
        raise ValueError(f"snapshot data must be 3D, got shape {data.shape}")
    if expected_shape is not None and tuple(data.shape) != tuple(expected_shape):
        raise ValueError(f"snapshot shape {data.shape} does not match expected {tuple(expected_shape)}; "
                         f"refusing to write {path}")
    body = np.asarray(data.real, dtype="<f8").ravel(order="F")  # x fastest
    try:
        with open(path, "wb") as fh:
            fh.write(_header(data.shape, step, sim_time))
            fh.write(body.tobytes())
    except OSError as exc:
        raise OSError(f"failed to write snapshot {path}: {exc}") from exc
    _sidecar(path, data.shape, step, sim_time, meta)
    return path


def read_snapshot(path) -> tuple[SnapshotHeader, np.ndarray]:
    """Header and (nx, ny, nz) float64 array; bit-exact round trip
    (snapshot.py:79-96).  Raises ValueError on a bad magic or a truncated
    file."""
    path = Path(path)
    raw = path.read_bytes()
    if raw[:8] != MAGIC:
        raise ValueError(f"{path}: not a snapshot file (bad magic {raw[:8]!r})")
    if len(raw) < HEADER_BYTES:
        raise ValueError(f"{path}: truncated snapshot header")
    _, nx, ny, nz, step, t = _HEAD.unpack_from(raw, 0)
    hdr = SnapshotHeader(nx=nx, ny=ny, nz=nz, step=step, sim_time=t)
    count = nx * ny * nz
    if len(raw) != HEADER_BYTES + 8 * count:
        raise ValueError(f"{path}: truncated snapshot ({len(raw)} bytes, expected {HEADER_BYTES + 8 * count})")
    data = np.frombuffer(raw, dtype="<f8", count=count, offset=HEADER_BYTES)
    return hdr, data.reshape(hdr.shape, order="F").copy()


def _pwrite_all(fd: int, data: memoryview, offset: int) -> None:
    """os.pwrite until every byte is written (short writes happen on network
    and parallel filesystems); a zero-byte write raises."""
    done = 0
    while done < len(data):
        n = os.pwrite(fd, data[done:], offset + done)
        if n <= 0:
            raise OSError(f"short snapshot write at offset {offset + done}")
        done += n


def write_snapshot_slabs(path, field, worker, step: int, sim_time: float, meta: dict | None = None,
                         chunk_planes: int | None = None) -> Path:
    """Collective snapshot of a physical field (3D Z_SLAB or 2D Y_SLAB)
    straight from the ranks' device slabs, no gather.  With x fastest in the
    file, rank r's slab (planes [p0, p0+c) of the split axis) is the byte
    range 48 + 8*plane*[p0, p0+c) with plane = nx*ny (z split) or nx (y
    split, nz = 1).  Rank 0 writes the header and the sidecar and sizes the
    file; after a barrier each rank writes its slab ``chunk_planes`` planes
    at a time (device transpose to x-fastest order, pinned staging,
    positional write).  Bytes identical to
    ``write_snapshot(path, gather(field).real, ...)``."""
    import torch

    from .distfft import Space, layout_for, physical_layout

    path = Path(path)
    grid = field.grid
    if field.space != Space.PHYSICAL or field.layout != physical_layout(grid):
        raise ValueError("write_snapshot_slabs needs a field in the physical slab layout")
    nx, ny, nz = grid.shape
    lay = layout_for(grid, field.layout, worker.size)
    axis = lay.axis  # 2 (z slabs) or 1 (y slabs, nz == 1)
    p0, cnt = lay.offsets[worker.rank], lay.counts[worker.rank]
    plane = nx * ny if axis == 2 else nx
    if worker.rank == 0:
        with open(path, "wb") as fh:
            fh.write(_header(grid.shape, step, sim_time))
            fh.truncate(HEADER_BYTES + 8 * nx * ny * nz)
        _sidecar(path, grid.shape, step, sim_time, meta)
    worker.barrier()
    local = field.dev
    if local.is_complex():
        local = local.real
    if chunk_planes is None:
        chunk_planes = max(1, min(max(cnt, 1), (256 << 20) // max(1, 8 * plane)))  # ~256 MiB staging
    fd = os.open(path, os.O_WRONLY)
    try:
        stage = None
        for c0 in range(0, cnt, chunk_planes):
            c1 = min(cnt, c0 + chunk_planes)
            # C-order (x, y, z) chunk of the split axis -> reversed axes = x fastest
            blk = (local[:, :, c0:c1] if axis == 2 else local[:, c0:c1, :]).permute(2, 1, 0).contiguous()
            if blk.is_cuda:
                if stage is None or stage.numel() < blk.numel():
                    stage = torch.empty(blk.numel(), dtype=torch.float64, pin_memory=True)
                host = stage[:blk.numel()]
                host.copy_(blk.reshape(-1))
                buf = host.numpy()
            else:
                buf = np.ascontiguousarray(blk.reshape(-1).numpy())
            _pwrite_all(fd, memoryview(buf).cast("B"), HEADER_BYTES + 8 * plane * (p0 + c0))
    finally:
        os.close(fd)
    worker.barrier()
    return path

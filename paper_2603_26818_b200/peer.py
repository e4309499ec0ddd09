"""Peer-mapped receive buffers for the fused exchanges.

The slab/pencil transposes can be fused into the FFT kernels: the last pass
before an exchange stores every element directly into the receive buffer of
the rank that owns it (csrc: PeerTable, pfcs_*_to / pfcs_fft_lines_scatter),
over NVLink, so there is no send buffer, no pack and no separate
all-to-all — the transfer overlaps the butterflies tile by tile and the
data crosses the link exactly once.  This module provides the buffers and
their mapping:

* `DeviceBuffer` — a raw cudaMalloc allocation (IPC-shareable, unlike a
  slice of torch's caching allocator) exposed as a torch tensor;
* `map_peers(worker, buf)` — collective: the device address of every rank's
  corresponding buffer.  Thread groups share the address space (peer access
  is enabled between distinct devices); process groups exchange CUDA IPC
  handles over torch.distributed and open them (lazy peer enable);
* `fence(worker)` — the ordering point of a fused exchange (writers done
  before readers read, readers done before the next writes): device-side
  event waits between thread ranks, drain + barrier between processes.
"""

from __future__ import annotations

import ctypes

import torch

from . import _native as nat


class _CAI:
    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


class DeviceBuffer:
    """cudaMalloc'd buffer (freed with the object) viewed as a 1-D tensor."""

    def __init__(self, numel: int, dtype=torch.complex128, device=None):
        lib = nat.load()
        item = torch.empty((), dtype=dtype).element_size()
        p = ctypes.c_void_p()
        nat.check(lib.pfcs_malloc(max(1, numel) * item, ctypes.byref(p)), "pfcs_malloc")
        self.ptr = p.value
        self.numel = numel
        typestr = {torch.complex128: "<c16", torch.float64: "<f8"}[dtype]
        self.tensor = torch.as_tensor(_CAI(self.ptr, (max(1, numel),), typestr),
                                      device=device or torch.device("cuda", torch.cuda.current_device()))
        self._lib = lib

    def __del__(self):
        try:
            if self.ptr:
                self._lib.pfcs_free(ctypes.c_void_p(self.ptr))
        except Exception:  # interpreter shutdown
            pass


class PeerMap:
    """Addresses of the same buffer on every rank (index = rank)."""

    def __init__(self, addrs, opened):
        self.addrs = list(addrs)
        self._opened = opened  # IPC mappings to close

    def __del__(self):
        try:
            lib = nat.load(require_cuda=False)
            for p in self._opened:
                lib.pfcs_ipc_close(ctypes.c_void_p(p))
        except Exception:
            pass


def map_peers(worker, buf: DeviceBuffer) -> PeerMap:
    """Collective: device addresses of `buf` on all ranks of `worker`."""
    lib = nat.load()
    dev = torch.cuda.current_device()
    if hasattr(worker, "_dist"):  # ProcessWorker: CUDA IPC handles
        h = ctypes.create_string_buffer(64)
        nat.check(lib.pfcs_ipc_get_handle(ctypes.c_void_p(buf.ptr), ctypes.addressof(h)), "pfcs_ipc_get_handle")
        handles = worker.all_to_all([bytes(h.raw)] * worker.size)
        addrs, opened = [], []
        for r, raw in enumerate(handles):
            if r == worker.rank:
                addrs.append(buf.ptr)
                continue
            p = ctypes.c_void_p()
            hb = ctypes.create_string_buffer(raw, 64)
            nat.check(lib.pfcs_ipc_open_handle(ctypes.addressof(hb), ctypes.byref(p)), "pfcs_ipc_open_handle")
            addrs.append(p.value)
            opened.append(p.value)
        return PeerMap(addrs, opened)
    infos = worker.all_to_all([(buf.ptr, dev)] * worker.size)
    for _, d in infos:
        if d != dev:
            nat.check(lib.pfcs_enable_peer_access(int(d)), "pfcs_enable_peer_access")
    return PeerMap([p for p, _ in infos], [])


def fence(worker) -> None:
    """Order a fused exchange: every rank's work issued so far (its stores
    into the peers' receive buffers, its reads of its own) completes before
    any rank's subsequent work does.

    Thread groups (one process, a GPU per thread: spawn_group) order it on
    the devices: each rank records an event on its stream, the ranks meet on
    the host — without draining anything — and every stream waits for its
    peers' events, so the GPUs never idle at a transpose and the host runs
    ahead.  Two events per rank, alternating: a rank cannot re-record an
    event before every peer has issued its wait on it (that needs the next
    fence's meeting).  Process groups drain the local stream and meet
    (dist.barrier), as CUDA IPC events would need a host barrier that does
    not synchronise the device."""
    if hasattr(worker, "_dist"):
        nat.check(nat.load().pfcs_stream_sync(ctypes.c_void_p(nat.stream_ptr())), "pfcs_stream_sync")
        worker.barrier()
        return
    st = worker.__dict__.get("_pfcs_fence")
    if st is None:
        st = worker.__dict__.setdefault("_pfcs_fence", {"k": 0, "ev": (torch.cuda.Event(), torch.cuda.Event())})
    ev = st["ev"][st["k"] & 1]
    st["k"] += 1
    stream = torch.cuda.current_stream()
    ev.record(stream)
    events = worker.all_to_all([ev] * worker.size)
    for h, e in enumerate(events):
        if h != worker.rank:
            stream.wait_event(e)


class Table:
    """Host uint64 array of destination addresses for the C ABI's `dst`
    argument (`.ptr` is passed; the object keeps the array alive)."""

    def __init__(self, addrs):
        self.arr = (ctypes.c_uint64 * len(addrs))(*[int(a) for a in addrs])
        self.ptr = ctypes.addressof(self.arr)

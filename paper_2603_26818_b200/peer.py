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
  event waits between thread ranks and between processes (interprocess
  events + a gloo host barrier).
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


class PeerUnavailable(RuntimeError):
    """Raised on EVERY rank of a group when any rank could not map a peer's
    buffer (no P2P between the devices, no CUDA IPC in this container): the
    callers fall back to the collective exchange, all ranks together."""


def _map_rank(worker, buf: DeviceBuffer, lib, dev: int) -> PeerMap:
    """This rank's side of map_peers (collective exchange of the handles or
    addresses, then the local mapping); raises if the mapping fails."""
    if hasattr(worker, "_dist"):  # ProcessWorker: CUDA IPC handles
        h = ctypes.create_string_buffer(64)
        got = lib.pfcs_ipc_get_handle(ctypes.c_void_p(buf.ptr), ctypes.addressof(h))
        # every rank takes part in the exchange, with None if it has no handle
        handles = worker.all_to_all([bytes(h.raw) if got == 0 else None] * worker.size)
        nat.check(got, "pfcs_ipc_get_handle")
        pm = PeerMap([], [])
        for r, raw in enumerate(handles):
            if r == worker.rank:
                pm.addrs.append(buf.ptr)
                continue
            if raw is None:
                raise RuntimeError(f"rank {r} has no IPC handle")
            p = ctypes.c_void_p()
            hb = ctypes.create_string_buffer(raw, 64)
            nat.check(lib.pfcs_ipc_open_handle(ctypes.addressof(hb), ctypes.byref(p)), "pfcs_ipc_open_handle")
            pm.addrs.append(p.value)
            pm._opened.append(p.value)
        return pm
    infos = worker.all_to_all([(buf.ptr, dev)] * worker.size)
    for _, d in infos:
        if d != dev:
            nat.check(lib.pfcs_enable_peer_access(int(d)), "pfcs_enable_peer_access")
    return PeerMap([p for p, _ in infos], [])


def map_peers(worker, buf: DeviceBuffer) -> PeerMap:
    """Collective: device addresses of `buf` on all ranks of `worker`.
    Raises PeerUnavailable on all ranks if any rank fails to map (the ranks
    agree through one more all-to-all, so none is left waiting in a fused
    exchange the others abandoned)."""
    lib = nat.load()
    err, pm = "", None
    try:
        pm = _map_rank(worker, buf, lib, torch.cuda.current_device())
    except Exception as exc:
        err = f"rank {worker.rank}: {exc}"
    errs = [e for e in worker.all_to_all([err] * worker.size) if e]
    if errs:
        del pm  # closes any IPC mappings this rank opened
        raise PeerUnavailable("; ".join(errs))
    return pm


class _IpcFence:
    """Per-process state of the device-ordered fence between processes: two
    interprocess events of this rank (alternating) and every peer's two,
    opened from their IPC handles, plus a host barrier that does not touch
    the device (gloo: the default group if it is gloo, else a gloo group
    over the same ranks, created collectively at the first fence)."""

    def __init__(self, worker):
        import torch.distributed as dist

        lib = nat.load()
        self.lib = lib
        self.own, handles = [], []
        for _ in range(2):
            ev = ctypes.c_void_p()
            h = ctypes.create_string_buffer(64)
            nat.check(lib.pfcs_ipc_event_create(ctypes.byref(ev), ctypes.addressof(h)), "pfcs_ipc_event_create")
            self.own.append(ev.value)
            handles.append(bytes(h.raw))
        all_h = worker.all_to_all([handles] * worker.size)
        self.peers = []
        for r, hs in enumerate(all_h):
            if r == worker.rank:
                continue
            evs = []
            for raw in hs:
                ev = ctypes.c_void_p()
                hb = ctypes.create_string_buffer(raw, 64)
                nat.check(lib.pfcs_ipc_event_open(ctypes.addressof(hb), ctypes.byref(ev)), "pfcs_ipc_event_open")
                evs.append(ev.value)
            self.peers.append(evs)
        if worker.backend == "gloo":
            self.barrier = worker.barrier
        else:
            hg = dist.new_group(worker._global, backend="gloo")
            self.barrier = lambda: dist.barrier(group=hg)
        self.k = 0

    def __del__(self):
        try:
            for ev in self.own + [e for evs in self.peers for e in evs]:
                self.lib.pfcs_event_destroy(ctypes.c_void_p(ev))
        except Exception:  # interpreter shutdown
            pass

    def __call__(self) -> None:
        st = ctypes.c_void_p(nat.stream_ptr())
        i = self.k & 1
        self.k += 1
        nat.check(self.lib.pfcs_event_record(ctypes.c_void_p(self.own[i]), st), "pfcs_event_record")
        self.barrier()
        for evs in self.peers:
            nat.check(self.lib.pfcs_stream_wait_event(st, ctypes.c_void_p(evs[i])), "pfcs_stream_wait_event")


def fence(worker) -> None:
    """Order a fused exchange: every rank's work issued so far (its stores
    into the peers' receive buffers, its reads of its own) completes before
    any rank's subsequent work does — on the devices, without draining:
    each rank records an event on its stream, the ranks meet on the host, and
    every stream waits for its peers' events, so the GPUs never idle at a
    transpose and the host runs ahead.  Two events per rank, alternating: a
    rank cannot re-record an event before every peer has issued its wait on
    it (that needs the next fence's meeting).

    Thread groups (one process, a GPU per thread: spawn_group) use ordinary
    CUDA events; process groups over the whole world use interprocess events
    (CUDA IPC handles) and a gloo host barrier; process sub-groups drain the
    local stream and meet (dist.barrier)."""
    if hasattr(worker, "_dist"):
        if worker.pg is not None:
            nat.check(nat.load().pfcs_stream_sync(ctypes.c_void_p(nat.stream_ptr())), "pfcs_stream_sync")
            worker.barrier()
            return
        f = worker.__dict__.get("_pfcs_ipc_fence")
        if f is None:
            f = worker.__dict__.setdefault("_pfcs_ipc_fence", _IpcFence(worker))
        f()
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

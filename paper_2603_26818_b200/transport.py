"""Worker groups: in-process threads (reference model) and one process per GPU.

The reference (transport.py:1-200) emulates the devices of a multi-GPU box
with G threads that exchange Python objects by reference.  This module keeps
that API — ``spawn_group(size, body, timeout)``, ``Worker.{rank, size,
send, receive, all_to_all, barrier, meter}``, the error types and their
messages — and adds the device data path the slab pipeline needs:

* ``Worker.exchange(send, send_counts, recv, recv_counts)`` — an
  all-to-all(v) of flat CUDA buffers.  In a thread group it is a set of
  device-to-device copies issued by the receiving rank after an event
  handshake (P2P over NVLink when the ranks sit on different GPUs).
* ``ProcessWorker`` — the same interface over ``torch.distributed``: one
  process per GPU, ``all_to_all_single`` on NCCL for the device exchange
  (NVLink/NVSwitch), object collectives for host payloads.  With the gloo
  backend the device exchange is staged through host memory (CPU tests and
  single-GPU multi-process tests).

Threads are bound to devices round-robin (thread r -> cuda:r % ndev), the
reference's one-thread-per-worker model (transport.py:191-197).
"""

from __future__ import annotations

import threading
from collections import deque
from typing import Any, Callable, Sequence

__all__ = [
    "TransportError",
    "DeadlockError",
    "WorkerFailure",
    "Worker",
    "WorkerGroup",
    "ProcessWorker",
    "spawn_group",
    "DEFAULT_TIMEOUT",
]

DEFAULT_TIMEOUT = 30.0


class TransportError(RuntimeError):
    """Protocol violation or cancelled collective (transport.py:28-29)."""


class DeadlockError(TransportError):
    """A blocking operation timed out; the message names the endpoints."""


class WorkerFailure(TransportError):
    """A worker body raised; ``rank`` and ``cause`` identify it."""

    def __init__(self, rank: int, cause: BaseException):
        super().__init__(f"worker {rank} failed: {cause!r}")
        self.rank = rank
        self.cause = cause


class WorkerGroup:
    """Shared state of G cooperating in-process workers.

    One condition variable guards every channel, the generation-counted
    barrier and the all-to-all staging table; the first failure cancels all
    waits.  Semantics follow transport.py:45-146.
    """

    def __init__(self, size: int, timeout: float = DEFAULT_TIMEOUT, channel_capacity: int = 64):
        if size < 1:
            raise ValueError(f"group size must be >= 1, got {size}")
        self.size = size
        self.timeout = timeout
        self.channel_capacity = channel_capacity
        self._cv = threading.Condition()
        self._queues: dict[tuple[int, int, int], deque] = {}
        self._gen = 0
        self._arrived: set[int] = set()
        self._table: list = [None] * size
        self._dev_table: list = [None] * size
        self._failure: WorkerFailure | None = None

    # -- cancellation ---------------------------------------------------------
    def _fail(self, rank: int, cause: BaseException) -> None:
        with self._cv:
            if self._failure is None:
                self._failure = WorkerFailure(rank, cause)
            self._cv.notify_all()
            subs = list(self.__dict__.get("_subgroups", {}).values())
        for sub in subs:  # cancel waits in row/column sub-groups too
            sub._fail(rank, cause)

    def _raise_if_cancelled(self) -> None:
        if self._failure is not None:
            raise TransportError(f"group cancelled: {self._failure}") from self._failure

    def _wait(self, pred: Callable[[], bool], on_timeout: Callable[[], str]) -> None:
        while not pred():
            self._raise_if_cancelled()
            if not self._cv.wait(self.timeout):
                if pred():
                    return
                raise DeadlockError(on_timeout())
        self._raise_if_cancelled()

    # -- point to point -------------------------------------------------------
    def _send(self, src: int, dst: int, tag: int, payload: Any) -> None:
        if not 0 <= dst < self.size:
            raise TransportError(f"send: destination rank {dst} out of range")
        if dst == src:
            raise TransportError(f"send: rank {src} cannot send to itself")
        with self._cv:
            q = self._queues.setdefault((src, dst, tag), deque())
            self._wait(lambda: len(q) < self.channel_capacity,
                       lambda: f"send timeout: rank {src} -> rank {dst} tag {tag} "
                               f"(channel full, receiver absent)")
            q.append(payload)
            self._cv.notify_all()

    def _receive(self, dst: int, src: int, tag: int) -> Any:
        if not 0 <= src < self.size:
            raise TransportError(f"receive: source rank {src} out of range")
        with self._cv:
            q = self._queues.setdefault((src, dst, tag), deque())
            self._wait(lambda: len(q) > 0,
                       lambda: f"receive timeout: rank {dst} waiting on src={src} tag={tag}")
            item = q.popleft()
            self._cv.notify_all()
            return item

    # -- collectives ------------------------------------------------------------
    def _barrier(self, rank: int) -> None:
        with self._cv:
            gen = self._gen
            self._arrived.add(rank)
            if len(self._arrived) == self.size:
                self._arrived.clear()
                self._gen += 1
                self._cv.notify_all()
                return
            self._wait(lambda: self._gen != gen,
                       lambda: f"barrier timeout at generation {gen}: absent ranks "
                               f"{sorted(set(range(self.size)) - self._arrived)}")

    def _all_to_all(self, rank: int, blocks: Sequence) -> list:
        if len(blocks) != self.size:
            err = TransportError(f"all_to_all: rank {rank} supplied {len(blocks)} blocks, "
                                 f"expected {self.size}")
            self._fail(rank, err)
            raise err
        self._table[rank] = blocks
        self._barrier(rank)
        out = [self._table[g][rank] for g in range(self.size)]
        self._barrier(rank)
        return out

    def _exchange(self, rank: int, send, send_counts, recv, recv_counts) -> None:
        """Device all-to-all(v): rank h receives, in source order, block h of
        every rank's flat ``send`` buffer into its flat ``recv`` buffer."""
        import torch

        G = self.size
        if len(send_counts) != G or len(recv_counts) != G:
            err = TransportError(f"exchange: rank {rank} supplied wrong count vectors")
            self._fail(rank, err)
            raise err
        stream = torch.cuda.current_stream(send.device)
        ready = torch.cuda.Event()
        ready.record(stream)
        soff = [0]
        for c in send_counts:
            soff.append(soff[-1] + int(c))
        self._dev_table[rank] = (send, soff, ready)
        self._barrier(rank)
        roff = 0
        for g in range(G):
            src, offs, ev = self._dev_table[g]
            n = int(recv_counts[g])
            if offs[rank + 1] - offs[rank] != n:
                err = TransportError(f"exchange: rank {g} sends {offs[rank + 1] - offs[rank]} "
                                     f"elements to rank {rank}, which expects {n}")
                self._fail(rank, err)
                raise err
            if n:
                stream.wait_event(ev)
                recv[roff:roff + n].copy_(src[offs[rank]:offs[rank] + n], non_blocking=True)
            roff += n
        done = torch.cuda.Event()
        done.record(stream)
        self._barrier(rank)
        # publish "my reads are done" so senders may reuse their buffers
        self._dev_table[rank] = (None, None, done)
        self._barrier(rank)
        for g in range(G):
            if g != rank:
                stream.wait_event(self._dev_table[g][2])
        self._barrier(rank)


class Worker:
    """Per-rank handle of an in-process group (transport.py:149-171)."""

    def __init__(self, group: WorkerGroup, rank: int, device=None):
        self.group = group
        self.rank = rank
        self.device = device
        self.meter = None

    @property
    def size(self) -> int:
        return self.group.size

    def send(self, dst: int, tag: int, payload: Any) -> None:
        self.group._send(self.rank, dst, tag, payload)

    def receive(self, src: int, tag: int) -> Any:
        return self.group._receive(self.rank, src, tag)

    def all_to_all(self, blocks: Sequence) -> list:
        return self.group._all_to_all(self.rank, blocks)

    def barrier(self) -> None:
        self.group._barrier(self.rank)

    def exchange(self, send, send_counts, recv, recv_counts) -> None:
        if self.group.size == 1:
            n = int(send_counts[0])
            if n and recv.data_ptr() != send.data_ptr():
                recv[:n].copy_(send[:n])
            return
        self.group._exchange(self.rank, send, send_counts, recv, recv_counts)

    def subgroup(self, ranks: Sequence[int]) -> "Worker":
        """Handle on the sub-group ``ranks`` (all members must call it with
        the same tuple).  Used for the row/column exchanges of a pencil
        decomposition."""
        ranks = tuple(int(r) for r in ranks)
        if self.rank not in ranks:
            raise TransportError(f"rank {self.rank} is not in sub-group {ranks}")
        g = self.group
        with g._cv:
            sub = g.__dict__.setdefault("_subgroups", {}).get(ranks)
            if sub is None:
                sub = WorkerGroup(len(ranks), timeout=g.timeout)
                g._subgroups[ranks] = sub
        return Worker(sub, ranks.index(self.rank), self.device)

    def pencil_groups(self, pr: int, pc: int) -> tuple:
        """(row, col) sub-workers of a pr x pc process grid, rank = r*pc + c:
        the row group shares c (size pr, ordered by r), the column group
        shares r (size pc, ordered by c)."""
        r, c = divmod(self.rank, pc)
        return (self.subgroup([rr * pc + c for rr in range(pr)]),
                self.subgroup([r * pc + cc for cc in range(pc)]))

    def send_tensor(self, dst: int, tag: int, t) -> None:
        """Device point-to-point send (handed over by reference in a thread
        group; the receiver copies).  The sender must not mutate ``t``
        afterwards (exclusive handoff, transport.py:4-6)."""
        import torch

        ev = torch.cuda.Event()
        ev.record(torch.cuda.current_stream(t.device))
        self.send(dst, tag, (t, ev))

    def recv_tensor(self, src: int, tag: int, out=None):
        import torch

        t, ev = self.receive(src, tag)
        stream = torch.cuda.current_stream()
        stream.wait_event(ev)
        if out is None:
            out = torch.empty_like(t, device=torch.cuda.current_device())
        out.copy_(t, non_blocking=True)
        return out

    def bcast_groups(self, sets: Sequence[Sequence[int]]) -> None:
        """Declare the broadcast rank sets (collective on process groups;
        nothing to set up in a thread group)."""

    def bcast_tensor(self, root: int, ranks: Sequence[int], tag: int, t=None, out=None):
        """``root`` sends ``t`` to every other member of ``ranks`` (all
        members call it; receivers pass ``out``); returns the member's copy.
        In a thread group: one reference handoff per receiver."""
        if self.rank == root:
            for r in ranks:
                if r != root:
                    self.send_tensor(r, tag, t)
            return t
        return self.recv_tensor(root, tag, out)


class ProcessWorker:
    """Worker over ``torch.distributed`` (one process per GPU).

    Host payloads use object collectives (tags are accepted for API
    compatibility; the hydro schedule relies only on per-pair ordering,
    which torch.distributed preserves).  ``exchange`` is NCCL
    ``all_to_all_single`` on CUDA tensors; under gloo it is staged through
    host memory.
    """

    def __init__(self, group=None, device=None, ranks=None):
        import torch.distributed as dist

        self._dist = dist
        self.pg = group
        # global ranks of the group members (sub-groups); point-to-point
        # calls take global ranks
        self._global = list(ranks) if ranks is not None else list(range(dist.get_world_size()))
        self.rank = self._global.index(dist.get_rank())
        self._size = len(self._global)
        self.device = device
        self.meter = None
        self.backend = dist.get_backend(group)

    @property
    def size(self) -> int:
        return self._size

    def barrier(self) -> None:
        self._dist.barrier(group=self.pg)

    def all_to_all(self, blocks: Sequence) -> list:
        if len(blocks) != self._size:
            raise TransportError(f"all_to_all: rank {self.rank} supplied {len(blocks)} blocks, "
                                 f"expected {self._size}")
        gathered: list = [None] * self._size
        self._dist.all_gather_object(gathered, list(blocks), group=self.pg)
        return [gathered[g][self.rank] for g in range(self._size)]

    def send(self, dst: int, tag: int, payload: Any) -> None:
        if dst == self.rank:
            raise TransportError(f"send: rank {self.rank} cannot send to itself")
        self._dist.send_object_list([tag, payload], dst=self._global[dst], group=self.pg)

    def receive(self, src: int, tag: int) -> Any:
        box = [None, None]
        self._dist.recv_object_list(box, src=self._global[src], group=self.pg)
        if box[0] != tag:
            raise TransportError(f"receive: rank {self.rank} expected tag {tag} from {src}, "
                                 f"got {box[0]}")
        return box[1]

    def exchange(self, send, send_counts, recv, recv_counts) -> None:
        import torch

        sc = [int(c) for c in send_counts]
        rc = [int(c) for c in recv_counts]
        s = send[:sum(sc)]
        r = recv[:sum(rc)]
        if self.backend == "nccl":
            self._dist.all_to_all_single(r, s, output_split_sizes=rc, input_split_sizes=sc,
                                         group=self.pg)
            return
        # gloo: stage through host memory (CPU tests, 1-GPU multi-process tests)
        s_h = s.cpu() if s.is_cuda else s
        r_h = torch.empty_like(r, device="cpu")
        if s_h.is_complex():
            s_h = torch.view_as_real(s_h)
            r_v = torch.view_as_real(r_h)
            sc2, rc2 = sc, rc
        else:
            r_v = r_h
            sc2, rc2 = sc, rc
        self._dist.all_to_all_single(r_v, s_h, output_split_sizes=rc2, input_split_sizes=sc2,
                                     group=self.pg)
        r.copy_(r_h)

    def pencil_groups(self, pr: int, pc: int) -> tuple:
        """(row, col) sub-workers of a pr x pc process grid (rank = r*pc + c).
        Collective: every rank creates every row and column group in the
        same order (torch.distributed.new_group semantics)."""
        key = (pr, pc)
        cache = self.__dict__.setdefault("_pencil", {})
        if key not in cache:
            if pr * pc != self._size:
                raise TransportError(f"process grid {pr}x{pc} does not match {self._size} ranks")
            rows, cols = {}, {}
            for c in range(pc):
                ranks = [r * pc + c for r in range(pr)]
                rows[c] = (ranks, self._dist.new_group(ranks))
            for r in range(pr):
                ranks = [r * pc + c for c in range(pc)]
                cols[r] = (ranks, self._dist.new_group(ranks))
            r, c = divmod(self.rank, pc)
            cache[key] = (ProcessWorker(rows[c][1], self.device, rows[c][0]),
                          ProcessWorker(cols[r][1], self.device, cols[r][0]))
        return cache[key]

    def bcast_groups(self, sets: Sequence[Sequence[int]]) -> None:
        """Create the communicators of the broadcast rank sets (group ranks).
        Collective: every rank of the group calls it with the same sets in
        the same order (torch.distributed.new_group semantics); cached."""
        cache = self.__dict__.setdefault("_bcast", {})
        for ranks in sets:
            key = tuple(sorted(int(r) for r in ranks))
            if key in cache:
                continue
            if len(key) == self._size:
                cache[key] = self.pg
            else:
                cache[key] = self._dist.new_group([self._global[r] for r in key])

    def bcast_tensor(self, root: int, ranks: Sequence[int], tag: int, t=None, out=None):
        """``root`` broadcasts ``t`` to the other members of ``ranks`` (all
        members call it; receivers pass ``out``): one NCCL broadcast over the
        set's communicator instead of a send per receiver, so the root's
        link carries the field once (NCCL pipelines it through the members
        or the switch).  The set must have been declared with
        bcast_groups."""
        key = tuple(sorted(int(r) for r in ranks))
        group = self.__dict__.get("_bcast", {}).get(key, "missing")
        if group == "missing":
            raise TransportError(f"bcast_tensor: rank set {key} was not declared with bcast_groups")
        buf = t.contiguous() if self.rank == root else out
        src = self._global[root]
        if self.backend == "nccl":
            self._dist.broadcast(buf, src=src, group=group)
        else:  # gloo: stage through host memory
            host = buf.cpu() if buf.is_cuda else buf
            self._dist.broadcast(host, src=src, group=group)
            if host is not buf:
                buf.copy_(host)
        return buf

    def send_tensor(self, dst: int, tag: int, t) -> None:
        if self.backend == "nccl":
            self._dist.send(t.contiguous(), dst=self._global[dst], group=self.pg)
        else:
            self._dist.send(t.contiguous().cpu(), dst=self._global[dst], group=self.pg)

    def recv_tensor(self, src: int, tag: int, out):
        if self.backend == "nccl":
            self._dist.recv(out, src=self._global[src], group=self.pg)
        else:
            tmp = out.cpu() if out.is_cuda else out
            self._dist.recv(tmp, src=self._global[src], group=self.pg)
            if tmp is not out:
                out.copy_(tmp)
        return out


def _bind_device(rank: int):
    try:
        import torch

        if torch.cuda.is_available():
            dev = rank % torch.cuda.device_count()
            torch.cuda.set_device(dev)
            return torch.device("cuda", dev)
    except Exception:  # pragma: no cover - torch import problems surface later
        pass
    return None


def spawn_group(size: int, body: Callable[[Worker], Any], timeout: float = DEFAULT_TIMEOUT) -> list:
    """Run ``body(worker)`` on ``size`` thread workers and return the
    per-rank results; the first failure cancels the group and is re-raised
    as :class:`WorkerFailure` (transport.py:174-200)."""
    group = WorkerGroup(size, timeout=timeout)
    results: list = [None] * size

    def run(rank: int) -> None:
        w = Worker(group, rank, _bind_device(rank))
        try:
            results[rank] = body(w)
        except BaseException as exc:  # noqa: BLE001 - the group must be cancelled
            group._fail(rank, exc)

    threads = [threading.Thread(target=run, args=(r,), name=f"worker-{r}", daemon=True)
               for r in range(size)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if group._failure is not None:
        raise group._failure
    return results

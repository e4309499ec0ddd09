"""The one-process-per-GPU transport (transport.ProcessWorker) on CPU with
the gloo backend, world size 2 and 3: host collectives, tagged point to
point, and the slab all-to-all(v) bookkeeping of distfft._Geometry — the
exact split sizes the NCCL exchange uses — checked against the reference's
concatenate semantics (distfft.py:110-124)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # pragma: no cover - surfaced below
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def spawn(fn, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return [out[r] for r in range(world)]


def _collectives(rank, world):
    from paper_2603_26818_b200.pfc import _reduce_max, _reduce_sum
    from paper_2603_26818_b200.transport import ProcessWorker

    w = ProcessWorker()
    got = w.all_to_all([(rank, h) for h in range(world)])
    if rank == 0:
        w.send(1, 2, {"psi": [1.0, 2.0]})
        msg = None
    elif rank == 1:
        msg = w.receive(0, 2)
    else:
        msg = None
    w.barrier()
    vals = [0.1, 1e16, -1e16][:world]
    return got, msg, _reduce_sum(w, vals[rank]), _reduce_max(w, vals[rank])


@pytest.mark.parametrize("world", [2, 3])
def test_process_worker_collectives(world):
    res = spawn(_collectives, world)
    for r, (got, msg, s, m) in enumerate(res):
        assert got == [(g, r) for g in range(world)]
    assert res[1][1] == {"psi": [1.0, 2.0]}
    assert len({x[2] for x in res}) == 1  # identical rank-ordered sum on every rank
    total = 0.0
    for v in [0.1, 1e16, -1e16][:world]:
        total += v
    assert res[0][2] == total


def _slab_exchange(rank, world):
    """Forward slab exchange of distfft with the real split sizes."""
    from paper_2603_26818_b200.distfft import _Geometry
    from paper_2603_26818_b200.grid import GridSpec, slab_layout
    from paper_2603_26818_b200.transport import ProcessWorker

    w = ProcessWorker()
    out = {}
    for shape, real in [((8, 6, 10), False), ((10, 4, 7), True), ((6, 5, 1), False)]:
        grid = GridSpec(shape, (1.0, 1.0, 1.0))
        g = _Geometry(grid, world, rank, real)
        full = np.arange(g.nxm * g.ny * g.nz, dtype=np.float64).reshape(g.nxm, g.ny, g.nz)
        zl = slab_layout(g.nz, world)
        zslab = np.ascontiguousarray(full[:, :, zl.offsets[rank]:zl.offsets[rank] + zl.counts[rank]])
        send = torch.from_numpy(zslab.reshape(-1).astype(np.complex128))
        sc, rc = g.fwd_counts()
        recv = torch.empty(sum(rc), dtype=torch.complex128)
        w.exchange(send, sc, recv, rc)
        # the kernel's blocked addressing: block g is (cx*ny, cz_g) at offset cx*ny*zoff_g
        xl = slab_layout(g.nxm, world)
        want = full[xl.offsets[rank]:xl.offsets[rank] + xl.counts[rank]]
        rebuilt = np.empty_like(want)
        off = 0
        for src in range(world):
            cz, z0 = zl.counts[src], zl.offsets[src]
            n = g.cx * g.ny * cz
            rebuilt[:, :, z0:z0 + cz] = recv[off:off + n].real.numpy().reshape(g.cx, g.ny, cz)
            off += n
        # and the inverse direction returns the original slab
        sc2, rc2 = g.inv_counts()
        back = torch.empty(sum(rc2), dtype=torch.complex128)
        w.exchange(recv, sc2, back, rc2)
        out[str(shape)] = (bool(np.array_equal(rebuilt, want)),
                           bool(np.array_equal(back.real.numpy().reshape(zslab.shape), zslab)))
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_slab_all_to_all_bookkeeping(world):
    for res in spawn(_slab_exchange, world):
        assert isinstance(res, dict), res
        for key, (fwd_ok, inv_ok) in res.items():
            assert fwd_ok and inv_ok, key


def _bcast(rank, world):
    """ProcessWorker.bcast_tensor over declared rank sets (the role maps'
    psi -> velocities and v_i -> (psi, c, helper) broadcasts), with the
    same call order on every member, plus an undeclared set."""
    from paper_2603_26818_b200.transport import ProcessWorker, TransportError

    w = ProcessWorker()
    sets = [(0, 1, 2, 3), (0, 1, 4), (0, 2, 4), (0, 3, 4)][: 1 if world == 4 else 4]
    w.bcast_groups(sets)
    got = {}
    x = torch.full((5,), 10.0 + rank, dtype=torch.float64)
    if rank in (0, 1, 2, 3):
        out = w.bcast_tensor(0, (0, 1, 2, 3), 2, t=x if rank == 0 else None,
                             out=None if rank == 0 else torch.empty(5, dtype=torch.float64))
        got["psi"] = out.tolist()
    if world == 5:
        for i in range(3):
            s = sets[1 + i]
            if rank in s:
                root = 1 + i
                out = w.bcast_tensor(root, s, 4 + i, t=x if rank == root else None,
                                     out=None if rank == root else torch.empty(5, dtype=torch.float64))
                got[f"v{i}"] = out.tolist()
    try:
        w.bcast_tensor(0, (0, 3), 9, t=x, out=x)
        got["undeclared"] = "no error"
    except TransportError:
        got["undeclared"] = "error"
    return got


@pytest.mark.parametrize("world", [4, 5])
def test_process_worker_bcast(world):
    res = spawn(_bcast, world)
    for r, got in enumerate(res):
        assert isinstance(got, dict), got
        assert got["undeclared"] == "error"
        if r < 4:
            assert got["psi"] == [10.0] * 5
        if world == 5:
            for i in range(3):
                if r in (0, 1 + i, 4):
                    assert got[f"v{i}"] == [11.0 + i] * 5

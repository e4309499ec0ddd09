"""Fused exchanges (transposes stored straight into the owners' receive
buffers from the FFT epilogues) against the collective path and the
single-rank result — bit-identical — for thread groups and for processes
(CUDA IPC between processes sharing the test GPU, gloo for host barriers)."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_26818_b200 as p

    return p


def _run(pkg, G, mode, real, steps=12, n=(16, 32, 16)):
    from paper_2603_26818_b200 import distfft, pfc

    os.environ["PFCS_EXCHANGE"] = mode
    try:
        grid = pkg.GridSpec(n, pfc.default_domain_length(n))
        psi0 = pfc.initial_field("constant_plus_noise", grid, seed=9, noise_amplitude=0.05)

        def body(w):
            sym = pkg.make_symbols(grid, -0.3)
            f = distfft.scatter(psi0, w, grid, distfft.Layout.Z_SLAB, real=real) if real else \
                distfft.scatter(psi0.astype(np.complex128), w, grid, distfft.Layout.Z_SLAB)
            st = pfc.PfcState(psi_hat=distfft.forward(f, w), grid=grid, symbols=sym, worker=w)
            pfc.pfc_run(st, pfc.PfcParams(), steps // 2)
            for _ in range(steps - steps // 2):
                pfc.pfc_step(st, pfc.PfcParams())
            assert st._engine.peer == (mode == "peer" and w.size > 1)
            return distfft.gather(distfft.inverse(st.psi_hat, w), w)

        return pkg.spawn_group(G, body)[0]
    finally:
        os.environ.pop("PFCS_EXCHANGE", None)


@pytest.mark.parametrize("G", [2, 3, 4])
@pytest.mark.parametrize("real", [True, False])
def test_peer_exchange_threads_bitwise(pkg, G, real):
    ref = _run(pkg, 1, "peer", real)
    np.testing.assert_array_equal(_run(pkg, G, "peer", real), ref)
    np.testing.assert_array_equal(_run(pkg, G, "collective", real), ref)


def _proc_body(rank, world, port, mode, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), PFCS_EXCHANGE=mode)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2603_26818_b200 as pkg
        from paper_2603_26818_b200 import distfft, pfc
        from paper_2603_26818_b200.transport import ProcessWorker

        w = ProcessWorker(device=torch.device("cuda", 0))
        n = (16, 32, 16)
        grid = pkg.GridSpec(n, pfc.default_domain_length(n))
        psi0 = pfc.initial_field("constant_plus_noise", grid, seed=9, noise_amplitude=0.05)
        f = distfft.scatter(psi0, w, grid, distfft.Layout.Z_SLAB, real=True)
        st = pfc.PfcState(psi_hat=distfft.forward(f, w), grid=grid, symbols=pkg.make_symbols(grid, -0.3),
                          worker=w)
        pfc.pfc_run(st, pfc.PfcParams(), 6)
        for _ in range(6):
            pfc.pfc_step(st, pfc.PfcParams())
        out = distfft.gather(distfft.inverse(st.psi_hat, w), w)
        q.put((rank, st._engine.peer, out))
    except Exception as e:  # pragma: no cover - reported below
        q.put((rank, None, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["peer", "collective"])
def test_exchange_processes_ipc_bitwise(pkg, mode):
    import torch.multiprocessing as mp

    ref = _run(pkg, 1, "peer", True)
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_proc_body, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
    for rank, peer, out in res:
        assert peer is not None, out
        assert peer == (mode == "peer")
        np.testing.assert_array_equal(out, ref)


@pytest.mark.parametrize("fail_rank", [0, 1])
def test_peer_mapping_failure_falls_back_on_every_rank(pkg, monkeypatch, fail_rank):
    """If ANY rank cannot map a peer buffer (no P2P / no CUDA IPC), every
    rank raises PeerUnavailable together and the step engine and the
    distributed FFT fall back to the collective exchange — same results."""
    from paper_2603_26818_b200 import peer

    real_map = peer._map_rank

    def flaky(worker, buf, lib, dev):
        pm = real_map(worker, buf, lib, dev)
        if worker.rank == fail_rank:
            raise RuntimeError("injected: no peer access")
        return pm

    monkeypatch.setattr(peer, "_map_rank", flaky)
    ref = _run(pkg, 1, "peer", True)
    with pytest.warns(UserWarning, match="fused peer exchange unavailable"):
        got = _run_fallback(pkg, 2)
    np.testing.assert_array_equal(got, ref)


def _run_fallback(pkg, G, steps=12, n=(16, 32, 16)):
    from paper_2603_26818_b200 import distfft, pfc

    grid = pkg.GridSpec(n, pfc.default_domain_length(n))
    psi0 = pfc.initial_field("constant_plus_noise", grid, seed=9, noise_amplitude=0.05)

    def body(w):
        sym = pkg.make_symbols(grid, -0.3)
        f = distfft.scatter(psi0, w, grid, distfft.Layout.Z_SLAB, real=True)
        st = pfc.PfcState(psi_hat=distfft.forward(f, w), grid=grid, symbols=sym, worker=w)
        pfc.pfc_run(st, pfc.PfcParams(), steps // 2)
        for _ in range(steps - steps // 2):
            pfc.pfc_step(st, pfc.PfcParams())
        assert not st._engine.peer
        return distfft.gather(distfft.inverse(st.psi_hat, w), w)

    return pkg.spawn_group(G, body)[0]

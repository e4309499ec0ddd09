"""Probe: y pass then z pass over chunks of x-planes, so the y pass's output
is still in L2 when the z pass reads it (half the HBM traffic of the two
full-array passes).  Not product code.

    python tools/probe_l2chain.py [n] [reps] [chunks...]

Times (CUDA events, in-place forward y + z over the (n/2+1, n, n) half
spectrum): the two full passes, then per chunk size P: one stream (y(c); z(c)),
and two streams (z(c) on its own stream after y(c); y(c + 2) waits for z(c)).
Checks every chunked result is bit-identical to the full passes."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))


def main():
    import torch

    from paper_2603_26818_b200 import _native as nat

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    chunks = [int(v) for v in sys.argv[3:]] or [2, 4, 8, 16, 32]
    torch.cuda.set_device(0)
    nh = n // 2 + 1
    plane = n * n
    src = torch.empty(nh * plane, dtype=torch.complex128, device="cuda")
    src.real.normal_()
    src.imag.normal_()
    a = src.clone()
    esz = 16
    S = {"s0": torch.cuda.current_stream(), "s1": torch.cuda.Stream()}

    def y(p0, p1, st):
        nat.call("pfcs_fft_axis_c2c", a.data_ptr() + p0 * plane * esz, a.data_ptr() + p0 * plane * esz, p1 - p0, n,
                 n, 1, 1, st.cuda_stream)

    def z(p0, p1, st):
        nat.call("pfcs_fft_axis_c2c", a.data_ptr() + p0 * plane * esz, a.data_ptr() + p0 * plane * esz, p1 - p0, n,
                 n, 2, 1, st.cuda_stream)

    def full():
        s0 = S["s0"]
        y(0, nh, s0)
        z(0, nh, s0)

    def one_stream(P):
        s0 = S["s0"]
        for p0 in range(0, nh, P):
            p1 = min(nh, p0 + P)
            y(p0, p1, s0)
            z(p0, p1, s0)

    def two_streams(P):
        s0, s1 = S["s0"], S["s1"]
        starts = list(range(0, nh, P))
        ydone = [torch.cuda.Event() for _ in starts]
        zdone = [torch.cuda.Event() for _ in starts]
        s1.wait_stream(s0)
        for i, p0 in enumerate(starts):
            p1 = min(nh, p0 + P)
            if i >= 2:
                s0.wait_event(zdone[i - 2])
            y(p0, p1, s0)
            ydone[i].record(s0)
            s1.wait_event(ydone[i])
            z(p0, p1, s1)
            zdone[i].record(s1)
        s0.wait_stream(s1)

    def graphed(fn):
        a.copy_(src)
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream()
        with torch.cuda.stream(cap):
            S["s0"] = cap
            with torch.cuda.graph(g, stream=cap):
                fn()
        S["s0"] = torch.cuda.current_stream()
        return g.replay

    def timed(fn):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        fn = graphed(fn)
        ms = []
        for _ in range(reps):
            a.copy_(src)
            ev[0].record()
            fn()
            ev[1].record()
            torch.cuda.synchronize()
            ms.append(ev[0].elapsed_time(ev[1]))
        return min(ms), sorted(ms)[len(ms) // 2]

    print(f"n={n}: full y + z: best/median %.4f / %.4f ms" % timed(full))
    a.copy_(src)
    full()
    want = a.clone()
    for P in chunks:
        for name, fn in (("1 stream", one_stream), ("2 streams", two_streams)):
            t = timed(lambda: fn(P))
            a.copy_(src)
            fn(P)
            torch.cuda.synchronize()
            same = bool(torch.equal(torch.view_as_real(a), torch.view_as_real(want)))
            print(f"n={n}: P={P:3d} {name:9s}: best/median {t[0]:.4f} / {t[1]:.4f} ms  bit-identical={same}")


if __name__ == "__main__":
    main()

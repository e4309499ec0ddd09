"""Concurrent H2D + D2H bandwidth of 1 GiB pinned transfers with k chunks
on k stream pairs (diagnostic for the bench's e2e pipeline)."""
import torch

n = 1 << 27  # 1 GiB of float64
hin = torch.empty(n, dtype=torch.float64).pin_memory()
hout = torch.empty(n, dtype=torch.float64).pin_memory()
din = torch.empty(n, dtype=torch.float64, device="cuda")
dout = torch.zeros(n, dtype=torch.float64, device="cuda")
for k in (1, 2, 4, 8):
    ups = [torch.cuda.Stream() for _ in range(k)]
    downs = [torch.cuda.Stream() for _ in range(k)]
    c = n // k
    torch.cuda.synchronize()
    for rep in range(2):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        for i in range(k):
            ups[i].wait_event(a)
            downs[i].wait_event(a)
            with torch.cuda.stream(ups[i]):
                din[i * c:(i + 1) * c].copy_(hin[i * c:(i + 1) * c], non_blocking=True)
            with torch.cuda.stream(downs[i]):
                hout[i * c:(i + 1) * c].copy_(dout[i * c:(i + 1) * c], non_blocking=True)
        cur = torch.cuda.current_stream()
        for s in ups + downs:
            cur.wait_stream(s)
        b.record()
        torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"k={k}: 1 GiB up + 1 GiB down concurrently in {ms:.2f} ms -> {2 * 8 * n / ms / 1e6:.1f} GB/s total")

# one direction at a time, and where the host memory sits relative to the GPU
for name, fn in (("H2D only", lambda: din.copy_(hin, non_blocking=True)),
                 ("D2H only", lambda: hout.copy_(dout, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(f"{name}: 1 GiB in {ms:.2f} ms -> {8 * n / ms / 1e6:.1f} GB/s")
try:
    import glob
    import subprocess

    print(subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id,pcie.link.gen.current,pcie.link.width.current",
                          "--format=csv,noheader"], capture_output=True, text=True).stdout.strip())
    for p in glob.glob("/sys/bus/pci/devices/*/numa_node"):
        pass
    print("host NUMA nodes:", len(glob.glob("/sys/devices/system/node/node[0-9]*")))
except Exception as exc:  # diagnostics only
    print("topology query failed:", exc)

"""Where fdog_create_from_plan's time goes on the default workload (MRF-LP):
the whole create (torch allocator and cudaMalloc), against a plain pinned
H2D copy of the same number of bytes (the transfer's floor)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2111_10270_b200 as F  # noqa: E402
import synth  # noqa: E402

p = synth.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "mrf_potts"](0)
pl = F.Plan(p, precision=32)
torch.cuda.init()
torch.zeros(1, device="cuda")
for alloc in ("torch", "cuda", "torch", "cuda"):
    torch.cuda.synchronize()
    t = time.perf_counter()
    s = F.Solver(plan=pl, precision=32, allocator=alloc)
    s.lower_bound()  # (synchronises the solver's stream)
    dt = time.perf_counter() - t
    st = s.stats()
    print(f"create ({alloc}): {dt * 1e3:.1f} ms, h2d {st['h2d_bytes'] / 1e6:.0f} MB, device {st['device_bytes'] / 1e6:.0f} MB", flush=True)
    s.close()
    del s
nb = pl.stats()["h2d_bytes"] if "h2d_bytes" in pl.stats() else st["h2d_bytes"]
h = torch.empty(int(nb), dtype=torch.uint8, pin_memory=True)
d = torch.empty(int(nb), dtype=torch.uint8, device="cuda")
for _ in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"pinned H2D of {nb / 1e6:.0f} MB: {dt * 1e3:.1f} ms ({nb / dt / 1e9:.1f} GB/s)", flush=True)
t = time.perf_counter()
x = torch.empty(int(nb), dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()
print(f"fresh torch allocation: {(time.perf_counter() - t) * 1e3:.1f} ms")

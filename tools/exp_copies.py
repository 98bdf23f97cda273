"""Copy-engine timing for the C2 e2e pipeline: 1 MB pinned H2D / D2H on one
stream, split over two / four streams, both directions at once."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

n = 65536
h_in = torch.randn(n, dtype=torch.complex128).pin_memory()
h_out = torch.empty(n, dtype=torch.complex128).pin_memory()
d_in = torch.empty(n, dtype=torch.complex128, device="cuda")
d_out = torch.randn(n, dtype=torch.complex128, device="cuda")
streams = [torch.cuda.Stream() for _ in range(4)]
R = 200


def run(nsplit, h2d=True, d2h=False):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for s in streams:
        s.wait_event(e0)
    part = n // nsplit
    for _ in range(R):
        for j in range(nsplit):
            sl = slice(j * part, (j + 1) * part)
            if h2d:
                with torch.cuda.stream(streams[j]):
                    d_in[sl].copy_(h_in[sl], non_blocking=True)
            if d2h:
                with torch.cuda.stream(streams[(j + 2) % 4]):
                    h_out[sl].copy_(d_out[sl], non_blocking=True)
    ends = []
    for s in streams:
        e = torch.cuda.Event(enable_timing=True)
        e.record(s)
        ends.append(e)
    torch.cuda.synchronize()
    return max(e0.elapsed_time(e) for e in ends) / R * 1e3


for rep in range(2):
    print(f"H2D 1 MB: 1 stream {run(1):.1f} us, 2 streams {run(2):.1f} us, 4 streams {run(4):.1f} us")
    print(f"D2H 1 MB: 1 stream {run(1, False, True):.1f} us, 2 streams {run(2, False, True):.1f} us")
    print(f"both: 1+1 streams {run(1, True, True):.1f} us, 2+2 streams {run(2, True, True):.1f} us")

"""Do stream events between consecutive persistent applies break the
programmatic (PDL) chaining? Back-to-back C2 applies: plain; with an event
recorded after every apply; with a wait on an (already complete) event of
another stream before every apply."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep  # noqa: E402

cfg = CONFIGS["C2"]
op = ToeplitzMatvec(ToeplitzRep.synthetic(cfg), max_nrhs=1)
st = torch.cuda.Stream()
other = torch.cuda.Stream()
op.set_stream(st.cuda_stream)
x = torch.randn(op.size(), dtype=torch.complex128, device="cuda")
y = torch.empty_like(x)
done = torch.cuda.Event()
done.record(other)
evs = [torch.cuda.Event() for _ in range(4)]
N = 1000
for mode in ("plain", "record", "wait", "record+wait", "plain"):
    for _ in range(20):
        op.apply_device(x.data_ptr(), y.data_ptr())
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for i in range(N):
        if "wait" in mode:
            st.wait_event(done)
        op.apply_device(x.data_ptr(), y.data_ptr())
        if "record" in mode:
            evs[i % 4].record(st)
    e1.record(st)
    st.synchronize()
    print(f"{mode:12s} {e0.elapsed_time(e1) / N * 1e3:6.2f} us per apply", flush=True)

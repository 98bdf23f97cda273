"""Two contexts on one GPU driven concurrently from two host threads (the
C ABI is thread-safe per context): persistent grid-barrier applies must not
interleave into a deadlock — with more than one live context on a device
they are launched cooperatively (csrc/api.cu plainLaunchOk) — and every
result stays bit-identical to the same apply run alone."""
import threading

import numpy as np
import pytest

from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep, gen

pytestmark = pytest.mark.gpu


@pytest.mark.timeout(600)
def test_two_contexts_concurrent_applies(gpu):
    import torch
    cfg = CONFIGS["C2"]
    rep = ToeplitzRep.synthetic(cfg)
    ops = [ToeplitzMatvec(rep), ToeplitzMatvec(rep)]
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    for op, st in zip(ops, streams):
        op.set_stream(st.cuda_stream)
    x = torch.from_numpy(np.asarray(gen.rhs_normal(cfg.n, 1, 5)[:, 0]).copy()).cuda()
    ref = torch.empty_like(x)
    ops[0].apply_device(x.data_ptr(), ref.data_ptr())
    torch.cuda.synchronize()
    outs = [torch.empty_like(x), torch.empty_like(x)]
    errors = []

    def run(k):
        try:
            for _ in range(300):
                ops[k].apply_device(x.data_ptr(), outs[k].data_ptr())
            streams[k].synchronize()
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=run, args=(k,)) for k in range(2)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in threads), "concurrent applies did not finish"
    assert not errors, errors
    for k in range(2):
        assert torch.equal(outs[k], ref), k

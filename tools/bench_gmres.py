"""GMRES time per inner iteration on a config (fixed budget), e.g.
    python tools/bench_gmres.py C3 20 smooth"""
import sys
import time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
from paper_2506_04710_b200 import CONFIGS, SolverOptions, ToeplitzMatvec, ToeplitzRep, rhs_for  # noqa: E402
cfg = CONFIGS[sys.argv[1]]
iters = int(sys.argv[2])
embed = sys.argv[3] if len(sys.argv) > 3 else "pow2"
orthog = int(sys.argv[4]) if len(sys.argv) > 4 else 1
rep = ToeplitzRep.synthetic(cfg)
op = ToeplitzMatvec(rep, max_nrhs=cfg.nrhs, embed=embed)
b = np.asarray(rhs_for(cfg))
opt = SolverOptions(tol=cfg.tol, maxIter=iters, restart=cfg.restart, orthog=orthog)
op.gmres(b, SolverOptions(tol=cfg.tol, maxIter=2, restart=cfg.restart, orthog=orthog), raise_on_fail=False)
t0 = time.perf_counter()
r = op.gmres(b, opt, raise_on_fail=False)
dt = time.perf_counter() - t0
print(f"{cfg.name} nrhs={cfg.nrhs} embed={embed} orthog={orthog}: {iters} iterations in {dt*1e3:.1f} ms "
      f"({dt / iters * 1e3:.3f} ms/iter incl. host copies), final residual {np.max(r.residual):.3e}")
# Device-resident b / x (no host copies): solver time only.
import torch  # noqa: E402
from paper_2506_04710_b200.toeplitz import TBT_DEVICE  # noqa: E402
ncol = 1 if b.ndim == 1 else b.shape[1]
bdc = torch.from_numpy(np.ascontiguousarray(b.reshape(cfg.n, -1).T)).cuda()  # column-major = [col][n]
xdc = torch.empty_like(bdc)
op.set_stream(torch.cuda.current_stream().cuda_stream)
for rep_i in range(2):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = op.gmres(None, opt, raise_on_fail=False, where=TBT_DEVICE, b_ptr=bdc.data_ptr(), x_ptr=xdc.data_ptr(),
                 nrhs=ncol)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"  device-resident solve {rep_i}: {ms:.1f} ms ({ms / iters:.3f} ms/iter)")

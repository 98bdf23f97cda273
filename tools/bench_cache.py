"""Row f3 measurement: operator setup with K1 (generators -> spectra) vs
from a persisted TBTS1 spectrum, on a BASELINE config."""
import json
import os
import sys
import tempfile
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2506_04710_b200 import CONFIGS, ToeplitzMatvec, ToeplitzRep  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C4"]
rep = ToeplitzRep.synthetic(cfg)
d = tempfile.mkdtemp()
path = os.path.join(d, "spec.tbts")
ToeplitzMatvec(rep).close()  # warm the CUDA context / module load
t0 = time.perf_counter()
op = ToeplitzMatvec(rep)
t_k1 = time.perf_counter() - t0
op.close()
t0 = time.perf_counter()
op = ToeplitzMatvec(rep, spectra_cache=path)
t_save = time.perf_counter() - t0
op.close()
t0 = time.perf_counter()
op = ToeplitzMatvec(rep, spectra_cache=path)
t_load = time.perf_counter() - t0
print(json.dumps({"config": cfg.name, "setup_with_k1_s": t_k1, "setup_k1_and_save_s": t_save,
                  "setup_from_cache_s": t_load, "cache_bytes": os.path.getsize(path)}))
os.remove(path)

"""Sharded apply on one NCCL rank (self exchanges) with a given chunk count
(TBT_DIST_CHUNKS, read once per process): device ms per matvec.

    for k in 1 2 4; do TBT_DIST_CHUNKS=$k python tools/dist_overlap.py C2 C4; done
"""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import bench  # noqa: E402

for name in sys.argv[1:]:
    r = bench.sharded_measure(name, 1, 0, 0, None, steps=50, gmres_iters=20)
    print(json.dumps({"config": name, "chunks": os.environ.get("TBT_DIST_CHUNKS", "default"), **r}), flush=True)

"""build_pocket (the step before the hot path): host (C++, OpenMP on all cores) vs the
device kernel (thread per node) on the synthetic pocket and its L2 variant; checks the grids are
identical and prints one JSON line."""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_05069_b200 import io, native  # noqa: E402

ctx = native.Context(0)
atoms = io.pocket_atoms(200, seed=7)
xyz = np.array([a.position for a in atoms], np.float32)
out = {"workload": "build_pocket, 200 synthetic pocket atoms (shell 7-10 A), padding 4 A", "cores": os.cpu_count()}
for spacing in (0.5, 0.375):
    t0 = time.perf_counter()
    host = io.build_pocket(atoms, spacing, 4.0)
    t_host = time.perf_counter() - t0
    ctx.build_pocket_grid(xyz, spacing, 4.0)  # warm-up
    ms = []
    for _ in range(5):
        o, d, v, k = ctx.build_pocket_grid(xyz, spacing, 4.0)
        ms.append(k)
    same = bool(np.array_equal(v, np.asarray(host.grid_values)))
    out[str(spacing)] = {"dims": list(d), "nodes": int(np.prod(d)), "host_ms": 1e3 * t_host,
                         "device_kernel_ms": float(np.median(ms)), "identical": same}
print(json.dumps(out))

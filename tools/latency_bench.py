"""BASELINE config 2: single large ligand (~90 atoms, 20 rotatable bonds) time-to-result.

Device-timed (CUDA events on the context stream, H2D + kernels + D2H) for the latency family
and the batched family on the same single ligand, plus the CPU oracle on one core.  Prints one
JSON line."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_05069_b200 import io, model, native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--no-cpu", action="store_true")
a = ap.parse_args()

pocket = io.synthetic_pocket()
table = native.InteractionTable.default()
cands = io.generate_dataset_batch(36, 20, 64, seed=2)
A = np.diff(cands.atom_off)
pick = int(np.nonzero((A >= 86) & (A <= 94))[0][0])
lig = cands.subset([pick])
packed = native.pack(lig)
cfg = model.DockConfig()
ctx = native.Context(0)
dp = ctx.pocket(pocket, table)
out = {"workload": "config2 single ligand", "atoms": int(A[pick]), "fragments": 20}
for name, fam in (("latency", native.FAMILY_LATENCY), ("batched", native.FAMILY_BATCHED)):
    for _ in range(3):
        ctx.dock(dp, packed, cfg, 0, fam)
    dev, wall = [], []
    for _ in range(a.reps):
        t0 = time.perf_counter()
        o = ctx.dock(dp, packed, cfg, 0, fam)
        wall.append(time.perf_counter() - t0)
        dev.append(o.stats.total_ms)
    out[name] = {"device_ms_median": float(np.median(dev)), "wall_ms_median": 1e3 * float(np.median(wall)),
                 "align_ms": float(o.stats.align_ms), "optimize_ms": float(o.stats.optimize_ms)}
if not a.no_cpu:
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    t0 = time.perf_counter()
    oracle.dock_batch(lig, pocket, table, cfg, threads=1)
    out["cpu_oracle_1core_ms"] = 1e3 * (time.perf_counter() - t0)
out["latency_speedup_vs_batched"] = out["batched"]["device_ms_median"] / out["latency"]["device_ms_median"]
print(json.dumps(out))

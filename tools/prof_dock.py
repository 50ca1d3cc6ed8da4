"""Profiling driver: dock one batch on resident inputs (warmup + measured launches).
Used under ncu (never for reported numbers)."""
import argparse
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_05069_b200 import io, model, native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ligands", type=int, default=20000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--heavy", type=int, default=0, help="homogeneous shape (heavy atoms); 0 = mixed")
ap.add_argument("--frags", type=int, default=0)
ap.add_argument("--spacing", type=float, default=0.5)
ap.add_argument("--family", default="batched", choices=["batched", "latency"])
ap.add_argument("--c2", action="store_true", help="the config-2 single ligand (~90 atoms, 20 bonds)")
a = ap.parse_args()
pocket = io.synthetic_pocket(spacing=a.spacing)
table = native.InteractionTable.default()
if a.c2:
    cands = io.generate_dataset_batch(36, 20, 64, seed=2)
    A = np.diff(cands.atom_off)
    batch = cands.subset([int(np.nonzero((A >= 86) & (A <= 94))[0][0])])
else:
    batch = (io.generate_dataset_batch(a.heavy, a.frags, a.ligands, seed=3) if a.heavy
             else io.generate_mixed_batch(a.ligands, seed=3))
fam = native.FAMILY_LATENCY if a.family == "latency" else native.FAMILY_BATCHED
ctx = native.Context(0)
dp = ctx.pocket(pocket, table)
rb = native.ResidentBatch(ctx, native.pack(batch))
for _ in range(a.reps):
    st = rb.dock(dp, model.DockConfig(), family=fam)
    print(f"align {st.align_ms:.3f} ms  optimize {st.optimize_ms:.3f} ms  total {st.total_ms:.3f} ms")

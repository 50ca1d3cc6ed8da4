"""Profiling driver: dock one mixed batch on resident inputs (warmup + measured launches).
Used under ncu (never for reported numbers)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_05069_b200 import io, model, native  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ligands", type=int, default=20000)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--heavy", type=int, default=0, help="homogeneous shape (heavy atoms); 0 = mixed")
ap.add_argument("--frags", type=int, default=0)
ap.add_argument("--spacing", type=float, default=0.5)
a = ap.parse_args()
pocket = io.synthetic_pocket(spacing=a.spacing)
table = native.InteractionTable.default()
batch = (io.generate_dataset_batch(a.heavy, a.frags, a.ligands, seed=3) if a.heavy
         else io.generate_mixed_batch(a.ligands, seed=3))
ctx = native.Context(0)
dp = ctx.pocket(pocket, table)
rb = native.ResidentBatch(ctx, native.pack(batch))
for _ in range(a.reps):
    st = rb.dock(dp, model.DockConfig())
    print(f"align {st.align_ms:.3f} ms  optimize {st.optimize_ms:.3f} ms  total {st.total_ms:.3f} ms")

"""Small latency-family calls that run the cluster-speculative kernel (k_optimize_latency_spec:
DSMEM outcome slots, TMA multicast, two thread groups per CTA) under compute-sanitizer:
single ligands, a forced multi-ligand batch, crowded ligands, early exit off, odd / even / no
fragments and a degenerate axis.

    compute-sanitizer --tool racecheck python tools/sanitize_spread.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_05069_b200 import io, model, native  # noqa: E402

os.environ["DS_LATENCY_SPEC"] = "1"
ctx = native.Context(0)
table = native.InteractionTable.default()
dp = ctx.pocket(io.synthetic_pocket(), table)
batch = io.generate_mixed_batch(6, seed=3)
crowded = io.generate_dataset_batch(36, 20, 2, seed=4)
crowded = native.LigandBatch(crowded.atom_off, (crowded.atom_xyz * np.float32(0.5)).astype(np.float32),
                             crowded.atom_type, crowded.bond_off, crowded.bonds, crowded.frag_off, crowded.frag_axis,
                             crowded.frag_mask, list(crowded.ids))
odd = io.generate_dataset_batch(12, 5, 2, seed=5)
none = io.generate_dataset_batch(8, 0, 2, seed=6)
degen = io.generate_dataset_batch(20, 6, 2, seed=21)
xyz = degen.atom_xyz.copy()
b, e = degen.frag_axis[1]
xyz[e] = xyz[b]
degen = native.LigandBatch(degen.atom_off, xyz, degen.atom_type, degen.bond_off, degen.bonds, degen.frag_off,
                           degen.frag_axis, degen.frag_mask, list(degen.ids))
for b in (batch.subset([0]), batch, crowded, odd, none, degen):
    for cfg in (model.DockConfig(), model.DockConfig(early_exit=False, restarts_n=3, rescore_top_k=2)):
        out = ctx.dock(dp, native.pack(b), cfg, 1, native.FAMILY_LATENCY, coords=True, detail=True)
        assert out.stats.lat_spread == 10
print("sanitize spread run ok")

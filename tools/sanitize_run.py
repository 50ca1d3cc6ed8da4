"""Small docking calls that launch every hot kernel once (run under compute-sanitizer):
k_align_batched, k_torsion_batched (early exit on and off), k_select_batched, k_align_latency_cl,
k_optimize_latency (shared-memory and global grid), the ds_op_* kernels and the device generator.

    compute-sanitizer --tool racecheck python tools/sanitize_run.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_05069_b200 import io, kernels, model, native  # noqa: E402

ctx = native.Context(0)
table = native.InteractionTable.default()
batch = io.generate_mixed_batch(24, seed=3)
crowded = io.generate_dataset_batch(36, 20, 4, seed=4)
crowded = native.LigandBatch(crowded.atom_off, (crowded.atom_xyz * np.float32(0.5)).astype(np.float32),
                             crowded.atom_type, crowded.bond_off, crowded.bonds, crowded.frag_off, crowded.frag_axis,
                             crowded.frag_mask, list(crowded.ids))
for spacing in (0.5, 0.375):
    dp = ctx.pocket(io.synthetic_pocket(spacing=spacing), table)
    for b in (batch, crowded):
        for cfg in (model.DockConfig(), model.DockConfig(early_exit=False, restarts_n=3, rescore_top_k=2)):
            for fam in (native.FAMILY_BATCHED, native.FAMILY_LATENCY):
                out = ctx.dock(dp, native.pack(b), cfg, 1, fam, coords=True, detail=True)
                assert (out.results["status"] >= 0).all()
    dp.close()
rb = native.ResidentBatch.generated(ctx, 5, 0, io.mixed_shapes(16, 5))
dp = ctx.pocket(io.synthetic_pocket(), table)
rb.dock(dp, model.DockConfig())
rb.download()
rb.close()
x = np.random.default_rng(1).uniform(-5, 5, size=(16, 20, 3)).astype(np.float32)
frag = model.Fragment(0, 1, frozenset(range(5, 20)))
kernels.apply_rigid(x, kernels.rot_x(30), np.zeros(3, np.float32))
kernels.apply_torsion(x, frag, 72)
kernels.bump_check(x, frag)
print("sanitize run ok")

# the batched engine's device-resident stream (ds_stream_*): producers, merged dispatches, download
from paper_2209_05069_b200 import engines  # noqa: E402
eb = io.generate_mixed_batch(600, seed=9)
rep = engines.batched_engine.run(eb, io.synthetic_pocket(), model.DockConfig(), workers=2, table=table,
                                 capacities={0: 64, 1: 48, 2: 32, 3: 16, 4: 8}, chunk=128)
assert len(rep.results) + len(rep.errors) == eb.n
print("engine stream ok")

"""BASELINE config 4: shape sweep and database-size ladder on one B200, both kernel families.

  * shape grid: heavy in {8, 12, ..., 40} x rotatable bonds in {0, 1, 2, 4, 8, 12,
    16, 20} (infeasible F >= heavy - 1 skipped) plus the paper's Small / Medium / Large classes
    (PAPER.md:452, 620-622); per cell a resident batch of --count ligands, device-timed (CUDA
    events around the kernels), batched vs latency family;
  * size ladder {10, 10^2, 10^3, 10^4, 10^5} of the mixed config-3 distribution: ligands/s of each
    family against the database size (where the batched family overtakes the latency one).

Writes CSV files + a JSON summary to --out (default profiles/r01/) and prints the summary.
"""
import argparse
import csv
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_05069_b200 import io, model, native  # noqa: E402
from bench import ClockSampler  # noqa: E402  (NVML clocks and throttle reasons while timing)

ap = argparse.ArgumentParser()
ap.add_argument("--count", type=int, default=4096, help="ligands per shape cell")
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01"))
ap.add_argument("--max-size", type=int, default=100000)
a = ap.parse_args()

pocket = io.synthetic_pocket()
table = native.InteractionTable.default()
cfg = model.DockConfig()
ctx = native.Context(0)
dp = ctx.pocket(pocket, table)
FAM = {"batched": native.FAMILY_BATCHED, "latency": native.FAMILY_LATENCY}


def device_rate(batch, reps):
    """Ligands/s of each family on a resident batch (kernels only, best of reps after warm-up)."""
    rb = native.ResidentBatch(ctx, native.pack(batch))
    out = {}
    for name, fam in FAM.items():
        rb.dock(dp, cfg, family=fam)
        ms = min(rb.dock(dp, cfg, family=fam).total_ms for _ in range(reps))
        out[name] = {"ms": ms, "ligands_per_s": batch.n / (ms / 1e3)}
    rb.close()
    return out


os.makedirs(a.out, exist_ok=True)
clk = ClockSampler(0)
clk.__enter__()
cells = [(h, f) for h in range(8, 41, 4) for f in (0, 1, 2, 4, 8, 12, 16, 20) if f < h - 1]
classes = {"Small": (20, 1), "Medium": (35, 12), "Large": (50, 20)}
rows = []
for (h, f) in cells + list(classes.values()):
    batch = io.generate_dataset_batch(h, f, a.count, seed=4)
    r = device_rate(batch, a.reps)
    A = float(np.mean(np.diff(batch.atom_off)))
    name = next((k for k, v in classes.items() if v == (h, f)), "")
    rows.append([h, f, name, round(A, 1), r["batched"]["ligands_per_s"], r["latency"]["ligands_per_s"],
                 r["batched"]["ligands_per_s"] / r["latency"]["ligands_per_s"]])
    print(f"cell heavy={h} F={f} {name} A={A:.1f}: batched {rows[-1][4]:.0f}/s latency {rows[-1][5]:.0f}/s",
          flush=True)
with open(os.path.join(a.out, "shape_sweep.csv"), "w", newline="") as fh:
    w = csv.writer(fh, lineterminator="\n")
    w.writerow(["heavy_atoms", "fragments", "paper_class", "mean_atoms", "batched_ligands_per_s",
                "latency_ligands_per_s", "batched_over_latency"])
    w.writerows(rows)

ladder = [s for s in (10, 100, 1000, 10000, 100000) if s <= a.max_size]
lrows = []
for size in ladder:
    r = device_rate(io.generate_mixed_batch(size, seed=3), a.reps)
    lrows.append([size, r["batched"]["ligands_per_s"], r["latency"]["ligands_per_s"], r["batched"]["ms"],
                  r["latency"]["ms"]])
    print(f"size {size}: batched {lrows[-1][1]:.0f}/s latency {lrows[-1][2]:.0f}/s", flush=True)
with open(os.path.join(a.out, "size_ladder.csv"), "w", newline="") as fh:
    w = csv.writer(fh, lineterminator="\n")
    w.writerow(["ligands", "batched_ligands_per_s", "latency_ligands_per_s", "batched_ms", "latency_ms"])
    w.writerows(lrows)

clk.__exit__(None, None, None)
summary = {"workload": "config4 shape sweep + size ladder, synthetic pocket, DockConfig defaults, device-timed",
           "clocks": clk.summary(), "lib_src_sha16": native.source_sha16(),
           "count_per_cell": a.count,
           "classes": {r[2]: {"batched": r[4], "latency": r[5]} for r in rows if r[2]},
           "batched_over_latency_range": [min(r[6] for r in rows), max(r[6] for r in rows)],
           "size_ladder": {str(r[0]): {"batched": r[1], "latency": r[2]} for r in lrows}}
with open(os.path.join(a.out, "shape_sweep.json"), "w") as fh:
    json.dump(summary, fh, indent=1)
print(json.dumps(summary))

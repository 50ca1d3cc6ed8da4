"""The paper's early-exit ablation (SPEC.md:515-522 cmd_ablate_early_exit) on the
device: each database docked with the bump test's early exit on and off, both kernel families,
device-timed; the selected results must be identical (only the counters may differ) and
bump_checks(on) <= bump_checks(off).  Prints one JSON line and writes profiles/r01/ablate_early_exit.json."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2209_05069_b200 import io, model, native  # noqa: E402

ctx = native.Context(0)
dp = ctx.pocket(io.synthetic_pocket(), native.InteractionTable.default())
FIELDS = ("status", "geom_score", "chem_fx", "best_restart", "best_ax", "best_ay", "n_kept", "poses_scored")
dbs = {"config3 mixed (20k)": io.generate_mixed_batch(20000, seed=3),
       "Small 20/1 (4k)": io.generate_dataset_batch(20, 1, 4096, seed=4),
       "Medium 35/12 (4k)": io.generate_dataset_batch(35, 12, 4096, seed=4),
       "Large 50/20 (4k)": io.generate_dataset_batch(50, 20, 4096, seed=4)}
out = {"workload": "early-exit ablation, synthetic pocket, DockConfig defaults, device-timed (best of 3)"}
for name, batch in dbs.items():
    rb = native.ResidentBatch(ctx, native.pack(batch))
    row = {}
    for fam_name, fam in (("batched", native.FAMILY_BATCHED), ("latency", native.FAMILY_LATENCY)):
        res = {}
        for ee in (True, False):
            cfg = model.DockConfig(early_exit=ee)
            rb.dock(dp, cfg, family=fam)
            ms = min(rb.dock(dp, cfg, family=fam).total_ms for _ in range(3))
            res[ee] = (ms, rb.download())
        same = all(np.array_equal(res[True][1][f], res[False][1][f]) for f in FIELDS)
        on, off = res[True][1], res[False][1]
        row[fam_name] = {"ms_on": res[True][0], "ms_off": res[False][0], "speedup_on": res[False][0] / res[True][0],
                         "bump_checks_on": int(on["bump_checks"].astype(np.int64).sum()),
                         "bump_checks_off": int(off["bump_checks"].astype(np.int64).sum()),
                         "bump_early_exits_on": int(on["bump_early_exits"].astype(np.int64).sum()),
                         "results_identical": bool(same)}
    rb.close()
    out[name] = row
    print(name, json.dumps(row), flush=True)
with open(os.path.join(ROOT, "profiles", "r01", "ablate_early_exit.json"), "w") as fh:
    json.dump(out, fh, indent=1)
print(json.dumps(out))

"""Throughput of the reference-facing engines on the B200 (A/B of the batched engine's knobs).

    python tools/engine_probe.py [--ligands 200000] [--objects 20000]

Prints one JSON line per configuration: batched_engine.run on a LigandBatch stream (capacities
from the device, several dispatchers per device, producer threads) and on Ligand objects."""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2209_05069_b200 import engines, io, model  # noqa: E402
from paper_2209_05069_b200.native import InteractionTable  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--ligands", type=int, default=200_000)
ap.add_argument("--objects", type=int, default=20_000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
pocket, table, cfg = io.synthetic_pocket(), InteractionTable.default(), model.DockConfig()
b = io.generate_mixed_batch(a.ligands, seed=3)
engines.batched_engine.run(b.slice(0, 20000), pocket, cfg, table=table, capacities="device")  # warm-up
for caps in ("device", None):
    for disp in (1, 2, 3):
        for workers in (1, 4):
            ts = []
            for _ in range(a.reps):
                rep = engines.batched_engine.run(b, pocket, cfg, table=table, capacities=caps, workers=workers,
                                                 dispatchers_per_device=disp)
                ts.append(rep.wall_time)
            t = min(ts)
            print(json.dumps({"stream": "LigandBatch", "ligands": b.n, "capacities": caps or "spec",
                              "capacity": rep.dispatch_log[0]["capacity"], "dispatchers": disp, "workers": workers,
                              "wall_s": t, "ligands_per_s": b.n / t, "batches": rep.counters.batches_dispatched,
                              "device_ms_sum": rep.device_ms}), flush=True)
ligs = b.slice(0, a.objects).to_ligands()
rep = engines.batched_engine.run(ligs, pocket, cfg, table=table, capacities="device", workers=4)
print(json.dumps({"stream": "Ligand objects", "ligands": len(ligs), "wall_s": rep.wall_time,
                  "ligands_per_s": len(ligs) / rep.wall_time}), flush=True)

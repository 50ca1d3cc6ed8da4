"""Timeline of one batched_engine.run (the reference-facing entry point) on the B200: phase times
of the run and every dispatched batch (detached / started / finished, size, device ms).

    python tools/engine_timeline.py [--ligands 200000] [--reps 3]"""
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
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--workers", type=int, default=4)
ap.add_argument("--dispatchers", type=int, default=2)
ap.add_argument("--merge", type=int, default=1 << 16)
ap.add_argument("--chunk", type=int, default=8192)
ap.add_argument("--log", action="store_true")
a = ap.parse_args()
pocket, table, cfg = io.synthetic_pocket(), InteractionTable.default(), model.DockConfig()
b = io.generate_mixed_batch(a.ligands, seed=3)
kw = dict(table=table, capacities="device", workers=a.workers, dispatchers_per_device=a.dispatchers,
          merge_ligands=a.merge, chunk=a.chunk)
engines.batched_engine.run(b, pocket, cfg, **kw)  # warm-up
for r in range(a.reps):
    t0 = time.perf_counter()
    rep = engines.batched_engine.run(b, pocket, cfg, **kw)
    wall = time.perf_counter() - t0
    log = rep.dispatch_log
    print(json.dumps({"rep": r, "workers": a.workers, "dispatchers": a.dispatchers, "merge": a.merge, "chunk": a.chunk,
                      "waves": os.environ.get("DS_CAPACITY_WAVES", "default"), "wall_ms": 1e3 * wall, "ligands_per_s": b.n / wall,
                      "timings_ms": {k: 1e3 * v for k, v in getattr(rep, "timings", {}).items()},
                      "batches": len(log), "device_ms_sum": rep.device_ms,
                      "first_start_ms": 1e3 * min(e["started"] for e in log),
                      "last_finish_ms": 1e3 * max(e["finished"] for e in log)}), flush=True)
for e in (log if a.log else []):
    print(json.dumps({k: (round(1e3 * v, 2) if k in ("detached", "started", "finished") else v)
                      for k, v in e.items()}))

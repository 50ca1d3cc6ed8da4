"""bench-cli: the reference's experiment harness on the B200 engines.

    python -m paper_2209_05069_b200.cli dock --ligands L.ligq --pocket P.pock [--engine batched] --out DIR
    python -m paper_2209_05069_b200.cli heatmap  [--count 2000] --out DIR
    python -m paper_2209_05069_b200.cli scaling  [--full-scale] --out DIR
    python -m paper_2209_05069_b200.cli ablate-early-exit --out DIR

CSV layouts follow SPEC.md:487, 497, 507, 517.  Rows are deterministic for fixed arguments
(timestamps go to a separate run.log).  `sequential` runs the latency engine with
one worker.
"""
from __future__ import annotations

import argparse
import csv
import os
import sys
import time
from typing import List, Optional, Sequence

from . import engines, io, model
from .native import InteractionTable

HEATMAP_HEAVY = (8, 12, 16, 20, 24, 28, 32, 36, 40)
HEATMAP_FRAGS = (0, 1, 2, 4, 8, 12, 16, 20)


def _cfg(a) -> model.DockConfig:
    return model.DockConfig(restarts_n=a.restarts, rescore_top_k=a.top_k, early_exit=(a.early_exit == "on"))


def _caps(a):
    out = {}
    for s in a.capacity_override or ():
        k, v = s.split("=")
        out[int(k)] = int(v)
    return out or None


def _run(engine: str, ligs, pocket, cfg, a, table):
    if engine == "batched":
        return engines.batched_engine.run(ligs, pocket, cfg, workers=a.workers, seed=a.seed, table=table,
                                          capacities=_caps(a))
    workers = 1 if engine == "sequential" else a.workers
    return engines.latency_engine.run(ligs, pocket, cfg, workers=workers, seed=a.seed, table=table)


def _log(out: str, msg: str):
    with open(os.path.join(out, "run.log"), "a") as fh:
        fh.write(f"{time.strftime('%Y-%m-%dT%H:%M:%S')} {msg}\n")


def cmd_dock(a) -> int:
    for p in (a.ligands, a.pocket):
        if not p or not os.path.exists(p):
            print(f"error: no such file: {p}", file=sys.stderr)
            return 2
    ligs = io.parse_ligand_file(a.ligands, skip_invalid=True)
    pocket = io.parse_pocket_file(a.pocket)
    table = InteractionTable.default()
    rep = _run(a.engine, ligs, pocket, _cfg(a), a, table)
    os.makedirs(a.out, exist_ok=True)
    with open(os.path.join(a.out, "results.csv"), "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["ligand_id", "geom_score", "chem_score", "valid"])
        for r in rep.results:
            w.writerow([r.ligand_id, r.best_pose.geometric_score, repr(r.best_pose.chemical_score), 1])
        for seq, lid, msg in rep.errors:
            w.writerow([lid, "", "", 0])
    c = rep.counters
    print(f"engine={a.engine} workers={a.workers} ligands={len(ligs)} wall_time={rep.wall_time:.4f}s "
          f"throughput={rep.throughput:.1f}/s poses_scored={c.poses_scored} bump_checks={c.bump_checks} "
          f"bump_early_exits={c.bump_early_exits} batches_dispatched={c.batches_dispatched}")
    return 0


def _cells(a):
    heavy = [int(x) for x in a.heavy.split(",")] if a.heavy else list(HEATMAP_HEAVY)
    frags = [int(x) for x in a.frags.split(",")] if a.frags else list(HEATMAP_FRAGS)
    return [(h, f) for h in heavy for f in frags if not (f > 0 and f >= h - 1)]


def cmd_heatmap(a) -> int:
    os.makedirs(a.out, exist_ok=True)
    pocket = io.synthetic_pocket()
    table = InteractionTable.default()
    cfg = _cfg(a)
    rows = []
    for (h, f) in _cells(a):
        ligs = io.generate_dataset(h, f, a.count, seed=a.seed)
        lat = _run("latency", ligs, pocket, cfg, a, table)
        bat = _run("batched", ligs, pocket, cfg, a, table)
        rows.append([h, f, lat.throughput, bat.throughput, bat.throughput / lat.throughput])
        _log(a.out, f"heatmap cell {h},{f} latency={lat.wall_time:.4f}s batched={bat.wall_time:.4f}s")
    with open(os.path.join(a.out, "heatmap.csv"), "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["heavy_atoms", "fragments", "latency_tput", "batched_tput", "speedup"])
        w.writerows(rows)
    return 0


def cmd_scaling(a) -> int:
    os.makedirs(a.out, exist_ok=True)
    pocket = io.synthetic_pocket()
    table = InteractionTable.default()
    cfg = _cfg(a)
    ladder = [10, 100, 1000, 10000, 100000] + ([1000000] if a.full_scale else [])
    if a.max_size:
        ladder = [s for s in ladder if s <= a.max_size]
    rows = []
    for size in ladder:
        for mode in ("homogeneous", "heterogeneous"):
            batch = (io.generate_dataset_batch(35, 12, size, seed=a.seed) if mode == "homogeneous"
                     else io.generate_mixed_batch(size, seed=a.seed))
            ligs = batch.to_ligands()
            for engine in ("latency", "batched"):
                rep = _run(engine, ligs, pocket, cfg, a, table)
                c = rep.counters
                fill = c.batch_fill_ratio_sum / c.batches_dispatched if c.batches_dispatched else 0.0
                rows.append([size, mode, engine, rep.throughput, c.batches_dispatched, fill])
                _log(a.out, f"scaling {size} {mode} {engine} wall={rep.wall_time:.4f}s")
    with open(os.path.join(a.out, "scaling.csv"), "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["size", "mode", "engine", "throughput", "batches_dispatched", "mean_fill_ratio"])
        w.writerows(rows)
    return 0


def cmd_ablate_early_exit(a) -> int:
    os.makedirs(a.out, exist_ok=True)
    pocket = io.synthetic_pocket()
    table = InteractionTable.default()
    rows = []
    for (h, f) in _cells(a):
        ligs = io.generate_dataset(h, f, a.count, seed=a.seed)
        res = {}
        for ee in ("on", "off"):
            cfg = model.DockConfig(restarts_n=a.restarts, rescore_top_k=a.top_k, early_exit=(ee == "on"))
            lat = _run("latency", ligs, pocket, cfg, a, table)
            bat = _run("batched", ligs, pocket, cfg, a, table)
            res[ee] = (lat, bat)
        sig = lambda rep: [(r.ligand_id, r.best_pose.geometric_score, r.best_pose.chem_fx) for r in rep.results]
        if sig(res["on"][1]) != sig(res["off"][1]) or sig(res["on"][0]) != sig(res["off"][0]):
            print(f"ScoreMismatch in cell {h},{f}", file=sys.stderr)   # SPEC.md:518 (fatal)
            return 3
        on, off = res["on"][1].counters, res["off"][1].counters
        rows.append([h, f, res["on"][1].throughput / res["on"][0].throughput,
                     res["off"][1].throughput / res["off"][0].throughput, on.bump_checks, off.bump_checks,
                     on.bump_early_exits, (on.bump_checks / off.bump_checks) if off.bump_checks else 1.0])
    with open(os.path.join(a.out, "ablate_early_exit.csv"), "w", newline="") as fh:
        w = csv.writer(fh, lineterminator="\n")
        w.writerow(["heavy_atoms", "fragments", "speedup_on", "speedup_off", "bump_checks_on", "bump_checks_off",
                    "bump_early_exits_on", "bump_checks_ratio"])
        w.writerows(rows)
    return 0


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="dockscreen")
    sub = p.add_subparsers(dest="cmd", required=True)

    def common(s):
        s.add_argument("--engine", default="batched", choices=["latency", "batched", "sequential"])
        s.add_argument("--workers", type=int, default=os.cpu_count() or 1)
        s.add_argument("--seed", type=int, default=0)
        s.add_argument("--restarts", type=int, default=8)
        s.add_argument("--top-k", type=int, default=4)
        s.add_argument("--early-exit", default="on", choices=["on", "off"])
        s.add_argument("--capacity-override", action="append")
        s.add_argument("--out", default="out")
    d = sub.add_parser("dock")
    common(d)
    d.add_argument("--ligands")
    d.add_argument("--pocket")
    for name in ("heatmap", "ablate-early-exit"):
        h = sub.add_parser(name)
        common(h)
        h.add_argument("--count", type=int, default=2000)
        h.add_argument("--heavy")
        h.add_argument("--frags")
    s = sub.add_parser("scaling")
    common(s)
    s.add_argument("--full-scale", action="store_true")
    s.add_argument("--max-size", type=int, default=0)
    return p


def console_main(argv: Optional[Sequence[str]] = None) -> int:
    """Exit status: 0 ok, 2 missing input file, 1 any error that ended a run (an invalid
    configuration, a device or library failure re-raised by an engine): never a short CSV with 0."""
    a = build_parser().parse_args(argv)
    try:
        return {"dock": cmd_dock, "heatmap": cmd_heatmap, "scaling": cmd_scaling,
                "ablate-early-exit": cmd_ablate_early_exit}[a.cmd](a)
    except (model.DockscreenError, RuntimeError, ValueError) as e:
        print(f"error: {type(e).__name__}: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(console_main())

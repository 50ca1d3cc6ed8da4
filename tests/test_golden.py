"""Golden fixtures (tests/golden/*.json, written by tests/golden/make_golden.py from the pinned
oracle) replayed on the oracle (CPU) and on the device (GPU), bit for bit."""
import glob
import json
import os

import numpy as np
import pytest

import oracle
from paper_2209_05069_b200 import io, model, native
from paper_2209_05069_b200.native import InteractionTable

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FILES = sorted(glob.glob(os.path.join(HERE, "*.json")))


def _load(path):
    with open(path) as fh:
        doc = json.load(fh)
    c = doc["case"]
    batch = (io.generate_dataset_batch(c["heavy"], c["frags"], c["count"], seed=c["seed"]) if c["kind"] == "shape"
             else io.generate_mixed_batch(c["count"], seed=c["seed"]))
    return doc, c, batch


def _check(doc, batch, res, restarts, rtors, coords):
    for i, g in enumerate(doc["ligands"]):
        assert batch.ids[i] == g["id"]
        r = res[i]
        assert int(r["status"]) == g["status"]
        if g["status"] != 0:
            continue
        assert (int(r["geom_score"]), int(r["chem_fx"]), int(r["best_restart"]), int(r["best_ax"]), int(r["best_ay"]),
                int(r["n_kept"]), int(r["poses_scored"]), int(r["bump_early_exits"])) == \
            (g["geom"], g["chem_fx"], g["best_restart"], g["ax"], g["ay"], g["n_kept"], g["poses_scored"],
             g["bump_early_exits"])
        got = [[int(x["align_score"]), int(x["final_geom"]), int(x["ax"]), int(x["ay"]), int(x["valid"]),
                int(x["kept"])] for x in restarts[i]]
        assert got == g["restarts"]
        f0, f1 = batch.frag_off[i], batch.frag_off[i + 1]
        assert [[int(v) for v in rtors[f]] for f in range(f0, f1)] == g["torsion"]
        a0, a1 = batch.atom_off[i], batch.atom_off[i + 1]
        assert coords[a0:a1].tobytes().hex() == g["best_coords_hex"]


def test_golden_files_exist():
    assert len(FILES) >= 4


@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
def test_golden_oracle(path):
    doc, c, batch = _load(path)
    out = oracle.dock_batch(batch, io.synthetic_pocket(), InteractionTable.default(), model.DockConfig(),
                            seed=c["dock_seed"], threads=4)
    _check(doc, batch, out.results, out.restarts, out.restart_torsion, out.best_coords)


@pytest.mark.gpu
@pytest.mark.parametrize("family", [native.FAMILY_BATCHED, native.FAMILY_LATENCY])
@pytest.mark.parametrize("path", FILES, ids=[os.path.basename(f) for f in FILES])
def test_golden_device(gpu_ctx, path, family):
    doc, c, batch = _load(path)
    dp = gpu_ctx.pocket(io.synthetic_pocket(), InteractionTable.default())
    out = gpu_ctx.dock(dp, native.pack(batch), model.DockConfig(), c["dock_seed"], family, coords=True, detail=True)
    _check(doc, batch, out.results, out.restarts, out.restart_torsion, out.best_coords)

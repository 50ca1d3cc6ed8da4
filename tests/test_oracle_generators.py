"""The oracle-side input makers (oracle/gen_oracle.c) produce the same inputs as the product's
generators (csrc/ds_host.cpp), array for array — so bench.py's reference arm can build its workload
without loading libdockscreen.so and still dock exactly the ligands the GPU arm docks."""
import numpy as np

import oracle
from paper_2209_05069_b200 import io
from paper_2209_05069_b200.native import InteractionTable


def test_mixed_batch_identical():
    for first in (0, 123_457):
        o = oracle.generate_mixed_batch(500, seed=3, first_index=first)
        p = io.generate_mixed_batch(500, seed=3, first_index=first)
        for f in ("atom_off", "atom_xyz", "atom_type", "frag_off", "frag_axis", "frag_mask"):
            assert np.array_equal(getattr(o, f), getattr(p, f)), f
        assert list(o.ids) == list(p.ids)
        assert o.id_bytes()[0] == p.id_bytes()[0]
        assert np.array_equal(o.id_bytes()[1], p.id_bytes()[1])


def test_fixed_shapes_identical():
    shapes = np.array([[12, 5], [36, 20], [1, 0], [70, 60], [80, 0]], np.int32)
    o = oracle.generate_batch(shapes, seed=2, first_index=7)
    p = io.generate_batch(shapes, seed=2, first_index=7)
    for f in ("atom_off", "atom_xyz", "atom_type", "frag_off", "frag_axis", "frag_mask"):
        assert np.array_equal(getattr(o, f), getattr(p, f)), f


def test_pocket_and_table_identical():
    for spacing in (0.5, 0.375):
        o = oracle.synthetic_pocket(spacing=spacing)
        p = io.synthetic_pocket(spacing=spacing)
        assert o.grid_origin == p.grid_origin and o.grid_dims == p.grid_dims and o.grid_spacing == p.grid_spacing
        assert np.array_equal(o.grid_values, p.grid_values)
        assert o.pocket_atoms == p.pocket_atoms
    assert np.array_equal(oracle.default_table().table, InteractionTable.default().table)
    assert oracle.default_table().bins == InteractionTable.default().bins


def test_oracle_docks_oracle_inputs_like_product_inputs():
    """dock_batch on the oracle-made inputs == dock_batch on the product-made inputs."""
    from paper_2209_05069_b200 import model
    cfg = model.DockConfig()
    a = oracle.dock_batch(oracle.generate_mixed_batch(12, seed=3), oracle.synthetic_pocket(), oracle.default_table(),
                          cfg, seed=0, threads=4)
    b = oracle.dock_batch(io.generate_mixed_batch(12, seed=3), io.synthetic_pocket(), InteractionTable.default(), cfg,
                          seed=0, threads=4)
    assert np.array_equal(a.results, b.results)
    assert np.array_equal(a.best_coords, b.best_coords)


def test_latency_shaped_oracle_equals_batched():
    """The oracle's latency-engine shape (restarts on an inner pool) == the sequential per-ligand
    oracle, including a DegenerateAxis ligand (counters and torsion records up to the stop)."""
    from paper_2209_05069_b200 import model
    b = oracle.generate_mixed_batch(10, seed=5)
    xyz = b.atom_xyz.copy()
    i, f0 = 3, int(b.frag_off[3])
    if b.frag_off[4] > f0:
        a0 = int(b.atom_off[i])
        bb, e = b.frag_axis[f0]
        xyz[a0 + e] = xyz[a0 + bb]
    b2 = oracle.OracleBatch(b.atom_off, xyz, b.atom_type, b.frag_off, b.frag_axis, b.frag_mask, b.ids)
    pk, tb = oracle.synthetic_pocket(), oracle.default_table()
    for cfg in (model.DockConfig(), model.DockConfig(early_exit=False, restarts_n=5, rescore_top_k=2)):
        a = oracle.dock_batch(b2, pk, tb, cfg, seed=1, threads=4)
        c = oracle.dock_batch(b2, pk, tb, cfg, seed=1, threads=8, latency=True)
        assert np.array_equal(a.results, c.results)
        assert np.array_equal(a.restarts, c.restarts)
        assert np.array_equal(a.restart_torsion, c.restart_torsion)
        assert np.array_equal(a.best_coords, c.best_coords)


def test_bench_reference_arm_contract():
    """bench.py --impl reference (the driver's reference arm) on a tiny sample: one JSON line with the
    contract's keys, the CPU oracle as a port, e2e == value with no copies, and the product library
    never mapped into that process."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--cpu-sample", "16"], capture_output=True, text=True, timeout=600,
                         env=dict(os.environ, OMP_NUM_THREADS="4"))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "cpu_baseline", "e2e", "config"):
        assert k in line, k
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "port" and line["value"] > 0
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]

"""io: generators, build_pocket and the text formats."""
import numpy as np
import pytest

from paper_2209_05069_b200 import io, model, native
from paper_2209_05069_b200.bucketizer import classify


def test_generate_dataset_examples():
    ligs = io.generate_dataset(20, 1, 500, seed=4)                      # SPEC.md:449 (scaled count)
    assert len(ligs) == 500
    for l in ligs:
        model.validate_ligand(l)
        assert l.heavy_atom_count == 20 and len(l.fragments) == 1
        assert 20 + 20 <= len(l.atoms) <= min(160, 60)
    assert len(io.generate_dataset(50, 20, 10, seed=4)) == 10
    a = io.generate_dataset_batch(12, 5, 50, seed=9)                    # SPEC.md:451 determinism
    b = io.generate_dataset_batch(12, 5, 50, seed=9)
    for f in ("atom_xyz", "atom_type", "frag_mask", "bonds"):
        assert np.array_equal(getattr(a, f), getattr(b, f))
    with pytest.raises(model.InfeasibleShape):
        io.generate_dataset(5, 4, 1, seed=1)


def test_generated_geometry():
    b = io.generate_dataset_batch(30, 8, 20, seed=3)
    for l in b.to_ligands():
        xyz = l.coords().astype(np.float64)
        for (i, j) in l.bonds:
            d = np.linalg.norm(xyz[i] - xyz[j])
            assert abs(d - (1.5 if l.atoms[j].is_heavy else 1.0)) < 1e-4   # 1.5 Å chain steps, 1.0 Å X-H


def test_shard_generation_matches_whole():
    """Any index range generates identically on its own (multi-GPU shards, config 5)."""
    whole = io.generate_mixed_batch(300, seed=5)
    part = io.generate_mixed_batch(100, seed=5, first_index=150)
    for k in range(100):
        a0, a1 = whole.atom_off[150 + k], whole.atom_off[151 + k]
        b0, b1 = part.atom_off[k], part.atom_off[k + 1]
        assert np.array_equal(whole.atom_xyz[a0:a1], part.atom_xyz[b0:b1])
        assert whole.ids[150 + k] == part.ids[k]


def test_bucket_diversity():
    """heavy atoms near a range boundary land in >= 2 atom ranges."""
    ligs = io.generate_dataset(15, 1, 200, seed=6)       # 15 heavy + 15..30 H -> 30..45 atoms
    assert len({classify(l).atom_range_index for l in ligs}) >= 2


def test_build_pocket_known_answers():
    p = io.build_pocket([model.Atom.of(0.0, 0.0, 0.0, 3)], spacing=1.0, padding=4.0)
    nx, ny, nz = p.grid_dims
    vals = p.grid_values.reshape(nz, ny, nx)
    o = np.array(p.grid_origin)
    # node at exactly 4 Å from the atom -> 10; node at 0 Å -> -10
    i0 = np.round(-o).astype(int)
    assert vals[i0[2], i0[1], i0[0]] == -10
    assert vals[i0[2], i0[1], i0[0] + 4] == 10
    with pytest.raises(model.EmptyPocket):
        io.build_pocket([], 1.0, 4.0)


def test_build_pocket_brute_force():
    """every node matches an independent per-node nearest-atom oracle."""
    atoms = io.pocket_atoms(30, seed=2, rmin=3.0, rmax=5.0)
    p = io.build_pocket(atoms, spacing=0.8, padding=2.0)
    nx, ny, nz = p.grid_dims
    xyz = np.array([a.position for a in atoms], np.float64)
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).astype(np.float64)
    nodes = np.array(p.grid_origin, np.float64) + g * np.float64(np.float32(0.8))
    d = np.sqrt(((nodes[..., None, :] - xyz) ** 2).sum(-1)).min(-1)
    gfun = np.where(d <= 3, -1 + 2 * d / 3, np.where(d <= 5, 1.0, np.where(d <= 8, 1 - 2 * (d - 5) / 3, -1.0)))
    want = np.rint(10 * gfun).astype(np.int32)            # x-fastest layout
    got = p.grid_values.reshape(nz, ny, nx).transpose(2, 1, 0)
    # values exactly at a .5 rounding boundary may differ by float noise; require >99.9% equal, all within 1
    assert np.mean(got == want) > 0.999 and np.abs(got - want).max() <= 1


def test_synthetic_pocket_shape():
    p = io.synthetic_pocket()
    assert len(p.pocket_atoms) == 200
    assert all(abs(d - 57) <= 3 for d in p.grid_dims)
    assert p.grid_values.min() >= -10 and p.grid_values.max() <= 10


def test_ligand_file_roundtrip(tmp_path):
    assert io.parse_ligand_file(str(_write(tmp_path / "e.ligq", ""))) == []
    ligs = io.generate_dataset(6, 2, 5, seed=8)
    f1 = tmp_path / "a.ligq"
    io.write_ligand_file(str(f1), ligs)
    back = io.parse_ligand_file(str(f1))
    assert [l.id for l in back] == [l.id for l in ligs]
    for a, b in zip(ligs, back):
        assert np.array_equal(a.coords(), b.coords()) and a.bonds == b.bonds and a.fragments == b.fragments
    f2 = tmp_path / "b.ligq"
    io.write_ligand_file(str(f2), back)
    assert f1.read_bytes() == f2.read_bytes()
    bad = tmp_path / "bad.ligq"
    _write(bad, "MOL x\nATOM 0 1 0 0 0 heavy\nATOM 1 1 1.5 0 0 heavy\nATOM 2 1 3 0 0 heavy\n"
                "BOND 0 1\nBOND 1 2\nFRAG 0 1 1 2\nEND\n")
    with pytest.raises(model.ValidationError):
        io.parse_ligand_file(str(bad))
    assert io.parse_ligand_file(str(bad), skip_invalid=True) == []


def test_pocket_file_roundtrip(tmp_path):
    p = io.build_pocket(io.pocket_atoms(20, seed=3), spacing=1.0, padding=2.0)
    f = tmp_path / "p.pock"
    io.write_pocket_file(str(f), p)
    q = io.parse_pocket_file(str(f))
    assert q.grid_dims == p.grid_dims and q.grid_origin == p.grid_origin and q.grid_spacing == p.grid_spacing
    assert np.array_equal(q.grid_values, p.grid_values)
    assert [a.position for a in q.pocket_atoms] == [a.position for a in p.pocket_atoms]


def _write(path, text):
    path.write_text(text)
    return path


def _same_batch(a, b):
    for f in ("atom_off", "atom_xyz", "atom_type", "bond_off", "bonds", "frag_off", "frag_axis", "frag_mask"):
        assert np.array_equal(getattr(a, f), getattr(b, f)), f
    assert list(a.ids) == list(b.ids)


def test_native_ligq_parser_matches_reference_parser(tmp_path):
    """ds_ligq_parse (SURVEY §8(f) host ingest) == io.parse_ligand_file on a mixed database."""
    ligs = io.generate_mixed_batch(300, seed=12).to_ligands()
    f = tmp_path / "db.ligq"
    io.write_ligand_file(str(f), ligs)
    fast = io.parse_ligand_batch(str(f))
    ref = native.LigandBatch.from_ligands(io.parse_ligand_file(str(f)))
    _same_batch(fast, ref)
    assert fast.to_ligands() == io.parse_ligand_file(str(f))
    empty = io.parse_ligand_batch(str(_write(tmp_path / "e.ligq", "\n\n")))
    assert empty.n == 0


VALID = ("MOL m{}\nATOM 0 1 0 0 0 heavy\nATOM 1 1 1.5 0 0 heavy\nATOM 2 0 2.5 0 0 H\n"
         "BOND 0 1\nBOND 1 2\nFRAG 0 1 2\nEND\n")


@pytest.mark.parametrize("text", [
    "ATOM 0 1 0 0 0 heavy\n",                                   # record outside MOL
    VALID.format(1) + "BOND 0 1\n",                             # record outside MOL after END
    "MOL a\nATOM 0 1 0 0 0\nEND\n",                             # missing field
    "MOL a\nATOM 1 1 0 0 0 heavy\nEND\n",                       # atom index out of order
    "MOL a\nATOM 0 1 x 0 0 heavy\nEND\n",                       # bad float
    "MOL a\nATOM 0 1 0 0 0 heavy\nFOO 1\nEND\n",                # unknown record
    VALID.format(1) + "MOL b\nATOM 0 1 0 0 0 heavy\n",          # missing final END
])
def test_native_ligq_parse_errors(tmp_path, text):
    f = _write(tmp_path / "bad.ligq", text)
    with pytest.raises(model.ParseError):
        io.parse_ligand_file(str(f))
    with pytest.raises(model.ParseError):
        io.parse_ligand_batch(str(f))


@pytest.mark.parametrize("frag", ["FRAG 0 1 1 2", "FRAG 0 2 2", "FRAG 0 1 7", "FRAG 0 1", "FRAG 0 2 1"])
def test_native_ligq_validation_errors(tmp_path, frag):
    """invalid fragments: raised (ValidationError) or skipped exactly like the reference parser;
    a molecule cut short by the next MOL is dropped by both."""
    text = ("MOL x\nATOM 0 1 0 0 0 heavy\nATOM 1 1 1.5 0 0 heavy\nATOM 2 1 3 0 0 heavy\nBOND 0 1\nBOND 1 2\n"
            + frag + "\nEND\n" + "MOL cut\nATOM 0 1 0 0 0 heavy\n" + VALID.format(2))
    f = _write(tmp_path / "v.ligq", text)
    with pytest.raises(model.ValidationError):
        io.parse_ligand_file(str(f))
    with pytest.raises(model.ValidationError):
        io.parse_ligand_batch(str(f))
    ref = io.parse_ligand_file(str(f), skip_invalid=True)
    fast = io.parse_ligand_batch(str(f), skip_invalid=True)
    assert [l.id for l in ref] == list(fast.ids) == ["m2"]
    _same_batch(fast, native.LigandBatch.from_ligands(ref))


def test_generated_ids_lazy_sequence():
    """Generated ligands carry a lazy id sequence (native.GeneratedIds): the same strings as
    ds_generated_id, slices stay lazy, and the packed id bytes come from one native call."""
    from paper_2209_05069_b200.native import GeneratedIds
    ids = GeneratedIds(-7, 99, 50)
    want = [io.generated_id(-7, 99 + i) for i in range(50)]
    assert list(ids) == want and len(ids) == 50 and ids[-1] == want[-1]
    assert isinstance(ids[10:20], GeneratedIds) and list(ids[10:20]) == want[10:20]
    assert ids[::7] == want[::7]
    blob, off = ids.id_blob()
    assert blob == b"".join(s.encode() for s in want)
    assert off.tolist() == np.cumsum([0] + [len(s) for s in want]).tolist()
    b = io.generate_mixed_batch(20, seed=3, first_index=5)
    assert isinstance(b.ids, GeneratedIds) and b.ids[0] == "lig_3_5"
    assert list(b.slice(4, 9).ids) == [f"lig_3_{5 + k}" for k in range(4, 9)]
    with pytest.raises(IndexError):
        ids[50]

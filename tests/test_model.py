"""core-model invariants and validate_ligand."""
import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from paper_2209_05069_b200 import io, model
from paper_2209_05069_b200.native import LigandBatch, pack


def chain(n, frags=(), types=None):
    types = types or [1] * n
    atoms = tuple(model.Atom.of(1.5 * i, 0.0, 0.0, types[i]) for i in range(n))
    bonds = tuple((i, i + 1) for i in range(n - 1))
    return model.Ligand("c", atoms, bonds, tuple(frags))


def test_validate_examples():
    with pytest.raises(model.TooManyAtoms):
        model.validate_ligand(chain(161))
    assert model.validate_ligand(chain(1)) is not None
    with pytest.raises(model.MalformedFragment):
        model.validate_ligand(chain(5, [model.Fragment(1, 2, frozenset({1, 3, 4}))]))


def test_validate_ok_fragment_both_sides():
    model.validate_ligand(chain(6, [model.Fragment(2, 3, frozenset({4, 5}))]))
    model.validate_ligand(chain(6, [model.Fragment(2, 3, frozenset({0, 1}))]))
    with pytest.raises(model.MalformedFragment):
        model.validate_ligand(chain(6, [model.Fragment(2, 3, frozenset({4}))]))      # not a whole side
    with pytest.raises(model.IndexOutOfRange):
        model.validate_ligand(chain(6, [model.Fragment(2, 9, frozenset({4, 5}))]))
    with pytest.raises(model.MalformedFragment):
        model.validate_ligand(chain(6, [model.Fragment(2, 4, frozenset({5}))]))      # axis not a bond


def test_config_invariants():
    model.DockConfig()
    with pytest.raises(ValueError):
        model.DockConfig(alignment_step_deg=7)
    with pytest.raises(ValueError):
        model.DockConfig(restarts_n=2, rescore_top_k=3)


def _reference_checker(n, bonds, frag):
    """Independent checker: BFS components after removing the axis bond."""
    b, e, mask = frag
    if not (0 <= b < n and 0 <= e < n) or any(not 0 <= m < n for m in mask):
        return "range"
    adj = {i: set() for i in range(n)}
    for x, y in bonds:
        if {x, y} != {b, e}:
            adj[x].add(y)
            adj[y].add(x)
    if b == e or b in mask or e in mask or not mask or len(mask) >= n or (b, e) not in bonds and (e, b) not in bonds:
        return "malformed"

    def comp(s):
        seen, st_ = {s}, [s]
        while st_:
            v = st_.pop()
            for w in adj[v]:
                if w not in seen:
                    seen.add(w)
                    st_.append(w)
        return seen
    cb, ce = comp(b), comp(e)
    if cb & ce or len(cb | ce) != n:
        return "malformed"
    if set(mask) not in (cb - {b, e}, ce - {b, e}):
        return "malformed"
    return "ok"


@settings(max_examples=200, deadline=None)
@given(st.integers(2, 12), st.data())
def test_validate_matches_reference_checker(n, data):
    """Random tree topologies + random fragments: accept/reject matches a reference checker."""
    parents = [data.draw(st.integers(0, i - 1)) for i in range(1, n)]
    bonds = tuple((parents[i - 1], i) for i in range(1, n))
    b = data.draw(st.integers(0, n - 1))
    e = data.draw(st.integers(0, n - 1))
    mask = frozenset(data.draw(st.sets(st.integers(0, n - 1), max_size=n)))
    lig = model.Ligand("h", tuple(model.Atom.of(i, 0, 0, 1) for i in range(n)), bonds,
                       (model.Fragment(b, e, mask),))
    want = _reference_checker(n, bonds, (b, e, mask))
    try:
        model.validate_ligand(lig)
        got = "ok"
    except model.IndexOutOfRange:
        got = "range"
    except model.MalformedFragment:
        got = "malformed"
    assert got == want


def test_generated_ligands_validate_and_pack_roundtrip():
    b = io.generate_mixed_batch(200, seed=31)
    for l in b.to_ligands():
        model.validate_ligand(l)
    b2 = LigandBatch.from_ligands(b.to_ligands())
    for f in ("atom_off", "atom_xyz", "atom_type", "frag_off", "frag_axis", "frag_mask", "bonds"):
        assert np.array_equal(getattr(b, f), getattr(b2, f)), f
    p = pack(b)
    A = np.diff(b.atom_off)
    for i in (0, 7, 199):
        a0, a1 = b.atom_off[i], b.atom_off[i + 1]
        c0 = (b.atom_xyz[a0:a1].astype(np.float64).sum(0) / A[i]).astype(np.float32)
        assert np.allclose(p.atom_xyzt[a0:a1, :3], b.atom_xyz[a0:a1] - c0, atol=1e-5)
        assert np.array_equal(p.atom_xyzt[a0:a1, 3], b.atom_type[a0:a1].astype(np.float32))


def test_pack_rejects_invalid():
    b = io.generate_dataset_batch(8, 2, 3, seed=1)
    b.frag_axis[1, 0] = b.frag_axis[1, 1]
    with pytest.raises(model.MalformedFragment):
        pack(b)

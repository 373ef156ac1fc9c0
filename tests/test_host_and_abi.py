"""CPU-side checks: host constant preparation, the C ABI surface, loud failure without a GPU."""

import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2411_13507_b200 import _native as nat
from paper_2411_13507_b200 import configs
from paper_2411_13507_b200.bezier import BezierSpec, boundary_matrix
from paper_2411_13507_b200.geometry import Box, Polytope, recover_box
from tests.helpers import inputs_from_golden

ROOT = Path(__file__).resolve().parents[1]


def test_host_constants_match_reference_goldens(golden):
    """F, G, D and inflated obstacles from the host mirror equal the live reference's."""
    g = golden("demo200")
    w = configs.demo(200)
    assert w.oracle.F.tobytes() == g["F"].tobytes()
    assert w.oracle.G.tobytes() == g["G"].tobytes()
    assert boundary_matrix(w.spec).tobytes() == g["D"].tobytes()
    A = np.vstack([o.A for o in w.obstacles])
    b = np.concatenate([o.b for o in w.obstacles])
    assert A.tobytes() == g["obs_A"].tobytes() and b.tobytes() == g["obs_b"].tobytes()
    assert w.oracle.tube.error.lo.tobytes() == g["tube_lo"].tobytes()


def test_cfg2_and_hop_constants(golden):
    g = golden("cfg2_rf2000")
    w = configs.random_field(1, 20, 2000)
    assert w.oracle.F.tobytes() == g["F"].tobytes() and w.oracle.G.tobytes() == g["G"].tobytes()
    assert np.vstack([o.A for o in w.obstacles]).tobytes() == g["obs_A"].tobytes()
    assert np.concatenate([o.b for o in w.obstacles]).tobytes() == g["obs_b"].tobytes()
    h = golden("hop1500")
    wh = configs.hopping_deg5(graph_n=1500, n_obstacles=12, clear_endpoints=False)
    assert wh.oracle.F.tobytes() == h["F"].tobytes() and wh.oracle.G.tobytes() == h["G"].tobytes()
    assert np.vstack([o.A for o in wh.obstacles]).tobytes() == h["obs_A"].tobytes()
    assert np.concatenate([o.b for o in wh.obstacles]).tobytes() == h["obs_b"].tobytes()


def test_boundary_matrix_residue():
    D = boundary_matrix(BezierSpec(2, 2, 1.0))
    # LAPACK residue the device must never recompute in closed form
    assert D[0, 1] != 0.0 and abs(D[0, 1]) < 1e-15


def test_recover_box():
    P = Box(np.array([0.0, 1.0]), np.array([2.0, 3.0])).to_polytope()
    bx = recover_box(P.A, P.b)
    assert np.array_equal(bx.lo, [0.0, 1.0]) and np.array_equal(bx.hi, [2.0, 3.0])
    tri = Polytope(np.array([[1.0, 1.0], [-1.0, 0.0], [0.0, -1.0]]), np.array([1.0, 0.0, 0.0]))
    assert recover_box(tri.A, tri.b) is None


def test_obstacle_arrays_match_scalar_box_recovery():
    """The vectorised obstacle preparation equals Polytope.normalized + as_box per obstacle."""
    from paper_2411_13507_b200 import graph as G

    rng = np.random.default_rng(3)
    obs = list(configs.hopping_deg5(graph_n=50).obstacles)
    obs.append(Polytope(np.array([[0.6, 0.8], [-0.8, 0.6], [-0.6, -0.8], [0.8, -0.6]]), np.ones(4)))  # rotated
    obs.append(Polytope(np.array([[0.0, 2.0], [-3.0, 0.0], [0.0, -1.0], [1.0, 0.0]]), np.array([2.0, 3.0, 1.0, 4.0])))
    obs.append(Polytope(np.array([[1.0, 1.0], [-1.0, 0.0], [0.0, -1.0]]), np.array([1.0, 0.0, 0.0])))  # triangle
    obs.append(Polytope(np.array([[1.0, 1e-13], [0.0, 1.0], [-1.0, 0.0], [0.0, -1.0]]), rng.uniform(1, 2, 4)))
    offs, A, b, is_box, lo, hi = G._obstacle_arrays(obs, 2)
    for o, ob in enumerate(obs):
        nrm = np.linalg.norm(ob.A, axis=1)
        An, bn = ob.A / nrm[:, None], ob.b / nrm
        assert A[offs[o]:offs[o + 1]].tobytes() == An.tobytes() and b[offs[o]:offs[o + 1]].tobytes() == bn.tobytes()
        bx = recover_box(An, bn)
        assert bool(is_box[o]) == (bx is not None)
        if bx is not None:
            assert lo[o].tobytes() == bx.lo.tobytes() and hi[o].tobytes() == bx.hi.tobytes()


def _header_symbols():
    text = (ROOT / "include" / "bzg.h").read_text()
    return sorted(set(re.findall(r"\b(bzg_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    lib = nat.load()
    syms = _header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(nat.EXPORTS)
    assert lib.bzg_abi_version() == 1


def test_context_fails_loudly_without_device():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(nat.BzgError) as ei:
        nat.Context(0)
    assert ei.value.code == nat.BZG_ENODEV


def test_pcg_words_roundtrip():
    from paper_2411_13507_b200.graph import _pcg_words

    hi, lo, ihi, ilo = _pcg_words(7)
    st = np.random.default_rng(7).bit_generator.state["state"]
    assert (hi << 64 | lo) == st["state"] and (ihi << 64 | ilo) == st["inc"]

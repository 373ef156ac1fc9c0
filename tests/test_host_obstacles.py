"""Host obstacle preparation: the per-obstacle cached path (graph._obstacle_arrays_rows, used by
cut_graph and the Replanner) is bitwise the vectorised restatement of Polytope.normalized +
as_box (graph._obstacle_arrays_uncached; reference geometry.py:135-185) -- boxes, rotated and
nearly-axis-aligned boxes, degenerate boxes, general polytopes, m = 1..3, and translated copies
sharing one frozen A (the replanning case the A-constant cache serves)."""

import numpy as np
import pytest

from paper_2411_13507_b200 import graph as G
from paper_2411_13507_b200.geometry import Box, Polytope


def _random_obstacles(rng, m, n):
    out = []
    for k in range(n):
        kind = k % 6
        c = rng.uniform(-5, 5, m)
        if kind == 0:  # axis-aligned box
            h = rng.uniform(0.1, 1.0, m)
            out.append(Box(c - h, c + h).to_polytope())
        elif kind == 1:  # box rows scaled (normalisation matters)
            h = rng.uniform(0.1, 1.0, m)
            P = Box(c - h, c + h).to_polytope()
            s = rng.uniform(0.5, 3.0, 2 * m)
            out.append(Polytope(P.A * s[:, None], P.b * s))
        elif kind == 2:  # nearly axis-aligned (inside / outside the 1e-12 tolerance)
            h = rng.uniform(0.1, 1.0, m)
            P = Box(c - h, c + h).to_polytope()
            A = P.A.copy()
            A[0, (0 + 1) % m] += (5e-13 if k % 12 == 2 else 5e-11) if m > 1 else 0.0
            out.append(Polytope(A, P.b))
        elif kind == 3:  # degenerate: lo > hi on one axis
            h = rng.uniform(0.1, 1.0, m)
            P = Box(c - h, c + h).to_polytope()
            b = P.b.copy()
            b[0] = -b[m] - 1.0
            out.append(Polytope(P.A, b))
        elif kind == 4:  # rotated square / general 2m-row polytope
            A = rng.normal(size=(2 * m, m))
            out.append(Polytope(A, np.abs(rng.normal(size=2 * m)) + 0.5))
        else:  # general, other row count
            r = 2 * m + 1 + k % 3
            A = rng.normal(size=(r, m))
            out.append(Polytope(A, np.abs(rng.normal(size=r)) + 0.5))
    return out


@pytest.mark.parametrize("m", [1, 2, 3])
def test_rows_path_is_bitwise_the_vectorised_path(m):
    rng = np.random.default_rng(m)
    obs = _random_obstacles(rng, m, 60)
    for rep in range(3):  # cold, then A-constant and per-obstacle cache hits, then translated copies
        got = G._obstacle_arrays_rows(obs, m)
        want = G._obstacle_arrays_uncached(obs, m)
        for x, y in zip(got, want):
            assert x.dtype == y.dtype and x.shape == y.shape and x.tobytes() == y.tobytes()
        obs = [Polytope(ob.A, ob.b + ob.A @ rng.normal(0, 0.1, m)) for ob in obs]
    assert G._obstacle_arrays_rows([], m)[0].tolist() == [0]

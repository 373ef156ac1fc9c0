"""Seeded synthetic workloads for the graph-construction stage (BASELINE.json configs).

Recipes follow SURVEY.md §8(d).  Scenes are built from the same primitives
as the reference generators (reference scenario.py:305-392 `_box_obstacle`,
`_standard_sets`, `demo_scenario`, `random_field_scenario`; sim.py:36-70
`design_tube`; sim.py:214-217 `_inflated`) so the numbers are identical to
what the reference pipeline feeds `build_graph`/`cut_graph`/`find_path`,
without needing the reference package at run time.

Each builder returns a ``Workload``: everything the hot path consumes.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from .bezier import BezierSpec
from .geometry import Box, Polytope, inflate
from .reachability import ReachOracle, TrackingTube, build_oracle


@dataclass
class Workload:
    name: str
    spec: BezierSpec
    oracle: ReachOracle
    sample_bounds: Box
    N: int
    seed: int
    include: np.ndarray | None
    obstacles: list  # tube-inflated keep-out polytopes, list order = cut order
    start: np.ndarray
    goal: np.ndarray
    goals: np.ndarray | None = None  # cfg4 replanning goals
    extra: dict = field(default_factory=dict)

    @property
    def num_vertices(self) -> int:
        return self.N + (0 if self.include is None else len(self.include))


def design_tube(spec, gains, w_max, headroom=1.2, state_slack=0.02, input_slack=0.25) -> TrackingTube:
    """Lyapunov-box tracking tube (same construction as reference sim.py:36-70)."""
    import scipy.linalg

    g = spec.gamma
    A = np.zeros((g, g))
    A[: g - 1, 1:] = np.eye(g - 1)
    A[-1, :] = -np.asarray(gains, dtype=np.float64)
    B = np.zeros(g)
    B[-1] = 1.0
    P = scipy.linalg.solve_continuous_lyapunov(A.T, -np.eye(g))
    radius = 2.0 * np.linalg.norm(P @ B) * w_max
    level = float(np.linalg.eigvalsh(P).max()) * radius**2
    Pinv = np.linalg.inv(P)
    axis_box = headroom * np.sqrt(level * np.diag(Pinv))
    e = np.concatenate([np.full(spec.m, axis_box[k]) for k in range(g)])
    e = e + state_slack
    fb = float(np.dot(np.abs(np.asarray(gains)), axis_box))
    margin = np.full(spec.m, fb + input_slack)
    return TrackingTube(Box(-e, e), Box(-margin, margin))


def box_obstacle(cx, cy, wx, wy) -> Polytope:
    return Box(np.array([cx - wx / 2, cy - wy / 2]), np.array([cx + wx / 2, cy + wy / 2])).to_polytope()


def standard_sets(v_max=1.5, u_max=6.0, side=5.0, v_sample=0.6):
    xd = Box(np.array([0.0, 0.0, -v_max, -v_max]), np.array([side, side, v_max, v_max])).to_polytope()
    u = Box(np.array([-u_max, -u_max]), np.array([u_max, u_max]))
    sample = Box(np.array([0.0, 0.0, -v_sample, -v_sample]), np.array([side, side, v_sample, v_sample]))
    return xd, u, sample


def _inflated(obstacles, tube, m):
    pos = tube.position_box(m)
    return [inflate(o, pos) for o in obstacles]


def demo(graph_n: int = 200, seed: int = 7) -> Workload:
    """cfg1 keep-out variant: the reference demo scene (3 boxes), 200 samples + start/goal."""
    spec = BezierSpec(m=2, gamma=2, T=1.0)
    xd, u, sample = standard_sets()
    tube = design_tube(spec, (6.0, 5.0), 0.02)
    obs = [box_obstacle(2.5, 2.5, 1.0, 1.0), box_obstacle(1.2, 3.8, 0.8, 0.8), box_obstacle(3.8, 1.2, 0.8, 0.8)]
    start = np.array([0.5, 0.5, 0.0, 0.0])
    goal = np.array([4.5, 4.5, 0.0, 0.0])
    oracle = build_oracle(spec, xd, u, tube)
    return Workload("cfg1-demo", spec, oracle, sample, graph_n, seed, np.array([start, goal]),
                    _inflated(obs, tube, spec.m), start, goal)


def random_field(seed: int = 1, n_obstacles: int = 20, graph_n: int = 2000, side: float = 5.0,
                 obstacle_size=(0.25, 0.7)) -> Workload:
    """cfg2: random box field with start/goal in opposite corners."""
    rng = np.random.default_rng(seed)
    spec = BezierSpec(m=2, gamma=2, T=1.0)
    xd, u, sample = standard_sets(side=side)
    tube = design_tube(spec, (6.0, 5.0), 0.02)
    start = np.array([0.4, 0.4, 0.0, 0.0])
    goal = np.array([side - 0.4, side - 0.4, 0.0, 0.0])
    obs = []
    while len(obs) < n_obstacles:
        c = rng.uniform(0.4, side - 0.4, 2)
        w = rng.uniform(*obstacle_size, 2)
        if np.linalg.norm(c - start[:2]) < 0.9 or np.linalg.norm(c - goal[:2]) < 0.9:
            continue
        obs.append(box_obstacle(c[0], c[1], w[0], w[1]))
    oracle = build_oracle(spec, xd, u, tube)
    return Workload(f"cfg2-random-field-{seed}", spec, oracle, sample, graph_n, seed,
                    np.array([start, goal]), _inflated(obs, tube, spec.m), start, goal)


def hopping_deg5(graph_n: int = 20000, n_obstacles: int = 50, seed: int = 1, obstacle_seed: int = 11,
                 clear_endpoints: bool = True) -> Workload:
    """cfg3: gamma=3 (degree-5 curves), 20k samples, 50 boxes.

    With ``clear_endpoints`` obstacle centres within 0.9 of start/goal are redrawn, the
    rule of the reference's random field (scenario.py:373-374), so a path exists.
    """
    spec = BezierSpec(m=2, gamma=3, T=1.0)
    xd = Box(np.array([0.0, 0.0, -1.5, -1.5, -4.0, -4.0]), np.array([5.0, 5.0, 1.5, 1.5, 4.0, 4.0])).to_polytope()
    u = Box(np.array([-30.0, -30.0]), np.array([30.0, 30.0]))
    sample = Box(np.array([0.0, 0.0, -0.6, -0.6, -1.0, -1.0]), np.array([5.0, 5.0, 0.6, 0.6, 1.0, 1.0]))
    tube = design_tube(spec, (6.0, 11.0, 6.0), 0.02)
    start = np.array([0.4, 0.4, 0.0, 0.0, 0.0, 0.0])
    goal = np.array([4.6, 4.6, 0.0, 0.0, 0.0, 0.0])
    rng = np.random.default_rng(obstacle_seed)
    obs = []
    while len(obs) < n_obstacles:
        c = rng.uniform(0.4, 4.6, 2)
        w = rng.uniform(0.25, 0.7, 2)
        if clear_endpoints and (np.linalg.norm(c - start[:2]) < 0.9 or np.linalg.norm(c - goal[:2]) < 0.9):
            continue
        obs.append(box_obstacle(c[0], c[1], w[0], w[1]))
    oracle = build_oracle(spec, xd, u, tube)
    return Workload("cfg3-hop-deg5-20k", spec, oracle, sample, graph_n, seed, np.array([start, goal]),
                    _inflated(obs, tube, spec.m), start, goal)


def keepin_quadrants(per_region: int = 50, seed: int = 4) -> Workload:
    """cfg1: 2D double integrator, 4 overlapping quadrant keep-in regions x 50 samples (200 states)
    + start/goal, the demo's 3 boxes as keep-out obstacles (regions.py semantics)."""
    w = demo(200, seed)
    quads = [((0.0, 0.0), (3.0, 3.0)), ((2.0, 0.0), (5.0, 3.0)), ((0.0, 2.0), (3.0, 5.0)), ((2.0, 2.0), (5.0, 5.0))]
    w.name = "cfg1-keepin-4"
    w.N = per_region * len(quads)
    w.extra = {"regions": [Box(np.array(lo), np.array(hi)).to_polytope() for lo, hi in quads],
               "per_region": per_region}
    return w


def scaling_sweep(nodes: int = 20000, n_regions=(20, 10), n_obstacles: int = 50, seed: int = 1) -> Workload:
    """cfg5: gamma=2 graph of `nodes` states over 200 keep-in cells (20 x 10 grid, 10% overlap) on a
    map of side 5 sqrt(N/2000) (mean out-degree held near cfg2's), 50 random boxes."""
    from .regions import grid_regions

    spec = BezierSpec(m=2, gamma=2, T=1.0)
    side = 5.0 * float(np.sqrt(nodes / 2000.0))
    xd, u, sample = standard_sets(side=side)
    tube = design_tube(spec, (6.0, 5.0), 0.02)
    regs = grid_regions(n_regions[0], n_regions[1], side, side)
    per = max(1, nodes // len(regs))
    rng = np.random.default_rng(seed + 100)
    start = np.array([0.4, 0.4, 0.0, 0.0])
    goal = np.array([side - 0.4, side - 0.4, 0.0, 0.0])
    obs = []
    while len(obs) < n_obstacles:
        c = rng.uniform(0.4, side - 0.4, 2)
        wd = rng.uniform(0.25, 0.7, 2)
        if np.linalg.norm(c - start[:2]) < 0.9 or np.linalg.norm(c - goal[:2]) < 0.9:
            continue
        obs.append(box_obstacle(c[0], c[1], wd[0], wd[1]))
    oracle = build_oracle(spec, xd, u, tube)
    return Workload(f"cfg5-sweep-{nodes}", spec, oracle, sample, per * len(regs), seed, np.array([start, goal]),
                    _inflated(obs, tube, spec.m), start, goal, extra={"regions": regs, "per_region": per})


def replanning_goals(w: Workload, count: int = 100, seed: int = 0) -> np.ndarray:
    """cfg4: goal positions U(0.3, 4.7)^2 with zero higher derivatives."""
    rng = np.random.default_rng(seed)
    pos = rng.uniform(0.3, 4.7, size=(count, 2))
    goals = np.zeros((count, w.spec.n))
    goals[:, :2] = pos
    return goals


BUILDERS = {
    "cfg1": keepin_quadrants,
    "cfg1-demo": demo,
    "cfg2": random_field,
    "cfg3": hopping_deg5,
    "cfg5": scaling_sweep,
}

"""Wire the device stage into the reference package ``beziergraph``.

The reference simulator imports its graph module as ``graphmod`` and calls
``graphmod.build_graph`` / ``graphmod.cut_graph`` / ``graphmod.find_path``
(sim.py:20, 202-209, 255-257, 324-335), so replacing those module attributes is
enough for ``plan_once`` and ``run_closed_loop`` to run on the GPU stage::

    import beziergraph
    from paper_2411_13507_b200 import shim
    shim.install(beziergraph)          # beziergraph.graph.* now run on the B200
    beziergraph.plan_once(beziergraph.demo_scenario())
    shim.uninstall(beziergraph)

The reference's own ``CutProvenance`` enum is used for ``CutMask.provenance`` while
installed, so masks compare equal to the reference's.
"""

from __future__ import annotations

from . import graph as _dev

_PATCHED = ("build_graph", "cut_graph", "find_path", "path_cost", "cut_heuristic", "cut_qp")
_saved: dict = {}


def _build_with_cache(cut_cache):
    def build_graph(N, spec, oracle, bounds, seed, include=None, k_nearest=None):
        g = _dev.build_graph(N, spec, oracle, bounds, seed, include, k_nearest)
        g.set_cut_cache(cut_cache)
        return g
    build_graph.__wrapped__ = _dev.build_graph
    return build_graph


def install(beziergraph_pkg, cut_cache: int = 0) -> None:
    """Patch ``beziergraph.graph`` (and the package re-exports) with the device functions.

    ``cut_cache`` > 0 turns on the re-cut cache of every graph built while installed
    (BezierGraph.set_cut_cache): the simulator's re-cuts of a fixed graph (sim.py:324-330)
    then screen and QP only the obstacles that moved.  The masks are identical either way."""
    gmod = beziergraph_pkg.graph
    if _saved:
        return
    for name in _PATCHED:
        fn = _build_with_cache(cut_cache) if (name == "build_graph" and cut_cache > 0) else getattr(_dev, name)
        _saved[("graph", name)] = getattr(gmod, name)
        setattr(gmod, name, fn)
        if hasattr(beziergraph_pkg, name):
            _saved[("pkg", name)] = getattr(beziergraph_pkg, name)
            setattr(beziergraph_pkg, name, fn)
    sim = getattr(beziergraph_pkg, "sim", None)
    if sim is not None and hasattr(sim, "_project_on_path"):  # sim.py:220-239 -> device
        from . import replan

        _saved[("sim", "_project_on_path")] = sim._project_on_path
        sim._project_on_path = replan.project_on_path
    _saved[("prov",)] = _dev._PROV_ENUM
    _dev._PROV_ENUM = gmod.CutProvenance
    _saved[("verdict",)] = _dev._VERDICT_ENUM
    _dev._VERDICT_ENUM = gmod.CutVerdict


def uninstall(beziergraph_pkg) -> None:
    gmod = beziergraph_pkg.graph
    for key, fn in list(_saved.items()):
        if key[0] == "graph":
            setattr(gmod, key[1], fn)
        elif key[0] == "pkg":
            setattr(beziergraph_pkg, key[1], fn)
        elif key[0] == "sim":
            setattr(beziergraph_pkg.sim, key[1], fn)
        elif key[0] == "prov":
            _dev._PROV_ENUM = fn
        elif key[0] == "verdict":
            _dev._VERDICT_ENUM = fn
    _saved.clear()

"""Per-phase wall time vs summed kernel time of one build -> cut -> find_path step."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2411_13507_b200 import _native as nat, configs, graph as G  # noqa: E402


def main(name="cfg3", reps=4):
    ctx = nat.Context(0)
    w = configs.BUILDERS[name]()
    for r in range(int(reps)):
        ctx.reset_stats()
        ctx.set_profiling(True)
        t0 = time.perf_counter()
        g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include, ctx=ctx)
        ctx.synchronize()
        t1 = time.perf_counter()
        mask = G.cut_graph(g, w.obstacles)
        ctx.synchronize()
        t2 = time.perf_counter()
        path = G.find_path(g, mask, w.start, w.goal)
        ctx.synchronize()
        t3 = time.perf_counter()
        _, st = ctx.stats()
        ctx.set_profiling(False)
        build_k = sum(v[0] for k, v in st.items() if k in ("k_sample_candidates", "cub_scan_sample", "k_sample_scatter",
                                                          "k_morton", "cub_sort_morton", "k_project_sorted",
                                                          "k_group_bounds", "k_pair_tiles", "cub_scan_rows", "k_expand",
                                                          "k_row_ptr_global"))
        cut_k = sum(v[0] for k, v in st.items() if k.startswith(("k_cut", "k_qp", "k_fill", "k_mask", "k_unpack")))
        path_k = sum(v[0] for k, v in st.items() if k.startswith(("k_snap", "k_bf", "k_parent", "k_init", "k_back",
                                                                  "k_reach")))
        print(f"rep {r}: build {1e3*(t1-t0):7.2f} ms (kernels {build_k:6.2f})  cut {1e3*(t2-t1):7.2f} ms "
              f"(kernels {cut_k:6.2f})  path {1e3*(t3-t2):6.2f} ms (kernels {path_k:5.2f})  hops {len(path or [])}")


if __name__ == "__main__":
    main(*sys.argv[1:])

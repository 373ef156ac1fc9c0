#!/usr/bin/env python
"""Benchmark of the B200 graph-construction stage (BASELINE.json metric).

One step = the whole hot path on one synthetic scene: sample V states (PCG64 on
device) -> all-pairs reachability test -> ordered CSR + edge costs -> obstacle cut
(box heuristic + batched Cut-QP + aggregation) -> snapping + Bellman-Ford shortest
path.  Default workload: cfg3 (degree-5 / gamma=3 hopping model, 20,000 samples +
start/goal, 50 boxes), i.e. 4.0e8 ordered pairs.

metric: edge evaluations/s = V^2 / t_step (whole job, all GPUs); ms_per_step is the
build+cut+solve latency.  ``value`` is timed with CUDA events on the library's stream
with L2 flushed before every step; ``e2e`` times the same call with host inputs and the
path read back.  On one GPU the step is the captured Planner (build -> cut -> find_path
as one CUDA graph, paths checked equal to the eager API's); the eager public API
(build_graph -> cut_graph -> find_path, one synchronisation per call) is reported
under "eager" and headlines with --no-planner and on several GPUs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg3] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (row-block sharding, NCCL gather)
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "edge evaluations/sec (V^2 / graph-build+cut+solve latency)"
UNIT = "edge_evals/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg3", choices=["cfg1", "cfg1-demo", "cfg2", "cfg3", "cfg4", "cfg5"])
    ap.add_argument("--nodes", type=int, default=0, help="cfg5: number of states (10k-100k)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-planner", action="store_true", help="headline the eager public-API step")
    ap.add_argument("--cpu-rows", type=int, default=0, help="source rows in the CPU sample (0 = auto)")
    ap.add_argument("--breakdown", action="store_true", help="print the per-kernel table to stderr")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(name, nodes=0):
    from paper_2411_13507_b200 import configs

    if name == "cfg5" and nodes:
        return configs.scaling_sweep(nodes)
    return configs.BUILDERS[name]()


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "20"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        rows = []
        for line in Path(self.path).read_text().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower().startswith("active")})
        busy = [s for s in sm if mx and s > 0.5 * max(mx)] or sm
        return {"sm_mhz": statistics.median(busy) if busy else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max((float(r[3]) for r in rows if r[3].replace(".", "").isdigit()), default=None)}


# ----------------------------------------------------------------------------- device step
class DeviceStep:
    """build -> cut -> (gather) -> find_path through libbzg, host constants prepared once."""

    def __init__(self, ctx, w, rank=0, world=1):
        from paper_2411_13507_b200 import graph as G
        from paper_2411_13507_b200 import shard

        self.G, self.ctx, self.w = G, ctx, w
        self.rank, self.world = rank, world
        V = w.num_vertices
        self.rows = shard.row_block(V, rank, world) if world > 1 else None
        regs = w.extra.get("regions")
        if regs:
            # keep-in regions (cfg1/cfg5): every step samples all regions on the device (one call,
            # bzg_sample_region_states) into a pinned-size host buffer the build reads its vertices from
            from paper_2411_13507_b200 import regions as R

            rr, self.sampling = region_constants(w)
            self.Vh = np.empty((self.sampling.total, w.spec.n))
            Vh = self.Vh
            self.desc, self._keep, self.D = G._build_desc(Vh.shape[0], w.spec, w.oracle, w.sample_bounds, w.seed,
                                                           w.include, vertices=Vh, rows=self.rows)
            off = np.concatenate([[0], np.cumsum([f.shape[0] for f in rr.F])]).astype(np.int32)
            RF, RG = G._f64(np.vstack(rr.F)), G._f64(np.concatenate(rr.G))
            blo, bhi = R.region_boxes(regs)
            self._keep += [off, RF, RG, blo, bhi]
            self.desc.n_regions = len(regs)
            self.desc.region_row_off, self.desc.region_F, self.desc.region_G = (nat_ptr(off), nat_ptr(RF),
                                                                                nat_ptr(RG))
            self.desc.region_box_lo, self.desc.region_box_hi = nat_ptr(blo), nat_ptr(bhi)
        else:
            self.desc, self._keep, self.D = G._build_desc(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, w.include,
                                                           rows=self.rows)
            self.sampling = None
        self.obs = G._obstacle_arrays(w.obstacles, w.spec.m)
        self.cfg = G._cut_cfg(G.CutConfig())
        self.last = {}

    def run(self):
        G, lib, ctx, w = self.G, self.ctx.lib, self.ctx, self.w
        from paper_2411_13507_b200 import _native as nat

        t0 = time.perf_counter()
        if self.sampling is not None:  # a2 for keep-in regions: all regions' samplers, one device call
            s = self.sampling
            nat.check(lib.bzg_sample_region_states(ctx.handle, w.spec.n, len(s.N), nat.ptr(s.N), nat.ptr(s.pcg),
                                                   nat.ptr(s.lo), nat.ptr(s.hi), nat.ptr(s.row_off), nat.ptr(s.A),
                                                   nat.ptr(s.b), G.EPS_GEO, nat.ptr(self.Vh)))
        h = C.c_void_p()
        nat.check(lib.bzg_build_graph(ctx.handle, C.byref(self.desc), C.byref(h)))
        graph = G.BezierGraph(h, ctx, w.spec, w.oracle, w.seed, w.sample_bounds, self.D)
        desc, keep = self.desc, self._keep  # no reference back to self: graph <-> step would be a cycle
        graph._desc_fn = lambda: (desc, keep)
        t1 = time.perf_counter()
        offs, A, b, is_box, lo, hi = self.obs
        mh = C.c_void_p()
        nat.check(lib.bzg_cut_graph(ctx.handle, h, len(is_box), nat.ptr(offs), nat.ptr(A), nat.ptr(b), nat.ptr(is_box),
                                    nat.ptr(lo), nat.ptr(hi), C.byref(self.cfg), C.byref(mh)))
        cnt = np.zeros(6, dtype=np.int64)
        nat.check(lib.bzg_mask_copy(mh, None, None, nat.ptr(cnt)))
        mask = G.CutMask(mh, graph, cnt)
        t2 = time.perf_counter()
        self.local_mask = mask
        E_all = graph.num_edges
        if self.world > 1:
            from paper_2411_13507_b200 import shard

            local_E = graph.num_edges
            graph, mask = shard.gather_to_root(graph, mask)
            self.last["local_edges"] = local_E
            if mask is not None:
                self.last["gather_bytes"] = mask.gather_bytes  # alive edges only travel to rank 0
                E_all = mask.pairs_total // len(w.obstacles) if w.obstacles else graph.num_edges
        t3 = time.perf_counter()
        path = None
        if self.rank == 0:
            path = G.find_path(graph, mask, w.start, w.goal)
        t4 = time.perf_counter()
        self.last.update(E=E_all if graph is not None else None, qp=int(cnt[3]), alive=None, path=path,
                         counters=cnt.tolist(),
                         host_phase_ms={"build": 1e3 * (t1 - t0), "cut": 1e3 * (t2 - t1), "gather": 1e3 * (t3 - t2),
                                        "path": 1e3 * (t4 - t3)})
        self.last_graph, self.last_mask = graph, mask
        return path


def region_constants(w):
    """Host constants of a keep-in workload, built once like the oracle itself (a1): the rows each
    region oracle adds (regions.region_rows) and the per-region sampler arrays."""
    if "_region_consts" not in w.extra:
        from paper_2411_13507_b200 import regions as R

        regs = w.extra["regions"]
        rr = R.region_rows(w.oracle, R.region_oracles(w.spec, w.oracle.Xd, w.oracle.U, w.oracle.tube, regs))
        s = R.region_sampling(w.extra["per_region"], w.spec, w.oracle.Xd, regs, w.sample_bounds, w.seed)
        w.extra["_region_consts"] = (rr, s)
    return w.extra["_region_consts"]


def nat_ptr(a):
    from paper_2411_13507_b200 import _native as nat

    return nat.ptr(a)


def public_api_step(w, ctx, rank, world):
    """The call sequence a user makes (reference sim.plan_once order), host inputs, path read back."""
    from paper_2411_13507_b200 import graph as G
    from paper_2411_13507_b200 import shard

    rows = shard.row_block(w.num_vertices, rank, world) if world > 1 else None
    if w.extra.get("regions"):
        from paper_2411_13507_b200 import regions as R

        rr, s = region_constants(w)
        g = R.build_region_graph(w.extra["per_region"], w.spec, w.oracle, w.extra["regions"], w.sample_bounds,
                                 w.seed, include=w.include, ctx=ctx, rows=rows, rows_added=rr, sampling=s)
    else:
        g = G.build_graph(w.N, w.spec, w.oracle, w.sample_bounds, w.seed, include=w.include, ctx=ctx, rows=rows)
    mask = G.cut_graph(g, w.obstacles)
    if world > 1:
        g, mask = shard.gather_to_root(g, mask)
    path = G.find_path(g, mask, w.start, w.goal) if rank == 0 else None
    return path


def h2d_d2h_bytes(w, path_len):
    n = w.spec.n
    h2d = (w.oracle.F.nbytes + w.oracle.G.nbytes + 8 * (w.spec.p + 1) * 2 * w.spec.gamma + w.oracle.Xd.A.nbytes
           + w.oracle.Xd.b.nbytes + 2 * 8 * n + (0 if w.include is None else np.asarray(w.include).nbytes)
           + sum(o.A.nbytes + o.b.nbytes + 2 * 8 * w.spec.m + 5 for o in w.obstacles) + 4 * 8 * n)
    d2h = 8 * path_len + 8 + 6 * 8 + 3 * 8  # path, dist, counters, E/sample/qp counts
    return int(h2d), int(d2h)


# ----------------------------------------------------------------------------- roofline
def algorithmic_work(kernel, w, step_info, world):
    """Algorithmic work of one launch of `kernel`: (amount, unit, bound)."""
    V = w.num_vertices
    g = w.spec.gamma
    m = w.spec.m
    E = step_info["E"]
    O = len(w.obstacles)
    if kernel in ("k_pair_bits", "k_pair_tiles", "k_pair_list"):
        # all-pairs interval test as the reference evaluates it (every ordered pair, every
        # coupled row); the tile cull skips provably failing blocks, so frac can exceed 1
        F = np.asarray(w.oracle.F)
        n = w.spec.n
        coupled = int((np.any(F[:, :n] != 0, axis=1) & np.any(F[:, n:] != 0, axis=1)).sum())
        K = coupled // 2  # negation-paired coupled rows -> two-sided intervals (1 add + 2 compares)
        pairs = V * V / world
        return pairs * 3 * K, "fp64"
    if kernel == "k_cut_heuristic":
        J = 2 * g
        per = J * 2 * m * (2 * m) + J * (3 * m + 1) + 2 * m * 4 + J * (2 * m)  # SURVEY.md §8(d) box pair
        return E * O * per, "fp64"
    if kernel == "k_qp_admm":
        canon = all(np.array_equal(np.asarray(o.A), np.vstack([np.eye(m), -np.eye(m)])) for o in w.obstacles)
        return step_info["qp_iterations"] * admm_ops_per_iteration(2 * g, m, canon), "fp64"
    return None, None


def admm_ops_per_iteration(J: int, M: int, canonical: bool) -> int:
    """FP64 operations of one reduced-form ADMM iteration as k_qp_admm performs them (DESIGN.md
    "Roofline").  Generic obstacle rows (C = 2M): KKT step 3C + 1 + J(3+C) + J^2, relaxation /
    projection / dual update 15J + C(J+15) + 6 (relaxations fused: RELAX in k_admm.cuh),
    termination test J + 2 + C(J+3) + J(C+2) + 3C (363 at J=6, M=2).  Canonical boxes keep only
    the M rows of P: 277 at J=6, M=2."""
    C = 2 * M
    fused = 2 * J + 2 * C + 1  # one DMUL + DADD per relaxation replaced by the FMA
    if not canonical:
        return ((3 * C + 1 + J * (3 + C) + J * J) + (17 * J + C * (J + 17) + 7)
                + (J + 2 + C * (J + 3) + J * (C + 2) + 3 * C)) - fused
    return (3 * C + 1 + M + J * (3 + M) + J * J + 12 * J + M * J + 14 * C + 7 + J + 2 + M * J + 3 * C + M
            + J * (2 + M) + 3 * C) - fused


_BYTE_UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def ncu_traffic(kernel: str, config: str):
    """dram read+write bytes per launch of `kernel` from the newest committed `ncu --set full`
    capture of this config (profiles/r*_ncu_full_<config>.json, tools/summarize_ncu.py; one
    step, so one launch per kernel), else None."""
    files = sorted((ROOT / "profiles").glob(f"r*_ncu_full_{config}.json"))
    if not files:
        return None, None
    recs = [r for r in json.loads(files[-1].read_text())["kernels"] if r.get("kernel") == kernel]
    if not recs:
        return None, None
    tot = 0.0
    for key in ("dram_read_bytes", "dram_write_bytes"):
        v = recs[0].get(key)
        if not isinstance(v, dict):
            return None, None
        tot += float(v["value"]) * _BYTE_UNITS.get(v["unit"], 1.0)
    return tot, files[-1].name


def main():
    args = parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        return reference_arm(args, rank, world)

    import gc

    import torch

    from paper_2411_13507_b200 import _native as nat

    # Python's cyclic GC can pause the host thread between the start event and the graph launch
    # of a sub-millisecond step (cfg1 showed one 1.4 ms step in ten); nothing here builds
    # reference cycles worth collecting during a few minutes of benchmarking
    gc.collect()
    gc.disable()

    # BZG_BENCH_DEVICE / BZG_DIST_BACKEND=gloo: functional check of the N>1 path with every rank
    # on one GPU and host-side collectives (never a performance number: ranks share the device)
    if os.environ.get("BZG_BENCH_DEVICE") is not None:
        local = int(os.environ["BZG_BENCH_DEVICE"])
    backend = os.environ.get("BZG_DIST_BACKEND", "nccl")
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = nat.Context(local, stream=stream.cuda_stream)
    nat.set_default_context(ctx)
    if args.config == "cfg4":
        return replanning_bench(args, ctx, stream, rank, world)
    w = workload(args.config, args.nodes)
    V = w.num_vertices
    step = DeviceStep(ctx, w, rank, world)

    def barrier():
        if world > 1:
            torch.distributed.barrier()

    fp64_rate = ctx.probe_fp64(True)  # DFMA instructions/s on this device
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(max(args.warmup, 0)):
        step.run()
    torch.cuda.synchronize()
    # breakdown pass (untimed): every launch timed with events, names the dominant kernel
    ctx.reset_stats()
    ctx.set_profiling(True)
    flush.zero_()
    step.run()
    torch.cuda.synchronize()
    _, breakdown = ctx.stats()
    dom = max(breakdown, key=lambda k: breakdown[k][0])

    # ---------------- timed region (device): K steps, L2 flushed before each; only the
    # dominant kernel's launches carry event pairs (its live duration feeds the roofline)
    ctx.reset_stats()
    ctx.profile_only(dom)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.4)  # let nvidia-smi attach before the first timed step
    barrier()
    torch.cuda.synchronize()
    evs = []
    for _ in range(args.steps):
        flush.zero_()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step.run()
        b.record(stream)
        evs.append((a, b))
    torch.cuda.synchronize()
    barrier()
    launches, kstats = ctx.stats()
    ctx.set_profiling(False)
    ctx.profile_only(None)
    step_ms = [a.elapsed_time(b) for a, b in evs]
    coll_dev = "cuda" if backend == "nccl" else "cpu"
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device=coll_dev)
    if world > 1:
        torch.distributed.all_reduce(tot, op=torch.distributed.ReduceOp.MAX)
    total_ms = float(tot.item())
    ms_per_step = total_ms / args.steps
    value = V * V / (ms_per_step * 1e-3)

    # ---------------- e2e through the public API
    e2e_ms = []
    path = None
    for k in range(args.steps + 1):
        flush.zero_()
        barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        path = public_api_step(w, ctx, rank, world)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        if k > 0:  # first call re-warms the Python path
            e2e_ms.append((t1 - t0) * 1e3)
    # ---------------- the same step through the captured Planner (one CUDA graph per step);
    # when the scene allows it (one GPU, no keep-in regions) it is the headline step
    planner = None
    if rank == 0 and world == 1 and not args.no_planner:
        planner = planner_block(w, ctx, stream, flush, args.steps)
    clk = clocks.stop()  # sampled over the timed region and the e2e pass that follows it
    clk["window"] = "device-timed steps + e2e steps" + (" + planner steps" if planner else "")
    et = torch.tensor([sum(e2e_ms) / len(e2e_ms)], dtype=torch.float64, device=coll_dev)
    if world > 1:
        torch.distributed.all_reduce(et, op=torch.distributed.ReduceOp.MAX)
    e2e_step_ms = float(et.item())
    h2d, d2h = h2d_d2h_bytes(w, len(path or []))

    # ---------------- roofline of the dominant kernel
    if step.local_mask is not None and step.local_mask.pairs_qp:
        step.last["qp_iterations"] = int(step.local_mask.qp_records()["iterations"].astype(np.int64).sum())
    else:
        step.last["qp_iterations"] = 0
    per_step = {k: (ms / args.steps, n / args.steps) for k, (ms, n) in kstats.items()}
    roof = {"kernel": dom}
    work, bound = algorithmic_work(dom, w, step.last, world)
    dom_ms, dom_n = per_step[dom]
    if work is not None and dom_n > 0:
        avg_launch_s = dom_ms / dom_n * 1e-3
        achieved = work / dom_n / avg_launch_s
        traffic, tsrc = ncu_traffic(dom, args.config)
        roof.update(bound=bound, achieved=achieved / 1e9, peak=fp64_rate / 1e9, unit="Gop/s (FP64 instr)",
                    frac=achieved / fp64_rate, traffic=traffic, traffic_source=tsrc,
                    algorithmic_ops_per_launch=work / dom_n, avg_launch_ms=dom_ms / dom_n,
                    peak_source="measured DFMA issue rate (bzg_probe_fp64, this run); "
                                "MEASURED_PEAKS.json has no FP64 figure")
        if dom == "k_cut_heuristic":
            roof["note"] = ("algorithmic work = the full box code of SURVEY.md 8(d) for every (edge, obstacle) "
                            "pair; the exact bounding-box certificate settles most pairs with a few compares, so "
                            "frac > 1 means the certificate beats the brute-force roofline")
        if dom in ("k_pair_tiles", "k_pair_list"):
            roof["note"] = ("algorithmic work = every ordered pair x every interval, as the reference "
                            "evaluates it; the exact tile cull skips provably failing blocks, so frac > 1 "
                            "means the cull beats the brute-force roofline")
    else:
        roof.update(bound=None, achieved=None, peak=None, frac=None, traffic=None)
    share = dom_ms / ms_per_step

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "vertices": V, "ordered_pairs": V * V, "edges": step.last["E"],
                   "obstacles": len(w.obstacles), "gamma": w.spec.gamma, "degree": w.spec.p,
                   "qp_instances": step.last["qp"], "parallelism": f"row-block x{world}",
                   "l2": "flushed before every step (256 MiB write)", "seed": w.seed},
        "latency_ms": ms_per_step,
        "step_ms": [round(x, 4) for x in step_ms],
        "path_hops": len(step.last["path"] or []) if rank == 0 else None,
        "clocks": clk,
        "e2e": {"value": V * V / (e2e_step_ms * 1e-3), "unit": UNIT, "ms_per_step": e2e_step_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "paper_2411_13507_b200.build_graph -> cut_graph -> find_path"},
        "gpu_launches": int(launches),
        "gpu_launches_per_step": launches / args.steps,
        "roofline": roof,
        "dominant_kernel_share": share,
        "kernels_ms_breakdown_pass": {k: round(v[0], 4) for k, v in sorted(breakdown.items(), key=lambda kv: -kv[1][0])},
        "fp64_peak_instr_per_s": fp64_rate,
        "host_phase_ms_last_step": {k: round(v, 3) for k, v in step.last.get("host_phase_ms", {}).items()},
    }
    if args.breakdown and rank == 0:
        for k, (ms, n) in sorted(breakdown.items(), key=lambda kv: -kv[1][0]):
            print(f"{k:28s} {ms:9.4f} ms/step  {n:7d} launches/step", file=sys.stderr)
    if planner is not None:
        # headline = the Planner's step; the eager public-API step (one host sync per call) kept
        out["eager"] = {"ms_per_step": ms_per_step, "value": value, "step_ms": out["step_ms"],
                        "e2e_ms_per_step": e2e_step_ms, "e2e_value": V * V / (e2e_step_ms * 1e-3),
                        "gpu_launches_per_step": launches / args.steps,
                        "api": "paper_2411_13507_b200.build_graph -> cut_graph -> find_path (eager)"}
        out["ms_per_step"] = out["latency_ms"] = planner["ms_per_step"]
        out["value"] = planner["value"]
        out["step_ms"] = planner["step_ms"]
        out["e2e"] = {"value": planner["e2e_value"], "unit": UNIT, "ms_per_step": planner["wall_ms_per_step"],
                      "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "api": planner["api"]}
        out["gpu_launches"] = planner["kernels_per_step"] * args.steps
        out["gpu_launches_per_step"] = planner["kernels_per_step"]
        out["dominant_kernel_share"] = dom_ms / planner["ms_per_step"]
        out["config"]["step_api"] = "Planner: build -> cut -> find_path as one captured CUDA graph"
        out["planner"] = {k: v for k, v in planner.items() if k not in ("step_ms",)}
    if rank == 0 and world == 1:
        out["parity"] = parity_block(w, step)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(w, step, args.cpu_rows)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def planner_block(w, ctx, stream, flush, steps):
    """The same step through the captured Planner (build -> cut -> find_path as ONE CUDA graph,
    bzg_planner): host inputs (seed words, include rows, obstacles, start, goal) staged in pinned
    memory, one graph launch, one synchronisation; device ms (events around the call, L2
    flushed) and wall ms per step; its path must equal the eager step's."""
    import torch

    from paper_2411_13507_b200.plan import Planner

    kw = {}
    if w.extra.get("regions"):  # keep-in regions (cfg1, cfg5): the same host constants as the eager step
        rr, smp = region_constants(w)
        kw = dict(regions=w.extra["regions"], per_region=w.extra["per_region"], rows_added=rr, sampling=smp)
    pl = Planner(w.N, w.spec, w.oracle, w.sample_bounds, w.obstacles, seed=w.seed, include=w.include, ctx=ctx,
                 **kw)
    want = public_api_step(w, ctx, 0, 1)
    dev, wall = [], []
    for k in range(steps + 3):
        flush.zero_()
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(stream)
        path = pl(w.seed, w.obstacles, w.start, w.goal, include=w.include)
        b.record(stream)
        b.synchronize()
        if k >= 3:
            wall.append(1e3 * (time.perf_counter() - t0))
            dev.append(a.elapsed_time(b))
    assert path == want, "planner path differs from the eager step's"
    info = pl.info()
    pl.close()
    V = w.num_vertices
    ms = float(np.mean(dev))
    return {"ms_per_step": ms, "value": V * V / (ms * 1e-3), "wall_ms_per_step": float(np.mean(wall)),
            "step_ms": [round(x, 4) for x in dev],
            "e2e_value": V * V / (float(np.mean(wall)) * 1e-3), "unit": UNIT,
            "kernels_per_step": info["kernels_per_call"], "eager_calls": info["eager_calls"],
            "edge_capacity": info["edge_capacity"], "path_equal_eager": True,
            "api": "paper_2411_13507_b200.plan.Planner (bzg_planner: build -> cut -> find_path as one captured "
                   "CUDA graph, host inputs)"}


# ----------------------------------------------------------------------------- cfg4 replanning
def replanning_bench(args, ctx, stream, rank, world):
    """BASELINE config 4: cfg2's graph and mask held fixed, 100 sequential goal
    updates find_path(g, mask, start, goal_k); latency p50/p99 per update.  "tree-cached" is the
    goal-only update (the shortest-path tree of (mask, v0) is reused, bitwise the same answer);
    "moving start" alternates two starts so every update recomputes the tree."""
    import torch

    from paper_2411_13507_b200 import configs
    from paper_2411_13507_b200 import graph as G

    if rank != 0:
        return
    w = configs.BUILDERS["cfg2"]()
    step = DeviceStep(ctx, w)
    step.run()
    graph, mask = step.last_graph, step.last_mask
    goals = configs.replanning_goals(w, 100)
    # a second start exactly at another vertex near the first: alternating the two changes v0
    # (and so invalidates the cached shortest-path tree) on every call
    Vx = graph.vertices
    near = np.argsort(np.linalg.norm(Vx - np.asarray(w.start), axis=1))
    start2 = Vx[int(near[1])].copy()

    query = G.PathQuery(graph, mask)  # the same search captured as one CUDA graph

    def timed(starts, fn=None):
        fn = fn or (lambda st, gl: G.find_path(graph, mask, st, gl))
        dev, wall, paths = [], [], []
        for k, gl in enumerate(goals):
            st = starts[k % len(starts)]
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record(stream)
            p = fn(st, gl)
            b.record(stream)
            b.synchronize()
            wall.append(1e3 * (time.perf_counter() - t0))
            dev.append(a.elapsed_time(b))
            paths.append(p)
        return np.array(dev), np.array(wall), paths

    for _ in range(max(args.warmup, 1)):
        timed([w.start])
        timed([w.start, start2], query)
    ctx.reset_stats()
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.4)
    dev_c, wall_c, paths = timed([w.start])
    dev_m, wall_m, paths_m = timed([w.start, start2])
    launches_eager, _ = ctx.stats()
    ctx.reset_stats()
    qdev_c, qwall_c, qpaths = timed([w.start], query)
    qdev_m, qwall_m, qpaths_m = timed([w.start, start2], query)
    launches, _ = ctx.stats()  # the captured queries' kernels (the headline)
    clk = clocks.stop()
    assert qpaths == paths and qpaths_m == paths_m, "captured query differs from find_path"
    pct = lambda a, q: float(np.percentile(a, q))  # noqa: E731
    out = {
        "metric": "goal-update latency p50 (find_path on a fixed graph+mask)", "value": pct(qdev_c, 50), "unit": "ms",
        "n_gpus": 1, "steps": len(goals), "warmup": args.warmup, "ms_per_step": pct(qdev_c, 50),
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "cfg4-replanning (cfg2 graph + mask fixed, 100 goals U(0.3,4.7)^2)",
                   "vertices": graph.num_vertices, "edges": graph.num_edges, "alive": mask.alive_count,
                   "step_api": "PathQuery: find_path captured as one CUDA graph (same paths as find_path)"},
        "p99_ms": pct(qdev_c, 99), "p50_ms": pct(qdev_c, 50),
        "moving_start": {"p50_ms": pct(qdev_m, 50), "p99_ms": pct(qdev_m, 99)},
        # the same updates through the eager find_path (one synchronisation per call)
        "eager": {"p50_ms": pct(dev_c, 50), "p99_ms": pct(dev_c, 99), "moving_start_p50_ms": pct(dev_m, 50),
                  "moving_start_p99_ms": pct(dev_m, 99), "wall_p50_ms": pct(wall_c, 50),
                  "wall_moving_start_p50_ms": pct(wall_m, 50), "api": "paper_2411_13507_b200.find_path"},
        "e2e": {"value": pct(qwall_c, 50), "unit": "ms", "p99": pct(qwall_c, 99),
                "moving_start_p50": pct(qwall_m, 50), "h2d_bytes_per_step": 2 * 8 * w.spec.n,
                "d2h_bytes_per_step": int(np.mean([8 * (len(p or []) + 1) for p in paths])),
                "api": "paper_2411_13507_b200.PathQuery", "kernels_per_query": query.kernels_per_query},
        "paths_found": int(sum(p is not None for p in paths)),
        "gpu_launches": int(launches), "gpu_launches_eager": int(launches_eager), "clocks": clk,
        "roofline": {"kernel": "k_bf_persistent", "bound": "latency", "achieved": None, "peak": None, "frac": None,
                     "traffic": None, "note": "a goal update is a few dependent small launches; latency-bound"},
    }
    out["recut_moving_obstacle"] = recut_bench(ctx, stream, w, graph, steps=20)
    print(json.dumps(out), flush=True)


def recut_bench(ctx, stream, w, graph, steps=20):
    """Replanning with a moving obstacle (sim.py:324-330, ObstacleTrack.at): every cycle obstacle
    0 moves a few cm along its track and the graph is re-cut, then searched (relaxed snap, as
    run_closed_loop mid-run).  Device ms per cycle: the eager full cut, the eager re-cut cache
    (BezierGraph.set_cut_cache), and the Replanner (cut + search as one captured CUDA graph),
    re-cutting every obstacle or only the moving one (static / dynamic split); and whether all
    masks agree on every cycle."""
    import torch

    from paper_2411_13507_b200 import graph as G
    from paper_2411_13507_b200.geometry import Polytope

    obs = list(w.obstacles)
    m = w.spec.m

    def lists():
        cur = list(obs)
        for k in range(steps):
            A = np.asarray(cur[0].A, dtype=np.float64)
            cur[0] = Polytope(A, np.asarray(cur[0].b, dtype=np.float64) + A @ np.full(m, 0.01 * (1 + k % 3)))
            yield list(cur)

    res, masks = {}, {}
    for mode, cache in (("full", 0), ("cached", 4 * len(obs))):
        graph.set_cut_cache(cache)
        G.cut_graph(graph, obs)  # warm (and fill the cache with the static obstacles)
        ms, ms_cut, ms_all = [], [], []
        masks[mode] = []
        for lst in lists():
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            c = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            mk = G.cut_graph(graph, lst)
            b.record(stream)
            G.find_path(graph, mk, w.start, w.goal, position_only_snap=True, require_tube_snap=False)
            c.record(stream)
            c.synchronize()
            ms_cut.append(a.elapsed_time(b))
            ms_all.append(a.elapsed_time(c))
            masks[mode].append(np.packbits(mk.alive).tobytes() + mk.provenance_codes.tobytes())
        res[mode] = {"cut_p50_ms": float(np.percentile(ms_cut, 50)), "cycle_p50_ms": float(np.percentile(ms_all, 50)),
                     "cycle_p99_ms": float(np.percentile(ms_all, 99))}
    graph.set_cut_cache(0)
    # the same cycles through the Replanner: cut + search captured as one CUDA graph
    from paper_2411_13507_b200.replan import Replanner

    for mode, dyn in (("captured", None), ("captured_split", [True] + [False] * (len(obs) - 1))):
        rp = Replanner(graph, obs, position_only_snap=True, require_tube_snap=False, dynamic=dyn)
        rp(obs, w.start, w.goal)
        ms_all, masks[mode], walls = [], [], []
        for lst in lists():
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            t0 = time.perf_counter()
            a.record(stream)
            rp(lst, w.start, w.goal)
            b.record(stream)
            b.synchronize()
            walls.append(1e3 * (time.perf_counter() - t0))
            ms_all.append(a.elapsed_time(b))
            mk = rp.mask()
            masks[mode].append(np.packbits(mk.alive).tobytes() + mk.provenance_codes.tobytes())
        info = rp.info()
        rp.close()
        res[mode] = {"cycle_p50_ms": float(np.percentile(ms_all, 50)), "cycle_p99_ms": float(np.percentile(ms_all, 99)),
                     "wall_p50_ms": float(np.percentile(walls, 50)), "kernels_per_cycle": info["kernels_per_cycle"],
                     "eager_cycles": info["eager_cycles"], "api": "paper_2411_13507_b200.replan.Replanner"}
    res["masks_equal_every_cycle"] = (masks["full"] == masks["cached"] == masks["captured"] ==
                                      masks["captured_split"])
    res["workload"] = f"{w.name}: obstacle 0 of {len(obs)} moves every cycle, {steps} cycles, cut + relaxed-snap search"
    return res


# ----------------------------------------------------------------------------- CPU baselines
def _cpu_sample_rows(w, rows):
    """Oracle port on source rows [r0, r1): (t_build_rows, t_cut, n_edges, n_qp)."""
    import oracle
    from paper_2411_13507_b200.bezier import boundary_matrix

    D = boundary_matrix(w.spec)
    n = w.spec.n
    V_ = oracle.sample_states(w.N, w.sample_bounds.lo, w.sample_bounds.hi, w.oracle.Xd.A, w.oracle.Xd.b, w.seed,
                              w.include)
    A1, A2 = oracle.project(V_, w.oracle.F, n)
    t0 = time.perf_counter()
    E = oracle.pair_edges(A1, A2, w.oracle.G, rows=rows)
    pts = oracle.edge_points(V_, E, D, w.spec.gamma, w.spec.m)
    oracle.edge_costs(pts)
    t1 = time.perf_counter()
    res = oracle.cut_graph(pts, [(o.A, o.b) for o in w.obstacles])
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, E.shape[0], res["pairs_qp"]


def cpu_baseline(w, step, rows_opt):
    """One host core on a bounded row sample: the unmodified reference package where the config
    has a reference generator (cfg2, cfg3: build_graph's pair test + cut_graph's own
    _heuristic_batch / solve_batch, _ref_live_rows; its own find_path on the full graph the device
    produced), else the oracle port (numpy restatement of the reference)."""
    import types

    V = w.num_vertices
    S = rows_opt or max(8, min(V, int(round(V * 0.005))))  # ~0.5% of the source rows
    g, mk = step.last_graph, step.last_mask
    if _import_reference() is not None and w.name.startswith(("cfg2", "cfg3")):
        from beziergraph import graph as rg

        name = "cfg3" if w.name.startswith("cfg3") else "cfg2"
        t0 = time.perf_counter()
        _ref_live_init(name)  # scene + sampler (graph.py:147-159) on reference objects
        t_sample = time.perf_counter() - t0
        t0 = time.perf_counter()
        e_s, q_s = _ref_live_rows((0, S))
        t_rows = time.perf_counter() - t0
        spec, oracle = _REF_SCENE[0], _REF_SCENE[1]
        gref = types.SimpleNamespace(vertices=g.vertices, edges=g.edges, costs=g.costs, spec=spec, oracle=oracle,
                                     num_vertices=g.num_vertices)
        mref = types.SimpleNamespace(alive=mk.alive)
        t0 = time.perf_counter()
        rg.find_path(gref, mref, w.start, w.goal)
        t_path = time.perf_counter() - t0
        t_full = t_sample + t_rows * (V / S) + t_path
        return {"value": V * V / t_full, "unit": UNIT, "cores": 1, "kind": "reference",
                "ms_per_step_extrapolated": t_full * 1e3,
                "sample": (f"unmodified reference package (baseline/_ref) in one process: scene + sampler "
                           f"({t_sample:.2f}s), build_graph's pair test + points + costs and cut_graph's "
                           f"_heuristic_batch + solve_batch on source rows [0,{S}) ({S * V} pairs, {e_s} edges, "
                           f"{q_s} QPs, {t_rows:.2f}s) extrapolated x{V / S:.1f}, the reference's find_path on the "
                           f"full {g.num_edges}-edge graph ({t_path:.2f}s)"),
                "cpu_model": _cpu_model()}
    import oracle

    t0 = time.perf_counter()
    oracle.sample_states(w.N, w.sample_bounds.lo, w.sample_bounds.hi, w.oracle.Xd.A, w.oracle.Xd.b, w.seed, w.include)
    t_sample = time.perf_counter() - t0
    tb, tc, e_s, q_s = _cpu_sample_rows(w, (0, S))
    # Dijkstra (heapq) on the full graph the device produced (same arrays the reference would search)
    t0 = time.perf_counter()
    oracle.find_path(g.vertices, g.edges, g.costs, mk.alive, w.start, w.goal, w.spec.m, w.oracle.tube.error.lo,
                     w.oracle.tube.error.hi)
    t_path = time.perf_counter() - t0
    t_full = t_sample + (tb + tc) * (V / S) + t_path
    return {"value": V * V / t_full, "unit": UNIT, "cores": 1, "kind": "port",
            "ms_per_step_extrapolated": t_full * 1e3,
            "sample": (f"oracle port (numpy restatement of reference graph.py) single process: sampling of all "
                       f"{V} states, pair test + control points + costs + box cut + Cut-QP on source rows [0,{S}) "
                       f"({S * V} pairs, {e_s} edges, {q_s} QPs) extrapolated x{V / S:.1f}, heapq Dijkstra on the "
                       f"full {g.num_edges}-edge graph; measured build {tb:.2f}s cut {tc:.2f}s path {t_path:.2f}s"),
            "cpu_model": _cpu_model()}


def parity_block(w, step):
    """The step's outputs against the live-reference golden of this workload (tests/golden,
    captured by make_golden.py from the unmodified reference on the same inputs): outside the
    timed region.  None when no golden exists for the config."""
    import hashlib

    name = {"cfg3-hop-deg5-20k": "cfg3_hop20k", "cfg2-random-field-1": "cfg2_rf2000"}.get(w.name)
    path = ROOT / "tests" / "golden" / f"{name}.npz"
    if name is None or not path.exists() or step.world > 1:
        return None
    gd = np.load(path)
    g, mk = step.last_graph, step.last_mask
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    alive = mk.alive
    cnt = [mk.pairs_total, mk.pairs_point_hit, mk.pairs_hyperplane, mk.pairs_qp, mk.qp_safe, mk.qp_unsafe]
    ref_cnt = [int(x) for x in gd["counters"]]
    band = g.eps_band(1e-11)["band"] if g._desc_fn is not None else None
    return {"golden": f"tests/golden/{name}.npz (live reference, {str(gd['env'])[:60]}...)",
            "vertices_bitwise": sha(g.vertices) == str(gd["sha_vertices"]),
            "edges_bitwise": sha(g.edges) == str(gd["sha_edges"]),
            "costs_bitwise": sha(g.costs) == str(gd["sha_costs"]),
            "heuristic_counters_equal": cnt[:4] == ref_cnt[:4],
            "qp_counters": {"device": cnt[4:], "reference": ref_cnt[4:]},
            "alive_mismatch": int((alive != gd["alive"]).sum()),
            "provenance_mismatch": int((mk.provenance_codes != gd["provenance"]).sum()),
            "path_equal": step.last["path"] == [int(x) for x in gd["path"]],
            "eps_band_1e-11": {"device": band, "reference": int(gd["eps_band_1e-11"])} if "eps_band_1e-11" in gd else None,
            "note": "QP verdict differences are solver-sensitive (tests/helpers.py qp_solver_sensitive)"}


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _import_reference():
    """The unmodified reference package: baseline/_ref (pip-installed by __graft_entry__.build(),
    travels to the GPU box) or /root/reference/pkg/src (the build container); None if absent."""
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "beziergraph" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import beziergraph

            return beziergraph
    return None


_REF_SCENE = None


def _ref_scene(name):
    """Reference objects of a BASELINE workload built with the reference's own generators:
    (spec, oracle, V, inflated obstacles, CutConfig).  cfg2 = random_field_scenario(1, 20, 2000)
    through sim.build_pipeline's inputs; cfg3 = the recipe of tests/golden/make_golden.py
    case_cfg3.  Vertices by build_graph's own sampler loop (graph.py:147-159) on reference
    Box/Polytope objects.  None for the keep-in configs (no reference function)."""
    bg = _import_reference()
    if bg is None or name not in ("cfg2", "cfg3"):
        return None
    from beziergraph import geometry as rgeo
    from beziergraph import graph as rg
    from beziergraph import scenario as rsc
    from beziergraph import sim as rsim

    if name == "cfg2":
        s = rsc.random_field_scenario(1, n_obstacles=20, graph_n=2000)
        spec, oracle = s.spec, bg.build_oracle(s.spec, s.xd, s.u_bounds, s.tube)
        N, bounds, seed, include = s.graph_n, s.sample_bounds, s.seed_graph, np.array([s.start, s.goal])
        obstacles = rsim._inflated(s, 0.0)
    else:
        spec = bg.BezierSpec(m=2, gamma=3, T=1.0)
        xd = rgeo.Box(np.array([0.0, 0.0, -1.5, -1.5, -4.0, -4.0]), np.array([5.0, 5.0, 1.5, 1.5, 4.0, 4.0])).to_polytope()
        u = rgeo.Box(np.array([-30.0, -30.0]), np.array([30.0, 30.0]))
        bounds = rgeo.Box(np.array([0.0, 0.0, -0.6, -0.6, -1.0, -1.0]), np.array([5.0, 5.0, 0.6, 0.6, 1.0, 1.0]))
        tube = rsim.design_tube(spec, (6.0, 11.0, 6.0), 0.02)
        oracle = bg.build_oracle(spec, xd, u, tube)
        start = np.array([0.4, 0.4, 0, 0, 0, 0.0])
        goal = np.array([4.6, 4.6, 0, 0, 0, 0.0])
        rng = np.random.default_rng(11)
        obs = []
        while len(obs) < 50:
            c = rng.uniform(0.4, 4.6, 2)
            w_ = rng.uniform(0.25, 0.7, 2)
            if np.linalg.norm(c - start[:2]) < 0.9 or np.linalg.norm(c - goal[:2]) < 0.9:
                continue
            obs.append(rsc._box_obstacle(c[0], c[1], w_[0], w_[1]).shape)
        obstacles = [rgeo.inflate(o, tube.position_box(2)) for o in obs]
        N, seed, include = 20000, 1, np.array([start, goal])
    rng = np.random.default_rng(seed)  # graph.py:147-159
    got, need = [], N
    while need > 0:
        cand = bounds.sample(rng, need)
        ok = oracle.Xd.contains_many(cand)
        if ok.any():
            got.append(cand[ok])
            need -= int(ok.sum())
    V = np.vstack([np.vstack(got)[:N], include])
    return spec, oracle, V, obstacles, rg.CutConfig()


def _ref_live_init(name):
    global _REF_SCENE
    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    _REF_SCENE = _ref_scene(name)


def _ref_live_rows(payload):
    """Source rows [r0, r1) through the reference: the pair test as build_graph evaluates it
    (graph.py:172-197, its own projections and 32-row chunks), then the reference's own
    _heuristic_batch and qpsolver.solve_batch on those edges, as cut_graph calls them
    (graph.py:312-337).  Returns (edges, QPs)."""
    from beziergraph import bezier as rbz
    from beziergraph import graph as rg
    from beziergraph import qpsolver as rqp

    r0, r1 = payload
    spec, oracle, V, obstacles, cfg = _REF_SCENE
    n = spec.n
    A1 = V[r0:r1] @ oracle.F1.T
    A2 = V @ oracle.F2.T
    thresh = oracle.G + rg.EPS_GEO
    src_l, dst_l = [], []
    for lo in range(0, r1 - r0, rg._PAIR_CHUNK):
        hi = min(lo + rg._PAIR_CHUNK, r1 - r0)
        feas = np.all(A1[lo:hi][:, None, :] + A2[None, :, :] <= thresh, axis=2)
        feas[np.arange(hi - lo), np.arange(r0 + lo, r0 + hi)] = False
        s_, d_ = np.nonzero(feas)
        src_l.append(s_ + r0 + lo)
        dst_l.append(d_)
    E = np.stack([np.concatenate(src_l), np.concatenate(dst_l)], axis=1).astype(np.int64)
    D = rbz.boundary_matrix(spec)
    x1 = V[E[:, 0]].reshape(-1, spec.gamma, spec.m)
    x2 = V[E[:, 1]].reshape(-1, spec.gamma, spec.m)
    pts = np.einsum("pq,eqm->emp", D, np.concatenate([x1, x2], axis=1))
    np.linalg.norm(np.diff(pts, axis=2), axis=1).sum(axis=1)
    del n
    n_qp = 0
    for ob in obstacles:
        codes = rg._heuristic_batch(pts, ob, cfg)
        pending = np.nonzero(codes == 2)[0]
        n_qp += pending.size
        if pending.size:
            O = ob.normalized()
            rqp.solve_batch([rg._cut_qp_problem(pts[e], O) for e in pending], cfg.qp)
    return E.shape[0], n_qp


def _ref_worker(payload):
    name, r0, r1 = payload
    w = workload(name)
    return _cpu_sample_rows(w, (r0, r1))


def reference_arm(args, rank, world):
    """`--impl reference`: the reference's CPU path on all host cores (rank 0 only).

    cfg2 / cfg3: the unmodified reference package (baseline/_ref) in a pool of one process per
    host core, each running the reference's own build arithmetic and its _heuristic_batch /
    solve_batch on a block of source rows (SURVEY.md §8(d) "ref-Np").  A step is a bounded
    row sample, extrapolated linearly to all rows (the whole reference step at cfg3 is
    ~2,900 s on one core: tests/golden/cfg3_hop20k.npz t_build + t_cut).  Keep-in configs have
    no reference function: the oracle port stands in there."""
    if rank != 0:
        return
    import multiprocessing as mp

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    w = workload(args.config)
    V = w.num_vertices
    cores = len(os.sched_getaffinity(0))
    live = _import_reference() is not None and args.config in ("cfg2", "cfg3")
    S = args.cpu_rows or min(V, cores * (48 if args.config == "cfg3" else 64))
    times = []
    if live:
        chunks = [(S * k // cores, S * (k + 1) // cores) for k in range(cores)]
        pool = mp.get_context("spawn").Pool(cores, initializer=_ref_live_init, initargs=(args.config,))
        fn = _ref_live_rows
    else:
        chunks = [(args.config, S * k // cores, S * (k + 1) // cores) for k in range(cores)]
        pool = mp.get_context("spawn").Pool(cores)
        fn = _ref_worker
    with pool:
        for k in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            res = pool.map(fn, chunks)
            t = time.perf_counter() - t0
            if k >= args.warmup:
                times.append(t)
    ms_sample = statistics.mean(times) * 1e3
    ms_full = ms_sample * V / S
    value = V * V / (ms_full * 1e-3)
    if live:
        e_s = sum(r[0] for r in res)
        q_s = sum(r[1] for r in res)
        kind = "reference"
        sample = (f"unmodified reference package (baseline/_ref beziergraph) in a {cores}-process pool: each step "
                  f"= build_graph's pair test + control points + costs (graph.py:172-197) and cut_graph's "
                  f"_heuristic_batch + qpsolver.solve_batch (graph.py:312-337) on source rows [0,{S}) of {w.name} "
                  f"({S * V} pairs, {e_s} edges, {q_s} QPs), extrapolated x{V / S:.1f} to all rows; Dijkstra "
                  f"excluded (the reference's heapq search: 1.2 s of its 2,902 s single-core step at cfg3, 93 ms "
                  f"of 76 s at cfg2)")
    else:
        e_s = sum(r[2] for r in res)
        q_s = sum(r[3] for r in res)
        kind = "port"
        sample = (f"oracle port (numpy restatement of reference graph.py/qpsolver.py; the keep-in regions have no "
                  f"reference function) in a {cores}-process pool: each step = pair test + control points + costs + "
                  f"box cut + Cut-QP on source rows [0,{S}) of {w.name} ({S * V} pairs, {e_s} edges, {q_s} QPs), "
                  f"extrapolated x{V / S:.1f} to all rows; Dijkstra excluded")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_full, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": w.name, "vertices": V, "ordered_pairs": V * V, "obstacles": len(w.obstacles),
                      "gamma": w.spec.gamma, "degree": w.spec.p, "parallelism": f"cpu x{cores}",
                      "seed": w.seed},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                            "cpu_model": _cpu_model()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

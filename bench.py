#!/usr/bin/env python
"""Benchmark of the exact 2D LMS fit (BASELINE.json metric, config 2).

One step = one complete exact LMS fit of n = 16,384 points (49% gross
outliers, q = n//2 + 1, fp64) over all n(n-1)/2 arrangement vertices: slope
bands and their lower bounds, band-seeded bound, one collect pass over every
vertex, window counts of the collected vertices, exact re-evaluation of the
survivors, argmin.  With
N > 1 processes (torchrun) the vertex-rank space of the SAME fit is split
into N contiguous partitions and the per-rank records are combined with one
NCCL all_gather each step (strong scaling).

Prints one JSON line on rank 0.  ``value`` is vertex-line evaluations per
second in the reference's counting (n * n(n-1)/2 per fit / device time);
``time_to_fit_s`` is the per-fit device time.  ``--impl reference`` times
the CPU restatement of the reference's algorithm (oracle/, C++ port with
std::nth_element in place of np.sort, all host threads) on a bounded sample
of the same workload and extrapolates to the same metric.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "exact 2D LMS vertex-line evals/s (time-to-fit) at n=16384, fp64"
UNIT = "vertex-line evals/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=50)
    p.add_argument("--warmup", type=int, default=5)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--n", type=int, default=16384)
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--cpu-vertices-per-thread", type=int, default=3000)
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-extra", action="store_true", help="skip the configs 1/4/5 side measurements")
    return p.parse_args()


def workload(n: int, seed: int):
    from paper_1510_01041_b200 import workloads

    pts = workloads.contaminated_line_points(n, seed)
    return pts, n // 2 + 1


def config(n: int, world: int) -> dict:
    return {
        "workload": f"config2: exact LMS fit, n={n} points, 49% gross outliers, q=n//2+1, fp64",
        "n": n,
        "pairs": n * (n - 1) // 2,
        "q": n // 2 + 1,
        "partitioning": (f"contiguous vertex-rank partitions x{world}; sharded band search: each rank "
                         "bounds 1/N of the slope bands, NCCL all_gather of the band table, then of "
                         "the per-rank records") if world > 1 else "one GPU, whole pair space",
        "l2": "flushed between timed steps (256 MiB write); the 256 KiB line set is re-read from "
              "L2 within a fit by design",
    }


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi-equivalent NVML sampling of SM clocks / throttle reasons."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
        0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._t = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
            return self
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(0.01)

    def stop(self) -> dict:
        self._stop.set()
        if self._t:
            self._t.join()
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


# --------------------------------------------------------------------------- cpu baseline
def cpu_baseline(a, b, q, n, per_thread: int) -> dict:
    """Oracle (C++ restatement of the reference's scan) on 16 evenly spaced
    rank slices of the same fit, all host threads."""
    import oracle

    oracle.build()
    threads = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else (os.cpu_count() or 1)
    total = n * (n - 1) // 2
    slices = 16
    per_slice = max(1, (per_thread * threads) // slices)
    t0 = time.perf_counter()
    verts = 0
    for s in range(slices):
        r0 = (s * total) // slices
        r1 = min(total, r0 + per_slice)
        oracle.min_bracelet(a, b, q, r0, r1, threads=threads)
        verts += r1 - r0
    dt = time.perf_counter() - t0
    rate = n * verts / dt
    return {
        "value": rate,
        "unit": UNIT,
        "cores": threads,
        "kind": "port",
        "sample": f"{verts} vertices ({slices} evenly spaced rank slices of the n={n} fit) x {n} lines "
                  f"in {dt:.2f}s; full fit extrapolates to {n * total / rate:.0f}s",
        "time_to_fit_s_extrapolated": n * total / rate,
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    pts, q = workload(args.n, args.seed)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    for _ in range(max(0, min(args.warmup, 1))):
        cpu_baseline(a, b, q, args.n, max(50, args.cpu_vertices_per_thread // 10))
    vals = []
    last = None
    for _ in range(args.steps):
        last = cpu_baseline(a, b, q, args.n, max(50, args.cpu_vertices_per_thread // 3))
        vals.append(last["value"])
    value = float(statistics.median(vals))
    n = args.n
    total = n * (n - 1) // 2
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": value,
        "unit": UNIT,
        "n_gpus": args.gpus,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * n * total / value,
        "time_to_fit_s": n * total / value,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (workloads.contaminated_line_points, seed 0)",
        "config": config(n, 1),
        "cpu_baseline": {**last, "value": value},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "note": "CPU restatement of the reference's exact scan (oracle/lms_oracle.cpp), each step a "
                "bounded rank sample of the fit extrapolated to the full fit; the reference package "
                "itself is pure Python+numpy with no GPU path",
    }
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- configs 1, 4, 5
def other_configs(device: int, reps: int = 3) -> dict:
    """Device / end-to-end times of BASELINE.json configs 1, 3, 4 and 5 (median
    of `reps` after one warm-up), reported beside the headline config 2."""
    import paper_1510_01041_b200 as lms
    from paper_1510_01041_b200 import _native, workloads

    res = {}
    ctx = _native.Context(device)

    def timed(fn):
        fn()
        ms = []
        for _ in range(reps):
            ctx.record(2)
            fn()
            ctx.record(3)
            ms.append(ctx.elapsed_ms(2, 3))
        return statistics.median(ms)

    # config 1: n = 1000, exact inliers on y = 2x + 1, 45% outliers, q = 501
    pts = workloads.config1_points(0)
    ctx.upload(pts[:, 0], pts[:, 1])
    ms = timed(lambda: ctx.solve(501, 0, 1000 * 999 // 2))
    res["config1"] = {"workload": "n=1000, 45% outliers, q=501", "ms_per_fit": ms,
                      "evals_per_s": 1000 * 499500 / (ms / 1e3)}
    # config 3: n = 65,536 on this one GPU (the multi-GPU case shards this rank space)
    n3 = 65536
    pts3 = workloads.contaminated_line_points(n3, 0)
    ctx.upload(pts3[:, 0], pts3[:, 1])
    P3 = n3 * (n3 - 1) // 2
    ms = timed(lambda: ctx.solve(n3 // 2 + 1, 0, P3))
    res["config3"] = {"workload": "n=65536, 49% outliers, q=32769, one GPU (all 2,147,450,880 pairs)",
                      "ms_per_fit": ms, "evals_per_s": n3 * P3 / (ms / 1e3)}
    # config 4: 8,192 fits of bench_points(512) (experiments.py:247-254)
    F, m = 8192, 512
    sets = [workloads.bench_points(m, seed=f) for f in range(F)]
    X = np.concatenate([t[:, 0] for t in sets])
    Y = np.concatenate([t[:, 1] for t in sets])
    offs = np.arange(F + 1, dtype=np.int64) * m
    qs = np.full(F, m // 2 + 1, dtype=np.int64)
    ctx.upload(X, Y)
    ms = timed(lambda: ctx.solve_batch(offs, qs))
    lms.solve_lms_batch(sets)  # warm-up of the public batch path
    walls4 = []
    for _ in range(reps):
        t0 = time.perf_counter()
        lms.solve_lms_batch(sets)  # host arrays in, LmsFit objects (with contact sets) out
        walls4.append(time.perf_counter() - t0)
    res["config4"] = {"workload": "8192 fits x n=512 (bench_points), q=257", "ms_per_batch": ms,
                      "evals_per_s": F * m * (m * (m - 1) // 2) / (ms / 1e3),
                      "e2e_ms": 1e3 * statistics.median(walls4),
                      "e2e_path": "solve_lms_batch(list of (512, 2) arrays) -> list[LmsFit]"}
    # config 5: detect_lines end to end (host image in, LineDetections out)
    img = workloads.line_image(4096, 4096, 64, 0.30, seed=0)
    params = lms.HoughParams.for_image(4096, 4096, 20.0, 20.0)
    lms.detect_lines(img, params, "lms", 64)
    walls = []
    for _ in range(reps):
        t0 = time.perf_counter()
        dets = lms.detect_lines(img, params, "lms", 64)
        walls.append(time.perf_counter() - t0)
    res["config5"] = {"workload": "detect_lines, 4096^2 image, 64 lines, 30% salt, 64 peaks, cap 256",
                      "e2e_ms": 1e3 * statistics.median(walls), "peaks": len(dets),
                      "lit_points": int((img >= 128).sum())}
    ctx.close()
    return res


# --------------------------------------------------------------------------- ours
def load_profile(name: str) -> dict:
    """ncu summary (scripts/ncu_summary.py) of one kernel on this workload."""
    path = os.path.join(ROOT, "profiles", name)
    try:
        with open(path) as fh:
            return json.load(fh)["launches"][0]
    except Exception:
        return {}


def run_ours(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # LMSB_DIST_BACKEND=gloo: a functional check of the N > 1 path with several
    # ranks sharing the visible GPUs (CPU collectives; its timings mean nothing)
    backend = os.environ.get("LMSB_DIST_BACKEND", "nccl")
    import torch as _t

    if backend != "nccl" and _t.cuda.device_count() > 0:
        local %= _t.cuda.device_count()
    import torch

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    coll_dev = torch.device("cuda", local) if backend == "nccl" else None
    from paper_1510_01041_b200 import _native, distributed, solve_lms
    from paper_1510_01041_b200.backend import record_from_native

    n = args.n
    pts, q = workload(n, args.seed)
    a, b = pts[:, 0].copy(), pts[:, 1].copy()
    total = n * (n - 1) // 2
    r0, r1 = distributed.partition(total, world, rank)

    ctx = _native.Context(local)
    ctx.upload(a, b)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=f"cuda:{local}")

    def step():
        if world > 1:  # sharded band search: band-table all_gather, record all_gather
            return distributed.solve_sharded(ctx, q, device=coll_dev)
        return record_from_native(ctx.solve(q, r0, r1))

    for _ in range(args.warmup):
        step()

    sampler = ClockSampler(local).start()
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    dev_ms = 0.0
    phase = {"ms_bound": 0.0, "ms_partition": 0.0, "ms_collect": 0.0, "ms_band_filter": 0.0}
    launches = 0
    survivors = 0
    band_stats = {}
    recs = []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        ctx.record(0)
        rec = step()
        ctx.record(1)
        dev_ms += ctx.elapsed_ms(0, 1)
        st = ctx.stats()
        for k in phase:
            phase[k] += st[k]
        launches += st["launches"]
        survivors += st["survivors"]
        band_stats = {k: st[k] for k in ("bands", "bands_searched", "filtered_vertices",
                                         "band_survivors", "survivors", "seed_height")}
        recs.append(rec)
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    clocks = sampler.stop()

    t_max = dev_ms
    if dist:
        tt = torch.tensor([dev_ms], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_max = float(tt.item())
    ms_per_step = t_max / args.steps
    value = args.steps * n * total / (t_max / 1e3)
    assert all(r == recs[0] for r in recs), "non-deterministic result across steps"

    # ---- e2e through the public API (host arrays in, LmsFit out), wall clock
    def e2e_once():
        if world == 1:
            return solve_lms(pts)
        from paper_1510_01041_b200.solver import fit_from_record, validated

        x, y, qq = validated(pts, None)
        return fit_from_record(x, y, qq, distributed.solve_distributed(x, y, qq))

    for _ in range(max(1, min(args.warmup, 3))):
        e2e_once()  # warm-up: the public API's shared context allocates on first use
    e2e_s = 0.0
    for _ in range(max(1, args.steps)):
        if dist:
            dist.barrier()
        t0 = time.perf_counter()
        fit = e2e_once()
        e2e_s += time.perf_counter() - t0
        assert fit.coverage == q
    if dist:
        tt = torch.tensor([e2e_s], dtype=torch.float64, device=coll_dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s = float(tt.item())
    e2e_value = max(1, args.steps) * n * total / e2e_s

    # ---- roofline of the dominant kernel: the collect pass, one test per
    # arrangement vertex; instruction-issue bound (no tensor-core or HBM
    # bound applies: its DRAM traffic is the collected list only, the lines
    # stay in L1/L2).  achieved = warp instructions per launch (ncu, same
    # workload, committed under profiles/) / live event time of the kernel.
    prof = load_profile("r01_collect_ncu.json")
    coll_ms = phase["ms_collect"] / args.steps
    sm_mhz = clocks.get("sm_mhz") or 1965.0
    sms = torch.cuda.get_device_properties(local).multi_processor_count
    peak = sms * 4 * sm_mhz * 1e6  # warp instructions / s: 4 schedulers per SM
    inst = prof.get("smsp__inst_executed.sum")
    pairs = r1 - r0
    if inst:  # the profile is of the whole-fit launch: scale to this rank's partition
        inst *= pairs / total
    achieved = inst / (coll_ms / 1e3) if inst and coll_ms > 0 else None
    traffic = None
    if prof.get("dram__bytes_read.sum") is not None:
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        traffic = (prof["dram__bytes_read.sum"] * scale.get(prof.get("dram__bytes_read.sum.unit"), 1)
                   + prof["dram__bytes_write.sum"] * scale.get(prof.get("dram__bytes_write.sum.unit"), 1))
    roofline = {
        "bound": "issue",
        "kernel": "band_collect_kernel (fp32 slope-run pre-test of every vertex, exact band of the "
                  "candidates)",
        "achieved": achieved,
        "peak": peak,
        "unit": "warp-instructions/s",
        "frac": achieved / peak if achieved else None,
        "traffic": traffic,
        "algorithmic": f"{pairs} vertex tests per launch ({pairs / (coll_ms / 1e3):.3e} vertices/s); "
                       "achieved = ncu smsp__inst_executed.sum of the launch (profiles/"
                       "r01_collect_ncu.json) / live CUDA-event time of the launch",
        "peak_source": f"{sms} SMs x 4 warp schedulers x 1 instruction/clk at the median SM clock "
                       "sampled during the timed region",
        "collect_share_of_step": coll_ms / ms_per_step if ms_per_step else None,
        "phase_ms_per_step": {k: v / args.steps for k, v in phase.items()},
        "reference_evals_per_step": n * total,
    }

    out = None
    if rank == 0:
        best = recs[0]
        out = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "time_to_fit_s": ms_per_step / 1e3,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic (workloads.contaminated_line_points, seed 0)",
            "config": config(n, world),
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 16 * n,
                    "d2h_bytes_per_step": 56 + (8 * 7 * world if world > 1 else 0),
                    "seconds_per_fit": e2e_s / max(1, args.steps),
                    "path": "solve_lms(points) -> LmsFit" if world == 1 else
                            "distributed.solve_distributed (sharded band search) + fit_from_record"},
            "gpu_launches": launches,
            "roofline": roofline,
            "clocks": clocks,
            "survivors_per_step": survivors / args.steps,
            "band_stage": band_stats,
            "result": {"i": best.i, "j": best.j, "height": best.height, "u": best.u},
        }
        if world == 1 and not args.no_extra:
            out["other_configs"] = other_configs(local)
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline(a, b, q, n, args.cpu_vertices_per_thread)
        print(json.dumps(out), flush=True)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())

#!/usr/bin/env python
"""SparseConv3d fwd+bwd throughput on B200 (BASELINE.json metric), plus the reference arm.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config cfg1..cfg5]

Workload (default, N=1): BASELINE.json configs[1] — the ScanNet-scale sphere shell
``sphere_shell_coords(470, band=1.5)`` (1,018,216 voxels, 21,229,376 kernel-map pairs), SparseConv3d 3×3×3
64→64, bf16 inputs / fp32 accumulation, forward + input gradient + weight gradient.  A "step" is one fwd+bwd
pass over that grid with inputs resident in HBM; the kernel map is built once outside the timed region (as the
reference's bench-conv, cli.py:353) and its build is reported separately (``stages``).

Multi-GPU (torchrun, one process per GPU, NCCL):
* cfg2: weak scaling — every rank runs its own cfg2 grid;
* cfg3: strong scaling — the 8 LiDAR grids are split across ranks by kernel-map pairs (dist.partition_by_cost),
  each rank builds its share as one jagged batch (one batched build, one batched kernel map);
* cfg5: strong scaling — the 19.4M-voxel grid's output rows are split at leaf boundaries (dist.RowShard);
every step ends with the sum all-reduce of the fp32 weight gradient, started right after the wgrad kernel and
overlapped with the input-gradient kernel.

Timing: W warm-up steps; K timed steps, each preceded by a 256 MB L2-flush write (untimed), timed with CUDA
events on the launching stream; ms_per_step = mean, max over ranks.  ``e2e`` is the same step through the public
API with host data: the features are copied host->device (pinned bf16; --e2e-dtype fp32) every step, the loss (½‖y‖², whose
gradient y seeds the backward) and the weight gradient are read back.  ``cpu_baseline`` times the reference
itself (the unmodified ``idxgrid`` package installed in baseline/_ref; the oracle port if it is absent) on a
leaf-aligned sample of the same workload.
"""

from __future__ import annotations

import argparse
import json
import os
import pathlib
import statistics
import sys
import threading
import time

# The reference arm (numpy + OpenBLAS) runs with every host thread the process may use.  torchrun exports
# OMP_NUM_THREADS=1 to each rank, which OpenBLAS reads when numpy loads, so override it before the import.
HOST_THREADS = len(os.sched_getaffinity(0))


def _reference_arm(argv) -> bool:
    for i, a in enumerate(argv):
        if a == "--impl=reference" or (a == "--impl" and i + 1 < len(argv) and argv[i + 1] == "reference"):
            return True
    return False


if _reference_arm(sys.argv):
    for _v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[_v] = str(HOST_THREADS)

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "SparseConv3d fwd+bwd active voxels/s & TFLOPS at 1/2/4/8 B200 vs CPU ref"
UNIT = "voxels/s"
PEAKS_FILE = ROOT / "MEASURED_PEAKS.json"
TRAFFIC_FILE = ROOT / "profiles" / "ncu_traffic.json"
REF_DIR = ROOT / "baseline" / "_ref"

CONFIGS = {
    "cfg1": dict(desc="single GridBatch from a random 100k-point cloud (sigma 1, voxel 0.05), SparseConv3d 3x3x3 "
                      "32->32 fp32 forward (CUDA-core exact path)", points=True, cin=32, cout=32, fp32_fwd=True),
    "cfg2": dict(desc="ScanNet-scale sphere shell sphere_shell_coords(470, band=1.5), SparseConv3d 3x3x3 64->64 "
                      "bf16 fwd+bwd", res=470, cin=64, cout=64, scaling="weak"),
    "cfg3": dict(desc="batch of 8 simulated KITTI-scale LiDAR grids (seeds 0-7, 128 beams x 2048 azimuths, voxel "
                      "0.05 m), SparseConv3d 3x3x3 128->128 bf16 fwd+bwd, batch-sharded across ranks by kernel-map "
                      "pairs", lidar=8, cin=128, cout=128, scaling="strong"),
    "cfg4": dict(desc="sparse U-Net stage: build from jagged points (cfg2 shell as f64 voxel centres), coarsen, "
                      "stride-2 conv 64->128 + transposed conv 128->64, fwd+bwd, bf16", res=470, cin=64, cout=128,
                 unet=True),
    # the reference's dense-window regime (leaf / brick schedules): fully occupied blocks
    "dense32": dict(desc="dense 160^3 block (4.1M voxels, 100% leaf occupancy), SparseConv3d 3x3x3 32->32 bf16 fwd+bwd",
                    dense=160, cin=32, cout=32, scaling="weak"),
    "dense64": dict(desc="dense 128^3 block (2.1M voxels, 100% leaf occupancy), SparseConv3d 3x3x3 64->64 bf16 fwd+bwd",
                    dense=128, cin=64, cout=64, scaling="weak"),
    "dense128": dict(desc="dense 96^3 block (0.88M voxels, 100% leaf occupancy), SparseConv3d 3x3x3 128->128 bf16 "
                          "fwd+bwd", dense=96, cin=128, cout=128, scaling="weak"),
    "cfg5": dict(desc="2048^3 surface shell sphere_shell_coords(2048, band=1.5), SparseConv3d 3x3x3 32->32 bf16 "
                      "fwd+bwd, output rows sharded across ranks at leaf boundaries", res=2048, cin=32, cout=32,
                 rowshard=True, scaling="strong"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=None)
    ap.add_argument("--e2e-dtype", default="bf16", choices=["bf16", "fp32"],
                    help="host dtype of the features the e2e step uploads (bf16: the config's compute dtype)")
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def peaks():
    try:
        return json.loads(PEAKS_FILE.read_text())
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "_fallback": True}


# ----------------------------------------------------------------------------- inputs

def make_coords(cfg, rank):
    from paper_2407_01781_b200.workloads import random_points, sphere_shell_coords
    if cfg.get("points"):
        return None, random_points(np.random.default_rng(rank), 100_000, sigma=1.0)
    if cfg.get("dense"):
        r = np.arange(cfg["dense"])
        return np.stack(np.meshgrid(r, r, r, indexing="ij"), -1).reshape(-1, 3), None
    return sphere_shell_coords(cfg["res"], band=1.5), None


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """NVML sampling of SM clock + clocks-event reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x1: "gpu_idle"}

    def __init__(self, index, interval=float(os.environ.get("FVDB_CLOCK_INTERVAL", "0.005"))):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self.interval = interval
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
        self.t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
            except Exception:
                pass
            time.sleep(self.interval)

    def __enter__(self):
        if self.nv is not None:
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        reasons = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": reasons, "samples": len(self.samples)}


# ----------------------------------------------------------------------------- timing helpers

def stage(torch, fn, reps=1):
    """(result, device ms from CUDA events on the current stream, wall ms incl. host work and syncs): best of reps.
    With reps > 1 the previous result is released before each repetition, so the repetitions after the first
    run with a warm caching allocator (a training loop's steady state); the first includes any cudaMalloc."""
    best = None
    res = None
    for _ in range(reps):
        res = None
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record()
        res = fn()
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) * 1e3
        dev = e0.elapsed_time(e1)
        if best is None or dev < best[0]:
            best = (dev, wall)
    return res, round(best[0], 4), round(best[1], 4)


def max_over_ranks(torch, dist, dev, v, use_dist):
    if not use_dist:
        return v
    t = torch.tensor([v], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(torch, dist, dev, v, use_dist):
    if not use_dist:
        return v
    t = torch.tensor([v], device=dev, dtype=torch.float64)
    dist.all_reduce(t)
    return float(t.item())


# ----------------------------------------------------------------------------- problem setup (per config)

def setup_problem(args, cfg, rank, world, dev, torch, P):
    """This rank's share of the workload: tables, inputs and the stage measurements of building them."""
    from paper_2407_01781_b200 import dist as D
    stages = {}
    if cfg.get("lidar"):
        from paper_2407_01781_b200.workloads import lidar_scan_points
        pts = [lidar_scan_points(s) for s in range(cfg["lidar"])]
        tf = P.VoxelTransform.uniform(0.05)
        # partition the batch by kernel-map pairs (the same on every rank; setup, untimed)
        full, _ = P.build_from_points(P.jagged_from_list([torch.from_numpy(p) for p in pts]), tf)
        kfull = P.build_batch_kernel_map(full, full, 1)
        costs = [int((kfull.fwd.t[:, s:e] >= 0).sum().item()) for s, e in full.voxel_joffsets.tolist()]
        s, e = D.partition_by_cost(costs, world)[rank]
        del full, kfull
        jag = P.jagged_from_list([torch.from_numpy(p).to(dev) for p in pts[s:e]])  # points resident, as cfg2's coords
        batch, dv, wl = stage(torch, lambda: P.build_from_points(jag, tf)[0], reps=3)
        stages["grid_build"] = dict(device_ms=dv, wall_ms=wl, inputs=int(jag.jdata.shape[0]), grids=e - s,
                                    batched=True)
        km, dv, wl = stage(torch, lambda: P.build_batch_kernel_map(batch, batch, 1), reps=3)
        stages["kernel_map"] = dict(device_ms=dv, wall_ms=wl, batched=True)
        n = batch.total_voxels
        return dict(t_fwd=km.fwd, t_dgrad=km.bwd, n_in=n, n_out=n, rows=slice(0, n), pairs=km.total_pairs, km=km,
                    batch=batch, leaves=sum(g.num_leaf_nodes for g in batch.grids), units=n,
                    share=f"grids {s}..{e - 1} of {len(pts)}"), stages
    coords, _ = make_coords(cfg, rank if cfg.get("scaling") == "weak" else 0)
    c_dev = torch.from_numpy(coords).to(dev)
    grid, dv, wl = stage(torch, lambda: P.build_from_coords(c_dev)[0], reps=3)
    stages["grid_build"] = dict(device_ms=dv, wall_ms=wl, inputs=int(coords.shape[0]), grids=1, batched=False)
    if cfg.get("rowshard"):
        r0, r1, l0, l1 = D.leaf_aligned_ranges(grid.leaf_value_offset, grid.num_voxels, world)[rank]
        sh, dv, wl = stage(torch, lambda: D.RowShard(grid, r0, r1, l0, l1), reps=3)
        stages["kernel_map"] = dict(device_ms=dv, wall_ms=wl, rows=f"[{r0}, {r1})")
        n = grid.num_voxels
        return dict(t_fwd=sh.fwd, t_dgrad=sh.dgrad, n_in=n, n_out=r1 - r0, rows=slice(r0, r1), pairs=sh.total_pairs,
                    shard=sh, grid=grid, leaves=l1 - l0, units=r1 - r0,
                    share=f"rows [{r0}, {r1}) of {n} (leaves [{l0}, {l1}))"), stages
    km, dv, wl = stage(torch, lambda: P.build_kernel_map(grid, grid, 1), reps=3)
    stages["kernel_map"] = dict(device_ms=dv, wall_ms=wl)
    n = grid.num_voxels
    return dict(t_fwd=km.fwd, t_dgrad=km.bwd, n_in=n, n_out=n, rows=slice(0, n), pairs=km.total_pairs, km=km,
                grid=grid, leaves=grid.num_leaf_nodes, units=n, share="whole grid"), stages


def stage_rooflines(stages, prob, pk):
    """Algorithmic bytes and fraction of measured HBM bandwidth of the map / grid stages."""
    hbm = pk["hbm_gbs"]
    out = {}
    gb = stages["grid_build"]
    # read 24 B per int64 input coordinate; write the leaf payload (80 B record + 8 B key + 24 B origin)
    gbytes = 24 * gb["inputs"] + (80 + 8 + 24) * prob["leaves"]
    out["grid_build"] = dict(gb, algorithmic_bytes=gbytes,
                             achieved_gbs=round(gbytes / (gb["device_ms"] * 1e-3) / 1e9, 1),
                             frac_hbm=round(gbytes / (gb["device_ms"] * 1e-3) / 1e9 / hbm, 4),
                             host_overhead_ms=round(gb["wall_ms"] - gb["device_ms"], 3))
    km = stages["kernel_map"]
    # read 24 B per output coordinate, write the int32 neighbour table (27 x 4 B per output row)
    kbytes = (24 + 27 * 4) * prob["n_out"]
    out["kernel_map"] = dict(km, algorithmic_bytes=kbytes,
                             achieved_gbs=round(kbytes / (km["device_ms"] * 1e-3) / 1e9, 1),
                             frac_hbm=round(kbytes / (km["device_ms"] * 1e-3) / 1e9 / hbm, 4),
                             host_overhead_ms=round(km["wall_ms"] - km["device_ms"], 3))
    for k, v in stages.items():
        if k not in out:
            out[k] = v
    return out


# ----------------------------------------------------------------------------- our arm

def run_ours(args, rank, world, local_rank):
    cfg = CONFIGS[args.config]
    if cfg.get("fp32_fwd") or cfg.get("unet"):
        return run_special(args, rank, world, local_rank, cfg)
    import torch
    import torch.distributed as dist

    import paper_2407_01781_b200 as P
    from paper_2407_01781_b200.conv import conv_impl, gather_conv, pack_weights_umma, steady_impl, wgrad

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    cin, cout = cfg["cin"], cfg["cout"]
    use_dist = world > 1
    pk = peaks()

    prob, stages = setup_problem(args, cfg, rank, world, dev, torch, P)
    t_fwd, t_dgrad = prob["t_fwd"], prob["t_dgrad"]
    n_in, n_out, rows, pairs = prob["n_in"], prob["n_out"], prob["rows"], prob["pairs"]

    # per-table preprocessing (cached on the tables, outside the timed step): the kernels "auto" settles on for a
    # reused map (conv.steady_impl: the halo kernel, or the sorted gather for sparse wide layers).
    forced = conv_impl()

    def steady(tab, k, n):
        return (forced, False) if forced != "auto" else steady_impl(tab, k, n)

    impl_f, sorted_f = steady(t_fwd, cin, cout)
    impl_b, sorted_b = steady(t_dgrad, cout, cin)
    from paper_2407_01781_b200 import _lib as _L
    from paper_2407_01781_b200.conv import HaloPlan
    for name, tab, k, n, on in (("halo_plan_fwd", t_fwd, cin, cout, impl_f == "halo"),
                                ("halo_plan_dgrad", t_dgrad, cout, cin, impl_b == "halo")):
        if on and getattr(tab, "rev_src", None) is not None and _L.lib().fvdb_halo_reversed_ok(k, n) and \
                os.environ.get("FVDB_PLAN_SHARE", "1") != "0":
            stages[name] = dict(device_ms=0.0, wall_ms=0.0, shared="the forward plan, run with offsets reversed")
            continue
        if on:  # steady state (warm allocator: a loop that rebuilds its maps), then cache the table's own plan
            cap = int(_L.lib().fvdb_halo_cap(k, n))
            _, dv, wl = stage(torch, lambda: HaloPlan(tab, cap), reps=3)
            stages[name] = dict(device_ms=dv, wall_ms=wl)
            tab.halo_plan(k, n)
    for name, fn in (("sort_fwd", lambda: t_fwd.signature_sorted() if sorted_f else None),
                     ("sort_dgrad", lambda: t_dgrad.signature_sorted() if sorted_b else None)):
        _, dv, wl = stage(torch, fn)
        if dv > 0.05 or wl > 0.05:
            stages[name] = dict(device_ms=dv, wall_ms=wl, note="first use (cold allocator)")
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    x = torch.randn(n_in, cin, device=dev, generator=gen).to(torch.bfloat16)
    # a row shard's input gradient reads grad_out of every row; its weight gradient only its own rows
    gy = torch.randn(n_in if cfg.get("rowshard") else n_out, cout, device=dev, generator=gen).to(torch.bfloat16)
    gy_rows = gy[rows] if cfg.get("rowshard") else gy
    w = torch.randn(cout, cin, 3, 3, 3, device=dev, generator=gen) / (27 * cin) ** 0.5
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    for _ in range(3):  # reach the steady kernels of every table (halo / sorted gather / pair-list wgrad)
        gather_conv(x, t_fwd, w)
        gather_conv(gy, t_dgrad, w, transpose=True)
        wgrad(x, gy_rows, t_fwd)

    def step(ev=None):
        img_f = pack_weights_umma(w, False, impl_f)
        img_b = pack_weights_umma(w, True, impl_b)
        if ev is not None:
            ev[0].record()
        y = gather_conv(x, t_fwd, w, transpose=False, out_dtype=torch.bfloat16, w_image=img_f)
        if ev is not None:
            ev[1].record()
        gw = wgrad(x, gy_rows, t_fwd)
        if ev is not None:
            ev[2].record()
        h = dist.all_reduce(gw, async_op=True) if use_dist else None  # overlaps the dgrad kernel
        gx = gather_conv(gy, t_dgrad, w, transpose=True, out_dtype=torch.bfloat16, w_image=img_b)
        if ev is not None:
            ev[3].record()
        if h is not None:
            h.wait()
        if ev is not None:
            ev[4].record()
        return y, gx, gw

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(args.steps)]
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            flush.fill_(k & 0xFF)          # untimed L2 flush (256 MB > 126 MB L2)
            starts[k].record()
            step(evs[k])
        torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    torch.cuda.synchronize()
    step_ms = [s.elapsed_time(e[4]) for s, e in zip(starts, evs)]
    phase = {"fwd": [e[0].elapsed_time(e[1]) for e in evs], "wgrad": [e[1].elapsed_time(e[2]) for e in evs],
             "dgrad": [e[2].elapsed_time(e[3]) for e in evs], "allreduce_tail": [e[3].elapsed_time(e[4]) for e in evs],
             "pack": [s.elapsed_time(e[0]) for s, e in zip(starts, evs)]}
    ms = max_over_ranks(torch, dist, dev, statistics.mean(step_ms), use_dist)
    total_units = int(sum_over_ranks(torch, dist, dev, prob["units"], use_dist))
    total_pairs = int(sum_over_ranks(torch, dist, dev, pairs, use_dist))
    value = total_units / (ms / 1e3)

    # ---- fresh-map step (cfg2, rank-local): build + kernel map + first-use kernels (no halo plan) ----
    fresh = run_fresh(torch, P, dev, x, gy, w) if args.config == "cfg2" else None
    # ---- schedules side by side (the reference's igemm vs its dense-window leaf / brick regime) ----
    schedules = compare_schedules(torch, flush, x, t_fwd, w) if cfg.get("dense") or args.config == "cfg2" else None

    # ---- end-to-end through the public API with host data ----
    e2e = run_e2e(args, cfg, P, torch, dist, prob, cin, cout, dev, use_dist, world)

    # ---- roofline of the dominant kernel ----
    flops_kernel = 2.0 * pairs * cin * cout
    means = {k: statistics.mean(v) for k, v in phase.items()}
    dom = max(("fwd", "dgrad", "wgrad"), key=lambda k: means[k])
    achieved = flops_kernel / (means[dom] / 1e3) / 1e12
    traffic = None
    try:
        tr = json.loads(TRAFFIC_FILE.read_text())
        traffic = tr.get(args.config, {}).get(dom)
    except Exception:
        pass
    from paper_2407_01781_b200.conv import halo_kernel_name
    fk = halo_kernel_name(cin, cout) if impl_f == "halo" else f"k_conv_fwd_tc<{cin},{cout},bf16>"
    dk = (f"{halo_kernel_name(cout, cin)} (dgrad)" if impl_b == "halo"
          else f"k_conv_fwd_tc<{cout},{cin},bf16> (dgrad form)")
    wk = "k_wgrad_pairs" if t_fwd._pairs is not None else f"k_wgrad_tc<{cin},{cout}>"
    roof = {"bound": "tensor", "kernel": {"fwd": fk, "dgrad": dk, "wgrad": wk}[dom],
            "achieved": round(achieved, 2), "peak": pk["bf16_tflops"], "unit": "TFLOP/s",
            "frac": round(achieved / pk["bf16_tflops"], 4), "traffic": traffic,
            "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst)" if not pk.get("_fallback") else "fallback",
            "algorithmic_flop_per_launch": flops_kernel}
    # HBM view of the same launch (both fractions near the ridge, e.g. cfg5 at 32 channels):
    # features in + features out (bf16) + the int32 neighbour table
    k_, n_ = (cout, cin) if dom == "dgrad" else (cin, cout)
    hbm_bytes = 2 * (n_in * k_ + n_out * n_) + 27 * 4 * n_out
    roof["hbm"] = {"algorithmic_bytes": hbm_bytes, "achieved_gbs": round(hbm_bytes / (means[dom] / 1e3) / 1e9, 1),
                   "peak_gbs": pk["hbm_gbs"], "frac": round(hbm_bytes / (means[dom] / 1e3) / 1e9 / pk["hbm_gbs"], 4)}
    step_tflops = 3 * 2.0 * total_pairs * cin * cout / (ms / 1e3) / 1e12

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(cfg, args)

    if rank == 0:
        how = ("batch-sharded" if cfg.get("lidar") else "row-sharded" if cfg.get("rowshard") else "one grid per rank")
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": cfg.get("scaling", "weak"), "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "voxels_total": total_units,
                       "pairs_total": total_pairs, "rank0_share": prob["share"], "cin": cin, "cout": cout,
                       "parallelism": (f"dp{world} ({how}, NCCL wgrad all-reduce overlapped with dgrad)"
                                       if world > 1 else "single GPU"),
                       "l2": "flushed (256 MB write) before every timed step",
                       "kernel_map": "prebuilt outside the timed step (reference cli.py:353); see stages",
                       "conv_kernel": {"fwd": impl_f + (" (signature-sorted)" if sorted_f else ""),
                                       "dgrad": impl_b + (" (signature-sorted)" if sorted_b else ""),
                                       "wgrad": "pair lists" if t_fwd._pairs is not None else "table"}},
            "tflops_effective": round(step_tflops, 2),
            "frac_of_bf16_peak": round(step_tflops / pk["bf16_tflops"], 4),
            "phases_ms": {k: round(v, 4) for k, v in means.items()},
            "stages": stage_rooflines(stages, prob, pk),
            "roofline": roof,
            "e2e": e2e,
            "gpu_launches": 6 * args.steps,
            "clocks": clk.summary(),
        }
        if fresh is not None:
            line["fresh_map_step"] = fresh
        if schedules is not None:
            line["schedules_fwd_ms"] = schedules
        if cpu is not None:
            line["cpu_baseline"] = cpu
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


def compare_schedules(torch, flush, x, table, w, reps=10):
    """Forward time of the gather kernel (igemm schedule: every pair's row gathered from L2) and of the halo
    kernel (dense-window schedule: each tile's neighbourhood staged once), median of reps with L2 flushes."""
    from paper_2407_01781_b200.conv import gather_conv, pack_weights_umma
    out = {}
    for impl in ("gather", "halo"):
        img = pack_weights_umma(w, False, impl)
        gather_conv(x, table, w, w_image=img, impl=impl)
        ts = []
        for _ in range(reps):
            flush.fill_(3)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            gather_conv(x, table, w, w_image=img, impl=impl)
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        out[{"gather": "igemm (gather kernel)", "halo": "leaf/brick (halo kernel)"}[impl]] = round(sorted(ts)[reps // 2], 4)
    v = list(out.values())
    out["speedup"] = round(v[0] / v[1], 3)
    return out


def run_fresh(torch, P, dev, x, gy, w):
    """A step on a map seen for the first time (a training loop that rebuilds grids per batch): grid build,
    kernel map, transposed table and fwd + dgrad + wgrad with the kernels `auto` picks for a new map."""
    from paper_2407_01781_b200.conv import gather_conv, wgrad
    from paper_2407_01781_b200.workloads import sphere_shell_coords
    c = torch.from_numpy(sphere_shell_coords(470, band=1.5)).to(dev)

    def one():
        g, _ = P.build_from_coords(c)
        km = P.build_kernel_map(g, g, 1)
        gather_conv(x, km.fwd, w)
        gather_conv(gy, km.bwd, w, transpose=True)
        wgrad(x, gy, km.fwd)

    one()
    best = None
    for _ in range(3):
        _, dv, wl = stage(torch, one)
        if best is None or wl < best[0]:
            best = (wl, dv)
    return {"wall_ms": round(best[0], 3), "device_ms": round(best[1], 3),
            "what": "build_from_coords + build_kernel_map + transposed table + fwd/dgrad/wgrad as the auto policy runs a "
                    "map's first step (same-grid map: the halo kernel with one plan shared by fwd and dgrad)"}


def run_special(args, rank, world, local_rank, cfg):
    """cfg1 (fp32 forward, exact path) and cfg4 (U-Net stage incl. grid build) — timed like the main arm."""
    import torch
    import torch.distributed as dist

    import paper_2407_01781_b200 as P
    from paper_2407_01781_b200.conv import gather_conv
    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    use_dist = world > 1
    coords, points = make_coords(cfg, rank)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)
    pk = peaks()
    extra = {}
    if cfg.get("fp32_fwd"):
        grid, _ = P.build_from_points(points, P.VoxelTransform.uniform(0.05))
        km = P.build_kernel_map(grid, grid, 1)
        x = torch.randn(grid.num_voxels, cfg["cin"], device=dev, generator=gen)
        w = torch.randn(cfg["cout"], cfg["cin"], 3, 3, 3, device=dev, generator=gen) / (27 * cfg["cin"]) ** 0.5
        n_vox, pairs = grid.num_voxels, km.total_pairs
        flops = 2.0 * pairs * cfg["cin"] * cfg["cout"]

        def step():
            return gather_conv(x, km.fwd, w)
        ffma = ffma_peak(torch)
        if ffma:
            extra["fp32_simt_peak_tflops"] = ffma
    else:
        pts = torch.from_numpy(coords.astype(np.float64)).to(dev)        # jagged points, B=1, on device
        tf = P.VoxelTransform.uniform(1.0)
        down = P.SparseConv3d(64, 128, stride=2).to(dev)
        up = P.SparseConv3d(128, 64, stride=2, transposed=True).to(dev)
        n_vox = coords.shape[0]
        x = torch.randn(n_vox, 64, device=dev, generator=gen).to(torch.bfloat16)  # bf16 features (compute dtype)
        if use_dist:
            P.dist.attach_grad_reducer(down)
            P.dist.attach_grad_reducer(up)

        def step():
            g, _ = P.build_from_points(pts, tf)
            fine = P.GridBatch([g])
            coarse, h = down(fine, fine.jagged(x))
            _, y = up(coarse, h, out_grid=fine)
            y.jdata.sum(dtype=torch.float32).backward()  # fp32 accumulation, no fp32 copy of y
            return y

        g0, _ = P.build_from_points(pts, tf)
        k2 = P.build_kernel_map(g0, P.coarsen(g0, 2), 2)
        pairs = k2.total_pairs
        flops = 2 * 6.0 * pairs * 64 * 128   # s2 conv fwd+bwd and transposed fwd+bwd (2 x 3 GEMMs)
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local_rank) as clk:
        for a, b in ev:
            flush.fill_(1)
            a.record()
            step()
            b.record()
        torch.cuda.synchronize()
    ms = max_over_ranks(torch, dist, dev, statistics.mean(a.elapsed_time(b) for a, b in ev), use_dist)
    if rank == 0:
        tfl = flops / (ms / 1e3) / 1e12
        line = {
            "metric": METRIC, "value": round(n_vox * world / (ms / 1e3), 1), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32" if cfg.get("fp32_fwd") else "bf16",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "voxels_per_gpu": n_vox, "pairs": pairs,
                       "l2": "flushed (256 MB write) before every timed step",
                       "step": "forward only" if cfg.get("fp32_fwd") else "build+coarsen+kmaps+fwd+bwd"},
            "tflops_effective": round(tfl, 3),
            "frac_of_bf16_peak": None if cfg.get("fp32_fwd") else round(tfl / pk["bf16_tflops"], 4),
            "clocks": clk.summary(),
        }
        if extra.get("fp32_simt_peak_tflops"):
            line["roofline"] = {"bound": "fp32 SIMT", "achieved": round(tfl, 3),
                                "peak": extra["fp32_simt_peak_tflops"], "unit": "TFLOP/s",
                                "frac": round(tfl / extra["fp32_simt_peak_tflops"], 4),
                                "peak_source": "fvdb_probe_ffma (FFMA microbenchmark, this run)"}
        print(json.dumps(line), flush=True)
    if use_dist:
        dist.barrier()
        dist.destroy_process_group()


def ffma_peak(torch):
    """FP32 FFMA throughput of this GPU (TFLOP/s), from the library's probe kernel."""
    import ctypes as C
    from paper_2407_01781_b200 import _lib
    L = _lib.lib()
    out = torch.empty(1 << 20, dtype=torch.float32, device="cuda")
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        flop = C.c_double(0)
        e0.record()
        _lib.check(L.fvdb_probe_ffma(4096, out.data_ptr(), out.numel(), C.byref(flop), _lib.stream_ptr()),
                   "probe_ffma")
        e1.record()
        torch.cuda.synchronize()
        t = flop.value / (e0.elapsed_time(e1) * 1e-3) / 1e12
        best = t if best is None else max(best, t)
    return round(best, 2)


def run_e2e(args, cfg, P, torch, dist, prob, cin, cout, dev, use_dist, world):
    """The same step through the public API with host data, every copy inside the timed region.

    Each step uploads that step's features from pinned host memory (bf16, the configs' compute dtype, as a
    training pipeline would keep them; ``--e2e-dtype fp32`` uploads fp32 and casts on the device), runs
    SparseConv3d forward (or, for a
    row shard, dist.RowShard.forward), takes the loss ½‖y‖² (its gradient, y itself, seeds the backward: dgrad +
    wgrad) and reads the loss and the fp32 weight gradient back to the host.  As a training loop with a
    prefetching loader would, step k+1's features upload on a copy stream during step k (double-buffered,
    ordered by events).  Row shards (cfg5) upload only their own rows and all-gather the features and the
    output gradient over NCCL (the exchange a row-sharded layer needs).
    """
    steps = args.e2e_steps or max(3, min(args.steps, 50))
    rng = np.random.default_rng(7)
    main = torch.cuda.current_stream(dev)
    s_in = torch.cuda.Stream(dev)
    rowshard = cfg.get("rowshard")
    n_up = (prob["rows"].stop - prob["rows"].start) if rowshard else prob["n_in"]
    hdt = torch.bfloat16 if args.e2e_dtype == "bf16" else torch.float32
    x_h = [torch.from_numpy(rng.normal(size=(n_up, cin)).astype(np.float32)).to(hdt).pin_memory() for _ in range(2)]
    x_d = [torch.empty((n_up, cin), dtype=hdt, device=dev) for _ in range(2)]
    loss_h = torch.empty(2, dtype=torch.float32).pin_memory()
    gw_h = torch.empty((cout, cin, 3, 3, 3), dtype=torch.float32).pin_memory()
    ev_in = [torch.cuda.Event() for _ in range(2)]
    ev_used = [torch.cuda.Event() for _ in range(2)]
    for e in ev_used:
        e.record(main)
    if rowshard:
        sh = prob["shard"]
        w = torch.randn(cout, cin, 3, 3, 3, device=dev) / (27 * cin) ** 0.5
        n_all = prob["n_in"]
        x_full = torch.empty((n_all, cin), dtype=torch.bfloat16, device=dev)
        gy_full = torch.empty((n_all, cout), dtype=torch.bfloat16, device=dev)
        # leaf-aligned shards differ in rows: all_gather into per-rank slices of the full tensor
        if use_dist:
            t = torch.tensor([n_up], device=dev, dtype=torch.int64)
            allc = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(allc, t)
            counts = [int(c.item()) for c in allc]
        else:
            counts = [n_up]
        starts = np.concatenate([[0], np.cumsum(counts)]).astype(int).tolist()

        def gather_rows(local, full):
            if not use_dist:
                full.copy_(local)
                return
            dist.all_gather([full[starts[r]:starts[r + 1]] for r in range(world)], local.contiguous())

        def compute(k):
            b = k % 2
            main.wait_event(ev_in[b])
            xl = x_d[b].to(torch.bfloat16)
            ev_used[b].record(main)
            gather_rows(xl, x_full)
            y = sh.forward(x_full, w, out_dtype=torch.bfloat16)
            loss = 0.5 * torch.linalg.vector_norm(y, dtype=torch.float32) ** 2
            gather_rows(y, gy_full)                       # d loss / d y = y
            gw = sh.weight_grad(x_full, y)
            h = dist.all_reduce(gw, async_op=True) if use_dist else None
            sh.input_grad(gy_full, w, out_dtype=torch.bfloat16)
            if h is not None:
                h.wait()
            loss_h[b:b + 1].copy_(loss.reshape(1), non_blocking=True)
            gw_h.copy_(gw, non_blocking=True)
        api = "paper_2407_01781_b200.dist.RowShard forward / weight_grad / input_grad + NCCL all-gathers"
    else:
        m = P.SparseConv3d(cin, cout).to(dev)
        if use_dist:
            P.dist.attach_grad_reducer(m)
        gb = prob.get("batch") or P.as_grid_batch(prob["grid"])
        from paper_2407_01781_b200.conv import cache_batch_kernel_map
        cache_batch_kernel_map(gb, gb, 1, prob["km"])

        def compute(k):
            b = k % 2
            main.wait_event(ev_in[b])
            m.weight.grad = None
            x = x_d[b].detach().requires_grad_(True)
            _, y = m(gb, gb.jagged(x))
            loss = 0.5 * torch.linalg.vector_norm(y.jdata, dtype=torch.float32) ** 2
            y.jdata.backward(y.jdata.detach())            # d loss / d y = y
            ev_used[b].record(main)
            loss_h[b:b + 1].copy_(loss.detach().reshape(1), non_blocking=True)
            gw_h.copy_(m.weight.grad, non_blocking=True)
        api = "paper_2407_01781_b200.SparseConv3d (autograd) fwd + bwd"

    def upload(k):
        b = k % 2
        with torch.cuda.stream(s_in):
            s_in.wait_event(ev_used[b])  # step k-2 no longer reads buffer b
            x_d[b].copy_(x_h[b], non_blocking=True)
            ev_in[b].record(s_in)

    def run(nsteps):
        upload(0)
        for k in range(nsteps):
            if k + 1 < nsteps:
                upload(k + 1)
            compute(k)

    run(2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(main)
    s_in.wait_stream(main)
    run(steps)
    e1.record(main)
    torch.cuda.synchronize()
    ms = max_over_ranks(torch, dist, dev, e0.elapsed_time(e1) / steps, use_dist)
    units = int(sum_over_ranks(torch, dist, dev, prob["units"], use_dist))
    h2d = x_h[0].numel() * x_h[0].element_size()
    d2h = 4 + gw_h.numel() * 4
    return {"value": round(units / (ms / 1e3), 1), "unit": UNIT, "ms_per_step": round(ms, 4),
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h), "steps": steps, "api": api,
            "step": f"upload {args.e2e_dtype} features (pinned) -> forward -> loss 0.5*|y|^2 -> backward (dgrad + wgrad"
                    + (", NCCL all-reduce" if use_dist else "") + ") -> read back loss + fp32 weight gradient",
            "pipeline": "features of step k+1 uploaded on a copy stream during step k; every copy inside the "
                        "timed region"}


# ----------------------------------------------------------------------------- CPU: the reference itself

def _reference_module():
    """The unmodified reference package (baseline/_ref, pip-installed from /root/reference/pkg), or None."""
    if REF_DIR.is_dir() and str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    try:
        import idxgrid
        return idxgrid
    except Exception:
        return None


def _cpu_problem(cfg, frac):
    """The grid and the kernel map of a leaf-aligned prefix of ~frac of its output rows; (kind, n, lim, pairs,
    run(features, weights, grad_out))."""
    ig = _reference_module()
    if cfg.get("lidar"):
        from paper_2407_01781_b200.workloads import lidar_scan_points
        src = ("points", lidar_scan_points(0), 0.05)
    else:
        coords, points = make_coords(cfg, 0)
        src = ("points", points, 0.05) if points is not None else ("coords", coords, None)
    if ig is not None:
        from idxgrid.conv import STENCIL, KernelMap
        if src[0] == "points":
            g, _ = ig.build_from_points(src[1], ig.VoxelTransform.uniform(src[2]))
        else:
            g, _ = ig.build_from_coords(src[1])
        n = g.num_voxels
        starts = np.asarray(g.leaf_value_offset, np.int64) - 1
        i = int(np.searchsorted(starts, int(n * frac)))
        lim = int(starts[i]) if 0 < i < len(starts) else n
        out_coords = g.active_coords()[:lim]
        rows = np.arange(lim, dtype=np.int64)
        ins, outs = [], []
        for d in STENCIL:  # the reference's build_kernel_map (conv.py:105-122) restricted to the sample rows
            idx = g.coord_to_index_many(out_coords + d)
            sel = idx > 0
            ins.append(idx[sel] - 1)
            outs.append(rows[sel])
        km = KernelMap(ins, outs, n, lim, 1)

        def run(f, w, go):
            ig.conv(g, f, w, kmap=km, variant="igemm")
            ig.conv_backward(km, go, f, w)
        return "reference", n, lim, sum(len(o) for o in outs), run
    import oracle as O
    if src[0] == "points":
        g = O.build_from_points(src[1], [src[2]] * 3, [0.0] * 3)
    else:
        g = O.build_from_coords(src[1])
    ins, outs = O.kernel_map(g, g, 1)
    n = g.num_voxels
    lim = max(1, int(n * frac))
    si, so = [], []
    for a, b in zip(ins, outs):
        k = np.searchsorted(b, lim)
        si.append(a[:k])
        so.append(b[:k])

    def run(f, w, go):
        O.conv_igemm(f, w, si, so, lim)
        O.conv_backward(si, so, go, f, w)
    return "port", n, lim, sum(len(o) for o in so), run


def _cpu_inputs(n, lim, cin, cout):
    rng = np.random.default_rng(0)  # cli.py:349-352
    f = rng.normal(size=(n, cin)).astype(np.float32)
    w = (rng.normal(size=(cout, cin, 3, 3, 3)) / np.sqrt(27 * cin)).astype(np.float32)
    go = rng.normal(size=(lim, cout)).astype(np.float32)
    return f, w, go


def _cpu_what(kind):
    return ("idxgrid.conv(variant='igemm') + idxgrid.conv_backward, the unmodified reference (baseline/_ref)"
            if kind == "reference" else "oracle port of reference conv.py:180-191, 339-368")


def cpu_baseline(cfg, args, frac=1 / 8, repeats=2):
    """The reference's igemm conv + conv_backward on the host cores, on a leaf-aligned 1/8 of the grid."""
    kind, n, lim, pairs, run = _cpu_problem(cfg, frac)
    f, w, go = _cpu_inputs(n, lim, cfg["cin"], cfg["cout"])
    best = float("inf")
    for _ in range(repeats):
        t0 = time.perf_counter()
        run(f, w, go)
        best = min(best, time.perf_counter() - t0)
    return {"value": round(lim / best, 1), "unit": UNIT, "cores": HOST_THREADS, "kind": kind,
            "sample": f"first {lim} of {n} output voxels (leaf-aligned prefix, {lim / n:.3f} of the grid), {pairs} "
                      f"pairs; fp32 {_cpu_what(kind)}; best of {repeats}",
            "seconds_per_sample": round(best, 4)}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU path on the host cores (rank 0 only; other ranks exit)."""
    if rank != 0:
        return
    cfg = CONFIGS[args.config]
    frac = 1 / 8 if args.steps + args.warmup <= 30 else 1 / 32
    kind, n, lim, pairs, run = _cpu_problem(cfg, frac)
    f, w, go = _cpu_inputs(n, lim, cfg["cin"], cfg["cout"])
    for _ in range(args.warmup):
        run(f, w, go)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run(f, w, go)
        times.append(time.perf_counter() - t0)
    ms = statistics.mean(times) * 1e3
    value = lim / (ms / 1e3)
    sample = f"first {lim} of {n} output voxels (leaf-aligned prefix, {lim / n:.3f}), {pairs} pairs; fp32 {_cpu_what(kind)}"
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": cfg.get("scaling", "weak"), "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "voxels": n, "cin": cfg["cin"], "cout": cfg["cout"]},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": HOST_THREADS, "kind": kind, "sample": sample},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    args = parse()
    rank, world, local_rank = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        # FVDB_DIST_BACKEND=gloo runs the multi-rank code paths on fewer GPUs than ranks (functional check only:
        # NCCL needs one GPU per rank); ranks then share devices round-robin
        backend = os.environ.get("FVDB_DIST_BACKEND", "nccl")
        if backend != "nccl":
            local_rank = local_rank % torch.cuda.device_count()
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    elif args.gpus > 1:
        print(json.dumps({"error": "--gpus > 1 needs torchrun (one process per GPU)"}), file=sys.stderr)
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()

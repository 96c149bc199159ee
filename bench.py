#!/usr/bin/env python
"""Benchmark of the Trick-GS rasterizer training step on B200 (BASELINE.json config 3).

Workload (`c3`): 1,000,000 Gaussians, SH degree 3, 8 cameras at 1920x1080 on a
radius U(4,6) sphere, Gaussian-mask threshold 0.01, SH-band masks 0.1.  One
step = for each view: render_forward -> (0.8 L1 + 0.2 D-SSIM) loss ->
render_backward, gradients summed over the 8 views, NCCL all-reduce (N > 1),
Adam over all 8 parameter groups.  Views are sharded over ranks (weak scaling
of per-GPU render work is NOT used: the 8-view batch is fixed, so "scaling":
"strong").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0 (see the repo's bench contract).  The reference
arm (`--impl reference`) times the CPU oracle port (oracle/, float64 C++
restatement of the reference's algorithm; the Python reference cannot travel to
the GPU box) on the host's cores for the same workload.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train step/s & render FPS at 1M Gaussians 1080p, 1/2/4/8 B200; HBM % of peak"
VIEWS = 8
LAMBDA_SSIM = 0.2


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--n", type=int, default=1_000_000, help="Gaussians (default: config 3)")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-threads", type=int, default=0, help="reference arm threads (0 = all cores)")
    p.add_argument("--config", choices=["c3", "c4", "c5"], default="c3",
                   help="c3: training step (default, the metric's config); c4: 3M-Gaussian 4K render orbit; "
                        "c5: progressive-schedule sweep (2000 steps with pruning)")
    p.add_argument("--c5-steps", type=int, default=2000, help="c5: schedule length")
    p.add_argument("--rank-share", type=int, default=0,
                   help="N > 1: time rank 0's share of an N-GPU ZeRO-1 step on this one GPU and print a projected "
                        "N-GPU step (measured share + an NCCL reduce-scatter/all-gather bandwidth model)")
    p.add_argument("--nvlink-gbs", type=float, default=720.0,
                   help="--rank-share model: NCCL reduce-scatter / all-gather / all-to-all bus bandwidth per GPU, GB/s")
    p.add_argument("--dp", choices=("zero", "gaussians"), default="gaussians",
                   help="data-parallel design for N > 1 and --rank-share (train.Trainer dp_mode)")
    a = p.parse_args()
    a.warmup = max(a.warmup, 3)
    return a


def settings_kwargs():
    return dict(near=0.2, tile_size=16, lowpass_s=0.3, active_sh_degree=3, mask_threshold=0.01,
                sh_mask_threshold=0.1, compute_sh_rest_grads=True, background=(0.0, 0.0, 0.0))


DP_DESIGNS = {"gaussians": "Gaussian-sharded: this rank's rows of every view's preprocess, NCCL all-to-all of the "
                            "preprocess outputs and splat partials, preprocess backward + Adam on this rank's rows",
              "zero": "ZeRO-1: NCCL reduce-scatter of the flat gradient, Adam on this rank's 1/N, all-gather of the "
                      "parameters"}


def config_dict(n, world, dp="gaussians"):
    return {"workload": "c3: BASELINE.json configs[2] training step", "gaussians": n, "sh_degree": 3,
            "views_per_step": VIEWS, "resolution": "1920x1080", "tile": 16, "loss": "0.8*L1 + 0.2*D-SSIM (11x11)",
            "mask_threshold": 0.01, "sh_mask_threshold": 0.1, "optimizer": "Adam, 8 groups",
            "parallelism": f"dp{world} (views sharded; {DP_DESIGNS[dp]})" if world > 1 else "dp1 (one GPU, no exchange)",
            "l2": "inputs larger than L2: params+grads+Adam moments = 1.0 GB touched per step",
            "timing": "fixed workload: each timed step starts from the initial parameters and Adam state "
                      "(restored outside the step's CUDA events); per-step device times summed, max over ranks"}


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = tempfile.mktemp(suffix=".csv")

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.idx), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self) -> dict:
        rows = []
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) >= 7:
                    rows.append(f)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[0]) for r in rows if r[0].replace(".", "").isdigit()]
        busy = [v for v in sm if v > 500] or sm
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(busy) if busy else None,
                "sm_max_mhz": float(rows[0][1]) if rows[0][1].replace(".", "").isdigit() else None,
                "reasons": reasons, "samples": len(rows)}


# ------------------------------------------------------------ roofline
def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def stage_bytes(n, vis_n, inst, entries, pixels, views):
    """Algorithmic bytes per stage launch as designed.

    n Gaussians, vis_n selected (on-screen) Gaussians, inst instances, entries
    (Gaussian, 8x8-tile super-tile) pairs and pixels are per view."""
    return {
        # one multi-view launch per step: 252 B of parameters read once, per view a 48 B record
        # + 1 visible + 4 tiles + 8 depth key written
        "preprocess_fwd": n * (252 + views * (48 + 1 + 4 + 8)),
        # value-bucket depth sort: select (tiles 4 + mean/radius 20 + rect 8 written) + key 8, bucket
        # count (rect 4, key 8), scatter (rect 4, key 8 in; key + id 12 out), in-bucket rank
        # (key + id 12 in, id 4 + rect 8 gathered + rect 8 out); the 2^17-bucket scan
        "bin_gaussians": n * (32 + 4 + 4) + vis_n * (8 + 8 + 8 + 12 + 12 + 20) + (1 << 17) * 12,
        # rects read by the chunk counts and the level-1 scatter (2 x 8 B per Gaussian); per entry:
        # level-1 write 4, level-2 count (entry 4 + rect 8), level-2 write (entry 4 + rect 8 + id 4);
        # per instance the final id written
        "bin_instances": vis_n * 16 + entries * (4 + 12 + 16) + inst * 4,
        # per instance: 4 B id + 48 B record staged; per pixel 28 B out (rgb, T, w, n, last)
        "blend_fwd": inst * 52 + pixels * 28,
        # per instance 52 B; per pixel 20 B in (dimage, T, last); 36 B partials RMW per Gaussian
        "blend_bwd": inst * 52 + pixels * 20 + vis_n * 72,
        # one launch per step: parameters 252 B, per view partials 36 B + visible 1 B, gradients 260 B
        "preprocess_bwd": n * (252 + views * 37 + 260),
        # image + target 24 B in, dimage 12 B out, SSIM partials 36 B written and read back per pixel
        "loss": pixels * (36 + 72),
        # 63 floats x (read p, g, m, v; write p, m, v), one fused launch per step
        "adam": n * 63 * 28,
    }


# Stages whose roof is instruction issue, not HBM (ncu: issue slots ~75% busy, DRAM ~3% of
# peak; the splat records they stage are L2-served): packed-FP32 per-pixel arithmetic with
# barrier-free warps.  Their roofline is the SM issue rate, 148 SMs x 4 schedulers x one
# warp instruction per clock at the measured SM clock.
ISSUE_BOUND = {"blend_fwd", "blend_bwd"}
SMS, SCHEDULERS = 148, 4


def ncu_stage(stage):
    """The stage's entry in the newest committed ncu --set full capture
    (profiles/r0N_ncu_traffic.json, written by profiles/ncu_summary.py)."""
    for rnd in ("r02", "r01"):
        try:
            d = json.load(open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_traffic.json")))
        except (OSError, ValueError):
            continue
        if stage in d:
            return dict(d[stage], capture=f"profiles/{rnd}_ncu_traffic.json")
    return {}


def roofline(prof_ms: dict, counts: dict, sbytes: dict, peak: float, peak_kind: str, pairs: float,
             sm_mhz) -> tuple[dict, dict]:
    """Per-stage achieved bytes/s (algorithmic bytes over the live CUDA-event time) and the
    roofline object of the dominant stage by device time.  For an issue-bound stage the
    roofline is the SM issue rate (achieved = the stage's executed warp instructions per
    launch from the committed ncu capture / the live launch time), with the HBM view
    (algorithmic and DRAM bytes) and the evaluated (pixel, splat) pairs per second beside it."""
    stages = {}
    for k, ms in prof_ms.items():
        c = counts.get(k, 0)
        if not c or k not in sbytes:
            stages[k] = {"ms_total": round(ms, 4), "launches": c}
            continue
        per = ms / c
        gbs = sbytes[k] / (per * 1e-3) / 1e9
        stages[k] = {"ms_per_launch": round(per, 4), "launches": c, "ms_total": round(ms, 4),
                     "algorithmic_gbs": round(gbs, 1), "frac": round(gbs / peak, 4),
                     "bound": "issue" if k in ISSUE_BOUND else "hbm"}
        nc = ncu_stage(k)
        if nc.get("dram_bytes_per_launch"):
            stages[k]["dram_gbs"] = round(nc["dram_bytes_per_launch"] / (per * 1e-3) / 1e9, 1)
            stages[k]["dram_frac"] = round(stages[k]["dram_gbs"] / peak, 4)
        for key in ("issue_busy_pct", "fma_pipe_pct"):
            if nc.get(key) is not None:
                stages[k][key] = nc[key]
    dom = max((k for k in stages if "algorithmic_gbs" in stages[k]), key=lambda k: stages[k]["ms_total"])
    d = stages[dom]
    nc = ncu_stage(dom)
    per_s = d["ms_per_launch"] * 1e-3
    hbm = {"algorithmic_bytes": int(sbytes[dom]), "algorithmic_gbs": d["algorithmic_gbs"],
           "frac_algorithmic": d["frac"], "dram_bytes_per_launch": nc.get("dram_bytes_per_launch"),
           "dram_gbs": d.get("dram_gbs"), "frac_dram": d.get("dram_frac"), "peak_gbs": peak, "peak_source": peak_kind}
    if dom in ISSUE_BOUND and nc.get("warp_insts") and sm_mhz:
        achieved = nc["warp_insts"] / per_s / 1e9
        ipk = SMS * SCHEDULERS * float(sm_mhz) * 1e6 / 1e9
        rf = {"kernel": dom, "bound": "issue", "achieved": round(achieved, 1), "peak": round(ipk, 1),
              "unit": "Gwarp-inst/s", "frac": round(achieved / ipk, 4),
              "traffic": nc.get("dram_bytes_per_launch"),
              "peak_source": f"{SMS} SMs x {SCHEDULERS} schedulers x 1 warp-inst/clk at the measured "
                             f"median SM clock {sm_mhz} MHz",
              "warp_insts_per_launch": nc["warp_insts"], "ncu_issue_busy_pct": nc.get("issue_busy_pct"),
              "ncu_fma_pipe_pct": nc.get("fma_pipe_pct"), "ncu_capture": nc.get("capture"),
              "pairs_per_launch": int(pairs), "pairs_per_s": round(pairs / per_s / 1e9, 2),
              "pairs_unit": "G (pixel, list entry) pairs/s: sum over pixels of last_pos", "hbm": hbm}
    else:
        rf = {"kernel": dom, "bound": "hbm", "achieved": d["algorithmic_gbs"], "peak": peak, "unit": "GB/s",
              "frac": d["frac"], "traffic": nc.get("dram_bytes_per_launch"), "peak_source": peak_kind, "hbm": hbm}
    return rf, stages


def super_tile_entries(splats, tiles_touched, width, height, ts=16, st=8):
    """(Gaussian, 8x8-tile super-tile) pairs of a view: the rect of bin_tiles
    (rasterizer.py:112-128) in super-tile units, summed over on-screen Gaussians."""
    import torch
    on = tiles_touched > 0
    m, r = splats[on, 0:2], splats[on, 10:11]
    tx, ty = (width + ts - 1) // ts, (height + ts - 1) // ts
    lo = torch.floor((m - r) / ts).clamp(min=0)
    hi = torch.floor((m + r) / ts)
    hi = torch.stack([hi[:, 0].clamp(max=tx - 1), hi[:, 1].clamp(max=ty - 1)], 1)
    span = (torch.div(hi, st, rounding_mode="floor") - torch.div(lo, st, rounding_mode="floor") + 1).clamp(min=0)
    return int((span[:, 0] * span[:, 1]).sum())


# ------------------------------------------------------- CPU reference
def cpu_view_step(fields, cam, target, st, threads_note=""):
    """One view: oracle fp64 render fwd -> loss -> render bwd (the reference algorithm)."""
    from oracle import loss_ref, oracle
    f = oracle.render_forward(fields, cam, st, "f64")
    _, _, dimg = loss_ref.total_loss_image(f["image"], target, LAMBDA_SSIM)
    g = oracle.render_backward(fields, cam, st, dimg, f, "f64")
    return g


def cpu_adam_seconds(n_floats):
    rng = np.random.default_rng(0)
    p, g = rng.standard_normal(n_floats), rng.standard_normal(n_floats)
    m, v = np.zeros(n_floats), np.zeros(n_floats)
    t = time.perf_counter()
    m = 0.9 * m + 0.1 * g  # optim.py:45-49
    v = 0.999 * v + 0.001 * g * g
    p -= 1e-3 * (m / 0.1) / (np.sqrt(v / 0.001) + 1e-15)
    return time.perf_counter() - t


def host_info() -> dict:
    """The CPU the baseline ran on (lscpu model, cores) and the BLAS/OpenMP thread environment."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    if model is None:
        try:
            model = next(line.split(":", 1)[1].strip() for line in open("/proc/cpuinfo") if line.startswith("model name"))
        except (OSError, StopIteration):
            model = "unknown"
    env = {k: os.environ.get(k) for k in ("OMP_NUM_THREADS", "MKL_NUM_THREADS", "OPENBLAS_NUM_THREADS",
                                          "NUMBA_NUM_THREADS")}
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "affinity_cpus": len(os.sched_getaffinity(0)),
            "thread_env": env, "numpy": np.__version__}


def cpu_baseline(sc, st, views_to_time=1):
    """Bounded sample: `views_to_time` view-steps on 1 core, scaled to the 8-view step."""
    t0 = time.perf_counter()
    for v in range(views_to_time):
        cpu_view_step(sc.fields, sc.cameras[v], sc.targets[v], st)
    t_view = (time.perf_counter() - t0) / views_to_time
    t_adam = cpu_adam_seconds(sc.n * 63)
    t_step = VIEWS * t_view + t_adam
    return {"value": round(1.0 / t_step, 6), "unit": "train step/s", "cores": 1, "kind": "port", "host": host_info(),
            "sample": f"{views_to_time} of 8 views (fwd+loss+bwd, float64 oracle/oracle.cpp) timed "
                      f"({t_view:.1f} s/view) + numpy Adam over {sc.n * 63} floats ({t_adam:.1f} s); "
                      f"step = 8 x view + Adam = {t_step:.1f} s"}


def reference_arm(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from concurrent.futures import ThreadPoolExecutor
    from types import SimpleNamespace

    from paper_2501_14534_b200 import scenes
    sc = scenes.config3(n=args.n)
    st = SimpleNamespace(record_hits=False, **settings_kwargs())
    threads = args.cpu_threads or os.cpu_count() or 1
    workers = max(1, min(threads, VIEWS))
    steps = max(1, min(args.steps, 2))  # bounded: each step is ~10-30 s of CPU work per view

    def step():
        with ThreadPoolExecutor(workers) as ex:  # ctypes releases the GIL: views run in parallel
            list(ex.map(lambda v: cpu_view_step(sc.fields, sc.cameras[v], sc.targets[v], st), range(VIEWS)))
        cpu_adam_seconds(sc.n * 63)

    step()  # warm-up (page-in, oracle build)
    t = time.perf_counter()
    for _ in range(steps):
        step()
    dt = (time.perf_counter() - t) / steps
    v = 1.0 / dt
    line = {"metric": METRIC, "value": round(v, 6), "unit": "train step/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": steps, "warmup": 1, "ms_per_step": round(dt * 1e3, 1),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (seeded BASELINE.json config 3 generator)", "config": config_dict(args.n, 1),
            "cpu_baseline": {"value": round(v, 6), "unit": "train step/s", "cores": workers, "kind": "port",
                             "host": host_info(),
                             "sample": f"full 8-view step: views in {workers} threads of the float64 oracle "
                                       f"(oracle/oracle.cpp + oracle/loss_ref.py), numpy Adam; "
                                       f"{steps} timed step(s) after 1 warm-up"},
            "e2e": {"value": round(v, 6), "unit": "train step/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------- ours
def main():
    args = parse()
    if args.config == "c4":
        return render_c4(args)
    if args.config == "c5":
        return schedule_c5(args)
    if args.impl == "reference":
        return reference_arm(args)
    if args.rank_share > 1:
        return rank_share(args)
    import torch
    import torch.distributed as dist

    from paper_2501_14534_b200 import GaussianCloud, RenderSettings, _lib, profiler, scenes
    from paper_2501_14534_b200.train import Trainer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    _lib.load()

    sc = scenes.config3(n=args.n)
    views = list(range(rank, VIEWS, world))
    st = RenderSettings(**settings_kwargs())
    cloud = GaussianCloud.from_fields(sc.fields, device=dev)
    h, w = sc.cameras[0].height, sc.cameras[0].width
    host_targets = {v: torch.from_numpy(sc.targets[v]).pin_memory() for v in views}
    targets = [None] * VIEWS
    for v in views:
        targets[v] = host_targets[v].to(dev)
    trainer = Trainer(cloud, sc.cameras, targets, st, LAMBDA_SSIM, process_group=pg, views=views, dp_mode=args.dp)

    def barrier():
        if pg is not None:
            dist.barrier()

    def timed(k, body):
        """K consecutive steps bracketed by one event pair (the scene evolves under training)."""
        torch.cuda.synchronize()
        barrier()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(k):
            body()
        e.record()
        torch.cuda.synchronize()
        barrier()
        t = torch.tensor([s.elapsed_time(e) / 1e3], device=dev)
        if pg is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t)

    # A FIXED workload: training changes the scene (the reference's mask lr of 0.5 prunes
    # occluded Gaussians within ~13 steps), so every timed step starts from the same initial
    # parameters and Adam state, restored before the step and outside its events; the
    # per-step device times are summed (max over ranks of the sum).
    init = (cloud.flat.clone(), trainer.opt.m.clone(), trainer.opt.v.clone(), dict(trainer.opt.steps))

    def reset(tr):
        cloud.flat.copy_(init[0])
        tr.opt.m.copy_(init[1])
        tr.opt.v.copy_(init[2])
        tr.opt.steps = dict(init[3])
        torch.cuda.synchronize()

    each = {}

    def timed_fixed(k, body, tr, label="device"):
        total, inst, ms = 0.0, [], []
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gc.collect()
        gc.disable()  # no collector pause inside a timed step (the host enqueues the step)
        try:
            for _ in range(k):
                reset(tr)
                barrier()
                s.record()
                body()
                e.record()
                e.synchronize()
                ms.append(s.elapsed_time(e))
                total += ms[-1] / 1e3
                inst.append(sum(tr.instances))
        finally:
            gc.enable()
        each[label] = [round(x, 3) for x in ms]
        torch.cuda.synchronize()
        barrier()
        t = torch.tensor([total], device=dev)
        if pg is not None:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t), inst

    for _ in range(args.warmup):
        trainer.step()
    trainer.check_divergence()
    # ---- device-resident timed region (inputs already in HBM), views pipelined on 4 streams
    with ClockSampler(local) as clk:
        t_dev, inst_steps = timed_fixed(args.steps, trainer.step, trainer)
    clocks = clk.summary()
    trainer.check_divergence()
    value = args.steps / t_dev
    # the same K steps back to back without the per-step restore (the scene prunes itself
    # as it trains): reported for comparison only
    reset(trainer)
    t_cont = timed(args.steps, trainer.step)
    trainer.check_divergence()
    # ---- end-to-end through the public API: targets H2D from pinned host memory, loss D2H
    terms_host = torch.empty((VIEWS, 2), dtype=torch.float64).pin_memory()

    def e2e_step():
        # targets stream in on the trainer's copy stream, overlapped with earlier views
        trainer.step(host_targets=host_targets)
        terms_host.copy_(trainer.terms, non_blocking=True)

    e2e_step()
    t_e2e, _ = timed_fixed(args.steps, e2e_step, trainer, "e2e")
    trainer.check_divergence()
    h2d = sum(host_targets[v].numel() * 4 for v in views)
    d2h = terms_host.numel() * 8

    # ---- per-kernel roofline: the same fixed-workload steps with views serialised on one
    # stream, so the CUDA-event duration of each stage is its own (no overlap with the other
    # views)
    serial = Trainer(cloud, sc.cameras, targets, st, LAMBDA_SSIM, process_group=pg, views=views, streams=1)
    serial.opt = trainer.opt
    serial.step()
    with profiler.StageTimer() as prof:
        t_serial, _ = timed_fixed(args.steps, serial.step, serial, "serial_views")
    reset(serial)
    from paper_2501_14534_b200.rasterizer import render_forward
    inst, ents, vis, pairs = [], [], [], []
    for v in views:
        out = render_forward(cloud, sc.cameras[v], st)
        inst.append(int(out._tiles.indices.numel()))
        tt = out._state.tiles_touched[: len(cloud)]
        vis.append(int((tt > 0).sum()))
        ents.append(super_tile_entries(out._state.splats[: len(cloud)], tt, w, h))
        pairs.append(int(out.last_pos.to(torch.int64).sum()))  # per-pixel list entries walked
    inst_mean, ent_mean, vis_n, pairs_mean = (sum(x) / len(x) for x in (inst, ents, vis, pairs))
    pk, pk_kind = peaks()
    sb = stage_bytes(len(cloud), vis_n, inst_mean, ent_mean, h * w, VIEWS)
    rf, stages = roofline(prof.durations_ms(), prof.counts(), sb, float(pk["hbm_gbs"]), pk_kind, pairs_mean,
                          clocks.get("sm_mhz"))
    launches = trainer_launches(prof.counts(), args.steps)

    # ---- render FPS (forward only, initial scene) as a secondary number: this rank's views
    # through render_views (one multi-view preprocess pass, binning + blending pipelined over
    # three streams), device-timed
    from paper_2501_14534_b200.rasterizer import render_views

    def render_all():
        render_views(cloud, [sc.cameras[v] for v in views], st)

    render_all()  # learns the batch's instance counts (Python pipeline)
    render_all()  # first native batch: its workspaces and arenas are allocated here, untimed
    fps_t = timed(args.steps, render_all)
    render_fps = args.steps * len(views) * world / fps_t
    compat = compat_cost(sc, st, dev) if world == 1 else None

    if rank != 0:
        return
    line = {"metric": METRIC, "value": round(value, 4), "unit": "train step/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_dev / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded BASELINE.json config 3 generator; random-init Gaussians, U[0,1] targets)",
            "config": config_dict(len(cloud), world, args.dp),
            "e2e": {"value": round(args.steps / t_e2e, 4), "unit": "train step/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches, "clocks": clocks, "roofline": rf, "stages": stages,
            "ms_each_step": each,
            "ms_per_step_serial_views": round(t_serial / args.steps * 1e3, 3),
            "ms_per_step_continuous": round(t_cont / args.steps * 1e3, 3),
            "render_fps": round(render_fps, 2), "instances_per_view": int(inst_mean),
            "instances_per_step_first_last": [inst_steps[0], inst_steps[-1]] if inst_steps else None,
            "entries_per_view": int(ent_mean), "selected_per_view": int(vis_n),
            "pairs_per_view": int(pairs_mean)}
    if compat is not None:
        line["compat_drop_in"] = compat
    if world == 1 and not args.no_cpu_baseline:
        from types import SimpleNamespace
        line["cpu_baseline"] = cpu_baseline(sc, SimpleNamespace(record_hits=False, **settings_kwargs()))
    print(json.dumps(line), flush=True)
    if pg is not None:
        dist.destroy_process_group()


def compat_cost(sc, st, dev) -> dict:
    """The literal drop-in (compat.py: the reference's own float64 numpy objects in and out,
    what its training.py:296-309 iteration calls): one c3 view's render_forward +
    render_backward per iteration, wall time per iteration (the cloud's upload and the
    outputs' / gradients' download included), against the same view's device time."""
    import types

    import torch

    from paper_2501_14534_b200 import compat
    cloud64 = types.SimpleNamespace(**{k: np.asarray(v, dtype=np.float64) for k, v in sc.fields.items()})
    cam = sc.cameras[0]
    dimg = np.random.default_rng(0).standard_normal((cam.height, cam.width, 3))
    for _ in range(2):
        compat.render_backward(cloud64, cam, st, dimg, compat.render_forward(cloud64, cam, st))
    torch.cuda.synchronize()
    k = 3
    t0 = time.perf_counter()
    for _ in range(k):
        out = compat.render_forward(cloud64, cam, st)
        compat.render_backward(cloud64, cam, st, dimg, out)
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / k
    return {"ms_per_view_iteration": round(wall * 1e3, 2),
            "what": "compat.render_forward + compat.render_backward of one c3 view with float64 numpy "
                    "inputs / outputs: the cloud (63 float64 per Gaussian) converted and uploaded, the "
                    "image, auxiliaries and 9 gradient fields downloaded and widened to float64 — the "
                    "reference's per-iteration call pattern; a training loop keeping the cloud on the "
                    "GPU (train.Trainer) does not pay it"}


def gpu_busy(fn, k: int) -> dict:
    """Run fn k times under a CUDA activity trace; GPU busy = the union of the kernel
    intervals, span = first kernel start to last kernel end (profiles/gpu_idle.py)."""
    import torch
    from torch.profiler import ProfilerActivity, profile
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(k):
            fn()
        torch.cuda.synchronize()
    wall = time.perf_counter() - w0
    iv = sorted((e.time_range.start, e.time_range.end) for e in prof.events()
                if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0
                and "Memcpy" not in e.name and "Memset" not in e.name)
    if not iv:
        return {}
    busy, cs, ce = 0.0, iv[0][0], iv[0][1]
    for a, b in iv[1:]:
        if a > ce:
            busy += ce - cs
            cs, ce = a, b
        else:
            ce = max(ce, b)
    busy += ce - cs
    span = max(b for _, b in iv) - iv[0][0]
    return {"steps": k, "gpu_busy_ms_per_step": round(busy / k / 1e3, 3), "span_ms_per_step": round(span / k / 1e3, 3),
            "busy_fraction": round(busy / max(span, 1e-9), 3), "wall_ms_per_step_traced": round(wall / k * 1e3, 3)}


def rank_share(args):
    """Projection of the N-GPU c3 step from ONE GPU (only one GPU is available to this
    build): rank 0's share of an N-rank step, timed exactly like the bench's fixed-workload
    step, plus the step's NCCL exchange at an assumed bus bandwidth (--nvlink-gbs), NOT
    overlapped with compute.  --dp gaussians (default, train.Trainer(gshard_sim=(0, N))):
    its views (0, N, 2N, ...), the preprocess forward / backward of every view over its 1/N
    rows of the cloud and Adam on those rows; exchange = the all-to-alls of its views'
    preprocess outputs and splat partials.  --dp zero (Trainer(zero_sim=(0, N))): its views,
    the multi-view preprocess forward / backward of those views over the whole cloud and
    Adam on its 1/N parameter shard; exchange = reduce-scatter + all-gather of the step's
    parameter range.  Measured for the bench's step (every gradient, SH-rest included) and
    for the SH-cadence steps in between (compute_sh_rest_grads off, rasterizer.py:88-92:
    sh_rest neither differentiated nor updated), as the schedule average of one cadence
    step per 16, and with steps enqueued back to back ("continuous")."""
    import dataclasses

    import torch

    from paper_2501_14534_b200 import GaussianCloud, RenderSettings, _lib, scenes
    from paper_2501_14534_b200.parallel import zero_plan
    from paper_2501_14534_b200.train import Trainer
    N = args.rank_share
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    _lib.load()
    sc = scenes.config3(n=args.n)
    st_full = RenderSettings(**settings_kwargs())
    cloud = GaussianCloud.from_fields(sc.fields, device=dev)
    views = list(range(0, VIEWS, N))
    gs = args.dp == "gaussians"
    share_kw = (dict(views=views, dp_mode="gaussians", gshard_sim=(0, N),
                     all_views=[list(range(d, VIEWS, N)) for d in range(N)]) if gs else dict(views=views, zero_sim=(0, N)))
    targets = [None] * VIEWS
    for v in views:
        targets[v] = torch.from_numpy(sc.targets[v]).to(dev)
    out, cont = {}, {}
    for rest in (True, False):
        st = dataclasses.replace(st_full, compute_sh_rest_grads=rest)
        for label, kw in (("share", share_kw), ("full", dict(views=list(range(VIEWS))))):
            if label == "full":
                for v in range(VIEWS):
                    targets[v] = torch.from_numpy(sc.targets[v]).to(dev)
            tr = Trainer(cloud, sc.cameras, targets, st, LAMBDA_SSIM, **kw)
            init = (cloud.flat.clone(), tr.opt.m.clone(), tr.opt.v.clone(), dict(tr.opt.steps))
            for _ in range(args.warmup):
                tr.step()
            total = 0.0
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            for _ in range(args.steps):
                cloud.flat.copy_(init[0])
                tr.opt.m.copy_(init[1])
                tr.opt.v.copy_(init[2])
                tr.opt.steps = dict(init[3])
                torch.cuda.synchronize()
                s.record()
                tr.step()
                e.record()
                e.synchronize()
                total += s.elapsed_time(e)
            tr.check_divergence()
            # the same fixed workload without the host synchronisation before every step:
            # each step's restore is enqueued ahead of it (outside its events), so the host
            # prepares step k+1 while the GPU runs step k, as in back-to-back training
            evs = []
            for _ in range(args.steps):
                cloud.flat.copy_(init[0])
                tr.opt.m.copy_(init[1])
                tr.opt.v.copy_(init[2])
                tr.opt.steps = dict(init[3])
                s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s.record()
                tr.step()
                e.record()
                evs.append((s, e))
            torch.cuda.synchronize()
            tr.check_divergence()
            cont[(rest, label)] = sum(a.elapsed_time(b) for a, b in evs) / args.steps
            cloud.flat.copy_(init[0])
            out[(rest, label)] = total / args.steps
        for v in range(VIEWS):
            targets[v] = torch.from_numpy(sc.targets[v]).to(dev) if v in views else None
    res = {}
    from paper_2501_14534_b200.parallel import GSHARD_BWD_BYTES, GSHARD_FWD_BYTES
    for rest in (True, False):
        if gs:  # per rank: its views' preprocess outputs in, their splat partials out (all-to-alls)
            pbytes = len(views) * len(cloud) * (GSHARD_FWD_BYTES + GSHARD_BWD_BYTES)
            comm_ms = (N - 1) / N * pbytes / (args.nvlink_gbs * 1e9) * 1e3
        else:
            pbytes = sum(ch.end - ch.begin for ch in zero_plan(cloud._layout_map, N, rest_grads=rest)) * 4
            comm_ms = 2 * (N - 1) / N * pbytes / (args.nvlink_gbs * 1e9) * 1e3
        res[rest] = dict(share=out[(rest, "share")], full=out[(rest, "full")], comm=comm_ms, bytes=pbytes,
                         proj=out[(rest, "share")] + comm_ms)
    avg = lambda k: (res[True][k] + 15 * res[False][k]) / 16  # noqa: E731
    proj, full = res[True]["proj"], res[True]["full"]
    design = "Gaussian-sharded" if gs else "ZeRO-1"
    print(json.dumps({"metric": f"projected c3 train step/s at {N} GPUs ({design}: 1-GPU rank-share measurement + "
                                f"NCCL model)",
                      "value": round(1e3 / proj, 3), "unit": "train step/s", "n_gpus": 1, "projected_n_gpus": N,
                      "ms_per_step_projected": round(proj, 3), "ms_rank_share_measured": round(res[True]["share"], 3),
                      "ms_comm_model": round(res[True]["comm"], 3), "ms_per_step_1gpu_measured": round(full, 3),
                      "projected_speedup": round(full / proj, 3), "dp": args.dp,
                      "continuous": {"ms_rank_share_measured": round(cont[(True, "share")], 3),
                                     "ms_per_step_1gpu_measured": round(cont[(True, "full")], 3),
                                     "ms_per_step_projected": round(cont[(True, "share")] + res[True]["comm"], 3),
                                     "projected_speedup": round(cont[(True, "full")] /
                                                                (cont[(True, "share")] + res[True]["comm"]), 3),
                                     "how": "same fixed workload, steps enqueued back to back (no host sync "
                                            "between steps; restores enqueued outside each step's events)"},
                      "projected_speedup_at_half_bandwidth": round(full / (proj + res[True]["comm"]), 3),
                      "sh_cadence_step": {"ms_rank_share_measured": round(res[False]["share"], 3),
                                          "ms_comm_model": round(res[False]["comm"], 3),
                                          "exchanged_bytes": res[False]["bytes"],
                                          "ms_per_step_projected": round(res[False]["proj"], 3),
                                          "ms_per_step_1gpu_measured": round(res[False]["full"], 3),
                                          "projected_speedup": round(res[False]["full"] / res[False]["proj"], 3)},
                      "schedule_average_1_in_16": {"ms_per_step_projected": round(avg("proj"), 3),
                                                   "ms_per_step_1gpu_measured": round(avg("full"), 3),
                                                   "projected_speedup": round(avg("full") / avg("proj"), 3)},
                      "views_on_rank0": views,
                      "comm_model": (f"all-to-all of rank 0's views' preprocess outputs ({GSHARD_FWD_BYTES} B per "
                                     f"Gaussian and view) and splat partials ({GSHARD_BWD_BYTES} B): {res[True]['bytes']} B "
                                     f"x (N-1)/N at {args.nvlink_gbs} GB/s NCCL bus bandwidth, not overlapped" if gs else
                                     f"reduce-scatter + all-gather of the step's parameter range ({res[True]['bytes']} B; "
                                     f"{res[False]['bytes']} B on SH-cadence steps) at {args.nvlink_gbs} GB/s NCCL bus "
                                     f"bandwidth, not overlapped"),
                      "higher_is_better": True, "dtype": "f32", "data": "synthetic (seeded BASELINE.json config 3)",
                      "config": config_dict(len(cloud), N, args.dp)}), flush=True)


def _c5_shell_targets(sc, views, st0, args, dev):
    """c5 on the shell scene (TGS_C5_SCENE=shell): targets are renders of a HELD-OUT SUBSET —
    30% of the Gaussians, drawn from the rows the 8 cameras see (hit counts > 0,
    significance.count_hits) — rendered opaquer than the trained cloud starts."""
    import torch

    from paper_2501_14534_b200 import GaussianCloud, significance
    from paper_2501_14534_b200.rasterizer import render_forward
    init = GaussianCloud.from_fields(sc.fields, device=dev)
    hits = significance.count_hits(init, sc.cameras, st0)
    seen = torch.nonzero(hits > 0).flatten().cpu().numpy()
    keep_n = min(int(0.3 * args.n), seen.size)
    if os.environ.get("TGS_C5_SUBSET", "top") == "top":  # the most-hit rows: the best-supported 30%
        subset = np.sort(torch.topk(hits.to(torch.float64), keep_n).indices.cpu().numpy())
    else:
        subset = np.sort(np.random.default_rng(5).choice(seen, keep_n, replace=False))
    # the subset is rendered OPAQUER than the trained cloud starts (opacity logits + boost):
    # its rows' photometric gradient then asks for more opacity step after step, a
    # consistent sign that holds their mask logits up against the lr-0.5 Adam random walk
    boost = float(os.environ.get("TGS_C5_BOOST", "2.0"))
    sub = {k: np.ascontiguousarray(v[subset]) for k, v in sc.fields.items()}
    sub["opacity_logits"] = (sub["opacity_logits"] + np.float32(boost)).astype(np.float32)
    held = GaussianCloud.from_fields(sub, device=dev)
    full_t = {}
    for v in views:
        full_t[v] = render_forward(held, sc.cameras[v], st0).image.contiguous()
    del init, held
    full_t["_meta"] = (keep_n, seen, boost)
    return full_t


def schedule_c5(args):
    """BASELINE.json configs[4]: the progressive-training schedule on 1M Gaussians — render
    resolution stepped 1/8 -> 1/4 -> 1/2 -> 1 of 1920x1080 (targets area-resized on the GPU),
    the EWA low-pass scale decaying with a blur factor 4 -> 1 (lowpass_s = max(HW/(9 pi N),
    0.3 f^2); the reference's progressive scale, schedule.py:166-170), SH bands enabled
    0 -> 3 (one per quarter), SH-rest gradients every 16 steps (rasterizer.py:88-92), mask
    pruning every 500 steps with cloud + Adam compaction (masking.py:70-81, optim.py:51-55).
    Each step = the c3 8-view training step at the current resolution.  Opacity noise has no
    counterpart in the reference (a non-goal there) and is not modelled."""
    import torch
    import torch.distributed as dist

    from paper_2501_14534_b200 import GaussianCloud, RenderSettings, _lib, images, scenes, schedule
    from paper_2501_14534_b200.rasterizer import sh_rest_update_step
    from paper_2501_14534_b200.train import Trainer

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    pg = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        pg = dist.group.WORLD
    _lib.load()
    c5_scene = os.environ.get("TGS_C5_SCENE", "sfm")
    if c5_scene == "sfm":  # the reference's own recipe: ground-truth renders, SfM-seeded cloud
        sc, gt_fields = scenes.config5_sfm(n=args.n, views=VIEWS)
    else:
        sc, gt_fields = scenes.config5(n=args.n, views=VIEWS), None
    views = list(range(rank, VIEWS, world))
    from paper_2501_14534_b200.rasterizer import render_forward
    st0 = RenderSettings(**settings_kwargs())
    if gt_fields is not None:
        gt = GaussianCloud.from_fields(gt_fields, device=dev)
        full_t = {v: render_forward(gt, sc.cameras[v], st0).image.contiguous() for v in views}
        keep_n, seen, boost = len(gt), np.zeros(0), 0.0
        del gt
    else:
        full_t = _c5_shell_targets(sc, views, st0, args, dev)
        keep_n, seen, boost = full_t.pop("_meta")
    steps = args.c5_steps
    phase_len = max(1, steps // 4)
    kw = settings_kwargs()
    cloud = GaussianCloud.from_fields(sc.fields, device=dev)
    # mask learning: the paper-scale rates (mask lr 0.5, lambda 0.05; config.py:76-92) make every
    # mask logit whose photometric gradient changes sign random-walk by ~0.5 per step into
    # the absorbing hard-mask threshold (a masked Gaussian has zero scale and no
    # photometric gradient left), so ~96% are gone by the first prune on synthetic
    # targets; TGS_C5_MASK=preset uses the reference's own synthetic-scene rates
    # (synthetic.py preset_config: mask / SH-mask lr 0.02, lambda 2e-3)
    lrs, lam = None, {}
    mask_mode = os.environ.get("TGS_C5_MASK", "preset")
    if mask_mode == "preset":
        from paper_2501_14534_b200.train import DEFAULT_LRS
        lrs = {**DEFAULT_LRS, "mask_logits": 0.02, "sh_mask_logits": 0.02}
        lam = dict(lambda_m=2e-3, lambda_sh=2e-3)
    trainer = Trainer(cloud, sc.cameras, {}, RenderSettings(**kw), LAMBDA_SSIM, lrs=lrs, process_group=pg,
                      views=views, dp_mode=args.dp, **lam)
    prunes, counts, phase_res = [], [len(cloud)], {}

    def setup(i):
        ph = min(3, i // phase_len)
        div = (8, 4, 2, 1)[ph]
        w, h = 1920 // div, 1080 // div
        if ph not in phase_res:  # per-phase cameras and area-resized targets (images.py:58-87)
            cams = [c.resized(w, h) for c in sc.cameras]
            tg = {v: (images.area_resize(full_t[v], h, w) if div > 1 else full_t[v]) for v in views}
            phase_res[ph] = (cams, tg)
        cams, tg = phase_res[ph]
        trainer.cameras, trainer.targets = cams, tg
        f = 4.0 - 3.0 * min(1.0, i / max(1, 3 * phase_len))  # blur factor 4 -> 1
        n = len(trainer.cloud)
        trainer.settings = RenderSettings(**{**kw, "lowpass_s": max(schedule.lowpass_s_at(n, h, w), 0.3 * f * f),
                                             "active_sh_degree": schedule.active_sh_degree(i, 3, phase_len),
                                             "compute_sh_rest_grads": sh_rest_update_step(i, 16)})

    def run(i0, i1):
        for i in range(i0, i1):
            if i > 0 and i % 500 == 0:
                prunes.append(i)
                counts.append(trainer.prune(kw["mask_threshold"]))
            setup(i)
            trainer.step()

    run(0, 3)  # warm-up (page-in, kernel attributes); the timed sweep restarts from the initial scene
    trainer.check_divergence()
    trainer.cloud = GaussianCloud.from_fields(sc.fields, device=dev)
    trainer.opt = type(trainer.opt)(trainer.cloud, trainer.opt.lrs)
    from paper_2501_14534_b200.cloud import CloudGrads
    trainer.grads = CloudGrads(len(trainer.cloud), dev)
    trainer.dsplats = {}
    prunes.clear()
    counts[:] = [len(trainer.cloud)]
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        w0 = time.perf_counter()
        s.record()
        run(0, steps)
        e.record()
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
    trainer.check_divergence()
    t = torch.tensor([s.elapsed_time(e) / 1e3], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    # host vs device: the GPU-busy share (union of kernel intervals, CUPTI via torch.profiler)
    # of 16 steps at the first and at the last phase's settings, after the timed sweep
    busy = {}
    for label, i in (("phase1_240x135", 0), ("phase4_1920x1080", steps - 1)):
        setup(i)
        busy[label] = gpu_busy(trainer.step, 16)
    trainer.check_divergence()
    if rank == 0:
        print(json.dumps({"metric": "c5 progressive-schedule sweep: train steps/s", "value": round(steps / float(t), 3),
                          "unit": "train step/s", "n_gpus": world, "steps": steps, "warmup": 3,
                          "ms_per_step": round(float(t) / steps * 1e3, 3), "higher_is_better": True,
                          "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                          "data": ("synthetic (seeded ground-truth shell + SfM-seeded cloud, scenes.config5_sfm; "
                                   "schedule of BASELINE.json config 5)" if c5_scene == "sfm" else
                                   "synthetic (seeded c5 shell scene, scenes.config5; schedule of BASELINE.json config 5)"),
                          "config": {"workload": "c5: BASELINE.json configs[4] schedule sweep", "gaussians": args.n,
                                     "resolution_steps": ["240x135", "480x270", "960x540", "1920x1080"],
                                     "views_per_step": VIEWS, "prune_steps": prunes, "gaussians_after_prunes": counts,
                                     "final_fraction": round(counts[-1] / args.n, 3),
                                     "targets": (f"renders of a {keep_n}-Gaussian ground-truth shell cloud; the trained "
                                                 f"cloud seeded from {args.n} SfM-like points around its centres "
                                                 f"(the reference's synthetic.py / seed_from_sfm recipe)"
                                                 if c5_scene == "sfm" else
                                                 f"renders of a held-out {keep_n}-row subset of the {seen.size} "
                                                 f"rows seen by the cameras, opacity logits +{boost}"),
                                     "mask_learning": ("reference synthetic preset: mask/sh-mask lr 0.02, lambda 2e-3"
                                                       if mask_mode == "preset" else
                                                       "paper scale: mask lr 0.5, sh-mask lr 0.05, lambda 0.05"),
                                     "parallelism": f"dp{world}"},
                          "total_s": round(float(t), 3), "host_wall_s": round(wall, 3),
                          "host_ms_per_step": round(wall / steps * 1e3, 3),
                          "device_ms_per_step": round(float(t) / steps * 1e3, 3),
                          "gpu_busy_sample": busy,
                          "clocks": clk.summary()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def render_c4(args):
    """BASELINE.json configs[3]: 3M Gaussians in 64 anisotropic clusters (radius 10), 3840x2160,
    render-only: the WHOLE 200-frame orbit is timed (after two untimed passes over its
    first 16 frames).  One GPU: batches of 8 frames through render_views (one preprocess pass
    per batch, binning + blending pipelined over three streams).  N ranks: tile rows sharded
    (parallel.ShardedRenderer: replicated preprocess, bands from the previous batch's
    replicated row histogram, the band rows of a batch gathered to rank 0 in one call)."""
    import torch
    import torch.distributed as dist

    from paper_2501_14534_b200 import GaussianCloud, RenderSettings, _lib, parallel, scenes
    from paper_2501_14534_b200.rasterizer import render_views

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _lib.load()
    n = 3_000_000 if args.n == 1_000_000 else args.n
    sc = scenes.config4(n=n)
    cloud = GaussianCloud.from_fields(sc.fields, device=dev)
    st = RenderSettings(near=0.2, tile_size=16)
    frames = sc.cameras
    renderer = parallel.ShardedRenderer(cloud, st) if world > 1 else None

    def orbit(k0, count):
        cams = [frames[(k0 + j) % len(frames)] for j in range(count)]
        for b in range(0, count, 8):
            if renderer is not None:
                renderer.render(cams[b:b + 8])
            else:
                render_views(cloud, cams[b:b + 8], st)

    # untimed: the first batch learns the instance counts (Python pipeline), the second
    # allocates the native batch path's buffers
    orbit(0, 16)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    count = len(frames)
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        s.record()
        orbit(0, count)
        e.record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t = torch.tensor([s.elapsed_time(e) / 1e3], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    fps = count / float(t)
    if rank == 0:
        print(json.dumps({"metric": "render FPS at 3M Gaussians 3840x2160 (c4 orbit)", "value": round(fps, 3),
                          "unit": "frames/s", "n_gpus": world, "steps": count, "warmup": 16,
                          "ms_per_step": round(float(t) / count * 1e3, 3), "higher_is_better": True,
                          "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                          "data": "synthetic (seeded BASELINE.json config 4 generator)",
                          "config": {"workload": "c4: BASELINE.json configs[3] render-only, the full orbit timed",
                                     "gaussians": n, "resolution": "3840x2160", "frames": len(frames),
                                     "parallelism": f"tile-row sharding x{world}" if world > 1 else "single GPU"},
                          "clocks": clk.summary()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def trainer_launches(counts: dict, steps: int) -> int:
    """Kernels of libtgs.so launched in the timed region: per stage call, the kernel count
    fixed by the host code in csrc/ (checked against the ncu launch list,
    profiles/r01_launches_bench_c3.summary.txt).  Memsets and torch's own kernels are
    not counted."""
    per_call = {"preprocess_fwd": 1,                # k_preprocess_fwd_views (all views)
                # k_bs_init, select, hist, scan, scatter, rank, the idle LSD fallback
                "bin_gaussians": 7,
                # k_seg_count, seg_base, scatter, unit_table, place_count, tile_scan, place_write
                "bin_instances": 7,
                "blend_fwd": 1,                      # k_blend_fwd16w
                "loss": 3,                           # k_ssim_fwd, k_ssim_adj, k_loss_finalize
                "blend_bwd": 1,                      # k_blend_bwd16w
                "preprocess_bwd": 1,                 # k_preprocess_bwd_views (all views)
                "adam": 1}                           # k_adam_groups (all groups)
    return int(sum(per_call[k] * c for k, c in counts.items() if k in per_call))


if __name__ == "__main__":
    main()

"""Summarise ncu --set full reports into profiles/<prefix>_ncu_summary.txt and the per-stage
DRAM traffic JSON that bench.py reports as roofline.traffic.

    python profiles/ncu_summary.py <view.ncu-rep> <step.ncu-rep>

Runs here (no GPU): `ncu -i <rep> --page raw --csv`.
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

STAGE_OF = [  # kernel-name prefix -> bench stage
    ("k_preprocess_fwd", "preprocess_fwd"), ("k_bs_", "bin_gaussians"), ("k_depth_sort", "bin_gaussians"),
    ("k_seg_", "bin_instances"), ("k_scatter", "bin_instances"), ("k_unit_table", "bin_instances"),
    ("k_place_", "bin_instances"), ("k_tile_scan", "bin_instances"), ("k_blend_fwd", "blend_fwd"),
    ("k_ssim_", "loss"), ("k_loss_finalize", "loss"), ("k_blend_bwd", "blend_bwd"),
    ("k_preprocess_bwd", "preprocess_bwd"), ("k_adam", "adam"), ("k_exact", "exact_records"),
]
UNIT = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,  # -> microseconds
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
METRICS = {
    "time_us": ("gpu__time_duration.sum", 1.0),
    "dram_read": ("dram__bytes_read.sum", 1.0),
    "dram_write": ("dram__bytes_write.sum", 1.0),
    "issue_busy_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
    "occupancy_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "regs": ("launch__registers_per_thread", 1.0),
    "fma_pipe_pct": ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "warp_insts": ("smsp__inst_executed.sum", 1.0),
}


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], dict(zip(r[0], r[1]))
    for x in r[2:]:
        d = dict(zip(hdr, x))
        rec = {"kernel": d["Kernel Name"].split("(")[0].replace("void ", "").replace("tgs::", "")}
        for k, (m, scale) in METRICS.items():
            try:
                rec[k] = float(d[m].replace(",", "")) * scale * UNIT.get(units.get(m, ""), 1.0)
            except (KeyError, ValueError):
                rec[k] = None
        yield rec


def stage(name):
    short = name.split("<")[0]
    for pre, st in STAGE_OF:
        if short.startswith(pre):
            return st
    return None


PER_STEP = {"preprocess_fwd", "preprocess_bwd", "adam", "exact_records"}  # one launch per 8-view step (step report)


def main(reps):
    # reps[0]: one view (profile_step.py), reps[1]: one 8-view step (profile_train.py).
    # The per-view stages come from the view report, the per-step ones from the step
    # report only (the view report's single-view preprocess launches are not the step's).
    recs, stage_recs = [], []
    for ri, rep in enumerate(reps):
        for r in rows(rep):
            recs.append(r)
            st = stage(r["kernel"])
            if st and (st in PER_STEP) == (ri == len(reps) - 1 and len(reps) > 1):
                stage_recs.append((st, r))
    lines = ["ncu --set full --clock-control none (one c3 view via profile_step.py; the per-step kernels via",
             "profile_train.py, 8 views).  Cold-cache, serialised replays: compare shares, not absolute times.", "",
             f"{'kernel':34s} {'us':>8s} {'DRAM MB':>9s} {'TB/s':>6s} {'issue%':>7s} {'occ%':>6s} {'fma%':>6s} {'regs':>5s}"]
    per_stage = defaultdict(lambda: {"dram_bytes_per_launch": 0.0, "time_us": 0.0, "kernels": [], "issue_w": 0.0,
                                     "fma_w": 0.0, "insts": 0.0})
    for r in recs:
        mb = ((r["dram_read"] or 0) + (r["dram_write"] or 0)) / 1e6
        tbs = mb / 1e6 / (r["time_us"] * 1e-6) if r["time_us"] else 0
        lines.append(f"{r['kernel'][:34]:34s} {r['time_us']:8.1f} {mb:9.2f} {tbs:6.2f} "
                     f"{r['issue_busy_pct'] or 0:7.1f} {r['occupancy_pct'] or 0:6.1f} {r['fma_pipe_pct'] or 0:6.1f} "
                     f"{int(r['regs'] or 0):5d}")
    for st, r in stage_recs:
        mb = ((r["dram_read"] or 0) + (r["dram_write"] or 0)) / 1e6
        per_stage[st]["dram_bytes_per_launch"] += mb * 1e6
        per_stage[st]["time_us"] += r["time_us"]
        per_stage[st]["kernels"].append(r["kernel"])
        per_stage[st]["issue_w"] += (r["issue_busy_pct"] or 0.0) * r["time_us"]
        per_stage[st]["fma_w"] += (r["fma_pipe_pct"] or 0.0) * r["time_us"]
        per_stage[st]["insts"] += r["warp_insts"] or 0.0
    # a stage's kernels can repeat (the step report profiles two steps): per launch of the
    # stage = the sums over its kernel list divided by the repeat count
    def reps(v):
        names = v["kernels"]
        return max(names.count(k) for k in set(names)) if names else 1
    json.dump({k: {"dram_bytes_per_launch": int(v["dram_bytes_per_launch"] / reps(v)),
                   "time_us": round(v["time_us"] / reps(v), 1),
                   "issue_busy_pct": round(v["issue_w"] / max(v["time_us"], 1e-9), 1),
                   "fma_pipe_pct": round(v["fma_w"] / max(v["time_us"], 1e-9), 1),
                   "warp_insts": int(v["insts"] / reps(v)), "kernels": sorted(set(v["kernels"]), key=v["kernels"].index)}
               for k, v in per_stage.items()},
              open(f"profiles/{PREFIX}_ncu_traffic.json", "w"), indent=1)
    open(f"profiles/{PREFIX}_ncu_summary.txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    # python profiles/ncu_summary.py [--prefix r02] <view.ncu-rep> <step.ncu-rep>
    args = sys.argv[1:]
    PREFIX = "r01"
    if args[:1] == ["--prefix"]:
        PREFIX, args = args[1], args[2:]
    main(args)

"""Builds profiles/<round>_summary.md from a gpu_full.sh run (gpurun_out/):
bench lines, ncu launch lists (kernel shares) and the key metrics of the
`ncu --set full` captures.  Usage: python scripts/make_profiles.py r01"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.path.join(ROOT, "profiles")

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("gpc__cycles_elapsed.avg.per_second", "SM clock (GHz)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("sm__cycles_active.max", "max SM active cycles"),
    ("sm__cycles_active.avg", "avg SM active cycles"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__occupancy_limit_shared_mem", "CTA limit (smem)"),
    ("launch__block_size", "block size"),
    ("launch__grid_size", "grid size"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = OrderedDict()
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        if r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        k = r[hdr.index("Kernel Name")]
        v = float(r[hdr.index("Metric Value")].replace(",", ""))
        unit = r[hdr.index("Metric Unit")]
        v = v / 1e3 if unit in ("nsecond", "ns") else v
        agg.setdefault(k, []).append(v)
    tot = sum(sum(v) for v in agg.values()) or 1.0
    lines = ["| kernel | launches | total us | share | mean us |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        name = k if len(k) < 90 else k[:87] + "..."
        lines.append(f"| `{name}` | {len(v)} | {sum(v):.1f} | {100 * sum(v) / tot:.1f}% | "
                     f"{sum(v) / len(v):.2f} |")
    return "\n".join(lines)


def ncu_metrics(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return "(no data)"
    hdr, units = rows[0], rows[1]
    out = []
    for li, r in enumerate(rows[2:]):
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        out.append(f"\n**launch {li}: `{name[:100]}`**\n\n| metric | value |\n|---|---|")
        for key, label in METRICS:
            if key in hdr:
                i = hdr.index(key)
                out.append(f"| {label} (`{key}`) | {r[i]} {units[i]} |")
    return "\n".join(out)


def bench_line(path):
    try:
        d = json.load(open(path))
    except Exception:  # noqa: BLE001
        return None
    d.pop("rounds", None)
    return d


def main(tag):
    os.makedirs(PROF, exist_ok=True)
    script = sys.argv[2] if len(sys.argv) > 2 else f"scripts/gpu_{tag}_final.sh"
    md = [f"# {tag} — measured on one B200 (gpurun), `{script}`", ""]
    gpu = os.path.join(OUT, "gpu.txt")
    if os.path.exists(gpu):
        md += ["```", open(gpu).read().strip(), open(os.path.join(OUT, "nproc.txt")).read().strip(),
               "```", ""]
    md += ["## bench lines (`python bench.py [--instance X]`; `--impl reference`)", "",
           "| run | value (bounded/s) | ms/step | e2e (bounded/s) | K2 share | roofline frac | cpu baseline |",
           "|---|---|---|---|---|---|---|"]
    for f in ["bench.json", "bench_ref.json", "bench_ta001.json", "bench_ta051.json",
              "bench_ta081.json", "bench_ta101.json", "bench_ta051_tuner.json"]:
        d = bench_line(os.path.join(OUT, f))
        if not d:
            continue
        rf = d.get("roofline") or {}
        cpu = (d.get("cpu_baseline") or {}).get("value")
        e2e = (d.get("e2e") or {}).get("value")
        md.append(f"| {f} | {d['value']:.4g} | {d['ms_per_step']:.4f} | "
                  f"{e2e:.4g} | {rf.get('k2_share_of_round', 0):.3f} | {rf.get('frac', 0):.3f} | "
                  f"{cpu if cpu is None else f'{cpu:.4g}'} |")
        shutil.copy(os.path.join(OUT, f), os.path.join(PROF, f"{tag}_{f}"))
    d = bench_line(os.path.join(OUT, "bench.json"))
    if d and d.get("small_pool_batches"):
        sp = d["small_pool_batches"]
        md += ["", f"### small pools in the default line (`small_pool_batches`: {sp['rounds_per_call']} rounds per "
                   f"explorer call, persistent batch kernel, {sp['l2']})", "",
               "| children per round | device bounded/s | us/round device | wall bounded/s | us/round wall | launches |",
               "|---|---|---|---|---|---|"]
        for T, v in sp["targets"].items():
            md.append(f"| {T} | {v['device_value'] / 1e6:.1f} M | {v['us_per_round_device']:.1f} | "
                      f"{v['wall_value'] / 1e6:.1f} M | {v['us_per_round_wall']:.1f} | {v['gpu_launches']} "
                      f"for {v['rounds']} rounds |")
    header = False
    for f in ["bench_bound_ta101.json", "bench_bound_ta051.json", "bench_bound_ta021.json",
              "bench_bound_ref.json"]:
        d = bench_line(os.path.join(OUT, f))
        if d:
            if not header:
                header = True
                md += ["", "## bound-only stress (`bench.py --mode bound`, K1 over a synthetic pool in HBM)", "",
                       "| run | value (bounded/s) | ms/pass | e2e (bounded/s) | roofline frac | cpu baseline |",
                       "|---|---|---|---|---|---|"]
            rf = d.get("roofline") or {}
            e2e = (d.get("e2e") or {}).get("value")
            cpu = (d.get("cpu_baseline") or {}).get("value")
            md.append(f"| {f} | {d['value']:.4g} | {d['ms_per_step']:.3f} | {e2e:.4g} | "
                      f"{rf.get('frac', 0):.3f} | {cpu if cpu is None else f'{cpu:.4g}'} |")
            shutil.copy(os.path.join(OUT, f), os.path.join(PROF, f"{tag}_{f}"))
    sw = os.path.join(OUT, "sweep_table.md")
    if os.path.exists(sw):
        md += ["", "## Ta021 pool-size sweep (BASELINE configs[1]; `scripts/gpu_sweep.sh`)", "",
               open(sw).read().strip()]
    dr = os.path.join(OUT, "dropin.txt")
    if os.path.exists(dr):
        md += ["", "## reference API driven by the GPU drop-in (`oracle/_ref/dropin_test`)", "", "```",
               open(dr).read().strip(), "```"]
    for lf, title in [("launches.csv", "Ta021 (bench.py --steps 5 --warmup 3)"),
                      ("launches_ta081.csv", "Ta081 (bench.py --instance ta081 --steps 5 --warmup 3)")]:
        p = os.path.join(OUT, lf)
        if os.path.exists(p):
            md += ["", f"## ncu launch list: {title}",
                   "", "`ncu --metrics gpu__time_duration.sum --clock-control none -c 400` (cold, "
                       "serialised: compare shares, not absolute times)", "", launches(p)]
            shutil.copy(p, os.path.join(PROF, f"{tag}_{lf}"))
    for rep, title in [("prof_k2_final.ncu-rep", "K2 (v2, Ta021) and place"),
                       ("prof_k2v2_pool.ncu-rep", "K2 (v2) on a fixed 262K-child Ta021 pool (k2_pool_bench)"),
                       ("prof_k2v3_ta081.ncu-rep", "K2 (v3, Ta081)"),
                       ("prof_k1v2_ta101.ncu-rep", "K1 (v2, 200x20 bound-only pool)"),
                       ("prof_k1v3_ta101.ncu-rep", "K1 (v3, 200x20 bound-only pool of 1 M nodes)"),
                       ("prof_k1v3_ta021.ncu-rep", "K1 (v3, 20x20 bound-only pool of 2 M nodes)"),
                       ("prof_persistent.ncu-rep", "persistent batch kernel (K2 v2, BATCH; one launch = a "
                                                   "batch of 4 K-child Ta021 rounds)")]:
        p = os.path.join(OUT, rep)
        if os.path.exists(p):
            md += ["", f"## ncu --set full: {title}", ncu_metrics(p)]
    extra = []
    for f, title in [("solve_ta001.json", "Ta001 solve() from the identity UB, one context"),
                     ("solve_ta001_group2.json", "Ta001 solve() over an fbb_group of 2 (GPU 0 twice)"),
                     ("exhaust_group2.json", "Ta021 exhaustion at UB 2298 over an fbb_group of 2"),
                     ("exhaust_ta021.json", "Ta021 exhaustion at UB 2298, one context"),
                     ("bench_bound_ta101_max.json", "Ta101 K1 over a pool filling the GPU's HBM")]:
        d = bench_line(os.path.join(OUT, f))
        if not d:
            continue
        keep = {k: d[k] for k in ("value", "explore_seconds", "device_seconds", "exhausted", "optimum",
                                  "incumbent", "bounded", "group", "proof", "config", "cpu_baseline",
                                  "roofline") if k in d}
        extra += ["", f"### {title} (`{f}`)", "", "```json", json.dumps(keep, indent=1)[:3000], "```"]
        shutil.copy(os.path.join(OUT, f), os.path.join(PROF, f"{tag}_{f}"))
    if extra:
        md += ["", "## other configs (solve, group, HBM-filling pool)"] + extra
    for f in ["sanitize_memcheck.txt", "sanitize_racecheck.txt", "sanitize_synccheck.txt"]:
        q = os.path.join(OUT, f)
        if os.path.exists(q):
            lines = open(q).read().strip().splitlines()
            md += ["", f"## {f}", "", "```", "\n".join(lines[-8:]), "```"]
            shutil.copy(q, os.path.join(PROF, f"{tag}_{f}"))
    out = os.path.join(PROF, f"{tag}_summary.md")
    with open(out, "w") as f:
        f.write("\n".join(md) + "\n")
    print(out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r01")

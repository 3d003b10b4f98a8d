"""Turn gpurun_out/ ncu artefacts into the committed summaries under profiles/.

  python tools/summarize_profiles.py --tag r01 --launches gpurun_out/launches.csv \
      --rep gpurun_out/condense_C4.ncu-rep --config C4 [--bench gpurun_out/bench_default.log]

Writes profiles/<tag>_launches.md (per-kernel launch list of the bench command: count, mean, share of step),
profiles/<tag>_<kernel>_<config>.md (key counters + stall hot lines of the one `ncu --set full` capture) and
updates profiles/traffic.json ({config: dram bytes read+write per launch of the dominant kernel}) which
bench.py copies into roofline.traffic.
"""
import argparse
import csv
import json
import os
import subprocess
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe (DMMA) active %"),
    ("sm__ops_path_tensor_src_fp64.sum", "DMMA fp64 operations (FMA) total"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 (DFMA) pipe active %"),
    ("sm__inst_executed.sum", "instructions executed"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers / thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared-memory wavefronts % of peak"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate %"),
]


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    h = rows[hdr]
    tot, cnt = defaultdict(float), defaultdict(int)
    unit = "ns"
    for r in rows[hdr + 1:]:
        d = dict(zip(h, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        k = d["Kernel Name"]
        v = float(d["Metric Value"].replace(",", ""))
        unit = d["Metric Unit"]
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        tot[k] += v * scale
        cnt[k] += 1
    return tot, cnt


def raw_metrics(rep, kernel=None):
    """Counters of one captured launch: the first one, or the first whose name contains `kernel`."""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h, u = r[0], r[1]
    ki = h.index("Kernel Name") if "Kernel Name" in h else None
    v = r[2]
    if kernel and ki is not None:
        v = next((row for row in r[2:] if kernel in row[ki]), r[2])
    return {a: (c, b) for a, b, c in zip(h, u, v)}, v[ki] if ki is not None else "?"


# source files whose change makes a stored traffic figure stale (bench.py recomputes the same hash)
KERNEL_SOURCES = {"sweep_kernel": "condense_sweep.cu", "condense_kernel": "condense.cu", "warp_kernel": "condense_warp.cu",
                  "adjoint_kernel": "adjoint.cu", "backsub_saved_kernel": "solutions.cu", "save_kernel": "solutions.cu",
                  "backsub_kernel": "backsub.cu", "rows_kernel": "condense_rows.cu"}


def source_sha(kname):
    import hashlib
    csrc = os.path.join(ROOT, "paper_1308_3995_b200", "csrc")
    f = next((v for k, v in KERNEL_SOURCES.items() if k in kname), None)
    if f is None:
        return None
    h = hashlib.sha256()
    for name in (f, "dev_common.cuh", "hdg_internal.cuh"):
        h.update(open(os.path.join(csrc, name), "rb").read())
    return h.hexdigest()[:16]


def hot_lines(rep, top=25):
    out = subprocess.run(["python", os.path.join(ROOT, "tools", "ncu_hot.py"), rep, str(top)], capture_output=True,
                         text=True).stdout
    return out


def to_bytes(val, unit):
    f = float(val.replace(",", ""))
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}.get(unit, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tag", required=True)
    ap.add_argument("--launches")
    ap.add_argument("--launch-config", default="C4")
    ap.add_argument("--rep", action="append", default=[])
    ap.add_argument("--config", action="append", default=[])
    ap.add_argument("--note", default="")
    ap.add_argument("--kernel", action="append", default=[], help="per --rep: the captured launch to summarise")
    a = ap.parse_args()
    os.makedirs(PROF, exist_ok=True)
    if a.launches:
        tot, cnt = launches(a.launches)
        path = os.path.join(PROF, f"{a.tag}_launches_{a.launch_config}.md")
        hot = [k for k in tot if any(s in k for s in ("condense_kernel", "sweep_kernel", "warp_kernel", "assemble", "backsub", "pack",
                                                       "accumulate"))]
        step = sum(tot[k] / max(1, cnt[k]) for k in hot)
        with open(path, "w") as f:
            f.write(f"# {a.tag} launch list — `bench.py --config {a.launch_config}` under "
                    f"`ncu --metrics gpu__time_duration.sum --clock-control none`\n\n")
            f.write("Cold-cache, serialised per-launch times (ncu): compare SHARES of the step, not absolutes.\n")
            if a.note:
                f.write(f"\n{a.note}\n")
            f.write("\n| kernel | launches | mean µs | share of hot-path step |\n|---|---|---|---|\n")
            for k in sorted(tot, key=lambda k: -tot[k]):
                m = tot[k] / cnt[k]
                share = f"{100 * m / step:.1f}%" if k in hot else "(not in step: generator / peaks / plan)"
                f.write(f"| `{k[:90]}` | {cnt[k]} | {m:.1f} | {share} |\n")
        print("wrote", path)
    tpath = os.path.join(PROF, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    kernels = a.kernel + [None] * (len(a.rep) - len(a.kernel))
    for rep, cfg, kf in zip(a.rep, a.config, kernels):
        m, kname = raw_metrics(rep, kf)
        short = ("condense_sweep" if "sweep_kernel" in kname else "condense_warp" if "warp_kernel" in kname else
                 "adjoint" if "adjoint" in kname else
                 "condense" if "condense" in kname else "backsub_saved" if "backsub_saved" in kname else
                 "save_solutions" if "save_kernel" in kname else
                 "backsub" if "backsub" in kname else "".join(ch for ch in kname.split("(")[0][-30:] if ch.isalnum()))
        path = os.path.join(PROF, f"{a.tag}_{short}_{cfg}_ncu.md")
        with open(path, "w") as f:
            f.write(f"# {a.tag} — `ncu --set full --clock-control none --import-source on` of `{kname[:100]}` "
                    f"({cfg})\n\n| counter | value | unit |\n|---|---|---|\n")
            for key, label in KEYS:
                if key in m:
                    f.write(f"| {label} (`{key}`) | {m[key][0]} | {m[key][1]} |\n")
            f.write("\nWarp-stall samples by source line (tools/ncu_hot.py):\n\n```\n" + hot_lines(rep) + "```\n")
        if "dram__bytes_read.sum" in m:
            rd = to_bytes(*m["dram__bytes_read.sum"])
            wr = to_bytes(*m["dram__bytes_write.sum"])
            key = cfg if short.startswith("condense") else f"{cfg}_{short}"
            traffic[key] = {"bytes": rd + wr, "kernel": kname[:120], "source_sha": source_sha(kname),
                            "profile": os.path.relpath(path, ROOT)}
        print("wrote", path)
    json.dump(traffic, open(tpath, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()

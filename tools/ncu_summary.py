"""Summarise ncu captures of bench.py into profiles/ (markdown + a JSON the bench reads).

    python tools/ncu_summary.py <tag> [--launches gpurun_out/launches_<tag>.csv]
                                      [--full gpurun_out/prof_gemm_<tag>.ncu-rep]

Launch list: `--metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active...,dram__bytes_*`
(cold, serialised: shares, not absolutes). Full capture: `ncu --set full -k regex:gemm_kernel`.
Writes profiles/<tag>_launches.md, profiles/<tag>_launches.csv (per kernel), and
profiles/<tag>_gemm_traffic.json (mean DRAM bytes per GEMM launch, the roofline `traffic`).
"""
from __future__ import annotations

import argparse
import collections
import csv
import io
import json
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def read_ncu_csv(path):
    text = open(path).read().splitlines()
    start = next(i for i, ln in enumerate(text) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(text[start:]))))
    launches = collections.OrderedDict()
    for r in rows:
        d = launches.setdefault(r["ID"], {"name": r["Kernel Name"], "grid": r["Grid Size"], "block": r["Block Size"]})
        v = r["Metric Value"].replace(",", "")
        try:
            d[r["Metric Name"]] = float(v)
        except ValueError:
            d[r["Metric Name"]] = v
    return list(launches.values())


def short(name: str) -> str:
    name = re.sub(r"\(.*\)$", "", name)
    name = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("jg_gemm::", "")
    return name[:70]


def summarize_launches(tag, path):
    L = read_ncu_csv(path)
    tot = sum(d.get("gpu__time_duration.sum", 0) for d in L)
    agg = collections.OrderedDict()
    for d in L:
        k = short(d["name"])
        a = agg.setdefault(k, {"n": 0, "ns": 0.0, "rd": 0.0, "wr": 0.0, "tc": 0.0})
        a["n"] += 1
        a["ns"] += d.get("gpu__time_duration.sum", 0)
        a["rd"] += d.get("dram__bytes_read.sum", 0)
        a["wr"] += d.get("dram__bytes_write.sum", 0)
        a["tc"] += d.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0) * d.get("gpu__time_duration.sum", 0)
    rows = sorted(agg.items(), key=lambda kv: -kv[1]["ns"])
    out = [f"# {tag} — ncu launch list of the bench command (1 B200)",
           "# gpu__time_duration.sum per launch, --clock-control none, serialised and cold: compare SHARES, not absolutes",
           f"# {len(L)} launches, {tot / 1e6:.2f} ms total", "",
           "| kernel | launches | total ms | share | tensor-pipe active (time-weighted) | DRAM GB/s |",
           "|---|---|---|---|---|---|"]
    for k, a in rows:
        bw = (a["rd"] + a["wr"]) / a["ns"] if a["ns"] else 0.0
        out.append(f"| {k} | {a['n']} | {a['ns'] / 1e6:.3f} | {100 * a['ns'] / tot:.1f}% | "
                   f"{a['tc'] / a['ns'] if a['ns'] else 0:.1f}% | {bw:.0f} |")
    outdir = os.environ.get("NCU_SUMMARY_OUT", os.path.join(ROOT, "profiles"))
    os.makedirs(outdir, exist_ok=True)
    with open(os.path.join(outdir, f"{tag}_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["kernel", "launches", "total_ns", "share", "dram_read_bytes", "dram_write_bytes", "tensor_active_pct"])
        for k, a in rows:
            w.writerow([k, a["n"], int(a["ns"]), round(a["ns"] / tot, 4), int(a["rd"]), int(a["wr"]),
                        round(a["tc"] / a["ns"], 2) if a["ns"] else 0])
    gem = [d for d in L if "gemm_kernel" in d["name"]]
    traffic = None
    if gem:
        traffic = sum(d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0) for d in gem) / len(gem)
        out += ["", f"GEMM launches: {len(gem)}; mean DRAM traffic per launch {traffic / 1e9:.3f} GB "
                f"(read {sum(d.get('dram__bytes_read.sum', 0) for d in gem) / len(gem) / 1e9:.3f} GB)."]
    return out, traffic


def summarize_full(path):
    try:
        txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True,
                             timeout=600).stdout
    except (OSError, subprocess.TimeoutExpired):
        return []
    lines = txt.splitlines()
    if len(lines) < 3:
        return []
    rd = list(csv.reader(io.StringIO("\n".join(lines))))
    hdr, units, data = rd[0], rd[1], rd[2:]
    want = ["gpu__time_duration.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
            "sm__cycles_elapsed.avg.per_second", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "lts__t_sector_hit_rate.pct", "launch__grid_size", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x", "smsp__inst_executed_pipe_uniform.sum"]
    idx = {h: i for i, h in enumerate(hdr)}
    out = ["", "## Top kernel (`ncu --set full -k regex:gemm_kernel`)", "",
           "| metric | " + " | ".join(f"launch {r[idx['ID']]}" for r in data) + " |",
           "|---|" + "---|" * len(data)]
    for w in want:
        if w in idx:
            out.append(f"| {w} ({units[idx[w]]}) | " + " | ".join(r[idx[w]] for r in data) + " |")
    if "Kernel Name" in idx:
        out.append("| kernel | " + " | ".join(short(r[idx['Kernel Name']]) for r in data) + " |")
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--full")
    a = ap.parse_args()
    lp = a.launches or os.path.join(ROOT, "gpurun_out", f"launches_{a.tag}.csv")
    fp = a.full or os.path.join(ROOT, "gpurun_out", f"prof_gemm_{a.tag}.ncu-rep")
    out, traffic = summarize_launches(a.tag, lp)
    if os.path.exists(fp):
        out += summarize_full(fp)
    outdir = os.environ.get("NCU_SUMMARY_OUT", os.path.join(ROOT, "profiles"))
    os.makedirs(outdir, exist_ok=True)
    md = os.path.join(outdir, f"{a.tag}_launches.md")
    open(md, "w").write("\n".join(out) + "\n")
    json.dump({"tag": a.tag, "kernel": "gemm_kernel (all launches of one step)",
               "traffic_bytes_per_launch": traffic, "source": os.path.basename(lp)},
              open(os.path.join(outdir, f"{a.tag}_gemm_traffic.json"), "w"), indent=1)
    print("\n".join(out))


if __name__ == "__main__":
    main()

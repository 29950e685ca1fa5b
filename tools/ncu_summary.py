"""Summarise ncu outputs into profiles/: a launch list (gpu__time_duration per launch) and the
key metrics of a `--set full` capture, one row per profiled kernel launch.

    python tools/ncu_summary.py --launches gpurun_out/launches.csv --full gpurun_out/prof.ncu-rep --out profiles/r1_x
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size", "launch__occupancy_limit_registers"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, ni = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    return [{"kernel": r[ki].split("(")[0], "ns": float(r[mi].replace(",", ""))} for r in rows[hi + 1:]
            if len(r) > mi and r[ni] == "gpu__time_duration.sum"]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for k in KEYS:
            if k in h:
                v = r[h.index(k)].replace(",", "")
                try:
                    d[k] = float(v)
                except ValueError:
                    d[k] = v
                d[k + ".unit"] = units[h.index(k)]
        out.append(d)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--out", required=True)
    a = ap.parse_args()
    res = {}
    if a.launches:
        L = launches(a.launches)
        res["launches"] = L
        agg = {}
        for x in L:
            agg.setdefault(x["kernel"], []).append(x["ns"])
        res["launch_summary"] = {k: {"n": len(v), "mean_us": sum(v) / len(v) / 1e3} for k, v in agg.items()}
    if a.full:
        res["full"] = full(a.full)
    json.dump(res, open(a.out + ".json", "w"), indent=1)
    lines = [f"# ncu summary {a.out}", ""]
    if "launch_summary" in res:
        lines += ["## launch list (gpu__time_duration, cold-cache serialised)", "", "| kernel | launches | mean us |", "|---|---|---|"]
        for k, v in res["launch_summary"].items():
            lines.append(f"| {k} | {v['n']} | {v['mean_us']:.2f} |")
    if "full" in res:
        lines += ["", "## --set full capture", "",
                  "| kernel | us | DRAM rd MB | DRAM wr MB | DRAM % peak | L2 hit % | issue active % | warps active % | regs |",
                  "|---|---|---|---|---|---|---|---|---|"]
        for d in res["full"]:
            def g(k, s=1.0):
                v = d.get(k)
                return f"{v * s:.1f}" if isinstance(v, float) else str(v)
            t = d.get("gpu__time_duration.sum")
            tu = d.get("gpu__time_duration.sum.unit", "")
            us = t / 1e3 if tu == "nsecond" else (t if tu == "usecond" else t)
            rd = d.get("dram__bytes_read.sum"); ru = d.get("dram__bytes_read.sum.unit", "")
            wr = d.get("dram__bytes_write.sum"); wu = d.get("dram__bytes_write.sum.unit", "")
            sc = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
            lines.append(f"| {d['kernel']} | {us:.1f} | {rd * sc.get(ru, 1):.1f} | {wr * sc.get(wu, 1):.1f} | "
                         f"{g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')} | {g('lts__t_sector_hit_rate.pct')} | "
                         f"{g('smsp__issue_active.avg.pct_of_peak_sustained_active')} | "
                         f"{g('sm__warps_active.avg.pct_of_peak_sustained_active')} | {g('launch__registers_per_thread')} |")
    open(a.out + ".md", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))

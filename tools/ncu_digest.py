"""Digest an ncu report into small text: key raw metrics + the source lines with most warp stall samples."""
import csv, io, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
KEYS = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed", "local_", "smsp__pcsamp_warps_issue_stalled",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__cycles_active.avg", "l1tex__data_pipe_lsu_wavefronts_mem_shared",
        "smsp__sass_inst_executed_op_local", "l1tex__t_sectors_pipe_lsu_mem_local", "smsp__average_warp_latency_issue_stalled")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
with open(out, "w") as f:
    if len(rows) > 2:
        hdr = rows[0]
        for r in rows[2:]:
            f.write("launch " + " ".join(r[:3]) + "\n")
            for i, h in enumerate(hdr):
                if any(k in h for k in KEYS) and i < len(r):
                    f.write(f"  {h} = {r[i]}\n")
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"], capture_output=True,
                         text=True).stdout
    srows = list(csv.reader(io.StringIO(src)))
    if srows:
        h = srows[0]
        f.write("source columns: " + "|".join(h) + "\n")
        try:
            si = next(i for i, x in enumerate(h) if "Warp Stall Sampling (All" in x)
        except StopIteration:
            si = None
        body = [r for r in srows[1:] if len(r) == len(h)]
        if si is not None:
            def num(x):
                try:
                    return float(x.replace(",", ""))
                except ValueError:
                    return 0.0
            tot = sum(num(r[si]) for r in body) or 1.0
            for r in sorted(body, key=lambda r: -num(r[si]))[:60]:
                f.write(f"{num(r[si]) / tot:6.3f} " + " | ".join(x[:140] for x in r[:3]) + "\n")

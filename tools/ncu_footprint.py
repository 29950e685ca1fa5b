"""Executed-code footprint of one kernel launch in an ncu report (--import-source, source page): the SASS
bytes executed at least once, split by how often (warp-level executions per instruction), and the
instruction-fetch stalls.  Code that runs once per launch is fetched cold from L2 every launch
(tools/icache_bench.cu: ~0.27 us per KB of straight-line code), so its size is a latency cost.
    python tools/ncu_footprint.py report.ncu-rep <kernel-name-substring> [nth-match]"""
import csv, io, subprocess, sys

rep, want = sys.argv[1], sys.argv[2]
nth = int(sys.argv[3]) if len(sys.argv) > 3 else 0  # [4]: optional per-instruction CSV
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks = txt.split('"Kernel Name",')
seen = 0
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if want not in name:
        continue
    if seen != nth:
        seen += 1
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    h = rows[0]
    ie = h.index("Instructions Executed")
    si = h.index("Warp Stall Sampling (All Samples)")
    body = [r for r in rows[1:] if len(r) > ie]
    tot = len(body)
    ex = [(float(r[ie] or 0), float(r[si] or 0)) for r in body]
    print(name[:100])
    print(f"  SASS instructions in the kernel: {tot} ({tot * 16 / 1024:.1f} KB)")
    bins = [(1, 600), (600, 4000), (4000, 20000), (20000, 1e18)]
    for lo, hi in bins:
        sel = [e for e in ex if lo <= e[0] < hi]
        print(f"  executed {lo:>6}..{hi:<8.0f} times (warp-level): {len(sel):6d} instructions = {len(sel) * 16 / 1024:7.1f} KB, "
              f"stall samples {sum(e[1] for e in sel):.0f}")
    run = sum(1 for e in ex if e[0] > 0)
    print(f"  executed at least once: {run} instructions = {run * 16 / 1024:.1f} KB")
    if len(sys.argv) > 4:  # per-instruction dump: offset from the kernel's first instruction, executions
        ai = h.index("Address")
        base = min(int(r[ai], 16) for r in body)
        with open(sys.argv[4], "w") as f:
            for r in body:
                f.write(f"{int(r[ai], 16) - base},{float(r[ie] or 0):.0f},{float(r[si] or 0):.0f}\n")
    break

"""Top stall-sampled SASS instructions of one kernel launch in an ncu report.
    python tools/ncu_hot.py report.ncu-rep <kernel-name-substring> [nth-match] [top]"""
import csv, io, subprocess, sys
rep, want = sys.argv[1], sys.argv[2]
nth = int(sys.argv[3]) if len(sys.argv) > 3 else 0
ntop = int(sys.argv[4]) if len(sys.argv) > 4 else 30
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
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
    si = h.index("Warp Stall Sampling (All Samples)")
    ai, src = h.index("Address"), h.index("Source")
    ie = h.index("Instructions Executed")
    body = [r for r in rows[1:] if len(r) > si]
    tot = sum(float(r[si] or 0) for r in body)
    print(name[:110], "| samples", tot, "| instructions", sum(float(r[ie] or 0) for r in body))
    for r in sorted(body, key=lambda r: -float(r[si] or 0))[:ntop]:
        print(f"{float(r[si] or 0):7.0f} {100 * float(r[si] or 0) / max(tot, 1):5.1f}%  {r[ai]:>6} {r[src].strip()[:90]}")
    break

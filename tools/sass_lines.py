"""Join an ncu per-instruction dump (tools/ncu_footprint.py ... out.csv: offset,executions,stall samples) with
the line info of the same build's SASS (nvdisasm -gi), and print where the code that runs once per
launch comes from: bytes executed rarely (the cold-fetched tail) per source line of tk_kernels.cuh.
    python tools/sass_lines.py <libtk.so> <mangled kernel name> <pcs.csv> [max_exec]"""
import collections, os, re, subprocess, sys, tempfile

so, fn, pcs = sys.argv[1], sys.argv[2], sys.argv[3]
max_exec = float(sys.argv[4]) if len(sys.argv) > 4 else 4000
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-gi", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
start = txt.index(f".text.{fn}:")
end = txt.find("\n.text.", start + 10)
body = txt[start:end if end > 0 else None]
loc = {}
cur = "?"
fresh = True  # the first location line after an instruction is the innermost one
for ln in body.splitlines():
    m = re.match(r'\s*//## File ".*/([^/"]+)", line (\d+)(?: inlined at ".*/([^/"]+)", line (\d+))?', ln)
    if m:
        if fresh:
            cur = f"{m.group(1)}:{m.group(2)}"
            fresh = False
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m:
        loc[int(m.group(1), 16)] = cur
        fresh = True
rows = [tuple(float(x) for x in l.split(",")) for l in open(pcs) if l.strip()]
by = collections.Counter()
stall = collections.Counter()
tot = 0
for off, ex, st in rows:
    if 0 < ex <= max_exec:
        by[loc.get(int(off), "?")] += 16
        stall[loc.get(int(off), "?")] += st
        tot += 16
print(f"{tot / 1024:.1f} KB of SASS executed 1..{max_exec:.0f} times (warp-level); top source lines:")
for k, v in by.most_common(60):
    print(f"  {v:6d} B  stall {stall[k]:5.0f}  {k}")

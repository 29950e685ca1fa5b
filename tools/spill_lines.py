"""Where the local-memory (LDL/STL) instructions of one kernel come from (needs a -lineinfo build)."""
import os, re, subprocess, sys, tempfile
so = os.path.realpath(sys.argv[1] if len(sys.argv) > 1 else "paper_2010_10458_b200/libtk.so")
fn = sys.argv[2] if len(sys.argv) > 2 else "_ZN2tk10k_compressILb1ELi0ELi0EEEvNS_5FusedE"
lo, hi = (int(sys.argv[3]), int(sys.argv[4])) if len(sys.argv) > 4 else (0, 10 ** 9)
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=d, capture_output=True)
cub = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")][0]
out = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(out) if l.startswith(f".text.{fn}:"))
end = next((i for i in range(start + 1, len(out)) if out[i].startswith(".text.") or out[i].startswith("\t.section")), len(out))
cur, cnt = None, {}
for l in out[start:end]:
    if "//##" in l:
        m = re.search(r'File "(.*?)", line (\d+)', l)
        cur = (os.path.basename(m.group(1)), int(m.group(2))) if m else cur
        continue
    if re.search(r"\b(LDL|STL)", l):
        cnt[cur] = cnt.get(cur, 0) + 1
src = open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2010_10458_b200", "csrc", "tk_kernels.cuh")).read().splitlines()
for k, v in sorted(cnt.items(), key=lambda x: -x[1])[:40]:
    if k and k[0] == "tk_kernels.cuh" and lo <= k[1] <= hi:
        print(v, k[1], src[k[1] - 1].strip()[:110])
    elif k and k[0] != "tk_kernels.cuh":
        print(v, k)

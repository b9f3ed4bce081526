"""Per-CUDA-source-line dynamic instruction counts and stall samples of one kernel (dev tool).
Joins the ncu source page (SASS, in address order) with nvdisasm -g line info of the same object.
    python tools/ncu_lines.py <rep.ncu-rep> <object.o> <kernel-substring> [top]"""
import collections, csv, io, os, re, subprocess, sys, tempfile
rep, obj, kern = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO("\n".join(out.splitlines()[1:]))))
hdr = rows[0]; ix = {h: i for i, h in enumerate(hdr)}
prof = []
for r in rows[1:]:
    if len(r) < len(hdr): continue
    prof.append((int(r[ix["Address"]], 16), r[ix["Source"]].strip(), int(float(r[ix["Instructions Executed"]] or 0)),
                 int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))))
prof.sort()
base = prof[0][0]
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
on, line, addr2line = False, None, {}
for l in txt.splitlines():
    if ".text." in l and "section" in l: on = kern in l
    if not on: continue
    m = re.search(r"line (\d+)", l)
    if m and "//##" in l:
        line = int(m.group(1)) if os.path.basename(os.environ.get("SRC", "kernels.cu")) in l else line
        continue
    m = re.search(r"/\*([0-9a-f]{4,})\*/\s+\S", l)
    if m: addr2line[int(m.group(1), 16)] = line
inst = collections.Counter(); samp = collections.Counter(); ti = ts = 0
ops = collections.defaultdict(collections.Counter)
for a, src, n, s in prof:
    ln = addr2line.get(a - base, -1)
    inst[ln] += n; samp[ln] += s; ti += n; ts += s
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    ops[ln][op.rstrip(";")] += n
src = open(os.environ.get("SRC", os.path.join(os.path.dirname(os.path.abspath(obj)), "..", "csrc", "kernels.cu"))).read().splitlines()
print(f"{'line':>5} {'%inst':>6} {'%samp':>6}  source")
for ln, n in sorted(inst.items(), key=lambda kv: -kv[1])[:top]:
    s = src[ln - 1].strip()[:90] if 0 < ln <= len(src) else "?"
    top3 = ", ".join(f"{o} {c / n * 100:.0f}%" for o, c in ops[ln].most_common(3))
    print(f"{ln:5d} {n / ti * 100:6.2f} {samp[ln] / ts * 100:6.2f}  {s[:70]:70s} | {top3}")

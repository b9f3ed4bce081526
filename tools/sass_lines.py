"""Static SASS opcode histogram per CUDA source line of one kernel (dev tool; needs -lineinfo).
    python tools/sass_lines.py <object.o> <kernel-substring> [opcode-regex]"""
import collections, os, re, subprocess, sys, tempfile
obj, kern = sys.argv[1], sys.argv[2]
pat = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
txt = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cub)], capture_output=True, text=True).stdout
on, line, by = False, None, collections.defaultdict(collections.Counter)
for l in txt.splitlines():
    if ".text." in l and "section" in l:
        on = kern in l
    if not on:
        continue
    m = re.search(r"line (\d+)", l)
    if m and "//##" in l:
        line = int(m.group(1))
        continue
    m = re.search(r"/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", l)
    if m and line and (pat is None or pat.search(m.group(2))):
        by[line][m.group(2)] += 1
for ln in sorted(by):
    print(ln, dict(by[ln]))

"""Dynamic SASS opcode histogram + stall samples per opcode from an ncu report (dev tool).
    python tools/sass_profile.py rep.ncu-rep [kernel-regex]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
ops = collections.Counter(); samp = collections.Counter(); tot = 0; stot = 0
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
st_by = collections.defaultdict(collections.Counter)
for r in rows[1:]:
    if len(r) < len(hdr): continue
    src = r[ix["Source"]].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"): op = src.split()[1]
    op = op.rstrip(";")
    n = int(float(r[ix["Instructions Executed"]] or 0))
    s = int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
    ops[op] += n; tot += n; samp[op] += s; stot += s
    for h in stalls:
        v = float(r[ix[h]] or 0)
        if v: st_by[op][h] += v
print(f"total warp-instr {tot:.3e}, samples {stot}")
for op, n in ops.most_common(45):
    top = ", ".join(f"{k[6:]}={v/max(1,samp[op])*100:.0f}%" for k, v in st_by[op].most_common(3))
    print(f"{op:28s} {n/tot*100:6.2f}% instr  {samp[op]/max(1,stot)*100:6.2f}% samples  [{top}]")

"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into per-kernel shares (dev tool)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[i], rows[i + 1:]
ix = {h: k for k, h in enumerate(hdr)}
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}
t, n = collections.Counter(), collections.Counter()
for r in data:
    if len(r) < len(hdr) or r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    name = r[ix["Kernel Name"]].split("(")[0]
    t[name] += float(r[ix["Metric Value"]].replace(",", "")) * scale.get(r[ix["Metric Unit"]], 1.0)
    n[name] += 1
tot = sum(t.values())
print(f"{'kernel':45s} {'launches':>8s} {'total_ms':>12s} {'avg_ms':>10s} {'share':>7s}")
for k, v in t.most_common():
    print(f"{k:45s} {n[k]:8d} {v / 1e3:12.3f} {v / 1e3 / n[k]:10.4f} {v / tot * 100:6.1f}%")
print("(cold-cache, serialised ncu timings: compare shares, not absolutes)")

"""Summarise an ncu --csv launch list (gpu__time_duration.sum per kernel)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
h = rows[hdr]
ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
tot, cnt = collections.defaultdict(float), collections.Counter()
seq = []
for r in rows[hdr + 1:]:
    if len(r) <= vi:
        continue
    v = float(r[vi].replace(",", "")) * {"nsecond": 1, "ns": 1, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6}.get(r[ui], 1)
    name = r[ki].split("(")[0].split("<")[0]
    tot[name] += v
    cnt[name] += 1
    seq.append((name, v))
T = sum(tot.values())
print(f"{'kernel':28s} {'n':>5s} {'total ms':>10s} {'avg us':>10s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:28s} {cnt[k]:5d} {tot[k]/1e6:10.3f} {tot[k]/cnt[k]/1e3:10.2f} {tot[k]/T:6.1%}")
if len(sys.argv) > 2:
    for name, v in seq[: int(sys.argv[2])]:
        print(f"  {name:28s} {v/1e3:9.2f} us")

"""Summarise an ncu --csv launch list (gpu__time_duration.sum): count, total and mean time per kernel."""
import collections, csv, sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
agg = collections.OrderedDict()
for d in data:
    k = d["Kernel Name"].split("(")[0][:56]
    v = float(d["Metric Value"].replace(",", "")) * scale.get(d["Metric Unit"], 1.0)
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
print(f"{'kernel':56s} {'count':>6s} {'total ms':>9s} {'share':>6s} {'mean us':>9s}")
for k, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:56s} {c:6d} {t / 1000:9.2f} {t / tot:6.1%} {t / c:9.1f}")
print(f"total {tot / 1000:.2f} ms over {len(data)} launches")

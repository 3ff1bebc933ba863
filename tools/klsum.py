"""Summarise an ncu launch-list CSV: total us per kernel name, launches, us per launch."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
h = rows[i]
c, t = collections.Counter(), collections.defaultdict(float)
for r in rows[i + 1:]:
    d = dict(zip(h, r))
    if d.get("Metric Name") != "gpu__time_duration.sum":
        continue
    k = d["Kernel Name"].split("(")[0]
    c[k] += 1
    t[k] += float(d["Metric Value"].replace(",", "")) / 1e3
print("==", sys.argv[2] if len(sys.argv) > 2 else sys.argv[1], f"total {sum(t.values()):.1f} us")
for k, v in sorted(t.items(), key=lambda x: -x[1])[:16]:
    print(f"  {v:9.1f} us  x{c[k]:<4d} {v / c[k]:8.1f} us/launch  {k}")

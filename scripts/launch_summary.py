"""Summarise an ncu --csv launch list: per launch of the last evaluation, duration (us) and other metrics."""
import collections, csv, io, sys
txt = open(sys.argv[1]).read()
rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
by = collections.OrderedDict()
for r in rows:
    d = by.setdefault(r["ID"], {"k": r["Kernel Name"][:24] + r["Grid Size"]})
    d[r["Metric Name"]] = r["Metric Value"]
items = list(by.values())
# the last complete evaluation: last pmat launch followed by a ratio/reduce launch
starts = [i for i, v in enumerate(items) if "pmat" in v["k"]]
ends = [i for i, v in enumerate(items) if "ratio" in v["k"] or "reduce" in v["k"]]
start = max([s for s in starts if any(e > s for e in ends)] or [0])
stop = min([e for e in ends if e > start] or [len(items) - 1])
tot = collections.defaultdict(float)
for v in items[start:stop + 1]:
    extra = {k.split(".")[0][-28:]: v[k] for k in v if k not in ("k", "gpu__time_duration.sum")}
    print(f"{v['k']:40s} {float(v['gpu__time_duration.sum'])/1000:8.1f} us  {extra}")
    tot[v["k"][:18]] += float(v["gpu__time_duration.sum"]) / 1000
print({k: round(t, 1) for k, t in tot.items()}, "total", round(sum(tot.values()), 1))

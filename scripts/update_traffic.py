"""Refresh profiles/ncu_traffic.json (the bench's roofline `traffic`) from ncu output.

  dengue fp64: dram__bytes_read.sum + dram__bytes_write.sum of the traversal
               kernel in an ncu --set full capture (gpurun_out/prof_trav.ncu-rep)
  MMM:         the same metrics of the traversal launch in a launch list
  yeast codon: those bytes summed over the launches of one evaluation
usage: python scripts/update_traffic.py [gpurun_out]"""
import collections, csv, io, json, os, subprocess, sys

out_dir = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path = os.path.join(root, "profiles", "ncu_traffic.json")
d = json.load(open(path)) if os.path.exists(path) else {}
d["_what"] = ("DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) per launch of the dominant kernel "
              "(per evaluation for the multi-launch codon path), from ncu captures under profiles/r01/.")


def raw_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    return dict(zip(rows[0], rows[2])), dict(zip(rows[0], rows[1]))


def to_bytes(v, unit):
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1)
    return int(float(v.replace(",", "")) * scale)


rep = os.path.join(out_dir, "prof_trav.ncu-rep")
if os.path.exists(rep):
    v, u = raw_metrics(rep)
    rd = to_bytes(v["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
    wr = to_bytes(v["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
    d["config1_fp64"] = {"bytes": rd + wr, "read": rd, "write": wr, "kernel": v.get("Kernel Name", "traverse_small_kernel"),
                         "source": "profiles/r01/ncu_traverse_dengue_fp64.txt (ncu --set full)"}


def launches(fn):
    txt = open(fn).read()
    rows = list(csv.DictReader(io.StringIO(txt[txt.index('"ID"'):])))
    by = collections.OrderedDict()
    for r in rows:
        e = by.setdefault(r["ID"], {"k": r["Kernel Name"]})
        e[r["Metric Name"]] = (r["Metric Value"], r["Metric Unit"])
    return list(by.values())


fn = os.path.join(out_dir, "launches_yeast.csv")
if os.path.exists(fn) and not os.path.exists(os.path.join(out_dir, "prof_flow.ncu-rep")):
    items = launches(fn)
    starts = [i for i, e in enumerate(items) if "pmat" in e["k"]]
    ends = [i for i, e in enumerate(items) if "ratio" in e["k"]]
    s = max(x for x in starts if any(y > x for y in ends))
    t = min(y for y in ends if y > s)
    tot = sum(to_bytes(*e["dram__bytes_read.sum"]) + to_bytes(*e["dram__bytes_write.sum"]) for e in items[s:t + 1])
    d["config3_fp64"] = {"bytes": tot, "kernel": f"codon pmat + level kernels + ratio ({t - s + 1} launches, one evaluation)",
                         "source": "profiles/r01/ncu_launches_yeast.csv"}
# codon flow kernel (the dominant launch since the one-launch schedule): ncu --set full captures
for cfg, name in ((3, "prof_flow"), (4, "prof_flow_wnv"), (5, "prof_flow_s122")):
    rep = os.path.join(out_dir, name + ".ncu-rep")
    if os.path.exists(rep):
        v, u = raw_metrics(rep)
        rd = to_bytes(v["dram__bytes_read.sum"], u["dram__bytes_read.sum"])
        wr = to_bytes(v["dram__bytes_write.sum"], u["dram__bytes_write.sum"])
        d[f"config{cfg}_fp64"] = {"bytes": rd + wr, "read": rd, "write": wr,
                                  "kernel": v.get("Kernel Name", "codon_flow_kernel"),
                                  "source": f"profiles/r01/ncu_flow_config{cfg}.txt (ncu --set full)"}
fn = os.path.join(out_dir, "launches_mmm.csv")
if os.path.exists(fn):
    tr = [e for e in launches(fn) if "traverse" in e["k"]][-1]
    rd, wr = to_bytes(*tr["dram__bytes_read.sum"]), to_bytes(*tr["dram__bytes_write.sum"])
    d["config2_fp64"] = {"bytes": rd + wr, "read": rd, "write": wr, "kernel": tr["k"], "source": "profiles/r01/ncu_launches_mmm.csv"}
json.dump(d, open(path, "w"), indent=1)
print(json.dumps(d, indent=1))

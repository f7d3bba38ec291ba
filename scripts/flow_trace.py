"""Flow-kernel item trace (PG_FLOW_TRACE) of one codon evaluation: per task
level, when its items were taken / became ready / finished (us from the first
take), and the mean item phases.  Usage: flow_trace.py <config> <virtual shards>"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_04390_b200 as pg  # noqa: E402
import phylo_synth as ps  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 8
path = "gpurun_out/flow_trace.bin"
os.environ["PG_FLOW_TRACE"] = path
pb = ps.make_config(cfg)
C = len(pb.pattern_weights)
lo, hi = pg.shard_range(C, shards, 0) if shards > 1 else (0, C)
inst = pg.from_problem(pb, lo=lo, hi=hi)
for _ in range(5):
    inst.compute()
t = np.fromfile(path, dtype=np.uint64).reshape(-1, 8).astype(np.int64)
info = inst.plan_info()
t0 = t[:, 1].min()
take, ready, done = (t[:, 1] - t0) / 1e3, (t[:, 2] - t0) / 1e3, (t[:, 3] - t0) / 1e3
R = len(pb.cat_rates)
ntiles = (hi - lo + 31) // 32
tch = info.get("flow_tiles", 1) or 1
nch = (ntiles + tch - 1) // tch
per_task = R * nch
ntask = len(t) // per_task
print(f"items {len(t)}  tasks {ntask}  span {done.max():.1f} us  mean wait {np.mean(ready - take):.2f} us  "
      f"mean run {np.mean(done - ready):.2f} us  SMs used {len(np.unique(t[:, 0]))}")
ph = np.where(t[:, 4:8] > 0, (t[:, 4:8] - t0) / 1e3, np.nan)
post = np.arange(len(t)) < info.get("npost_items", 0)
def phase_means(sel, label):
    r0, p0, p1, p2, end = ready[sel], ph[sel, 0], ph[sel, 1], ph[sel, 2], ph[sel, 3]
    print(f"{label}: loads {np.nanmean(p0 - r0):.2f}  ph1 {np.nanmean(p1 - p0):.2f}  ph2 {np.nanmean(p2 - p1):.2f}  "
          f"rest {np.nanmean(end - np.where(np.isnan(p2), p1, p2)):.2f}  publish {np.mean(done[sel] - end):.2f} us")
rows = []
for k in range(ntask):
    s = slice(k * per_task, (k + 1) * per_task)
    rows.append((k, take[s].min(), ready[s].min(), ready[s].max(), done[s].max(), np.mean(done[s] - ready[s])))
npost_task = sum(1 for k in range(ntask) if not np.isnan(ph[k * per_task, 1]) and np.isnan(ph[k * per_task, 2]))
isp = np.isnan(ph[:, 2])
phase_means(isp, "post items (loads = wait+stage, ph1 = GEMM, rest = epilogue)")
phase_means(~isp, "pre items (loads, ph1 = Eq.8 GEMMs, ph2 = x form, rest = q GEMMs)")
for k, a, b, c, d, m in rows:
    print(f"task {k:3d}  take {a:7.1f}  ready {b:7.1f}..{c:7.1f}  done {d:7.1f}  run/item {m:6.2f}")

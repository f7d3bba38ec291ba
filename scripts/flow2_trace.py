"""codon_flow2_kernel item trace (PG_FLOW_TRACE) of one evaluation: per item
{smid, claim, inputs ready, stage full (consumers start), GEMM done, published,
released, cta}; prints the mean phase latencies and, per task (tree level
entry), when its items became ready / finished.
Usage: flow2_trace.py <config> <virtual shards>"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_04390_b200 as pg  # noqa: E402
import phylo_synth as ps  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
shards = int(sys.argv[2]) if len(sys.argv) > 2 else 8
path = f"gpurun_out/flow2_trace_{cfg}_{shards}.bin"
os.environ["PG_FLOW_TRACE"] = path
pb = ps.make_config(cfg)
C = len(pb.pattern_weights)
lo, hi = pg.shard_range(C, shards, 0) if shards > 1 else (0, C)
inst = pg.from_problem(pb, lo=lo, hi=hi)
for _ in range(5):
    inst.compute()
info = inst.plan_info()
t = np.fromfile(path, dtype=np.uint64).reshape(-1, 8).astype(np.int64)
R = len(pb.cat_rates)
ntiles = (hi - lo + 31) // 32
split = os.environ.get("PG_FLOW_SPLIT", "1" if ntiles * R < 296 else "0") != "0"
npost = pb.n_tips - 1
n_items = npost * R * ntiles * (3 if split else 2)
t = t[:n_items]
# per task rows: post tasks R*ntiles items, pre tasks (2 if split) R*ntiles
bounds = [k * R * ntiles for k in range(npost + 1)]
bounds += [bounds[-1] + (k + 1) * R * ntiles * (2 if split else 1) for k in range(npost)]
ntask = len(bounds) - 1
t0 = t[:, 1].min()
claim, ready, full, gemm, pub, end = [(t[:, i] - t0) / 1e3 for i in range(1, 7)]
print(f"config {cfg} shards {shards}: items {len(t)} tasks {ntask} span {end.max():.1f} us  CTAs {len(np.unique(t[:, 7]))}"
      f"  plan {info}")
print(f"mean us: claim->ready {np.mean(ready - claim):.2f}  ready->full {np.mean(full - ready):.2f}  "
      f"full->gemm {np.mean(gemm - full):.2f}  gemm->pub {np.mean(pub - gemm):.2f}  pub->end {np.mean(end - pub):.2f}  "
      f"full->end {np.mean(end - full):.2f}")
npost = info.get("npost", None)
for k in range(ntask):
    s = slice(bounds[k], bounds[k + 1])
    print(f"task {k:3d}  claim {claim[s].min():7.1f}  ready {ready[s].min():7.1f}..{ready[s].max():7.1f}  "
          f"full {full[s].min():7.1f}..{full[s].max():7.1f}  pub {pub[s].max():7.1f}  end {end[s].max():7.1f}  "
          f"item {np.mean(end[s] - full[s]):5.2f} (gemm {np.mean(gemm[s] - full[s]):5.2f})")

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
# task order of schedule.cpp: post tasks by height, pre tasks by depth (stable
# in op order); a split pre task has one item group per child only when both
# children are internal
N = pb.n_tips
ops = np.asarray(pb.ops)
height, depth = {}, {}
for d, a_, b_ in ops:
    height[d] = 1 + max(height.get(a_, 0), height.get(b_, 0))
depth[ops[-1][0]] = 0
for d, a_, b_ in ops[::-1]:
    depth[a_] = depth[b_] = depth[d] + 1
post_order = sorted(range(len(ops)), key=lambda o: (height[ops[o][0]], o))
pre_order = sorted(range(len(ops)), key=lambda o: (depth[ops[o][0]], -o))
bounds = [0]
for o in post_order:
    bounds.append(bounds[-1] + R * ntiles)
for o in pre_order:
    two = split and ops[o][1] >= N and ops[o][2] >= N
    bounds.append(bounds[-1] + R * ntiles * (2 if two else 1))
t = t[:bounds[-1]]
ntask = len(bounds) - 1
t0 = t[:, 1].min()
claim, ready, full, gemm, pub, end = [(t[:, i] - t0) / 1e3 for i in range(1, 7)]
print(f"config {cfg} shards {shards}: items {len(t)} tasks {ntask} span {end.max():.1f} us  CTAs {len(np.unique(t[:, 7]))}"
      f"  plan {info}")
print(f"mean us: claim->ready {np.mean(ready - claim):.2f}  ready->full {np.mean(full - ready):.2f}  "
      f"full->gemm {np.mean(gemm - full):.2f}  gemm->pub {np.mean(pub - gemm):.2f}  pub->end {np.mean(end - pub):.2f}  "
      f"full->end {np.mean(end - full):.2f}")
npi = npost * R * ntiles
for name, sl in (("post", slice(0, npi)), ("pre", slice(npi, None))):
    print(f"{name:4s} items {len(t[sl])}: claim->ready {np.mean((ready - claim)[sl]):.2f}  ready->full "
          f"{np.mean((full - ready)[sl]):.2f}  full->gemm {np.mean((gemm - full)[sl]):.2f}  gemm->pub "
          f"{np.mean((pub - gemm)[sl]):.2f}  pub->end {np.mean((end - pub)[sl]):.2f}  full->end {np.mean((end - full)[sl]):.2f}")
# consumer duty per CTA: time between one item's end and the next item's full
cta = t[:, 7]
gaps, busy = [], 0.0
for c in np.unique(cta):
    ii = np.where(cta == c)[0]
    ii = ii[np.argsort(full[ii])]
    gaps += list(full[ii][1:] - end[ii][:-1])
    busy += float(np.sum(end[ii] - full[ii]))
print(f"consumer idle between items: mean {np.mean(gaps):.2f} us; consumers busy {busy / (len(np.unique(cta)) * end.max()):.3f} of span")
if os.environ.get("TRACE_SUMMARY_ONLY"):
    sys.exit(0)
for k in range(ntask):
    s = slice(bounds[k], bounds[k + 1])
    print(f"task {k:3d}  claim {claim[s].min():7.1f}  ready {ready[s].min():7.1f}..{ready[s].max():7.1f}  "
          f"full {full[s].min():7.1f}..{full[s].max():7.1f}  pub {pub[s].max():7.1f}  end {end[s].max():7.1f}  "
          f"item {np.mean(end[s] - full[s]):5.2f} (gemm {np.mean(gemm[s] - full[s]):5.2f})")

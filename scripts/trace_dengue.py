"""Phase timing of the small-S traversal (trace build, PHYLOGRAD_LIB=...trace.so).

clock64 stamps of CTA 0 (producer lane 0, consumer warp 0 lane 0) per step:
producer 0 loop top, 1 after empty wait, 2 after issue; consumer post 3 op
decoded, 4 children ready, 5 next op waited, 6 rescaled, 7 u ready; consumer
pre 3 op decoded, 4 q + children ready, 5 next op waited, 6 q_c computed,
7 gradient terms + pushes done.
"""
import ctypes, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_04390_b200 as pg
import phylo_synth as ps
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 1
kw = {"C": int(os.environ["TRACE_C"])} if os.environ.get("TRACE_C") else {}
pb = ps.make_config(cfg, **kw)
inst = pg.from_problem(pb)
out = torch.zeros(2 * pb.n_tips - 1, dtype=torch.float64, device="cuda")
for _ in range(3):
    inst.compute_device(out)
inst.stream.synchronize()
N = pb.n_tips
n = 16 * 2 * N
buf = (ctypes.c_longlong * n)()
pg._lib.pg_trace_copy.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int]
pg._lib.pg_trace_copy(inst._h, buf, n)
tr = np.array(buf, dtype=np.int64).reshape(2 * N, 16)
steps = N - 1
for name, blk in (("post", tr[:steps]), ("pre", tr[steps:2 * steps])):
    print(f"== {name} ({steps} steps)")
    def stats(label, a, b):
        d = (blk[1:-1, b] - blk[1:-1, a]).astype(float)
        print(f"  {label:28s} mean {d.mean():8.1f}  median {np.median(d):8.1f}  p90 {np.percentile(d, 90):8.1f}")
    stats("3->4", 3, 4); stats("4->5", 4, 5); stats("5->6", 5, 6); stats("6->7", 6, 7)
    if name == "pre":
        stats("7->8 forwarding", 7, 8)
        f = blk[1:-1]; m = f[:, 9] > 0
        d = (f[m, 9] - f[m, 8]).astype(float)
        print(f"  {'flush (8->9, flush steps)':28s} mean {d.mean():8.1f}  median {np.median(d):8.1f}  n {m.sum()}")
        nx = blk[2:, 3]; cur = blk[1:-1]
        d = (nx - np.where(cur[:, 9] > 0, cur[:, 9], cur[:, 8])).astype(float)
        print(f"  {'loop back (->next 3)':28s} mean {d.mean():8.1f}  median {np.median(d):8.1f}")
    d = np.diff(blk[:, 3]).astype(float)
    print(f"  {'consumer step (3->3)':28s} mean {d.mean():8.1f}  median {np.median(d):8.1f}")
    stats("producer empty wait (0->1)", 0, 1); stats("producer issue (1->2)", 1, 2)
    if (blk[1:-1, 10] > 0).all():
        stats("  prod: wait -> op read (1->10)", 1, 10); stats("  prod: small copies (10->11)", 10, 11)
        stats("  prod: arrive+sync (11->12)", 11, 12); stats("  prod: bulk (12->2)", 12, 2)
    d = np.diff(blk[:, 0]).astype(float)
    print(f"  {'producer step (0->0)':28s} mean {d.mean():8.1f}  median {np.median(d):8.1f}")
    lag = (blk[:, 3] - blk[:, 2]).astype(float)
    print(f"  consumer start - producer issue: mean {lag.mean():.0f} median {np.median(lag):.0f}")
print("post total cycles", tr[steps - 1, 3] - tr[0, 3], " pre total", tr[2 * steps - 1, 3] - tr[steps, 3])

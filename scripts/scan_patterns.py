"""Traversal time vs pattern count (dengue tree): is the kernel latency-bound?

If the traversal time stays flat as the number of resident warps per SM
changes, the per-tile sequential chain (2(N-1) steps) sets the time."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2303_04390_b200 as pg
import phylo_synth as ps
for C in [int(x) for x in (sys.argv[1:] or ["1184", "2368", "4736", "7104", "10000"])]:
    pb = ps.config1_dengue(C=C)
    inst = pg.from_problem(pb)
    inst.set_kernel_timing(True)
    out = torch.zeros(2 * pb.n_tips - 1, dtype=torch.float64, device="cuda")
    ts = []
    for i in range(30):
        inst.compute_device(out)
        inst.stream.synchronize()
        if i >= 5:
            ts.append(inst.kernel_times()["traverse"])
    info = inst.plan_info()
    print(f"C={C:6d} grid={info['grid']} block={info['block']} smem={info['smem_bytes']} traverse ms median {np.median(ts):.4f}", flush=True)
    inst.close()

"""Device-resident HMC leapfrog throughput: leapfrog
steps per second through pg_hmc_leapfrog (one full gradient evaluation per
step, theta = log b, no host synchronisation inside a trajectory).
usage: python scripts/hmc_bench.py [config ...]   -> one JSON line per config"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2303_04390_b200 as pg  # noqa: E402
import phylo_synth as ps  # noqa: E402

for cfg in [int(c) for c in (sys.argv[1:] or ["1", "3"])]:
    pb = ps.make_config(cfg)
    inst = pg.from_problem(pb)
    B = 2 * pb.n_tips - 2
    dev = torch.device("cuda", 0)
    th = torch.tensor(np.log(np.maximum(pb.branch_lengths, 1e-6)), device=dev)
    th0 = th.clone()
    rng = np.random.default_rng(cfg)
    p = torch.tensor(rng.standard_normal(B), device=dev)
    out = torch.empty(B + 1, dtype=torch.float64, device=dev)
    eps, L, traj = 1e-4, 50, 10
    with torch.cuda.stream(inst.stream):
        inst.hmc_leapfrog(th, p, eps, L, out)                 # warm-up (graph capture)
        inst.stream.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(inst.stream)
        for _ in range(traj):
            th.copy_(th0)
            inst.hmc_leapfrog(th, p, eps, L, out)
        e1.record(inst.stream)
    inst.stream.synchronize()
    ms = e0.elapsed_time(e1)
    evals = traj * (L + 1)
    print(json.dumps({"metric": "HMC leapfrog steps/s (device-resident, theta = log b)",
                      "workload": pb.name, "value": round(traj * L / (ms * 1e-3), 1),
                      "gradient_evals_per_s": round(evals / (ms * 1e-3), 1), "trajectory_length": L,
                      "ms_per_trajectory": round(ms / traj, 4), "status": inst.check_status()}))
    inst.close()
